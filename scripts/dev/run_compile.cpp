// Dev harness (CPU, no GPU): plan a QFT / random circuit, encode its passes
// and NVRTC-compile the co-scheduled run kernels of its L2 groups (f2) --
// catches generator errors before spending GPU time.
//   g++ -std=c++17 -O1 -I include -I /usr/local/cuda/include scripts/dev/run_compile.cpp \
//       -L paper_2604_12256_b200 -lqs -Wl,-rpath,$PWD/paper_2604_12256_b200 -o /tmp/run_compile
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "../../paper_2604_12256_b200/csrc/planner.hpp"

namespace qs {
bool jit_prepare_run(const std::vector<const unsigned char*>& blobs, int sb, int device, JitPrepared& out,
                     bool compile_only);
}
using namespace qs;

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 24;
  const int W = argc > 2 ? atoi(argv[2]) : 18;
  std::vector<qs_gate_t> g;
  for (int i = n - 1; i >= 0; i--) {  // QFT
    qs_gate_t h = {};
    h.kind = QS_H;
    h.n_targets = 1;
    h.targets[0] = i;
    g.push_back(h);
    for (int j = i - 1; j >= 0; j--) {
      qs_gate_t c = {};
      c.kind = QS_CP;
      c.n_targets = 1;
      c.targets[0] = j;
      c.n_controls = 1;
      c.controls[0] = i;
      c.params[0] = M_PI / (double)(1ull << (i - j));
      g.push_back(c);
    }
  }
  std::vector<IrGate> ir;
  std::string err;
  if (ingest(n, g.data(), g.size(), ir, err)) { fprintf(stderr, "ingest: %s\n", err.c_str()); return 1; }
  PlanInput in;
  in.n = n;
  qs_default_config(&in.cfg);
  in.cfg.l2_block_qubits = W;
  in.product_state = true;
  in.basis = 12345 % (1ull << n);
  for (int q = 0; q < n; q++) in.map.push_back(q);
  Plan plan;
  if (make_plan(in, ir, plan, err)) { fprintf(stderr, "plan: %s\n", err.c_str()); return 1; }
  std::vector<std::vector<unsigned char>> bl;
  std::vector<const unsigned char*> run;
  int wm = 12;
  for (const Step& st : plan.steps) {
    if (st.type != Step::PASS || st.pass.l2_grp < 0) continue;
    bl.emplace_back();
    if (encode_pass(st.pass, 0, bl.back(), err)) { fprintf(stderr, "encode: %s\n", err.c_str()); return 1; }
    for (int c : st.pass.cpos) wm = std::max(wm, c + 1);
    for (int c : st.pass.opos) wm = std::max(wm, c + 1);
  }
  for (auto& b : bl) run.push_back(b.data());
  printf("run of %zu passes, sb %d\n", run.size(), wm - 12);
  JitPrepared jp;
  const bool ok = jit_prepare_run(run, wm - 12, 0, jp, true);
  printf("ok %d threads %d smem %zu err %s\n", ok, jp.threads, jp.smem, jp.err.substr(0, 3000).c_str());
  return ok ? 0 : 1;
}
