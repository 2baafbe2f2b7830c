// planner.hpp -- host-side optimiser of libqs (Alg. 4 "Swarm optimization",
// PAPER.md L391-416): ingest/validation, diagonal detector (Alg. 8), merge
// booster (Alg. 6/7), rank-level staging with global<->local swaps,
// machine-level cache blocking (Alg. 2) with a virtual qubit map, and
// cost-based fusion.  The output is a Plan: a list of device steps.
#pragma once
#include <complex>
#include <string>
#include <vector>

#include "../../include/qs.h"
#include "qs_internal.hpp"

namespace qs {

typedef std::complex<double> cd;

struct Mono {
  u64 mask;   // qubit mask (logical or physical depending on context)
  u64 coeff;  // angle in turns * 2^64 (mod 2^64)
};

// Intermediate representation of one (possibly fused) gate over LOGICAL
// qubits.
struct IrGate {
  enum Type { DENSE, DIAG, RELABEL } type = DENSE;
  std::vector<int> targets;   // DENSE: matrix bit i <-> targets[i]; RELABEL: {a,b}
  std::vector<int> controls;  // DENSE only (DIAG folds controls into monomials)
  std::vector<cd> mat;        // DENSE: 2^t x 2^t row-major
  std::vector<Mono> mono;     // DIAG: phase polynomial exp(2 pi i sum c_S [x_S])
  u64 support = 0;            // logical mask of every qubit the gate reads
  int kind = -1;              // qs_kind of the source gate (-1: fused)
  int n_src = 1;              // source gates merged into this one
  bool is_h = false, is_x = false;
};

// Physical-position op inside a pass (before register encoding).
struct POp {
  enum Type { DENSE, DIAG } type = DENSE;
  std::vector<int> tpos;      // DENSE: physical target positions
  u64 cmask = 0;              // DENSE: physical control mask
  std::vector<cd> mat;
  std::vector<Mono> mono;     // DIAG: physical masks
  bool is_h = false, is_x = false;
  int n_src = 1;
};

struct PassPlan {
  int buf = 0;                // 0 main shard, >0 sub-state id
  int nl = 0;                 // local qubits of the buffer
  int n_global = 0;           // global (rank) bits of the buffer
  int kernel = KK_CHUNK;
  std::vector<int> cpos;      // chunk positions (ascending) for K1/K2/K3
  std::vector<int> opos;      // output positions (relabel)
  std::vector<POp> ops;
  int src_mode = 0;           // 0 load, 1 expand (booster), 2 basis state
  std::vector<int> exp_bufs, exp_lo, exp_len;
  uint64_t basis = 0;
  // the following SWAP's exchange is fused into this pass's
  // stores -- output indices whose top x_j local bits are s go straight to the
  // receive buffer of the rank the swap sends piece s to (0: not fused)
  int x_j = 0;
  std::vector<int> x_pos;     // the swap's local positions (exported bit i)
  // push/pull split of a fused swap (NVLink time spread over two passes):
  // the exporting pass pushes only the chunks whose bit `x_split` is 0 (the
  // rest stay in place, -1: push all); the pass after the swap pulls those
  // from the source ranks' buffers (pull_j > 0: piece = its bits at
  // pull_pos, pull_z the split bit)
  int x_split = -1;
  int pull_j = 0, pull_z = -1;
  std::vector<int> pull_pos;
  // two-level blocking: id of the run of consecutive passes
  // executed wave by wave over L2-sized blocks (-1: none)
  int l2_grp = -1;
  // filled by encode_pass
  std::vector<std::vector<int>> phase_regs;  // per phase: chunk bits held in registers
  std::vector<int> op_phase;
};

struct Step {
  enum Type { INIT_BASIS, PASS, SWAP, EXPAND, SUB_INIT, SUB_MERGE, PERMUTE } type;
  // PERMUTE: exchange local bit positions gpos[i] <-> lpos[i] (full pass)
  PassPlan pass;              // PASS
  int buf = 0;                // SUB_INIT / SUB_MERGE destination, EXPAND uses subs
  uint64_t basis = 0;         // INIT_BASIS / SUB_INIT: basis index (physical)
  int j = 0;                  // SWAP: number of exchanged qubits
  std::vector<int> gpos;      // SWAP: global positions exchanged with
  std::vector<int> lpos;      //       local positions (top j)
  bool fusable = false;       // SWAP: the preceding pass may do the exchange
  int src_a = 0, src_b = 0;   // SUB_MERGE: dst = A (low) (x) B (high)
  std::vector<int> exp_bufs;  // EXPAND (and fused expand): sub-state ids
  std::vector<int> exp_lo, exp_len;
};

struct SubBuf {
  int nq = 0;                 // qubits
  int lo = 0;                 // lowest logical qubit of the contiguous group
};

struct PlanStats {
  uint64_t n_gates_in = 0, n_passes = 0, n_chunk = 0, n_dense = 0, n_diag = 0,
           n_small = 0, n_expand = 0, n_swaps = 0, n_sub_gates = 0,
           n_fused_diag = 0, paper_updates = 0, naive_updates = 0,
           bytes_hbm = 0, bytes_nvlink = 0, n_fusable_swaps = 0,
           n_l2_groups = 0, bytes_hbm_l2 = 0;  // f2: runs, HBM bytes with them
  std::vector<std::vector<int>> booster_rounds;  // gate counts per round/group
  bool wo_budget_hit = false;   // the FP64 budget closed the write-only pass
};

struct Plan {
  int n = 0, n_global = 0, nl = 0;
  std::vector<Step> steps;
  std::vector<SubBuf> subs;       // sub-state buffers (index 1..)
  std::vector<int> map_in;        // logical -> physical before the plan
  std::vector<int> map_out;       // logical -> physical after the plan
  PlanStats stats;
};

struct PlanInput {
  int n = 0;
  int n_global = 0;               // log2(#ranks)
  qs_config_t cfg;
  bool product_state = false;
  uint64_t basis = 0;             // valid if product_state
  std::vector<int> map;           // current logical -> physical map
};

// Validate and convert ABI gates.  Returns QS_OK or QS_EINVAL with `err`.
int ingest(int n, const qs_gate_t* gates, size_t n_gates,
           std::vector<IrGate>& out, std::string& err);

// Corrected Alg. 8 (readings c4-c7).
std::vector<IrGate> diagonal_detector(const std::vector<IrGate>& in, int n, int diag_cap,
                                      uint64_t* n_fused);

// Alg. 6.
void divider(int n, int div_size, std::vector<int>& que);

// Full optimiser: Plan from validated IR.
int make_plan(const PlanInput& in, const std::vector<IrGate>& gates, Plan& plan,
              std::string& err);

// Encode a pass into a device descriptor blob (KPass header + arrays).
// `rank` selects rank_base; sub-state pointers are patched by the executor.
int encode_pass(const PassPlan& p, int rank, std::vector<unsigned char>& blob,
                std::string& err);

std::string plan_to_json(const Plan& plan, bool detail);

// Product-side gate table (reading c3).
bool gate_matrix(int kind, const double* params, std::vector<cd>& m, int* t_out);
bool kind_is_diagonal(int kind);

// Angle (radians) -> turns * 2^64 mod 2^64.
u64 turns_of(long double radians);

}  // namespace qs
