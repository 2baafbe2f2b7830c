// planner.cpp -- host optimiser: Alg. 4 "Swarm optimization" (PAPER.md
// L391-416) re-designed for B200.
//
//   Booster            Alg. 6/7 with readings c8-c11.
//   DiagonalDetector   Alg. 8 with corrections c4-c7.
//   GBSA rank level stages whose non-diagonal targets are local;
//                      global<->local swaps between stages.
//   GBSA machine level cache blocking into chunk passes: every
//                      non-diagonal target of a pass lies in the pass's 12
//                      chunk positions; diagonals and controls need no
//                      locality (evaluated from index bits, incl. rank bits).
//   GBSA fuse=1 cost-based fusion of adjacent dense ops
//                      (FP64-FMA cost model, reading c15).
//   Virtual qubit map  logical -> physical; uncontrolled SWAPs are relabels
//                      (Eq. 4).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <map>
#include <sstream>
#include <unordered_set>

#include "planner.hpp"

namespace qs {

static inline int popc(u64 x) { return __builtin_popcountll(x); }

// ------------------------------------------------------------ Alg. 6
void divider(int n, int div_size, std::vector<int>& que) {
  if (n <= div_size) {
    que.push_back(n);
    return;
  }
  divider(n >> 1, div_size, que);
  n = (n & 1) ? n + 1 : n;
  divider(n >> 1, div_size, que);
}

// ------------------------------------------------------------ helpers
static void merge_mono(std::vector<Mono>& m) {
  std::sort(m.begin(), m.end(), [](const Mono& a, const Mono& b) { return a.mask < b.mask; });
  std::vector<Mono> out;
  for (const Mono& x : m) {
    if (!out.empty() && out.back().mask == x.mask) out.back().coeff += x.coeff;
    else out.push_back(x);
  }
  m.clear();
  for (const Mono& x : out)
    if (x.coeff != 0) m.push_back(x);
}

static u64 map_mask(u64 logical_mask, const std::vector<int>& map) {
  u64 r = 0;
  while (logical_mask) {
    int q = __builtin_ctzll(logical_mask);
    logical_mask &= logical_mask - 1;
    r |= 1ull << map[q];
  }
  return r;
}

// Matrix product C = A * B for gates given over target lists; result over
// `uni` (ascending union).  Matrix bit i <-> targets[i].
static std::vector<cd> embed(const std::vector<cd>& m, const std::vector<int>& tg,
                             const std::vector<int>& uni) {
  const int t = (int)tg.size(), u = (int)uni.size();
  const int D = 1 << u, d = 1 << t;
  std::vector<int> idx(t);
  for (int i = 0; i < t; i++)
    idx[i] = (int)(std::find(uni.begin(), uni.end(), tg[i]) - uni.begin());
  std::vector<cd> out((size_t)D * D, 0);
  for (int r = 0; r < D; r++)
    for (int c = 0; c < D; c++) {
      // identity on the non-target bits
      int rest_r = r, rest_c = c, sr = 0, sc = 0;
      for (int i = 0; i < t; i++) {
        sr |= ((r >> idx[i]) & 1) << i;
        sc |= ((c >> idx[i]) & 1) << i;
        rest_r &= ~(1 << idx[i]);
        rest_c &= ~(1 << idx[i]);
      }
      if (rest_r != rest_c) continue;
      out[(size_t)r * D + c] = m[(size_t)sr * d + sc];
    }
  return out;
}

static std::vector<cd> matmul(const std::vector<cd>& A, const std::vector<cd>& B, int D) {
  std::vector<cd> C((size_t)D * D, 0);
  for (int i = 0; i < D; i++)
    for (int k = 0; k < D; k++) {
      cd a = A[(size_t)i * D + k];
      if (a == cd(0, 0)) continue;
      for (int j = 0; j < D; j++) C[(size_t)i * D + j] += a * B[(size_t)k * D + j];
    }
  return C;
}

// ------------------------------------------------------------ Alg. 8
// Corrected diagonal detector (readings c4-c7):
//  c4  dependencies use the support (targets U controls);
//  c5  a non-diagonal is deferred (uList, stopTable) when its support meets
//      depSet OR a stopTable-marked qubit, else bypassed ahead of the fusion;
//  c6  a lone diagonal is kept (the printed Alg. 8 drops it);
//  c7  a diagonal touching a stopTable-marked qubit stops the scan; so does
//      exceeding the D cap on the fused support (diag_cap > 0).
std::vector<IrGate> diagonal_detector(const std::vector<IrGate>& in, int n, int diag_cap,
                                      uint64_t* n_fused) {
  (void)n;
  std::vector<IrGate> res;           // resList
  res.reserve(in.size());
  size_t it = 0;
  while (it < in.size()) {
    if (in[it].type != IrGate::DIAG) {
      res.push_back(in[it]);
      ++it;
      continue;
    }
    IrGate fused = in[it];             // diagList (merged as we go)
    std::vector<IrGate> ulist;         // uList
    u64 stop = 0;                      // stopTable
    u64 dep = in[it].support;          // depSet
    int diag_size = 1;
    size_t f = it + 1;
    for (; f < in.size(); ++f) {
      const IrGate& g = in[f];
      const u64 s = g.support;
      if (g.type != IrGate::DIAG) {
        if (s & (dep | stop)) {        // c5
          stop |= s;
          ulist.push_back(g);
        } else {
          res.push_back(g);
        }
      } else {
        if (s & stop) break;           // checkStop (c7)
        if (diag_cap > 0 && popc(dep | s) > diag_cap) break;
        dep |= s;
        fused.mono.insert(fused.mono.end(), g.mono.begin(), g.mono.end());
        fused.support |= s;
        fused.n_src += g.n_src;
        ++diag_size;
      }
    }
    if (diag_size > 1) {               // doDiagonalFusion
      merge_mono(fused.mono);
      fused.kind = -1;
      if (n_fused) ++*n_fused;
    }
    res.push_back(std::move(fused));   // c6: singletons are kept
    for (auto& g : ulist) res.push_back(std::move(g));
    it = f;
  }
  return res;
}

// ------------------------------------------------------------ scheduling
struct Sched {
  Plan* plan;
  const qs_config_t* cfg;
  int src_mode = 0;                 // pending source of the next main pass: 0 none,
                                    // 1 expand (booster), 2 basis
  std::vector<int> exp_bufs, exp_lo, exp_len;
  uint64_t basis_phys = 0;
  double wo_budget = 40.0;          // FP64/amp budget of the write-only first pass (c15)
};

static double dense_cost(int k) { return 4.0 * (1 << k); }  // FP64 FMA per amp

// FP64 instructions per output amplitude of a dense matrix as the
// specialised kernels execute it: 0 per zero entry, 2 per real or purely
// imaginary entry, 4 per complex entry (averaged over rows).
static double mat_cost(const std::vector<cd>& m) {
  size_t D = 1;
  while (D * D < m.size()) D++;
  double c = 0;
  for (const cd& z : m) c += (z == cd(0, 0)) ? 0.0 : (z.imag() == 0.0 || z.real() == 0.0) ? 2.0 : 4.0;
  return c / (double)D;
}

// A "unit-scaled" matrix: every nonzero entry is exactly +-lam or +-i lam
// for one complex lam (the first nonzero entry), e.g. SX = ((1+i)/2) [[1,-i],
// [-i,1]], SY = ((1+i)/2) [[1,-1],[1,1]], CZ-free Clifford products.  For an
// UNCONTROLLED op lam commutes with the whole pass (a global scalar of the
// shard), so the kernels apply the +-1/+-i matrix with additions only and
// fold lam into the pass scale (encode_pass).  unit_out (optional) receives
// the +-1/+-i/0 matrix (exact: built from the comparison, not a division).
static bool unit_scaled(const std::vector<cd>& m, cd* lam_out, std::vector<cd>* unit_out) {
  cd lam(0, 0);
  for (const cd& z : m)
    if (z != cd(0, 0)) {
      lam = z;
      break;
    }
  if (lam == cd(0, 0)) return false;
  const cd ilam(-lam.imag(), lam.real());  // i * lam, exact
  if (unit_out) unit_out->assign(m.size(), cd(0, 0));
  for (size_t k = 0; k < m.size(); k++) {
    const cd z = m[k];
    cd u;
    if (z == cd(0, 0)) u = cd(0, 0);
    else if (z == lam) u = cd(1, 0);
    else if (z == -lam) u = cd(-1, 0);
    else if (z == ilam) u = cd(0, 1);
    else if (z == -ilam) u = cd(0, -1);
    else return false;
    if (unit_out) (*unit_out)[k] = u;
  }
  if (lam_out) *lam_out = lam;
  return true;
}

// An uncontrolled one-qubit matrix [[a, b], [c, d]] is applied as
// lam [[a, b], [c, d]] / lam with lam = the larger of a, b (|lam| >= 1/sqrt2
// for a unitary, so every ratio has magnitude <= 1): entries equal to
// +-lam, +-i lam become exact units (built from the comparison, like
// unit_scaled) and lam joins the pass scale.  RX = cos [[1, -i tan],
// [-i tan, 1]] then costs 2 FP64 per output amplitude instead of 4 (the
// kernels bake units into additions, dense()), RY likewise.  false: no
// entry became a unit (nothing to gain).  QS_NO_ROWSCALE: A/B knob.
static bool row_scale_1q(std::vector<cd>& m, cd* lam_out) {
  static const bool off = getenv("QS_NO_ROWSCALE") != nullptr;
  if (off || m.size() != 4) return false;
  const cd lam = std::abs(m[0]) >= std::abs(m[1]) ? m[0] : m[1];
  if (lam == cd(0, 0)) return false;
  const cd ilam(-lam.imag(), lam.real());
  std::vector<cd> r(4);
  int units = 0;
  for (int k = 0; k < 4; k++) {
    const cd z = m[k];
    if (z == cd(0, 0)) r[k] = cd(0, 0);
    else if (z == lam) r[k] = cd(1, 0), units++;
    else if (z == -lam) r[k] = cd(-1, 0), units++;
    else if (z == ilam) r[k] = cd(0, 1), units++;
    else if (z == -ilam) r[k] = cd(0, -1), units++;
    else r[k] = z / lam;
  }
  // row 0 holds lam itself; the gain needs a unit in row 1 too (one-row
  // savings are offset by the complex ratios that appear)
  auto unit = [](const cd& z) {
    return (z.imag() == 0.0 && std::abs(z.real()) == 1.0) || (z.real() == 0.0 && std::abs(z.imag()) == 1.0);
  };
  if (units < 2 || !(unit(r[2]) || unit(r[3]))) return false;
  m.swap(r);
  *lam_out = lam;
  return true;
}

// FP64 instructions per output amplitude of an UNCONTROLLED op: a
// unit-scaled matrix needs only complex additions (nnz - 1 per row).
static double mat_cost_unc(const std::vector<cd>& m) {
  // (row-scaled one-qubit gates, r9b, are priced at their full-matrix cost:
  // pricing them at 2 FP64/amp lets the write-only pass take more gates,
  // which removed a pass of QAOA-32 on 4 GPUs but made one of its fused-swap
  // passes run at half the NVLink rate, 133 -> 152 ms)
  if (!unit_scaled(m, nullptr, nullptr)) return mat_cost(m);
  size_t D = 1;
  while (D * D < m.size()) D++;
  size_t nnz = 0;
  for (const cd& z : m) nnz += z != cd(0, 0);
  return 2.0 * ((double)nnz / (double)D - 1.0);
}
static double op_cost(const std::vector<cd>& m, bool is_h) { return is_h ? 2.0 : mat_cost(m); }
static double op_cost_unc(const std::vector<cd>& m, bool is_h) { return is_h ? 2.0 : mat_cost_unc(m); }

// Emit the pending source as a standalone step (before a swap / small pass).
static void flush_source(Sched& S) {
  if (S.src_mode == 1) {
    Step st;
    st.type = Step::EXPAND;
    st.buf = 0;
    st.exp_bufs = S.exp_bufs;
    st.exp_lo = S.exp_lo;
    st.exp_len = S.exp_len;
    S.plan->steps.push_back(st);
    S.plan->stats.n_expand++;
    S.plan->stats.bytes_hbm += (16ull << S.plan->nl);
  } else if (S.src_mode == 2) {
    Step st;
    st.type = Step::INIT_BASIS;
    st.buf = 0;
    st.basis = S.basis_phys;
    S.plan->steps.push_back(st);
    S.plan->stats.bytes_hbm += (16ull << S.plan->nl);
  }
  S.src_mode = 0;
}

static POp dense_pop(const IrGate& g, const std::vector<int>& map) {
  POp op;
  op.type = POp::DENSE;
  for (int q : g.targets) op.tpos.push_back(map[q]);
  u64 cm = 0;
  for (int q : g.controls) cm |= 1ull << map[q];
  op.cmask = cm;
  op.mat = g.mat;
  op.is_h = g.is_h;
  op.is_x = g.is_x;
  op.n_src = g.n_src;
  return op;
}

static void add_diag_op(std::vector<POp>& ops, const IrGate& g, const std::vector<int>& map) {
  if (ops.empty() || ops.back().type != POp::DIAG) {
    POp op;
    op.type = POp::DIAG;
    op.n_src = 0;
    ops.push_back(op);
  }
  POp& d = ops.back();
  for (const Mono& m : g.mono) d.mono.push_back({map_mask(m.mask, map), m.coeff});
  d.n_src += g.n_src;
}

// GBSA fuse=1: fuse adjacent uncontrolled dense ops when the fused
// gate's FP64 cost does not exceed the sum of the parts (reading c15).  First
// the longest run of such ops whose targets fit F (<= 4) qubits is tried as
// one unitary (many small gates on few qubits: e.g. 12 two-qubit gates on 4
// qubits cost 192 FP64/amp, one 16x16 costs 64); a 4-qubit result runs as a
// shared-memory op (two more chunk exchanges), so it must at least halve the
// cost.  Otherwise pairs are fused greedily up to 3 qubits (register ops).
static std::vector<cd> fuse_pair(const POp& a, const POp& b, std::vector<int>& uni) {
  uni = a.tpos;
  for (int p : b.tpos)
    if (std::find(uni.begin(), uni.end(), p) == uni.end()) uni.push_back(p);
  std::sort(uni.begin(), uni.end());
  std::vector<cd> A = embed(a.mat, a.tpos, uni);
  std::vector<cd> B = embed(b.mat, b.tpos, uni);
  return matmul(B, A, 1 << (int)uni.size());  // later gate applied after
}

static void fuse_ops(std::vector<POp>& ops, int fuse_cap) {
  if (fuse_cap < 2) return;
  // Fusion must make the op strictly cheaper: at equal FP64 cost (e.g. RX x
  // RX: 8 = 4 + 4 per amplitude) the fused 4x4 needs 16 matrix constants
  // instead of 2 x 4, which the compiler keeps in registers (spills in
  // QAOA's write-only pass).  QS_FUSE_TIES=1: the round-1 rule (ties fuse).
  static const bool ties = getenv("QS_FUSE_TIES") != nullptr;
  auto pays = [](double fused, double parts) { return ties ? fused <= parts : fused < parts; };
  const int cap = std::min(fuse_cap, kRegBits);          // run fusion
  const int pcap = std::min(fuse_cap, kRegBits - 1);     // pairwise (register ops)
  auto fusable = [](const POp& o) { return o.type == POp::DENSE && o.cmask == 0 && (int)o.tpos.size() < kRegBits; };
  std::vector<POp> out;
  for (size_t i = 0; i < ops.size();) {
    if (fusable(ops[i])) {
      // longest run from i whose union fits `cap` qubits
      size_t j = i + 1;
      u64 um = 0;
      for (int p : ops[i].tpos) um |= 1ull << p;
      double parts = op_cost_unc(ops[i].mat, ops[i].is_h);
      while (j < ops.size() && fusable(ops[j])) {
        u64 nm = um;
        for (int p : ops[j].tpos) nm |= 1ull << p;
        if (popc(nm) > cap) break;
        um = nm;
        parts += op_cost_unc(ops[j].mat, ops[j].is_h);
        j++;
      }
      if (j - i >= 3) {
        POp f = ops[i];
        for (size_t q = i + 1; q < j; q++) {
          std::vector<int> uni;
          f.mat = fuse_pair(f, ops[q], uni);
          f.tpos = uni;
          f.n_src += ops[q].n_src;
        }
        if (pays(mat_cost_unc(f.mat) * (f.tpos.size() >= (size_t)kRegBits ? 2.0 : 1.0), parts)) {
          f.is_h = f.is_x = false;
          out.push_back(std::move(f));
          i = j;
          continue;
        }
      }
    }
    POp& op = ops[i];
    if (!out.empty() && fusable(op) && fusable(out.back())) {
      POp& prev = out.back();
      u64 um = 0;
      for (int p : prev.tpos) um |= 1ull << p;
      for (int p : op.tpos) um |= 1ull << p;
      const int ku = popc(um);
      const double parts = op_cost_unc(prev.mat, prev.is_h) + op_cost_unc(op.mat, op.is_h);
      if (ku <= pcap && dense_cost(ku) / 2 <= parts) {
        std::vector<int> uni;
        std::vector<cd> F = fuse_pair(prev, op, uni);
        if (pays(mat_cost_unc(F), parts)) {
          prev.mat = F;
          prev.tpos = uni;
          prev.is_h = prev.is_x = false;
          prev.n_src += op.n_src;
          i++;
          continue;
        }
      }
    }
    out.push_back(std::move(op));
    i++;
  }
  ops.swap(out);
}

// Inside a pass, a phase monomial commutes with every dense op whose targets
// it does not touch (controls do not matter: a diagonal on the control commutes
// with the control projector).  Move each monomial forward into the furthest
// later diagonal group it can reach, so groups merge and fewer per-thread
// sincos are needed (the diagonal detector's commutation, Alg. 8, applied at
// monomial granularity inside a pass).
static void sink_monomials(std::vector<POp>& ops) {
  for (size_t i = 0; i < ops.size(); i++) {
    if (ops[i].type != POp::DIAG) continue;
    std::vector<Mono> keep;
    for (const Mono& m : ops[i].mono) {
      size_t dest = i;
      for (size_t j = i + 1; j < ops.size(); j++) {
        if (ops[j].type == POp::DIAG) {
          dest = j;
          continue;
        }
        u64 tm = 0;
        for (int pos : ops[j].tpos) tm |= 1ull << pos;
        if (m.mask & tm) break;
      }
      if (dest == i) keep.push_back(m);
      else ops[dest].mono.push_back(m);
    }
    ops[i].mono.swap(keep);
  }
  std::vector<POp> out;
  for (POp& op : ops) {
    if (op.type == POp::DIAG) {
      merge_mono(op.mono);
      if (op.mono.empty()) continue;
    }
    out.push_back(std::move(op));
  }
  ops.swap(out);
}

// Thread-bit order of a register layout: tid bits 0..2 take the lowest
// non-register chunk bits of distinct residues mod 3 (bank-conflict-free
// swizzled exchange), then the rest ascending.
static std::vector<int> phase_thread_order(const std::vector<int>& regs, int m) {
  std::vector<int> rest;
  for (int c = 0; c < m; c++)
    if (std::find(regs.begin(), regs.end(), c) == regs.end()) rest.push_back(c);
  std::vector<int> order;
  for (int res = 0; res < 3; res++)
    for (int c : rest)
      if (c % 3 == res && std::find(order.begin(), order.end(), c) == order.end()) {
        order.push_back(c);
        break;
      }
  std::sort(order.begin(), order.end());
  for (int c : rest)
    if (std::find(order.begin(), order.end(), c) == order.end()) order.push_back(c);
  return order;
}

// Assign register layouts ("phases") to the dense ops of a chunk pass.
static void assign_phases(PassPlan& p) {
  const int m = (int)p.cpos.size();
  auto cbit = [&](int pos) {
    return (int)(std::find(p.cpos.begin(), p.cpos.end(), pos) - p.cpos.begin());
  };
  p.phase_regs.clear();
  p.op_phase.assign(p.ops.size(), 0);
  std::vector<int> cur;
  int ph = 0;
  for (size_t i = 0; i < p.ops.size(); i++) {
    const POp& op = p.ops[i];
    if (op.type == POp::DENSE && (int)op.tpos.size() >= kRegBits) {
      // wide op (4-6 targets): applied to the chunk in shared memory at the
      // exchange INTO a new layout, so it is the first op of that layout
      p.phase_regs.push_back(cur);
      ++ph;
      cur.clear();
    } else if (op.type == POp::DENSE) {
      std::vector<int> need;
      for (int pos : op.tpos) need.push_back(cbit(pos));
      std::vector<int> uni = cur;
      for (int c : need)
        if (std::find(uni.begin(), uni.end(), c) == uni.end()) uni.push_back(c);
      if ((int)uni.size() > kRegBits) {
        p.phase_regs.push_back(cur);
        ++ph;
        cur = need;
      } else {
        cur = uni;
      }
    }
    p.op_phase[i] = ph;
  }
  p.phase_regs.push_back(cur);
  // fill every layout to kRegBits register bits, preferring high chunk bits
  for (auto& regs : p.phase_regs) {
    for (int c = m - 1; c >= 0 && (int)regs.size() < kRegBits; c--)
      if (std::find(regs.begin(), regs.end(), c) == regs.end()) regs.push_back(c);
    std::sort(regs.begin(), regs.end());
  }
  if (p.kernel != KK_DIAG) p.kernel = (p.phase_regs.size() > 1) ? KK_CHUNK : KK_DENSE;
}

static void finalize_chunk_pass(Sched& S, PassPlan& p, u64 need_pos, int nl,
                                std::vector<int>* map, const std::vector<IrGate>* upcoming) {
  const int m = kChunkBits;
  // chunk positions: the needed ones, filled with the lowest free positions
  u64 c = need_pos;
  for (int pos = 0; pos < nl && popc(c) < m; pos++) c |= 1ull << pos;
  p.cpos.clear();
  for (int pos = 0; pos < nl; pos++)
    if (c >> pos & 1) p.cpos.push_back(pos);
  p.opos = p.cpos;
  for (POp& op : p.ops)
    if (op.type == POp::DIAG) merge_mono(op.mono);
  if (S.cfg->flags & QS_OPT_DIAG) {
    // keep the sunk order only if it lowers the estimated per-thread sincos
    // count: 1 + (dense-target qubits a group touches) per diagonal group
    auto est = [](const std::vector<POp>& ops) {
      u64 T = 0;
      for (const POp& op : ops)
        if (op.type == POp::DENSE)
          for (int pos : op.tpos) T |= 1ull << pos;
      int c = 0;
      for (const POp& op : ops)
        if (op.type == POp::DIAG) {
          u64 s = 0;
          for (const Mono& m : op.mono) s |= m.mask;
          c += 1 + popc(s & T);
        }
      return c;
    };
    std::vector<POp> sunk = p.ops;
    sink_monomials(sunk);
    if (est(sunk) < est(p.ops)) p.ops.swap(sunk);
  }
  bool all_diag = true;
  for (const POp& op : p.ops)
    if (op.type != POp::DIAG) all_diag = false;
  p.kernel = all_diag ? KK_DIAG : KK_CHUNK;
  fuse_ops(p.ops, (S.cfg->flags & QS_OPT_FUSE) ? S.cfg->fuse_cap : 1);
  assign_phases(p);
  // Store relabel (reading r2, virtual qubit map): if the last register
  // layout holds the lowest chunk bits, each thread would store 2^run
  // contiguous amplitudes and the lanes would write 64+ B apart.  Instead
  // the pass writes its output with the chunk bits permuted -- the last
  // layout's thread bits onto the lowest positions, its register bits on
  // top -- and the map records where every qubit went (no extra exchange,
  // coalesced stores).
  static const bool relabel_on = !getenv("QS_NO_STORE_RELABEL");  // A/B knob
  if (map && relabel_on) {
    const std::vector<int>& last = p.phase_regs.back();
    int run = 0;
    while (std::find(last.begin(), last.end(), run) != last.end()) run++;
    if (run >= 2) {
      std::vector<int> order = phase_thread_order(last, (int)p.cpos.size());
      order.insert(order.end(), last.begin(), last.end());
      std::vector<int> opos(p.cpos.size());
      for (size_t i = 0; i < order.size(); i++) opos[order[i]] = p.cpos[i];
      std::vector<int>& mp = *map;
      std::vector<int> moved(mp.size());
      for (size_t q = 0; q < mp.size(); q++) {
        moved[q] = mp[q];
        for (size_t c = 0; c < p.cpos.size(); c++)
          if (mp[q] == p.cpos[c]) moved[q] = opos[c];
      }
      mp.swap(moved);
      p.opos = opos;
    }
  }
  // Low-slot steering (reading r7): the 3 lowest positions are in every
  // chunk, so every pass can act on the qubits that sit there.  The store
  // puts there, among the qubits the last layout keeps on lane bits (so the
  // 128 B store runs stay coalesced), those whose next dense gate comes
  // soonest; the map records the relabel.
  static const bool steer_on = !getenv("QS_NO_LOW_STEER");  // A/B knob
  if (map && upcoming && steer_on && p.cpos.size() >= 3 && p.cpos[0] == 0 && p.cpos[1] == 1 &&
      p.cpos[2] == 2) {
    std::vector<int>& mp = *map;  // logical -> physical, already after the store relabel
    const std::vector<int> order = phase_thread_order(p.phase_regs.back(), (int)p.cpos.size());
    const int nlane = std::min<int>(5, (int)order.size());
    // output position -> logical qubit (for this chunk's qubits)
    auto qubit_at = [&](int pos) {
      for (size_t q = 0; q < mp.size(); q++)
        if (mp[q] == pos) return (int)q;
      return -1;
    };
    auto next_use = [&](int q) {
      for (size_t i = 0; i < upcoming->size(); i++) {
        const IrGate& g = (*upcoming)[i];
        if (g.type != IrGate::DENSE) continue;
        for (int t : g.targets)
          if (t == q) return (long)i;
      }
      return (long)1 << 40;
    };
    struct Cand { int c; long use; };
    std::vector<Cand> cand;
    for (int t = 0; t < nlane; t++) {
      const int c = order[t];
      const int q = qubit_at(p.opos[c]);
      cand.push_back({c, q >= 0 ? next_use(q) : ((long)1 << 41)});
    }
    std::stable_sort(cand.begin(), cand.end(), [](const Cand& a, const Cand& b) { return a.use < b.use; });
    // give output positions 0,1,2 to the 3 best lane-bit chunk bits; the
    // chunk bits that fed them take the vacated positions.  Position 3 too
    // when this chunk has it: a chunk with position 3 (or 5) streams at full
    // HBM bandwidth, one with neither at ~0.75-0.8 of it (address-pattern
    // probe, scripts/dev/pattern_bw.cu), so the next pass should find a
    // target there (QS_NO_STEER3: A/B knob)
    static const bool steer3 = !getenv("QS_NO_STEER3");
    const int nslot = (steer3 && nlane >= 4 && std::find(p.opos.begin(), p.opos.end(), 3) != p.opos.end()) ? 4 : 3;
    for (int slot = 0; slot < nslot; slot++) {
      const int c = cand[slot].c;
      if (p.opos[c] == slot) continue;
      int holder = -1;
      for (size_t k = 0; k < p.opos.size(); k++)
        if (p.opos[k] == slot) holder = (int)k;
      const int qa = qubit_at(p.opos[c]), qb = qubit_at(slot);
      std::swap(p.opos[c], p.opos[holder]);
      if (qa >= 0) mp[qa] = slot;
      if (qb >= 0) mp[qb] = p.opos[holder];
    }
    // position 5 is the other fast-pattern position: any chunk bit may be
    // stored there (coalescing needs only 0,1,2 on lane bits), so it could
    // get the soonest-needed qubit of the rest of the chunk.  QS_STEER5=1
    // (A/B knob, off: on the plans it trades QAOA-30's fast-pattern passes
    // 7 -> 5 for rand-30's 19 -> 23, and rand's fast/slow gap is small)
    static const bool steer5 = getenv("QS_STEER5") != nullptr && atoi(getenv("QS_STEER5")) != 0;
    int h5 = -1;
    for (size_t k = 0; k < p.opos.size(); k++)
      if (p.opos[k] == 5) h5 = (int)k;
    if (steer3 && steer5 && h5 >= 0) {
      int best = -1;
      long bu = (long)1 << 40;
      for (size_t k = 0; k < p.opos.size(); k++) {
        if (p.opos[k] < nslot) continue;  // placed on 0..3 above
        const int q = qubit_at(p.opos[k]);
        const long u = q >= 0 ? next_use(q) : ((long)1 << 41);
        if (u < bu) {
          bu = u;
          best = (int)k;
        }
      }
      if (best >= 0 && best != h5) {
        const int qa = qubit_at(p.opos[best]), qb = qubit_at(5);
        std::swap(p.opos[best], p.opos[h5]);
        if (qa >= 0) mp[qa] = 5;
        if (qb >= 0) mp[qb] = p.opos[h5];
      }
    }
  }
  if (S.src_mode && p.buf == 0) {
    p.src_mode = S.src_mode;
    p.exp_bufs = S.exp_bufs;
    p.exp_lo = S.exp_lo;
    p.exp_len = S.exp_len;
    p.basis = S.basis_phys;
    S.src_mode = 0;
  }
}

// Schedule `gates` (logical) on buffer `buf` (nq qubits of which nl local,
// map logical->physical).  Appends steps; updates `map` (relabels, swaps).
static int schedule(Sched& S, int buf, int nq, int nl, std::vector<int>& map,
                    std::vector<IrGate> gates, std::string& err) {
  Plan& plan = *S.plan;
  const int n_global = nq - nl;
  const bool blocking = (S.cfg->flags & QS_OPT_BLOCK) != 0;
  // low positions always in a chunk (128 B runs); 3,4 added when room.
  // QS_PLAN_LOW: A/B knob for the forced low run
  static const int l = getenv("QS_PLAN_LOW") ? atoi(getenv("QS_PLAN_LOW")) : 3;
  std::vector<IrGate> rem;
  // A fused diagonal with more distinct monomials than one pass can encode
  // (kMaxShapes) is split into commuting factors (phase polynomials add).
  for (IrGate& g : gates) {
    if (g.type != IrGate::DIAG || g.mono.size() <= (size_t)kMaxShapes || nl <= kSmallMax) {
      rem.push_back(std::move(g));
      continue;
    }
    merge_mono(g.mono);
    for (size_t b = 0; b < g.mono.size(); b += kMaxShapes) {
      IrGate part = g;
      part.mono.assign(g.mono.begin() + b, g.mono.begin() + std::min(g.mono.size(), b + kMaxShapes));
      part.n_src = b ? 0 : g.n_src;
      rem.push_back(std::move(part));
    }
  }
  gates.clear();
  int guard = 0;
  while (!rem.empty()) {
    if (++guard > 1000000) {
      err = "planner failed to make progress";
      return QS_EINVAL;
    }
    PassPlan p;
    p.buf = buf;
    p.nl = nl;
    p.n_global = n_global;
    const bool small = nl <= kSmallMax;
    u64 need = 0;
    if (!small)
      for (int i = 0; i < l; i++) need |= 1ull << i;
    u64 blocked_all = 0, blocked_nd = 0;
    std::vector<IrGate> deferred;
    bool stop = false;
    bool progress = false;
    // FP64-instruction budget per amplitude (reading c15).  A pass whose
    // source is fused (booster expand / basis: write-only, 16 B/amp) is
    // given about the FP64 work the HBM time of a write-only pass covers
    // (~48/amp at 6.5 TB/s and ~18 TFLOP/s FP64), so ALU-heavy work moves to
    // the following read+write passes; other passes are capacity-limited.
    const double budget = (buf == 0 && S.src_mode && !small) ? S.wo_budget : 400.0;
    double cost = 0;
    // Encoder limit (kMaxShapes diagonal shapes per pass).  A diagonal op's
    // shapes are at most its distinct physical masks, and neither the
    // in-pass monomial sinking nor the fast-path split raises the sum over
    // ops, so the pass closes before that sum could exceed the limit.
    size_t shapes_done = 0;            // distinct masks of the earlier diagonal ops
    std::unordered_set<u64> cur_masks;  // the last diagonal op (open or just closed)
    int dense_taken = 0;
    u64 dense_union = 0;  // dense target positions taken (no-blocking fusion)
    u64 cur_regs = 0;
    int nphase = 1;
    for (size_t gi = 0; gi < rem.size(); gi++) {
      IrGate& g = rem[gi];
      const u64 s = g.support;
      auto defer = [&]() {
        blocked_all |= s;
        if (g.type != IrGate::DIAG) blocked_nd |= s;
        deferred.push_back(std::move(g));
      };
      if (stop) { defer(); continue; }
      if (g.type == IrGate::RELABEL) {
        if (s & blocked_all) { defer(); continue; }
        std::swap(map[g.targets[0]], map[g.targets[1]]);
        progress = true;
        continue;
      }
      if (g.type == IrGate::DIAG) {
        if (s & blocked_nd) { defer(); continue; }
        const bool open = !p.ops.empty() && p.ops.back().type == POp::DIAG;
        if (!small) {
          std::unordered_set<u64> fresh;
          for (const Mono& m : g.mono) {
            const u64 pm = map_mask(m.mask, map);
            if (!(open && cur_masks.count(pm))) fresh.insert(pm);
          }
          const size_t have = shapes_done + cur_masks.size();
          if (have + fresh.size() > (size_t)kMaxShapes && have > 0) { stop = true; defer(); continue; }
          if (!open) {
            shapes_done += cur_masks.size();
            cur_masks.clear();
          }
          cur_masks.insert(fresh.begin(), fresh.end());
        }
        if (!open) cost += 8;
        add_diag_op(p.ops, g, map);
        progress = true;
        continue;
      }
      // DENSE
      if (s & blocked_all) { defer(); continue; }
      u64 tp = 0;
      bool global = false;
      for (int q : g.targets) {
        if (map[q] >= nl) global = true;
        tp |= 1ull << map[q];
      }
      if (global) { defer(); continue; }
      if (!small) {
        const bool wide = (int)g.targets.size() >= kRegBits;  // 4-6 targets: shared-memory op
        u64 nn = need | tp;
        if (popc(nn) > kChunkBits) { defer(); continue; }
        const double c = (g.controls.empty() ? op_cost_unc(g.mat, g.is_h) : op_cost(g.mat, g.is_h)) + 0.5;
        if (cost + c > budget && dense_taken > 0) {
          if (budget == S.wo_budget) plan.stats.wo_budget_hit = true;
          stop = true;
          defer();
          continue;
        }
        // register layouts (assign_phases' greedy, on positions): a new
        // layout costs a shared-memory exchange; keep <= kMaxPhases/2
        {
          const u64 uni = cur_regs | tp;
          int ph = nphase, cnt = popc(uni);
          u64 nr = uni;
          if (wide) {  // starts a new layout (applied at the exchange into it)
            ph++;
            nr = 0;
          } else if ((tp & ~cur_regs) && cnt > kRegBits) {
            ph++;
            nr = tp;
          }
          if (ph > kMaxPhases / 2) { stop = true; defer(); continue; }
          nphase = ph;
          cur_regs = nr;
        }
        // without cache blocking a pass is one state sweep for one gate -- or,
        // with fusion, for the gates whose targets fuse into one <= F-qubit
        // unitary (the paper's Naive_f, L782)
        if (!blocking && dense_taken > 0 &&
            (!(S.cfg->flags & QS_OPT_FUSE) || popc(dense_union | tp) > S.cfg->fuse_cap)) {
          stop = true;
          defer();
          continue;
        }
        need = nn;
        cost += c;
        dense_union |= tp;
      }
      p.ops.push_back(dense_pop(g, map));
      ++dense_taken;
      progress = true;
    }
    rem.swap(deferred);
    if (!p.ops.empty()) {
      if (small) {
        if (S.src_mode && buf == 0) {
          p.src_mode = S.src_mode;
          p.exp_bufs = S.exp_bufs;
          p.exp_lo = S.exp_lo;
          p.exp_len = S.exp_len;
          p.basis = S.basis_phys;
          S.src_mode = 0;
        }
        p.kernel = KK_SMALL;
        p.cpos.clear();
      } else {
        finalize_chunk_pass(S, p, need, nl, buf == 0 ? &map : nullptr, &deferred);
      }
      plan.steps.push_back(Step{Step::PASS, p});
      if (buf == 0) {  // statistics count full-state passes only
        if (p.kernel == KK_CHUNK) plan.stats.n_chunk++;
        else if (p.kernel == KK_DENSE) plan.stats.n_dense++;
        else if (p.kernel == KK_DIAG) plan.stats.n_diag++;
        else plan.stats.n_small++;
        plan.stats.n_passes++;
        plan.stats.bytes_hbm += ((p.src_mode ? 16ull : 32ull) << nl);
      }
      continue;
    }
    if (progress) continue;  // only relabels were taken
    // Nothing applicable: the first pending dense gate has a global target.
    if (n_global == 0) {
      err = "internal: no progress on a single-rank buffer";
      return QS_EINVAL;
    }
    // rem[0] is the blocked gate (a diagonal or relabel at the head would
    // have been taken): bring its global targets in, keep its local targets,
    // and bring further globals needed by later gates while room remains.
    std::vector<int> gpos;
    u64 protect = 0;
    for (int q : rem[0].targets) {
      if (map[q] >= nl) gpos.push_back(map[q]);
      else protect |= 1ull << map[q];
    }
    for (const IrGate& g : rem) {
      if (g.type != IrGate::DENSE) continue;
      for (int q : g.targets)
        if (map[q] >= nl && std::find(gpos.begin(), gpos.end(), map[q]) == gpos.end() &&
            (int)gpos.size() < n_global && (int)gpos.size() + 1 + popc(protect) <= nl)
          gpos.push_back(map[q]);
      if ((int)gpos.size() == n_global) break;
    }
    std::sort(gpos.begin(), gpos.end());
    const int j = (int)gpos.size();
    if (j > nl) {
      err = "too few local qubits for the swap";
      return QS_EINVAL;
    }
    for (const IrGate& g : rem)
      if (g.type == IrGate::DENSE && (int)g.targets.size() > nl) {
        err = "a gate has more targets than there are local qubits";
        return QS_EINVAL;
      }
    if (buf == 0) flush_source(S);
    std::vector<int> inv(nq);
    for (int q = 0; q < nq; q++) inv[map[q]] = q;
    // Victims: the j local qubits whose next use as a dense target is the
    // farthest (Belady), preferring those already at the top positions.
    std::vector<size_t> next(nq, (size_t)-1);
    for (size_t i = rem.size(); i-- > 0;)
      if (rem[i].type == IrGate::DENSE)
        for (int q : rem[i].targets) next[q] = i;
    std::vector<int> cand;
    for (int p = 0; p < nl; p++)
      if (!(protect >> p & 1)) cand.push_back(p);
    std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) {
      const size_t na = next[inv[a]], nb = next[inv[b]];
      if (na != nb) return na > nb;
      return a > b;  // prefer high (top) positions
    });
    std::vector<int> victims(cand.begin(), cand.begin() + j);
    std::vector<int> top;
    for (int i = 0; i < j; i++) top.push_back(nl - j + i);
    // f1: the exchange can ride on the stores of the pass right before it
    // (no expand in between; a specialised kernel, which picks each store's
    // destination from the exported bits of its index).  Then the victims
    // need not be moved to the top positions first: the swap exchanges the
    // globals directly with the victims' positions (a victim already on top
    // pairs with its own top slot, so that the swap equals "permute the
    // victims to the top, swap, permute back" -- the unfused fallback).
    PassPlan* fuse_into = nullptr;
    if (buf == 0 && j <= kMaxXBits && !plan.steps.empty() && plan.steps.back().type == Step::PASS) {
      PassPlan& lp = plan.steps.back().pass;
      if (lp.buf == 0 && lp.kernel != KK_SMALL && lp.nl >= S.cfg->jit_min_qubits) fuse_into = &lp;
    }
    static const bool direct_on = !getenv("QS_NO_DIRECT_SWAP");  // A/B knob
    std::vector<int> lpos = top;
    if (fuse_into && direct_on) {
      std::vector<int> rest;
      for (int v : victims)
        if (v >= nl - j) lpos[v - (nl - j)] = -1 - v;  // placeholder: fixed below
        else rest.push_back(v);
      size_t ri = 0;
      for (int i = 0; i < j; i++) lpos[i] = (lpos[i] < 0) ? -1 - lpos[i] : rest[ri++];
    } else {
      // local bit permutation bringing the victims to the top positions
      std::vector<int> tv, vv;  // top non-victims, victims not on top
      for (int t : top)
        if (std::find(victims.begin(), victims.end(), t) == victims.end()) tv.push_back(t);
      for (int v : victims)
        if (v < nl - j) vv.push_back(v);
      if (!tv.empty()) {
        Step ps;
        ps.type = Step::PERMUTE;
        for (size_t i = 0; i < tv.size(); i++) {
          ps.gpos.push_back(tv[i]);
          ps.lpos.push_back(vv[i]);
          std::swap(map[inv[tv[i]]], map[inv[vv[i]]]);
          std::swap(inv[tv[i]], inv[vv[i]]);
        }
        plan.steps.push_back(ps);
        plan.stats.n_passes++;
        plan.stats.bytes_hbm += (32ull << nl);
        fuse_into = nullptr;
      }
    }
    Step st;
    st.type = Step::SWAP;
    st.j = j;
    st.gpos = gpos;
    st.lpos = lpos;
    if (fuse_into) {
      fuse_into->x_j = j;
      fuse_into->x_pos = lpos;
      st.fusable = true;
      plan.stats.n_fusable_swaps++;
    }
    // relabel: logical at gpos[i] <-> logical at lpos[i]
    for (int i = 0; i < j; i++) std::swap(map[inv[st.gpos[i]]], map[inv[st.lpos[i]]]);
    plan.steps.push_back(st);
    plan.stats.n_swaps++;
    plan.stats.bytes_nvlink += (16ull << nl) - (16ull << (nl - j));
  }
  return QS_OK;
}

// ------------------------------------------------------------ Alg. 7
// Merge booster (readings c8-c11).  Sub-state buffers are simulated with the
// same scheduler (replicated on every rank); the final merge into the full
// state is fused into the load of the first full-state pass (K5 as a source).
static int booster(Sched& S, int n, std::vector<IrGate>& gates, std::string& err) {
  Plan& plan = *S.plan;
  const int B = std::max(1, S.cfg->boost_div);
  std::vector<int> que;
  divider(n, (n + B - 1) / B, que);
  if (que.size() <= 1) return QS_OK;  // nothing to divide: plain basis source
  struct Grp { int lo, len, buf; };
  std::vector<Grp> groups;
  int lo = 0;
  auto new_sub = [&](int len, int glo) {
    plan.subs.push_back(SubBuf{len, glo});
    return (int)plan.subs.size();  // ids start at 1
  };
  for (int len : que) {
    Grp g{lo, len, new_sub(len, lo)};
    Step st;
    st.type = Step::SUB_INIT;
    st.buf = g.buf;
    st.basis = (S.basis_phys >> lo) & ((1ull << len) - 1);
    plan.steps.push_back(st);
    groups.push_back(g);
    lo += len;
  }
  uint64_t sub_gates = 0;
  while (groups.size() > 1) {
    std::vector<int> round_counts;
    for (Grp& g : groups) {
      const u64 gm = ((g.len >= 64) ? ~0ull : ((1ull << g.len) - 1)) << g.lo;
      // genGateBlock (c11): support within the group and every earlier
      // unscheduled gate overlapping it already scheduled.
      std::vector<IrGate> mine, rest;
      u64 blocked = 0;
      for (IrGate& x : gates) {
        if ((x.support & ~gm) == 0 && !(x.support & blocked)) {
          mine.push_back(std::move(x));
        } else {
          blocked |= x.support;
          rest.push_back(std::move(x));
        }
      }
      gates.swap(rest);
      round_counts.push_back((int)mine.size());
      plan.stats.paper_updates += (uint64_t)mine.size() << g.len;
      sub_gates += mine.size();
      if (!mine.empty()) {
        // remap to sub-state qubits; relabels become physical SWAPs here
        for (IrGate& x : mine) {
          if (x.type == IrGate::RELABEL) {
            x.type = IrGate::DENSE;
            int t = 0;
            gate_matrix(QS_SWAP, nullptr, x.mat, &t);
          }
          for (int& q : x.targets) q -= g.lo;
          for (int& q : x.controls) q -= g.lo;
          x.support >>= g.lo;
          for (Mono& mo : x.mono) mo.mask >>= g.lo;
        }
        std::vector<int> smap(g.len);
        for (int i = 0; i < g.len; i++) smap[i] = i;
        int rc = schedule(S, g.buf, g.len, g.len, smap, std::move(mine), err);
        if (rc) return rc;
      }
    }
    plan.stats.booster_rounds.push_back(round_counts);
    // merge pairwise, c8: odd leftover kept as its own group
    std::vector<Grp> next;
    if (groups.size() == 2 && groups[0].len + groups[1].len == n) {
      // final merge: fused into the first full-state pass (or standalone)
      S.src_mode = 1;
      S.exp_bufs.clear(); S.exp_lo.clear(); S.exp_len.clear();
      for (Grp& g : groups) {
        S.exp_bufs.push_back(g.buf);
        S.exp_lo.push_back(g.lo);
        S.exp_len.push_back(g.len);
      }
      plan.stats.paper_updates += 1ull << n;
      groups.clear();
      groups.push_back(Grp{0, n, 0});
      break;
    }
    for (size_t i = 0; i + 1 < groups.size(); i += 2) {
      Grp a = groups[i], b = groups[i + 1];
      Grp m{a.lo, a.len + b.len, new_sub(a.len + b.len, a.lo)};
      Step st;
      st.type = Step::SUB_MERGE;
      st.buf = m.buf;
      st.src_a = a.buf;
      st.src_b = b.buf;
      plan.steps.push_back(st);
      plan.stats.paper_updates += 1ull << m.len;
      next.push_back(m);
    }
    if (groups.size() & 1) next.push_back(groups.back());
    groups.swap(next);
  }
  plan.stats.n_sub_gates = sub_gates;
  if (S.src_mode != 1) {
    // que had a single group: nothing to boost
    S.src_mode = 2;
  }
  return QS_OK;
}

// ------------------------------------------------------------ make_plan
static int make_plan_budget(const PlanInput& in, const std::vector<IrGate>& gates_in, Plan& plan,
                            std::string& err, double wo_budget);
static void mark_pull_splits(Plan& plan, const qs_config_t& cfg);
static void mark_l2_groups(Plan& plan, const qs_config_t& cfg);

// The write-only first pass (booster / basis source fused) gets an FP64
// budget (c15): about the work its 16 B/amp of writes hide (~40 FP64/amp).
// A larger budget can save a whole read/write pass later (QAOA-30: 12 -> 11
// passes at 64), so the optimiser plans with both and keeps the plan with
// fewer full-state passes (candidates 40, 48, 64; ties: the smaller, more
// balanced budget).  QS_WO_BUDGET pins one.
int make_plan(const PlanInput& in, const std::vector<IrGate>& gates_in, Plan& plan,
              std::string& err) {
  const char* e = getenv("QS_WO_BUDGET");  // experiment knob
  if (e && *e) {
    const int rc = make_plan_budget(in, gates_in, plan, err, atof(e));
    if (rc == QS_OK) {
      mark_pull_splits(plan, in.cfg);
      mark_l2_groups(plan, in.cfg);
    }
    return rc;
  }
  // (more than 2 ranks: 40/48 only -- QAOA-32 on 4 GPUs takes 13 passes at
  // 64 but two of its fused-swap passes then run at half the NVLink rate:
  // 160.6 vs 135.7 ms with push/pull, measured per launch; on 2 GPUs the
  // 64-plan wins, 111.8 vs 116.2 ms.  QFT-32 on 4 GPUs needs 48 for 2 passes)
  // Alternatives are planned only when the budget actually closed the
  // write-only pass (otherwise they would produce the same plan).
  int rc = make_plan_budget(in, gates_in, plan, err, 40.0);
  if (rc) return rc;
  if (in.product_state && plan.stats.n_passes >= 3 && plan.stats.wo_budget_hit)
    for (double b : {48.0, 64.0}) {
      if (in.n_global > 1 && b > 48.0) break;
      Plan alt;
      std::string err2;
      if (make_plan_budget(in, gates_in, alt, err2, b) == QS_OK && alt.stats.n_passes < plan.stats.n_passes)
        plan = std::move(alt);
    }
  mark_pull_splits(plan, in.cfg);
  mark_l2_groups(plan, in.cfg);
  return QS_OK;
}

static int make_plan_budget(const PlanInput& in, const std::vector<IrGate>& gates_in, Plan& plan,
                            std::string& err, double wo_budget) {
  plan = Plan();
  plan.n = in.n;
  plan.n_global = in.n_global;
  plan.nl = in.n - in.n_global;
  plan.map_in = in.map;
  plan.stats.n_gates_in = gates_in.size();
  plan.stats.naive_updates = (uint64_t)gates_in.size() << in.n;
  Sched S;
  S.plan = &plan;
  S.cfg = &in.cfg;
  S.wo_budget = wo_budget;
  std::vector<int> map = in.map;
  std::vector<IrGate> gates = gates_in;
  if (in.product_state) {
    // a basis state is stored at the identity map (qs_set_basis_state)
    S.basis_phys = in.basis;
    S.src_mode = 2;
  }
  const bool boost = in.product_state && (in.cfg.flags & QS_OPT_BOOST) && in.n >= 2;
  if (boost) {
    int rc = booster(S, in.n, gates, err);
    if (rc) return rc;
  }
  const uint64_t before = plan.stats.paper_updates;
  if (in.cfg.flags & QS_OPT_DIAG)
    gates = diagonal_detector(gates, in.n, in.cfg.diag_cap, &plan.stats.n_fused_diag);
  uint64_t full_gates = 0;
  for (const IrGate& g : gates) full_gates += g.n_src;
  plan.stats.paper_updates = before + (full_gates << in.n);
  static const bool tdump = getenv("QS_PLAN_TIMING") != nullptr;  // diagnostics
  auto ts = std::chrono::steady_clock::now();
  int rc = schedule(S, 0, in.n, plan.nl, map, std::move(gates), err);
  if (tdump)
    fprintf(stderr, "qs_plan schedule(full) %.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts).count());
  if (rc) return rc;
  if (S.src_mode) flush_source(S);  // circuit left nothing to fuse the source into
  plan.map_out = map;
  return QS_OK;
}

// Push/pull split of fused swaps.  A fused pass is
// NVLink-bound: it exports (1 - 2^-j) of the shard while it streams only
// 32 B/amp through HBM.  When the pass after the swap is a full-state
// specialised pass and a free split position z is a chunk-id bit of both
// passes, the exporting pass pushes the chunks with z = 0 and leaves the
// z = 1 chunks in place; the next pass loads those elements straight from
// the source ranks' buffers (NVLink reads; the source of an element is its
// piece = its bits at the swap's local positions), so both passes carry half
// the link traffic.  Data placement after the next pass is unchanged.
static void mark_pull_splits(Plan& plan, const qs_config_t& cfg) {
  if (plan.n_global == 0 || getenv("QS_NO_PULL")) return;
  for (size_t i = 0; i + 2 < plan.steps.size(); i++) {
    Step& a = plan.steps[i];
    Step& sw = plan.steps[i + 1];
    Step& b = plan.steps[i + 2];
    if (a.type != Step::PASS || sw.type != Step::SWAP || !sw.fusable || b.type != Step::PASS) continue;
    PassPlan& pk = a.pass;
    PassPlan& pn = b.pass;
    if (pk.buf != 0 || pn.buf != 0 || pk.x_j == 0 || pn.kernel == KK_SMALL || pn.src_mode != 0 ||
        pn.nl < cfg.jit_min_qubits || pn.x_j)
      continue;
    u64 ck = 0, cn = 0, lp = 0;
    for (int c : pk.cpos) ck |= 1ull << c;
    for (int c : pn.cpos) cn |= 1ull << c;
    for (int q : sw.lpos) lp |= 1ull << q;
    // the pull pass loads each element from the buffer its piece (bits at
    // lpos, usually chunk bits: the swap brings in the qubits it acts on)
    // selects; a contiguous low run of the chunk must not straddle pieces
    int l = 0;
    while (l < (int)pn.cpos.size() && pn.cpos[l] == l) l++;
    if (lp & ((1ull << l) - 1)) continue;
    int z = -1;
    for (int q = pk.nl - 1; q >= 0 && z < 0; q--)
      if (!(ck >> q & 1) && !(cn >> q & 1) && !(lp >> q & 1)) z = q;
    if (z < 0) continue;
    pk.x_split = z;
    pn.pull_j = sw.j;
    pn.pull_z = z;
    pn.pull_pos = sw.lpos;
  }
}

// Two-level blocking (the state of a gate block
// is "accommodated in the higher-level memory ... and processed
// consecutively"; C "within the cache capacity").  Level 1 is the
// 2^12-amplitude chunk of one CTA (shared memory, Alg. 2).  Level 2 is a
// contiguous block of 2^W amplitudes (W = cfg.l2_block_qubits): a pass whose
// chunk and output positions all lie below W maps every such block onto
// itself, so a run of consecutive such passes can be executed block by block
// -- a wave of chunks [b 2^(W-12), (b+1) 2^(W-12)) through every pass of the
// run before the next wave -- and every pass after a wave's first finds the
// wave in L2.  The run's HBM traffic is one read (none for a write-only
// first pass) and one write of the state.  Fused-swap exporters and pull
// passes talk to peers and stay outside.
static void mark_l2_groups(Plan& plan, const qs_config_t& cfg) {
  const int W = cfg.l2_block_qubits;
  plan.stats.bytes_hbm_l2 = plan.stats.bytes_hbm;
  if (W <= 0 || plan.nl <= W) return;
  auto eligible = [&](const Step& st) {
    if (st.type != Step::PASS) return false;
    const PassPlan& p = st.pass;
    if (p.buf != 0 || p.nl != plan.nl || p.kernel == KK_SMALL || p.nl < cfg.jit_min_qubits) return false;
    if (p.x_j || p.x_split >= 0 || p.pull_j) return false;
    for (int c : p.cpos)
      if (c >= W) return false;
    for (int c : p.opos)
      if (c >= W) return false;
    return true;
  };
  int g = 0;
  for (size_t i = 0; i < plan.steps.size();) {
    size_t j = i;
    while (j < plan.steps.size() && eligible(plan.steps[j])) j++;
    if (j - i >= 2) {
      for (size_t k = i; k < j; k++) {
        plan.steps[k].pass.l2_grp = g;
        // every pass after the first: L2 only (algorithmic HBM bytes)
        if (k > i) plan.stats.bytes_hbm_l2 -= (uint64_t)32 << plan.nl;
      }
      // the first pass's write reaches HBM only through the last one
      g++;
    }
    i = j > i ? j : i + 1;
  }
  plan.stats.n_l2_groups = (uint64_t)g;
}

// ------------------------------------------------------------ encoding
namespace {
struct Blob {
  std::vector<unsigned char> b;
  size_t align(size_t a) {
    while (b.size() % a) b.push_back(0);
    return b.size();
  }
  template <class T>
  size_t put(const T* p, size_t n) {
    size_t off = align(16);
    const unsigned char* c = reinterpret_cast<const unsigned char*>(p);
    b.insert(b.end(), c, c + n * sizeof(T));
    return off;
  }
};

int pair_code(int a, int b) {
  static const int codes[4][4] = {{-1, 0, 1, 2}, {0, -1, 3, 4}, {1, 3, -1, 5}, {2, 4, 5, -1}};
  return codes[a][b];
}
}  // namespace

int encode_pass(const PassPlan& p, int rank, std::vector<unsigned char>& out, std::string& err) {
  KPass h;
  memset(&h, 0, sizeof h);
  h.kernel = p.kernel;
  h.nl = p.nl;
  h.rank_base = (u64)rank << p.nl;
  h.local_mask = (p.nl >= 64) ? ~0ull : ((1ull << p.nl) - 1);
  h.src_mode = p.src_mode;
  h.basis = p.basis;
  if (p.src_mode == 1) {  // structure of the expansion; pointers patched by the executor
    h.expand.n = (int)p.exp_lo.size();
    for (int g = 0; g < h.expand.n && g < kMaxExpand; g++) {
      h.expand.lo[g] = p.exp_lo[g];
      h.expand.len[g] = p.exp_len[g];
    }
  }
  h.scale = 1.0;
  h.scale_im = 0.0;
  cd lam_total(1.0, 0.0);  // scalars factored out of unit-scaled ops
  if (p.x_j < 0 || p.x_j > kMaxXBits) {
    err = "internal: fused swap exports more than 3 qubits";
    return QS_EINVAL;
  }
  h.x_split = (int8_t)p.x_split;
  h.pull_j = (int8_t)p.pull_j;
  h.pull_z = (int8_t)p.pull_z;
  for (int i = 0; i < 5; i++) h.pull_pos[i] = (int8_t)(i < (int)p.pull_pos.size() ? p.pull_pos[i] : 0);
  if (p.pull_j > kMaxXBits) {
    err = "internal: pull of more than 3 qubits";
    return QS_EINVAL;
  }
  h.x_shift = p.x_j ? p.nl - p.x_j : 0;
  h.x_mask = p.x_j ? (1 << p.x_j) - 1 : 0;
  memset(h.x_pos, 0, sizeof h.x_pos);
  for (int i = 0; i < p.x_j && i < (int)sizeof h.x_pos; i++) h.x_pos[i] = (int8_t)p.x_pos[i];
  int n_hu = 0;
  std::vector<KOp> kops;
  std::vector<KGroup> kgroups;
  std::vector<KShape> kshapes;
  std::vector<KTerm> kterms;
  std::vector<double> pool;
  auto put_mat = [&](const std::vector<cd>& m) {
    while (pool.size() % 2) pool.push_back(0);
    int off = (int)pool.size();
    for (const cd& z : m) {
      pool.push_back(z.real());
      pool.push_back(z.imag());
    }
    return off;
  };

  if (p.kernel == KK_SMALL) {
    h.n_chunks = 1;
    for (const POp& op : p.ops) {
      KOp k;
      memset(&k, 0, sizeof k);
      if (op.type == POp::DIAG) {
        k.type = OP_SDIAG;
        k.data = (int)kterms.size();
        for (const Mono& m : op.mono) kterms.push_back({m.mask, m.coeff});
        k.data2 = (int)op.mono.size();
      } else {
        k.type = OP_SDENSE;
        k.k = (uint8_t)op.tpos.size();
        for (size_t i = 0; i < op.tpos.size(); i++) k.tpos[i] = (int8_t)op.tpos[i];
        k.ncm = op.cmask;
        k.data = put_mat(op.mat);
      }
      kops.push_back(k);
    }
    h.n_ops = (int)kops.size();
  } else {
    const int m = (int)p.cpos.size();
    if (m != kChunkBits) {
      err = "internal: chunk size";
      return QS_EINVAL;
    }
    for (int c = 0; c < m; c++) {
      h.cpos[c] = (int8_t)p.cpos[c];
      h.opos[c] = (int8_t)p.opos[c];
    }
    // chunk-id deposit runs over the free local positions
    u64 cm = 0;
    for (int c : p.cpos) cm |= 1ull << c;
    std::vector<int> freep;
    for (int pos = 0; pos < p.nl; pos++)
      if (!(cm >> pos & 1)) freep.push_back(pos);
    h.n_chunks = 1ull << freep.size();
    int nr = 0;
    for (size_t i = 0; i < freep.size();) {
      size_t j = i;
      while (j + 1 < freep.size() && freep[j + 1] == freep[j] + 1) j++;
      if (nr >= kMaxRuns) {
        err = "internal: too many runs";
        return QS_EINVAL;
      }
      h.run_src[nr] = (int8_t)i;
      h.run_dst[nr] = (int8_t)freep[i];
      h.run_len[nr] = (int8_t)(j - i + 1);
      nr++;
      i = j + 1;
    }
    h.n_runs = nr;
    const int nph = (int)p.phase_regs.size();
    if (nph > kMaxPhases) {
      err = "internal: too many phases";
      return QS_EINVAL;
    }
    h.n_phases = nph;
    // per-phase layouts
    std::vector<std::vector<int>> thr(nph);
    for (int ph = 0; ph < nph; ph++) {
      const std::vector<int>& regs = p.phase_regs[ph];
      KPhase& kp = h.phases[ph];
      for (int k = 0; k < kRegBits; k++) kp.reg_c[k] = (int8_t)regs[k];
      const std::vector<int> order = phase_thread_order(regs, m);
      for (int i = 0; i < kLogT; i++) kp.thr_c[i] = (int8_t)order[i];
      thr[ph] = order;
    }
    auto cbit = [&](int pos) {
      return (int)(std::find(p.cpos.begin(), p.cpos.end(), pos) - p.cpos.begin());
    };
    int cur_phase = -1;
    for (size_t oi = 0; oi < p.ops.size(); oi++) {
      const POp& op = p.ops[oi];
      const int ph = p.op_phase[oi];
      while (cur_phase < ph) {
        if (cur_phase >= 0) h.phases[cur_phase].op_end = (int16_t)kops.size();
        cur_phase++;
        h.phases[cur_phase].op_begin = (int16_t)kops.size();
      }
      const std::vector<int>& regs = p.phase_regs[ph];
      auto regidx = [&](int c) {
        return (int)(std::find(regs.begin(), regs.end(), c) - regs.begin());
      };
      KOp k;
      memset(&k, 0, sizeof k);
      if (op.type == POp::DENSE && (int)op.tpos.size() >= kRegBits) {
        // wide op: chunk-bit targets and controls (shared-memory matvec; a
        // 16x16 in registers would hold 16 inputs + 16 outputs = all 128
        // registers of a 2-CTA/SM thread and spill)
        if (oi != 0 && p.op_phase[oi - 1] == ph) {
          err = "internal: wide op is not the first op of its layout";
          return QS_EINVAL;
        }
        if (ph == 0) {
          err = "internal: wide op in the first layout";
          return QS_EINVAL;
        }
        u64 ncm = 0;
        uint32_t ccm = 0;
        for (u64 c = op.cmask; c;) {
          const int pos = __builtin_ctzll(c);
          c &= c - 1;
          const int cb = (pos < p.nl) ? cbit(pos) : m;
          if (cb < m) ccm |= 1u << cb;
          else ncm |= 1ull << pos;
        }
        k.type = OP_DW;
        k.k = (uint8_t)op.tpos.size();
        for (size_t i = 0; i < op.tpos.size(); i++) {
          const int cb = cbit(op.tpos[i]);
          if (cb >= m) {
            err = "internal: wide-op target not in the chunk";
            return QS_EINVAL;
          }
          k.tpos[i] = (int8_t)cb;
        }
        k.rcm = ccm;
        k.ncm = ncm;
        k.data = put_mat(op.mat);
      } else if (op.type == POp::DENSE) {
        // controls: register bits -> rho mask; the rest stay physical
        u64 ncm = 0;
        uint32_t rcm = 0;
        for (u64 c = op.cmask; c;) {
          int pos = __builtin_ctzll(c);
          c &= c - 1;
          int cb = (pos < p.nl) ? cbit(pos) : m;
          int ri = (cb < m) ? regidx(cb) : kRegBits;
          if (ri < kRegBits) rcm |= 1u << ri;
          else ncm |= 1ull << pos;
        }
        k.rcm = rcm;
        k.ncm = ncm;
        const int t = (int)op.tpos.size();
        std::vector<int> rbits(t);
        for (int i = 0; i < t; i++) {
          int cb = cbit(op.tpos[i]);
          rbits[i] = regidx(cb);
          if (rbits[i] >= kRegBits) {
            err = "internal: target not in register layout";
            return QS_EINVAL;
          }
        }
        // permute the matrix so that its bit j <-> j-th smallest register bit
        std::vector<int> sorted = rbits;
        std::sort(sorted.begin(), sorted.end());
        std::vector<int> newbit(t);
        for (int i = 0; i < t; i++)
          newbit[i] = (int)(std::find(sorted.begin(), sorted.end(), rbits[i]) - sorted.begin());
        const int D = 1 << t;
        std::vector<cd> pm((size_t)D * D);
        for (int r = 0; r < D; r++)
          for (int c = 0; c < D; c++) {
            int r2 = 0, c2 = 0;
            for (int i = 0; i < t; i++) {
              r2 |= ((r >> i) & 1) << newbit[i];
              c2 |= ((c >> i) & 1) << newbit[i];
            }
            pm[(size_t)r2 * D + c2] = op.mat[(size_t)r * D + c];
          }
        // uncontrolled unit-scaled op: +-1/+-i matrix, scalar into the pass scale
        {
          cd lam;
          std::vector<cd> unit;
          if (op.cmask == 0 && !op.is_h && !op.is_x && unit_scaled(pm, &lam, &unit)) {
            pm.swap(unit);
            lam_total *= lam;
          } else if (t == 1 && op.cmask == 0 && !op.is_h && !op.is_x && row_scale_1q(pm, &lam)) {
            lam_total *= lam;
          }
        }
        if (t == 1) {
          k.sel = (uint8_t)rbits[0];
          if (op.is_h && rcm == 0 && ncm == 0) {
            k.type = OP_HU;  // unnormalised; the pass scale restores 1/sqrt2
            n_hu++;
          } else if (op.is_h) k.type = OP_H;
          else if (op.is_x) k.type = OP_X;
          else { k.type = OP_D1; k.data = put_mat(pm); }
        } else if (t == 2) {
          k.type = OP_D2;
          k.sel = (uint8_t)pair_code(sorted[0], sorted[1]);
          k.data = put_mat(pm);
        } else if (t == 3) {
          k.type = OP_D3;
          int missing = 0;
          while (std::find(sorted.begin(), sorted.end(), missing) != sorted.end()) missing++;
          k.sel = (uint8_t)missing;
          k.data = put_mat(pm);
        } else {
          err = "internal: dense op too wide";
          return QS_EINVAL;
        }
      } else {
        // DIAG: shapes keyed by (register subset R, thread mask)
        k.type = OP_DIAG;
        std::map<std::pair<int, uint32_t>, std::vector<KTerm>> shapes;
        const std::vector<int>& order = thr[ph];
        for (const Mono& mo : op.mono) {
          u64 ncmask = 0;
          int R = 0;
          uint32_t tm = 0;
          for (u64 x = mo.mask; x;) {
            int pos = __builtin_ctzll(x);
            x &= x - 1;
            int cb = (pos < p.nl) ? cbit(pos) : m;
            if (cb >= m) { ncmask |= 1ull << pos; continue; }
            int ri = regidx(cb);
            if (ri < kRegBits) { R |= 1 << ri; continue; }
            int ti = (int)(std::find(order.begin(), order.end(), cb) - order.begin());
            tm |= 1u << ti;
          }
          shapes[{R, tm}].push_back({ncmask, mo.coeff});
        }
        KGroup G;
        memset(&G, 0, sizeof G);
        G.ck_off = -1;
        // Fast path (OP_DIAGF) when every shape with >= 2 register bits is
        // constant (no thread bits, no chunk-dependent terms): those go to a
        // host table CK16[rho] = exp(2 pi i sum_{R subset rho, |R|>=2} K_R).
        bool fast = true;
        for (auto& kv : shapes) {
          if (popc((u64)kv.first.first) < 2) continue;
          if (kv.first.second != 0) fast = false;
          for (const KTerm& tt : kv.second)
            if (tt.ncmask != 0) fast = false;
        }
        if (fast) {
          u64 K[kNReg] = {0};
          bool any_pair = false;
          for (auto it = shapes.begin(); it != shapes.end();) {
            const int R = it->first.first;
            if (popc((u64)R) >= 2) {
              for (const KTerm& tt : it->second) K[R] += tt.coeff;
              any_pair = true;
              it = shapes.erase(it);
            } else {
              ++it;
            }
          }
          int lin = 0, hc = 0;
          for (auto& kv : shapes) {
            if (kv.first.first) lin |= kv.first.first;
            else hc = 1;
          }
          uint32_t touch = 0;
          std::vector<cd> ck(kNReg, cd(1, 0));
          for (int r = 0; r < kNReg; r++) {
            u64 ang = 0;
            bool nz = false;
            for (int R = 0; R < kNReg; R++)
              if (popc((u64)R) >= 2 && (R & ~r) == 0 && K[R]) {
                ang += K[R];
                nz = true;
              }
            if (nz) {
              if ((ang & ((1ull << 62) - 1)) == 0) {  // quarter turns: exact units
                static const cd unit[4] = {cd(1, 0), cd(0, 1), cd(-1, 0), cd(0, -1)};
                ck[r] = unit[ang >> 62];
              } else {
                const long double th = (long double)ang / 18446744073709551616.0L * 6.283185307179586476925286766559L;
                ck[r] = cd((double)cosl(th), (double)sinl(th));
              }
            }
            if (hc || (r & lin) || nz) touch |= 1u << r;
          }
          if (any_pair) G.ck_off = put_mat(ck);
          k.type = OP_DIAGF;
          k.rcm = touch;
          int cnt[kNReg + 1] = {0};
          for (auto& kv : shapes) cnt[kv.first.first]++;
          G.rbeg[0] = (int)kshapes.size();
          for (int R = 0; R < kNReg; R++) G.rbeg[R + 1] = G.rbeg[R] + cnt[R];
          int fill[kNReg];
          std::vector<KShape> tmp(shapes.size());
          for (int R = 0; R < kNReg; R++) fill[R] = G.rbeg[R] - (int)kshapes.size();
          for (auto& kv : shapes) {
            KShape s;
            memset(&s, 0, sizeof s);
            s.tmask = kv.first.second;
            s.term_begin = (int)kterms.size();
            kterms.insert(kterms.end(), kv.second.begin(), kv.second.end());
            s.term_end = (int)kterms.size();
            tmp[fill[kv.first.first]++] = s;
          }
          kshapes.insert(kshapes.end(), tmp.begin(), tmp.end());
          k.sel = (uint8_t)lin;
          k.has_const = (uint8_t)hc;
          k.data = (int)kgroups.size();
          kgroups.push_back(G);
          kops.push_back(k);
          continue;
        }
        int active = 0, has_const = 0;
        int cnt[kNReg + 1] = {0};
        for (auto& kv : shapes) cnt[kv.first.first]++;
        G.rbeg[0] = (int)kshapes.size();
        for (int R = 0; R < kNReg; R++) G.rbeg[R + 1] = G.rbeg[R] + cnt[R];
        std::vector<KShape> tmp(shapes.size());
        int fill[kNReg];
        for (int R = 0; R < kNReg; R++) fill[R] = G.rbeg[R] - (int)kshapes.size();
        for (auto& kv : shapes) {
          const int R = kv.first.first;
          if (R) active |= R;
          else has_const = 1;
          KShape s;
          memset(&s, 0, sizeof s);
          s.tmask = kv.first.second;
          s.term_begin = (int)kterms.size();
          kterms.insert(kterms.end(), kv.second.begin(), kv.second.end());
          s.term_end = (int)kterms.size();
          tmp[fill[R]++] = s;
        }
        kshapes.insert(kshapes.end(), tmp.begin(), tmp.end());
        k.sel = (uint8_t)active;
        k.has_const = (uint8_t)has_const;
        k.data = (int)kgroups.size();
        kgroups.push_back(G);
      }
      kops.push_back(k);
    }
    while (cur_phase < nph - 1) {
      if (cur_phase >= 0) h.phases[cur_phase].op_end = (int16_t)kops.size();
      cur_phase++;
      h.phases[cur_phase].op_begin = (int16_t)kops.size();
    }
    h.phases[nph - 1].op_end = (int16_t)kops.size();
    h.n_ops = (int)kops.size();
    h.n_shapes = (int)kshapes.size();
    h.n_groups = (int)kgroups.size();
    // OP_HU leaves a factor sqrt2 per gate: restore 2^{-n_hu/2} at the store
    const double hs = std::ldexp(1.0, -(n_hu / 2)) * ((n_hu & 1) ? 0.70710678118654752440 : 1.0);
    h.scale = hs * lam_total.real();
    h.scale_im = hs * lam_total.imag();
    if (h.n_shapes > kMaxShapes) {
      err = "internal: too many diagonal shapes in one pass";
      return QS_EINVAL;
    }
  }
  Blob B;
  B.put(&h, 1);
  h.off_ops = (uint32_t)B.put(kops.data(), kops.size());
  h.off_groups = (uint32_t)B.put(kgroups.data(), kgroups.size());
  h.off_shapes = (uint32_t)B.put(kshapes.data(), kshapes.size());
  h.off_terms = (uint32_t)B.put(kterms.data(), kterms.size());
  h.off_pool = (uint32_t)B.put(pool.data(), pool.size());
  B.align(16);
  h.total_bytes = (uint32_t)B.b.size();
  memcpy(B.b.data(), &h, sizeof h);
  out.swap(B.b);
  return QS_OK;
}

// ------------------------------------------------------------ JSON
static const char* kname(int k) {
  switch (k) {
    case KK_CHUNK: return "K1_chunk";
    case KK_DENSE: return "K2_dense";
    case KK_DIAG: return "K3_diag";
    case KK_SMALL: return "small";
    default: return "?";
  }
}

std::string plan_to_json(const Plan& plan, bool detail) {
  std::ostringstream o;
  const PlanStats& s = plan.stats;
  o << "{\"n\":" << plan.n << ",\"n_global\":" << plan.n_global << ",\"nl\":" << plan.nl;
  o << ",\"stats\":{\"n_gates_in\":" << s.n_gates_in << ",\"n_passes\":" << s.n_passes
    << ",\"n_chunk\":" << s.n_chunk << ",\"n_dense\":" << s.n_dense << ",\"n_diag\":" << s.n_diag
    << ",\"n_small\":" << s.n_small << ",\"n_expand\":" << s.n_expand
    << ",\"n_swaps\":" << s.n_swaps << ",\"n_fusable_swaps\":" << s.n_fusable_swaps << ",\"n_sub_gates\":" << s.n_sub_gates
    << ",\"n_fused_diag\":" << s.n_fused_diag << ",\"paper_updates\":" << s.paper_updates
    << ",\"naive_updates\":" << s.naive_updates << ",\"bytes_hbm\":" << s.bytes_hbm
    << ",\"bytes_nvlink\":" << s.bytes_nvlink << ",\"n_l2_groups\":" << s.n_l2_groups
    << ",\"bytes_hbm_l2\":" << s.bytes_hbm_l2 << ",\"booster_rounds\":[";
  for (size_t r = 0; r < s.booster_rounds.size(); r++) {
    o << (r ? "," : "") << "[";
    for (size_t g = 0; g < s.booster_rounds[r].size(); g++)
      o << (g ? "," : "") << s.booster_rounds[r][g];
    o << "]";
  }
  o << "]},\"subs\":[";
  for (size_t i = 0; i < plan.subs.size(); i++)
    o << (i ? "," : "") << "{\"nq\":" << plan.subs[i].nq << ",\"lo\":" << plan.subs[i].lo << "}";
  o << "],\"map_in\":[";
  for (size_t i = 0; i < plan.map_in.size(); i++) o << (i ? "," : "") << plan.map_in[i];
  o << "],\"map_out\":[";
  for (size_t i = 0; i < plan.map_out.size(); i++) o << (i ? "," : "") << plan.map_out[i];
  o << "],\"steps\":[";
  for (size_t i = 0; i < plan.steps.size(); i++) {
    const Step& st = plan.steps[i];
    o << (i ? "," : "") << "{";
    switch (st.type) {
      case Step::INIT_BASIS:
        o << "\"type\":\"init_basis\",\"basis\":\"" << st.basis << "\"";
        break;
      case Step::SUB_INIT:
        o << "\"type\":\"sub_init\",\"buf\":" << st.buf << ",\"basis\":\"" << st.basis << "\"";
        break;
      case Step::SUB_MERGE:
        o << "\"type\":\"sub_merge\",\"buf\":" << st.buf << ",\"a\":" << st.src_a
          << ",\"b\":" << st.src_b;
        break;
      case Step::EXPAND:
        o << "\"type\":\"expand\",\"bufs\":[";
        for (size_t k = 0; k < st.exp_bufs.size(); k++) o << (k ? "," : "") << st.exp_bufs[k];
        o << "],\"exp_lo\":[";
        for (size_t k = 0; k < st.exp_lo.size(); k++) o << (k ? "," : "") << st.exp_lo[k];
        o << "],\"exp_len\":[";
        for (size_t k = 0; k < st.exp_len.size(); k++) o << (k ? "," : "") << st.exp_len[k];
        o << "]";
        break;
      case Step::SWAP:
      case Step::PERMUTE:
        o << "\"type\":\"" << (st.type == Step::SWAP ? "swap" : "permute") << "\",\"j\":" << st.j
          << ",\"gpos\":[";
        for (size_t k = 0; k < st.gpos.size(); k++) o << (k ? "," : "") << st.gpos[k];
        o << "],\"lpos\":[";
        for (size_t k = 0; k < st.lpos.size(); k++) o << (k ? "," : "") << st.lpos[k];
        o << "]";
        if (st.type == Step::SWAP) o << ",\"fusable\":" << (st.fusable ? "true" : "false");
        break;
      case Step::PASS: {
        const PassPlan& p = st.pass;
        o << "\"type\":\"pass\",\"kernel\":\"" << kname(p.kernel) << "\",\"buf\":" << p.buf
          << ",\"nl\":" << p.nl << ",\"src_mode\":" << p.src_mode << ",\"x_j\":" << p.x_j
          << ",\"x_split\":" << p.x_split << ",\"pull_j\":" << p.pull_j << ",\"pull_z\":" << p.pull_z << ",\"l2_grp\":" << p.l2_grp
          << ",\"x_pos\":[" << (p.x_j > 0 ? std::to_string(p.x_pos[0]) : "")
          << (p.x_j > 1 ? "," + std::to_string(p.x_pos[1]) : "") << (p.x_j > 2 ? "," + std::to_string(p.x_pos[2]) : "")
          << "]"
          << ",\"cpos\":[";
        for (size_t k = 0; k < p.cpos.size(); k++) o << (k ? "," : "") << p.cpos[k];
        o << "],\"opos\":[";
        for (size_t k = 0; k < p.opos.size(); k++) o << (k ? "," : "") << p.opos[k];
        o << "],\"basis\":\"" << p.basis << "\",\"exp_bufs\":[";
        for (size_t k = 0; k < p.exp_bufs.size(); k++) o << (k ? "," : "") << p.exp_bufs[k];
        o << "],\"exp_lo\":[";
        for (size_t k = 0; k < p.exp_lo.size(); k++) o << (k ? "," : "") << p.exp_lo[k];
        o << "],\"exp_len\":[";
        for (size_t k = 0; k < p.exp_len.size(); k++) o << (k ? "," : "") << p.exp_len[k];
        o << "],\"phase_regs\":[";
        for (size_t k = 0; k < p.phase_regs.size(); k++) {
          o << (k ? "," : "") << "[";
          for (size_t q = 0; q < p.phase_regs[k].size(); q++) o << (q ? "," : "") << p.phase_regs[k][q];
          o << "]";
        }
        o << "],\"phases\":" << p.phase_regs.size() << ",\"ops\":[";
        for (size_t k = 0; k < p.ops.size(); k++) {
          const POp& op = p.ops[k];
          o << (k ? "," : "") << "{\"t\":\"" << (op.type == POp::DIAG ? "diag" : "dense")
            << "\",\"n_src\":" << op.n_src;
          if (op.type == POp::DIAG) {
            o << ",\"n_mono\":" << op.mono.size();
            if (detail) {
              o << ",\"mono\":[";
              for (size_t q = 0; q < op.mono.size(); q++)
                o << (q ? "," : "") << "[\"" << op.mono[q].mask << "\",\"" << op.mono[q].coeff << "\"]";
              o << "]";
            }
          } else {
            o << ",\"tpos\":[";
            for (size_t q = 0; q < op.tpos.size(); q++) o << (q ? "," : "") << op.tpos[q];
            o << "],\"cmask\":\"" << op.cmask << "\"";
            if (detail) {
              char b[64];
              o << ",\"mat\":[";
              for (size_t q = 0; q < op.mat.size(); q++) {
                snprintf(b, sizeof b, "%.17g,%.17g", op.mat[q].real(), op.mat[q].imag());
                o << (q ? "," : "") << b;
              }
              o << "]";
            }
          }
          o << "}";
        }
        o << "]";
        break;
      }
    }
    o << "}";
  }
  o << "]}";
  return o.str();
}

}  // namespace qs
