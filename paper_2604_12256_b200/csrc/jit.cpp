// jit.cpp -- per-pass specialisation of the chunk / dense / diagonal kernels
// (K1/K2/K3) with NVRTC for sm_100a.
//
// The planner's pass descriptor (KPass blob) fixes the pass STRUCTURE: chunk
// positions, register layouts, op sequence, register bits, controls, the
// diagonal shape masks.  This file turns that structure into straight-line
// CUDA: every register index, address offset, swizzled shared-memory slot
// and control test becomes a compile-time constant, X gates become register
// renames, and the op dispatch of the interpreter kernels (kernels.cu)
// disappears.  NUMBERS (matrix entries, phase coefficients, constant tables,
// sub-state pointers, the basis index) are still read from the descriptor at
// run time, so a circuit with new angles reuses the compiled kernel.
//
// Compiled cubins are cached in memory (per device) and on disk
// (QS_JIT_CACHE, default <libdir>/jit_cache) keyed by a hash of the source.
// The driver API is reached through cudaGetDriverEntryPoint (no link-time
// libcuda dependency, so the library still loads on a CPU-only host).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <map>
#include <thread>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "planner.hpp"
#include "qs_internal.hpp"

namespace qs {

// ------------------------------------------------------------- source gen
static const char* kPrelude = R"PRELUDE(
typedef unsigned long long u64;
typedef unsigned int u32;
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cmac(double2 acc, double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)),
                      fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
// exp(2 pi i t / 2^64); polynomials: fdlibm's __kernel_sin/__kernel_cos
// coefficients (see kernels.cu)
__device__ __forceinline__ double2 cis_turns(u64 t) {
  const u64 q = (t + (1ull << 61)) >> 62;
  const long long f = (long long)(t - (q << 62));
  const double x = (double)f * 3.4061215800865545e-19;
  const double z = x * x;
  const double s = fma(x * z,
      fma(z, fma(z, fma(z, fma(z, fma(z, 1.58969099521155010221e-10,
      -2.50507602534068634195e-08), 2.75573137070700676789e-06),
      -1.98412698298579493134e-04), 8.33333333332248946124e-03),
      -1.66666666666666324348e-01), x);
  const double c = fma(z * z,
      fma(z, fma(z, fma(z, fma(z, fma(z, -1.13596475577881948265e-11,
      2.08757232129817482790e-09), -2.75573143513906633035e-07),
      2.48015872894767294178e-05), -1.38888888888741095749e-03),
      4.16666666666666019037e-02), fma(-0.5, z, 1.0));
  switch ((int)(q & 3)) {
    case 0: return make_double2(c, s);
    case 1: return make_double2(-s, c);
    case 2: return make_double2(-c, -s);
    default: return make_double2(s, -c);
  }
}
// exp(2 pi i t / 2^64) = T[k] * exp(i x): k = nearest 1/256 turn (T in shared
// memory, filled with cis_turns), |x| <= pi/256; the polynomials' first
// omitted terms are x^7/7! and x^8/8! (< 1e-17).
__device__ __forceinline__ double2 cis_tab(u64 t, const double2* __restrict__ T) {
  const u64 k = (t + (1ull << 55)) >> 56;
  const long long f = (long long)(t - (k << 56));
  const double x = (double)f * 3.4061215800865545e-19;
  const double z = x * x;
  const double s = x * fma(z, fma(z, 8.3333333333333333e-03, -1.6666666666666667e-01), 1.0);
  const double c = fma(z, fma(z, fma(z, -1.3888888888888889e-03, 4.1666666666666667e-02), -0.5), 1.0);
  const double2 b = T[k & 255];
  return make_double2(fma(b.x, c, -b.y * s), fma(b.x, s, b.y * c));
}
__device__ __forceinline__ int swz(int c) {
  return c ^ (((c >> 3) ^ (c >> 6) ^ (c >> 9) ^ (c >> 12)) & 7);
}
__device__ __forceinline__ u32 sa(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* b, u32 n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(u64* b, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* b, u32 parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
               :: "r"(sa(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(sa(dst)), "l"(src) : "memory");
}
// the mbarrier sees one arrival once all of this thread's prior cp.async land
__device__ __forceinline__ void cp_async_mbar_arrive(u64* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(sa(b)) : "memory");
}
// exact unit (1, i, -1, -i) -> quarter index 0..3 (integer bit tests)
__device__ __forceinline__ u32 qof(double2 e) {
  const u64 bx = (u64)__double_as_longlong(e.x), by = (u64)__double_as_longlong(e.y);
  const u32 sw = (bx << 1) == 0ull ? 1u : 0u;
  const u32 ng = (u32)((sw ? by : bx) >> 63);
  return sw | (ng << 1);
}
// a * i^q by sign/swap of the bit patterns (no FP64 instruction)
__device__ __forceinline__ double2 rotq(double2 a, u32 q) {
  const u64 ax = (u64)__double_as_longlong(a.x), ay = (u64)__double_as_longlong(a.y);
  const bool s = (q & 1u) != 0u;
  const u64 sg = (u64)((q >> 1) & 1u) << 63;
  const u64 nx = (s ? (ay ^ 0x8000000000000000ull) : ax) ^ sg;
  const u64 ny = (s ? ax : ay) ^ sg;
  return make_double2(__longlong_as_double((long long)nx), __longlong_as_double((long long)ny));
}
// barrier of one 256-thread chunk group (named barrier 1 + group)
__device__ __forceinline__ void gbar(u32 id) { asm volatile("bar.sync %0, 256;" :: "r"(id) : "memory"); }
)PRELUDE";

static int host_swz(int c) { return c ^ (((c >> 3) ^ (c >> 6) ^ (c >> 9) ^ (c >> 12)) & 7); }

// Kernel parameters are limited to 32764 bytes (CUDA 12.1+, sm_70+); the
// pool is passed by value up to this many doubles (else read from the blob).
static const size_t kMaxParamPool = 3900;

static const int kPairA[6] = {0, 0, 0, 1, 1, 2};
static const int kPairB[6] = {1, 2, 3, 2, 3, 3};

namespace {
// The per-chunk table of a specialised pass (TabCols).  A diagonal slot (a
// fast diagonal's E0 or E_k, a sum of shapes) whose chunk-dependent shapes
// all have an empty thread mask is chunk-only up to a per-thread constant:
// it becomes a cis column (its sincos is taken once per chunk by the table
// kernel; the chunk-independent shapes with an empty thread mask are folded
// in), and its thread-dependent constant shapes are hoisted.  Every other
// chunk-dependent shape is an angle column.  slot_col: (op index * 32 + R)
// -> cis column.  false: nothing chunk-dependent, or over the limits.
bool table_columns(const unsigned char* blob, TabCols* v, std::map<int, int>* slot_col) {
  KPass h;
  memcpy(&h, blob, sizeof h);
  memset(v, 0, sizeof *v);
  if (getenv("QS_JIT_NOTAB")) return false;  // tests: force the in-kernel level-1 sums
  const KOp* ops = reinterpret_cast<const KOp*>(blob + h.off_ops);
  const KGroup* groups = reinterpret_cast<const KGroup*>(blob + h.off_groups);
  const KShape* shapes = reinterpret_cast<const KShape*>(blob + h.off_shapes);
  const KTerm* terms = reinterpret_cast<const KTerm*>(blob + h.off_terms);
  auto vary = [&](int j) {
    for (int q = shapes[j].term_begin; q < shapes[j].term_end; q++)
      if (terms[q].ncmask) return true;
    return false;
  };
  std::vector<int> ang;
  std::vector<std::vector<int>> cis;
  const int nph = h.kernel == KK_CHUNK ? h.n_phases : 1;
  for (int p = 0; p < nph; p++)
    for (int i = h.phases[p].op_begin; i < h.phases[p].op_end; i++) {
      const KOp& op = ops[i];
      if (op.type == OP_DIAG) {
        const KGroup& G = groups[op.data];
        for (int j = G.rbeg[0]; j < G.rbeg[kNReg]; j++)
          if (vary(j)) ang.push_back(j);
      } else if (op.type == OP_DIAGF) {
        const KGroup& G = groups[op.data];
        std::vector<int> slots;
        if (op.has_const) slots.push_back(0);
        for (int k = 0; k < kRegBits; k++)
          if (op.sel >> k & 1) slots.push_back(1 << k);
        for (int R : slots) {
          bool any_vary = false, vary_thread = false;
          for (int j = G.rbeg[R]; j < G.rbeg[R + 1]; j++)
            if (vary(j)) any_vary = true, vary_thread |= shapes[j].tmask != 0;
          if (!any_vary) continue;
          if (vary_thread) {
            for (int j = G.rbeg[R]; j < G.rbeg[R + 1]; j++)
              if (vary(j)) ang.push_back(j);
            continue;
          }
          std::vector<int> c;
          for (int j = G.rbeg[R]; j < G.rbeg[R + 1]; j++)
            if (vary(j) || shapes[j].tmask == 0) c.push_back(j);
          if (slot_col) (*slot_col)[i * 32 + R] = (int)cis.size();
          cis.push_back(c);
        }
      }
    }
  std::sort(ang.begin(), ang.end());
  ang.erase(std::unique(ang.begin(), ang.end()), ang.end());
  if (ang.empty() && cis.empty()) return false;
  if ((int)ang.size() > kMaxVaryTab || (int)cis.size() > kMaxTabCis) return false;
  v->n_ang = (int)ang.size();
  for (size_t t = 0; t < ang.size(); t++) v->ang[t] = (int16_t)ang[t];
  v->n_cis = (int)cis.size();
  int nref = 0;
  for (size_t e = 0; e < cis.size(); e++) {
    v->cis_beg[e] = (int16_t)nref;
    for (int j : cis[e]) {
      if (nref == kMaxTabRefs) return false;
      v->cis_shape[nref++] = (int16_t)j;
    }
  }
  v->cis_beg[cis.size()] = (int16_t)nref;
  v->width = ((v->n_ang + 1) & ~1) + 2 * v->n_cis;
  return true;
}

// TMA tensor view of a load pass whose chunk has short contiguous runs
// (l < 5, where per-run bulk copies lose): the shard as a <= 5-d float64
// tensor whose dims are the runs of consecutive positions (chunk and
// non-chunk runs alternate; runs longer than 8 bits split), dim 0 being the
// low chunk run in doubles.  One cp.async.bulk.tensor per chunk, box = the
// chunk dims in full and 1 along the others; the smem image is the linear
// chunk-index layout, like the bulk stage.
// More runs than 5 dims (round 2): dims 0-3 are the lowest four runs and
// dim 4 ("rest") spans every higher position with box 1; the chunk positions
// inside it (`extra`) are enumerated by 2^|extra| <= 32 copies per chunk (one
// per lane), copy e landing at e * 2^(covered chunk bits) -- still the linear
// chunk-index layout (chunk bits are numbered by ascending position).
struct TPlan {
  int rank = 0;
  int pos[5], len[5];
  bool chunk[5];
  int n_extra = 0;
  int extra[kChunkBits];     // chunk positions inside the rest dim
  int covered = kChunkBits;  // chunk bits covered by one copy
};
bool tensor_plan(const KPass& h, TPlan* t) {
  if (getenv("QS_JIT_NOTENSOR")) return false;  // A/B knob
  static const int max_copies = getenv("QS_JIT_TENSOR_COPIES") ? atoi(getenv("QS_JIT_TENSOR_COPIES")) : 64;
  u64 cm = 0;
  for (int c = 0; c < kChunkBits; c++) cm |= 1ull << h.cpos[c];
  int l = 0;
  while (l < kChunkBits && h.cpos[l] == l) l++;
  if (l < 3 || l >= 5) return false;
  std::vector<int> rp, rl;
  std::vector<bool> rc;
  int p = 0;
  while (p < h.nl) {
    const bool in = (cm >> p) & 1;
    int q = p;
    while (q < h.nl && (((cm >> q) & 1) != 0) == in && (!in || q - p < 8)) q++;
    rp.push_back(p);
    rl.push_back(q - p);
    rc.push_back(in);
    p = q;
  }
  if (!rc[0] || rp[0] != 0 || rl[0] != l) return false;
  t->n_extra = 0;
  t->covered = kChunkBits;
  if (rp.size() <= 5) {
    t->rank = (int)rp.size();
    for (int d = 0; d < t->rank; d++) t->pos[d] = rp[d], t->len[d] = rl[d], t->chunk[d] = rc[d];
    return true;
  }
  if (max_copies <= 1) return false;
  t->rank = 5;
  t->covered = 0;
  for (int d = 0; d < 4; d++) {
    t->pos[d] = rp[d], t->len[d] = rl[d], t->chunk[d] = rc[d];
    if (rc[d]) t->covered += rl[d];
  }
  t->pos[4] = rp[4];
  t->len[4] = h.nl - rp[4];
  t->chunk[4] = false;
  for (int q = rp[4]; q < h.nl; q++)
    if (cm >> q & 1) t->extra[t->n_extra++] = q;
  return (1 << t->n_extra) <= max_copies && t->len[4] <= 32;
}

struct Gen {
  std::ostringstream o;
  const KPass& h;
  const KOp* ops;
  const KGroup* groups;
  const KShape* shapes;
  const KTerm* terms;
  const double* pool;  // host copy of the matrix pool (structure detection)
  // per-chunk table (qs_kshape_table): columns and diagonal slot -> cis column
  TabCols tc;
  std::map<int, int> slot_col;
  bool use_vtab = false;
  size_t sc_cis = 0;  // u64 offset of the cis columns in a shape-sum copy
  // table rows of <= 32 entries are kept per warp (each warp loads its next
  // chunk's row, lane t holding entry t, published with __syncwarp): no
  // CTA-wide barrier per chunk.  ang_col: shape -> its angle column.
  bool warp_tab = false;
  std::map<int, int> ang_col;
  std::string sref(int j) const {
    if (warp_tab) {
      auto it = ang_col.find(j);
      if (it != ang_col.end()) return "wrow[" + std::to_string(it->second) + "]";
    }
    return "scoef[" + std::to_string(j) + "]";
  }
  int nm[kNReg];  // register slot -> variable index (X renames)
  // per-thread factors that multiply every register, not yet applied:
  // folded into the next full-width diagonal's E0, else applied at the store
  std::vector<std::string> pend_c;
  bool pend_scale = false;
  int sc_kind = 0, sc_sx = 1, sc_sy = 1;  // unit part of the pass scale (see build)
  double sc_mag = 1.0;                     // its real magnitude (folded like the H scale)
  // pass constants (matrices, CK tables) as a by-value kernel parameter:
  // FP64 instructions then read them as constant-bank operands
  bool param_pool = false;
  std::string pv(int off) const {
    return (param_pool ? "P.v[" : "pool[") + std::to_string(off) + "]";
  }
  // The CK register-pair phase tables of fast diagonals live in a per-CTA
  // shared-memory copy (cks[], filled once): as loop-invariant parameter
  // loads the compiler hoists them into registers, which spills the
  // 16-amplitude register tile (QFT-30 write-only pass: 88 B of spills,
  // none with the table in shared memory).
  std::map<int, int> ck_slot;  // complex pool offset (doubles) -> cks index
  bool ck_smem = false;        // single-layout passes (multi-layout ones keep
                               // constant-bank operands: no spills there, and
                               // the extra loads would cost registers)
  std::string ckv(int off) {
    if (!ck_smem) return "make_double2(" + pv(off) + ", " + pv(off + 1) + ")";
    auto it = ck_slot.find(off);
    int k;
    if (it == ck_slot.end()) {
      k = (int)ck_slot.size();
      ck_slot[off] = k;
    } else {
      k = it->second;
    }
    return "cks[" + std::to_string(k) + "]";
  }
  // Dense-op matrix entries from a per-CTA shared-memory copy (csm[]) instead
  // of constant-bank operands: QS_JIT_MSMEM=1 (A/B knob; measured worse).
  std::map<int, int> m_slot;   // pool offset (doubles) -> csm index
  bool mat_smem = false;
  std::string mat_ref(int off) {
    if (!mat_smem) return pv(off);
    auto it = m_slot.find(off);
    int k;
    if (it == m_slot.end()) {
      k = (int)m_slot.size();
      m_slot[off] = k;
    } else {
      k = it->second;
    }
    return "csm[" + std::to_string(k) + "]";
  }
  int n_mat_doubles() const {  // upper bound of the register ops' matrix entries
    int c = 0;
    for (int i = 0; i < h.n_ops; i++) {
      const int t = ops[i].type;
      c += t == OP_D1 ? 8 : t == OP_D2 ? 32 : t == OP_D3 ? 128 : 0;
    }
    return c;
  }
  int n_ck_entries() const {  // upper bound, before generation
    int c = 0;
    for (int i = 0; i < h.n_ops; i++)
      if (ops[i].type == OP_DIAGF && groups[ops[i].data].ck_off >= 0) c += kNReg;
    return c;
  }
  // loop-invariant per-thread values hoisted out of the chunk loop
  std::ostringstream pre;
  int n_hoist = 0;
  int max_hoist = 0;
  size_t hz_off = 0;  // byte offset of the hoisted-value slots in shared memory
  int nthreads = kThreads;  // threads per CTA (chunk groups x 256)
  // fast-diagonal product scheme: 0 two-level, 1 Gray walk (default: best or
  // tied on QFT/QAOA/diag-chain A/B runs on one box), 2 product tree
  static int diag_scheme() {
    const char* e = getenv("QS_JIT_DIAGPROD");
    return e ? atoi(e) : 1;
  }
  int n_table = 0;          // sincos evaluations left in the loop (need the table)
  bool hoist_capped = false;  // a loop-invariant sincos did not fit in smem
  bool table_free = false;    // generation assumes no table: 4 KB more for hoists
  bool bad_op = false;        // an op type the generator does not know
  int variant = 0;            // chunk refill engine (JitVariant)
  int grid_mult = 1;          // the grid must be a multiple of this (hoisted expand gathers)
  // Member of a co-scheduled run (two-level blocking): the
  // pass is emitted as a device function qs_body() (the run kernel deals its
  // CTAs to the passes of the run); run_wait: every chunk load first waits
  // until the previous pass has stored its whole 2^(12+run_sb)-amplitude
  // block (qs_fin counter); run_signal: every chunk's store is counted on
  // its block (qs_fout) for the next pass.
  bool run_mode = false, run_wait = false, run_signal = false;
  // run_throttle (first member): chunk processing waits until the last
  // member is done with the block qs_lag blocks back, so the run's blocks
  // stay within L2 instead of the first pass racing ahead
  bool run_throttle = false;
  int run_sb = 0;             // chunk-id bits inside one block of the run
  std::string run_wait_of(const std::string& c) const {
    return run_wait ? "qs_wait(qs_fin + ((" + c + ") >> " + std::to_string(run_sb) + "), " +
                          std::to_string(1 << run_sb) + "u); "
                    : "";
  }
  // Chunk groups per CTA: multi-layout load passes (compute-heavy between
  // their load and their store) run two groups over three buffers so a load
  // is always in flight; the others run one group (two CTAs per SM, one
  // buffer refilled right after its last read).  QS_JIT_GROUPS=1|2 forces.
  static int groups_per_cta(bool pipe, int nlay) {
    const char* e = getenv("QS_JIT_GROUPS");
    if (e && (atoi(e) == 1 || atoi(e) == 2)) return atoi(e);
    // write-only passes: two groups per CTA too (QFT-30's K2 3.73 -> 3.37 ms:
    // the groups share the CTA's hoisted per-thread values); QS_JIT_WO_GROUPS
    // is the A/B knob
    const char* w = getenv("QS_JIT_WO_GROUPS");
    if (!pipe) return (w && atoi(w) == 1) ? 1 : 2;
    return nlay > 1 ? 2 : 1;
  }
  Gen(const KPass& hh, const unsigned char* blob)
      : h(hh),
        ops(reinterpret_cast<const KOp*>(blob + hh.off_ops)),
        groups(reinterpret_cast<const KGroup*>(blob + hh.off_groups)),
        shapes(reinterpret_cast<const KShape*>(blob + hh.off_shapes)),
        terms(reinterpret_cast<const KTerm*>(blob + hh.off_terms)),
        pool(reinterpret_cast<const double*>(blob + hh.off_pool)) {
    for (int r = 0; r < kNReg; r++) nm[r] = r;
    use_vtab = table_columns(blob, &tc, &slot_col);
    // (not for diagonal-only passes: there the per-chunk barrier keeps the
    // CTA's warps on one chunk, which the streaming stores prefer -- A/B:
    // QFT-30 K2 4.50 -> 3.85 ms, RZZ-30 K3 3.33 -> 3.72 ms with warp rows)
    warp_tab = use_vtab && tc.width <= 32 && hh.kernel != KK_DIAG && !getenv("QS_JIT_CTATAB");
    for (int t = 0; t < tc.n_ang; t++) ang_col[tc.ang[t]] = t;
  }
  std::string A(int r) const { return "a" + std::to_string(nm[r]); }

  // Register layouts: the pass's phases, plus (when the last one would store
  // with lanes off the low chunk bits) a store layout reached by one more
  // shared-memory exchange.
  std::vector<KPhase> L;
  // number of consecutive low chunk bits (0, 1, ...) held in registers: a
  // thread then owns 2^run contiguous amplitudes of every register group
  static int low_run(const KPhase& k) {
    int run = 0;
    for (;;) {
      bool has = false;
      for (int i = 0; i < kRegBits; i++)
        if (k.reg_c[i] == run) has = true;
      if (!has) return run;
      run++;
    }
  }
  // low_run of the store: consecutive lowest output positions that are
  // register bits of layout k under the pass's output relabel (opos)
  int low_run_out(const KPhase& k) const {
    int run = 0;
    for (;;) {
      bool has = false;
      for (int i = 0; i < kRegBits; i++)
        if (h.opos[k.reg_c[i]] == h.cpos[run]) has = true;
      if (!has || run + 1 >= kChunkBits) return run + (has ? 1 : 0);
      run++;
    }
  }
  static KPhase default_layout() {
    KPhase k;
    memset(&k, 0, sizeof k);
    for (int i = 0; i < kRegBits; i++) k.reg_c[i] = (int8_t)(kChunkBits - kRegBits + i);
    for (int i = 0; i < kLogT; i++) k.thr_c[i] = (int8_t)i;
    return k;
  }
  u64 reg_phys(int p, int r, bool out) const {
    const int8_t* pos = out ? h.opos : h.cpos;
    u64 o = 0;
    for (int k = 0; k < kRegBits; k++)
      if (r >> k & 1) o |= 1ull << pos[L[p].reg_c[k]];
    return o;
  }
  int reg_slot(int p, int r) const {
    int c = 0;
    for (int k = 0; k < kRegBits; k++)
      if (r >> k & 1) c |= 1 << L[p].reg_c[k];
    return host_swz(c);
  }
  std::string tphys_expr(int p, bool out) const {
    const int8_t* pos = out ? h.opos : h.cpos;
    std::string s = "(0ull";
    for (int i = 0; i < kLogT; i++)
      s += " | ((u64)((tid >> " + std::to_string(i) + ") & 1u) << " +
           std::to_string(pos[L[p].thr_c[i]]) + ")";
    return s + ")";
  }
  std::string tc_expr(int p) const {
    std::string s = "(0";
    for (int i = 0; i < kLogT; i++)
      s += " | (int)(((tid >> " + std::to_string(i) + ") & 1u) << " +
           std::to_string(L[p].thr_c[i]) + ")";
    return s + ")";
  }
  static std::string hex(double d) {
    char b[64];
    snprintf(b, sizeof b, "%a", d);
    return b;
  }
  static std::string u(u64 v) { return std::to_string(v) + "ull"; }

  void pred(const KOp& op, int p) {
    if (op.ncm)
      o << "    const bool tp = ((cphys | tp" << p << ") & " << u(op.ncm) << ") == " << u(op.ncm)
        << ";\n    if (tp) {\n";
    else
      o << "    {\n";
  }

  void dense(const KOp& op, int p, int W, const int* bits) {
    const int D = 1 << W;
    int tm = 0;
    for (int b = 0; b < W; b++) tm |= 1 << bits[b];
    o << "  { // dense " << W << "q\n";
    pred(op, p);
    // Entry structure (zero / real / imaginary / complex) is baked into the
    // code -- e.g. RX, RY, SX need 4 FP64 per output instead of 8; values stay
    // run-time data.
    const double* mv = pool + op.data;
    // 0 zero, 1 real, 2 imag, 3 complex; exact units (unit-scaled ops,
    // encode_pass): 4 +1, 5 -1, 6 +i, 7 -i -- additions only
    std::vector<int> kind(D * D);
    for (int i = 0; i < D * D; i++) {
      const double re = mv[2 * i], im = mv[2 * i + 1];
      kind[i] = (re == 0.0 && im == 0.0) ? 0 : (im == 0.0 && re == 1.0) ? 4 : (im == 0.0 && re == -1.0) ? 5
              : (re == 0.0 && im == 1.0) ? 6 : (re == 0.0 && im == -1.0) ? 7
              : (im == 0.0) ? 1 : (re == 0.0) ? 2 : 3;
      const std::string e = std::to_string(i);
      if (W <= 2) {
        if (kind[i] == 1 || kind[i] == 3) o << "    const double mr" << e << " = " << mat_ref(op.data + 2 * i) << ";\n";
        if (kind[i] == 2 || kind[i] == 3) o << "    const double mi" << e << " = " << mat_ref(op.data + 2 * i + 1) << ";\n";
      }
    }
    auto mr = [&](int i) { return (W <= 2) ? "mr" + std::to_string(i) : mat_ref(op.data + 2 * i); };
    auto mi = [&](int i) { return (W <= 2) ? "mi" + std::to_string(i) : mat_ref(op.data + 2 * i + 1); };
    for (int base = 0; base < kNReg; base++) {
      if (base & tm) continue;
      if ((base & (int)op.rcm) != (int)op.rcm) continue;
      int idx[16];
      for (int i = 0; i < D; i++) {
        int r = base;
        for (int b = 0; b < W; b++)
          if (i >> b & 1) r |= 1 << bits[b];
        idx[i] = r;
      }
      o << "    {\n";
      for (int i = 0; i < D; i++) o << "      const double2 v" << i << " = " << A(idx[i]) << ";\n";
      for (int r = 0; r < D; r++) {
        std::string re, im;
        auto add = [](std::string& acc, const std::string& t, bool neg) {
          if (acc.empty()) acc = neg ? "-(" + t + ")" : t;
          else acc += (neg ? " - " : " + ") + t;
        };
        for (int c = 0; c < D; c++) {
          const int i = r * D + c;
          const std::string v = "v" + std::to_string(c);
          switch (kind[i]) {
            case 1:
              add(re, mr(i) + " * " + v + ".x", false);
              add(im, mr(i) + " * " + v + ".y", false);
              break;
            case 2:
              add(re, mi(i) + " * " + v + ".y", true);
              add(im, mi(i) + " * " + v + ".x", false);
              break;
            case 3:
              add(re, mr(i) + " * " + v + ".x", false);
              add(re, mi(i) + " * " + v + ".y", true);
              add(im, mr(i) + " * " + v + ".y", false);
              add(im, mi(i) + " * " + v + ".x", false);
              break;
            case 4:  // +1
              add(re, v + ".x", false);
              add(im, v + ".y", false);
              break;
            case 5:  // -1
              add(re, v + ".x", true);
              add(im, v + ".y", true);
              break;
            case 6:  // +i: i (x + iy) = -y + ix
              add(re, v + ".y", true);
              add(im, v + ".x", false);
              break;
            case 7:  // -i
              add(re, v + ".y", false);
              add(im, v + ".x", true);
              break;
            default:
              break;
          }
        }
        if (re.empty()) re = "0.0";
        if (im.empty()) im = "0.0";
        o << "      " << A(idx[r]) << " = make_double2(" << re << ", " << im << ");\n";
      }
      o << "    }\n";
    }
    o << "    }\n  }\n";
  }

  void hadamard(const KOp& op, int p, bool norm) {
    const int K = op.sel;
    o << "  { // H" << (norm ? "" : "u") << "\n";
    pred(op, p);
    // The first unnormalised H of a pass (uncontrolled: touches every
    // register) also applies the pass's whole 2^{-n/2} scale.
    std::string f;
    if (norm) f = "0x1.6a09e667f3bcdp-1";
    else if (pend_scale && op.rcm == 0 && op.ncm == 0) {
      f = hex(sc_mag);
      pend_scale = false;
    }
    for (int r = 0; r < kNReg; r++) {
      if (r >> K & 1) continue;
      if ((r & (int)op.rcm) != (int)op.rcm) continue;
      const int r1 = r | (1 << K);
      o << "      { const double2 x = " << A(r) << ", y = " << A(r1) << ";\n";
      if (!f.empty()) {
        o << "        " << A(r) << " = make_double2((x.x + y.x) * " << f << ", (x.y + y.y) * " << f << ");\n";
        o << "        " << A(r1) << " = make_double2((x.x - y.x) * " << f << ", (x.y - y.y) * " << f << "); }\n";
      } else {
        o << "        " << A(r) << " = make_double2(x.x + y.x, x.y + y.y);\n";
        o << "        " << A(r1) << " = make_double2(x.x - y.x, x.y - y.y); }\n";
      }
    }
    o << "    }\n  }\n";
  }

  void pauli_x(const KOp& op, int p) {
    const int K = op.sel;
    if (op.ncm == 0 && op.rcm == 0) {  // pure register rename: no instructions
      for (int r = 0; r < kNReg; r++)
        if (!(r >> K & 1)) std::swap(nm[r], nm[r | (1 << K)]);
      return;
    }
    o << "  { // X (controlled)\n";
    pred(op, p);
    for (int r = 0; r < kNReg; r++) {
      if (r >> K & 1) continue;
      if ((r & (int)op.rcm) != (int)op.rcm) continue;
      const int r1 = r | (1 << K);
      o << "      { const double2 x = " << A(r) << "; " << A(r) << " = " << A(r1) << "; " << A(r1)
        << " = x; }\n";
    }
    o << "    }\n  }\n";
  }

  // Per-thread sum of the shapes with register subset R.
  std::string shape_sum(const KGroup& G, int R) const {
    std::string s = "0ull";
    for (int j = G.rbeg[R]; j < G.rbeg[R + 1]; j++) {
      const uint32_t tm = shapes[j].tmask;
      if (tm == 0) s += " + " + sref(j);
      else
        s += " + (((tid & " + std::to_string(tm) + "u) == " + std::to_string(tm) + "u) ? " + sref(j) +
             " : 0ull)";
    }
    return s;
  }

  std::string shape_sum_list(const std::vector<int>& js) const {
    std::string s = "0ull";
    for (int j : js) {
      const uint32_t tm = shapes[j].tmask;
      if (tm == 0) s += " + " + sref(j);
      else
        s += " + (((tid & " + std::to_string(tm) + "u) == " + std::to_string(tm) + "u) ? " + sref(j) +
             " : 0ull)";
    }
    return s;
  }

  // quarter index of an exact unit (1, i, -1, -i -> 0..3); -1 otherwise
  static int unit_q(double re, double im) {
    if (re == 1.0 && im == 0.0) return 0;
    if (re == 0.0 && im == 1.0) return 1;
    if (re == -1.0 && im == 0.0) return 2;
    if (re == 0.0 && im == -1.0) return 3;
    return -1;
  }
  bool quarter_group(const KGroup& G) const {
    static const bool off = getenv("QS_JIT_NOQUARTER") != nullptr;  // A/B knob
    if (off) return false;
    for (int j = G.rbeg[0]; j < G.rbeg[kNReg]; j++)
      for (int q = shapes[j].term_begin; q < shapes[j].term_end; q++)
        if (terms[q].coeff & ((1ull << 62) - 1)) return false;
    if (G.ck_off >= 0)
      for (int r = 0; r < kNReg; r++)
        if (unit_q(pool[G.ck_off + 2 * r], pool[G.ck_off + 2 * r + 1]) < 0) return false;
    return true;
  }
  bool uses_rotq = false;

  void diag_fast(const KOp& op) {
    const KGroup& G = groups[op.data];
    const int L = op.sel;
    const bool hc = op.has_const != 0;
    o << "  { // diagonal (fast)\n";
    // A slot whose shapes have no chunk-dependent term is loop-invariant per
    // thread: its sincos is hoisted out of the chunk loop.
    auto slot_const = [&](int R) {
      for (int j = G.rbeg[R]; j < G.rbeg[R + 1]; j++)
        for (int q = shapes[j].term_begin; q < shapes[j].term_end; q++)
          if (terms[q].ncmask) return false;
      return true;
    };
    // Hoisted values live in per-thread shared-memory slots (registers are
    // the scarce resource: keeping them live across the loop spills).
    // (computed once per thread: the table-free sincos; the 256-entry table,
    // whose random lookups cost shared-memory bank conflicts, is only
    // instantiated for the sincos left inside the chunk loop)
    const int opi = (int)(&op - ops);
    auto evar = [&](int R) -> std::string {
      auto it = use_vtab ? slot_col.find(opi * 32 + R) : slot_col.end();
      if (it != slot_col.end()) {
        // chunk part from the table's cis column, times the hoisted
        // thread-dependent constant part (if any)
        const std::string cv = "cisv[" + std::to_string(it->second) + "]";
        std::vector<int> tpart;
        for (int j = G.rbeg[R]; j < G.rbeg[R + 1]; j++)
          if (shapes[j].tmask != 0) tpart.push_back(j);
        if (tpart.empty()) return cv;
        if (n_hoist < max_hoist) {
          const std::string slot = "hz[" + std::to_string(n_hoist++ * kThreads) + " + tid]";
          pre << "  " << slot << " = cis_turns(" << shape_sum_list(tpart) << ");\n";
          return "cmul(" + slot + ", " + cv + ")";
        }
        hoist_capped = true;
        n_table++;
        return "cmul(cis_tab(" + shape_sum_list(tpart) + ", ctab), " + cv + ")";
      }
      if (slot_const(R)) {
        if (n_hoist < max_hoist) {
          const std::string slot = "hz[" + std::to_string(n_hoist++ * kThreads) + " + tid]";
          pre << "  " << slot << " = cis_turns(" << shape_sum(G, R) << ");\n";
          return slot;
        }
        hoist_capped = true;
      }
      n_table++;
      return "cis_tab(" + shape_sum(G, R) + ", ctab)";
    };
    // Quarter-turn group (every coefficient a multiple of 1/4 turn, e.g. CZ,
    // S, CP(pi/2) chains): every factor is exactly one of 1, i, -1, -i, so the
    // phases are applied with integer sign/swap operations on the amplitude
    // bits (rotq) instead of FP64 complex products.
    if (quarter_group(G)) {
      // the quarter index of a factor: straight from its angle (top 2 bits)
      // when it is summed here, else from the exact unit value
      std::function<std::string(const std::string&)> qv = [&](const std::string& e) -> std::string {
        const std::string tab = "cis_tab(", suf = ", ctab)";
        if (e.compare(0, tab.size(), tab) == 0 && e.size() > tab.size() + suf.size() &&
            e.compare(e.size() - suf.size(), suf.size(), suf) == 0) {
          n_table--;  // no sincos needed
          return "((u32)((" + e.substr(tab.size(), e.size() - tab.size() - suf.size()) + ") >> 62))";
        }
        const std::string cm = "cmul(";
        if (e.compare(0, cm.size(), cm) == 0) {  // cmul(thread part, table column): two exact units
          const size_t c = e.rfind(", ");
          return "(" + qv(e.substr(cm.size(), c - cm.size())) + " + " + qv(e.substr(c + 2, e.size() - c - 3)) + ")";
        }
        return "qof(" + e + ")";
      };
      o << "    u32 Q = 0u;\n";
      if (hc) o << "    Q = " << qv(evar(0)) << ";\n";
      std::vector<int> lbq;
      for (int k = 0; k < kRegBits; k++)
        if (L >> k & 1) {
          lbq.push_back(k);
          o << "    const u32 Q" << k + 1 << " = " << qv(evar(1 << k)) << ";\n";
        }
      uses_rotq = true;
      const int m = (int)lbq.size();
      for (int i = 0; i < (1 << m); i++) {
        const int g = i ^ (i >> 1);
        if (i > 0) {
          const int b = __builtin_ctz(g ^ ((i - 1) ^ ((i - 1) >> 1)));
          o << "    Q = (Q " << ((g >> b & 1) ? "+" : "-") << " Q" << lbq[b] + 1 << ") & 3u;\n";
        }
        int sub = 0;
        for (int t = 0; t < m; t++)
          if (g >> t & 1) sub |= 1 << lbq[t];
        for (int r = 0; r < kNReg; r++) {
          if (!(op.rcm >> r & 1) || (r & L) != sub) continue;
          int cq = 0;
          if (G.ck_off >= 0) cq = unit_q(pool[G.ck_off + 2 * r], pool[G.ck_off + 2 * r + 1]);
          o << "    " << A(r) << " = rotq(" << A(r) << ", Q + " << cq << "u);\n";
        }
      }
      o << "  }\n";
      return;
    }
    if (hc) {
      o << "    double2 E0 = " << evar(0) << ";\n";
      if (op.rcm == 0xFFFFu) {  // multiplies every register: absorb pending factors
        for (const std::string& f : pend_c) o << "    E0 = cmul(E0, " << f << ");\n";
        if (pend_scale)
          o << "    E0 = make_double2(E0.x * " << hex(sc_mag) << ", E0.y * " << hex(sc_mag) << ");\n";
        pend_c.clear();
        pend_scale = false;
      }
    }
    std::vector<int> lb;  // active register bits
    for (int k = 0; k < kRegBits; k++)
      if (L >> k & 1) {
        lb.push_back(k);
        o << "    const double2 E" << k + 1 << " = " << evar(1 << k) << ";\n";
      }
    const int scheme = diag_scheme();
    if (scheme == 1) {
    // Gray-code walk: one running factor F, one multiplication (by E or
    // conj E) per step -- minimal live registers, a 2^m - 1 deep chain.
    {
      bool fid = !hc;  // F is still the identity
      if (hc) o << "    double2 F = E0;\n";
      else o << "    double2 F;\n";
      const int m = (int)lb.size();
      for (int i = 0; i < (1 << m); i++) {
        const int g = i ^ (i >> 1);
        if (i > 0) {
          const int b = __builtin_ctz(g ^ ((i - 1) ^ ((i - 1) >> 1)));
          const std::string e = "E" + std::to_string(lb[b] + 1);
          if (fid) o << "    F = " << e << ";\n", fid = false;
          else o << "    F = " << ((g >> b & 1) ? "cmul" : "cmulc") << "(F, " << e << ");\n";
        }
        int s = 0;
        for (int t = 0; t < m; t++)
          if (g >> t & 1) s |= 1 << lb[t];
        for (int r = 0; r < kNReg; r++) {
          if (!(op.rcm >> r & 1) || (r & L) != s) continue;
          const bool ck = G.ck_off >= 0;
          const std::string c = ck ? ckv(G.ck_off + 2 * r) : "";
          if (fid && !ck) continue;
          if (fid) o << "    " << A(r) << " = cmul(" << A(r) << ", " << c << ");\n";
          else if (!ck) o << "    " << A(r) << " = cmul(" << A(r) << ", F);\n";
          else o << "    " << A(r) << " = cmul(cmul(" << A(r) << ", F), " << c << ");\n";
        }
      }
    }
    } else if (scheme == 2) {
    // Full product tree per register (the compiler shares the prefixes).
    for (int r = 0; r < kNReg; r++) {
      if (!(op.rcm >> r & 1)) continue;
      std::vector<std::string> f;
      if (hc) f.push_back("E0");
      for (int k = 0; k < kRegBits; k++)
        if ((L >> k & 1) && (r >> k & 1)) f.push_back("E" + std::to_string(k + 1));
      if (G.ck_off >= 0) f.push_back(ckv(G.ck_off + 2 * r));
      if (f.empty()) continue;
      std::string g = f[0];
      for (size_t i = 1; i < f.size(); i++) g = "cmul(" + g + ", " + f[i] + ")";
      o << "    " << A(r) << " = cmul(" << A(r) << ", " << g << ");\n";
    }
    } else {
    // Register r takes E0 * prod_{k in r & L} E_{k+1} * CK[r].  Two-level
    // products: the low half of L's bits gives P_l (all subsets, formed once),
    // the high half Q_h = E0 * prod (one scope per subset h), and register r
    // takes Q_h * P_l -- 2-3 cmuls deep (ILP for the FP64 pipe) with only Q_h
    // and the P_l live (a full product tree keeps up to 15 partial products).
    const int m = (int)lb.size();
    const int mlo = m / 2;
    // subset s (bits over lb[0..mlo)) -> expression of P_s ("" = identity)
    std::vector<std::string> P(1 << mlo);
    for (int sl = 1; sl < (1 << mlo); sl++) {
      const int top = 31 - __builtin_clz(sl);
      const std::string e = "E" + std::to_string(lb[top] + 1);
      const int rest = sl & ~(1 << top);
      if (!rest) {
        P[sl] = e;
      } else {
        o << "    const double2 P" << sl << " = cmul(" << P[rest] << ", " << e << ");\n";
        P[sl] = "P" + std::to_string(sl);
      }
    }
    const bool ck = G.ck_off >= 0;
    for (int sh = 0; sh < (1 << (m - mlo)); sh++) {
      o << "    {\n";
      // Q = E0 * prod of the high bits in sh
      std::string Q = hc ? "E0" : "";
      for (int t = 0; t < m - mlo; t++)
        if (sh >> t & 1) {
          const std::string e = "E" + std::to_string(lb[mlo + t] + 1);
          if (Q.empty()) {
            Q = e;
          } else {
            o << "      const double2 Q" << t << " = cmul(" << Q << ", " << e << ");\n";
            Q = "Q" + std::to_string(t);
          }
        }
      for (int sl = 0; sl < (1 << mlo); sl++) {
        int s = 0;
        for (int t = 0; t < mlo; t++)
          if (sl >> t & 1) s |= 1 << lb[t];
        for (int t = 0; t < m - mlo; t++)
          if (sh >> t & 1) s |= 1 << lb[mlo + t];
        std::string f;
        if (Q.empty()) f = P[sl];
        else if (P[sl].empty()) f = Q;
        else f = "cmul(" + Q + ", " + P[sl] + ")";
        for (int r = 0; r < kNReg; r++) {
          if (!(op.rcm >> r & 1) || (r & L) != s) continue;
          const std::string c = ck ? ckv(G.ck_off + 2 * r) : "";
          if (f.empty() && !ck) continue;
          if (f.empty()) o << "      " << A(r) << " = cmul(" << A(r) << ", " << c << ");\n";
          else if (!ck) o << "      " << A(r) << " = cmul(" << A(r) << ", " << f << ");\n";
          else o << "      " << A(r) << " = cmul(" << A(r) << ", cmul(" << f << ", " << c << "));\n";
        }
      }
      o << "    }\n";
    }
    }
    o << "  }\n";
  }

  void diag_general(const KOp& op) {
    const KGroup& G = groups[op.data];
    const int act = op.sel;
    o << "  { // diagonal (general)\n";
    for (int R = 0; R < kNReg; R++) o << "    u64 g" << R << " = " << shape_sum(G, R) << ";\n";
    for (int k = 0; k < kRegBits; k++)
      for (int S = 0; S < kNReg; S++)
        if (S >> k & 1) o << "    g" << S << " += g" << (S ^ (1 << k)) << ";\n";
    for (int S = 0; S < kNReg; S++) {
      if (S & ~act) continue;
      if (S == 0 && !op.has_const) continue;
      o << "    { const double2 e = cis_tab(g" << S << ", ctab);\n";
      n_table++;
      for (int r = 0; r < kNReg; r++)
        if ((r & act) == S) o << "      " << A(r) << " = cmul(" << A(r) << ", e);\n";
      o << "    }\n";
    }
    o << "  }\n";
  }

  // Wide dense op (OP_DW, 5-6 targets; Eq. 3 generalised) on the
  // chunk in shared memory: thread t owns base t >> (k-4) and output rows
  // (t & (2^(k-4)-1))*16 + j; it reads the base's 2^k inputs, accumulates
  // its 16 rows, and writes them after the group barrier.
  void wide(const KOp& op) {
    const int k = op.k, D = 1 << k, g = k - kRegBits;
    int tm = 0;
    for (int i = 0; i < k; i++) tm |= 1 << op.tpos[i];
    o << "    { // wide dense " << k << "q (shared memory)\n";
    o << "      const u32 wb = tid >> " << g << ", wr = tid & " << ((1 << g) - 1) << "u;\n";
    o << "      const int cbase = 0";
    for (int c = 0, bi = 0; c < kChunkBits; c++)
      if (!(tm >> c & 1)) o << " | (int)(((wb >> " << bi++ << ") & 1u) << " << c << ")";
    o << ";\n";
    o << "      const bool wact = ((cphys & " << u(op.ncm) << ") == " << u(op.ncm) << ") && ((cbase & "
      << op.rcm << ") == " << op.rcm << ");\n";
    std::string dep = "";
    for (int i = 0; i < k; i++) dep += " | (((c >> " + std::to_string(i) + ") & 1) << " + std::to_string((int)op.tpos[i]) + ")";
    o << "      const double* __restrict__ wm = pool + " << op.data << " + 2 * (size_t)(wr * " << kNReg * D << ");\n";
    for (int j = 0; j < kNReg; j++) o << "      double2 w" << j << " = make_double2(0.0, 0.0);\n";
    o << "      if (wact) {\n#pragma unroll 2\n        for (int c = 0; c < " << D << "; c++) {\n"
      << "          const double2 v = sch[swz(cbase" << dep << ")];\n";
    for (int j = 0; j < kNReg; j++)
      o << "          w" << j << " = cmac(w" << j << ", __ldg(reinterpret_cast<const double2*>(wm) + " << j * D << " + c), v);\n";
    o << "        }\n      }\n      gbar(1u + grp);\n      if (wact) {\n";
    for (int j = 0; j < kNReg; j++) {
      o << "        { const int c = (int)(wr << 4) + " << j << "; sch[swz(cbase" << dep << ")] = w" << j << "; }\n";
    }
    o << "      }\n    }\n";
  }

  void emit_ops(int p, bool diag_only) {
    const KPhase& ph = h.phases[p];
    for (int i = ph.op_begin; i < ph.op_end; i++) {
      const KOp& op = ops[i];
      switch (op.type) {
        case OP_DIAGF: diag_fast(op); break;
        case OP_DIAG: diag_general(op); break;
        default:
          if (diag_only) break;
          if (op.type == OP_HU) hadamard(op, p, false);
          else if (op.type == OP_H) hadamard(op, p, true);
          else if (op.type == OP_X) pauli_x(op, p);
          else if (op.type == OP_D1) { int b[1] = {op.sel}; dense(op, p, 1, b); }
          else if (op.type == OP_D2) { int b[2] = {kPairA[op.sel], kPairB[op.sel]}; dense(op, p, 2, b); }
          else if (op.type == OP_D3) {
            int b[3], n = 0;
            for (int k = 0; k < kRegBits; k++) if (k != op.sel) b[n++] = k;
            dense(op, p, 3, b);
          } else if (op.type == OP_DW) {
            // applied in shared memory at the exchange into this layout
          } else {
            bad_op = true;  // never skip an op silently: the pass fails to build
          }
          break;
      }
    }
  }

  std::string build(const char* kname, bool multi, bool diag_only) {
    const int nph = multi ? h.n_phases : 1;
    L.assign(h.phases, h.phases + nph);
    // >= 4 contiguous amplitudes per thread at the store: lanes would write
    // 64+ B apart; one more exchange to the default layout pays for itself
    const bool extra_store = low_run_out(L[nph - 1]) >= 2;
    if (extra_store) L.push_back(default_layout());
    const int nlay = (int)L.size();
    const bool xchg = nlay > 1;  // any shared-memory exchange
    ck_smem = !xchg;
    {
      static const int msm = getenv("QS_JIT_MSMEM") ? atoi(getenv("QS_JIT_MSMEM")) : -1;  // A/B knob
      mat_smem = msm > 0;  // default off: on the QAOA/rand-30 passes it spills MORE
                           // (54 of 62 kernels, 8.9 KB vs 10 kernels, 0.6 KB)
    }
    const int nsh = h.n_shapes;
    std::vector<int> vary, cons;
    for (int j = 0; j < nsh; j++) {
      bool v = false;
      for (int q = shapes[j].term_begin; q < shapes[j].term_end; q++)
        if (terms[q].ncmask) v = true;
      (v ? vary : cons).push_back(j);
    }
    o << kPrelude;
    // Processing order of the chunks.  A pass that exports a swap's pieces
    // (x_mask) rotates the chunk id so that its top bits -- the destination
    // rank -- change fastest: the CTAs in flight write to every destination
    // at once instead of all of them streaming into one peer at a time.
    {
      int B = 0;
      while ((1ull << B) < h.n_chunks) B++;
      // chunk-id bits that land on exported positions (the non-chunk
      // positions in ascending order are the chunk id's bits)
      std::vector<int> nonchunk, dbits;
      for (int p = 0; p < h.nl; p++) {
        bool in = false;
        for (int c = 0; c < kChunkBits; c++)
          if (h.cpos[c] == p) in = true;
        if (!in) nonchunk.push_back(p);
      }
      for (int i = 0; h.x_mask && (1 << i) <= h.x_mask; i++)
        for (size_t b = 0; b < nonchunk.size(); b++)
          if (nonchunk[b] == h.x_pos[i] && (int)b < B) dbits.push_back((int)b);
      if (dbits.empty()) {
        o << "__device__ __forceinline__ u64 corder(u64 c) { return c; }\n";
      } else {
        // loop index bit t < |dbits| -> chunk-id bit dbits[t]; the others in order
        std::vector<int> src(B, -1);
        for (size_t t = 0; t < dbits.size(); t++) src[dbits[t]] = (int)t;
        int next = (int)dbits.size();
        for (int b = 0; b < B; b++)
          if (src[b] < 0) src[b] = next++;
        o << "__device__ __forceinline__ u64 corder(u64 c) { return 0ull";
        for (int b = 0; b < B; b++) o << " | (((c >> " << src[b] << ") & 1ull) << " << b << ")";
        o << "; }\n";
      }
    }
    auto emit_arr = [&](const char* name, const std::vector<int>& v) {
      o << "__device__ const int " << name << "[" << std::max<size_t>(1, v.size()) << "] = {";
      for (size_t i = 0; i < v.size(); i++) o << (i ? "," : "") << v[i];
      if (v.empty()) o << "0";
      o << "};\n";
    };
    // chunk-dependent shapes: few terms -> one thread each; many -> one warp
    std::vector<int> vsmall, vbig;
    for (int j : vary) (shapes[j].term_end - shapes[j].term_begin <= 6 ? vsmall : vbig).push_back(j);
    emit_arr("vmap", vbig);
    emit_arr("smap", vsmall);
    emit_arr("cmap", cons);
    // chunk-dependent shapes read from the per-chunk table (qs_kshape_table)
    // destinations in a shape-sum copy of the table row's entries: angle
    // columns -> their shape's slot, the padding and cis columns -> the cis area
    const int W = use_vtab ? tc.width : 0;
    const size_t sc_pad = ((nsh * 8 + 15) / 16) * 16;
    sc_cis = sc_pad / 8;
    {
      std::vector<int> tm;
      const int apad = (tc.n_ang + 1) & ~1;
      for (int t = 0; t < W; t++)
        tm.push_back(t < tc.n_ang ? tc.ang[t] : t < apad ? (int)sc_cis + 2 * tc.n_cis : (int)sc_cis + t - apad);
      emit_arr("tmap", tm);
    }
    // Load passes stream their chunks through two shared-memory stages filled
    // by cp.async.bulk (the TMA bulk-copy engine) one chunk ahead.
    const bool pipe = (h.src_mode == 0);
    // Loop-invariant expand factors.  A CTA's chunks are blockIdx.x + k *
    // gridDim.x: when gridDim.x is a multiple of 2^b, chunk-id bits below b
    // are the same for all of them.  If the positions a register-dependent
    // booster sub-state reads come only from the chunk bits, those chunk-id
    // bits and the rank, every thread gathers the same 16 values for every
    // chunk: they are loaded once into the thread's shared-memory slots (a
    // runtime check of gridDim.x keeps the per-chunk gather as fallback).
    int xh_g = -1, xh_b = 0;
    if (h.src_mode == 1 && nlay == 1 && h.x_mask == 0 && !getenv("QS_JIT_NOXH")) {  // env: A/B knob
      u64 regpos = 0;
      for (int r = 0; r < kNReg; r++) regpos |= reg_phys(0, r, false);
      for (int g = 0; g < h.expand.n && xh_g < 0; g++) {
        const int glo = h.expand.lo[g], ghi = h.expand.lo[g] + h.expand.len[g];
        if (!(regpos & (((1ull << h.expand.len[g]) - 1) << glo))) continue;
        int b = 0;
        for (int i = 0; i < h.n_runs; i++)
          for (int t = 0; t < h.run_len[i]; t++) {
            const int pos = h.run_dst[i] + t;
            if (pos >= glo && pos < ghi) b = std::max(b, h.run_src[i] + t + 1);
          }
        if (b <= 3) xh_g = g, xh_b = b;  // the launcher keeps grids a multiple of 8 (grid_mult)
      }
    }
    const int CH = 1 << kChunkBits;
    int l = 0;
    while (l < kChunkBits && h.cpos[l] == l) l++;
    const int nseg = 1 << (kChunkBits - l);
    std::string cbexpr = "0ull";
    for (int i = 0; i < h.n_runs; i++)
      cbexpr += " | (((chunk >> " + std::to_string((int)h.run_src[i]) + ") & " +
                u((1ull << h.run_len[i]) - 1) + ") << " + std::to_string((int)h.run_dst[i]) + ")";
    // Refill engine: TMA bulk copies of the chunk's contiguous 2^l-amplitude
    // runs (l >= 5: >= 512 B each) into a linear stage; for shorter runs
    // (l = 3, 4: passes that trade coalescing width for target slots) each
    // thread cp.async's its own 16 layout-0 amplitudes (stage slot r*256+tid).
    // The linear TMA stage is read by layout 0 with a 2^run-way bank
    // conflict; for run >= 2 the chunk is instead copied with coalesced
    // per-thread cp.async in linear order into XOR-swizzled slots (the
    // exchange layout), conflict-free on both sides.
    // (bulk copies of 128 B runs are far slower than per-thread cp.async:
    // A/B with QS_JIT_TMA_L=3, QAOA-30 155 ms vs 90 ms, rand30 587 vs 333 ms)
    static const int tma_min_l = getenv("QS_JIT_TMA_L") ? atoi(getenv("QS_JIT_TMA_L")) : 5;  // A/B knob
    TPlan tp;
    const bool pull = h.pull_j > 0;
    const bool use_tensor = pipe && !pull && l < tma_min_l && low_run(L[0]) <= 1 && tensor_plan(h, &tp);
    static const bool pull_cpa = getenv("QS_JIT_PULL_CPASYNC") != nullptr;  // A/B knob: remote loads per thread
    const bool use_tma = (pipe && l >= tma_min_l && low_run(L[0]) <= 1 && !getenv("QS_JIT_NOTMA") &&
                          !(pull && pull_cpa)) || use_tensor;
    variant = !pipe ? JV_WRITE_ONLY : use_tensor ? JV_TENSOR : use_tma ? JV_BULK : JV_CPASYNC;
    o << "struct __align__(64) QsTmap { u64 v[16]; };\n";
    // buffer table (kernel parameter xp, copied to shared memory once: a
    // dynamically indexed parameter would be copied to local memory)
    if (pull || h.x_mask) o << "__shared__ u64 qs_ptab[16];\n";
    if (pull) {
      // pull pass: the buffer an element is read from -- table entry
      // (z << 3) | piece, piece = its bits at the swap's local positions
      o << ""
        << "__device__ __forceinline__ const double2* pull_src(u64 idx) {\n"
        << "  const u32 e = (u32)(((idx >> " << (int)h.pull_z << ") & 1ull) << 3)";
      for (int t = 0; t < h.pull_j; t++) o << " | (u32)(((idx >> " << (int)h.pull_pos[t] << ") & 1ull) << " << t << ")";
      o << ";\n  return reinterpret_cast<const double2*>(qs_ptab[e]);\n}\n";
    }
    if (use_tensor) {
      // one tensor copy per chunk (coordinates: the non-chunk runs' index
      // bits), or one per lane for the 2^n_extra sub-boxes of the rest dim
      const int ncopy = 1 << tp.n_extra;
      o << "__device__ __forceinline__ void issue(const double2* __restrict__ state, u64 chunk, double2* dst, u64* bar, u32 lane, const QsTmap* tm) {\n"
        << "  (void)state;\n"
        << "  if (lane == 0) mbar_expect(bar, " << CH * 16 << "u);\n"
        << "  __syncwarp();\n"
        << "  const u64 cb = " << cbexpr << ";\n"
        << "  for (u32 e = lane; e < " << ncopy << "u; e += 32u) {\n"
        << "    asm volatile(\"cp.async.bulk.tensor." << tp.rank << "d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {";
      for (int d = 0; d < tp.rank; d++) o << (d ? ", " : "") << "%" << d + 2;
      o << "}], [" << "%" << tp.rank + 2 << "];\"\n      :: \"r\"(sa(dst + e * " << (1 << tp.covered) << "u)), \"l\"(tm)";
      for (int d = 0; d < tp.rank; d++) {
        if (tp.chunk[d]) {
          o << ", \"r\"(0)";
        } else if (d == 4 && tp.n_extra) {
          o << ", \"r\"((u32)((cb >> " << tp.pos[d] << ") & " << ((1ull << tp.len[d]) - 1) << "ull)";
          for (int x = 0; x < tp.n_extra; x++)
            o << " | (((e >> " << x << ") & 1u) << " << tp.extra[x] - tp.pos[4] << ")";
          o << ")";
        } else {
          o << ", \"r\"((u32)((cb >> " << tp.pos[d] << ") & " << ((1ull << tp.len[d]) - 1) << "ull))";
        }
      }
      o << ", \"r\"(sa(bar)) : \"memory\");\n  }\n  __syncwarp();\n}\n";
    } else if (use_tma) {
      o << "__device__ __forceinline__ void issue(const double2* __restrict__ state, u64 chunk, double2* dst, u64* bar, u32 lane, const QsTmap* tm) {\n"
        << "  (void)tm;\n"
        << "  const u64 cb = " << cbexpr << ";\n"
        << "  if (lane == 0) mbar_expect(bar, " << CH * 16 << "u);\n"
        << "  __syncwarp();\n"
        << "  for (int seg = lane; seg < " << nseg << "; seg += 32) {\n"
        << "    const u64 off = 0ull";
      for (int i = 0; i < kChunkBits - l; i++)
        o << " | ((u64)((seg >> " << i << ") & 1) << " << (int)h.cpos[l + i] << ")";
      o << ";\n    bulk_g2s(dst + (seg << " << l << "), " << (pull ? "pull_src(cb | off)" : "state") << " + (cb | off), "
        << (16 << l) << "u, bar);\n"
        << "  }\n}\n";
    } else if (pipe) {
      // thread t copies chunk elements c = t + 256 i (coalesced 128 B+ runs)
      // into slot swz(c) = swz(t) ^ swz(256 i)
      o << "__device__ __forceinline__ void issue_async(const double2* __restrict__ state, u64 chunk, double2* stage, u64* bar, u64 tpd, int sd) {\n"
        << "  const u64 cb = " << cbexpr << ";\n"
        << "  const double2* sp = state + (cb | tpd);\n";
      for (int i = 0; i < kNReg; i++) {
        u64 off = 0;
        for (int k = 0; k < kRegBits; k++)
          if (i >> k & 1) off |= 1ull << h.cpos[kLogT + k];
        if (pull)
          o << "  cp_async16(stage + (sd ^ " << host_swz(i << kLogT) << "), pull_src(cb | tpd | " << u(off) << ") + (cb | tpd | "
            << u(off) << "));\n";
        else
          o << "  cp_async16(stage + (sd ^ " << host_swz(i << kLogT) << "), sp + " << u(off) << ");\n";
      }
      o << "  cp_async_mbar_arrive(bar);\n}\n";
    }
    // A CTA runs NG chunk groups of 256 threads; its chunk sequence
    // k = 0, 1, 2, ... (chunk blockIdx.x + k * gridDim.x) is dealt round-robin
    // to the groups.  Load passes keep NB = NG + 1 chunk buffers: chunk k
    // lives in buffer k % NB, and right after its last shared-memory read the
    // buffer is refilled with chunk k + NB, so a load is in flight while every
    // group computes.  Write-only passes need a buffer per group only for
    // their layout exchanges.
    const int NG = groups_per_cta(pipe, nlay);
    int NB = pipe ? (NG == 1 ? 1 : NG + 1) : (xchg ? NG : 0);
    {
      // QS_JIT_NB: A/B knob for the ring depth of multi-layout load passes
      // (more chunk loads in flight per SM)
      static const int nb_env = getenv("QS_JIT_NB") ? atoi(getenv("QS_JIT_NB")) : 0;
      if (pipe && xchg && nb_env > NB && (size_t)nb_env * CH * 16 <= 200 * 1024) NB = nb_env;
    }
    // L2 prefetch distance (chunks of the CTA's sequence beyond the
    // shared-memory ring): cp.async.bulk.prefetch.L2 of chunk k + NB + PF
    // when chunk k's buffer is refilled, so DRAM latency overlaps more than
    // the one chunk load the ring keeps in flight.  QS_JIT_L2PF: A/B knob.
    // Per engine: tensor passes prefetch with the same tensor copies
    // (cp.async.bulk.prefetch.tensor), bulk passes per contiguous run
    // (>= 512 B), per-thread cp.async passes one prefetch.global.L2 per
    // 128 B line (the threads holding a line's first element); round 1's
    // bulk prefetch of every 64-256 B run lost badly (QAOA-30 90 -> 151 ms).
    static const int l2pf = getenv("QS_JIT_L2PF") ? atoi(getenv("QS_JIT_L2PF")) : 0;
    const int PF = (pipe && !pull) ? l2pf : 0;
    const bool pf_all = PF > 0 && !use_tma;  // every thread of the group prefetches
    if (PF > 0 && use_tensor) {
      const int ncopy = 1 << tp.n_extra;
      o << "__device__ __forceinline__ void l2pf(const double2* __restrict__ state, u64 chunk, u32 lane, const QsTmap* tm) {\n"
        << "  (void)state;\n  const u64 cb = " << cbexpr << ";\n"
        << "  for (u32 e = lane; e < " << ncopy << "u; e += 32u) {\n"
        << "    asm volatile(\"cp.async.bulk.prefetch.tensor." << tp.rank << "d.L2.global.tile [%0, {";
      for (int d = 0; d < tp.rank; d++) o << (d ? ", " : "") << "%" << d + 1;
      o << "}];\"\n      :: \"l\"(tm)";
      for (int d = 0; d < tp.rank; d++) {
        if (tp.chunk[d]) {
          o << ", \"r\"(0)";
        } else if (d == 4 && tp.n_extra) {
          o << ", \"r\"((u32)((cb >> " << tp.pos[d] << ") & " << ((1ull << tp.len[d]) - 1) << "ull)";
          for (int x = 0; x < tp.n_extra; x++)
            o << " | (((e >> " << x << ") & 1u) << " << tp.extra[x] - tp.pos[4] << ")";
          o << ")";
        } else {
          o << ", \"r\"((u32)((cb >> " << tp.pos[d] << ") & " << ((1ull << tp.len[d]) - 1) << "ull))";
        }
      }
      o << " : \"memory\");\n  }\n}\n";
    } else if (PF > 0 && use_tma) {
      o << "__device__ __forceinline__ void l2pf(const double2* __restrict__ state, u64 chunk, u32 lane, const QsTmap* tm) {\n"
        << "  (void)tm;\n  const u64 cb = " << cbexpr << ";\n"
        << "  for (int seg = (int)lane; seg < " << nseg << "; seg += 32) {\n"
        << "    const u64 off = 0ull";
      for (int i = 0; i < kChunkBits - l; i++)
        o << " | ((u64)((seg >> " << i << ") & 1) << " << (int)h.cpos[l + i] << ")";
      o << ";\n    asm volatile(\"cp.async.bulk.prefetch.L2.global [%0], %1;\" :: \"l\"(state + (cb | off)), \"r\"("
        << (16 << l) << "u) : \"memory\");\n  }\n}\n";
    } else if (PF > 0) {
      // thread t's elements t + 256 i: chunk bits 0..2 are positions 0..2
      // (the forced low run), so threads t = 0 mod 8 start every line
      o << "__device__ __forceinline__ void l2pf(const double2* __restrict__ state, u64 chunk, u32 tid, const QsTmap* tm) {\n"
        << "  (void)tm;\n  if ((tid & 7u) != 0u) return;\n"
        << "  const u64 cb = " << cbexpr << ";\n"
        << "  const double2* sp = state + (cb";
      for (int i = 0; i < kLogT; i++) o << " | ((u64)((tid >> " << i << ") & 1u) << " << (int)h.cpos[i] << ")";
      o << ");\n";
      for (int i = 0; i < kNReg; i++) {
        u64 off = 0;
        for (int k = 0; k < kRegBits; k++)
          if (i >> k & 1) off |= 1ull << h.cpos[kLogT + k];
        o << "  asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(sp + " << u(off) << ") : \"memory\");\n";
      }
      o << "}\n";
    }
    nthreads = kThreads * NG;
    const size_t npool = (h.total_bytes - h.off_pool) / sizeof(double);
    param_pool = npool > 0 && npool <= kMaxParamPool && !run_mode;
    if (param_pool) o << "struct QsPool { double v[" << npool << "]; };\n";
    // fused swap: destination base per value of the exported
    // top local bits (receive buffers of this rank or its peers, by value)
    o << "struct QsXPeer { u64 v[16]; };\n";
    if (run_mode) {
      // QS_RUN_SLEEP (ns between polls), QS_RUN_NOPFENCE, QS_RUN_PROF
      // (per-CTA wait cycles, printed by the run kernel): A/B and diagnostics
      static const int sleep_ns = getenv("QS_RUN_SLEEP") ? atoi(getenv("QS_RUN_SLEEP")) : 64;
      static const bool pfence = getenv("QS_RUN_NOPFENCE") == nullptr;
      static const bool prof = getenv("QS_RUN_PROF") != nullptr;
      // (a wait that lasts ~10 s means a scheduling bug: trap -- the launch
      // fails with an error instead of hanging the device)
      o << "__device__ __forceinline__ void qs_wait(const u32* f, u32 need) {\n"
        << "  const long long t0_ = clock64();\n"
        << "  for (;;) {\n    u32 v;\n"
           "    asm volatile(\"ld.acquire.gpu.global.u32 %0, [%1];\" : \"=r\"(v) : \"l\"(f) : \"memory\");\n"
           "    if (v >= need) break;\n"
           "    if (clock64() - t0_ > 20000000000ll) __trap();\n"
        << (sleep_ns > 0 ? "    __nanosleep(" + std::to_string(sleep_ns) + ");\n" : "") << "  }\n"
        << (pfence ? "  asm volatile(\"fence.proxy.async.global;\" ::: \"memory\");\n" : "")
        << (prof ? "  if ((threadIdx.x & 31u) == 0) atomicAdd(&::qs_wcyc, (unsigned long long)(clock64() - t0_));\n" : "")
        << "}\n";
    }
    // QS_JIT_WO_MINB: A/B knob for the resident-CTA target of one-group passes
    static const int wo_minb = getenv("QS_JIT_WO_MINB") ? atoi(getenv("QS_JIT_WO_MINB")) : 2;
    if (run_mode)
      o << "__device__ __forceinline__ void qs_body(const unsigned char* __restrict__ blob, double2* __restrict__ state, "
           "u64 rank_base, const u64* __restrict__ vtab, const QsXPeer& xp, const QsTmap& tensmap, const u64 clo, "
           "const u64 cn, const u32 qs_bid, const u32 qs_nbid, const u32* qs_fin, u32* qs_fout, const u32* qs_back, "
           "const u32 qs_lag) {\n"
           "  (void)qs_fin; (void)qs_fout; (void)qs_back; (void)qs_lag;\n";
    else
      o << "extern \"C\" __global__ void __launch_bounds__(" << nthreads << ", " << (NG == 1 && NB <= 1 ? wo_minb : 1)
        << ")\n" << kname
        << "(const unsigned char* __restrict__ blob, double2* __restrict__ state, u64 rank_base, "
           "const u64* __restrict__ vtab, const QsXPeer xp, const __grid_constant__ QsTmap tensmap, "
           "const u64 clo, const u64 cn"
        << (param_pool ? ", const QsPool P" : "") << ") {\n";
    o << "  extern __shared__ __align__(128) unsigned char smem_raw[];\n";
    const size_t buf_bytes = (size_t)NB * CH * 16;
    // shape sums; with the per-chunk table, two copies: the chunk's and the
    // group's next chunk's (prefetched during the chunk)
    const size_t sc_copy = (use_vtab && !warp_tab) ? sc_pad + (2 * tc.n_cis + 2) * 8 : sc_pad;
    const size_t sc_bytes = warp_tab ? sc_pad + (kThreads / 32) * 64 * 8 : use_vtab ? 2 * sc_copy : sc_copy;
    const std::string SCN = std::to_string(sc_copy / 8);
    o << "  const u32 tid = threadIdx.x & 255u;\n";
    o << "  const u32 grp = threadIdx.x >> 8;\n  (void)grp;\n";
    o << "  double2* const bufs = reinterpret_cast<double2*>(smem_raw);\n  (void)bufs;\n";
    o << "  u64* const scbase = reinterpret_cast<u64*>(smem_raw + " << buf_bytes << " + grp * " << sc_bytes << ");\n";
    o << "  u64* scoef = scbase;\n  (void)scoef;\n";
    if (warp_tab)
      o << "  u64* const wbase = scbase + " << sc_pad / 8 << " + (tid >> 5) * 64;\n"
        << "  const u32 lane = tid & 31u;\n";
    const size_t mbar_off = buf_bytes + NG * sc_bytes;
    // issued[b]: loads issued into buffer b so far (two groups: see the wait)
    if (pipe)
      o << "  u64* mbar = reinterpret_cast<u64*>(smem_raw + " << mbar_off << ");\n"
        << "  volatile u32* issued = reinterpret_cast<volatile u32*>(smem_raw + " << mbar_off + NB * 8
        << ");\n  (void)issued;\n";
    hz_off = mbar_off + (pipe ? ((NB * 12 + 15) / 16) * 16 : 0);
    const size_t xh_off = hz_off;
    if (xh_g >= 0) {
      hz_off += (size_t)kNReg * kThreads * 16;
      static const bool xh_grid = getenv("QS_JIT_XHGRID") == nullptr || atoi(getenv("QS_JIT_XHGRID")) != 0;
      if (xh_grid) grid_mult = 1 << xh_b;  // e.g. 148 -> 144 CTAs: the gathers stay hoisted
    }
    // hoisted per-thread values (shared by the groups: they depend on tid only)
    // fill what shared memory is left: 227 KB per CTA (two CTAs per SM: half
    // of 228 KB, less the per-CTA reservation), minus the 4 KB sincos table
    // unless no sincos is left inside the loop (second generation pass)
    const long smem_cap = ((NG == 1 && NB <= 1) ? 113 * 1024 : 227 * 1024) - (table_free ? 0 : 4096) -
                          (run_mode ? 12 * 1024 : 0) -
                          (ck_smem ? 16l * n_ck_entries() : 0l) - (mat_smem ? 8l * n_mat_doubles() : 0l);
    max_hoist = (int)std::max<long>(0, (smem_cap - (long)hz_off) / (kThreads * 16));
    if (max_hoist > 24) max_hoist = 24;
    if (const char* e = getenv("QS_JIT_MAXHOIST")) max_hoist = std::min(max_hoist, atoi(e));  // experiments
    o << "  double2* hz = reinterpret_cast<double2*>(smem_raw + " << hz_off << ");\n  (void)hz;\n";
    o << "  const double* __restrict__ pool = reinterpret_cast<const double*>(blob + " << h.off_pool << ");\n";
    o << "  const int* __restrict__ shp = reinterpret_cast<const int*>(blob + " << h.off_shapes << ");\n";
    o << "  const u64* __restrict__ trm = reinterpret_cast<const u64*>(blob + " << h.off_terms << ");\n";
    o << "  (void)pool; (void)shp; (void)trm;\n";
    const size_t ctab_pos = o.str().size();  // the sincos table goes here if used
    for (int p = 0; p < nlay; p++) {
      o << "  const u64 tp" << p << " = " << tphys_expr(p, false) << ";\n";
      if (xchg || (pipe && !use_tma)) o << "  const int st" << p << " = swz(" << tc_expr(p) << ");\n";
    }
    o << "  const u64 tpo = " << tphys_expr(nlay - 1, true) << ";\n";
    // chunks [clo, clo + cn) of the pass's h.n_chunks: all of them, or one
    // wave of an L2-blocked pass group (executor)
    const std::string N = "cn";
    // Chunk pairs: a two-group load pass deals chunk PAIRS
    // (2m, 2m + 1; m = blockIdx.x + j gridDim.x) to its groups, so the loads
    // a CTA has in flight differ in chunk-id bit 0 (the lowest non-chunk
    // position) -- probe: a chunk without position 3 or 5 streams at 0.75 of
    // the bandwidth of one with it (scripts/dev/pattern_bw.cu)
    // Default: the passes whose chunk has neither position 3 nor 5 (the
    // slow address pattern); QS_JIT_PAIR=0 never, =1 every two-group load pass.
    static const int pair_env = getenv("QS_JIT_PAIR") ? atoi(getenv("QS_JIT_PAIR")) : -1;
    bool slow_pattern = true;
    for (int c = 0; c < kChunkBits; c++)
      if (h.cpos[c] == 3 || h.cpos[c] == 5) slow_pattern = false;
    const bool pair = (pair_env == 1 || (pair_env < 0 && slow_pattern)) && pipe && NG == 2 && xh_g < 0 &&
                      (h.n_chunks % 2) == 0;
    auto chunk_of = [&](const std::string& k) {
      return pair ? "(((((u64)blockIdx.x + (u64)((" + k + ") >> 1) * gridDim.x)) << 1) | (u64)((" + k + ") & 1u))"
                  : "(blockIdx.x + (u64)(" + k + ") * gridDim.x)";
    };

    if (pipe) {
      o << "  if (threadIdx.x == 0) {\n"
        << "    for (int b = 0; b < " << NB << "; b++) { mbar_init(mbar + b, " << (use_tma ? 1 : kThreads)
        << "); issued[b] = 0u; }\n"
        << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n  }\n";
    }
    if (pull || h.x_mask) {
      o << "  if (threadIdx.x == 0) {\n";
      for (int i = 0; i < 16; i++) o << "    qs_ptab[" << i << "] = xp.v[" << i << "];\n";
      o << "  }\n";
    }
    o << "  __syncthreads();\n";
    if (use_tma) {
      o << "  const int tcl0 = " << tc_expr(0) << ";\n";
      o << "  for (u32 k = grp; k < " << NB << "u; k += " << NG << "u)\n"
        << "    if (tid < 32 && " << chunk_of("k") << " < " << N << ") { "
        << run_wait_of("corder(clo + " + chunk_of("k") + ")") << "issue(state, corder(clo + " << chunk_of("k") << ")"
        << ", bufs + k * " << CH << ", mbar + k, tid, &tensmap); if (tid == 0) issued[k] = 1u; }\n";
    } else if (pipe) {
      std::string tpd = "(0ull";
      for (int i = 0; i < kLogT; i++)
        tpd += " | ((u64)((tid >> " + std::to_string(i) + ") & 1u) << " + std::to_string((int)h.cpos[i]) + ")";
      o << "  const u64 tpd = " << tpd << ");\n  const int sd = swz((int)tid);\n";
      o << "  for (u32 k = grp; k < " << NB << "u; k += " << NG << "u)\n"
        << "    if (" << chunk_of("k") << " < " << N << ") { "
        << run_wait_of("corder(clo + " + chunk_of("k") + ")") << "issue_async(state, corder(clo + " << chunk_of("k") << ")"
        << ", bufs + k * " << CH << ", mbar + k, tpd, sd); if (tid == 0) issued[k] = 1u; }\n";
    }
    if (PF > 0)
      o << "  for (u32 k = " << NB << "u + grp; k < " << NB + PF << "u; k += " << NG << "u)\n"
        << "    if (" << (pf_all ? "" : "tid < 32 && ") << chunk_of("k") << " < " << N << ") l2pf(state, corder(clo + "
        << chunk_of("k") << "), tid, &tensmap);\n";
    // level 1, constant shapes: once
    // level 1: one warp per shape, lanes over its terms, shuffle reduction
    auto level1 = [&](const char* map, size_t n, bool use_cphys) {
      o << "    for (int jj = (int)(tid >> 5); jj < " << n << "; jj += 8) {\n"
        << "      const int j = " << map << "[jj];\n"
        << "      const int b = __ldg(shp + 4 * j + 1), e = __ldg(shp + 4 * j + 2);\n"
        << "      u64 acc = 0ull;\n"
        << "      for (int q = b + (int)(tid & 31u); q < e; q += 32) {\n";
      if (use_cphys)
        o << "        const u64 mk = __ldg(trm + 2 * q);\n"
          << "        if ((cphys & mk) == mk) acc += __ldg(trm + 2 * q + 1);\n";
      else
        o << "        acc += __ldg(trm + 2 * q + 1);\n";
      o << "      }\n"
        << "      for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);\n"
        << "      if ((tid & 31u) == 0) { scoef[j] = acc;" << (use_vtab && !warp_tab && !use_cphys ? " scoef[j + " + SCN + "] = acc;" : "")
        << " }\n    }\n";
    };
    if (!cons.empty()) {
      o << "  {\n";
      level1("cmap", cons.size(), false);
      o << "  }\n  __syncthreads();\n";
    }
    const std::string NV = std::to_string(W);
    if (warp_tab)
      o << "  { const u64 c0 = " << chunk_of("grp") << ";\n    if (lane < " << NV << "u && c0 < " << N
        << ") wbase[lane] = __ldg(vtab + corder(clo + c0) * " << NV << "ull + lane);\n    __syncwarp(); }\n";
    else if (use_vtab)
      o << "  { const u64 c0 = " << chunk_of("grp") << ";\n    if (tid < " << NV << "u && c0 < " << N
        << ") scoef[tmap[tid]] = __ldg(vtab + corder(clo + c0) * " << NV << "ull + tid); }\n  __syncthreads();\n";
    if (xh_g >= 0) {
      const int g = xh_g;
      o << "  double2* const xh = reinterpret_cast<double2*>(smem_raw + " << xh_off << ");\n"
        << "  const bool xinv = (gridDim.x & " << ((1u << xh_b) - 1) << "u) == 0u;\n"
        << "  if (xinv) {\n"
        << "    const double2* __restrict__ xsv = reinterpret_cast<const double2*>(*reinterpret_cast<const u64*>(blob + "
        << (size_t)((const unsigned char*)&h.expand.ptr[g] - (const unsigned char*)&h) << "));\n"
        << "    const u64 chunk = corder(clo + " << chunk_of("grp") << ");\n"
        << "    const u64 xph = (" << cbexpr << ") | rank_base | tp0;\n";
      for (int r = 0; r < kNReg; r++)
        o << "    xh[" << r * kThreads << " + tid] = __ldg(xsv + (((xph | " << u(reg_phys(0, r, false)) << ") >> "
          << h.expand.lo[g] << ") & " << u((1ull << h.expand.len[g]) - 1) << "));\n";
      o << "  }\n";
    }
    o << "  double2 a0, a1, a2, a3, a4, a5, a6, a7, a8, a9, a10, a11, a12, a13, a14, a15;\n";
    const size_t loop_pos = o.str().size();  // hoisted code goes here
    o << "  for (u32 k = grp;; k += " << NG << "u) {\n"
      << "    const u64 craw = " << chunk_of("k") << ";\n"
      << "    if (craw >= " << N << ") break;\n"
      << "    const u64 chunk = corder(clo + craw);\n";
    if (run_throttle)
      o << "    if ((chunk >> " << run_sb << ") >= qs_lag) {\n"
        << "      if (tid == 0) qs_wait(qs_back + ((chunk >> " << run_sb << ") - qs_lag), " << (1 << run_sb) << "u);\n"
        << "      gbar(1u + grp);\n    }\n";
    if (pipe) o << "    const u32 kb = k % " << NB << "u;\n    double2* const sch = bufs + kb * " << CH << ";\n";
    else if (xchg) o << "    double2* const sch = bufs + grp * " << CH << ";\n";
    const std::string nxt = chunk_of("k + " + std::to_string(NB));
    const std::string pfc = chunk_of("k + " + std::to_string(NB + PF));
    const std::string pf_issue =
        PF > 0 ? "    if (" + std::string(pf_all ? "" : "tid < 32 && ") + pfc + " < " + N + ") l2pf(state, corder(clo + " + pfc +
                     "), tid, &tensmap);\n"
               : "";
    const std::string count = "if (tid == 0) { __threadfence_block(); issued[kb] = k / " +
                              std::to_string(NB) + "u + 2u; }";
    // QS_JIT_CHECK (debug builds of the kernels; compute-sanitizer is not
    // available on the GPU pool): the consumed buffer is overwritten with NaN
    // before its refill is issued, so a read that races the refill (or a
    // stale-phase wait) poisons the result instead of silently reusing data;
    // and the ring's phase bookkeeping is asserted (trap on violation).
    static const bool check = getenv("QS_JIT_CHECK") != nullptr;
    const std::string poison =
        check ? "    gbar(1u + grp);\n    for (int i = 0; i < 16; i++) sch[(int)tid + 256 * i] = make_double2(__longlong_as_double(0x7ff8dead7ff8deadll), __longlong_as_double(0x7ff8dead7ff8deadll));\n"
              : "";
    const std::string refill = poison +
        (use_tma ? "    gbar(1u + grp);  // every thread is done reading the buffer\n"
                  "    if (tid < 32 && " + nxt + " < " + N +
                  ") { " + run_wait_of("corder(clo + " + nxt + ")") + "fence_proxy_async(); issue(state, corder(clo + " + nxt + "), sch, mbar + kb, tid, &tensmap); " + count + " }\n" + pf_issue
                : "    gbar(1u + grp);  // every thread is done reading the buffer\n"
                  "    if (" + nxt + " < " + N + ") { " + run_wait_of("corder(clo + " + nxt + ")") + "issue_async(state, corder(clo + " + nxt + "), sch, mbar + kb, tpd, sd); " +
                  count + " }\n" + pf_issue);
    o << "    const u64 cb = " << cbexpr << ";\n";
    o << "    const u64 cphys = cb | rank_base;\n    (void)cphys;\n";
    // (cp.async row prefetch unless the pass's own chunk refill uses
    // per-thread cp.async, whose uncommitted copies a row group would absorb;
    // A/B on one box: diag-chain-30 K2 6.26 -> 5.09 ms, QFT-30 K2 3.84 ->
    // 3.91 ms.  Tried for the CTA-wide rows too: RZZ-30 K3 3.33 -> 3.36 ms)
    const bool row_async = warp_tab && (!pipe || use_tma) && !getenv("QS_JIT_ROWREG");  // env: A/B knob
    if (warp_tab) {
      // per-warp table rows (two copies: this chunk's, the next one's)
      o << "    u64 nxrow = 0ull;\n    (void)nxrow;\n";
      o << "    const u64* const wrow = wbase + (((k / " << NG << "u) & 1u) ? 32 : 0);\n"
        << "    u64* const wnx = wbase + (((k / " << NG << "u) & 1u) ? 0 : 32);\n"
        << "    const double2* const cisv = reinterpret_cast<const double2*>(wrow + " << ((tc.n_ang + 1) & ~1) << ");\n"
        << "    (void)cisv; (void)wrow;\n"
        << "    { const u64 nc = " << chunk_of("k + " + std::to_string(NG)) << ";\n";
      if (row_async)
        // the next row goes straight into the other copy with cp.async (a
        // register load gets sunk by the compiler next to its use)
        o << "      if (lane < " << NV << "u && nc < " << N << ") cp_async8(wnx + lane, vtab + corder(clo + nc) * " << NV
          << "ull + lane);\n      cp_async_commit(); }\n";
      else
        o << "      u64 nxv = 0ull;\n      if (lane < " << NV << "u && nc < " << N << ") nxv = __ldg(vtab + corder(clo + nc) * "
          << NV << "ull + lane);\n      nxrow = nxv; }\n";
    } else if (use_vtab) {
      // one coalesced table row per chunk instead of the level-1 term loops,
      // loaded one chunk ahead (stored to the other copy at the chunk's end)
      o << "    u64* const scoef = scbase + (((k / " << NG << "u) & 1u) ? " << SCN << " : 0);\n"
        << "    u64* const scnx = scbase + (((k / " << NG << "u) & 1u) ? 0 : " << SCN << ");\n"
        << "    const double2* const cisv = reinterpret_cast<const double2*>(scoef + " << sc_cis << ");\n"
        << "    (void)cisv;\n"
        << "    u64 nxv = 0ull;\n"
        << "    { const u64 nc = " << chunk_of("k + " + std::to_string(NG)) << ";\n"
        << "      if (tid < " << NV << "u && nc < " << N << ") nxv = __ldg(vtab + corder(clo + nc) * " << NV << "ull + tid); }\n";
    } else if (!vary.empty()) {
      o << "    gbar(1u + grp);\n";
      if (!vbig.empty()) level1("vmap", vbig.size(), true);
      if (!vsmall.empty())
        o << "    for (int jj = (int)tid; jj < " << vsmall.size() << "; jj += " << kThreads << ") {\n"
          << "      const int j = smap[jj];\n"
          << "      const int b = __ldg(shp + 4 * j + 1), e = __ldg(shp + 4 * j + 2);\n"
          << "      u64 acc = 0ull;\n"
          << "      for (int q = b; q < e; q++) {\n"
          << "        const u64 mk = __ldg(trm + 2 * q);\n"
          << "        if ((cphys & mk) == mk) acc += __ldg(trm + 2 * q + 1);\n"
          << "      }\n      scoef[j] = acc;\n    }\n";
      o << "    gbar(1u + grp);\n";
    }
    // loads (phase 0)
    for (int r = 0; r < kNReg; r++) nm[r] = r;
    pend_c.clear();
    // pass scale S = (scale, scale_im) = m * u: the real m is folded into an
    // unnormalised H / a full-width diagonal / the store as before; the unit
    // u is applied at the end: +-1 (sign of m), +-i (swap + sign), an eighth
    // turn (+-1 +- i)/|.| (two additions), else a constant complex product
    {
      const double sr = h.scale, si = h.scale_im;
      if (si == 0.0) { sc_kind = 0; sc_mag = sr; }
      else if (sr == 0.0) { sc_kind = 1; sc_mag = si; }                          // S = i * si
      else if (std::fabs(sr) == std::fabs(si)) { sc_kind = 2; sc_mag = std::fabs(sr); sc_sx = sr > 0 ? 1 : -1; sc_sy = si > 0 ? 1 : -1; }
      else { sc_kind = 3; sc_mag = 1.0; }
    }
    pend_scale = (sc_mag != 1.0);
    static const bool xsm_off = getenv("QS_JIT_NOXSM") != nullptr;  // A/B knob
    if (h.src_mode == 1 && xchg && !xsm_off) {
      // Multi-layout write-only pass: the tensor product is expanded into the
      // chunk buffer in LINEAR chunk order (thread t makes chunk elements
      // t + 256 i), so consecutive lanes gather consecutive sub-state entries
      // (coalesced, L1-friendly), then layout 0 is read from the buffer like
      // an exchange.  Groups with no chunk position are per-chunk constants.
      u64 cmask = 0;
      for (int c = 0; c < kChunkBits; c++) cmask |= 1ull << h.cpos[c];
      std::vector<int> varying;
      std::string tpd = "(0ull";
      for (int i = 0; i < kLogT; i++)
        tpd += " | ((u64)((tid >> " + std::to_string(i) + ") & 1u) << " + std::to_string((int)h.cpos[i]) + ")";
      tpd += ")";
      for (int g = 0; g < h.expand.n; g++) {
        o << "    const double2* __restrict__ sv" << g << " = reinterpret_cast<const double2*>(*reinterpret_cast<const u64*>(blob + "
          << (size_t)((const unsigned char*)&h.expand.ptr[g] - (const unsigned char*)&h) << "));\n";
        const u64 gmask = ((1ull << h.expand.len[g]) - 1) << h.expand.lo[g];
        if (cmask & gmask) {
          varying.push_back(g);
        } else {
          o << "    const double2 pf" << g << " = __ldg(sv" << g << " + ((cphys >> " << h.expand.lo[g] << ") & "
            << u((1ull << h.expand.len[g]) - 1) << "));\n";
          pend_c.push_back("pf" + std::to_string(g));
        }
      }
      // (the group may still be reading the previous chunk's last layout)
      o << "    gbar(1u + grp);\n    { const u64 xb = cphys | " << tpd << ";\n";
      for (int i = 0; i < kNReg; i++) {
        u64 off = 0;
        for (int k = 0; k < kRegBits; k++)
          if (i >> k & 1) off |= 1ull << h.cpos[kLogT + k];
        o << "      { const u64 ph = xb | " << u(off) << "; double2 v = ";
        if (varying.empty()) o << "make_double2(1.0, 0.0)";
        for (size_t q = 0; q < varying.size(); q++) {
          const int g = varying[q];
          const std::string ld = "__ldg(sv" + std::to_string(g) + " + ((ph >> " + std::to_string(h.expand.lo[g]) +
                                 ") & " + u((1ull << h.expand.len[g]) - 1) + "))";
          if (q == 0) o << ld;
          else o << "; v = cmul(v, " << ld << ")";
        }
        o << "; sch[swz((int)tid ^ " << (i << kLogT) << ")] = v; }\n";
      }
      o << "    }\n    gbar(1u + grp);\n";
      for (int r = 0; r < kNReg; r++) o << "    " << A(r) << " = sch[st0 ^ " << reg_slot(0, r) << "];\n";
    } else if (h.src_mode == 1) {
      // groups whose sub-state index ignores the register bits contribute a
      // per-thread constant factor (loaded once, folded later)
      u64 regpos = 0;
      for (int r = 0; r < kNReg; r++) regpos |= reg_phys(0, r, false);
      std::vector<int> varying;
      for (int g = 0; g < h.expand.n; g++) {
        o << "    const double2* __restrict__ sv" << g << " = reinterpret_cast<const double2*>(*reinterpret_cast<const u64*>(blob + "
          << (size_t)((const unsigned char*)&h.expand.ptr[g] - (const unsigned char*)&h) << "));\n";
        const u64 gmask = ((1ull << h.expand.len[g]) - 1) << h.expand.lo[g];
        if (regpos & gmask) {
          varying.push_back(g);
        } else {
          o << "    const double2 pf" << g << " = __ldg(sv" << g << " + (((cphys | tp0) >> " << h.expand.lo[g]
            << ") & " << u((1ull << h.expand.len[g]) - 1) << "));\n";
          pend_c.push_back("pf" + std::to_string(g));
        }
      }
      o << "    {\n";
      for (int r = 0; r < kNReg; r++) {
        if (varying.empty()) {
          o << "      " << A(r) << " = make_double2(1.0, 0.0);\n";
          continue;
        }
        o << "      { const u64 ph = cphys | tp0 | " << u(reg_phys(0, r, false)) << "; double2 v = ";
        for (size_t i = 0; i < varying.size(); i++) {
          const int g = varying[i];
          std::string ld = "__ldg(sv" + std::to_string(g) + " + ((ph >> " + std::to_string(h.expand.lo[g]) +
                           ") & " + u((1ull << h.expand.len[g]) - 1) + "))";
          if (g == xh_g) ld = "(xinv ? xh[" + std::to_string(r * kThreads) + " + tid] : " + ld + ")";
          if (i == 0) o << ld;
          else o << "; v = cmul(v, " << ld << ")";
        }
        o << "; " << A(r) << " = v; }\n";
      }
      o << "    }\n";
    } else if (h.src_mode == 2) {
      o << "    { const u64 bz = *reinterpret_cast<const u64*>(blob + "
        << (size_t)((const unsigned char*)&h.basis - (const unsigned char*)&h) << ");\n";
      for (int r = 0; r < kNReg; r++)
        o << "      " << A(r) << " = make_double2(((cphys | tp0 | " << u(reg_phys(0, r, false))
          << ") == bz) ? 1.0 : 0.0, 0.0);\n";
      o << "    }\n";
    } else {
      // staged chunk (linear chunk-index layout) -> registers of layout 0
      // The j-th use of buffer b (chunk k = j * NB + b) is its mbarrier's
      // phase j.  With two groups, phase j - 1 belongs to the other group and
      // may still be in flight, and a parity wait on j would then alias to the
      // completed phase j - 2.  The load of phase j is issued only after phase
      // j - 1 was consumed, so first wait until it has been issued.
      if (NG > 1) o << "    while (issued[kb] < k / " << NB << "u + 1u) {}\n";
      o << "    mbar_wait(mbar + kb, (k / " << NB << "u) & 1u);\n";
      if (check && NG > 1) o << "    if (issued[kb] != k / " << NB << "u + 1u) __trap();\n";
      if (use_tma) {
        for (int r = 0; r < kNReg; r++) {
          int rc = 0;
          for (int k = 0; k < kRegBits; k++)
            if (r >> k & 1) rc |= 1 << L[0].reg_c[k];
          o << "    " << A(r) << " = sch[tcl0 | " << rc << "];\n";
        }
      } else {
        for (int r = 0; r < kNReg; r++) o << "    " << A(r) << " = sch[st0 ^ " << reg_slot(0, r) << "];\n";
      }
      if (nlay == 1) o << refill;
    }
    for (int p = 0; p < nlay; p++) {
      if (p > 0) {
        o << "    gbar(1u + grp);\n";
        for (int r = 0; r < kNReg; r++)
          o << "    sch[st" << p - 1 << " ^ " << reg_slot(p - 1, r) << "] = " << A(r) << ";\n";
        o << "    gbar(1u + grp);\n";
        if (p < nph && h.phases[p].op_begin < h.phases[p].op_end && ops[h.phases[p].op_begin].type == OP_DW) {
          wide(ops[h.phases[p].op_begin]);
          o << "    gbar(1u + grp);\n";
        }
        for (int r = 0; r < kNReg; r++)
          o << "    " << A(r) << " = sch[st" << p << " ^ " << reg_slot(p, r) << "];\n";
        if (pipe && p == nlay - 1) o << refill;
      }
      if (p < nph) emit_ops(p, diag_only);
    }
    if (!pend_c.empty()) {
      o << "    { double2 F = " << pend_c[0] << ";\n";
      for (size_t i = 1; i < pend_c.size(); i++) o << "      F = cmul(F, " << pend_c[i] << ");\n";
      if (pend_scale) o << "      F = make_double2(F.x * " << hex(sc_mag) << ", F.y * " << hex(sc_mag) << ");\n";
      for (int r = 0; r < kNReg; r++) o << "      " << A(r) << " = cmul(" << A(r) << ", F);\n";
      o << "    }\n";
    } else if (pend_scale) {
      for (int r = 0; r < kNReg; r++)
        o << "    " << A(r) << " = make_double2(" << A(r) << ".x * " << hex(sc_mag) << ", " << A(r)
          << ".y * " << hex(sc_mag) << ");\n";
    }
    if (sc_kind == 1) {         // * i
      for (int r = 0; r < kNReg; r++)
        o << "    " << A(r) << " = make_double2(-" << A(r) << ".y, " << A(r) << ".x);\n";
    } else if (sc_kind == 2) {  // * (sx + i sy), magnitude folded
      const char* px = sc_sx > 0 ? "" : "-";
      const char* py = sc_sy > 0 ? "" : "-";
      for (int r = 0; r < kNReg; r++)
        o << "    " << A(r) << " = make_double2(" << px << A(r) << ".x - " << py << "(" << A(r) << ".y), "
          << py << A(r) << ".x + " << px << "(" << A(r) << ".y));\n";
    } else if (sc_kind == 3) {  // general complex scale (read from the descriptor)
      o << "    { const double2 S = make_double2(*reinterpret_cast<const double*>(blob + "
        << (size_t)((const unsigned char*)&h.scale - (const unsigned char*)&h) << "), *reinterpret_cast<const double*>(blob + "
        << (size_t)((const unsigned char*)&h.scale_im - (const unsigned char*)&h) << "));\n";
      for (int r = 0; r < kNReg; r++) o << "      " << A(r) << " = cmul(" << A(r) << ", S);\n";
      o << "    }\n";
    }
    if (h.x_mask) {
      // exported piece s = the output index's top x_j local bits; they may
      // come from the chunk index, the thread or the register (disjoint bits)
      int xj = 0;
      while ((1 << xj) <= h.x_mask) xj++;
      if (h.x_split >= 0) {
        // push/pull split: chunks with bit x_split set stay in place (the
        // pass after the swap pulls them from this buffer)
        o << "    if ((cb >> " << (int)h.x_split << ") & 1ull) { double2* __restrict__ so = state + (cb | tpo);\n";
        for (int r = 0; r < kNReg; r++)
          o << "      so[" << u(reg_phys(nlay - 1, r, true)) << "] = " << A(r) << ";\n";
        o << "    } else\n";
      }
      o << "    { const u64 xi = cb | tpo;\n      const u32 sct = 0u";
      for (int i = 0; i < xj; i++) o << " | ((u32)((xi >> " << (int)h.x_pos[i] << ") & 1ull) << " << i << ")";
      o << ";\n";
      for (int r = 0; r < kNReg; r++) {
        const u64 ro = reg_phys(nlay - 1, r, true);
        u64 sr = 0;
        for (int i = 0; i < xj; i++) sr |= ((ro >> h.x_pos[i]) & 1ull) << i;
        o << "      reinterpret_cast<double2*>(qs_ptab[sct | " << sr << "u])[xi + " << u(ro) << "] = " << A(r)
          << ";\n";
      }
      o << "    }\n";
    } else {
      o << "    { double2* __restrict__ so = state + (cb | tpo);\n";
      for (int r = 0; r < kNReg; r++)
        o << "      so[" << u(reg_phys(nlay - 1, r, true)) << "] = " << A(r) << ";\n";
      o << "    }\n";
    }
    if (warp_tab && row_async) o << "    cp_async_wait_group0();\n    __syncwarp();\n";
    else if (warp_tab) o << "    if (lane < " << NV << "u) wnx[lane] = nxrow;\n    __syncwarp();\n";
    else if (use_vtab) o << "    if (tid < " << NV << "u) scnx[tmap[tid]] = nxv;\n    gbar(1u + grp);\n";
    if (run_signal)
      // the group's stores of this chunk, then one release increment of its
      // block's counter (cumulative over the barrier: the next pass's
      // acquire sees all of them)
      o << "    gbar(1u + grp);\n    if (tid == 0) asm volatile(\"red.release.gpu.global.add.u32 [%0], 1;\" :: \"l\"(qs_fout + (chunk >> "
        << run_sb << ")) : \"memory\");\n";
    o << "  }\n";
    // peer stores must be performed before the barrier that publishes them
    if (h.x_mask) o << "  __threadfence_system();\n";
    o << "}\n";
    std::string s = o.str();
    if (n_hoist) s.insert(loop_pos, "  if (grp == 0) {\n" + pre.str() + "  }\n  __syncthreads();\n");
    if (!m_slot.empty()) {
      std::string t = "  __shared__ double csm[" + std::to_string(m_slot.size()) + "];\n  {\n";
      t += "    const unsigned short csoff[" + std::to_string(m_slot.size()) + "] = {";
      bool first = true;
      for (auto& kv : m_slot) {  // m_slot is ordered by offset; indices by first use
        (void)kv;
      }
      std::vector<int> offs(m_slot.size());
      for (auto& kv : m_slot) offs[kv.second] = kv.first;
      for (int v : offs) {
        t += (first ? "" : ",") + std::to_string(v);
        first = false;
      }
      t += "};\n    for (int i = (int)threadIdx.x; i < " + std::to_string(m_slot.size()) + "; i += " +
           std::to_string(nthreads) + ") csm[i] = __ldg(pool + csoff[i]);\n  }\n";
      s.insert(ctab_pos, t);
    }
    if (!ck_slot.empty()) {
      std::string t = "  __shared__ double2 cks[" + std::to_string(ck_slot.size()) + "];\n  {\n";
      for (auto& kv : ck_slot)
        t += "    if (threadIdx.x == " + std::to_string(kv.second % nthreads) + "u) cks[" + std::to_string(kv.second) +
             "] = __ldg(reinterpret_cast<const double2*>(pool) + " + std::to_string(kv.first / 2) + ");\n";
      t += "  }\n";
      s.insert(ctab_pos, t);
    }
    if (n_table)
      s.insert(ctab_pos, "  __shared__ double2 ctab[256];\n  for (int i = (int)threadIdx.x; i < 256; i += " +
                             std::to_string(nthreads) + ") ctab[i] = cis_turns((u64)i << 56);\n");
    return s;
  }
};

// 64-bit word-wise hash of a descriptor (the memo key; the kernel cache key
// is fnv1a of the generated source)
u64 blob_hash(const unsigned char* p, size_t n) {
  u64 h = 0x9E3779B97F4A7C15ull ^ n;
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    u64 w;
    memcpy(&w, p + i, 8);
    h = (h ^ w) * 0xff51afd7ed558ccdull;
    h ^= h >> 29;
  }
  for (; i < n; i++) h = (h ^ p[i]) * 1099511628211ull;
  return h ^ (h >> 31);
}

u64 fnv1a(const std::string& s) {
  u64 h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

// ---------------------------------------------------------- driver access
typedef CUresult (*PFN_ModuleLoadData)(CUmodule*, const void*);
typedef CUresult (*PFN_ModuleGetFunction)(CUfunction*, CUmodule, const char*);
typedef CUresult (*PFN_LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                                     unsigned, unsigned, CUstream, void**, void**);
typedef CUresult (*PFN_LaunchCoop)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                   unsigned, CUstream, void**);
typedef CUresult (*PFN_FuncSetAttribute)(CUfunction, CUfunction_attribute, int);
typedef CUresult (*PFN_OccupancyMax)(int*, CUfunction, int, size_t);
typedef CUresult (*PFN_TensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Driver {
  bool ok = false;
  PFN_ModuleLoadData load = nullptr;
  PFN_ModuleGetFunction getf = nullptr;
  PFN_LaunchKernel launch = nullptr;
  PFN_FuncSetAttribute setattr = nullptr;
  PFN_OccupancyMax occ = nullptr;
  PFN_TensorMapEncodeTiled tmap = nullptr;
  PFN_LaunchCoop launch_coop = nullptr;
};

Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    d.ok = get("cuModuleLoadData", (void**)&d.load) && get("cuModuleGetFunction", (void**)&d.getf) &&
           get("cuLaunchKernel", (void**)&d.launch) &&
           get("cuFuncSetAttribute", (void**)&d.setattr) &&
           get("cuOccupancyMaxActiveBlocksPerMultiprocessor", (void**)&d.occ);
    if (d.ok && !get("cuTensorMapEncodeTiled", (void**)&d.tmap)) d.tmap = nullptr;
    if (d.ok && !get("cuLaunchCooperativeKernel", (void**)&d.launch_coop)) d.launch_coop = nullptr;
  });
  return d;
}

struct Compiled {
  CUfunction f = nullptr;
  int threads = kThreads;
  int blocks_per_sm = 1;
  size_t smem = 0;
  int variant = 0;
  int grid_mult = 1;
};

std::mutex g_mu;
std::unordered_map<u64, Compiled> g_cache;  // key: hash ^ device
std::unordered_map<void*, int> g_threads;   // function -> threads per CTA
struct BlobMemo {
  std::vector<unsigned char> bytes;  // the descriptor (a hit compares it in full)
  u64 src_hash = 0;
};
std::unordered_map<u64, BlobMemo> g_blob_src;  // descriptor hash -> source hash
double g_compile_ms = 0;
uint64_t g_compiles = 0, g_disk_hits = 0;

std::string cache_dir() {
  const char* e = getenv("QS_JIT_CACHE");
  if (e && *e) return e;
  Dl_info info;
  if (dladdr((void*)&fnv1a, &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    size_t k = p.rfind('/');
    if (k != std::string::npos) return p.substr(0, k) + "/jit_cache";
  }
  return "/tmp/qs_jit_cache";
}

bool compile_cubin(const std::string& src, const char* kname, std::vector<char>& cubin,
                   std::string& err) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "qs_pass.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    err = "nvrtcCreateProgram failed";
    return false;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo",
                        "--fmad=true", "-default-device"};
  nvrtcResult rc = nvrtcCompileProgram(prog, 5, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, 0);
    nvrtcGetProgramLog(prog, &log[0]);
    err = std::string("NVRTC: ") + nvrtcGetErrorString(rc) + "\n" + log.substr(0, 2000);
    nvrtcDestroyProgram(&prog);
    return false;
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin.resize(n);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  (void)kname;
  return true;
}
}  // namespace

const char* jit_kernel_name(int kernel) {
  switch (kernel) {
    case KK_CHUNK: return "qs_k1_chunk_jit";
    case KK_DENSE: return "qs_k2_dense_jit";
    default: return "qs_k3_diag_jit";
  }
}

namespace {
struct Source {
  std::string src, err;
  u64 hash = 0;
  size_t smem = 0;
  int threads = kThreads;
  int variant = 0;
  int grid_mult = 1;
  bool ok = false;
};

// run membership of a pass's generated code (f2; see Gen::run_mode)
struct RunOpt {
  bool wait = false, signal = false, throttle = false;
  int sb = 0;
};

Source make_source(const unsigned char* blob, const RunOpt* ro = nullptr) {
  Source r;
  KPass h;
  memcpy(&h, blob, sizeof h);
  const char* kname = jit_kernel_name(h.kernel);
  const bool multi = h.kernel == KK_CHUNK, diag_only = h.kernel == KK_DIAG;
  auto set_run = [&](Gen& x) {
    if (!ro) return;
    x.run_mode = true;
    x.run_wait = ro->wait;
    x.run_signal = ro->signal;
    x.run_throttle = ro->throttle;
    x.run_sb = ro->sb;
  };
  Gen g(h, blob);
  set_run(g);
  r.src = g.build(kname, multi, diag_only);
  r.smem = g.hz_off + (size_t)g.n_hoist * kThreads * 16;
  r.threads = g.nthreads;
  r.variant = g.variant;
  r.grid_mult = g.grid_mult;
  bool bad = g.bad_op;
  // hoists were capped only by the table's 4 KB: if the extra room takes
  // every loop-invariant sincos out of the loop, no table is needed at all
  if (g.hoist_capped) {
    Gen g2(h, blob);
    set_run(g2);
    g2.table_free = true;
    std::string s2 = g2.build(kname, multi, diag_only);
    if (g2.n_table == 0) {
      r.src.swap(s2);
      r.smem = g2.hz_off + (size_t)g2.n_hoist * kThreads * 16;
      r.threads = g2.nthreads;
      r.variant = g2.variant;
      r.grid_mult = g2.grid_mult;
      bad = g2.bad_op;
    }
  }
  if (bad) {
    r.err = "pass contains an op type the kernel generator does not implement";
    return r;
  }
  r.hash = fnv1a(r.src);
  r.ok = true;
  return r;
}

// Run fn(i) for i in [0, n) on up to QS_JIT_THREADS (default: all host
// cores, <= 32) threads.
template <class F>
void parallel_for(size_t n, F fn) {
  int nt = (int)std::thread::hardware_concurrency();
  if (const char* e = getenv("QS_JIT_THREADS")) nt = atoi(e);
  nt = std::max(1, std::min<int>(nt, 32));
  if ((size_t)nt > n) nt = (int)n;
  if (nt <= 1) {
    for (size_t i = 0; i < n; i++) fn(i);
    return;
  }
  std::atomic<size_t> next(0);
  std::vector<std::thread> th;
  for (int t = 0; t < nt; t++)
    th.emplace_back([&] {
      for (size_t i; (i = next.fetch_add(1)) < n;) fn(i);
    });
  for (auto& x : th) x.join();
}

bool read_file(const std::string& path, std::vector<char>& out) {
  FILE* f = fopen(path.c_str(), "rb");
  if (!f) return false;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  out.resize(n > 0 ? n : 0);
  if (n <= 0 || fread(out.data(), 1, n, f) != (size_t)n) out.clear();
  fclose(f);
  return !out.empty();
}
}  // namespace

std::string jit_source(const unsigned char* blob, size_t* smem_bytes = nullptr, int* threads = nullptr) {
  Source r = make_source(blob);
  if (smem_bytes) *smem_bytes = r.smem;
  if (threads) *threads = r.threads;
  return r.src;
}

// Compile (or fetch) the specialised kernels of many passes for `device`
// (the current device): sources are generated and unique sources compiled
// in parallel (NVRTC, one program per thread; disk cache first), then the
// modules are loaded.  compile_only: stop after the cubins (no GPU needed).
// Returns the number of passes that failed (their JitPrepared.err says why).
int jit_prepare_all(const std::vector<const unsigned char*>& blobs, int device,
                    std::vector<JitPrepared>& out, bool compile_only) {
  const size_t n = blobs.size();
  out.assign(n, JitPrepared());
  // Fast path: a descriptor seen before (same bytes: structure AND numbers,
  // e.g. the same circuit again) whose kernel is loaded on this device needs
  // no source generation at all.
  std::vector<u64> bh(n);
  std::vector<char> need(n, 1);
  size_t n_need = 0;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < n; i++) {
      KPass hh;
      memcpy(&hh, blobs[i], sizeof hh);
      bh[i] = blob_hash(blobs[i], hh.total_bytes);
      auto it = g_blob_src.find(bh[i]);
      if (!compile_only && it != g_blob_src.end() && it->second.bytes.size() == hh.total_bytes &&
          memcmp(it->second.bytes.data(), blobs[i], hh.total_bytes) == 0) {
        auto c = g_cache.find(it->second.src_hash ^ ((u64)(device + 1) * 0x9E3779B97F4A7C15ull));
        if (c != g_cache.end()) {
          JitPrepared& P = out[i];
          P.ok = true;
          P.fn = (void*)c->second.f;
          P.per_sm = c->second.blocks_per_sm;
          P.smem = c->second.smem;
          P.threads = c->second.threads;
          P.variant = c->second.variant;
          P.grid_mult = c->second.grid_mult;
          need[i] = 0;
          continue;
        }
      }
      n_need++;
    }
  }
  if (n_need == 0) return 0;
  std::vector<Source> srcs(n);
  std::vector<size_t> todo;
  for (size_t i = 0; i < n; i++)
    if (need[i]) todo.push_back(i);
  parallel_for(todo.size(), [&](size_t t) { srcs[todo[t]] = make_source(blobs[todo[t]]); });
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i : todo)
      if (srcs[i].ok) {
        KPass hh;
        memcpy(&hh, blobs[i], sizeof hh);
        BlobMemo& m = g_blob_src[bh[i]];
        m.bytes.assign(blobs[i], blobs[i] + hh.total_bytes);
        m.src_hash = srcs[i].hash;
      }
  }
  // unique sources that are not loaded on this device yet
  std::map<u64, size_t> uniq;  // hash -> first pass index
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < n; i++) {
      if (!need[i] || !srcs[i].ok) continue;
      const u64 key = srcs[i].hash ^ ((u64)(device + 1) * 0x9E3779B97F4A7C15ull);
      if (!compile_only && g_cache.count(key)) continue;
      uniq.emplace(srcs[i].hash, i);
    }
  }
  std::vector<std::pair<u64, size_t>> work(uniq.begin(), uniq.end());
  std::vector<std::vector<char>> cubins(work.size());
  std::vector<std::string> errs(work.size());
  const std::string dir = cache_dir();
  const char* dump = getenv("QS_JIT_DUMP");  // debugging: keep the generated sources
  parallel_for(work.size(), [&](size_t w) {
    const Source& S = srcs[work[w].second];
    char hx[32];
    snprintf(hx, sizeof hx, "%016llx", (unsigned long long)S.hash);
    KPass h;
    memcpy(&h, blobs[work[w].second], sizeof h);
    const char* kname = jit_kernel_name(h.kernel);
    if (dump) {
      if (FILE* f = fopen((std::string(dump) + "/" + hx + "_" + kname + ".cu").c_str(), "wb")) {
        fwrite(S.src.data(), 1, S.src.size(), f);
        fclose(f);
      }
    }
    const std::string path = dir + "/" + hx + ".cubin";
    if (read_file(path, cubins[w])) {
      std::lock_guard<std::mutex> lk(g_mu);
      g_disk_hits++;
      return;
    }
    auto t0 = std::chrono::steady_clock::now();
    if (!compile_cubin(S.src, kname, cubins[w], errs[w])) {
      cubins[w].clear();
      return;
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    mkdir(dir.c_str(), 0755);
    std::string tmp = path + ".tmp" + std::to_string(getpid()) + "_" + std::to_string(w);
    if (FILE* f = fopen(tmp.c_str(), "wb")) {
      fwrite(cubins[w].data(), 1, cubins[w].size(), f);
      fclose(f);
      rename(tmp.c_str(), path.c_str());
    }
    std::lock_guard<std::mutex> lk(g_mu);
    g_compile_ms += ms;
    g_compiles++;
  });
  std::map<u64, std::string> failed;  // hash -> error
  for (size_t w = 0; w < work.size(); w++)
    if (cubins[w].empty()) failed[work[w].first] = errs[w].empty() ? "compile failed" : errs[w];
  int bad = 0;
  if (compile_only) {
    for (size_t i = 0; i < n; i++) {
      JitPrepared& P = out[i];
      if (!need[i]) continue;
      P.variant = srcs[i].variant;
      P.threads = srcs[i].threads;
      P.smem = srcs[i].smem;
      if (!srcs[i].ok) P.err = srcs[i].err;
      else if (failed.count(srcs[i].hash)) P.err = failed[srcs[i].hash];
      else P.ok = true;
      bad += !P.ok;
    }
    return bad;
  }
  Driver& d = driver();
  std::lock_guard<std::mutex> lk(g_mu);
  for (size_t w = 0; w < work.size(); w++) {
    if (cubins[w].empty()) continue;
    const Source& S = srcs[work[w].second];
    const u64 key = S.hash ^ ((u64)(device + 1) * 0x9E3779B97F4A7C15ull);
    KPass h;
    memcpy(&h, blobs[work[w].second], sizeof h);
    const char* kname = jit_kernel_name(h.kernel);
    CUmodule mod;
    Compiled c;
    if (!d.ok) failed[S.hash] = "CUDA driver entry points unavailable";
    else if (d.load(&mod, cubins[w].data()) != CUDA_SUCCESS) failed[S.hash] = "cuModuleLoadData failed";
    else if (d.getf(&c.f, mod, kname) != CUDA_SUCCESS) failed[S.hash] = "cuModuleGetFunction failed";
    else if (S.smem > 48 * 1024 &&
             d.setattr(c.f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)S.smem) != CUDA_SUCCESS)
      failed[S.hash] = "shared memory request of " + std::to_string(S.smem) + " B refused";
    if (failed.count(S.hash)) continue;
    int nb = 1;
    if (d.occ(&nb, c.f, S.threads, S.smem) != CUDA_SUCCESS || nb < 1) nb = 1;
    c.blocks_per_sm = nb;
    c.smem = S.smem;
    c.threads = S.threads;
    c.variant = S.variant;
    c.grid_mult = S.grid_mult;
    g_cache[key] = c;
    g_threads[(void*)c.f] = S.threads;
  }
  for (size_t i = 0; i < n; i++) {
    JitPrepared& P = out[i];
    if (!need[i]) {
      continue;
    } else if (!srcs[i].ok) {
      P.err = srcs[i].err;
    } else if (failed.count(srcs[i].hash)) {
      P.err = failed[srcs[i].hash];
    } else {
      const u64 key = srcs[i].hash ^ ((u64)(device + 1) * 0x9E3779B97F4A7C15ull);
      auto it = g_cache.find(key);
      if (it == g_cache.end()) {
        P.err = "internal: kernel missing from the cache";
      } else {
        P.ok = true;
        P.fn = (void*)it->second.f;
        P.per_sm = it->second.blocks_per_sm;
        P.smem = it->second.smem;
        P.threads = it->second.threads;
        P.variant = it->second.variant;
        P.grid_mult = it->second.grid_mult;
      }
    }
    bad += !P.ok;
  }
  return bad;
}

// Single-pass form (plan inspection with detail >= 2 compiles one pass).
bool jit_prepare(const unsigned char* blob, int device, void** fn_out, int* grid_per_sm,
                 size_t* smem_out, std::string& err, bool compile_only) {
  std::vector<JitPrepared> r;
  jit_prepare_all({blob}, device, r, compile_only);
  if (!r[0].ok) {
    err = r[0].err;
    return false;
  }
  *fn_out = r[0].fn;
  *grid_per_sm = r[0].per_sm;
  *smem_out = r[0].smem;
  return true;
}

// Bytes of the by-value pool parameter of the specialised kernel of this
// pass (0: the kernel reads its constants from the blob).
size_t jit_param_bytes(const unsigned char* blob) {
  KPass h;
  memcpy(&h, blob, sizeof h);
  const size_t npool = (h.total_bytes - h.off_pool) / sizeof(double);
  return (npool > 0 && npool <= kMaxParamPool) ? npool * sizeof(double) : 0;
}

// Columns of the per-chunk table of this pass (0: no table -- nothing
// chunk-dependent, or too much; the kernel then sums the shapes itself).
int jit_table_cols(const unsigned char* blob, TabCols* v) {
  return table_columns(blob, v, nullptr) ? v->width : 0;
}

// The tensor map of a pass that loads through cp.async.bulk.tensor (see
// tensor_plan; the same conditions as the generator).  false: not such a
// pass (out is zeroed).
bool jit_tensor_map(const unsigned char* blob, const void* state, void* out128) {
  memset(out128, 0, 128);
  KPass h;
  memcpy(&h, blob, sizeof h);
  const int tma_min_l = getenv("QS_JIT_TMA_L") ? atoi(getenv("QS_JIT_TMA_L")) : 5;
  int l = 0;
  while (l < kChunkBits && h.cpos[l] == l) l++;
  TPlan tp;
  if (h.src_mode != 0 || h.kernel == KK_SMALL || l >= tma_min_l || Gen::low_run(h.phases[0]) > 1 ||
      h.pull_j > 0 || !tensor_plan(h, &tp))
    return false;
  Driver& d = driver();
  if (!d.tmap) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], estr[5];
  for (int k = 0; k < tp.rank; k++) {
    dims[k] = k == 0 ? (2ull << tp.len[0]) : (1ull << tp.len[k]);
    box[k] = tp.chunk[k] ? (cuuint32_t)dims[k] : 1u;
    estr[k] = 1;
    if (k > 0) strides[k - 1] = (cuuint64_t)16 << tp.pos[k];
  }
  return d.tmap((CUtensorMap*)out128, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)tp.rank,
                const_cast<void*>(state), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t jit_launch(void* fn, int grid, size_t smem, const unsigned char* dblob,
                       const unsigned char* hblob, double2* state, u64 rank_base, const u64* vtab,
                       const u64* xpeer8, const void* pool_host, size_t pool_bytes, cudaStream_t st,
                       u64 clo, u64 cn) {
  alignas(64) unsigned char tm[128];
  jit_tensor_map(hblob, state, tm);
  Driver& d = driver();
  int threads = kThreads;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_threads.find(fn);
    if (it != g_threads.end()) threads = it->second;
  }
  u64 xp[16];
  memset(xp, 0, sizeof xp);
  if (xpeer8) memcpy(xp, xpeer8, sizeof xp);
  void* args[] = {(void*)&dblob, (void*)&state, (void*)&rank_base, (void*)&vtab, (void*)xp,
                  (void*)tm, (void*)&clo, (void*)&cn, (void*)pool_host};
  if (!pool_bytes) args[8] = nullptr;
  CUresult r = d.launch((CUfunction)fn, (unsigned)grid, 1, 1, (unsigned)threads, 1, 1, (unsigned)smem,
                        (CUstream)st, args, nullptr);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

// ------------------------------------------- co-scheduled runs (f2)
// Two-level blocking (planner
// mark_l2_groups): the K passes of a run execute in ONE cooperative launch.
// Its CTAs are dealt to the passes (contiguous ranges, split.e[i] = first CTA
// after member i); each member runs its own specialised chunk loop (the
// generated pass code as qs_body in namespace qs_rI) over all chunks.  Member
// i > 0 loads a chunk only after member i - 1 has stored every chunk of the
// chunk's 2^(12 + sb)-amplitude block (per-block counters in `flags`, one
// row of nblk per link): the blocks stream through the passes in order a
// few MiB apart, so every member after the first reads them from L2 and the
// state crosses HBM once.  Dependencies only point to lower members and all
// CTAs are co-resident (cooperative launch), so the waits cannot deadlock.
static const char* kRunKernel = "qs_run_jit";

static std::string replace_all(std::string s, const std::string& a, const std::string& b) {
  for (size_t p = s.find(a); p != std::string::npos; p = s.find(a, p + b.size())) s.replace(p, a.size(), b);
  return s;
}

bool jit_prepare_run(const std::vector<const unsigned char*>& blobs, int sb, int device, JitPrepared& out,
                     bool compile_only) {
  out = JitPrepared();
  const int K = (int)blobs.size();
  if (K < 2 || K > kMaxRun) {
    out.err = "run length";
    return false;
  }
  std::vector<Source> m(K);
  for (int i = 0; i < K; i++) {
    RunOpt ro;
    ro.wait = i > 0;
    ro.signal = true;  // the last member's counters throttle the first
    ro.throttle = i == 0;
    ro.sb = sb;
    m[i] = make_source(blobs[i], &ro);
    if (!m[i].ok) {
      out.err = m[i].err;
      return false;
    }
    if (m[i].threads != m[0].threads) {
      out.err = "run members differ in threads per CTA";
      return false;
    }
  }
  std::ostringstream o;
  size_t smem = 0;
  int gm = 1;
  static const bool prof = getenv("QS_RUN_PROF") != nullptr;
  o << "__shared__ unsigned long long qs_wcyc;\n";
  for (int i = 0; i < K; i++) {
    o << "namespace qs_r" << i << " {\n"
      << replace_all(replace_all(m[i].src, "blockIdx.x", "qs_bid"), "gridDim.x", "qs_nbid") << "}\n";
    smem = std::max(smem, m[i].smem);
    gm = std::max(gm, m[i].grid_mult);
  }
  o << "struct __align__(64) QsTmapR { unsigned long long v[16]; };\n"
    << "struct QsSplitR { unsigned int e[" << kMaxRun << "]; };\n"
    << "extern \"C\" __global__ void __launch_bounds__(" << m[0].threads << ", 1)\n" << kRunKernel << "(";
  for (int i = 0; i < K; i++) o << "const unsigned char* __restrict__ b" << i << ", ";
  o << "double2* __restrict__ state, const unsigned long long rank_base, ";
  for (int i = 0; i < K; i++) o << "const unsigned long long* __restrict__ v" << i << ", ";
  for (int i = 0; i < K; i++) o << "const __grid_constant__ QsTmapR t" << i << ", ";
  o << "const unsigned long long n_chunks, unsigned int* __restrict__ flags, const unsigned int nblk, "
       "const QsSplitR split, const unsigned int lag) {\n"
    << "  const unsigned int b = blockIdx.x;\n"
    << (prof ? "  const long long qs_t0 = clock64();\n  if (threadIdx.x == 0) qs_wcyc = 0ull;\n  __syncthreads();\n" : "");
  for (int i = 0; i < K; i++) {
    const std::string lo = i ? "split.e[" + std::to_string(i - 1) + "]" : "0u";
    o << "  " << (i ? "else if" : "if") << " (b < split.e[" << i << "]) {\n"
      << "    const qs_r" << i << "::QsXPeer xz = {};\n"
      << "    qs_r" << i << "::qs_body(b" << i << ", state, rank_base, v" << i << ", xz, reinterpret_cast<const qs_r" << i
      << "::QsTmap&>(t" << i << "), 0ull, n_chunks, b - " << lo << ", split.e[" << i << "] - " << lo << ", "
      << (i ? "flags + (size_t)" + std::to_string(i - 1) + " * nblk" : "nullptr") << ", "
      << "flags + (size_t)" << i << " * nblk, flags + (size_t)" << K - 1 << " * nblk, lag);\n  }\n";
  }
  if (prof)
    o << "  __syncthreads();\n"
         "  if (threadIdx.x == 0 && (b % 8u) == 0u) {\n"
         "    unsigned int r = 0; while (r < " << K - 1 << "u && b >= split.e[r]) r++;\n"
         "    printf(\"qs_run_prof role %u cta %u cycles %lld wait_warp_cycles %llu\\n\", r, b, clock64() - qs_t0, qs_wcyc);\n  }\n";
  o << "}\n";
  const std::string src = o.str();
  const u64 hash = fnv1a(src);
  const u64 key = hash ^ ((u64)(device + 1) * 0x9E3779B97F4A7C15ull);
  static std::unordered_map<u64, std::string> failed;  // a run kernel that did not build: not retried
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto f = failed.find(key);
    if (f != failed.end()) {
      out.err = f->second;
      return false;
    }
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
      out.ok = true;
      out.fn = (void*)it->second.f;
      out.per_sm = it->second.blocks_per_sm;
      out.smem = it->second.smem;
      out.threads = it->second.threads;
      out.grid_mult = it->second.grid_mult;
      out.variant = it->second.variant;
      return true;
    }
  }
  char hx[32];
  snprintf(hx, sizeof hx, "%016llx", (unsigned long long)hash);
  const std::string dir = cache_dir();
  const std::string path = dir + "/" + hx + ".cubin";
  if (const char* dump = getenv("QS_JIT_DUMP"))
    if (FILE* f = fopen((std::string(dump) + "/" + hx + "_" + kRunKernel + ".cu").c_str(), "wb")) {
      fwrite(src.data(), 1, src.size(), f);
      fclose(f);
    }
  std::vector<char> cubin;
  if (read_file(path, cubin)) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_disk_hits++;
  } else {
    std::string err;
    auto t0 = std::chrono::steady_clock::now();
    if (!compile_cubin(src, kRunKernel, cubin, err)) {
      out.err = err;
      std::lock_guard<std::mutex> lk(g_mu);
      failed[key] = err;
      return false;
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    mkdir(dir.c_str(), 0755);
    const std::string tmp = path + ".tmp" + std::to_string(getpid());
    if (FILE* f = fopen(tmp.c_str(), "wb")) {
      fwrite(cubin.data(), 1, cubin.size(), f);
      fclose(f);
      rename(tmp.c_str(), path.c_str());
    }
    std::lock_guard<std::mutex> lk(g_mu);
    g_compile_ms += ms;
    g_compiles++;
  }
  if (compile_only) {
    out.ok = true;
    out.threads = m[0].threads;
    out.smem = smem;
    return true;
  }
  Driver& d = driver();
  if (!d.ok || !d.launch_coop) {
    out.err = "CUDA driver entry points unavailable";
    return false;
  }
  CUmodule mod;
  Compiled c;
  if (d.load(&mod, cubin.data()) != CUDA_SUCCESS || d.getf(&c.f, mod, kRunKernel) != CUDA_SUCCESS) {
    out.err = "run kernel: module load failed";
    return false;
  }
  if (smem > 48 * 1024 && d.setattr(c.f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem) != CUDA_SUCCESS) {
    out.err = "run kernel: shared memory request refused";
    return false;
  }
  int nb = 0;
  if (d.occ(&nb, c.f, m[0].threads, smem) != CUDA_SUCCESS || nb < 1) {
    out.err = "run kernel: does not fit on an SM";
    return false;
  }
  c.blocks_per_sm = nb;
  c.smem = smem;
  c.threads = m[0].threads;
  c.grid_mult = gm;
  c.variant = m[K - 1].variant;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_cache[key] = c;
    g_threads[(void*)c.f] = c.threads;
  }
  out.ok = true;
  out.fn = (void*)c.f;
  out.per_sm = nb;
  out.smem = smem;
  out.threads = c.threads;
  out.grid_mult = gm;
  out.variant = c.variant;
  return true;
}

cudaError_t jit_launch_run(const JitPrepared& jp, int grid, const std::vector<const unsigned char*>& dblobs,
                           const std::vector<const unsigned char*>& hblobs, double2* state, u64 rank_base,
                           const std::vector<const u64*>& vtabs, u64 n_chunks, unsigned* flags, unsigned nblk,
                           const unsigned* split, unsigned lag, cudaStream_t st) {
  const int K = (int)dblobs.size();
  alignas(64) unsigned char tm[kMaxRun][128];
  std::vector<void*> args;
  for (int i = 0; i < K; i++) args.push_back((void*)&dblobs[i]);
  args.push_back((void*)&state);
  args.push_back((void*)&rank_base);
  for (int i = 0; i < K; i++) args.push_back((void*)&vtabs[i]);
  for (int i = 0; i < K; i++) {
    jit_tensor_map(hblobs[i], state, tm[i]);
    args.push_back((void*)tm[i]);
  }
  unsigned sp[kMaxRun];
  for (int i = 0; i < kMaxRun; i++) sp[i] = i < K ? split[i] : 0u;
  args.push_back((void*)&n_chunks);
  args.push_back((void*)&flags);
  args.push_back((void*)&nblk);
  args.push_back((void*)sp);
  args.push_back((void*)&lag);
  Driver& d = driver();
  CUresult r = d.launch_coop((CUfunction)jp.fn, (unsigned)grid, 1, 1, (unsigned)jp.threads, 1, 1, (unsigned)jp.smem,
                             (CUstream)st, args.data());
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

void jit_stats(double* compile_ms, uint64_t* compiles, uint64_t* disk_hits) {
  std::lock_guard<std::mutex> lk(g_mu);
  *compile_ms = g_compile_ms;
  *compiles = g_compiles;
  *disk_hits = g_disk_hits;
}

}  // namespace qs
