// kernels.cu -- sm_100a kernels of the state-vector hot path.
//
//   K1 qs_k1_chunk : cache-blocked gate block (Alg. 2; all-in-one
//                    chunk arm of Alg. 5).  A CTA owns a chunk of
//                    2^12 amplitudes (64 KiB): it loads them with 128-bit
//                    coalesced loads straight into registers (16 amplitudes /
//                    thread), applies every op of the pass whose targets sit in
//                    the current register layout, re-shuffles the chunk through
//                    XOR-swizzled shared memory between layouts ("phases"), and
//                    writes the chunk back (optionally relabelled: the in-pass
//                    qubit reorder of Eq. 4 P:L165-179 at zero extra traffic).
//   K2 qs_k2_dense : the single-layout case (no shared-memory exchange):
//                    fused k<=4 qubit dense matvecs (Eq. 2/3 P:L125-155,
//                    "operate(fusedGate, chunk)" P:L448-449) + diagonals.
//   K3 qs_k3_diag  : diagonal-only pass: alpha_x <- lambda_x alpha_x
//                     with lambda_x = exp(2 pi i Q(x)) evaluated
//                    from the index bits (phase polynomial, see planner.cpp).
//   SMALL          : shards of <= 2^12 amplitudes: whole shard in one CTA.
//   K5             : tensor-product expansion / merge (Alg. 7).
//   K6             : logical-order readout gather.
//
// The path is HBM-bound streaming of complex128 (32 B per amplitude per
// pass); FP64 ALU is the secondary ceiling.  Tensor cores have no FP64 kind
// on tcgen05 and are not used.
#include <cuda_runtime.h>
#include <stdint.h>

#include "qs_internal.hpp"

namespace qs {

static int num_sms();

// ------------------------------------------------------------ primitives
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc + a*b
__device__ __forceinline__ double2 cmac(double2 acc, double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)),
                      fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}

// exp(2 pi i t / 2^64): quadrant from the top bits (exact), then the
// minimax kernel polynomials of fdlibm's __kernel_sin / __kernel_cos (Sun
// Microsystems' freely distributable libm; their published coefficients S1-S6
// and C1-C6) on |x| <= pi/4.
__device__ __forceinline__ double2 cis_turns(u64 t) {
  const u64 q = (t + (1ull << 61)) >> 62;
  const long long f = (long long)(t - (q << 62));
  const double x = (double)f * 3.4061215800865545e-19;  // 2 pi / 2^64
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

__device__ __forceinline__ int swz(int c) {
  return c ^ (((c >> 3) ^ (c >> 6) ^ (c >> 9) ^ (c >> 12)) & 7);
}

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// ------------------------------------------------------- register ops
template <int K>
__device__ __forceinline__ void op_d1(double2 (&a)[kNReg], const double* __restrict__ m,
                                      uint32_t rcm, bool tp) {
  if (!tp) return;
  const double2 u00 = ldg2(m), u01 = ldg2(m + 2), u10 = ldg2(m + 4), u11 = ldg2(m + 6);
#pragma unroll
  for (int r = 0; r < kNReg; r++) {
    if (r & (1 << K)) continue;
    if ((r & rcm) != rcm) continue;
    const int r1 = r | (1 << K);
    const double2 x = a[r], y = a[r1];
    a[r] = cmac(cmul(u00, x), u01, y);
    a[r1] = cmac(cmul(u10, x), u11, y);
  }
}

template <int K>
__device__ __forceinline__ void op_h(double2 (&a)[kNReg], uint32_t rcm, bool tp) {
  if (!tp) return;
  const double h = 0.70710678118654752440;
#pragma unroll
  for (int r = 0; r < kNReg; r++) {
    if (r & (1 << K)) continue;
    if ((r & rcm) != rcm) continue;
    const int r1 = r | (1 << K);
    const double2 x = a[r], y = a[r1];
    a[r] = make_double2((x.x + y.x) * h, (x.y + y.y) * h);
    a[r1] = make_double2((x.x - y.x) * h, (x.y - y.y) * h);
  }
}

template <int K>
__device__ __forceinline__ void op_x(double2 (&a)[kNReg], uint32_t rcm, bool tp) {
  if (!tp) return;
#pragma unroll
  for (int r = 0; r < kNReg; r++) {
    if (r & (1 << K)) continue;
    if ((r & rcm) != rcm) continue;
    const int r1 = r | (1 << K);
    const double2 x = a[r];
    a[r] = a[r1];
    a[r1] = x;
  }
}

// Dense 2^W x 2^W over register bits BITS[0..W) (ascending), matrix bit i <->
// BITS[i].  Loads matrix entries on the fly (uniform, L1-resident).
template <int W, int B0, int B1, int B2, int B3>
__device__ __forceinline__ void op_dn(double2 (&a)[kNReg], const double* __restrict__ m,
                                      uint32_t rcm, bool tp) {
  if (!tp) return;
  constexpr int D = 1 << W;
  constexpr int bits[4] = {B0, B1, B2, B3};
  constexpr int tmask = (W > 0 ? (1 << B0) : 0) | (W > 1 ? (1 << B1) : 0) |
                        (W > 2 ? (1 << B2) : 0) | (W > 3 ? (1 << B3) : 0);
#pragma unroll
  for (int base = 0; base < kNReg; base++) {
    if (base & tmask) continue;
    if ((base & rcm) != rcm) continue;
    double2 v[D];
#pragma unroll
    for (int i = 0; i < D; i++) {
      int r = base;
#pragma unroll
      for (int b = 0; b < W; b++)
        if (i >> b & 1) r |= 1 << bits[b];
      v[i] = a[r];
    }
#pragma unroll
    for (int o = 0; o < D; o++) {
      double2 acc = cmul(ldg2(m + 2 * (o * D)), v[0]);
#pragma unroll
      for (int i = 1; i < D; i++) acc = cmac(acc, ldg2(m + 2 * (o * D + i)), v[i]);
      int r = base;
#pragma unroll
      for (int b = 0; b < W; b++)
        if (o >> b & 1) r |= 1 << bits[b];
      a[r] = acc;
    }
  }
}

// Diagonal group: per-thread subset coefficients -> phases for the subsets of
// the active register bits A.
template <int A>
__device__ __forceinline__ void op_phase(double2 (&a)[kNReg], const u64 (&ang)[kNReg],
                                         bool has_const) {
#pragma unroll
  for (int S = 0; S < kNReg; S++) {
    if (S & ~A) continue;
    if (S == 0 && !has_const) continue;
    const double2 e = cis_turns(ang[S]);
#pragma unroll
    for (int r = 0; r < kNReg; r++)
      if ((r & A) == S) a[r] = cmul(a[r], e);
  }
}

__device__ __forceinline__ void op_diag(double2 (&a)[kNReg], const KOp& op,
                                        const KGroup* __restrict__ groups,
                                        const KShape* __restrict__ shapes,
                                        const u64* scoef, uint32_t tid) {
  const KGroup* G = groups + op.data;
  u64 ang[kNReg];
#pragma unroll
  for (int R = 0; R < kNReg; R++) {
    u64 acc = 0;
    const int e = __ldg(&G->rbeg[R + 1]);
    for (int j = __ldg(&G->rbeg[R]); j < e; j++) {
      const uint32_t tm = __ldg(&shapes[j].tmask);
      if ((tid & tm) == tm) acc += scoef[j];
    }
    ang[R] = acc;
  }
  // zeta transform: ang[S] = sum_{R subset S} coef[R]
#pragma unroll
  for (int k = 0; k < kRegBits; k++)
#pragma unroll
    for (int S = 0; S < kNReg; S++)
      if (S >> k & 1) ang[S] += ang[S ^ (1 << k)];
  const bool hc = op.has_const != 0;
  switch (op.sel) {
#define QS_PH(A) case A: op_phase<A>(a, ang, hc); break;
    QS_PH(0) QS_PH(1) QS_PH(2) QS_PH(3) QS_PH(4) QS_PH(5) QS_PH(6) QS_PH(7)
    QS_PH(8) QS_PH(9) QS_PH(10) QS_PH(11) QS_PH(12) QS_PH(13) QS_PH(14) QS_PH(15)
#undef QS_PH
    default: break;
  }
}

// Fast diagonal group: only the empty subset (if has_const) and the linear
// register bits L have per-thread angles; register-pair terms are constant
// and pre-multiplied on the host into ck[rho] (16 complex, or null).
// phase(rho) = E0 * prod_{k in rho & L} E_k * ck[rho]; rho outside `touch`
// has phase 1 and is skipped.
template <int L>
__device__ __forceinline__ void op_phase_fast(double2 (&a)[kNReg], const u64 (&cf)[kRegBits + 1],
                                              bool has_const, uint32_t touch,
                                              const double* __restrict__ ck) {
  double2 E[kRegBits];
#pragma unroll
  for (int k = 0; k < kRegBits; k++)
    if (L >> k & 1) E[k] = cis_turns(cf[1 + k]);
  const double2 E0 = has_const ? cis_turns(cf[0]) : make_double2(1.0, 0.0);
#pragma unroll
  for (int r = 0; r < kNReg; r++) {
    if (!(touch >> r & 1)) continue;
    double2 g = E0;
    bool first = !has_const;
#pragma unroll
    for (int k = 0; k < kRegBits; k++)
      if ((L >> k & 1) && (r >> k & 1)) {
        g = first ? E[k] : cmul(g, E[k]);
        first = false;
      }
    if (ck) g = first ? ldg2(ck + 2 * r) : cmul(g, ldg2(ck + 2 * r));
    a[r] = cmul(a[r], g);
  }
}

__device__ __forceinline__ void op_diag_fast(double2 (&a)[kNReg], const KOp& op,
                                             const KGroup* __restrict__ groups,
                                             const KShape* __restrict__ shapes,
                                             const double* __restrict__ pool,
                                             const u64* scoef, uint32_t tid) {
  const KGroup* G = groups + op.data;
  u64 cf[kRegBits + 1];
#pragma unroll
  for (int i = 0; i <= kRegBits; i++) {
    const int R = i ? (1 << (i - 1)) : 0;
    u64 acc = 0;
    const int e = __ldg(&G->rbeg[R + 1]);
    for (int j = __ldg(&G->rbeg[R]); j < e; j++) {
      const uint32_t tm = __ldg(&shapes[j].tmask);
      if ((tid & tm) == tm) acc += scoef[j];
    }
    cf[i] = acc;
  }
  const int cko = __ldg(&G->ck_off);
  const double* ck = (cko >= 0) ? pool + cko : nullptr;
  const bool hc = op.has_const != 0;
  const uint32_t touch = op.rcm;
  switch (op.sel) {
#define QS_PF(L) case L: op_phase_fast<L>(a, cf, hc, touch, ck); break;
    QS_PF(0) QS_PF(1) QS_PF(2) QS_PF(3) QS_PF(4) QS_PF(5) QS_PF(6) QS_PF(7)
    QS_PF(8) QS_PF(9) QS_PF(10) QS_PF(11) QS_PF(12) QS_PF(13) QS_PF(14) QS_PF(15)
#undef QS_PF
    default: break;
  }
}

template <int K>
__device__ __forceinline__ void op_hu(double2 (&a)[kNReg]) {
#pragma unroll
  for (int r = 0; r < kNReg; r++) {
    if (r & (1 << K)) continue;
    const int r1 = r | (1 << K);
    const double2 x = a[r], y = a[r1];
    a[r] = make_double2(x.x + y.x, x.y + y.y);
    a[r1] = make_double2(x.x - y.x, x.y - y.y);
  }
}

template <bool DIAG_ONLY>
__device__ __forceinline__ void apply_ops(double2 (&a)[kNReg], const KOp* __restrict__ ops,
                                          int ob, int oe, const double* __restrict__ pool,
                                          const KGroup* __restrict__ groups,
                                          const KShape* __restrict__ shapes,
                                          const u64* scoef, uint32_t tid, u64 tphys_full) {
  for (int o = ob; o < oe; o++) {
    KOp op;
    op.type = __ldg(&ops[o].type);
    op.sel = __ldg(&ops[o].sel);
    op.has_const = __ldg(&ops[o].has_const);
    op.rcm = __ldg(&ops[o].rcm);
    op.ncm = __ldg(&ops[o].ncm);
    op.data = __ldg(&ops[o].data);
    if (op.type == OP_DIAGF) {
      op_diag_fast(a, op, groups, shapes, pool, scoef, tid);
      continue;
    }
    if (op.type == OP_DIAG) {
      op_diag(a, op, groups, shapes, scoef, tid);
      continue;
    }
    if (op.type == OP_DW) continue;  // applied in shared memory (op_wide)
    if constexpr (!DIAG_ONLY) {
      if (op.type == OP_HU) {
        switch (op.sel) {
          case 0: op_hu<0>(a); break;
          case 1: op_hu<1>(a); break;
          case 2: op_hu<2>(a); break;
          default: op_hu<3>(a); break;
        }
        continue;
      }
      const bool tp = (tphys_full & op.ncm) == op.ncm;
      const double* m = pool + op.data;
      const uint32_t rcm = op.rcm;
      switch (op.type) {
        case OP_D1:
          switch (op.sel) {
            case 0: op_d1<0>(a, m, rcm, tp); break;
            case 1: op_d1<1>(a, m, rcm, tp); break;
            case 2: op_d1<2>(a, m, rcm, tp); break;
            default: op_d1<3>(a, m, rcm, tp); break;
          }
          break;
        case OP_H:
          switch (op.sel) {
            case 0: op_h<0>(a, rcm, tp); break;
            case 1: op_h<1>(a, rcm, tp); break;
            case 2: op_h<2>(a, rcm, tp); break;
            default: op_h<3>(a, rcm, tp); break;
          }
          break;
        case OP_X:
          switch (op.sel) {
            case 0: op_x<0>(a, rcm, tp); break;
            case 1: op_x<1>(a, rcm, tp); break;
            case 2: op_x<2>(a, rcm, tp); break;
            default: op_x<3>(a, rcm, tp); break;
          }
          break;
        case OP_D2:
          switch (op.sel) {
            case 0: op_dn<2, 0, 1, 0, 0>(a, m, rcm, tp); break;
            case 1: op_dn<2, 0, 2, 0, 0>(a, m, rcm, tp); break;
            case 2: op_dn<2, 0, 3, 0, 0>(a, m, rcm, tp); break;
            case 3: op_dn<2, 1, 2, 0, 0>(a, m, rcm, tp); break;
            case 4: op_dn<2, 1, 3, 0, 0>(a, m, rcm, tp); break;
            default: op_dn<2, 2, 3, 0, 0>(a, m, rcm, tp); break;
          }
          break;
        case OP_D3:
          switch (op.sel) {  // sel = the register bit NOT in the op
            case 0: op_dn<3, 1, 2, 3, 0>(a, m, rcm, tp); break;
            case 1: op_dn<3, 0, 2, 3, 0>(a, m, rcm, tp); break;
            case 2: op_dn<3, 0, 1, 3, 0>(a, m, rcm, tp); break;
            default: op_dn<3, 0, 1, 2, 0>(a, m, rcm, tp); break;
          }
          break;
        default:
          __trap();  // an op this kernel does not know: never skip silently
      }
    }
  }
}

// Wide dense op (OP_DW, k = 5..6 targets; Eq. 3 generalised) on
// the chunk staged in shared memory (swizzled slots, chunk index c at
// swz(c)).  Thread t owns base b = t >> (k-4) (the chunk index with the
// target bits zero, deposited over the other chunk bits) and the 16 output
// rows (t & (2^(k-4)-1)) * 16 + j: it reads the 2^k inputs of its base,
// accumulates its 16 rows, and after a CTA barrier writes them back.
__device__ void op_wide(double2* sch, const KOp& op, const double* __restrict__ pool, u64 cphys,
                        uint32_t tid) {
  const int k = op.k, D = 1 << k, g = k - kRegBits;
  int tm = 0;
  for (int i = 0; i < k; i++) tm |= 1 << op.tpos[i];
  const uint32_t b = tid >> g, rg = tid & ((1u << g) - 1);
  int cbase = 0, bi = 0;
  for (int c = 0; c < kChunkBits; c++)
    if (!(tm >> c & 1)) cbase |= (int)((b >> bi++) & 1u) << c;
  const bool act = ((cphys & op.ncm) == op.ncm) && ((cbase & (int)op.rcm) == (int)op.rcm);
  auto dep = [&](int r) {
    int x = cbase;
    for (int i = 0; i < k; i++) x |= ((r >> i) & 1) << op.tpos[i];
    return x;
  };
  const double* m = pool + op.data;
  double2 acc[kNReg];
#pragma unroll
  for (int j = 0; j < kNReg; j++) acc[j] = make_double2(0.0, 0.0);
  if (act)
    for (int c = 0; c < D; c++) {
      const double2 v = sch[swz(dep(c))];
#pragma unroll
      for (int j = 0; j < kNReg; j++) acc[j] = cmac(acc[j], ldg2(m + 2 * ((size_t)((rg << kRegBits) + j) * D + c)), v);
    }
  __syncthreads();
  if (act)
#pragma unroll
    for (int j = 0; j < kNReg; j++) sch[swz(dep((int)(rg << kRegBits) + j))] = acc[j];
}

// ---------------------------------------------------------- pass kernels
struct Layout {
  int tc;           // chunk index bits of this thread
  u64 tphys;        // physical offset of this thread (load positions)
  int rc[kRegBits];
  u64 rphys[kRegBits];
};

__device__ __forceinline__ void make_layout(const KPass& P, int p, uint32_t tid, bool out,
                                            Layout& L) {
  const KPhase& ph = P.phases[p];
  const int8_t* pos = out ? P.opos : P.cpos;
  int tc = 0;
  u64 tphys = 0;
#pragma unroll
  for (int i = 0; i < kLogT; i++)
    if (tid >> i & 1) {
      const int c = ph.thr_c[i];
      tc |= 1 << c;
      tphys |= 1ull << pos[c];
    }
  L.tc = tc;
  L.tphys = tphys;
#pragma unroll
  for (int k = 0; k < kRegBits; k++) {
    L.rc[k] = 1 << ph.reg_c[k];
    L.rphys[k] = 1ull << pos[ph.reg_c[k]];
  }
}

__device__ __forceinline__ u64 reg_off(const Layout& L, int r) {
  u64 o = 0;
#pragma unroll
  for (int k = 0; k < kRegBits; k++)
    if (r >> k & 1) o |= L.rphys[k];
  return o;
}
__device__ __forceinline__ int reg_c(const Layout& L, int r) {
  int o = 0;
#pragma unroll
  for (int k = 0; k < kRegBits; k++)
    if (r >> k & 1) o |= L.rc[k];
  return o;
}

__device__ __forceinline__ u64 deposit_runs(const KPass& P, u64 id) {
  u64 b = 0;
  for (int i = 0; i < P.n_runs; i++)
    b |= ((id >> P.run_src[i]) & ((1ull << P.run_len[i]) - 1)) << P.run_dst[i];
  return b;
}

__device__ __forceinline__ double2 expand_amp(const KPass& P, u64 phys) {
  double2 v = make_double2(1.0, 0.0);
  for (int g = 0; g < P.expand.n; g++) {
    const double2* s = reinterpret_cast<const double2*>(P.expand.ptr[g]);
    const u64 idx = (phys >> P.expand.lo[g]) & ((1ull << P.expand.len[g]) - 1);
    v = cmul(v, __ldg(s + idx));
  }
  return v;
}

// MODE 0: K1 multi-phase (smem exchange); 1: K2 single phase; 2: K3 diag only.
template <int MODE>
__global__ void __launch_bounds__(kThreads, 2)
qs_kpass(const unsigned char* __restrict__ blob, double2* __restrict__ state) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ KPass P;
  const uint32_t tid = threadIdx.x;
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(blob);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&P);
    for (uint32_t i = tid; i < sizeof(KPass) / 4; i += kThreads) dst[i] = src[i];
  }
  __syncthreads();
  constexpr int NC = 1 << kChunkBits;
  double2* sch = reinterpret_cast<double2*>(smem_raw);
  u64* scoef = reinterpret_cast<u64*>(smem_raw + (MODE == 0 ? NC * sizeof(double2) : 0));
  const KOp* ops = reinterpret_cast<const KOp*>(blob + P.off_ops);
  const KGroup* groups = reinterpret_cast<const KGroup*>(blob + P.off_groups);
  const KShape* shapes = reinterpret_cast<const KShape*>(blob + P.off_shapes);
  const KTerm* terms = reinterpret_cast<const KTerm*>(blob + P.off_terms);
  const double* pool = reinterpret_cast<const double*>(blob + P.off_pool);
  const int nph = (MODE == 0) ? P.n_phases : 1;
  const int nsh = P.n_shapes;

  for (u64 chunk = blockIdx.x; chunk < P.n_chunks; chunk += gridDim.x) {
    const u64 cb = deposit_runs(P, chunk);        // local bits of the chunk
    const u64 cphys = cb | P.rank_base;           // incl. rank bits
    if (nsh) {
      __syncthreads();
      for (int j = tid; j < nsh; j += kThreads) {
        u64 acc = 0;
        const int e = __ldg(&shapes[j].term_end);
        for (int q = __ldg(&shapes[j].term_begin); q < e; q++) {
          const u64 m = __ldg(&terms[q].ncmask);
          if ((cphys & m) == m) acc += __ldg(&terms[q].coeff);
        }
        scoef[j] = acc;
      }
      __syncthreads();
    }
    double2 a[kNReg];
    Layout L;
    make_layout(P, 0, tid, false, L);
    if (P.src_mode == 1) {
#pragma unroll
      for (int r = 0; r < kNReg; r++) a[r] = expand_amp(P, cphys | L.tphys | reg_off(L, r));
    } else if (P.src_mode == 2) {
#pragma unroll
      for (int r = 0; r < kNReg; r++)
        a[r] = make_double2((cphys | L.tphys | reg_off(L, r)) == P.basis ? 1.0 : 0.0, 0.0);
    } else {
#pragma unroll
      for (int r = 0; r < kNReg; r++) a[r] = state[cb | L.tphys | reg_off(L, r)];
    }
    int p = 0;
    for (;;) {
      const KPhase& ph = P.phases[p];
      apply_ops<MODE == 2>(a, ops, ph.op_begin, ph.op_end, pool, groups, shapes, scoef, tid,
                           cphys | L.tphys);
      if constexpr (MODE == 0) {
        if (++p >= nph) break;
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kNReg; r++) sch[swz(L.tc | reg_c(L, r))] = a[r];
        make_layout(P, p, tid, false, L);
        __syncthreads();
        {
          const int ob = P.phases[p].op_begin;
          if (ob < P.phases[p].op_end && __ldg(&ops[ob].type) == OP_DW) {
            KOp w;
            w.type = OP_DW;
            w.k = __ldg(&ops[ob].k);
            w.rcm = __ldg(&ops[ob].rcm);
            w.ncm = __ldg(&ops[ob].ncm);
            w.data = __ldg(&ops[ob].data);
            for (int i = 0; i < 8; i++) w.tpos[i] = __ldg(&ops[ob].tpos[i]);
            op_wide(sch, w, pool, cphys, tid);
            __syncthreads();
          }
        }
#pragma unroll
        for (int r = 0; r < kNReg; r++) a[r] = sch[swz(L.tc | reg_c(L, r))];
      } else {
        break;
      }
    }
    Layout O;
    make_layout(P, nph - 1, tid, true, O);
    if (P.scale_im != 0.0) {
      const double2 sc = make_double2(P.scale, P.scale_im);
#pragma unroll
      for (int r = 0; r < kNReg; r++) a[r] = cmul(a[r], sc);
    } else if (P.scale != 1.0) {
      const double sc = P.scale;
#pragma unroll
      for (int r = 0; r < kNReg; r++) a[r] = make_double2(a[r].x * sc, a[r].y * sc);
    }
#pragma unroll
    for (int r = 0; r < kNReg; r++) state[cb | O.tphys | reg_off(O, r)] = a[r];
  }
}

// --------------------------------------------------------------- SMALL
// Whole shard (nl <= 12) in shared memory; ops applied one by one.
__global__ void __launch_bounds__(kThreads)
qs_ksmall(const unsigned char* __restrict__ blob, double2* __restrict__ state) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* s = reinterpret_cast<double2*>(smem_raw);
  const KPass& P = *reinterpret_cast<const KPass*>(blob);
  const KOp* ops = reinterpret_cast<const KOp*>(blob + P.off_ops);
  const KTerm* terms = reinterpret_cast<const KTerm*>(blob + P.off_terms);
  const double* pool = reinterpret_cast<const double*>(blob + P.off_pool);
  const int nl = P.nl;
  const u64 rb = P.rank_base;
  const int size = 1 << nl;
  const int tid = threadIdx.x;
  for (int i = tid; i < size; i += blockDim.x) {
    if (P.src_mode == 1) s[i] = expand_amp(P, rb | (u64)i);
    else if (P.src_mode == 2) s[i] = make_double2((rb | (u64)i) == P.basis ? 1.0 : 0.0, 0.0);
    else s[i] = state[i];
  }
  __syncthreads();
  for (int o = 0; o < P.n_ops; o++) {
    const KOp& op = ops[o];
    if (op.type == OP_SDIAG) {
      const int tb = op.data, te = op.data + op.data2;
      for (int i = tid; i < size; i += blockDim.x) {
        const u64 ph = rb | (u64)i;
        u64 ang = 0;
        for (int q = tb; q < te; q++)
          if ((ph & terms[q].ncmask) == terms[q].ncmask) ang += terms[q].coeff;
        if (ang) s[i] = cmul(s[i], cis_turns(ang));
      }
    } else {
      const int k = op.k;
      const int D = 1 << k;
      int sorted[8];
      for (int i = 0; i < k; i++) sorted[i] = op.tpos[i];
      for (int i = 1; i < k; i++)
        for (int j = i; j > 0 && sorted[j - 1] > sorted[j]; j--) {
          int t = sorted[j]; sorted[j] = sorted[j - 1]; sorted[j - 1] = t;
        }
      const double* m = pool + op.data;
      const int nb = size >> k;
      for (int b = tid; b < nb; b += blockDim.x) {
        int idx = b;
        for (int i = 0; i < k; i++) {
          const int p = sorted[i];
          idx = ((idx >> p) << (p + 1)) | (idx & ((1 << p) - 1));
        }
        if ((((u64)idx | rb) & op.ncm) != op.ncm) continue;
        double2 v[64];
        for (int r = 0; r < D; r++) {
          int j = idx;
          for (int i = 0; i < k; i++)
            if (r >> i & 1) j |= 1 << op.tpos[i];
          v[r] = s[j];
        }
        for (int r = 0; r < D; r++) {
          double2 acc = make_double2(0.0, 0.0);
          for (int c = 0; c < D; c++) acc = cmac(acc, ldg2(m + 2 * (r * D + c)), v[c]);
          int j = idx;
          for (int i = 0; i < k; i++)
            if (r >> i & 1) j |= 1 << op.tpos[i];
          s[j] = acc;
        }
      }
    }
    __syncthreads();
  }
  for (int i = tid; i < size; i += blockDim.x) state[i] = s[i];
}

// ---------------------------------------------------------- K5 / init / K6
__global__ void qs_kexpand(double2* __restrict__ dst, u64 n_amps, u64 rank_base, KExpand e) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n_amps;
       i += (u64)gridDim.x * blockDim.x) {
    const u64 phys = rank_base | i;
    double2 v = make_double2(1.0, 0.0);
    for (int g = 0; g < e.n; g++) {
      const double2* s = reinterpret_cast<const double2*>(e.ptr[g]);
      v = cmul(v, __ldg(s + ((phys >> e.lo[g]) & ((1ull << e.len[g]) - 1))));
    }
    dst[i] = v;
  }
}

__global__ void qs_kmerge(double2* __restrict__ dst, const double2* __restrict__ A, int la,
                          const double2* __restrict__ B, int lb) {
  const u64 n = 1ull << (la + lb);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
       i += (u64)gridDim.x * blockDim.x)
    dst[i] = cmul(A[i & ((1ull << la) - 1)], B[i >> la]);
}

// Local bit permutation (exchange bit a[i] <-> b[i]): out[pi(x)] = in[x].
// Used before a global swap whose victim qubits are not at the top local
// positions (pieces must be contiguous for the exchange).
struct KPerm {
  int8_t a[8], b[8];
  int n;
};
__global__ void qs_kpermute(const double2* __restrict__ in, double2* __restrict__ out, u64 n_amps,
                            KPerm p) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n_amps;
       i += (u64)gridDim.x * blockDim.x) {
    u64 j = i;
    for (int k = 0; k < p.n; k++) {
      const u64 x = ((i >> p.a[k]) ^ (i >> p.b[k])) & 1ull;
      j ^= (x << p.a[k]) | (x << p.b[k]);
    }
    out[j] = in[i];
  }
}

cudaError_t launch_permute(const double2* in, double2* out, u64 n_amps, const int* a, const int* b,
                           int n, cudaStream_t st) {
  KPerm p;
  p.n = n;
  for (int k = 0; k < n && k < 8; k++) {
    p.a[k] = (int8_t)a[k];
    p.b[k] = (int8_t)b[k];
  }
  u64 blocks = (n_amps + 255) / 256;
  u64 cap = (u64)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  qs_kpermute<<<(unsigned)blocks, 256, 0, st>>>(in, out, n_amps, p);
  return cudaGetLastError();
}

__global__ void qs_kset_one(double2* __restrict__ dst, u64 idx) {
  dst[idx] = make_double2(1.0, 0.0);
}

// out[i] = amplitude of logical index off+i if it lives in this shard, else 0.
__global__ void qs_kgather(const double2* __restrict__ state, double2* __restrict__ out,
                           u64 off, u64 count, int n, const int8_t* __restrict__ map,
                           int nl, u64 rank, int probs) {
  __shared__ int8_t smap[64];
  if (threadIdx.x < 64) smap[threadIdx.x] = threadIdx.x < n ? map[threadIdx.x] : 0;
  __syncthreads();
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count;
       i += (u64)gridDim.x * blockDim.x) {
    const u64 L = off + i;
    u64 ph = 0;
    for (int q = 0; q < n; q++) ph |= ((L >> q) & 1ull) << smap[q];
    double2 v = make_double2(0.0, 0.0);
    if ((ph >> nl) == rank) v = state[ph & ((1ull << nl) - 1)];
    if (probs) {
      reinterpret_cast<double*>(out)[i] = v.x * v.x + v.y * v.y;
    } else {
      out[i] = v;
    }
  }
}

// ------------------------------------------------------------- launchers
static int g_num_sms = 0;

static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

cudaError_t launch_pass(int kernel, const unsigned char* dblob, const KPass& hdr,
                        double2* state, cudaStream_t st) {
  const size_t scoef_bytes = (size_t)hdr.n_shapes * sizeof(u64);
  if (kernel == KK_SMALL) {
    const size_t smem = ((size_t)1 << hdr.nl) * sizeof(double2);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(qs_ksmall, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    qs_ksmall<<<1, kThreads, smem, st>>>(dblob, state);
    return cudaGetLastError();
  }
  const u64 nchunks = hdr.n_chunks;
  int per_sm = 2;
  u64 grid = (u64)num_sms() * per_sm;
  if (grid > nchunks) grid = nchunks;
  if (kernel == KK_CHUNK) {
    const size_t smem = ((size_t)1 << kChunkBits) * sizeof(double2) + scoef_bytes;
    cudaFuncSetAttribute(qs_kpass<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    qs_kpass<0><<<(unsigned)grid, kThreads, smem, st>>>(dblob, state);
  } else if (kernel == KK_DENSE) {
    const size_t smem = scoef_bytes;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(qs_kpass<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    qs_kpass<1><<<(unsigned)grid, kThreads, smem, st>>>(dblob, state);
  } else {
    const size_t smem = scoef_bytes;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(qs_kpass<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    qs_kpass<2><<<(unsigned)grid, kThreads, smem, st>>>(dblob, state);
  }
  return cudaGetLastError();
}

cudaError_t launch_expand(double2* dst, u64 n_amps, u64 rank_base, const KExpand& e,
                          cudaStream_t st) {
  u64 blocks = (n_amps + 255) / 256;
  u64 cap = (u64)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  qs_kexpand<<<(unsigned)blocks, 256, 0, st>>>(dst, n_amps, rank_base, e);
  return cudaGetLastError();
}

cudaError_t launch_merge(double2* dst, const double2* A, int la, const double2* B, int lb,
                         cudaStream_t st) {
  u64 n = 1ull << (la + lb);
  u64 blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  qs_kmerge<<<(unsigned)blocks, 256, 0, st>>>(dst, A, la, B, lb);
  return cudaGetLastError();
}

// The per-chunk table of a specialised pass (TabCols, qs_internal.hpp): for
// every chunk c, the level-1 sums of the listed chunk-dependent shapes (the
// sum of the coefficients of the shape's terms whose non-chunk mask is set
// in chunk c's physical base -- what the interpreter computes per chunk in
// shared memory), and for each cis column exp(2 pi i S / 2^64) of the summed
// shapes S of one diagonal slot.
__device__ __forceinline__ u64 shape_level1(const KShape* S, const KTerm* T, int j, u64 cphys) {
  u64 acc = 0;
  for (int q = S[j].term_begin; q < S[j].term_end; q++) {
    const u64 mk = T[q].ncmask;
    if ((cphys & mk) == mk) acc += T[q].coeff;
  }
  return acc;
}

__global__ void qs_kshape_table(const unsigned char* __restrict__ blob, u64* __restrict__ tab,
                                u64 rank_base, TabCols v) {
  const KPass& P = *reinterpret_cast<const KPass*>(blob);
  const KShape* S = reinterpret_cast<const KShape*>(blob + P.off_shapes);
  const KTerm* T = reinterpret_cast<const KTerm*>(blob + P.off_terms);
  // One thread per chunk row, every column: the shape/term loops are the
  // same for all lanes (uniform branches, broadcast term loads) -- one
  // thread per (row, column) entry diverged across columns and ran ~8x
  // slower (QFT-30's write-only pass table: 148 us on the critical path)
  const int apad = (v.n_ang + 1) & ~1;
  if (P.n_chunks < 4096) {
    // few rows (sub-state passes): one thread per (row, column) entry keeps
    // the GPU busy (8 rows x all columns per thread took 12 vs 5 us)
    const int ncol = v.n_ang + v.n_cis;
    const u64 total = P.n_chunks * (u64)ncol;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (u64)gridDim.x * blockDim.x) {
      const u64 c = i / (u64)ncol;
      const int t = (int)(i - c * (u64)ncol);
      const u64 cphys = deposit_runs(P, c) | rank_base;
      u64* row = tab + c * (u64)v.width;
      if (t < v.n_ang) {
        row[t] = shape_level1(S, T, v.ang[t], cphys);
      } else {
        const int e = t - v.n_ang;
        u64 th = 0;
        for (int q = v.cis_beg[e]; q < v.cis_beg[e + 1]; q++) th += shape_level1(S, T, v.cis_shape[q], cphys);
        reinterpret_cast<double2*>(row + apad)[e] = cis_turns(th);
      }
    }
    return;
  }
  for (u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x; c < P.n_chunks; c += (u64)gridDim.x * blockDim.x) {
    const u64 cphys = deposit_runs(P, c) | rank_base;
    u64* row = tab + c * (u64)v.width;
    for (int t = 0; t < v.n_ang; t++) row[t] = shape_level1(S, T, v.ang[t], cphys);
    for (int e = 0; e < v.n_cis; e++) {
      u64 th = 0;
      for (int q = v.cis_beg[e]; q < v.cis_beg[e + 1]; q++) th += shape_level1(S, T, v.cis_shape[q], cphys);
      reinterpret_cast<double2*>(row + apad)[e] = cis_turns(th);
    }
  }
}

cudaError_t launch_shape_table(const unsigned char* dblob, u64* tab, u64 rank_base, u64 n_chunks,
                               const TabCols& v, cudaStream_t st) {
  u64 blocks = (n_chunks * (n_chunks < 4096 ? (u64)(v.n_ang + v.n_cis) : 1ull) + 255) / 256;
  u64 cap = (u64)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  qs_kshape_table<<<(unsigned)blocks, 256, 0, st>>>(dblob, tab, rank_base, v);
  return cudaGetLastError();
}

cudaError_t launch_set_one(double2* dst, u64 idx, cudaStream_t st) {
  qs_kset_one<<<1, 1, 0, st>>>(dst, idx);
  return cudaGetLastError();
}

cudaError_t launch_gather(const double2* state, double2* out, u64 off, u64 count, int n,
                          const int8_t* dmap, int nl, u64 rank, int probs, cudaStream_t st) {
  u64 blocks = (count + 255) / 256;
  u64 cap = (u64)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  qs_kgather<<<(unsigned)blocks, 256, 0, st>>>(state, out, off, count, n, dmap, nl, rank, probs);
  return cudaGetLastError();
}

}  // namespace qs
