/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * gate-by-gate state-vector simulator used to check the CUDA path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product library
 * (paper_2604_12256_b200/libqs.so) shares no code, header, table or helper
 * with this file, and neither side includes or links the other.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   - Alg. 1 "Gate-by-gate simulation scheme": for each
 *     gate in circuit order, traverse and update the whole state vector.
 *   - Eq. 2 (L125-137) and Eq. 3 (L139-155) generalised to t targets and c
 *     controls (SURVEY 8(c) "Definition"): for every index b whose target bits
 *     are 0 and whose control bits are all 1, gather v[r] = psi[b | sum_i
 *     r_i 2^targets[i]] for r in [0, 2^t), then psi[...] <- U v.
 *     Matrix index bit i <-> targets[i] (reading c2); listing the
 *     targets ascending reproduces Eq. 3's row order 0_j0_k,0_j1_k,1_j0_k,1_j1_k
 *     with j > k.
 *   - Qubit 0 is the least significant bit of the amplitude index (reading c1).
 *   - Amplitudes are complex128, "two 64-bit floating-point numbers"
 *     (PAPER.md L112).
 *   - Gate matrices: DESIGN.md reading c3 (the paper names gates but does not
 *     define matrices); written here independently of the product's table.
 *   - Diagonal gates (Z, S, T, RZ, U1, CZ, CP, RZZ, GENERIC_DIAGONAL) are
 *     applied through the same dense gather/matvec/scatter definition with
 *     their full 2^t x 2^t matrix: no diagonal shortcut, no fusion, no
 *     reordering.  (PAPER.md L634-650 defines the fused diagonal as
 *     "thread_i ... complex multiplication between lambda_i and alpha_i",
 *     which is the special case of this definition.)
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): brute-force Kronecker-product
 * unitaries for N<=6 built from PAPER.md L125's U_j = I^{N-j-1} (x) U (x) I^j,
 * tensor-contraction application, QFT / GHZ closed forms, norm preservation,
 * gate-table identities (expm of Pauli generators, squares of sqrt gates),
 * SPEC.md worked examples.
 *
 * Threading: one OpenMP "parallel for" over the base index b; no other change
 * to the plain loop.
 */
#define _GNU_SOURCE
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

/* Gate kinds of the oracle (its own numbering; the Python wrapper maps the
 * workload's kind names to these). */
enum {
  OK_H = 0, OK_X, OK_Y, OK_Z, OK_S, OK_T, OK_RX, OK_RY, OK_RZ, OK_U1, OK_U2,
  OK_U3, OK_CX, OK_CZ, OK_CP, OK_RZZ, OK_SWAP, OK_SX, OK_SY, OK_SW,
  OK_GENERIC_UNITARY, OK_GENERIC_DIAGONAL, OK_SDG, OK_TDG, OK_NKINDS
};

#define ORACLE_MAX_T 10

/* Number of target qubits a kind acts on (-1: given by the caller). */
static int kind_targets(int kind) {
  switch (kind) {
    case OK_RZZ: case OK_SWAP: return 2;
    case OK_GENERIC_UNITARY: case OK_GENERIC_DIAGONAL: return -1;
    default: return 1;
  }
}

/*
 * Fill out[dim*dim] (row-major, dim = 2^t) with the gate matrix over its
 * targets.  Reading c3 of DESIGN.md (c = cos(theta/2), s = sin(theta/2)).
 * Returns 0, or -1 for an unknown kind / bad arity.
 */
int oracle_gate_matrix(int kind, int t, const double *params,
                       const double *user, double *out_interleaved) {
  int dim = 1 << t;
  cplx *m = (cplx *)calloc((size_t)dim * dim, sizeof(cplx));
  if (!m) return -1;
  int want = kind_targets(kind);
  if (want >= 0 && want != t) { free(m); return -1; }
  const double r2 = 1.0 / sqrt(2.0);
  double th = params ? params[0] : 0.0;
  double c = cos(th / 2), s = sin(th / 2);
  switch (kind) {
    case OK_H:  m[0] = r2; m[1] = r2; m[2] = r2; m[3] = -r2; break;
    case OK_X: case OK_CX: m[1] = 1; m[2] = 1; break;
    case OK_Y:  m[1] = -I; m[2] = I; break;
    case OK_Z: case OK_CZ: m[0] = 1; m[3] = -1; break;
    case OK_S:  m[0] = 1; m[3] = I; break;
    case OK_SDG: m[0] = 1; m[3] = -I; break;
    case OK_T:  m[0] = 1; m[3] = cexp(I * M_PI / 4); break;
    case OK_TDG: m[0] = 1; m[3] = cexp(-I * M_PI / 4); break;
    case OK_RX: m[0] = c; m[1] = -I * s; m[2] = -I * s; m[3] = c; break;
    case OK_RY: m[0] = c; m[1] = -s; m[2] = s; m[3] = c; break;
    case OK_RZ: m[0] = cexp(-I * th / 2); m[3] = cexp(I * th / 2); break;
    case OK_U1: case OK_CP: m[0] = 1; m[3] = cexp(I * th); break;
    case OK_U2: {  /* OpenQASM 2.0: u2(phi, lambda) */
      double phi = params[0], lam = params[1];
      m[0] = r2; m[1] = -r2 * cexp(I * lam);
      m[2] = r2 * cexp(I * phi); m[3] = r2 * cexp(I * (phi + lam));
      break;
    }
    case OK_U3: {  /* OpenQASM 2.0: u3(theta, phi, lambda) */
      double phi = params[1], lam = params[2];
      m[0] = c; m[1] = -cexp(I * lam) * s;
      m[2] = cexp(I * phi) * s; m[3] = cexp(I * (phi + lam)) * c;
      break;
    }
    case OK_RZZ:  /* diag(e^{-i th/2}, e^{i th/2}, e^{i th/2}, e^{-i th/2}) */
      m[0] = cexp(-I * th / 2); m[5] = cexp(I * th / 2);
      m[10] = cexp(I * th / 2); m[15] = cexp(-I * th / 2);
      break;
    case OK_SWAP: m[0] = 1; m[6] = 1; m[9] = 1; m[15] = 1; break;
    /* sqrt(P) := ((1+i)/2)(I - iP) for P in {X, Y, W=(X+Y)/sqrt2} */
    case OK_SX: {
      cplx a = (1 + I) / 2;
      m[0] = a; m[1] = a * (-I); m[2] = a * (-I); m[3] = a;
      break;
    }
    case OK_SY: {
      cplx a = (1 + I) / 2;
      /* -iY = [[0,-1],[1,0]] */
      m[0] = a; m[1] = -a; m[2] = a; m[3] = a;
      break;
    }
    case OK_SW: {
      cplx a = (1 + I) / 2;
      /* W = (X+Y)/sqrt2 = [[0, (1-i)/sqrt2], [(1+i)/sqrt2, 0]] */
      cplx w01 = (1 - I) * r2, w10 = (1 + I) * r2;
      m[0] = a; m[1] = a * (-I) * w01; m[2] = a * (-I) * w10; m[3] = a;
      break;
    }
    case OK_GENERIC_UNITARY:
      for (int i = 0; i < dim * dim; i++)
        m[i] = user[2 * i] + I * user[2 * i + 1];
      break;
    case OK_GENERIC_DIAGONAL:
      for (int i = 0; i < dim; i++)
        m[i * dim + i] = user[2 * i] + I * user[2 * i + 1];
      break;
    default: free(m); return -1;
  }
  for (int i = 0; i < dim * dim; i++) {
    out_interleaved[2 * i] = creal(m[i]);
    out_interleaved[2 * i + 1] = cimag(m[i]);
  }
  free(m);
  return 0;
}

/*
 * Apply one gate (Eq. 2/3 generalised) to psi[2^n] (interleaved complex128).
 * Returns 0 or -1 on invalid input (index out of range, overlap, bad kind).
 */
int oracle_apply_gate(double *psi_interleaved, int n, int kind, int t,
                      const int *targets, int nc, const int *controls,
                      const double *params, const double *user_matrix) {
  if (t < 1 || t > ORACLE_MAX_T || nc < 0) return -1;
  uint64_t tmask = 0, cmask = 0;
  for (int i = 0; i < t; i++) {
    if (targets[i] < 0 || targets[i] >= n) return -1;
    if (tmask & (1ull << targets[i])) return -1;
    tmask |= 1ull << targets[i];
  }
  for (int i = 0; i < nc; i++) {
    if (controls[i] < 0 || controls[i] >= n) return -1;
    if ((tmask | cmask) & (1ull << controls[i])) return -1;
    cmask |= 1ull << controls[i];
  }
  int dim = 1 << t;
  double *mi = (double *)malloc(sizeof(double) * 2 * dim * dim);
  if (!mi) return -1;
  if (oracle_gate_matrix(kind, t, params, user_matrix, mi) != 0) {
    free(mi);
    return -1;
  }
  cplx *U = (cplx *)malloc(sizeof(cplx) * dim * dim);
  for (int i = 0; i < dim * dim; i++) U[i] = mi[2 * i] + I * mi[2 * i + 1];
  free(mi);

  /* offset of matrix index r: sum_i r_i 2^targets[i] */
  uint64_t *off = (uint64_t *)malloc(sizeof(uint64_t) * dim);
  for (int r = 0; r < dim; r++) {
    uint64_t o = 0;
    for (int i = 0; i < t; i++)
      if (r & (1 << i)) o |= 1ull << targets[i];
    off[r] = o;
  }
  cplx *psi = (cplx *)psi_interleaved;
  int64_t size = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < size; b++) {
    if ((uint64_t)b & tmask) continue;               /* target bits 0 */
    if (((uint64_t)b & cmask) != cmask) continue;    /* control bits 1 */
    cplx v[1 << ORACLE_MAX_T];
    cplx w[1 << ORACLE_MAX_T];
    for (int r = 0; r < dim; r++) v[r] = psi[(uint64_t)b | off[r]];
    for (int r = 0; r < dim; r++) {
      cplx acc = 0;
      for (int k = 0; k < dim; k++) acc += U[r * dim + k] * v[k];
      w[r] = acc;
    }
    for (int r = 0; r < dim; r++) psi[(uint64_t)b | off[r]] = w[r];
  }
  free(off);
  free(U);
  return 0;
}

/* Gate record as marshalled by oracle/__init__.py (oracle's own layout). */
typedef struct {
  int32_t kind, t, nc, pad;
  int32_t targets[ORACLE_MAX_T];
  int32_t controls[ORACLE_MAX_T];
  double params[3];
  const double *matrix;
} oracle_gate;

/* Alg. 1: for gate in circuit: stateVec <- operate(gate, stateVec). */
int oracle_apply_circuit(double *psi, int n, const oracle_gate *gates,
                         int64_t n_gates) {
  for (int64_t g = 0; g < n_gates; g++) {
    const oracle_gate *q = &gates[g];
    int rc = oracle_apply_gate(psi, n, q->kind, q->t, q->targets, q->nc,
                               q->controls, q->params, q->matrix);
    if (rc != 0) return (int)(-1 - g);
  }
  return 0;
}

/* |x> : all zeros except psi[x] = 1. */
void oracle_basis_state(double *psi, int n, uint64_t x) {
  memset(psi, 0, sizeof(double) * 2 * ((size_t)1 << n));
  psi[2 * x] = 1.0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
