// gates.cpp -- product-side gate table and ingest/validation (step a1 of
// SURVEY 8(a)).  Written independently of oracle/oracle.c (no shared code).
//
// Matrices: DESIGN.md reading c3 (the paper names gates but never writes
// their matrices; SPEC.md L98 adopts OpenQASM 2.0 conventions).
// Diagonal gates are turned into phase polynomials: a diagonal over t
// targets with entry angles f(y), y in {0,1}^t, equals
// exp(2 pi i sum_S c_S prod_{i in S} y_i) with c = Moebius(f) computed exactly
// in Z/2^64 (angles in turns * 2^64), controls multiplied into every monomial.
// This is the B200 form of "thread_i ... complex multiplication between
// lambda_i and alpha_i": the kernel evaluates lambda_i
// from the index bits instead of reading a 2^N table.
#include <cmath>
#include <cstring>

#include "planner.hpp"

namespace qs {

static const long double kPiL = 3.141592653589793238462643383279502884L;

u64 turns_of(long double radians) {
  long double t = radians / (2.0L * kPiL);
  t -= floorl(t);                                    // [0, 1)
  long double v = roundl(t * 18446744073709551616.0L);  // * 2^64
  if (v >= 18446744073709551616.0L) return 0;           // rounded up to a full turn
  return (u64)v;                                        // exact: v < 2^64, integral
}

bool kind_is_diagonal(int kind) {
  switch (kind) {
    case QS_Z: case QS_S: case QS_SDG: case QS_T: case QS_TDG: case QS_RZ:
    case QS_U1: case QS_CZ: case QS_CP: case QS_RZZ: case QS_DIAGONAL:
      return true;
    default:
      return false;
  }
}

static int kind_arity(int kind) {
  switch (kind) {
    case QS_RZZ: case QS_SWAP: return 2;
    case QS_UNITARY: case QS_DIAGONAL: return -1;
    default: return (kind >= 0 && kind < QS_NUM_KINDS) ? 1 : 0;
  }
}

// Full matrix of a named (non-generic) kind.  Returns false for generic kinds.
bool gate_matrix(int kind, const double* p, std::vector<cd>& m, int* t_out) {
  const double h = 0.70710678118654752440;
  const cd i1(0, 1);
  const double th = p ? p[0] : 0.0;
  const double c = std::cos(0.5 * th), s = std::sin(0.5 * th);
  auto set2 = [&](cd a, cd b, cd cc, cd d) { m = {a, b, cc, d}; *t_out = 1; };
  switch (kind) {
    case QS_H: set2(h, h, h, -h); return true;
    case QS_X: case QS_CX: set2(0, 1, 1, 0); return true;
    case QS_Y: set2(0, -i1, i1, 0); return true;
    case QS_Z: case QS_CZ: set2(1, 0, 0, -1); return true;
    case QS_S: set2(1, 0, 0, i1); return true;
    case QS_SDG: set2(1, 0, 0, -i1); return true;
    case QS_T: set2(1, 0, 0, cd(h, h)); return true;
    case QS_TDG: set2(1, 0, 0, cd(h, -h)); return true;
    case QS_RX: set2(c, cd(0, -s), cd(0, -s), c); return true;
    case QS_RY: set2(c, -s, s, c); return true;
    case QS_RZ: set2(std::polar(1.0, -0.5 * th), 0, 0, std::polar(1.0, 0.5 * th)); return true;
    case QS_U1: case QS_CP: set2(1, 0, 0, std::polar(1.0, th)); return true;
    case QS_U2: {
      const double phi = p[0], lam = p[1];
      set2(h, -h * std::polar(1.0, lam), h * std::polar(1.0, phi),
           h * std::polar(1.0, phi + lam));
      return true;
    }
    case QS_U3: {
      const double phi = p[1], lam = p[2];
      set2(c, -s * std::polar(1.0, lam), s * std::polar(1.0, phi),
           c * std::polar(1.0, phi + lam));
      return true;
    }
    case QS_SX: {  // e^{i pi/4} RX(pi/2)
      const cd a(0.5, 0.5), b(0.5, -0.5);
      set2(a, b, b, a);
      return true;
    }
    case QS_SY: {  // e^{i pi/4} RY(pi/2)
      const cd a(0.5, 0.5);
      set2(a, -a, a, a);
      return true;
    }
    case QS_SW: {  // e^{i pi/4} exp(-i pi/4 W), W = (X+Y)/sqrt2
      const cd a(0.5, 0.5);
      set2(a, cd(0, -h), cd(h, 0), a);
      return true;
    }
    case QS_RZZ: {
      cd e0 = std::polar(1.0, -0.5 * th), e1 = std::polar(1.0, 0.5 * th);
      m.assign(16, 0);
      m[0] = e0; m[5] = e1; m[10] = e1; m[15] = e0;
      *t_out = 2;
      return true;
    }
    case QS_SWAP:
      m.assign(16, 0);
      m[0] = 1; m[6] = 1; m[9] = 1; m[15] = 1;
      *t_out = 2;
      return true;
    default:
      return false;
  }
}

// Angles (turns*2^64) of the diagonal entries of a named diagonal kind.
static void diag_turns(int kind, const double* p, std::vector<u64>& f) {
  const u64 half = 1ull << 63, quarter = 1ull << 62, eighth = 1ull << 61;
  const long double th = p ? (long double)p[0] : 0.0L;
  switch (kind) {
    case QS_Z: case QS_CZ: f = {0, half}; break;
    case QS_S: f = {0, quarter}; break;
    case QS_SDG: f = {0, (u64)0 - quarter}; break;
    case QS_T: f = {0, eighth}; break;
    case QS_TDG: f = {0, (u64)0 - eighth}; break;
    case QS_RZ: f = {turns_of(-th / 2), turns_of(th / 2)}; break;
    case QS_U1: case QS_CP: f = {0, turns_of(th)}; break;
    case QS_RZZ: {
      u64 a = turns_of(-th / 2), b = turns_of(th / 2);
      f = {a, b, b, a};
      break;
    }
    default: f.clear();
  }
}

// Moebius transform over subsets (exact in Z/2^64) -> monomials.
static void diag_to_mono(const std::vector<u64>& f, const std::vector<int>& targets,
                         u64 cmask, std::vector<Mono>& out) {
  const int t = (int)targets.size();
  std::vector<u64> c(f);
  for (int i = 0; i < t; i++)
    for (size_t S = 0; S < c.size(); S++)
      if (S >> i & 1) c[S] -= c[S ^ (1u << i)];
  for (size_t S = 0; S < c.size(); S++) {
    if (c[S] == 0) continue;
    u64 mask = cmask;
    for (int i = 0; i < t; i++)
      if (S >> i & 1) mask |= 1ull << targets[i];
    out.push_back({mask, c[S]});
  }
}

static bool is_unitary(const std::vector<cd>& m, int dim) {
  for (int r = 0; r < dim; r++)
    for (int q = 0; q < dim; q++) {
      cd acc = 0;
      for (int k = 0; k < dim; k++) acc += m[r * dim + k] * std::conj(m[q * dim + k]);
      if (std::abs(acc - (r == q ? 1.0 : 0.0)) >= 1e-10) return false;
    }
  return true;
}

int ingest(int n, const qs_gate_t* gates, size_t n_gates, std::vector<IrGate>& out,
           std::string& err) {
  out.clear();
  out.reserve(n_gates);
  char msg[256];
  for (size_t gi = 0; gi < n_gates; gi++) {
    const qs_gate_t& g = gates[gi];
    auto fail = [&](const char* why) {
      snprintf(msg, sizeof msg, "gate %zu (kind %d): %s", gi, g.kind, why);
      err = msg;
      return QS_EINVAL;
    };
    if (g.kind < 0 || g.kind >= QS_NUM_KINDS) return fail("unknown kind");
    const int t = g.n_targets, nc = g.n_controls;
    if (t < 1 || t > QS_MAX_TARGETS) return fail("n_targets out of range");
    if (nc < 0 || nc > QS_MAX_CONTROLS) return fail("n_controls out of range");
    int ar = kind_arity(g.kind);
    if (ar > 0 && ar != t) return fail("wrong number of targets for kind");
    if ((g.kind == QS_CX || g.kind == QS_CZ || g.kind == QS_CP) && nc < 1)
      return fail("controlled kind without control");
    u64 tm = 0, cm = 0;
    for (int i = 0; i < t; i++) {
      int q = g.targets[i];
      if (q < 0 || q >= n) return fail("target index out of range");
      if (tm >> q & 1) return fail("duplicate target");
      tm |= 1ull << q;
    }
    for (int i = 0; i < nc; i++) {
      int q = g.controls[i];
      if (q < 0 || q >= n) return fail("control index out of range");
      if ((tm | cm) >> q & 1) return fail("control overlaps a target or control");
      cm |= 1ull << q;
    }
    IrGate ir;
    ir.kind = g.kind;
    ir.support = tm | cm;
    std::vector<int> targets(g.targets, g.targets + t);
    std::vector<int> controls(g.controls, g.controls + nc);
    const int dim = 1 << t;

    if (g.kind == QS_DIAGONAL) {
      if (!g.matrix) return fail("DIAGONAL without entries");
      std::vector<u64> f(dim);
      for (int r = 0; r < dim; r++) {
        double re = g.matrix[2 * r], im = g.matrix[2 * r + 1];
        if (!std::isfinite(re) || !std::isfinite(im)) return fail("non-finite entry");
        if (std::fabs(std::hypot(re, im) - 1.0) >= 1e-10) return fail("|lambda| != 1");
        f[r] = turns_of(atan2l((long double)im, (long double)re));
      }
      ir.type = IrGate::DIAG;
      diag_to_mono(f, targets, cm, ir.mono);
    } else if (kind_is_diagonal(g.kind)) {
      std::vector<u64> f;
      diag_turns(g.kind, g.params, f);
      ir.type = IrGate::DIAG;
      diag_to_mono(f, targets, cm, ir.mono);
    } else if (g.kind == QS_SWAP && nc == 0) {
      ir.type = IrGate::RELABEL;  // Eq. 4: a pure qubit relabel
      ir.targets = targets;
    } else {
      ir.type = IrGate::DENSE;
      ir.targets = targets;
      ir.controls = controls;
      if (g.kind == QS_UNITARY) {
        if (!g.matrix) return fail("UNITARY without matrix");
        ir.mat.resize((size_t)dim * dim);
        for (int r = 0; r < dim * dim; r++) {
          double re = g.matrix[2 * r], im = g.matrix[2 * r + 1];
          if (!std::isfinite(re) || !std::isfinite(im)) return fail("non-finite entry");
          ir.mat[r] = cd(re, im);
        }
        if (!is_unitary(ir.mat, dim)) return fail("matrix is not unitary (1e-10)");
        // A generic unitary with exactly-zero off-diagonal entries is diagonal.
        bool diag = true;
        for (int r = 0; r < dim && diag; r++)
          for (int q = 0; q < dim; q++)
            if (r != q && ir.mat[r * dim + q] != cd(0, 0)) { diag = false; break; }
        if (diag) {
          std::vector<u64> f(dim);
          for (int r = 0; r < dim; r++)
            f[r] = turns_of(atan2l((long double)ir.mat[r * dim + r].imag(),
                                   (long double)ir.mat[r * dim + r].real()));
          ir.type = IrGate::DIAG;
          ir.mat.clear();
          ir.targets.clear();
          ir.controls.clear();
          diag_to_mono(f, targets, cm, ir.mono);
        }
      } else {
        int tt = 0;
        if (!gate_matrix(g.kind, g.params, ir.mat, &tt) || tt != t)
          return fail("no matrix for kind");
        ir.is_h = (g.kind == QS_H);
        ir.is_x = (g.kind == QS_X || g.kind == QS_CX);
      }
    }
    out.push_back(std::move(ir));
  }
  return QS_OK;
}

}  // namespace qs
