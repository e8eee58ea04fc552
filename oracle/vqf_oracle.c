/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Not part of the shipped
 * product; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it, and only as the checker.
 *
 * Plain-C restatement of the reference VQE Forge hot path
 * (/root/reference/proj/include/vqeforge/*.hpp), written from the
 * reference's behaviour, not copied.  Each function cites the reference
 * file:line it follows.  Complex arithmetic is spelled out as
 * (ac - bd, ad + bc) and the file is compiled with -ffp-contract=off so the
 * operation order matches the reference's std::complex<double> code built
 * without FMA (the reference CMake build sets no -march).
 *
 * Parity pin: tests/test_oracle.py checks this file against
 *   - the golden vectors in the reference tests (test_chem.cpp:223-239,
 *     :265; test_vqe.cpp:129, :178, :235; test_statevector.cpp:116-132;
 *     test_sweep.cpp:52-57) and
 *   - oracle/_ref/libvqf_ref.so (the unmodified reference headers compiled
 *     against oracle/eigen_shim) on seeded random inputs.
 *
 * Error convention (same as oracle/ref_capi.cpp): return 0 on success,
 * 1 invalid_argument, 2 runtime_error, 3 logic_error, 4 domain_error, with a
 * message written to err.
 */
#include "vqf_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846

typedef struct {
  double re, im;
} cplx;

static cplx c_mk(double re, double im) {
  cplx r = {re, im};
  return r;
}
static cplx c_add(cplx a, cplx b) { return c_mk(a.re + b.re, a.im + b.im); }
static cplx c_sub(cplx a, cplx b) { return c_mk(a.re - b.re, a.im - b.im); }
static cplx c_mul(cplx a, cplx b) { return c_mk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static cplx c_scale(double s, cplx a) { return c_mk(s * a.re, s * a.im); }
static cplx c_conj(cplx a) { return c_mk(a.re, -a.im); }
static double c_norm(cplx a) { return a.re * a.re + a.im * a.im; }
static double c_abs(cplx a) { return hypot(a.re, a.im); }

static int fail(char* err, size_t cap, int code, const char* msg) {
  if (err && cap) {
    strncpy(err, msg, cap - 1);
    err[cap - 1] = '\0';
  }
  return code;
}

/* ---------------------------------------------------------------- pauli */

/* pauli.hpp:225-227 qubit_bit: qubit 0 is the MOST significant index bit. */
static uint64_t qubit_bit(uint32_t n, uint32_t q) { return (uint64_t)1 << (n - 1 - q); }

/* pauli.hpp:229-238 term_masks */
static void term_masks(const orc_ham* h, uint32_t t, uint64_t* flip, uint64_t* yz, unsigned* n_y) {
  *flip = 0;
  *yz = 0;
  *n_y = 0;
  for (uint32_t k = h->offsets[t]; k < h->offsets[t + 1]; ++k) {
    const uint64_t bit = qubit_bit(h->n_qubits, h->qubits[k]);
    const uint8_t a = h->axes[k];
    if (a == 1 || a == 2) *flip |= bit;
    if (a == 2 || a == 3) *yz |= bit;
    if (a == 2) ++*n_y;
  }
}

/* pauli.hpp:242-249 y_phase_base = (-i)^{n_y} */
static cplx y_phase_base(unsigned n_y) {
  switch (n_y % 4) {
    case 0: return c_mk(1, 0);
    case 1: return c_mk(0, -1);
    case 2: return c_mk(-1, 0);
    default: return c_mk(0, 1);
  }
}

/* Sparse term used while building/canonicalizing (pauli.hpp:65-95). */
typedef struct {
  cplx coeff;
  uint32_t n;
  uint32_t q[ORC_MAX_AXES];
  uint8_t a[ORC_MAX_AXES];
} sterm;

/* pauli.hpp:99-106 axes_less: lexicographic on (index, axis) pairs. */
static int axes_less(const sterm* x, const sterm* y) {
  uint32_t i = 0;
  for (;; ++i) {
    if (i == y->n) return 0;
    if (i == x->n) return 1;
    if (x->q[i] != y->q[i]) return x->q[i] < y->q[i];
    if (x->a[i] != y->a[i]) return x->a[i] < y->a[i];
  }
}
static int axes_equal(const sterm* x, const sterm* y) {
  if (x->n != y->n) return 0;
  for (uint32_t i = 0; i < x->n; ++i)
    if (x->q[i] != y->q[i] || x->a[i] != y->a[i]) return 0;
  return 1;
}

/* pauli.hpp:180-201 canonicalize: merge like terms in order of first
 * appearance, drop |c| < 1e-12, stable-sort by axes_less.  Operates in
 * place on `ts`, returns the new count. */
static uint32_t canonicalize_terms(sterm* ts, uint32_t n) {
  uint32_t m = 0;
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t j = 0;
    for (; j < m; ++j)
      if (axes_equal(&ts[j], &ts[i])) break;
    if (j == m) {
      if (m != i) ts[m] = ts[i];
      ++m;
    } else {
      ts[j].coeff = c_add(ts[j].coeff, ts[i].coeff);
    }
  }
  uint32_t k = 0;
  for (uint32_t i = 0; i < m; ++i)
    if (c_abs(ts[i].coeff) >= 1e-12) {
      if (k != i) ts[k] = ts[i];
      ++k;
    }
  /* insertion sort: stable, and the reference's std::sort never sees equal
   * keys after merging, so any correct sort yields the same order. */
  for (uint32_t i = 1; i < k; ++i) {
    sterm key = ts[i];
    uint32_t j = i;
    while (j > 0 && axes_less(&key, &ts[j - 1])) {
      ts[j] = ts[j - 1];
      --j;
    }
    ts[j] = key;
  }
  return k;
}

static int sterm_from(const orc_ham* h, uint32_t t, sterm* out, char* err, size_t cap) {
  out->coeff = c_mk(h->coeffs[2 * t], h->coeffs[2 * t + 1]);
  out->n = h->offsets[t + 1] - h->offsets[t];
  if (out->n > ORC_MAX_AXES) return fail(err, cap, 1, "oracle: too many axes");
  for (uint32_t i = 0; i < out->n; ++i) {
    out->q[i] = h->qubits[h->offsets[t] + i];
    out->a[i] = h->axes[h->offsets[t] + i];
  }
  /* PauliTerm constructor (pauli.hpp:73-88): sort by index, reject I and
   * duplicate indices, reject non-finite coefficients. */
  for (uint32_t i = 1; i < out->n; ++i) {
    uint32_t qk = out->q[i];
    uint8_t ak = out->a[i];
    uint32_t j = i;
    while (j > 0 && out->q[j - 1] > qk) {
      out->q[j] = out->q[j - 1];
      out->a[j] = out->a[j - 1];
      --j;
    }
    out->q[j] = qk;
    out->a[j] = ak;
  }
  for (uint32_t i = 0; i < out->n; ++i) {
    if (out->a[i] == 0) return fail(err, cap, 1, "explicit identity entry in PauliTerm");
    if (i > 0 && out->q[i] == out->q[i - 1]) return fail(err, cap, 1, "duplicate qubit index in PauliTerm");
  }
  if (!isfinite(out->coeff.re) || !isfinite(out->coeff.im))
    return fail(err, cap, 1, "non-finite PauliTerm coefficient");
  return 0;
}

static int write_terms(const sterm* ts, uint32_t n, orc_ham_out* o, char* err, size_t cap) {
  if (n > o->cap_terms) return fail(err, cap, 2, "oracle: term capacity");
  uint32_t k = 0;
  o->offsets[0] = 0;
  for (uint32_t t = 0; t < n; ++t) {
    o->coeffs[2 * t] = ts[t].coeff.re;
    o->coeffs[2 * t + 1] = ts[t].coeff.im;
    for (uint32_t i = 0; i < ts[t].n; ++i) {
      if (k >= o->cap_axes) return fail(err, cap, 2, "oracle: axis capacity");
      o->qubits[k] = ts[t].q[i];
      o->axes[k] = ts[t].a[i];
      ++k;
    }
    o->offsets[t + 1] = k;
  }
  *o->n_terms = n;
  return 0;
}

int orc_canonicalize(const orc_ham* h, orc_ham_out* out, char* err, size_t cap) {
  sterm* ts = (sterm*)malloc(sizeof(sterm) * (h->n_terms ? h->n_terms : 1));
  int rc = 0;
  for (uint32_t t = 0; t < h->n_terms && rc == 0; ++t) rc = sterm_from(h, t, &ts[t], err, cap);
  if (rc == 0) {
    for (uint32_t t = 0; t < h->n_terms; ++t)
      if (ts[t].n && ts[t].q[ts[t].n - 1] >= h->n_qubits) {
        rc = fail(err, cap, 1, "PauliTerm index exceeds register size");
        break;
      }
  }
  if (rc == 0) rc = write_terms(ts, canonicalize_terms(ts, h->n_terms), out, err, cap);
  free(ts);
  return rc;
}

/* ---------------------------------------------------------- statevector */

/* statevector.hpp:61-74 basis_state */
int orc_basis_state(uint32_t n, const int* bits, uint32_t n_bits, double* amps, char* err, size_t cap) {
  if (n_bits != n) return fail(err, cap, 1, "basis_state: bit count != qubit count");
  const uint64_t dim = (uint64_t)1 << n;
  memset(amps, 0, sizeof(double) * 2 * dim);
  uint64_t index = 0;
  for (uint32_t q = 0; q < n; ++q)
    if (bits[q]) index |= qubit_bit(n, q);
  amps[2 * index] = 1.0;
  return 0;
}

/* statevector.hpp:105-120 check_wires */
static int check_wires(uint32_t n, const orc_gate* g, uint32_t expected, char* err, size_t cap) {
  if (g->n_wires != expected) return fail(err, cap, 1, "gate wire count mismatch");
  for (uint32_t i = 0; i < g->n_wires; ++i) {
    if (g->wires[i] >= n) return fail(err, cap, 1, "gate wire exceeds register size");
    for (uint32_t j = i + 1; j < g->n_wires; ++j)
      if (g->wires[i] == g->wires[j]) return fail(err, cap, 1, "duplicate gate wire");
  }
  return 0;
}

/* statevector.hpp:148-203 apply_gate. amps: interleaved (re, im), 2^n. */
int orc_apply_gate(uint32_t n, double* amps, const orc_gate* g, char* err, size_t cap) {
  cplx* a = (cplx*)amps;
  const uint64_t dim = (uint64_t)1 << n;
  int rc;
  switch (g->kind) {
    case ORC_X:
    case ORC_RY: {
      if ((rc = check_wires(n, g, 1, err, cap))) return rc;
      /* statevector.hpp:124-134 for_each_pair */
      const uint64_t bit = qubit_bit(n, g->wires[0]);
      const uint64_t low = bit - 1, high = ~low;
      const double c = cos(0.5 * g->angle), s = sin(0.5 * g->angle);
      for (uint64_t k = 0; k < dim / 2; ++k) {
        const uint64_t i0 = ((k & high) << 1) | (k & low);
        const cplx t0 = a[i0], t1 = a[i0 | bit];
        if (g->kind == ORC_X) {
          a[i0] = t1;
          a[i0 | bit] = t0;
        } else { /* :160-164 */
          a[i0] = c_sub(c_scale(c, t0), c_scale(s, t1));
          a[i0 | bit] = c_add(c_scale(s, t0), c_scale(c, t1));
        }
      }
      return 0;
    }
    case ORC_CNOT: { /* :167-178 */
      if ((rc = check_wires(n, g, 2, err, cap))) return rc;
      const uint64_t cm = qubit_bit(n, g->wires[0]), tm = qubit_bit(n, g->wires[1]);
      for (uint64_t i = 0; i < dim; ++i)
        if ((i & cm) && !(i & tm)) {
          const cplx t = a[i];
          a[i] = a[i | tm];
          a[i | tm] = t;
        }
      return 0;
    }
    case ORC_DE: { /* :179-200 */
      if ((rc = check_wires(n, g, 4, err, cap))) return rc;
      const uint64_t m0 = qubit_bit(n, g->wires[0]), m1 = qubit_bit(n, g->wires[1]);
      const uint64_t m2 = qubit_bit(n, g->wires[2]), m3 = qubit_bit(n, g->wires[3]);
      const uint64_t sel = m0 | m1 | m2 | m3, occ = m0 | m1;
      const double c = cos(0.5 * g->angle), s = sin(0.5 * g->angle);
      for (uint64_t i = 0; i < dim; ++i)
        if ((i & sel) == occ) {
          const uint64_t j = i ^ sel;
          const cplx x = a[i], y = a[j];
          a[i] = c_sub(c_scale(c, x), c_scale(s, y));
          a[j] = c_add(c_scale(s, x), c_scale(c, y));
        }
      return 0;
    }
    case ORC_SE: { /* DE's loop (:179-200) on two wires: occupied = w0 */
      if ((rc = check_wires(n, g, 2, err, cap))) return rc;
      const uint64_t m0 = qubit_bit(n, g->wires[0]), m1 = qubit_bit(n, g->wires[1]);
      const uint64_t sel = m0 | m1;
      const double c = cos(0.5 * g->angle), s = sin(0.5 * g->angle);
      for (uint64_t i = 0; i < dim; ++i)
        if ((i & sel) == m0) {
          const uint64_t j = i ^ sel;
          const cplx x = a[i], y = a[j];
          a[i] = c_sub(c_scale(c, x), c_scale(s, y));
          a[j] = c_add(c_scale(s, x), c_scale(c, y));
        }
      return 0;
    }
  }
  return fail(err, cap, 3, "unknown gate kind");
}

/* statevector.hpp:217-249 expectation */
int orc_expectation(uint32_t n, const double* amps, const orc_ham* h, double* out, char* err, size_t cap) {
  if (h->n_qubits != n) return fail(err, cap, 1, "expectation: qubit count mismatch");
  const cplx* a = (const cplx*)amps;
  const uint64_t dim = (uint64_t)1 << n;
  cplx total = c_mk(0, 0);
  for (uint32_t t = 0; t < h->n_terms; ++t) {
    uint64_t flip, yz;
    unsigned n_y;
    term_masks(h, t, &flip, &yz, &n_y);
    const cplx base = y_phase_base(n_y);
    cplx acc = c_mk(0, 0);
    if (flip == 0) {
      double diag = 0.0;
      for (uint64_t i = 0; i < dim; ++i) {
        const double p = c_norm(a[i]);
        diag += (__builtin_popcountll(i & yz) & 1U) ? -p : p;
      }
      acc = c_mk(diag, 0.0);
    } else {
      for (uint64_t i = 0; i < dim; ++i) {
        const cplx v = c_mul(c_conj(a[i]), a[i ^ flip]);
        acc = (__builtin_popcountll(i & yz) & 1U) ? c_sub(acc, v) : c_add(acc, v);
      }
    }
    const cplx coeff = c_mk(h->coeffs[2 * t], h->coeffs[2 * t + 1]);
    total = c_add(total, c_mul(c_mul(coeff, base), acc));
  }
  if (fabs(total.im) >= 1e-10) {
    char msg[128];
    snprintf(msg, sizeof msg, "expectation has imaginary residue %f", total.im);
    return fail(err, cap, 2, msg);
  }
  *out = total.re;
  return 0;
}

/* ------------------------------------------------------------------ vqe */

/* vqe.hpp:54-62 n_parameters */
uint32_t orc_n_parameters(int kind, uint32_t layers, uint32_t n) { return kind == 0 ? 1u : layers * n; }

/* vqe.hpp:65-96 prepare_ansatz */
int orc_prepare_ansatz(int kind, uint32_t layers, const double* theta, uint32_t n_theta, uint32_t n,
                       double* amps, char* err, size_t cap) {
  if (n_theta != orc_n_parameters(kind, layers, n)) return fail(err, cap, 1, "parameter count mismatch for ansatz");
  if (kind == 0) {
    if (n != 4) return fail(err, cap, 1, "H2 double-excitation ansatz requires 4 qubits");
    const int bits[4] = {1, 1, 0, 0};
    orc_basis_state(4, bits, 4, amps, err, cap);
    orc_gate g = {ORC_DE, theta[0], 4, {0, 1, 2, 3}};
    return orc_apply_gate(4, amps, &g, err, cap);
  }
  const uint64_t dim = (uint64_t)1 << n;
  memset(amps, 0, sizeof(double) * 2 * dim);
  amps[0] = 1.0;
  uint32_t k = 0;
  for (uint32_t layer = 0; layer < layers; ++layer) {
    for (uint32_t q = 0; q < n; ++q) {
      orc_gate g = {ORC_RY, theta[k++], 1, {q, 0, 0, 0}};
      orc_apply_gate(n, amps, &g, err, cap);
    }
    for (uint32_t q = 0; q + 1 < n; ++q) {
      orc_gate g = {ORC_CNOT, 0.0, 2, {q, q + 1, 0, 0}};
      orc_apply_gate(n, amps, &g, err, cap);
    }
  }
  return 0;
}

/* vqe.hpp:99-104 energy */
int orc_energy(int kind, uint32_t layers, const double* theta, uint32_t n_theta, const orc_ham* h, double* out,
               char* err, size_t cap) {
  const uint32_t n = h->n_qubits;
  double* amps = (double*)malloc(sizeof(double) * 2 * ((size_t)1 << n));
  int rc = orc_prepare_ansatz(kind, layers, theta, n_theta, n, amps, err, cap);
  if (rc == 0) rc = orc_expectation(n, amps, h, out, err, cap);
  free(amps);
  return rc;
}

/* vqe.hpp:112-127 gradient (two-term parameter shift, shift pi/2) */
int orc_gradient(int kind, uint32_t layers, const double* theta, uint32_t n_theta, const orc_ham* h, double* grad,
                 char* err, size_t cap) {
  const double shift = ORC_PI / 2.0;
  double* shifted = (double*)malloc(sizeof(double) * (n_theta ? n_theta : 1));
  memcpy(shifted, theta, sizeof(double) * n_theta);
  int rc = 0;
  for (uint32_t k = 0; k < n_theta && rc == 0; ++k) {
    double plus, minus;
    shifted[k] = theta[k] + shift;
    rc = orc_energy(kind, layers, shifted, n_theta, h, &plus, err, cap);
    if (rc) break;
    shifted[k] = theta[k] - shift;
    rc = orc_energy(kind, layers, shifted, n_theta, h, &minus, err, cap);
    shifted[k] = theta[k];
    grad[k] = 0.5 * (plus - minus);
  }
  free(shifted);
  return rc;
}

/* vqe.hpp:152-174 adam_step (pure; step counts from 1) */
void orc_adam_step(const double* m, const double* v, int64_t step, const double* grad, const double* theta,
                   uint32_t n, const orc_adam* cfg, double* theta_out, double* m_out, double* v_out,
                   int64_t* step_out) {
  const int64_t t = step + 1;
  const double bc1 = 1.0 - pow(cfg->beta1, (double)t);
  const double bc2 = 1.0 - pow(cfg->beta2, (double)t);
  for (uint32_t k = 0; k < n; ++k) {
    m_out[k] = cfg->beta1 * m[k] + (1.0 - cfg->beta1) * grad[k];
    v_out[k] = cfg->beta2 * v[k] + (1.0 - cfg->beta2) * grad[k] * grad[k];
    const double m_hat = m_out[k] / bc1;
    const double v_hat = v_out[k] / bc2;
    theta_out[k] = theta[k] - cfg->learning_rate * m_hat / (sqrt(v_hat) + cfg->epsilon);
  }
  *step_out = t;
}

static int nonfinite_msg(int iter, const double* theta, uint32_t n, char* err, size_t cap) {
  /* vqe.hpp:216-221: "non-finite energy at iteration I; theta = x y ..."
   * with std::to_string (%f) formatting. */
  char msg[1024];
  int off = snprintf(msg, sizeof msg, "non-finite energy at iteration %d; theta =", iter);
  for (uint32_t k = 0; k < n && off < (int)sizeof msg - 32; ++k) off += snprintf(msg + off, sizeof msg - off, " %f", theta[k]);
  return fail(err, cap, 2, msg);
}

/* vqe.hpp:194-254 run_vqe.  traj must hold max_iterations + 1 doubles. */
int orc_run_vqe(const orc_ham* h, int kind, uint32_t layers, const orc_adam* cfg, const double* init, uint32_t n_init,
                orc_vqe_result* r, char* err, size_t cap) {
  const uint32_t P = orc_n_parameters(kind, layers, h->n_qubits);
  if (n_init != 0 && n_init != P) return fail(err, cap, 1, "initial parameter count mismatch");
  double* theta = (double*)calloc(P, sizeof(double));
  double* grad = (double*)calloc(P, sizeof(double));
  double* m = (double*)calloc(P, sizeof(double));
  double* v = (double*)calloc(P, sizeof(double));
  double* tn = (double*)calloc(P, sizeof(double));
  double* mn = (double*)calloc(P, sizeof(double));
  double* vn = (double*)calloc(P, sizeof(double));
  if (n_init) memcpy(theta, init, sizeof(double) * P);
  int64_t step = 0;
  int rc = 0, converged = 0;
  r->traj_len = 0;
  r->iterations_run = 0;
  r->circuit_evaluations = 0;
  for (int iter = 0; iter < cfg->max_iterations; ++iter) {
    double e;
    rc = orc_energy(kind, layers, theta, P, h, &e, err, cap);
    if (rc) goto done;
    ++r->circuit_evaluations;
    if (!isfinite(e)) {
      rc = nonfinite_msg(iter, theta, P, err, cap);
      goto done;
    }
    r->trajectory[r->traj_len++] = e;
    rc = orc_gradient(kind, layers, theta, P, h, grad, err, cap);
    if (rc) goto done;
    r->circuit_evaluations += 2 * (uint64_t)P;
    if (cfg->has_tolerance) {
      double g_inf = 0.0;
      for (uint32_t k = 0; k < P; ++k) g_inf = fmax(g_inf, fabs(grad[k]));
      if (g_inf < cfg->gradient_tolerance) {
        converged = 1;
        break;
      }
    }
    orc_adam_step(m, v, step, grad, theta, P, cfg, tn, mn, vn, &step);
    memcpy(theta, tn, sizeof(double) * P);
    memcpy(m, mn, sizeof(double) * P);
    memcpy(v, vn, sizeof(double) * P);
    r->iterations_run = iter + 1;
  }
  if (!converged) {
    double e;
    rc = orc_energy(kind, layers, theta, P, h, &e, err, cap);
    if (rc) goto done;
    ++r->circuit_evaluations;
    if (!isfinite(e)) {
      rc = nonfinite_msg(cfg->max_iterations, theta, P, err, cap);
      goto done;
    }
    r->trajectory[r->traj_len++] = e;
  }
  r->energy = r->trajectory[r->traj_len - 1];
  memcpy(r->theta, theta, sizeof(double) * P);
done:
  free(theta);
  free(grad);
  free(m);
  free(v);
  free(tn);
  free(mn);
  free(vn);
  return rc;
}

/* ---------------------------------------------------------------- sweep */

/* sweep.hpp:68-85 bond_grid */
int orc_bond_grid(double d_min, double d_max, int n_points, double* out, char* err, size_t cap) {
  if (n_points < 1) return fail(err, cap, 1, "grid needs >= 1 point");
  if (d_max < d_min) return fail(err, cap, 1, "d_max < d_min");
  if (n_points == 1) {
    out[0] = d_min;
    return 0;
  }
  const double span = d_max - d_min;
  for (int i = 0; i < n_points - 1; ++i) out[i] = d_min + span * (double)i / (double)(n_points - 1);
  out[n_points - 1] = d_max;
  return 0;
}

/* sweep.hpp:93-107 split_chunks: begin_end[2c], begin_end[2c+1] */
int orc_split_chunks(uint64_t n_items, uint64_t n_chunks, uint64_t* begin_end, char* err, size_t cap) {
  if (n_chunks == 0) return fail(err, cap, 1, "need >= 1 chunk");
  const uint64_t base = n_items / n_chunks, extra = n_items % n_chunks;
  uint64_t begin = 0;
  for (uint64_t c = 0; c < n_chunks; ++c) {
    const uint64_t len = base + (c < extra ? 1 : 0);
    begin_end[2 * c] = begin;
    begin_end[2 * c + 1] = begin + len;
    begin += len;
  }
  return 0;
}

/* sweep.hpp:209-223 build_tfim and :227-235 build_z_sum */
int orc_build_tfim(uint32_t n, double coupling, double field, orc_ham_out* out, char* err, size_t cap) {
  const uint32_t nt = 2 * n;
  sterm* ts = (sterm*)calloc(nt, sizeof(sterm));
  uint32_t k = 0;
  for (uint32_t q = 0; q + 1 < n; ++q) {
    ts[k].coeff = c_mk(-coupling, 0.0);
    ts[k].n = 2;
    ts[k].q[0] = q;
    ts[k].a[0] = 3;
    ts[k].q[1] = q + 1;
    ts[k].a[1] = 3;
    ++k;
  }
  for (uint32_t q = 0; q < n; ++q) {
    ts[k].coeff = c_mk(-field, 0.0);
    ts[k].n = 1;
    ts[k].q[0] = q;
    ts[k].a[0] = 1;
    ++k;
  }
  int rc = write_terms(ts, canonicalize_terms(ts, k), out, err, cap);
  free(ts);
  return rc;
}

int orc_build_z_sum(uint32_t n, orc_ham_out* out, char* err, size_t cap) {
  sterm* ts = (sterm*)calloc(n ? n : 1, sizeof(sterm));
  for (uint32_t q = 0; q < n; ++q) {
    ts[q].coeff = c_mk(1.0, 0.0);
    ts[q].n = 1;
    ts[q].q[0] = q;
    ts[q].a[0] = 3;
  }
  int rc = write_terms(ts, canonicalize_terms(ts, n), out, err, cap);
  free(ts);
  return rc;
}

/* ----------------------------------------------------------------- chem */
/* chem.hpp:32-36 constants */
#define K_ANG_TO_BOHR 1.8897259886
#define K_MIN_BOND 0.05
#define K_MAX_BOND 10.0
#define K_SCF_MAX 100
#define K_SCF_TOL 1e-10

typedef struct {
  double e[3], c[3], z; /* exponents, coefficients, center z (x = y = 0) */
} cgauss;

/* chem.hpp:66-89 sto3g_hydrogen */
static cgauss sto3g(double z) {
  static const double alpha[3] = {3.42525091, 0.62391373, 0.16885540};
  static const double contr[3] = {0.15432897, 0.53532814, 0.44463454};
  cgauss g;
  g.z = z;
  for (int i = 0; i < 3; ++i) {
    g.e[i] = alpha[i];
    g.c[i] = contr[i] * pow(2.0 * alpha[i] / ORC_PI, 0.75);
  }
  double self = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double p = alpha[i] + alpha[j];
      self += g.c[i] * g.c[j] * pow(ORC_PI / p, 1.5);
    }
  const double scale = 1.0 / sqrt(self);
  for (int i = 0; i < 3; ++i) g.c[i] *= scale;
  return g;
}

/* chem.hpp:93-99 boys_f0 */
static double boys_f0(double t) {
  if (t < 1e-12) return 1.0 - t / 3.0 + t * t / 10.0 - t * t * t / 42.0;
  const double sq = sqrt(t);
  return 0.5 * sqrt(ORC_PI / t) * erf(sq);
}

/* All centres lie on the z axis: dist2 reduces to dz^2 but is spelled out as
 * the reference's dx*dx + dy*dy + dz*dz (chem.hpp:103-107) with dx = dy = 0. */
static double dist2z(double a, double b) {
  const double dz = a - b;
  return 0.0 * 0.0 + 0.0 * 0.0 + dz * dz;
}
static double center_z(double a, double A, double b, double B) { return (a * A + b * B) / (a + b); }

/* chem.hpp:142-182 primitive integrals */
static double overlap_prim(double a, double A, double b, double B) {
  const double p = a + b, mu = a * b / p;
  return pow(ORC_PI / p, 1.5) * exp(-mu * dist2z(A, B));
}
static double kinetic_prim(double a, double A, double b, double B) {
  const double p = a + b, mu = a * b / p, r2 = dist2z(A, B);
  return mu * (3.0 - 2.0 * mu * r2) * pow(ORC_PI / p, 1.5) * exp(-mu * r2);
}
static double nuclear_prim(double a, double A, double b, double B, double C) {
  const double p = a + b, mu = a * b / p;
  const double P = center_z(a, A, b, B);
  return -2.0 * ORC_PI / p * exp(-mu * dist2z(A, B)) * boys_f0(p * dist2z(P, C));
}
static double eri_prim(double a, double A, double b, double B, double c, double C, double d, double D) {
  const double p = a + b, q = c + d;
  const double P = center_z(a, A, b, B), Q = center_z(c, C, d, D);
  const double pref = 2.0 * pow(ORC_PI, 2.5) / (p * q * sqrt(p + q));
  return pref * exp(-(a * b / p) * dist2z(A, B)) * exp(-(c * d / q) * dist2z(C, D)) *
         boys_f0(p * q / (p + q) * dist2z(P, Q));
}

typedef struct {
  double S[2][2], T[2][2], V[2][2], eri[16]; /* eri[((i*2+j)*2+k)*2+l] chemist */
} ao_ints;

/* chem.hpp:218-249 ao_integrals */
static void ao_integrals(double bond_bohr, ao_ints* out) {
  const cgauss bs[2] = {sto3g(0.0), sto3g(bond_bohr)};
  const double nuc[2] = {0.0, bond_bohr};
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      double s = 0, t = 0;
      for (int x = 0; x < 3; ++x)
        for (int y = 0; y < 3; ++y) {
          s += bs[i].c[x] * bs[j].c[y] * overlap_prim(bs[i].e[x], bs[i].z, bs[j].e[y], bs[j].z);
        }
      for (int x = 0; x < 3; ++x)
        for (int y = 0; y < 3; ++y) {
          t += bs[i].c[x] * bs[j].c[y] * kinetic_prim(bs[i].e[x], bs[i].z, bs[j].e[y], bs[j].z);
        }
      double v = 0.0;
      for (int n = 0; n < 2; ++n) {
        double vn = 0.0;
        for (int x = 0; x < 3; ++x)
          for (int y = 0; y < 3; ++y)
            vn += bs[i].c[x] * bs[j].c[y] * nuclear_prim(bs[i].e[x], bs[i].z, bs[j].e[y], bs[j].z, nuc[n]);
        v += vn;
      }
      out->S[i][j] = s;
      out->T[i][j] = t;
      out->V[i][j] = v;
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l) {
          double sum = 0.0;
          for (int x = 0; x < 3; ++x)
            for (int y = 0; y < 3; ++y)
              for (int z = 0; z < 3; ++z)
                for (int w = 0; w < 3; ++w)
                  sum += bs[i].c[x] * bs[j].c[y] * bs[k].c[z] * bs[l].c[w] *
                         eri_prim(bs[i].e[x], bs[i].z, bs[j].e[y], bs[j].z, bs[k].e[z], bs[k].z, bs[l].e[w],
                                  bs[l].z);
          out->eri[((i * 2 + j) * 2 + k) * 2 + l] = sum;
        }
    }
}

/* Symmetric 2x2 eigen-decomposition, ascending eigenvalues, unit columns. */
static void sym2(const double A[2][2], double ev[2], double V[2][2]) {
  const double p = A[0][0], q = A[1][1], r = 0.5 * (A[0][1] + A[1][0]);
  const double mean = 0.5 * (p + q), rad = hypot(0.5 * (p - q), r);
  ev[0] = mean - rad;
  ev[1] = mean + rad;
  if (rad == 0.0) {
    V[0][0] = 1;
    V[0][1] = 0;
    V[1][0] = 0;
    V[1][1] = 1;
    return;
  }
  double ux = r, uy = ev[0] - p;
  const double vx = ev[0] - q, vy = r;
  if (hypot(vx, vy) > hypot(ux, uy)) {
    ux = vx;
    uy = vy;
  }
  const double nrm = hypot(ux, uy);
  ux /= nrm;
  uy /= nrm;
  V[0][0] = ux;
  V[1][0] = uy;
  V[0][1] = -uy;
  V[1][1] = ux;
}

static void mm2(const double A[2][2], const double B[2][2], double C[2][2]) {
  double R[2][2];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) R[i][j] = A[i][0] * B[0][j] + A[i][1] * B[1][j];
  memcpy(C, R, sizeof R);
}
static void tr2(const double A[2][2], double B[2][2]) {
  double R[2][2] = {{A[0][0], A[1][0]}, {A[0][1], A[1][1]}};
  memcpy(B, R, sizeof R);
}

/* chem.hpp:280-372 run_hartree_fock.  Outputs core_h_mo, physicist eri_mo
 * and energies. */
static int hartree_fock(double bond_angstrom, double hmo[2][2], double eri_mo[16], double* e_nuc, double* hf_energy,
                        int* scf_iters, char* err, size_t cap) {
  if (!(bond_angstrom >= K_MIN_BOND && bond_angstrom <= K_MAX_BOND)) {
    char msg[160];
    snprintf(msg, sizeof msg, "bond length %f angstrom outside [%f, %f]", bond_angstrom, K_MIN_BOND, K_MAX_BOND);
    return fail(err, cap, 4, msg);
  }
  const double d = bond_angstrom * K_ANG_TO_BOHR;
  ao_ints I;
  ao_integrals(d, &I);
  double H[2][2];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) H[i][j] = I.T[i][j] + I.V[i][j];
  double sev[2], SV[2][2], X[2][2], D12[2][2], SVt[2][2];
  sym2(I.S, sev, SV);
  D12[0][0] = 1.0 / sqrt(sev[0]);
  D12[1][1] = 1.0 / sqrt(sev[1]);
  D12[0][1] = D12[1][0] = 0.0;
  /* X = V diag(1/sqrt(s)) V^T */
  double VD[2][2];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) VD[i][j] = SV[i][j] * D12[j][j];
  tr2(SV, SVt);
  mm2(VD, SVt, X);
#define ERI(a, b, c, e) I.eri[(((a)*2 + (b)) * 2 + (c)) * 2 + (e)]
  double P[2][2] = {{0, 0}, {0, 0}}, C[2][2] = {{0, 0}, {0, 0}}, F[2][2], G[2][2];
  double e_elec = 0.0;
  int converged = 0, iterations = 0;
  for (int iter = 1; iter <= K_SCF_MAX; ++iter) {
    for (int mu = 0; mu < 2; ++mu)
      for (int nu = 0; nu < 2; ++nu) {
        double g = 0.0;
        for (int lam = 0; lam < 2; ++lam)
          for (int sig = 0; sig < 2; ++sig) g += P[lam][sig] * (ERI(mu, nu, sig, lam) - 0.5 * ERI(mu, lam, sig, nu));
        G[mu][nu] = g;
      }
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) F[i][j] = H[i][j] + G[i][j];
    double Xt[2][2], T1[2][2], Fp[2][2], fev[2], FV[2][2];
    tr2(X, Xt);
    mm2(Xt, F, T1);
    mm2(T1, X, Fp);
    sym2(Fp, fev, FV);
    mm2(X, FV, C);
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) P[i][j] = (2.0 * C[i][0]) * C[j][0];
    double s = 0.0;
    for (int j = 0; j < 2; ++j)
      for (int i = 0; i < 2; ++i) s += P[i][j] * (H[i][j] + F[i][j]);
    const double e_new = 0.5 * s;
    iterations = iter;
    if (iter > 1 && fabs(e_new - e_elec) < K_SCF_TOL) {
      e_elec = e_new;
      converged = 1;
      break;
    }
    e_elec = e_new;
  }
  if (!converged) {
    char msg[160];
    snprintf(msg, sizeof msg, "SCF failed to converge within %d iterations at bond length %f angstrom", K_SCF_MAX,
             bond_angstrom);
    return fail(err, cap, 2, msg);
  }
  for (int mu = 0; mu < 2; ++mu)
    for (int nu = 0; nu < 2; ++nu) {
      double g = 0.0;
      for (int lam = 0; lam < 2; ++lam)
        for (int sig = 0; sig < 2; ++sig) g += P[lam][sig] * (ERI(mu, nu, sig, lam) - 0.5 * ERI(mu, lam, sig, nu));
      F[mu][nu] = H[mu][nu] + g;
    }
  double s = 0.0;
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i) s += P[i][j] * (H[i][j] + F[i][j]);
  e_elec = 0.5 * s;
  *e_nuc = 1.0 / d;
  *hf_energy = e_elec + *e_nuc;
  *scf_iters = iterations;
  double Ct[2][2], T2[2][2];
  tr2(C, Ct);
  mm2(Ct, H, T2);
  mm2(T2, C, hmo);
  double mo_chem[16];
  for (int p = 0; p < 2; ++p)
    for (int q = 0; q < 2; ++q)
      for (int r = 0; r < 2; ++r)
        for (int t = 0; t < 2; ++t) {
          double val = 0.0;
          for (int mu = 0; mu < 2; ++mu)
            for (int nu = 0; nu < 2; ++nu)
              for (int lam = 0; lam < 2; ++lam)
                for (int sig = 0; sig < 2; ++sig)
                  val += C[mu][p] * C[nu][q] * C[lam][r] * C[sig][t] * ERI(mu, nu, lam, sig);
          mo_chem[((p * 2 + q) * 2 + r) * 2 + t] = val;
        }
  /* chemist -> physicist: <ij|kl> = (ik|jl) (chem.hpp:366-370) */
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l) eri_mo[((i * 2 + j) * 2 + k) * 2 + l] = mo_chem[((i * 2 + k) * 2 + j) * 2 + l];
#undef ERI
  return 0;
}

int orc_hartree_fock(double bond_angstrom, double* out4, char* err, size_t cap) {
  double hmo[2][2], eri[16], en, hf;
  int it;
  int rc = hartree_fock(bond_angstrom, hmo, eri, &en, &hf, &it, err, cap);
  if (rc) return rc;
  out4[0] = hf;
  out4[1] = hf - en;
  out4[2] = en;
  out4[3] = it;
  return 0;
}

/* pauli.hpp:142-150 axis_product: a*b = phase * axis. */
static void axis_product(uint8_t a, uint8_t b, cplx* phase, uint8_t* axis) {
  if (a == 0) {
    *phase = c_mk(1, 0);
    *axis = b;
    return;
  }
  if (b == 0 || a == b) {
    *phase = c_mk(1, 0);
    *axis = (b == 0) ? a : 0;
    return;
  }
  const int ic = 6 - a - b;
  const int cyclic = ((b - a + 3) % 3) == 1;
  *phase = cyclic ? c_mk(0, 1) : c_mk(0, -1);
  *axis = (uint8_t)ic;
}

/* pauli.hpp:152-174 multiply_terms */
static sterm multiply_terms(const sterm* a, const sterm* b) {
  sterm out;
  out.coeff = c_mul(a->coeff, b->coeff);
  out.n = 0;
  uint32_t i = 0, j = 0;
  while (i < a->n || j < b->n) {
    if (j == b->n || (i < a->n && a->q[i] < b->q[j])) {
      out.q[out.n] = a->q[i];
      out.a[out.n++] = a->a[i++];
    } else if (i == a->n || b->q[j] < a->q[i]) {
      out.q[out.n] = b->q[j];
      out.a[out.n++] = b->a[j++];
    } else {
      cplx ph;
      uint8_t ax;
      axis_product(a->a[i], b->a[j], &ph, &ax);
      out.coeff = c_mul(out.coeff, ph);
      if (ax != 0) {
        out.q[out.n] = a->q[i];
        out.a[out.n++] = ax;
      }
      ++i;
      ++j;
    }
  }
  return out;
}

/* chem.hpp:380-393 jordan_wigner_ladder */
static void jw_ladder(uint32_t p, int dagger, sterm out[2]) {
  for (int k = 0; k < 2; ++k) {
    out[k].n = 0;
    for (uint32_t q = 0; q < p; ++q) {
      out[k].q[out[k].n] = q;
      out[k].a[out[k].n++] = 3;
    }
    out[k].q[out[k].n] = p;
    out[k].a[out[k].n++] = (k == 0) ? 1 : 2;
  }
  out[0].coeff = c_mk(0.5, 0.0);
  out[1].coeff = dagger ? c_mk(-0.0, -0.5) : c_mk(0.0, 0.5);
}

/* chem.hpp:397-410 accumulate_product */
static void accumulate(sterm* out, uint32_t* n_out, cplx weight, const sterm* const* factors, int n_factors) {
  sterm acc[16], next[16];
  uint32_t n_acc = 1;
  acc[0].coeff = weight;
  acc[0].n = 0;
  for (int f = 0; f < n_factors; ++f) {
    uint32_t nn = 0;
    for (uint32_t x = 0; x < n_acc; ++x)
      for (int y = 0; y < 2; ++y) next[nn++] = multiply_terms(&acc[x], &factors[f][y]);
    memcpy(acc, next, sizeof(sterm) * nn);
    n_acc = nn;
  }
  memcpy(out + *n_out, acc, sizeof(sterm) * n_acc);
  *n_out += n_acc;
}

/* chem.hpp:422-467 jordan_wigner + :473 build_h2_hamiltonian (no memo). */
int orc_build_h2_hamiltonian(double bond_angstrom, orc_ham_out* o, char* err, size_t cap) {
  double hmo[2][2], eri[16], en, hf;
  int it;
  int rc = hartree_fock(bond_angstrom, hmo, eri, &en, &hf, &it, err, cap);
  if (rc) return rc;
  sterm create[4][2], annih[4][2];
  for (uint32_t p = 0; p < 4; ++p) {
    jw_ladder(p, 1, create[p]);
    jw_ladder(p, 0, annih[p]);
  }
  const uint32_t max_terms = 1 + 16 * 4 + 256 * 16;
  sterm* ts = (sterm*)malloc(sizeof(sterm) * max_terms);
  uint32_t n = 0;
  ts[0].coeff = c_mk(en, 0.0);
  ts[0].n = 0;
  n = 1;
  for (uint32_t p = 0; p < 4; ++p)
    for (uint32_t q = 0; q < 4; ++q) {
      if (p % 2 != q % 2) continue;
      const double h = hmo[p / 2][q / 2];
      if (h == 0.0) continue;
      const sterm* f[2] = {create[p], annih[q]};
      accumulate(ts, &n, c_mk(h, 0.0), f, 2);
    }
  for (uint32_t p = 0; p < 4; ++p)
    for (uint32_t q = 0; q < 4; ++q)
      for (uint32_t r = 0; r < 4; ++r)
        for (uint32_t s = 0; s < 4; ++s) {
          if (p % 2 != r % 2 || q % 2 != s % 2) continue;
          const double g = eri[(((p / 2) * 2 + q / 2) * 2 + r / 2) * 2 + s / 2];
          if (g == 0.0) continue;
          const sterm* f[4] = {create[p], create[q], annih[s], annih[r]};
          accumulate(ts, &n, c_mk(0.5 * g, 0.0), f, 4);
        }
  n = canonicalize_terms(ts, n);
  /* pauli.hpp:205-214 check_hermitian_coefficients, then drop imag parts */
  for (uint32_t t = 0; t < n; ++t) {
    if (fabs(ts[t].coeff.im) >= 1e-10) {
      char msg[128];
      snprintf(msg, sizeof msg, "non-Hermitian Pauli coefficient: imag = %f", ts[t].coeff.im);
      free(ts);
      return fail(err, cap, 2, msg);
    }
    ts[t].coeff.im = 0.0;
  }
  rc = write_terms(ts, n, o, err, cap);
  free(ts);
  return rc;
}

/* sweep.hpp:128-178 run_sweep, serial (the oracle is the checker, not a
 * parallel baseline; chunking does not change per-point results). */
int orc_run_sweep(double d_min, double d_max, int n_points, const orc_adam* cfg, double* bond, double* energy,
                  double* theta_star, int* iterations, int* ok, char* errors, size_t err_stride, char* err,
                  size_t cap) {
  int rc = orc_bond_grid(d_min, d_max, n_points, bond, err, cap);
  if (rc) return rc;
  double coeffs[2 * 64];
  uint32_t offs[65], qb[256], nt;
  uint8_t ax[256];
  orc_ham_out ho = {&nt, coeffs, offs, qb, ax, 64, 256};
  double* traj = (double*)malloc(sizeof(double) * ((size_t)cfg->max_iterations + 1));
  for (int i = 0; i < n_points; ++i) {
    char perr[512] = {0};
    energy[i] = NAN;
    theta_star[i] = 0.0;
    iterations[i] = 0;
    ok[i] = 0;
    int prc = orc_build_h2_hamiltonian(bond[i], &ho, perr, sizeof perr);
    if (prc == 0) {
      orc_ham h = {4, nt, coeffs, offs, qb, ax};
      double th;
      orc_vqe_result r = {0};
      r.trajectory = traj;
      r.theta = &th;
      prc = orc_run_vqe(&h, 0, 0, cfg, NULL, 0, &r, perr, sizeof perr);
      if (prc == 0) {
        energy[i] = r.energy;
        theta_star[i] = th;
        iterations[i] = r.iterations_run;
        ok[i] = 1;
      }
    }
    if (errors && err_stride) {
      strncpy(errors + (size_t)i * err_stride, perr, err_stride - 1);
      errors[(size_t)i * err_stride + err_stride - 1] = '\0';
    }
  }
  free(traj);
  return 0;
}
