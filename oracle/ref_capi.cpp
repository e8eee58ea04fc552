// TEST INFRASTRUCTURE ONLY (oracle/_ref). Not part of the shipped product.
//
// extern "C" shim over the UNMODIFIED reference headers in
// /root/reference/proj/include/vqeforge (compiled in place with -I, never
// copied), so Python tests and bench.py's CPU-baseline leg can call the
// reference's own CPU path through ctypes.  Built by oracle/Makefile into
// oracle/_ref/libvqf_ref.so (git-ignored; travels to the GPU box with the
// snapshot).  Every entry point returns 0 on success or an error class:
//   1 std::invalid_argument   2 std::runtime_error   3 std::logic_error
//   4 std::domain_error       9 other std::exception
// with e.what() copied into `err` (may be NULL).
//
// Hamiltonians cross this boundary in sparse CSR form mirroring
// vqeforge::PauliTerm (pauli.hpp:65-95): coeffs[2T] (re,im), offsets[T+1],
// qubits[offsets[T]], axes[offsets[T]] (1=X 2=Y 3=Z, PauliAxis pauli.hpp:34).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "vqeforge/chem.hpp"
#include "vqeforge/pauli.hpp"
#include "vqeforge/statevector.hpp"
#include "vqeforge/sweep.hpp"
#include "vqeforge/vqe.hpp"
// the reference's own seeded fixtures (tests/test_helpers.hpp:28-69):
// random Pauli sums and random states for the config-3/4 parity tests
#include "test_helpers.hpp"

#include <chrono>

using namespace vqeforge;

namespace {

void put_err(char* err, std::size_t cap, const char* msg) {
  if (err == nullptr || cap == 0) return;
  std::strncpy(err, msg, cap - 1);
  err[cap - 1] = '\0';
}

template <typename F>
int guarded(char* err, std::size_t cap, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    put_err(err, cap, e.what());
    return 1;
  } catch (const std::domain_error& e) {
    put_err(err, cap, e.what());
    return 4;
  } catch (const std::runtime_error& e) {
    put_err(err, cap, e.what());
    return 2;
  } catch (const std::logic_error& e) {
    put_err(err, cap, e.what());
    return 3;
  } catch (const std::exception& e) {
    put_err(err, cap, e.what());
    return 9;
  }
}

// Raw construction (no PauliTerm validation) so tests can feed the same
// malformed inputs the reference tests build field by field
// (test_vqe.cpp:238-254 NaN coefficient).
QubitHamiltonian ham_in(std::uint32_t n_qubits, std::uint32_t n_terms, const double* coeffs,
                        const std::uint32_t* offsets, const std::uint32_t* qubits,
                        const std::uint8_t* axes) {
  QubitHamiltonian h;
  h.n_qubits = n_qubits;
  h.terms.resize(n_terms);
  for (std::uint32_t t = 0; t < n_terms; ++t) {
    h.terms[t].coefficient = {coeffs[2 * t], coeffs[2 * t + 1]};
    for (std::uint32_t k = offsets[t]; k < offsets[t + 1]; ++k) {
      h.terms[t].axes.emplace_back(qubits[k], static_cast<PauliAxis>(axes[k]));
    }
  }
  return h;
}

void ham_out(const QubitHamiltonian& h, std::uint32_t* n_terms, double* coeffs,
             std::uint32_t* offsets, std::uint32_t* qubits, std::uint8_t* axes,
             std::uint32_t cap_terms, std::uint32_t cap_axes) {
  if (h.terms.size() > cap_terms) throw std::runtime_error("ref_capi: term capacity");
  std::uint32_t k = 0;
  offsets[0] = 0;
  for (std::size_t t = 0; t < h.terms.size(); ++t) {
    coeffs[2 * t] = h.terms[t].coefficient.real();
    coeffs[2 * t + 1] = h.terms[t].coefficient.imag();
    for (const auto& [q, a] : h.terms[t].axes) {
      if (k >= cap_axes) throw std::runtime_error("ref_capi: axis capacity");
      qubits[k] = q;
      axes[k] = static_cast<std::uint8_t>(a);
      ++k;
    }
    offsets[t + 1] = k;
  }
  *n_terms = static_cast<std::uint32_t>(h.terms.size());
}

StateVector sv_in(std::uint32_t n, const double* amps) {
  StateVector psi;
  psi.n_qubits = n;
  psi.amplitudes.resize(std::size_t{1} << n);
  for (std::size_t i = 0; i < psi.amplitudes.size(); ++i) {
    psi.amplitudes[i] = {amps[2 * i], amps[2 * i + 1]};
  }
  return psi;
}

void sv_out(const StateVector& psi, double* amps) {
  for (std::size_t i = 0; i < psi.amplitudes.size(); ++i) {
    amps[2 * i] = psi.amplitudes[i].real();
    amps[2 * i + 1] = psi.amplitudes[i].imag();
  }
}

AnsatzSpec spec_in(int kind, std::uint32_t layers) {
  return kind == 0 ? AnsatzSpec::h2_double_excitation() : AnsatzSpec::hardware_efficient(layers);
}

AdamConfig adam_in(double lr, double b1, double b2, double eps, int max_iter, int has_tol,
                   double tol) {
  AdamConfig c;
  c.learning_rate = lr;
  c.beta1 = b1;
  c.beta2 = b2;
  c.epsilon = eps;
  c.max_iterations = max_iter;
  if (has_tol) c.gradient_tolerance = tol;
  return c;
}

}  // namespace

extern "C" {

#define HAM_IN_ARGS                                                                       \
  std::uint32_t n_qubits, std::uint32_t n_terms, const double *coeffs,                   \
      const std::uint32_t *offsets, const std::uint32_t *qubits, const std::uint8_t *axes
#define HAM_OUT_ARGS                                                                \
  std::uint32_t *o_n_terms, double *o_coeffs, std::uint32_t *o_offsets,            \
      std::uint32_t *o_qubits, std::uint8_t *o_axes, std::uint32_t cap_terms,       \
      std::uint32_t cap_axes
#define HAM_IN ham_in(n_qubits, n_terms, coeffs, offsets, qubits, axes)
#define HAM_OUT(h) ham_out(h, o_n_terms, o_coeffs, o_offsets, o_qubits, o_axes, cap_terms, cap_axes)

// chem.hpp:473 build_h2_hamiltonian (thread-local memo; HF + JW on miss).
int ref_build_h2_hamiltonian(double bond_angstrom, HAM_OUT_ARGS, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] { HAM_OUT(build_h2_hamiltonian(bond_angstrom)); });
}

// chem.hpp:280 run_hartree_fock -> {hf_energy, electronic, nuclear, scf_iterations}
int ref_hartree_fock(double bond_angstrom, double* out4, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    const auto s = run_hartree_fock(bond_angstrom);
    out4[0] = s.hf_energy;
    out4[1] = s.electronic_energy;
    out4[2] = s.nuclear_repulsion;
    out4[3] = s.scf_iterations;
  });
}

// sweep.hpp:209 / :227
int ref_build_tfim(std::uint32_t n, double coupling, double field, HAM_OUT_ARGS, char* err,
                   std::size_t errcap) {
  return guarded(err, errcap, [&] { HAM_OUT(build_tfim(n, coupling, field)); });
}
int ref_build_z_sum(std::uint32_t n, HAM_OUT_ARGS, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] { HAM_OUT(build_z_sum(n)); });
}

// pauli.hpp:180 canonicalize (input goes through the validating PauliTerm
// constructor first, as QubitHamiltonian users do).
int ref_canonicalize(HAM_IN_ARGS, HAM_OUT_ARGS, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    std::vector<PauliTerm> terms;
    for (std::uint32_t t = 0; t < n_terms; ++t) {
      std::vector<std::pair<std::uint32_t, PauliAxis>> ax;
      for (std::uint32_t k = offsets[t]; k < offsets[t + 1]; ++k)
        ax.emplace_back(qubits[k], static_cast<PauliAxis>(axes[k]));
      terms.emplace_back(std::complex<double>{coeffs[2 * t], coeffs[2 * t + 1]}, ax);
    }
    HAM_OUT(canonicalize(QubitHamiltonian{n_qubits, std::move(terms)}));
  });
}

// pauli.hpp:294 to_text
int ref_to_text(HAM_IN_ARGS, char* buf, std::size_t cap, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    const std::string s = to_text(HAM_IN);
    if (s.size() + 1 > cap) throw std::runtime_error("ref_capi: text capacity");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

// pauli.hpp:278 exact_ground_energy (dense, <= 12 qubits)
int ref_exact_ground_energy(HAM_IN_ARGS, double* out, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] { *out = exact_ground_energy(HAM_IN); });
}

// statevector.hpp:148 apply_gate, gate by gate. kinds: 0 X, 1 RY, 2 CNOT, 3 DE;
// wires4[4*g ...] holds up to 4 wires (n_wires per kind).
int ref_apply_gates(std::uint32_t n, double* amps, std::uint32_t n_gates, const int* kinds,
                    const double* angles, const std::uint32_t* n_wires,
                    const std::uint32_t* wires4, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    StateVector psi = sv_in(n, amps);
    for (std::uint32_t g = 0; g < n_gates; ++g) {
      Gate gate;
      gate.kind = static_cast<GateKind>(kinds[g]);
      gate.angle = angles[g];
      gate.wires.assign(wires4 + 4 * g, wires4 + 4 * g + n_wires[g]);
      apply_gate(psi, gate);
    }
    sv_out(psi, amps);
  });
}

// statevector.hpp:61 basis_state
int ref_basis_state(std::uint32_t n, const int* bits, std::uint32_t n_bits, double* amps,
                    char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    sv_out(basis_state(n, std::vector<int>(bits, bits + n_bits)), amps);
  });
}

// statevector.hpp:217 expectation
int ref_expectation(std::uint32_t sv_qubits, const double* amps, HAM_IN_ARGS, double* out,
                    char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] { *out = expectation(sv_in(sv_qubits, amps), HAM_IN); });
}

// vqe.hpp:65 prepare_ansatz
int ref_prepare_ansatz(int kind, std::uint32_t layers, const double* theta, std::uint32_t n_theta,
                       std::uint32_t n, double* amps, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    sv_out(prepare_ansatz(spec_in(kind, layers), std::vector<double>(theta, theta + n_theta), n),
           amps);
  });
}

// vqe.hpp:99 energy, :112 gradient
int ref_energy(int kind, std::uint32_t layers, const double* theta, std::uint32_t n_theta,
               HAM_IN_ARGS, double* out, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    *out = energy(std::vector<double>(theta, theta + n_theta), HAM_IN, spec_in(kind, layers));
  });
}
int ref_gradient(int kind, std::uint32_t layers, const double* theta, std::uint32_t n_theta,
                 HAM_IN_ARGS, double* out, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    const auto g =
        gradient(std::vector<double>(theta, theta + n_theta), HAM_IN, spec_in(kind, layers));
    for (std::size_t k = 0; k < g.size(); ++k) out[k] = g[k];
  });
}

// vqe.hpp:152 adam_step
int ref_adam_step(const double* m, const double* v, std::int64_t step, const double* grad,
                  const double* theta, std::uint32_t n, double lr, double b1, double b2,
                  double eps, double* theta_out, double* m_out, double* v_out,
                  std::int64_t* step_out, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    AdamState s(n);
    s.m.assign(m, m + n);
    s.v.assign(v, v + n);
    s.step = step;
    auto [t, ns] = adam_step(s, std::vector<double>(grad, grad + n),
                             std::vector<double>(theta, theta + n),
                             adam_in(lr, b1, b2, eps, 0, 0, 0.0));
    for (std::uint32_t k = 0; k < n; ++k) {
      theta_out[k] = t[k];
      m_out[k] = ns.m[k];
      v_out[k] = ns.v[k];
    }
    *step_out = ns.step;
  });
}

// vqe.hpp:194 run_vqe. traj must hold max_iter+1 doubles, theta_out P.
int ref_run_vqe(HAM_IN_ARGS, int kind, std::uint32_t layers, double lr, double b1, double b2,
                double eps, int max_iter, int has_tol, double tol, const double* init,
                std::uint32_t n_init, double* energy_out, double* theta_out, double* traj,
                std::uint32_t* traj_len, int* iters, std::uint64_t* evals, double* wall,
                char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    const auto r = run_vqe(HAM_IN, spec_in(kind, layers),
                           adam_in(lr, b1, b2, eps, max_iter, has_tol, tol),
                           std::vector<double>(init, init + n_init));
    *energy_out = r.energy;
    for (std::size_t k = 0; k < r.theta.size(); ++k) theta_out[k] = r.theta[k];
    for (std::size_t k = 0; k < r.trajectory.size(); ++k) traj[k] = r.trajectory[k];
    *traj_len = static_cast<std::uint32_t>(r.trajectory.size());
    *iters = r.iterations_run;
    *evals = r.circuit_evaluations;
    *wall = r.wall_seconds;
  });
}

// sweep.hpp:68 / :93 / :111
int ref_bond_grid(double d_min, double d_max, int n_points, double* out, char* err,
                  std::size_t errcap) {
  return guarded(err, errcap, [&] {
    const auto g = bond_grid(d_min, d_max, n_points);
    for (std::size_t i = 0; i < g.size(); ++i) out[i] = g[i];
  });
}
int ref_split_chunks(std::uint64_t n_items, std::uint64_t n_chunks, std::uint64_t* begin_end,
                     char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    const auto c = split_chunks(n_items, n_chunks);
    for (std::size_t i = 0; i < c.size(); ++i) {
      begin_end[2 * i] = c[i].first;
      begin_end[2 * i + 1] = c[i].second;
    }
  });
}
int ref_effective_workers(int requested, int* out, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] { *out = effective_workers(requested); });
}

// sweep.hpp:128 run_sweep. Per-point arrays sized n_points; theta_star is
// one parameter per point (H2 ansatz). Per-point error strings are packed
// into errors[n_points * err_stride].
int ref_run_sweep(double d_min, double d_max, int n_points, int workers, double lr, double b1,
                  double b2, double eps, int max_iter, int has_tol, double tol, double* bond,
                  double* energy, double* theta_star, int* iterations, double* point_wall,
                  int* ok, char* errors, std::size_t err_stride, double* per_worker,
                  double* total_wall, int* all_ok, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    SweepConfig c;
    c.d_min = d_min;
    c.d_max = d_max;
    c.n_points = n_points;
    c.workers = workers;
    c.adam = adam_in(lr, b1, b2, eps, max_iter, has_tol, tol);
    const SweepReport r = run_sweep(c);
    for (std::size_t i = 0; i < r.points.size(); ++i) {
      const auto& p = r.points[i];
      bond[i] = p.bond_angstrom;
      energy[i] = p.energy_hartree;
      theta_star[i] = p.theta_star.empty() ? 0.0 : p.theta_star[0];
      iterations[i] = p.iterations;
      point_wall[i] = p.wall_seconds;
      ok[i] = p.ok ? 1 : 0;
      if (errors != nullptr && err_stride > 0) put_err(errors + i * err_stride, err_stride, p.error.c_str());
    }
    for (std::size_t w = 0; w < r.per_worker_seconds.size(); ++w) per_worker[w] = r.per_worker_seconds[w];
    *total_wall = r.total_wall_seconds;
    *all_ok = r.all_ok ? 1 : 0;
  });
}

// sweep.hpp:265 run_scaling_study. Records: n_qubits, state_bytes,
// runtime_seconds, final_energy, iterations_run per width.
int ref_run_scaling_study(const std::uint32_t* widths, std::uint32_t n_widths, std::uint32_t layers,
                          int iterations, double lr, double coupling, double field, int z_sum,
                          double theta_init, int force, std::uint64_t* state_bytes,
                          double* runtime, double* final_energy, int* iters_run, char* err,
                          std::size_t errcap) {
  return guarded(err, errcap, [&] {
    ScalingConfig c;
    c.qubits.assign(widths, widths + n_widths);
    c.layers = layers;
    c.iterations = iterations;
    c.learning_rate = lr;
    c.coupling = coupling;
    c.field = field;
    c.z_sum_mode = z_sum != 0;
    c.theta_init = theta_init;
    c.force = force != 0;
    const auto recs = run_scaling_study(c);
    for (std::size_t i = 0; i < recs.size(); ++i) {
      state_bytes[i] = recs[i].state_bytes;
      runtime[i] = recs[i].runtime_seconds;
      final_energy[i] = recs[i].final_energy;
      iters_run[i] = recs[i].iterations_run;
    }
  });
}

// test_helpers.hpp:49-58 random_hamiltonian(mt19937(seed), n, T, real)
// (uncanonicalised; tests canonicalise through ref_canonicalize as the
// reference tests do, test_statevector.cpp:200).
int ref_random_hamiltonian(std::uint32_t seed, std::uint32_t n, int n_terms, int real, HAM_OUT_ARGS, char* err,
                           std::size_t errcap) {
  return guarded(err, errcap, [&] {
    std::mt19937 rng(seed);
    HAM_OUT(testutil::random_hamiltonian(rng, n, n_terms, real != 0));
  });
}

// test_helpers.hpp:61-69 random_state(mt19937(seed), n)
int ref_random_state(std::uint32_t seed, std::uint32_t n, double* amps, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    std::mt19937 rng(seed);
    sv_out(testutil::random_state(rng, n), amps);
  });
}

// CPU baselines for bench.py (configs 3/4): the reference's single-threaded
// apply_gate / expectation, one call timed by steady_clock on a state that
// is already resident (no copies inside the timed region), best of `reps`.
int ref_time_apply_gate(std::uint32_t n, const double* amps, int kind, double angle, std::uint32_t n_wires,
                        const std::uint32_t* wires, int reps, double* seconds, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    StateVector psi = sv_in(n, amps);
    Gate gate;
    gate.kind = static_cast<GateKind>(kind);
    gate.angle = angle;
    gate.wires.assign(wires, wires + n_wires);
    double best = 1e300;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      apply_gate(psi, gate);
      const auto t1 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    }
    *seconds = best;
  });
}

int ref_time_expectation(std::uint32_t sv_qubits, const double* amps, HAM_IN_ARGS, int reps, double* value,
                         double* seconds, char* err, std::size_t errcap) {
  return guarded(err, errcap, [&] {
    const StateVector psi = sv_in(sv_qubits, amps);
    const QubitHamiltonian h = HAM_IN;
    double best = 1e300;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      *value = expectation(psi, h);
      const auto t1 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    }
    *seconds = best;
  });
}

}  // extern "C"
