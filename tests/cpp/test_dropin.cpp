// The C++ drop-in (include/vqeforge_b200/vqeforge.hpp) exercised the way
// the reference's own Catch2 tests use vqeforge:: (test_statevector.cpp,
// test_vqe.cpp, test_sweep.cpp), with expected values taken from those
// tests and from tests/golden.  `--host-only` runs the subset that needs no
// GPU.  Prints "ok N" and exits 0, or reports the first failure and exits 1.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numbers>
#include <stdexcept>
#include <string>

#include "vqeforge_b200/vqeforge.hpp"

namespace {
int checks = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    ++checks;                                                               \
    if (!(cond)) {                                                          \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      std::exit(1);                                                         \
    }                                                                       \
  } while (0)
template <typename E, typename F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}
}  // namespace

using namespace vqeforge;

static void host_part() {
  // test_sweep.cpp:25-41
  const auto grid = bond_grid(0.5, 2.0, 7);
  CHECK(grid.size() == 7 && grid.front() == 0.5 && grid.back() == 2.0);
  CHECK(throws<std::invalid_argument>([] { bond_grid(1.0, 0.5, 4); }));
  // test_sweep.cpp:52-57
  const auto ch = split_chunks(100, 3);
  CHECK(ch[0].second - ch[0].first == 34 && ch[1].second - ch[1].first == 33);
  CHECK(throws<std::invalid_argument>([] { split_chunks(10, 0); }));
  // test_vqe.cpp:119-138
  const AdamState st(1);
  const auto [first, s2] = adam_step(st, {1.0}, {0.0}, AdamConfig{});
  CHECK(std::abs(first[0] - (-0.009999999900000002)) < 1e-15 && s2.step == 1);
  CHECK(throws<std::invalid_argument>([&] { adam_step(st, {1.0, 2.0}, {0.0}, AdamConfig{}); }));
  // test_chem.cpp:218-247 (15 terms at 0.7414 A)
  const auto h = build_h2_hamiltonian(0.7414);
  CHECK(h.n_qubits == 4 && h.terms.size() == 15);
  CHECK(h.terms[0].is_identity() && std::abs(h.terms[0].coefficient.real() - (-0.098863900993594683)) < 1e-12);
  CHECK(throws<BondLengthOutOfRange>([] { build_h2_hamiltonian(0.01); }));
  CHECK(throws<std::domain_error>([] { build_h2_hamiltonian(0.01); }));
  // pauli.hpp:180-201
  const auto c = canonicalize(QubitHamiltonian{2, {PauliTerm(0.5, {{1, PauliAxis::Z}}), PauliTerm(0.25, {{1, PauliAxis::Z}}),
                                                   PauliTerm(1e-13, {{0, PauliAxis::X}}), PauliTerm(2.0, {})}});
  CHECK(c.terms.size() == 2 && c.terms[0].is_identity() && c.terms[1].coefficient.real() == 0.75);
  CHECK(build_tfim(5, 1.0, 1.0).terms.size() == 9);
  CHECK(memory_estimate(26) == 1024ull * 1024 * 1024);
  CHECK(throws<std::invalid_argument>([] { PauliTerm(1.0, {{0, PauliAxis::I}}); }));
}

static void gpu_part() {
  // test_statevector.cpp:96-132
  StateVector psi(1);
  apply_gate(psi, Gate::pauli_x(0));
  CHECK(psi.amplitudes[1] == std::complex<double>(1.0, 0.0));
  StateVector full = basis_state(4, {1, 1, 0, 0});
  apply_gate(full, Gate::double_excitation(std::numbers::pi, 0, 1, 2, 3));
  CHECK(std::abs(full.amplitudes[3].real() - 1.0) < 1e-15 && std::abs(full.amplitudes[12]) < 1e-15);
  StateVector two(2);
  CHECK(throws<std::invalid_argument>([&] { apply_gate(two, Gate::cnot(0, 0)); }));
  CHECK(throws<std::invalid_argument>([&] { expectation(two, build_z_sum(3)); }));
  // test_statevector.cpp:185-196
  CHECK(std::abs(expectation(basis_state(4, {1, 1, 1, 1}), build_z_sum(4)) + 4.0) < 1e-15);
  // test_vqe.cpp:82-89 / :140-150 / :171-180 / :228-236
  const auto& kH2 = AnsatzSpec::h2_double_excitation();
  const auto h = build_h2_hamiltonian(0.7414);
  const auto r = run_vqe(h, kH2, AdamConfig{});
  CHECK(r.iterations_run == 200 && r.trajectory.size() == 201 && r.energy == r.trajectory.back());
  CHECK(std::abs(r.energy - (-1.1372701752231376)) < 1e-10);  // tests/golden/vqe_runs.json
  AdamConfig tol;
  tol.gradient_tolerance = 1e3;
  const auto r0 = run_vqe(h, kH2, tol);
  CHECK(r0.iterations_run == 0 && r0.circuit_evaluations == 3);
  AdamConfig five;
  five.max_iterations = 5;
  CHECK(run_vqe(build_h2_hamiltonian(0.9), kH2, five).circuit_evaluations == 16);
  CHECK(throws<std::invalid_argument>([&] { run_vqe(h, kH2, AdamConfig{}, {0.1, 0.2}); }));
  QubitHamiltonian bad;
  bad.n_qubits = 4;
  PauliTerm nan_term;
  nan_term.coefficient = {std::numeric_limits<double>::quiet_NaN(), 0.0};
  bad.terms.push_back(nan_term);
  bool threw = false;
  try {
    run_vqe(bad, kH2, AdamConfig{});
  } catch (const std::runtime_error& e) {
    threw = std::string(e.what()).find("non-finite energy at iteration") != std::string::npos;
  }
  CHECK(threw);
  // gradient vs finite differences (test_vqe.cpp:91-106)
  const double g = gradient({0.3}, h, kH2)[0];
  const double fd = (energy({0.3 + 1e-5}, h, kH2) - energy({0.3 - 1e-5}, h, kH2)) / 2e-5;
  CHECK(std::abs(g - fd) < 1e-7);
  // test_sweep.cpp:101-143
  SweepConfig base;
  base.d_min = 0.5;
  base.d_max = 2.0;
  base.n_points = 8;
  base.adam.max_iterations = 25;
  const auto a = run_sweep(base);
  base.workers = 3;
  const auto b = run_sweep(base);
  CHECK(a.all_ok && b.all_ok && b.per_worker_seconds.size() == 3);
  for (std::size_t i = 0; i < a.points.size(); ++i)
    CHECK(a.points[i].energy_hartree == b.points[i].energy_hartree && a.points[i].iterations == b.points[i].iterations);
  SweepConfig badc;
  badc.d_min = 0.01;
  badc.d_max = 1.0;
  badc.n_points = 2;
  badc.adam.max_iterations = 10;
  const auto rep = run_sweep(badc);
  CHECK(!rep.all_ok && !rep.points[0].ok && !rep.points[0].error.empty() && std::isnan(rep.points[0].energy_hartree));
  CHECK(rep.points[1].ok);
  // test_sweep.cpp:195-212
  ScalingConfig sc;
  sc.qubits = {4, 6};
  sc.layers = 1;
  sc.iterations = 150;
  sc.learning_rate = 0.1;
  sc.z_sum_mode = true;
  const auto recs = run_scaling_study(sc);
  CHECK(recs.size() == 2 && recs[0].state_bytes == 256 && recs[1].state_bytes == 1024);
  CHECK(std::abs(recs[0].final_energy - (-4.0)) < 0.08 && recs[1].final_energy < 0.0);
  ScalingConfig big;
  big.qubits = {28};
  CHECK(throws<std::invalid_argument>([&] { run_scaling_study(big); }));
  // device-resident state for large registers
  gpu::DeviceState d(20);
  std::vector<Gate> gs;
  for (std::uint32_t q = 0; q < 20; ++q) gs.push_back(Gate::ry(0.3, q));
  gpu::apply_circuit(d, gs);
  CHECK(std::abs(gpu::expectation(d, build_z_sum(20)) - 20 * std::cos(0.3)) < 1e-10);
  // distributed state (virtual ranks): an HEA layer + TFIM vs the single state
  std::vector<Gate> layer;
  for (std::uint32_t q = 0; q < 16; ++q) layer.push_back(Gate::ry(0.1 * (q + 1), q));
  for (std::uint32_t q = 0; q + 1 < 16; ++q) layer.push_back(Gate::cnot(q, q + 1));
  gpu::DistributedState ds(16, 8);
  gpu::apply_circuit(ds, layer);
  gpu::DeviceState one(16);
  gpu::apply_circuit(one, layer);
  const auto tfim = build_tfim(16, 1.0, 0.7);
  CHECK(std::abs(gpu::expectation(ds, tfim) - gpu::expectation(one, tfim)) < 1e-10);
  const auto lay = ds.layout();
  std::vector<std::uint32_t> sorted_lay(lay);
  std::sort(sorted_lay.begin(), sorted_lay.end());
  for (std::uint32_t q = 0; q < 16; ++q) CHECK(sorted_lay[q] == q);
  CHECK(throws<std::invalid_argument>([&] { gpu::DistributedState bad_world(16, 3); }));
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;
  host_part();
  if (!host_only) gpu_part();
  std::printf("ok %d\n", checks);
  return 0;
}
