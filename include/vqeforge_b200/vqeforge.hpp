// vqeforge_b200/vqeforge.hpp — C++ drop-in for the reference VQE Forge hot
// path (/root/reference/proj/include/vqeforge/{pauli,statevector,vqe,sweep,
// chem}.hpp), implemented over the C ABI in vqf_b200.h (libvqf_b200.so).
//
// Same namespace (vqeforge), type names, factory helpers, function
// signatures and exception types as the reference; link with
//   -I<repo>/include -L<repo>/paper_2601_09951_b200 -lvqf_b200
// Differences a caller can observe are listed in INTEGRATION.md; the main
// one: StateVector stays a host value type (public `amplitudes`, as in
// statevector.hpp:33-51), so apply_gate / expectation on it stage the state
// through the GPU per call.  The hot path — energy, gradient, run_vqe,
// run_sweep, run_scaling_study — runs entirely on the device; for large
// registers keep the state resident with vqeforge::gpu::DeviceState.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "vqf_b200.h"

namespace vqeforge {

// ---------------------------------------------------------------- errors
// chem.hpp:38-52
struct BondLengthOutOfRange : std::domain_error {
  explicit BondLengthOutOfRange(const std::string& what) : std::domain_error(what) {}
};

namespace detail {
// Maps a C-ABI status back onto the reference's exception types
// (SURVEY.md §8b): invalid_argument / runtime_error / logic_error /
// BondLengthOutOfRange.
inline void check(int rc) {
  if (rc == VQF_OK) return;
  const std::string msg = vqf_last_error();
  switch (rc) {
    case VQF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case VQF_LOGIC_ERROR: throw std::logic_error(msg);
    case VQF_DOMAIN_ERROR: throw BondLengthOutOfRange(msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace detail

// ----------------------------------------------------------------- pauli
enum class PauliAxis : std::uint8_t { I = 0, X = 1, Y = 2, Z = 3 };  // pauli.hpp:34

inline constexpr double kCoefficientDropThreshold = 1e-12;  // pauli.hpp:47
inline constexpr double kHermiticityTolerance = 1e-10;      // pauli.hpp:49

// pauli.hpp:65-95
struct PauliTerm {
  std::complex<double> coefficient{1.0, 0.0};
  std::vector<std::pair<std::uint32_t, PauliAxis>> axes;

  PauliTerm() = default;
  PauliTerm(std::complex<double> coeff, std::vector<std::pair<std::uint32_t, PauliAxis>> ops)
      : coefficient(coeff), axes(std::move(ops)) {
    std::sort(axes.begin(), axes.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (std::size_t i = 0; i < axes.size(); ++i) {
      if (axes[i].second == PauliAxis::I) throw std::invalid_argument("explicit identity entry in PauliTerm");
      if (i > 0 && axes[i].first == axes[i - 1].first) throw std::invalid_argument("duplicate qubit index in PauliTerm");
    }
    if (!std::isfinite(coefficient.real()) || !std::isfinite(coefficient.imag()))
      throw std::invalid_argument("non-finite PauliTerm coefficient");
  }
  bool is_identity() const { return axes.empty(); }
  std::uint32_t max_qubit_index() const { return axes.empty() ? 0 : axes.back().first; }
};

// pauli.hpp:116-129
struct QubitHamiltonian {
  std::uint32_t n_qubits = 0;
  std::vector<PauliTerm> terms;
  QubitHamiltonian() = default;
  QubitHamiltonian(std::uint32_t n, std::vector<PauliTerm> ts) : n_qubits(n), terms(std::move(ts)) {
    for (const auto& t : terms)
      if (!t.axes.empty() && t.max_qubit_index() >= n_qubits)
        throw std::invalid_argument("PauliTerm index exceeds register size");
  }
};

namespace detail {

// CSR view of a QubitHamiltonian for the C ABI (owns its arrays).
struct CsrHam {
  std::vector<double> coeffs;
  std::vector<std::uint32_t> offsets, qubits;
  std::vector<std::uint8_t> axes;
  vqf_hamiltonian view{};
  explicit CsrHam(const QubitHamiltonian& h) {
    offsets.push_back(0);
    for (const auto& t : h.terms) {
      coeffs.push_back(t.coefficient.real());
      coeffs.push_back(t.coefficient.imag());
      for (const auto& [q, a] : t.axes) {
        qubits.push_back(q);
        axes.push_back(static_cast<std::uint8_t>(a));
      }
      offsets.push_back(static_cast<std::uint32_t>(qubits.size()));
    }
    if (coeffs.empty()) coeffs.assign(2, 0.0);
    if (qubits.empty()) {
      qubits.push_back(0);
      axes.push_back(0);
    }
    view = {h.n_qubits, static_cast<std::uint32_t>(h.terms.size()), coeffs.data(), offsets.data(), qubits.data(),
            axes.data()};
  }
};

struct HamBuffer {
  std::vector<double> coeffs;
  std::vector<std::uint32_t> offsets, qubits;
  std::vector<std::uint8_t> axes;
  vqf_hamiltonian_out out{};
  HamBuffer(std::uint32_t cap_terms, std::uint32_t cap_axes)
      : coeffs(2 * cap_terms), offsets(cap_terms + 1), qubits(cap_axes), axes(cap_axes) {
    out = {0, coeffs.data(), offsets.data(), qubits.data(), axes.data(), cap_terms, cap_axes};
  }
  QubitHamiltonian result(std::uint32_t n_qubits) const {
    QubitHamiltonian h;
    h.n_qubits = n_qubits;
    for (std::uint32_t t = 0; t < out.n_terms; ++t) {
      PauliTerm term;
      term.coefficient = {coeffs[2 * t], coeffs[2 * t + 1]};
      for (std::uint32_t k = offsets[t]; k < offsets[t + 1]; ++k)
        term.axes.emplace_back(qubits[k], static_cast<PauliAxis>(axes[k]));
      h.terms.push_back(std::move(term));
    }
    return h;
  }
};

}  // namespace detail

// pauli.hpp:180-201
inline QubitHamiltonian canonicalize(const QubitHamiltonian& h) {
  detail::CsrHam in(h);
  detail::HamBuffer buf(static_cast<std::uint32_t>(h.terms.size()) + 1,
                        static_cast<std::uint32_t>(in.qubits.size()) + 1);
  detail::check(vqf_canonicalize(&in.view, &buf.out));
  return buf.result(h.n_qubits);
}

inline char axis_char(PauliAxis a) {
  switch (a) {
    case PauliAxis::I: return 'I';
    case PauliAxis::X: return 'X';
    case PauliAxis::Y: return 'Y';
    case PauliAxis::Z: return 'Z';
  }
  return '?';
}

// pauli.hpp:294-309: one term per line, "%.17g %.17g <axis><index>...".
inline std::string to_text(const QubitHamiltonian& h) {
  std::string out;
  char buf[64];
  for (const auto& t : h.terms) {
    std::snprintf(buf, sizeof buf, "%.17g", t.coefficient.real());
    out += buf;
    std::snprintf(buf, sizeof buf, "%.17g", t.coefficient.imag());
    out += ' ';
    out += buf;
    if (!t.axes.empty()) {
      out += ' ';
      for (const auto& [q, a] : t.axes) out += axis_char(a) + std::to_string(q);
    }
    out += '\n';
  }
  return out;
}

inline constexpr std::uint32_t kDenseOracleMaxQubits = 12;  // pauli.hpp:51

struct TooManyQubits : std::domain_error {  // pauli.hpp:53-58
  explicit TooManyQubits(std::uint32_t n)
      : std::domain_error("dense oracle limited to " + std::to_string(kDenseOracleMaxQubits) + " qubits, got " +
                          std::to_string(n)) {}
};

// pauli.hpp:278-285 exact_ground_energy: lowest eigenvalue of the dense
// realisation (host; the n x n Hermitian matrix is embedded as the 2n x 2n
// real symmetric [[A, -B], [B, A]] and diagonalised by cyclic Jacobi — the
// oracle used by the reference's variational-bound checks, not a hot path).
inline double exact_ground_energy(const QubitHamiltonian& h) {
  if (h.n_qubits > kDenseOracleMaxQubits) throw TooManyQubits(h.n_qubits);
  const std::size_t D = std::size_t{1} << h.n_qubits, M = 2 * D;
  std::vector<double> a(M * M, 0.0);
  for (const auto& t : h.terms) {
    std::uint64_t flip = 0, yz = 0;
    unsigned ny = 0;
    for (const auto& [q, ax] : t.axes) {
      const std::uint64_t bit = std::uint64_t{1} << (h.n_qubits - 1 - q);
      if (ax == PauliAxis::X || ax == PauliAxis::Y) flip |= bit;
      if (ax == PauliAxis::Y || ax == PauliAxis::Z) yz |= bit;
      if (ax == PauliAxis::Y) ++ny;
    }
    static const std::complex<double> base_tab[4] = {{1, 0}, {0, -1}, {-1, 0}, {0, 1}};
    const std::complex<double> cb = t.coefficient * base_tab[ny % 4];
    for (std::size_t i = 0; i < D; ++i) {
      const std::complex<double> v = (__builtin_popcountll(i & yz) & 1) ? -cb : cb;
      const std::size_t j = i ^ flip;
      a[i * M + j] += v.real();
      a[(i + D) * M + (j + D)] += v.real();
      a[i * M + (j + D)] -= v.imag();
      a[(i + D) * M + j] += v.imag();
    }
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (std::size_t i = 0; i < M; ++i)
      for (std::size_t j = i + 1; j < M; ++j) off += a[i * M + j] * a[i * M + j];
    if (off < 1e-30) break;
    for (std::size_t p = 0; p < M; ++p)
      for (std::size_t q = p + 1; q < M; ++q) {
        const double apq = a[p * M + q];
        if (std::abs(apq) < 1e-300) continue;
        const double theta = (a[q * M + q] - a[p * M + p]) / (2.0 * apq);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(tt * tt + 1.0), s = tt * c;
        for (std::size_t k = 0; k < M; ++k) {
          const double akp = a[k * M + p], akq = a[k * M + q];
          a[k * M + p] = c * akp - s * akq;
          a[k * M + q] = s * akp + c * akq;
        }
        for (std::size_t k = 0; k < M; ++k) {
          const double apk = a[p * M + k], aqk = a[q * M + k];
          a[p * M + k] = c * apk - s * aqk;
          a[q * M + k] = s * apk + c * aqk;
        }
      }
  }
  double e0 = a[0];
  for (std::size_t i = 1; i < M; ++i) e0 = std::min(e0, a[i * M + i]);
  return e0;
}

// ------------------------------------------------------------ statevector
// statevector.hpp:33-51 (host value type, as in the reference)
struct StateVector {
  std::uint32_t n_qubits = 0;
  std::vector<std::complex<double>> amplitudes;
  StateVector() = default;
  explicit StateVector(std::uint32_t n) : n_qubits(n), amplitudes(std::size_t{1} << n, {0.0, 0.0}) {
    amplitudes[0] = {1.0, 0.0};
  }
  std::uint64_t dimension() const { return std::uint64_t{1} << n_qubits; }
  double norm() const {
    double s = 0.0;
    for (const auto& a : amplitudes) s += std::norm(a);
    return std::sqrt(s);
  }
};

inline std::uint64_t memory_estimate(std::uint32_t n_qubits) { return vqf_memory_estimate(n_qubits); }

inline StateVector basis_state(std::uint32_t n_qubits, const std::vector<int>& bits) {
  if (bits.size() != n_qubits) throw std::invalid_argument("basis_state: bit count != qubit count");
  StateVector psi(n_qubits);
  psi.amplitudes[0] = {0.0, 0.0};
  std::uint64_t index = 0;
  for (std::uint32_t q = 0; q < n_qubits; ++q)
    if (bits[q]) index |= std::uint64_t{1} << (n_qubits - 1 - q);
  psi.amplitudes[index] = {1.0, 0.0};
  return psi;
}

// statevector.hpp:76-101 (+ SingleExcitation)
enum class GateKind : std::uint8_t { PauliX, RY, CNOT, DoubleExcitation, SingleExcitation };

struct Gate {
  GateKind kind = GateKind::PauliX;
  double angle = 0.0;
  std::vector<std::uint32_t> wires;
  static Gate pauli_x(std::uint32_t q) { return Gate{GateKind::PauliX, 0.0, {q}}; }
  static Gate ry(double theta, std::uint32_t q) { return Gate{GateKind::RY, theta, {q}}; }
  static Gate cnot(std::uint32_t c, std::uint32_t t) { return Gate{GateKind::CNOT, 0.0, {c, t}}; }
  static Gate double_excitation(double theta, std::uint32_t w0, std::uint32_t w1, std::uint32_t w2, std::uint32_t w3) {
    return Gate{GateKind::DoubleExcitation, theta, {w0, w1, w2, w3}};
  }
  static Gate single_excitation(double theta, std::uint32_t w0, std::uint32_t w1) {
    return Gate{GateKind::SingleExcitation, theta, {w0, w1}};
  }
};

namespace gpu {

// A device-resident state (batch 1, fp64 by default): the object to keep
// between gates when the register is large.
class DeviceState {
 public:
  explicit DeviceState(std::uint32_t n_qubits, int device = 0, bool fp32 = false) {
    detail::check(vqf_sv_create(n_qubits, 1, fp32 ? VQF_F32 : VQF_F64, device, &h_));
  }
  explicit DeviceState(const StateVector& psi, int device = 0) : DeviceState(psi.n_qubits, device) { upload(psi); }
  ~DeviceState() {
    if (h_) vqf_sv_destroy(h_);
  }
  DeviceState(const DeviceState&) = delete;
  DeviceState& operator=(const DeviceState&) = delete;
  void upload(const StateVector& psi) {
    detail::check(vqf_sv_upload(h_, reinterpret_cast<const double*>(psi.amplitudes.data())));
  }
  void download(StateVector& psi) const {
    std::uint32_t n = 0;
    detail::check(vqf_sv_info(h_, &n, nullptr, nullptr, nullptr));
    psi.n_qubits = n;
    psi.amplitudes.resize(std::size_t{1} << n);
    detail::check(vqf_sv_download(h_, reinterpret_cast<double*>(psi.amplitudes.data())));
  }
  vqf_sv handle() const { return h_; }

 private:
  vqf_sv h_ = nullptr;
};

inline vqf_gate to_c(const Gate& g) {
  vqf_gate c{};
  c.kind = static_cast<std::int32_t>(g.kind);
  c.n_wires = static_cast<std::uint32_t>(g.wires.size());
  for (std::size_t i = 0; i < g.wires.size() && i < 4; ++i) c.wires[i] = g.wires[i];
  c.angle = g.angle;
  return c;
}

inline void apply_gate(DeviceState& psi, const Gate& g) {
  const vqf_gate c = to_c(g);
  detail::check(vqf_apply_gate(psi.handle(), &c));
}

inline void apply_circuit(DeviceState& psi, const std::vector<Gate>& gates) {
  std::vector<vqf_gate> cs;
  for (const auto& g : gates) cs.push_back(to_c(g));
  detail::check(vqf_apply_circuit(psi.handle(), cs.data(), static_cast<std::uint32_t>(cs.size())));
}

inline double expectation(const DeviceState& psi, const QubitHamiltonian& h) {
  detail::CsrHam c(h);
  double e = 0.0;
  detail::check(vqf_expectation(psi.handle(), &c.view, &e));
  return e;
}

// An n-qubit state split over `world` = 2^g shards (BASELINE config 5, beyond
// one GPU's memory; the reference stops at 26 qubits, sweep.hpp:36-38).
// comm == nullptr: every shard on `device` (virtual ranks); otherwise one
// shard per process, exchanges through the caller's communicator (e.g.
// ncclSend / ncclRecv in sendrecv, ncclAllReduce in allreduce_sum; see
// INTEGRATION.md).  The qubit layout is updated lazily (layout()).
class DistributedState {
 public:
  DistributedState(std::uint32_t n_qubits, std::uint32_t world, int device = 0, bool fp32 = false,
                   const vqf_dsv_comm* comm = nullptr, std::uint64_t chunk_bytes = 0) {
    detail::check(vqf_dsv_create(n_qubits, world, fp32 ? VQF_F32 : VQF_F64, device, comm, chunk_bytes, &h_));
    n_ = n_qubits;
  }
  ~DistributedState() {
    if (h_) vqf_dsv_destroy(h_);
  }
  DistributedState(const DistributedState&) = delete;
  DistributedState& operator=(const DistributedState&) = delete;
  std::vector<std::uint32_t> layout() const {
    std::vector<std::uint32_t> pos(n_);
    detail::check(vqf_dsv_layout(h_, pos.data()));
    return pos;
  }
  vqf_dsv handle() const { return h_; }
  std::uint32_t n_qubits() const { return n_; }

 private:
  vqf_dsv h_ = nullptr;
  std::uint32_t n_ = 0;
};

inline void apply_circuit(DistributedState& psi, const std::vector<Gate>& gates) {
  std::vector<vqf_gate> cs;
  for (const auto& g : gates) cs.push_back(to_c(g));
  detail::check(vqf_dsv_apply_circuit(psi.handle(), cs.data(), static_cast<std::uint32_t>(cs.size())));
}

inline double expectation(const DistributedState& psi, const QubitHamiltonian& h) {
  if (h.n_qubits != psi.n_qubits()) throw std::invalid_argument("expectation: qubit count mismatch");
  detail::CsrHam c(h);
  double e = 0.0;
  detail::check(vqf_dsv_expectation(psi.handle(), &c.view, &e));
  return e;
}

}  // namespace gpu

// statevector.hpp:148-207: the host value is staged through the device.
inline void apply_gate(StateVector& psi, const Gate& g) {
  gpu::DeviceState d(psi);
  gpu::apply_gate(d, g);
  d.download(psi);
}

inline void apply_circuit(StateVector& psi, const std::vector<Gate>& gates) {
  gpu::DeviceState d(psi);
  gpu::apply_circuit(d, gates);
  d.download(psi);
}

// statevector.hpp:217-249
inline double expectation(const StateVector& psi, const QubitHamiltonian& h) {
  if (h.n_qubits != psi.n_qubits) throw std::invalid_argument("expectation: qubit count mismatch");
  gpu::DeviceState d(psi);
  return gpu::expectation(d, h);
}

// -------------------------------------------------------------------- vqe
enum class AnsatzKind : std::uint8_t { H2DoubleExcitation, HardwareEfficient };  // vqe.hpp:32

struct AnsatzSpec {  // vqe.hpp:42-52
  AnsatzKind kind = AnsatzKind::H2DoubleExcitation;
  std::uint32_t layers = 2;
  static AnsatzSpec h2_double_excitation() { return AnsatzSpec{AnsatzKind::H2DoubleExcitation, 0}; }
  static AnsatzSpec hardware_efficient(std::uint32_t layers) { return AnsatzSpec{AnsatzKind::HardwareEfficient, layers}; }
};

inline std::size_t n_parameters(const AnsatzSpec& spec, std::uint32_t n_qubits) {
  return vqf_n_parameters(static_cast<std::int32_t>(spec.kind), spec.layers, n_qubits);
}

inline StateVector prepare_ansatz(const AnsatzSpec& spec, const std::vector<double>& theta, std::uint32_t n_qubits) {
  gpu::DeviceState d(n_qubits);
  detail::check(vqf_prepare_ansatz(static_cast<std::int32_t>(spec.kind), spec.layers, theta.data(),
                                   static_cast<std::uint32_t>(theta.size()), d.handle()));
  StateVector psi;
  d.download(psi);
  return psi;
}

inline double energy(const std::vector<double>& theta, const QubitHamiltonian& h, const AnsatzSpec& spec) {
  detail::CsrHam c(h);
  double e = 0.0;
  detail::check(vqf_energy(theta.data(), static_cast<std::uint32_t>(theta.size()), &c.view,
                           static_cast<std::int32_t>(spec.kind), spec.layers, 0, &e));
  return e;
}

inline std::vector<double> gradient(const std::vector<double>& theta, const QubitHamiltonian& h,
                                    const AnsatzSpec& spec) {
  detail::CsrHam c(h);
  std::vector<double> g(theta.size());
  detail::check(vqf_gradient(theta.data(), static_cast<std::uint32_t>(theta.size()), &c.view,
                             static_cast<std::int32_t>(spec.kind), spec.layers, VQF_GRAD_PARAMETER_SHIFT, 0,
                             g.data()));
  return g;
}

struct AdamConfig {  // vqe.hpp:129-138
  double learning_rate = 0.01;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double epsilon = 1e-8;
  int max_iterations = 200;
  std::optional<double> gradient_tolerance{};
};

struct AdamState {  // vqe.hpp:140-146
  std::vector<double> m;
  std::vector<double> v;
  std::int64_t step = 0;
  explicit AdamState(std::size_t n = 0) : m(n, 0.0), v(n, 0.0) {}
};

namespace detail {
inline vqf_adam_config to_c(const AdamConfig& a) {
  return vqf_adam_config{a.learning_rate, a.beta1, a.beta2, a.epsilon, a.max_iterations,
                         a.gradient_tolerance ? 1 : 0, a.gradient_tolerance.value_or(0.0)};
}
}  // namespace detail

// vqe.hpp:152-174
inline std::pair<std::vector<double>, AdamState> adam_step(const AdamState& state, const std::vector<double>& grad,
                                                           const std::vector<double>& theta,
                                                           const AdamConfig& config) {
  if (grad.size() != theta.size() || state.m.size() != theta.size())
    throw std::invalid_argument("adam_step dimension mismatch");
  AdamState next(theta.size());
  std::vector<double> out(theta.size());
  const vqf_adam_config c = detail::to_c(config);
  detail::check(vqf_adam_step(state.m.data(), state.v.data(), state.step, grad.data(), theta.data(),
                              static_cast<std::uint32_t>(theta.size()), &c, out.data(), next.m.data(),
                              next.v.data(), &next.step));
  return {std::move(out), std::move(next)};
}

struct VqeResult {  // vqe.hpp:176-186
  double energy = 0.0;
  std::vector<double> theta;
  std::vector<double> trajectory;
  int iterations_run = 0;
  std::uint64_t circuit_evaluations = 0;
  double wall_seconds = 0.0;
};

namespace detail {
inline VqeResult run_vqe_on(const QubitHamiltonian& h, const AnsatzSpec& spec, const AdamConfig& config,
                            const std::vector<double>& initial_theta, std::int32_t method, std::int32_t dtype,
                            int device) {
  CsrHam c(h);
  const std::size_t P = n_parameters(spec, h.n_qubits);
  VqeResult r;
  r.theta.assign(P, 0.0);
  r.trajectory.assign(static_cast<std::size_t>(std::max(config.max_iterations, 0)) + 1, 0.0);
  vqf_vqe_result out{};
  out.theta = r.theta.data();
  out.trajectory = r.trajectory.data();
  out.trajectory_capacity = static_cast<std::uint32_t>(r.trajectory.size());
  const vqf_adam_config a = to_c(config);
  check(vqf_run_vqe_ex(&c.view, static_cast<std::int32_t>(spec.kind), spec.layers, &a,
                       initial_theta.empty() ? nullptr : initial_theta.data(),
                       static_cast<std::uint32_t>(initial_theta.size()), method, device, dtype, &out));
  r.energy = out.energy;
  r.trajectory.resize(out.trajectory_len);
  r.iterations_run = out.iterations_run;
  r.circuit_evaluations = out.circuit_evaluations;
  r.wall_seconds = out.wall_seconds;
  return r;
}
}  // namespace detail

// vqe.hpp:194-254 — the whole optimisation loop runs on the device.
inline VqeResult run_vqe(const QubitHamiltonian& h, const AnsatzSpec& spec, const AdamConfig& config,
                         const std::vector<double>& initial_theta = {}) {
  return detail::run_vqe_on(h, spec, config, initial_theta, VQF_GRAD_PARAMETER_SHIFT, VQF_F64, 0);
}

// Engine extensions beyond the reference signatures: state precision
// (complex128 as the reference, or complex64: energies within 1e-5,
// fixed-iteration runs only), gradient rule and device.
namespace gpu {
enum class Precision : std::int32_t { F64 = VQF_F64, F32 = VQF_F32 };
enum class Gradient : std::int32_t { ParameterShift = VQF_GRAD_PARAMETER_SHIFT, Adjoint = VQF_GRAD_ADJOINT };

inline double energy(const std::vector<double>& theta, const QubitHamiltonian& h, const AnsatzSpec& spec,
                     Precision p, int device = 0) {
  detail::CsrHam c(h);
  double e = 0.0;
  detail::check(vqf_energy_ex(theta.data(), static_cast<std::uint32_t>(theta.size()), &c.view,
                              static_cast<std::int32_t>(spec.kind), spec.layers, device, static_cast<std::int32_t>(p),
                              &e));
  return e;
}

inline std::vector<double> gradient(const std::vector<double>& theta, const QubitHamiltonian& h,
                                    const AnsatzSpec& spec, Gradient method, Precision p, int device = 0) {
  detail::CsrHam c(h);
  std::vector<double> g(theta.size());
  detail::check(vqf_gradient_ex(theta.data(), static_cast<std::uint32_t>(theta.size()), &c.view,
                                static_cast<std::int32_t>(spec.kind), spec.layers, static_cast<std::int32_t>(method),
                                device, static_cast<std::int32_t>(p), g.data()));
  return g;
}

inline VqeResult run_vqe(const QubitHamiltonian& h, const AnsatzSpec& spec, const AdamConfig& config,
                         const std::vector<double>& initial_theta, Gradient method, Precision p, int device = 0) {
  return detail::run_vqe_on(h, spec, config, initial_theta, static_cast<std::int32_t>(method),
                            static_cast<std::int32_t>(p), device);
}
}  // namespace gpu

// ------------------------------------------------------------------ chem
// chem.hpp:473-482 (HF + Jordan-Wigner, host build over the shared core)
inline QubitHamiltonian build_h2_hamiltonian(double bond_angstrom) {
  detail::HamBuffer buf(64, 256);
  detail::check(vqf_build_h2_hamiltonian(bond_angstrom, &buf.out));
  return buf.result(4);
}

// ----------------------------------------------------------------- sweep
inline constexpr std::uint32_t kScalingWarnQubits = 22;    // sweep.hpp:36
inline constexpr std::uint32_t kScalingRefuseQubits = 26;  // sweep.hpp:38

struct SweepConfig {  // sweep.hpp:40-46
  double d_min = 0.1;
  double d_max = 3.0;
  int n_points = 100;
  int workers = 1;  // on the GPU build: worker w -> device w % device_count
  AdamConfig adam{};
};

struct SweepPoint {  // sweep.hpp:48-56
  double bond_angstrom = 0.0;
  double energy_hartree = std::numeric_limits<double>::quiet_NaN();
  std::vector<double> theta_star;
  int iterations = 0;
  double wall_seconds = 0.0;
  bool ok = false;
  std::string error;
};

struct SweepReport {  // sweep.hpp:58-64
  SweepConfig config;
  std::vector<SweepPoint> points;
  std::vector<double> per_worker_seconds;
  double total_wall_seconds = 0.0;
  bool all_ok = true;
};

inline std::vector<double> bond_grid(double d_min, double d_max, int n_points) {
  std::vector<double> g(static_cast<std::size_t>(std::max(n_points, 0)));
  detail::check(vqf_bond_grid(d_min, d_max, n_points, g.data()));
  return g;
}

inline std::vector<std::pair<std::size_t, std::size_t>> split_chunks(std::size_t n_items, std::size_t n_chunks) {
  std::vector<std::uint64_t> be(2 * std::max<std::size_t>(n_chunks, 1));
  detail::check(vqf_split_chunks(n_items, n_chunks, be.data()));
  std::vector<std::pair<std::size_t, std::size_t>> out;
  for (std::size_t c = 0; c < n_chunks; ++c) out.emplace_back(be[2 * c], be[2 * c + 1]);
  return out;
}

inline int effective_workers(int requested) {
  std::int32_t out = 0;
  detail::check(vqf_effective_workers(requested, &out));
  return out;
}

// sweep.hpp:128-178 — HF + JW + VQE of every bond in one fused launch per worker.
inline SweepReport run_sweep(const SweepConfig& config) {
  if (config.workers < 1) throw std::invalid_argument("workers must be >= 1");
  const std::size_t n = static_cast<std::size_t>(std::max(config.n_points, 1));
  std::vector<double> bond(n), e(n), th(n), wall(n), per_worker(static_cast<std::size_t>(config.workers));
  std::vector<std::int32_t> iters(n), ok(n);
  constexpr std::size_t kStride = 256;
  std::vector<char> errors(n * kStride, '\0');
  vqf_sweep_config c{config.d_min, config.d_max, config.n_points, config.workers, detail::to_c(config.adam),
                     nullptr, 0, 0, 1};
  vqf_sweep_report rep{bond.data(), e.data(), th.data(), iters.data(), wall.data(), ok.data(), errors.data(),
                       kStride, nullptr, per_worker.data(), 0.0, 0, 0.0, 0, 0};
  detail::check(vqf_run_sweep(&c, &rep));
  SweepReport out;
  out.config = config;
  out.per_worker_seconds = per_worker;
  out.total_wall_seconds = rep.total_wall_seconds;
  out.all_ok = rep.all_ok != 0;
  for (std::size_t i = 0; i < static_cast<std::size_t>(config.n_points); ++i) {
    SweepPoint p;
    p.bond_angstrom = bond[i];
    p.energy_hartree = e[i];
    if (ok[i]) p.theta_star = {th[i]};
    p.iterations = iters[i];
    p.wall_seconds = wall[i];
    p.ok = ok[i] != 0;
    p.error = std::string(errors.data() + i * kStride);
    out.points.push_back(std::move(p));
  }
  return out;
}

// sweep.hpp:181-202 (host arithmetic)
inline double measured_speedup(double t_serial, double t_parallel) {
  if (!(t_serial > 0.0) || !(t_parallel > 0.0)) throw std::invalid_argument("speedup needs positive timings");
  return t_serial / t_parallel;
}
inline double parallel_efficiency(double t_serial, double t_parallel, int workers) {
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  return measured_speedup(t_serial, t_parallel) / workers;
}
inline double amdahl_speedup(double serial_fraction, int workers) {
  if (!(serial_fraction >= 0.0 && serial_fraction <= 1.0))
    throw std::invalid_argument("serial fraction must lie in [0, 1]");
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  return 1.0 / (serial_fraction + (1.0 - serial_fraction) / workers);
}

inline QubitHamiltonian build_tfim(std::uint32_t n_qubits, double coupling, double field) {  // sweep.hpp:209
  detail::HamBuffer buf(2 * n_qubits + 1, 4 * n_qubits + 1);
  detail::check(vqf_build_tfim(n_qubits, coupling, field, &buf.out));
  return buf.result(n_qubits);
}

inline QubitHamiltonian build_z_sum(std::uint32_t n_qubits) {  // sweep.hpp:227
  detail::HamBuffer buf(n_qubits + 1, n_qubits + 1);
  detail::check(vqf_build_z_sum(n_qubits, &buf.out));
  return buf.result(n_qubits);
}

struct ScalingConfig {  // sweep.hpp:237-249
  std::vector<std::uint32_t> qubits{4, 8, 12, 14, 16, 18, 20};
  std::uint32_t layers = 2;
  int iterations = 5;
  double learning_rate = 0.05;
  double coupling = 1.0;
  double field = 1.0;
  bool z_sum_mode = false;
  double theta_init = 0.1;
  bool force = false;
  bool adjoint = false;  // extension: adjoint gradients instead of parameter shift
  int device = 0;
  bool fp32 = false;     // extension: complex64 states (fixed-iteration runs)
};

struct ScalingRecord {  // sweep.hpp:251-257
  std::uint32_t n_qubits = 0;
  std::uint64_t state_bytes = 0;
  double runtime_seconds = 0.0;
  double final_energy = 0.0;
  int iterations_run = 0;
};

// sweep.hpp:265-307
inline std::vector<ScalingRecord> run_scaling_study(const ScalingConfig& config) {
  vqf_scaling_config c{config.qubits.data(), static_cast<std::uint32_t>(config.qubits.size()), config.layers,
                       config.iterations, config.learning_rate, config.coupling, config.field,
                       config.z_sum_mode ? 1 : 0, config.theta_init, config.force ? 1 : 0,
                       config.adjoint ? VQF_GRAD_ADJOINT : VQF_GRAD_PARAMETER_SHIFT, config.device,
                       config.fp32 ? VQF_F32 : VQF_F64};
  std::vector<vqf_scaling_record> recs(config.qubits.size());
  detail::check(vqf_run_scaling_study(&c, recs.data()));
  std::vector<ScalingRecord> out;
  for (const auto& r : recs)
    out.push_back(ScalingRecord{r.n_qubits, r.state_bytes, r.runtime_seconds, r.final_energy, r.iterations_run});
  return out;
}

}  // namespace vqeforge
