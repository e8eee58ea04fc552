// Host-side half of the C ABI: runtime queries, the pure host functions of
// the reference hot path (sweep.hpp bond_grid/split_chunks/effective_workers,
// vqe.hpp adam_step, pauli.hpp canonicalize, sweep.hpp TFIM/Z-sum builders)
// and Hamiltonian compilation into flip-grouped mask tables.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "pauli_host.h"

namespace vqf {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const char* msg) { g_last_error = msg; }

std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}

uint64_t qubit_bit(uint32_t n, uint32_t q) { return uint64_t{1} << (n - 1 - q); }

CompiledHam compile_hamiltonian(const vqf_hamiltonian* h) {
  if (h == nullptr) throw_invalid("null hamiltonian");
  if (h->n_qubits == 0 || h->n_qubits > 63) throw_invalid("hamiltonian: unsupported register size");
  CompiledHam c;
  c.n_qubits = h->n_qubits;
  std::vector<MaskTerm> raw(h->n_terms);
  for (uint32_t t = 0; t < h->n_terms; ++t) {
    MaskTerm m{0, 0, 0.0, 0.0};
    unsigned n_y = 0;
    for (uint32_t k = h->offsets[t]; k < h->offsets[t + 1]; ++k) {
      const uint32_t q = h->qubits[k];
      if (q >= h->n_qubits) throw_invalid("PauliTerm index exceeds register size");
      const uint64_t bit = qubit_bit(h->n_qubits, q);
      const uint8_t a = h->axes[k];
      if (a == VQF_AXIS_X || a == VQF_AXIS_Y) m.flip |= bit;
      if (a == VQF_AXIS_Y || a == VQF_AXIS_Z) m.yz |= bit;
      if (a == VQF_AXIS_Y) ++n_y;
    }
    // y_phase_base (pauli.hpp:242-249) times the coefficient, as the
    // reference's `t.coefficient * base` (statevector.hpp:242).
    double br = 1, bi = 0;
    switch (n_y % 4) {
      case 1: br = 0; bi = -1; break;
      case 2: br = -1; bi = 0; break;
      case 3: br = 0; bi = 1; break;
      default: break;
    }
    const double cr = h->coeffs[2 * t], ci = h->coeffs[2 * t + 1];
    m.cb_re = cr * br - ci * bi;
    m.cb_im = cr * bi + ci * br;
    raw[t] = m;
  }
  // Group by flip in order of first appearance, diagonal group first.
  c.group_flip.push_back(0);
  for (const auto& m : raw)
    if (m.flip != 0 && std::find(c.group_flip.begin(), c.group_flip.end(), m.flip) == c.group_flip.end())
      c.group_flip.push_back(m.flip);
  c.group_offset.push_back(0);
  for (uint64_t f : c.group_flip) {
    for (const auto& m : raw)
      if (m.flip == f) c.terms.push_back(m);
    c.group_offset.push_back(static_cast<uint32_t>(c.terms.size()));
  }
  return c;
}

}  // namespace vqf

using namespace vqf;

extern "C" {

const char* vqf_version(void) { return "vqeforge-b200 0.1.0 (sm_100a)"; }

const char* vqf_last_error(void) { return g_last_error.c_str(); }

int vqf_device_count(int32_t* out) {
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
    *out = n;
  });
}

int vqf_init(int32_t device) {
  return guarded([&] {
    VQF_CUDA(cudaSetDevice(device));
    VQF_CUDA(cudaFree(nullptr));  // forces context creation
  });
}

uint64_t vqf_kernel_launches(void) { return launch_counter().load(); }

uint64_t vqf_memory_estimate(uint32_t n_qubits) { return (uint64_t{1} << n_qubits) * 16u; }

uint32_t vqf_n_parameters(int32_t kind, uint32_t layers, uint32_t n_qubits) {
  switch (kind) {
    case VQF_ANSATZ_H2_DOUBLE_EXCITATION: return 1;
    case VQF_ANSATZ_HARDWARE_EFFICIENT: return layers * n_qubits;
    default: return 0;
  }
}

int vqf_bond_grid(double d_min, double d_max, int32_t n_points, double* out) {
  return guarded([&] {
    if (n_points < 1) throw_invalid("grid needs >= 1 point");
    if (d_max < d_min) throw_invalid("d_max < d_min");
    host::bond_grid(d_min, d_max, n_points, out);
  });
}

int vqf_split_chunks(uint64_t n_items, uint64_t n_chunks, uint64_t* begin_end) {
  return guarded([&] {
    if (n_chunks == 0) throw_invalid("need >= 1 chunk");
    host::split_chunks(n_items, n_chunks, begin_end);
  });
}

int vqf_effective_workers(int32_t requested, int32_t* out) {
  return guarded([&] {
    if (requested < 1) throw_invalid("workers must be >= 1");
    const char* env = std::getenv("VQE_FORGE_THREADS");
    int32_t r = requested;
    if (env != nullptr && *env != '\0') {
      char* end = nullptr;
      const long cap = std::strtol(env, &end, 10);
      if (!(end == env || *end != '\0' || cap < 1)) r = static_cast<int32_t>(std::min<long>(requested, cap));
    }
    *out = r;
  });
}

int vqf_adam_step(const double* m, const double* v, int64_t step, const double* grad, const double* theta,
                  uint32_t n, const vqf_adam_config* cfg, double* theta_out, double* m_out, double* v_out,
                  int64_t* step_out) {
  return guarded([&] {
    if (cfg == nullptr) throw_invalid("adam_step: null config");
    host::adam_step(m, v, step, grad, theta, n, *cfg, theta_out, m_out, v_out, step_out);
  });
}

int vqf_canonicalize(const vqf_hamiltonian* h, vqf_hamiltonian_out* out) {
  return guarded([&] {
    auto terms = host::terms_from_csr(h, /*validate=*/true);
    host::canonicalize(terms);
    host::terms_to_csr(terms, out);
  });
}

int vqf_build_tfim(uint32_t n, double coupling, double field, vqf_hamiltonian_out* out) {
  return guarded([&] { host::terms_to_csr(host::build_tfim(n, coupling, field), out); });
}

int vqf_build_z_sum(uint32_t n, vqf_hamiltonian_out* out) {
  return guarded([&] { host::terms_to_csr(host::build_z_sum(n), out); });
}

}  // extern "C"
