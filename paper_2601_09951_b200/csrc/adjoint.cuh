// Adjoint-differentiation plan for the HBM engine (see adjoint.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "sv.cuh"

namespace vqf {

// One ansatz gate for the backward sweep; param = -1 when not parameterised.
struct AdjGate {
  int32_t kind;
  uint32_t wires[4];
  int32_t param;
};

// Device view of the compiled Hamiltonian for k_apply_ham: the diagonal
// group split by tile (low-bit / high-bit / mixed terms) and the
// off-diagonal flip groups.
struct HamDevC {
  const MaskTerm* lo_t;
  const MaskTerm* hi_t;
  const MaskTerm* mx_t;
  uint32_t n_lo, n_hi, n_mx;
  const uint64_t* flips;
  const uint32_t* group_off;
  const uint32_t* group_hi;  // per group: its first group_hi terms have Z/Y only at or above the tile bits
  const MaskTerm* terms;
  uint32_t n_groups;
};

struct AdjointPlan {
  vqf_statevector* psi = nullptr;  // forward state (consumed by the sweep)
  vqf_statevector* lam = nullptr;  // H psi, swept backwards
  uint32_t P = 0, tile_bits = 0, nb = 0, nb_ham = 0;
  void* dev = nullptr;
  double* hout = nullptr;           // thread-local pinned block (not owned)
  cudaStream_t free_stream = nullptr;  // the state's own stream: dev is freed there
  HamDevC hd{};
  double* gpart = nullptr;
  double* epart = nullptr;
  double* dout = nullptr;

  AdjointPlan() = default;
  AdjointPlan(const AdjointPlan&) = delete;
  ~AdjointPlan();
  void init(vqf_statevector* psi, vqf_statevector* lam, const CompiledHam& h, uint32_t n_params);
  // Whether init() can table this Hamiltonian on an n-qubit register (at most
  // 64 diagonal terms straddling the tile boundary, 256 flip groups, 1024
  // off-diagonal terms).  Callers run the parameter-shift engine otherwise,
  // so method = adjoint never fails on a large Hamiltonian.
  static bool supports(const CompiledHam& h, uint32_t n_qubits);
  // Gradient of <psi(theta)|H|psi(theta)> for the prepared forward state in
  // psi (destroyed); e_out = {Re, Im} of the energy, grad_out[P].
  void run(const std::vector<AdjGate>& prog, const std::vector<double>& theta, double* e_out, double* grad_out);
};

}  // namespace vqf
