// Launch interface of the register-resident batched VQE engine (n <= 5).
#pragma once

#include <cstdint>

#include "chem.cuh"
#include "common.cuh"

namespace vqf {

constexpr int kSmallMaxN = 5;
constexpr int kSmallMaxD = 1 << kSmallMaxN;
constexpr int kSmallMaxP = 64;

// Per-problem status written by the kernel (0 = ok).
enum : int32_t {
  kStatusOk = 0,
  kStatusConverged = 1,  // internal only
  kStatusImag = 2,       // expectation has imaginary residue (statevector.hpp:245)
  kStatusNonFinite = 3,  // non-finite energy at iteration (vqe.hpp:217)
  kStatusScf = 4,        // NonConvergence (chem.hpp:46-52)
  kStatusHermitian = 5,  // non-Hermitian Pauli coefficient (pauli.hpp:205-214)
  kStatusBond = 6,       // BondLengthOutOfRange (host-side check, chem.hpp:38-44)
  kStatusAbort = 7       // block engine: grid barrier watchdog fired
};

struct SmallParams {
  int32_t n_qubits, ansatz_kind, layers, n_params;
  int32_t max_iterations, has_tol;
  double tol, lr, beta1, beta2, eps;
  const double* bc1;  // max_iterations entries: 1 - beta1^t
  const double* bc2;
  // generic mode: grouped-by-problem mask terms
  const MaskTerm* terms;
  const uint32_t* term_off;  // batch + 1
  // PES mode: bonds[] (staged), or, when grid_n > 0, bond grid_first + b of
  // bond_grid(grid_min, grid_max, grid_n) computed on device (sweep.hpp:68-85
  // arithmetic, bitwise) with the range check done there too (no H2D copy)
  const double* bonds;
  double grid_min, grid_max;
  int32_t grid_n, grid_first;
  chem::ChemConsts chem;
  const chem::JwTable* jw;
  const double* init_theta;  // batch * P, or null (theta0 = 0)
  // outputs
  double* energy;
  double* theta_out;  // batch * P
  double* traj;       // batch * traj_stride
  int32_t traj_stride;
  int32_t* iters;
  int32_t* converged;
  int32_t* status;  // in: 0 or kStatusBond (staged PES); out: status
  double* err_val;
  int32_t* err_iter;
  double* err_theta;  // batch * P
  // optional PES diagnostics (may be null)
  int32_t* ham_keys;    // batch * 16
  double* ham_coeffs;   // batch * 16
  int32_t* ham_count;   // batch
  double* hf_out;       // batch * 4
  // optional device timing (may be null): %globaltimer at CTA entry and at
  // the CTA's result write, 2 per problem (ns); replaces host-side events
  unsigned long long* clk;
};

size_t small_smem_bytes();
int small_amps_per_lane(int n_qubits, int n_params);
void launch_vqe_small(const SmallParams& p, uint32_t batch, bool pes, cudaStream_t stream);

}  // namespace vqf
