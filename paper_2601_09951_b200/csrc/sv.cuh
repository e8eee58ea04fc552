// Device-resident state-vector batches and the HBM-bound kernels that act
// on them (statevector.hpp:33-249 semantics, MSB-first qubit order).
#pragma once

#include <cstdint>
#include <vector>

#include "common.cuh"

struct vqf_statevector {
  uint32_t n_qubits = 0;
  uint32_t batch = 1;
  int32_t dtype = VQF_F64;
  int32_t device = 0;
  void* amps = nullptr;  // batch * 2^n complex (double2 or float2), entry-major
  cudaStream_t stream = nullptr;      // active stream (own or caller's)
  cudaStream_t own_stream = nullptr;
  // reduction scratch: per (entry, group, block) complex partials
  double* partials = nullptr;
  size_t partial_cap = 0;  // in doubles
  double* host_out = nullptr;  // pinned, >= 2 * batch doubles
  double* dev_out = nullptr;   // device, >= 2 * batch doubles
  size_t out_cap = 0;          // doubles in host_out / dev_out
  void* terms_dev = nullptr;   // compiled Hamiltonian terms (MaskTerm)
  size_t terms_cap = 0;        // bytes
  double* cs_dev = nullptr;    // per-entry (cos, sin) scratch for batched gates
  size_t cs_cap = 0;           // in doubles
  uint64_t dim() const { return uint64_t{1} << n_qubits; }
  size_t amp_bytes() const { return dtype == VQF_F64 ? 16 : 8; }
};

namespace vqf {

// Per-entry gate angle source for batched circuits.  When `cs` is non-null,
// entry b uses (cs[2b], cs[2b+1]) = (cos(angle/2), sin(angle/2)); otherwise
// every entry uses (c, s).
struct GateArgs {
  int32_t kind;
  uint32_t n_wires;
  uint32_t wires[4];
  double c, s;
  const double* cs;
};

void sv_check_gate(const vqf_statevector* sv, const vqf_gate& g);
void sv_apply(vqf_statevector* sv, const GateArgs& g);
void sv_reset(vqf_statevector* sv, uint64_t basis_index);
// Expectation of a compiled Hamiltonian for every entry, returned as
// interleaved (re, im) in `out` (host, 2*batch).  Synchronises the stream.
void sv_expectation(vqf_statevector* sv, const CompiledHam& h, double* out);
// Same, but leaves the per-entry complex totals on the device in `dev_out`
// (2*batch doubles) without synchronising.
void sv_expectation_async(vqf_statevector* sv, const CompiledHam& h, double* dev_out);
void sv_norms(vqf_statevector* sv, double* out);
void sv_ensure_cs(vqf_statevector* sv, size_t n_doubles);
// Keeps freed stream-ordered allocations of `device` cached in its pool.
void retain_pool(int device);

}  // namespace vqf
