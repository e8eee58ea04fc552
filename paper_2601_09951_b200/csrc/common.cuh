// Shared internals of libvqf_b200.so: error plumbing for the C ABI, CUDA
// checks, complex helpers and the compiled (mask-form) Hamiltonian.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "vqf_b200.h"

namespace vqf {

// ------------------------------------------------------------------ errors
// The C ABI returns an int class and keeps the message thread-locally
// (vqf_last_error).  Internally we throw these and translate at the edge.
struct Error : std::exception {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(VQF_INVALID_ARGUMENT, m); }
[[noreturn]] inline void throw_runtime(const std::string& m) { throw Error(VQF_RUNTIME_ERROR, m); }

void set_last_error(const char* msg);
std::atomic<uint64_t>& launch_counter();

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return VQF_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return VQF_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return VQF_RUNTIME_ERROR;
  }
}

#define VQF_CUDA(call)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (call);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      throw ::vqf::Error(VQF_CUDA_ERROR, std::string("CUDA: ") + cudaGetErrorString(_e) +    \
                                             " at " __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

#define VQF_LAUNCHED() ::vqf::launch_counter().fetch_add(1, std::memory_order_relaxed)

// Formats a double like std::to_string (printf "%f"), which is what the
// reference uses inside its exception messages (statevector.hpp:245,
// vqe.hpp:218-219, chem.hpp:40-51).
inline std::string fstr(double x) { return std::to_string(x); }

// ----------------------------------------------------------------- complex
struct cd {
  double re, im;
};

__host__ __device__ inline double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// --------------------------------------------------------- Hamiltonian ABI
// Mask form of one Pauli term (pauli.hpp:217-249): flip = X|Y bits,
// yz = Y|Z bits (MSB-first), cb = coefficient * (-i)^{n_y}.
struct MaskTerm {
  uint64_t flip;
  uint64_t yz;
  double cb_re, cb_im;
};

// A Hamiltonian grouped by flip mask: all terms of a group read the same
// amplitude pairs, so one pass over the state serves the whole group.
// group 0 is always the diagonal group (flip == 0), possibly empty.
struct CompiledHam {
  uint32_t n_qubits = 0;
  std::vector<uint64_t> group_flip;      // G
  std::vector<uint32_t> group_offset;    // G + 1 into terms
  std::vector<MaskTerm> terms;           // grouped, original order inside a group
};

// Validates the CSR (QubitHamiltonian ctor, pauli.hpp:120-127, minus the
// PauliTerm checks the reference only runs at construction) and compiles it.
CompiledHam compile_hamiltonian(const vqf_hamiltonian* h);

uint64_t qubit_bit(uint32_t n, uint32_t q);

}  // namespace vqf
