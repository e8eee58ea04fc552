// Launch interface of the shared-memory VQE engine (mid widths, one launch
// per run_vqe).  See vqe_block.cu.
#pragma once

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace vqf {

constexpr int kBlockMinN = 4;
constexpr int kBlockMaxP = 256;
constexpr int kBlockMaxR = 4;  // register bits per rotation pass

// Largest register whose state fits one CTA's shared memory; one qubit
// more runs with the state in an L2-resident global buffer per CTA
// (everything else on chip).  Measured (run_scaling_study, 5 iterations):
// n = 14 1.42 ms vs 2.38 / 2.91 ms on the HBM engine (adjoint / shift); at
// n = 15-16 one CTA per circuit is bound by its SM's L2 bandwidth
// (2.8 / 5.7 ms, no better than the HBM engine), so the engine stops at 14.
inline int block_smem_max_n(int32_t dtype) { return dtype == VQF_F32 ? 14 : 13; }
inline int block_max_n(int32_t dtype) { return dtype == VQF_F32 ? 15 : 14; }

// One shared-memory pass: up to R commuting RY rotations applied in
// registers.  Amplitude member m of a thread's coset sits at physical index
// base ^ (XOR of vec[j] over the set bits j of m); base has zeros at the
// pivot bits (ascending).  Logical bit of rotation j at base =
// parity(row[j] & base) ^ cbit_j (the frame, see vqe_block.cu).
struct BlockPass {
  uint32_t vec[kBlockMaxR];
  uint32_t svec[kBlockMaxR];  // block_slot(vec): the slot map is linear over GF(2)
  uint32_t row[kBlockMaxR];
  uint32_t piv[kBlockMaxR];
  int32_t param[kBlockMaxR];
  uint32_t cbits;
  int32_t r;
};

// Shared-memory slot of physical index p (16-byte amplitudes: one 128-byte
// wavefront holds 8 slots; XOR-ing bits 3..5 into bits 0..2 spreads strided
// patterns -- a pivot or pair bit among bits 0..2 -- over all 8).  Linear
// over GF(2): slot(p ^ q) = slot(p) ^ slot(q).
__host__ __device__ inline uint32_t block_slot(uint32_t p) { return p ^ ((p >> 3) & 7u); }

// Expectation term in the final frame: flip' = M^-1 flip, yz' = M^T yz,
// cb' = cb * (-1)^popc(yz & c).
struct BlockTerm {
  uint32_t yz;
  uint32_t pad;
  double cb_re, cb_im;
};

// Real form of a Hermitian term (every coefficient real, the usual case):
// with v = conj(psi_i) psi_{i ^ flip}, a pair contributes
// a (-1)^popc(yz' & i) w, w = 2 Re v (even Y count) or 2 Im v (odd), and the
// diagonal group is one real operator value per amplitude.
struct BlockRTerm {
  uint32_t yz;
  uint32_t odd;
  double a;
};

// Dynamic shared memory of one CTA (byte offsets), shared by host and kernel.
// `slots` states and angle tables: one per team (see Team in vqe_block.cu).
struct BlockSmem {
  uint32_t Pp, psi, theta, mom, vel, cs, e_all, otab, rterms, gflip, goff, total;
  __host__ __device__ BlockSmem(uint32_t n, uint32_t amp, uint32_t P, uint32_t obytes, uint32_t T, uint32_t G,
                                uint32_t slots = 1) {
    Pp = (P + 1u) & ~1u;
    uint32_t o = 0;
    psi = o;
    o += slots * (amp << n);
    theta = o;
    o += 8u * Pp;
    mom = o;
    o += 8u * Pp;
    vel = o;
    o += 8u * Pp;
    cs = o;
    o += (slots > 1 ? 3u : 1u) * 16u * Pp;  // teams: (theta, +pi/2, -pi/2) per parameter
    e_all = o;
    o += 16u * (2u * Pp + 2u);
    otab = o;
    o += obytes << n;
    rterms = o;
    o += 16u * T;
    gflip = o;
    o += 4u * G;
    goff = o;
    o += 4u * (G + 1u);
    total = (o + 15u) & ~15u;
  }
};

// Host-compiled ansatz + Hamiltonian for the engine (frame tracking of the
// permutation gates, rotation passes, transformed term tables).
struct BlockProgram {
  uint32_t n = 0, R = 0, init_index = 0;
  std::vector<BlockPass> passes;
  std::vector<uint32_t> group_flip;  // physical flip per group (group 0 diagonal)
  std::vector<uint32_t> group_off;   // G + 1
  std::vector<BlockTerm> terms;
  bool herm = false;                 // every term has a real form (rterms valid)
  std::vector<BlockRTerm> rterms;    // same order as terms
  uint32_t obytes = 0;               // diagonal operator table: 8 (double), 4 (float) or 0 (none)
  // launch shape: teams of `lanes` threads in one CTA (teams = true), or a
  // cooperative grid of CTAs of `threads`, one circuit per CTA
  bool teams = false;
  bool gmem = false;  // state in a global (L2-resident) buffer per CTA
  uint32_t lanes = 0, threads = 0, slots = 1;
};

// HEA / H2 ansatz of vqe.hpp:65-96 compiled for the engine; throws
// invalid_argument for kinds the engine does not hold (DoubleExcitation is
// not a rotation of one wire).
BlockProgram compile_block_program(int32_t kind, uint32_t layers, uint32_t n, const CompiledHam& h, int32_t dtype);

struct BlockParams {
  int32_t n, P, NC, max_iterations, has_tol, dtype;
  double tol, lr, beta1, beta2, eps;
  const double* bc;  // 2 * max(T, 1): (1 - beta1^t, 1 - beta2^t), t = 1..T
  const BlockPass* passes;
  int32_t n_passes;
  uint32_t init_index;
  const uint32_t* group_flip;
  const uint32_t* group_off;
  int32_t n_groups;
  const BlockTerm* terms;
  int32_t herm, n_terms;
  uint32_t obytes;
  int32_t team_lanes;
  void* gstate;  // gmem programs: gridDim.x states of 2^n amplitudes (CTA b uses state b)
  const BlockRTerm* rterms;
  const double* init_theta;  // P or null
  // grid exchange
  double2* energies;  // 2 * NC (by iteration parity)
  unsigned* barrier;  // [0] arrivals, [1] abort, [2] exits; zero at launch, reset by the last CTA out
  // outputs
  double* energy;
  double* theta_out;  // P
  double* traj;       // max_iterations + 1
  int32_t* iters;
  int32_t* converged;
  int32_t* status;
  double* err_val;
  int32_t* err_iter;
  double* err_theta;  // P
  unsigned long long* clk;  // 2: %globaltimer at entry / result
};

// Launch arguments: small problems carry every input inside the kernel
// parameter block (no host-to-device copy before the launch); the input
// pointers of `p` then hold byte offsets into `blob` (inl = 1).
// Two parameter-block sizes: the launch call's cost grows with it (8 KB
// costs ~6 us more than 1 KB on the host), so small inputs take the 1 KB one.
constexpr int kBlockInline = 8192;
constexpr int kBlockInlineSmall = 1024;
template <int NB>
struct __align__(16) BlockArgsN {
  BlockParams p;
  int32_t inl;
  alignas(16) unsigned char blob[NB];
};
using BlockArgs = BlockArgsN<kBlockInline>;

// Grid size of the cooperative launch for this program (<= NC).
int block_grid(const BlockProgram& prog, int32_t dtype, int NC, int device);
size_t block_smem_bytes(const BlockProgram& prog, int32_t dtype, int32_t P);
// `used`: bytes of a.blob holding inputs (a.inl = 1).
void launch_vqe_block(const BlockArgs& a, size_t used, const BlockProgram& prog, int grid, cudaStream_t stream);

}  // namespace vqf
