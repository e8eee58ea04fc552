// Register-resident batched VQE engine for small registers (n <= 5) and the
// fused H2 potential-energy-surface kernel.
//
// The reference evaluates each bond serially: per Adam iteration one energy
// plus 2P parameter-shifted energies, each a fresh heap-allocated
// StateVector (vqe.hpp:99-127, :226-243).  Here ONE WARP owns one problem
// (one bond) for its whole optimisation, with no block barriers:
//   * every circuit of an iteration (base + 2P shifts) is simulated at once
//     in the warp: a circuit occupies L lanes x A amplitudes per lane
//     (index i = a*L + lane), gates on lane bits are warp shuffles, gates on
//     slot bits are register permutations (H2: 3 circuits x 8 lanes x 2);
//   * each (cos, sin) is computed once per parameter and shift;
//   * expectation is a per-amplitude table lookup: the Hamiltonian is folded
//     once into per-flip-group tables O_g(i) = sum_t cb_t (-1)^popc(i&yz_t),
//     <psi|H|psi> = sum_i sum_g O_g(i) conj(psi_i) psi_{i^f_g}, reduced in a
//     fixed order (slots, then an xor butterfly) so results do not depend on
//     where the problem runs;
//   * Adam runs in the lane that owns the parameter, with host-computed
//     bias-correction tables (bitwise the reference's std::pow,
//     vqe.hpp:161-162);
//   * in PES mode the CTA first builds its bond's Hamiltonian from scratch
//     (STO-3G integrals -> RHF -> Jordan-Wigner, chem.cuh) with 4 warps, then
//     warp 0 runs the optimisation: a whole PES is ONE launch.
// The path is latency bound (a bond's state is 256 B): nothing touches HBM
// beyond the outputs.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

#include "chem.cuh"
#include "fastmath.cuh"
#include "vqe_small.cuh"

namespace vqf {

namespace {

constexpr double kShift = 1.5707963267948966;  // std::numbers::pi / 2 (vqe.hpp:115)
#ifndef VQF_PES_THREADS
#define VQF_PES_THREADS 288
#endif
// Chemistry prologue width; warps 1.. exit before the loop.  288 threads:
// the 273 distinct Boys evaluations run in one round, and the register cap
// stays at 224 for the optimisation loop (512 threads cap it at 128 and the
// loop then spills its constants through uniform registers).
constexpr int kPesThreads = VQF_PES_THREADS;
constexpr int kMaxGates = 2 * kSmallMaxP + 8;

enum : int { G_X = 0, G_RY = 1, G_CNOT = 2, G_DE = 3 };

struct PGate {
  int kind;
  int param;  // -1 if not parameterised
  int m0;     // RY/X: bit mask; CNOT: control mask; DE: sel mask
  int m1;     // CNOT: target mask; DE: occ (1100) mask
};

struct Shared {
  // problem description
  int n_groups, n_gates, n_terms;
  int flip[kSmallMaxD];
  double2 tab[kSmallMaxD * kSmallMaxD];  // [group][index]
  PGate prog[kMaxGates];
  MaskTerm terms[256];
  // per-iteration exchange
  double theta[kSmallMaxP];
  double2 cs[kSmallMaxP][3];  // (cos, sin) of 0.5 * (theta, theta + pi/2, theta - pi/2)
  double init_state[16];      // PES whole-state lanes: basis_state(4, {1,1,0,0})
  double2 energy[2 * kSmallMaxP + 1];
  double grad[kSmallMaxP];
  int stop;
  // PES prologue scratch
  chem::PairFactor pf[36];
  int pf_rep[21];                     // a pair-factor index per distinct pair factor
  double eri_pref[231], eri_boys[231];  // per unordered pair of distinct pair factors
  double nuc_boys[42];                // per distinct pair factor x nucleus
  double prim[1296];
  double prim1[144];
  chem::AoInts ints;
  chem::HfOut hf;
  double C[2][2];
  double mo[16];
  double integ[20];  // hmo (4) then physicist eri_mo (16)
  double kre[256], kim[256];
  int kflag[256];
  int wlive[8], wbad[8];  // per-warp survivor counts / first non-Hermitian key
  unsigned char cpart[chem::kNumContrib];  // Jordan-Wigner contribution part (0 re, 1 im)
};

#ifdef VQF_STAGE_CLOCKS
__device__ __forceinline__ unsigned __mysmid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#endif

__device__ __forceinline__ double2 shfl_xor2(double2 v, int m, int width) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m, width);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, m, width);
  return v;
}
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  v.x = __shfl_sync(0xffffffffu, v.x, src);
  v.y = __shfl_sync(0xffffffffu, v.y, src);
  return v;
}

// a' = c a - s b and b' = s a + c b as the reference writes them (complex *
// real, then subtract / add): statevector.hpp:160-163, :195-196.
__device__ __forceinline__ double2 rot_lo(double c, double s, double2 a, double2 b) {
  return make_double2(c * a.x - s * b.x, c * a.y - s * b.y);
}
__device__ __forceinline__ double2 rot_hi(double c, double s, double2 a, double2 b) {
  return make_double2(s * a.x + c * b.x, s * a.y + c * b.y);
}

// out[a] = amplitude at index (a*L + lane) ^ m, m split into lane / slot
// bits.  m is warp-uniform, so every branch is uniform.
template <int A>
__device__ __forceinline__ void fetch_partner(const double2 (&amp)[A], double2 (&out)[A], int m, int L, int lgL) {
  const int ml = m & (L - 1), ms = m >> lgL;
#pragma unroll
  for (int a = 0; a < A; ++a) out[a] = ml ? shfl_xor2(amp[a], ml, L) : amp[a];
#pragma unroll
  for (int k = 1; k < A; k <<= 1) {
    if (ms & k) {
#pragma unroll
      for (int a = 0; a < A; ++a) {
        if (!(a & k)) {
          const double2 t = out[a];
          out[a] = out[a | k];
          out[a | k] = t;
        }
      }
    }
  }
}

// Runs the circuit program for circuit c (0 = base, 2k+1 = +pi/2 on k,
// 2k+2 = -pi/2 on k) on this lane's A amplitudes.  H2 = true compiles the
// H2 ansatz (vqe.hpp:72-80) as constants: |1100> = 12, DoubleExcitation on
// wires 0..3 (sel 1111).
template <int A, bool H2>
__device__ __forceinline__ void run_circuit(const Shared& sh, double2 (&amp)[A], int c, int lane, int L, int lgL,
                                            int basis) {
#pragma unroll
  for (int a = 0; a < A; ++a) amp[a] = make_double2((a * L + lane) == basis ? 1.0 : 0.0, 0.0);
  if (H2) {
    double2 part[A];
    fetch_partner<A>(amp, part, 15, L, lgL);
    const double2 t = sh.cs[0][c == 1 ? 1 : c == 2 ? 2 : 0];
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int pat = (a * L + lane) & 15;
      if (pat == 12) amp[a] = rot_lo(t.x, t.y, amp[a], part[a]);
      else if (pat == 3) amp[a] = rot_hi(t.x, t.y, part[a], amp[a]);
    }
    return;
  }
  for (int gi = 0; gi < sh.n_gates; ++gi) {
    const PGate g = sh.prog[gi];
    double2 part[A];
    if (g.kind == G_RY || g.kind == G_X) {
      fetch_partner<A>(amp, part, g.m0, L, lgL);
      if (g.kind == G_X) {
#pragma unroll
        for (int a = 0; a < A; ++a) amp[a] = part[a];
      } else {
        const int j = (c == 2 * g.param + 1) ? 1 : (c == 2 * g.param + 2) ? 2 : 0;
        const double2 t = sh.cs[g.param][j];
#pragma unroll
        for (int a = 0; a < A; ++a) {
          const int i = a * L + lane;
          amp[a] = (i & g.m0) ? rot_hi(t.x, t.y, part[a], amp[a]) : rot_lo(t.x, t.y, amp[a], part[a]);
        }
      }
    } else if (g.kind == G_CNOT) {
      fetch_partner<A>(amp, part, g.m1, L, lgL);
#pragma unroll
      for (int a = 0; a < A; ++a)
        if ((a * L + lane) & g.m0) amp[a] = part[a];
    } else {  // DoubleExcitation: sel = m0, |1100> = m1, |0011> = m0 ^ m1
      fetch_partner<A>(amp, part, g.m0, L, lgL);
      const int j = (c == 2 * g.param + 1) ? 1 : (c == 2 * g.param + 2) ? 2 : 0;
      const double2 t = sh.cs[g.param][j];
#pragma unroll
      for (int a = 0; a < A; ++a) {
        const int pat = (a * L + lane) & g.m0;
        if (pat == g.m1) amp[a] = rot_lo(t.x, t.y, amp[a], part[a]);
        else if (pat == (g.m0 ^ g.m1)) amp[a] = rot_hi(t.x, t.y, part[a], amp[a]);
      }
    }
  }
}

// <psi|H|psi> of this lane's circuit, complete on every lane of the segment.
template <int A>
__device__ __forceinline__ double2 circuit_energy(const Shared& sh, const double2 (&amp)[A], int lane, int L, int lgL,
                                                  int D) {
  double2 acc = make_double2(0.0, 0.0);
  for (int g = 0; g < sh.n_groups; ++g) {
    double2 part[A];
    fetch_partner<A>(amp, part, sh.flip[g], L, lgL);
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const double2 x = amp[a], y = part[a];
      const double vr = x.x * y.x + x.y * y.y, vi = x.x * y.y - x.y * y.x;  // conj(x) * y
      const double2 o = sh.tab[g * D + a * L + lane];
      acc.x += o.x * vr - o.y * vi;
      acc.y += o.x * vi + o.y * vr;
    }
  }
  for (int o = L >> 1; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o, L);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o, L);
  }
  return acc;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Folds the mask terms into per-flip-group amplitude tables (warp 0).
// Groups are numbered in order of first appearance after the diagonal
// group 0: lane t flags term t when no earlier term has its flip, and a
// ballot prefix count gives its group index (no serial scan).
__device__ void build_tables(Shared& sh, int D, int lane) {
  const int T = sh.n_terms;
  int n_new = 0;
  for (int t0 = 0; t0 < T; t0 += 32) {
    const int t = t0 + lane;
    int f = -1;
    bool first = false;
    if (t < T) {
      f = static_cast<int>(sh.terms[t].flip);
      first = f != 0;
      for (int u = 0; u < t && first; ++u) first = static_cast<int>(sh.terms[u].flip) != f;
    }
    const unsigned m = __ballot_sync(0xffffffffu, first);
    if (first) sh.flip[1 + n_new + __popc(m & ((1u << lane) - 1))] = f;
    n_new += __popc(m);
  }
  if (lane == 0) {
    sh.flip[0] = 0;
    sh.n_groups = 1 + n_new;
  }
  __syncwarp();
  const int G = 1 + n_new;
  for (int idx = lane; idx < G * D; idx += 32) {
    const int g = idx / D, i = idx % D;
    const int fg = sh.flip[g];
    double re = 0.0, im = 0.0;
    for (int t = 0; t < T; ++t) {
      const MaskTerm m = sh.terms[t];
      if (static_cast<int>(m.flip) != fg) continue;
      const bool odd = __popcll(static_cast<uint64_t>(i) & m.yz) & 1;
      re += odd ? -m.cb_re : m.cb_re;
      im += odd ? -m.cb_im : m.cb_im;
    }
    sh.tab[g * D + i] = make_double2(re, im);
  }
  __syncwarp();
}

// prepare_ansatz (vqe.hpp:65-96) as a gate program; returns the basis index.
__device__ int build_program(Shared& sh, int kind, int n, int layers) {
  int ng = 0;
  if (kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION) {
    // basis_state(4, {1,1,0,0}) = 12; DoubleExcitation(theta0, 0, 1, 2, 3)
    sh.prog[ng++] = PGate{G_DE, 0, 15, 12};
    sh.n_gates = ng;
    return 12;
  }
  int k = 0;
  for (int layer = 0; layer < layers; ++layer) {
    for (int q = 0; q < n; ++q) sh.prog[ng++] = PGate{G_RY, k++, 1 << (n - 1 - q), 0};
    for (int q = 0; q + 1 < n; ++q) sh.prog[ng++] = PGate{G_CNOT, -1, 1 << (n - 1 - q), 1 << (n - 2 - q)};
  }
  sh.n_gates = ng;
  return 0;
}

// Bond length of problem `prob`: staged, or bond_grid's own arithmetic.
__device__ __forceinline__ double pes_bond(const SmallParams& p, int prob) {
  if (p.grid_n <= 0) return p.bonds[prob];
  const int i = p.grid_first + prob;
  if (p.grid_n == 1) return p.grid_min;
  if (i == p.grid_n - 1) return p.grid_max;
  const double span = p.grid_max - p.grid_min;
  return p.grid_min + span * static_cast<double>(i) / static_cast<double>(p.grid_n - 1);
}

// PES prologue: this CTA's H2 Hamiltonian as mask terms in smem (all
// kPesThreads threads).  Sets sh.stop to kStatusScf / kStatusHermitian.
//   1. 36 pair factors (one exp each) shared by every primitive;
//   2. 1296 ERI + 36 overlap + 36 kinetic + 72 nuclear primitive terms, one
//      per thread-slot;
//   3. contractions summed in the reference's loop order;
//   4. RHF (thread 0), MO transform (16 threads), Jordan-Wigner per string.
__device__ void build_h2_device(Shared& sh, const SmallParams& p, int prob) {
  using namespace chem;
  const ChemConsts& k = p.chem;
  const double d = pes_bond(p, prob) * kAngstromToBohr;
#ifdef VQF_STAGE_CLOCKS
  long long t_start = clock64(), t_pf, t_boys, t_prim, t_sum, t_scf, t_mo, t_jw;
#endif
  // The Jordan-Wigner contribution map is bond-independent: issue its loads
  // now so their latency hides under the integral work.
  const JwTable& jw = *p.jw;
  constexpr int kContribPerThread = (kNumContrib + kPesThreads - 1) / kPesThreads;
  int c_slot[kContribPerThread], c_part[kContribPerThread];
  double c_coef[kContribPerThread];
#pragma unroll
  for (int u = 0; u < kContribPerThread; ++u) {
    const int e = threadIdx.x + u * kPesThreads;
    const bool in = e < kNumContrib;
    c_slot[u] = in ? jw.slot[e] : 0;
    c_part[u] = in ? jw.part[e] : 0;
    c_coef[u] = in ? jw.coef[e] : 0.0;
  }
  for (int idx = threadIdx.x; idx < 36; idx += blockDim.x) {
    const int ij = idx / 9, x = (idx % 9) / 3, y = idx % 3;
    sh.pf[idx] = pair_factor(k, d, ij, idx % 9);
    if (ij == 1 || ((ij == 0 || ij == 3) && x <= y)) sh.pf_rep[pf_uid(ij, x, y)] = idx;
  }
  __syncthreads();
#ifdef VQF_STAGE_CLOCKS
  t_pf = clock64();
#endif
  // The transcendental part of every primitive (Boys function, ERI
  // prefactor) depends on its pair factors only through values that are
  // exactly symmetric under bra <-> ket and under swapping the two
  // primitives of a same-centre pair, so it is evaluated once per unordered
  // pair of the 21 distinct pair factors (231 + 42 nuclear instead of
  // 1296 + 72) - bitwise the values eri_prim / nuclear_prim compute.
  for (int idx = threadIdx.x; idx < 231 + 42; idx += blockDim.x) {
    if (idx < 231) {
      int u = 0;  // decode pf_pair: row u starts at u * 21 - u * (u - 1) / 2
      while (u < 20 && pf_pair(u + 1, u + 1) <= idx) ++u;
      const int v = u + (idx - pf_pair(u, u));
      const PairFactor& a = sh.pf[sh.pf_rep[u]];
      const PairFactor& b = sh.pf[sh.pf_rep[v]];
      sh.eri_pref[idx] = eri_pref(k, a.p, b.p);
      sh.eri_boys[idx] = boys_f0(a.p * b.p / (a.p + b.p) * d2z(a.P, b.P));
    } else {
      const int o = idx - 231, u = o >> 1;
      const PairFactor& f = sh.pf[sh.pf_rep[u]];
      sh.nuc_boys[o] = boys_f0(f.p * d2z(f.P, (o & 1) ? d : 0.0));
    }
  }
  __syncthreads();
#ifdef VQF_STAGE_CLOCKS
  t_boys = clock64();
#endif
  constexpr int kOne = 36 * 4;  // S, T, V(nucleus 0), V(nucleus 1) per (ij, xy)
  for (int idx = threadIdx.x; idx < 1296 + kOne; idx += blockDim.x) {
    if (idx < 1296) {
      const int ijkl = idx / 81, r = idx % 81;
      const int x = r / 27, y = (r / 9) % 3, z = (r / 3) % 3, w = r % 3;
      const int bra = (ijkl >> 2) * 9 + x * 3 + y, ket = (ijkl & 3) * 9 + z * 3 + w;
      const int u = pf_uid(ijkl >> 2, x, y), v = pf_uid(ijkl & 3, z, w);
      const int pi = u <= v ? pf_pair(u, v) : pf_pair(v, u);
      sh.prim[idx] = eri_term_tab(k, sh.pf[bra], sh.pf[ket], sh.eri_pref[pi], sh.eri_boys[pi], x, y, z, w);
    } else {
      const int o = idx - 1296, which = o / 36, e = o % 36;
      const int ij = e / 9, x = (e % 9) / 3, y = e % 3;
      const double nb = which >= 2 ? sh.nuc_boys[2 * pf_uid(ij, x, y) + (which - 2)] : 0.0;
      sh.prim1[o] = one_e_term_tab(k, sh.pf[e], e % 9, which < 2 ? which : 2, nb);
    }
  }
  __syncthreads();
#ifdef VQF_STAGE_CLOCKS
  t_prim = clock64();
#endif
  if (threadIdx.x < 16) {  // contract4's loop order (chem.hpp:197-212)
    double s = 0.0;
    for (int r = 0; r < 81; ++r) s += sh.prim[threadIdx.x * 81 + r];
    sh.ints.eri[threadIdx.x] = s;
  } else if (threadIdx.x >= 32 && threadIdx.x < 36) {  // ao_integrals (chem.hpp:224-239)
    const int ij = threadIdx.x - 32, i = ij >> 1, j = ij & 1;
    double s = 0.0, t = 0.0, v0 = 0.0, v1 = 0.0;
    for (int xy = 0; xy < 9; ++xy) s += sh.prim1[0 * 36 + ij * 9 + xy];
    for (int xy = 0; xy < 9; ++xy) t += sh.prim1[1 * 36 + ij * 9 + xy];
    for (int xy = 0; xy < 9; ++xy) v0 += sh.prim1[2 * 36 + ij * 9 + xy];
    for (int xy = 0; xy < 9; ++xy) v1 += sh.prim1[3 * 36 + ij * 9 + xy];
    double v = 0.0;
    v += v0;
    v += v1;
    sh.ints.S[i][j] = s;
    sh.ints.T[i][j] = t;
    sh.ints.V[i][j] = v;
  }
  __syncthreads();
#ifdef VQF_STAGE_CLOCKS
  t_sum = clock64();
#endif
  if (threadIdx.x == 0) {
    scf(sh.ints, d, sh.hf, sh.C);
    sh.stop = sh.hf.converged ? 0 : kStatusScf;
    for (int i = 0; i < 4; ++i) sh.integ[i] = sh.hf.hmo[i >> 1][i & 1];
  }
  __syncthreads();
#ifdef VQF_STAGE_CLOCKS
  t_scf = clock64();
#endif
  if (sh.stop) return;
  if (threadIdx.x < 16) sh.mo[threadIdx.x] = mo_chem(sh.C, sh.ints.eri, threadIdx.x);
  __syncthreads();
  if (threadIdx.x < 16) {  // chemist -> physicist: <ij|kl> = (ik|jl)
    const int i = threadIdx.x >> 3, j = (threadIdx.x >> 2) & 1, kk = (threadIdx.x >> 1) & 1, l = threadIdx.x & 1;
    sh.integ[4 + threadIdx.x] = sh.mo[((i * 2 + kk) * 2 + j) * 2 + l];
  }
  __syncthreads();
#ifdef VQF_STAGE_CLOCKS
  t_mo = clock64();
#endif
  // Jordan-Wigner: per Pauli string, its contributions in generation order
  // (canonicalize merges in order of first appearance, pauli.hpp:180-190).
  // contribution values, block-parallel, staged in smem (sh.prim is free
  // again); then each string sums its own run sequentially, in generation
  // order, from smem
  static_assert(kNumContrib <= 1296, "contribution values reuse sh.prim");
#pragma unroll
  for (int u = 0; u < kContribPerThread; ++u) {
    const int e = threadIdx.x + u * kPesThreads;
    if (e < kNumContrib) {
      sh.prim[e] = c_slot[u] < 0 ? sh.hf.e_nuc : c_coef[u] * sh.integ[c_slot[u]];
      sh.cpart[e] = static_cast<unsigned char>(c_part[u]);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < jw.n_keys; t += blockDim.x) {
    double re = 0.0, im = 0.0;
    const int e1 = jw.start[t + 1];
    int e = jw.start[t];
    for (; e + 4 <= e1; e += 4) {  // loads batched ahead of the ordered adds
      double v[4];
      unsigned char pt[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = sh.prim[e + u];
        pt[u] = sh.cpart[e + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (pt[u]) im += v[u];
        else re += v[u];
      }
    }
    for (; e < e1; ++e) {
      const double v = sh.prim[e];
      if (sh.cpart[e]) im += v;
      else re += v;
    }
    sh.kre[t] = re;
    sh.kim[t] = im;
    // canonicalize drop (|c| < 1e-12) and check_hermitian_coefficients
    // (pauli.hpp:195-214), decided per string in parallel
    sh.kflag[t] = hypot(re, im) < 1e-12 ? 0 : (fabs(im) >= 1e-10 ? 2 : 1);
  }
  __syncthreads();
  // Compaction in canonical order (the table order), block-parallel: a
  // survivor's slot is the number of survivors before it (warp ballots +
  // per-warp counts).  The first non-Hermitian survivor raises, as the
  // reference's check loop does (pauli.hpp:207-214).
  static_assert(kPesThreads >= 256, "one thread per Jordan-Wigner key");
  {
    const int t = threadIdx.x, w = t >> 5, ln = t & 31;
    const int flag = t < jw.n_keys ? sh.kflag[t] : 0;
    const unsigned live = __ballot_sync(0xffffffffu, flag == 1), bad = __ballot_sync(0xffffffffu, flag == 2);
    if (w < 8 && ln == 0) {
      sh.wlive[w] = __popc(live);
      sh.wbad[w] = bad ? w * 32 + __ffs(bad) - 1 : 1 << 30;
    }
    __syncthreads();
    int base = 0, total = 0, first_bad = 1 << 30;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      base += u < w ? sh.wlive[u] : 0;
      total += sh.wlive[u];
      first_bad = min(first_bad, sh.wbad[u]);
    }
    if (first_bad < (1 << 30)) {
      if (t == 0) {
        sh.stop = kStatusHermitian;
        p.err_val[prob] = sh.kim[first_bad];
        sh.n_terms = 0;
      }
    } else if (flag == 1) {
      const int nt = base + __popc(live & ((1u << ln) - 1u));
      const int key = jw.keys[t], x = key & 15, z = key >> 4;
      uint64_t flip = 0, yz = 0;  // MSB-first: qubit q -> bit (3 - q)
      for (int q = 0; q < 4; ++q) {
        if ((x >> q) & 1) flip |= uint64_t{1} << (3 - q);
        if ((z >> q) & 1) yz |= uint64_t{1} << (3 - q);
      }
      const double c = sh.kre[t];  // imaginary part discarded (chem.hpp:465)
      MaskTerm mt{flip, yz, 0.0, 0.0};
      switch (__popc(x & z) & 3) {  // c * (-i)^{n_y}
        case 0: mt.cb_re = c; break;
        case 1: mt.cb_im = -c; break;
        case 2: mt.cb_re = -c; break;
        default: mt.cb_im = c; break;
      }
      if (p.ham_keys != nullptr && nt < 16) {
        p.ham_keys[prob * 16 + nt] = key;
        p.ham_coeffs[prob * 16 + nt] = c;
      }
      sh.terms[nt] = mt;
    }
    if (t == 0 && first_bad >= (1 << 30)) sh.n_terms = total;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nt = sh.n_terms;
#ifdef VQF_STAGE_CLOCKS
    t_jw = clock64();
    if (prob == 0)
      printf("PROLOGUE pair=%lld boys=%lld prims=%lld sums=%lld scf=%lld mo=%lld jw=%lld total=%lld (scf iters %d)\n",
             t_pf - t_start, t_boys - t_pf, t_prim - t_boys, t_sum - t_prim, t_scf - t_sum, t_mo - t_scf, t_jw - t_mo,
             t_jw - t_start, sh.hf.scf_iterations);
#endif
    if (p.ham_count != nullptr) p.ham_count[prob] = sh.stop ? 0 : nt;
    if (p.hf_out != nullptr) {
      p.hf_out[4 * prob + 0] = sh.hf.hf_energy;
      p.hf_out[4 * prob + 1] = sh.hf.e_elec;
      p.hf_out[4 * prob + 2] = sh.hf.e_nuc;
      p.hf_out[4 * prob + 3] = sh.hf.scf_iterations;
    }
  }
  __syncthreads();
}

// Common kernel prologue: bias tables to smem, the problem's Hamiltonian as
// mask terms (built on device in PES mode), then the lane tables.  Returns
// false for threads that take no part in the optimisation (warps 1..3 of a
// PES CTA, or a problem that already failed).
#ifdef VQF_STAGE_CLOCKS
__device__ unsigned long long g_marks[4];  // bond 0: after bias tables, Hamiltonian, lane tables
__device__ __forceinline__ void gmark(int prob, int i) {
  if (prob == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_marks[i] = t;
  }
}
#else
__device__ __forceinline__ void gmark(int, int) {}
#endif

template <bool PES>
__device__ __forceinline__ bool prologue(Shared& sh, const SmallParams& p, int prob, double* bc, int D) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sh.stop = 0;
    if (p.clk) p.clk[2 * prob] = global_ns();
  }
  for (int t = threadIdx.x; t < p.max_iterations; t += blockDim.x) {
    bc[2 * t] = p.bc1[t];
    bc[2 * t + 1] = p.bc2[t];
  }
  // single-warp CTAs read bc after build_tables' __syncwarp; PES CTAs after
  // the chemistry's first __syncthreads, so the copy's load latency overlaps
  // the pair-factor stage instead of stalling the whole CTA here
  if (!PES) __syncthreads();
  gmark(prob, 0);
  if (PES) {
    if (p.grid_n > 0) {  // grid mode: the range check (chem.hpp:33-34) is ours
      const double b = pes_bond(p, prob);
      const int32_t st = (b >= chem::kMinBond && b <= chem::kMaxBond) ? 0 : kStatusBond;
      if (threadIdx.x == 0) p.status[prob] = st;
      if (st != 0) return false;
    } else if (p.status[prob] != 0) {
      return false;  // rejected on the host (bond out of range)
    }
    build_h2_device(sh, p, prob);
    if (sh.stop) {
      if (threadIdx.x == 0) p.status[prob] = sh.stop;
      return false;
    }
    gmark(prob, 1);
    if (threadIdx.x >= 32) return false;  // warp 0 runs the optimisation
  } else {
    const uint32_t t0 = p.term_off[prob], t1 = p.term_off[prob + 1];
    for (uint32_t t = t0 + lane; t < t1; t += 32) sh.terms[t - t0] = p.terms[t];
    if (lane == 0) sh.n_terms = static_cast<int>(t1 - t0);
    __syncwarp();
  }
  build_tables(sh, D, lane);
  if (lane < 16) sh.init_state[lane] = lane == 12 ? 1.0 : 0.0;  // basis_state(4, {1,1,0,0}) (vqe.hpp:77)
  __syncwarp();
  gmark(prob, 2);
  return true;
}

// Failure of checked_energy / gradient at iteration `iter` (vqe.hpp:213-229):
// decoded off the hot path.
__device__ __forceinline__ void h2_fail(const SmallParams& p, int prob, int iter, double th, double2 e0, double2 ep,
                                     double2 em) {
  int st;
  double val = 0.0;
  if (fabs(e0.y) >= 1e-10) {
    st = kStatusImag;
    val = e0.y;
  } else if (!isfinite(e0.x)) {
    st = kStatusNonFinite;
  } else {
    st = kStatusImag;
    val = fabs(ep.y) >= 1e-10 ? ep.y : em.y;
  }
  p.status[prob] = st;
  p.err_val[prob] = val;
  p.err_iter[prob] = iter;
  p.err_theta[prob] = th;
}

// The three circuits of one H2 iteration, E(theta), E(theta + pi/2) and
// E(theta - pi/2) (vqe.hpp:115-127).  Lanes 8c..8c+7 hold circuit c with
// amplitude indices {sl, 8 + sl} (lanes 24..31 repeat circuit 0).  G: the
// number of flip groups, compile-time so the group loop has no branches
// (1..4, tables in registers); 0 = any count, tables read from smem.
// The ansatz (basis_state |1100>, then DoubleExcitation, a real rotation)
// keeps every amplitude real: imaginary parts are exactly zero in the
// reference's complex arithmetic too, so they are not carried (real parts
// are the same sums; the energy's imaginary part comes from the Hamiltonian
// tables' imaginary parts alone and is still formed and checked).
struct H2Lane {
  int sl, circ, G;
  double shift;  // 0, +pi/2, -pi/2 (theta + shift is the reference's sum)
  int fl[4], fs[4];
  double2 o0[4], o1[4];
  double in0, in1, q0, q1;  // |1100> and its DoubleExcitation partners
  // G < 0 (whole-state lanes, PES): lane c < 3 holds circuit c's complete
  // 16-amplitude state in registers; real operator tables of the diagonal
  // group and the flip-15 group (XXYY-type strings), the input state
  double fo0[16], fo1[16], fin[16];
};

// own: this lane's circuit total (lane 0 holds E(theta)); ep_re / em_re:
// the real parts of the two shifted energies on every lane.
template <int G, bool FAST>
__device__ __forceinline__ void h2_energies(const Shared& sh, const H2Lane& L, double th, double2& own,
                                            double& ep_re, double& em_re) {
  // gradient(): shifted[k] = theta[k] +- pi/2 (vqe.hpp:119-121)
  const double t = th + L.shift;
  double sn, cs;
  if (FAST) sincos_reduced(0.5 * t, &sn, &cs);
  else sincos(0.5 * t, &sn, &cs);
  if constexpr (G < 0) {
    // whole-state lanes: the circuit's 16 amplitudes in this lane.
    // DoubleExcitation(0,1,2,3) rotates indices 12 (wires 0,1 set) and 3
    // (statevector.hpp:186-197); every other amplitude passes through.  The
    // expectation runs over all 16 amplitudes: sum_i O_0(i) psi_i^2 +
    // sum_i O_15(i) psi_i psi_{i^15}, eight independent partial sums.  No
    // shuffle until the three circuit energies are exchanged.
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = L.fin[i];
    x[12] = fma(cs, L.fin[12], -(sn * L.fin[3]));
    x[3] = fma(sn, L.fin[12], cs * L.fin[3]);
    double part[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) part[i] = L.fo0[i] * (x[i] * x[i]);
#pragma unroll
    for (int i = 8; i < 16; ++i) part[i & 7] = fma(L.fo0[i], x[i] * x[i], part[i & 7]);
#pragma unroll
    for (int i = 0; i < 16; ++i) part[i & 7] = fma(L.fo1[i], x[i] * x[i ^ 15], part[i & 7]);
    const double e = ((part[0] + part[1]) + (part[2] + part[3])) + ((part[4] + part[5]) + (part[6] + part[7]));
    own = make_double2(e, 0.0);  // real tables and amplitudes: no imaginary part (checked at setup)
    ep_re = __shfl_sync(0xffffffffu, e, 1);
    em_re = __shfl_sync(0xffffffffu, e, 2);
    return;
  }
  // DoubleExcitation(0,1,2,3) on the fixed input |1100>: indices 12 and 3
  // rotate; every other amplitude and its partner are zero, so the same
  // rotation formula on all lanes leaves them zero (no per-lane select).
  const double a1 = fma(cs, L.in1, -sn * L.q1);
  const double a0 = fma(sn, L.q0, cs * L.in0);
  // expectation: sum_g O_g(i) conj(psi_i) psi_{i ^ f_g}.  Group 0 is the
  // diagonal (flip 0, build_tables puts it first): O_0(i) |psi_i|^2 with no
  // exchange; the flip groups exchange partners by shuffle (xor 0 when a
  // group flips only the slot bit).  Group terms are formed independently,
  // then added in group order.
  double2 acc;
  if (G > 0) {
    // conj(psi_i) psi_j is the real a_i a_j: O(i) times a real product
    double2 term[4];
    {
      const double n0 = a0 * a0, n1 = a1 * a1;
      term[0] = make_double2(fma(L.o0[0].x, n0, L.o1[0].x * n1), fma(L.o0[0].y, n0, L.o1[0].y * n1));
    }
#pragma unroll
    for (int g = 1; g < 4; ++g) {
      term[g] = make_double2(0.0, 0.0);
      if (g < G) {
        double r0 = L.fs[g] ? a1 : a0, r1 = L.fs[g] ? a0 : a1;
        r0 = __shfl_xor_sync(0xffffffffu, r0, L.fl[g], 8);
        r1 = __shfl_xor_sync(0xffffffffu, r1, L.fl[g], 8);
        const double v0 = a0 * r0, v1 = a1 * r1;
        term[g] = make_double2(fma(L.o0[g].x, v0, L.o1[g].x * v1), fma(L.o0[g].y, v0, L.o1[g].y * v1));
      }
    }
    if (G == 1) acc = term[0];
    else if (G == 2) acc = make_double2(term[0].x + term[1].x, term[0].y + term[1].y);
    else if (G == 3) acc = make_double2((term[0].x + term[1].x) + term[2].x, (term[0].y + term[1].y) + term[2].y);
    else acc = make_double2((term[0].x + term[1].x) + (term[2].x + term[3].x),
                            (term[0].y + term[1].y) + (term[2].y + term[3].y));
  } else {
    acc = make_double2(0.0, 0.0);
    for (int g = 0; g < L.G; ++g) {
      const int f = sh.flip[g], fl = f & 7;
      double r0 = (f & 8) ? a1 : a0, r1 = (f & 8) ? a0 : a1;
      r0 = __shfl_xor_sync(0xffffffffu, r0, fl, 8);
      r1 = __shfl_xor_sync(0xffffffffu, r1, fl, 8);
      const double2 o0 = sh.tab[g * 16 + L.sl], o1 = sh.tab[g * 16 + 8 + L.sl];
      const double v0 = a0 * r0, v1 = a1 * r1;
      acc.x += fma(o0.x, v0, o1.x * v1);
      acc.y += fma(o0.y, v0, o1.y * v1);
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o, 8);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o, 8);
  }
  own = acc;
  ep_re = __shfl_sync(0xffffffffu, acc.x, 8);
  em_re = __shfl_sync(0xffffffffu, acc.x, 16);
}

// One iteration of run_vqe's loop (vqe.hpp:225-243) on one warp: energies,
// checks, trajectory, gradient, tolerance, Adam.  Every lane carries theta /
// m / v and runs Adam itself (identical values in all lanes, no broadcast).
// Returns 0 continue, 1 converged, 2 failed (status written), 3 theta left
// the fast-trig range (FAST only; nothing written, redo with FAST = false).
struct H2State {
  double th, m, v;
};

template <int G, bool FAST>
__device__ __forceinline__ int h2_step(const Shared& sh, const SmallParams& p, int prob, const double* bc,
                                       const H2Lane& L, int iter, H2State& s, double tol, double* traj) {
  const int lane = threadIdx.x & 31;
  const bool range_bad = FAST && !(fabs(s.th) < kFastTrigTheta);  // warp-uniform
  const double2 bcs = reinterpret_cast<const double2*>(bc)[iter];  // issued early, used by Adam
  double2 own;
  double ep_re, em_re;
  h2_energies<G, FAST>(sh, L, s.th, own, ep_re, em_re);

  // gradient and the Adam update (vqe.hpp:152-174, t = iter + 1; bias
  // corrections as host-computed reciprocals 1 / (1 - beta^t)) are formed
  // first and committed after the checks, so their latency overlaps the vote
  const double g = 0.5 * (ep_re - em_re);
  const double mk = p.beta1 * s.m + (1.0 - p.beta1) * g;
  const double vk = p.beta2 * s.v + (1.0 - p.beta2) * g * g;
  const double th_next = s.th - adam_delta_fast(p.lr, mk * bcs.x, vk * bcs.y, p.eps);
  // checked_energy, then the gradient's two expectations (vqe.hpp:227-229):
  // each lane checks its own circuit, one vote
  const bool my_bad = range_bad || fabs(own.y) >= 1e-10 || (L.circ == 0 && !isfinite(own.x));
  if (__any_sync(0xffffffffu, my_bad)) {
    if (range_bad) return 3;
    const double2 e0 = shfl2(own, 0), ep = shfl2(own, 8), em = shfl2(own, 16);
    if (lane == 0) h2_fail(p, prob, iter, s.th, e0, ep, em);
    return 2;
  }
  if (lane == 0) traj[iter] = own.x;
  if (fabs(g) < tol) return 1;
  s.th = th_next;
  s.m = mk;
  s.v = vk;
  return 0;
}

// run_vqe's loop (vqe.hpp:225-247) for one bond: the fast-trig loop, and
// the library-sincos continuation should theta ever leave its range.
template <int G>
__device__ __forceinline__ void h2_optimise(const Shared& sh, const SmallParams& p, int prob, const double* bc,
                                            const H2Lane& L, unsigned long long g_entry, unsigned long long g_loop) {
  const int lane = threadIdx.x & 31;
  double* traj = p.traj + (size_t)prob * p.traj_stride;
  H2State s{p.init_theta ? p.init_theta[prob] : 0.0, 0.0, 0.0};
  const double tol = p.has_tol ? p.tol : -1.0;  // |g| < -1 never holds
  const int T = p.max_iterations;
#ifdef VQF_STAGE_CLOCKS
  long long c100 = 0, c101 = 0;
#endif
  int iter = 0, rc = 0;
  for (; iter < T; ++iter) {
#ifdef VQF_STAGE_CLOCKS
    if (iter == 100) c100 = clock64();
    if (iter == 101) c101 = clock64();
#endif
    rc = h2_step<G, true>(sh, p, prob, bc, L, iter, s, tol, traj);
    if (rc != 0) break;
  }
  if (rc == 3) {
    for (rc = 0; iter < T; ++iter) {
      rc = h2_step<G, false>(sh, p, prob, bc, L, iter, s, tol, traj);
      if (rc != 0) break;
    }
  }
  if (rc == 2) return;
  const int converged = rc == 1, iters = iter;
  double e_final;
  if (converged) {
    e_final = traj[iters];
  } else {  // the final checked_energy (vqe.hpp:244-247)
    double2 own;
    double ep_re, em_re;
    if (fabs(s.th) < kFastTrigTheta) h2_energies<G, true>(sh, L, s.th, own, ep_re, em_re);
    else h2_energies<G, false>(sh, L, s.th, own, ep_re, em_re);
    const double2 e0 = shfl2(own, 0);
    if (fabs(e0.y) >= 1e-10 || !isfinite(e0.x)) {
      if (lane == 0) h2_fail(p, prob, T, s.th, e0, make_double2(0.0, 0.0), make_double2(0.0, 0.0));
      return;
    }
    if (lane == 0) traj[T] = e0.x;
    e_final = e0.x;
  }
#ifdef VQF_STAGE_CLOCKS
  if (prob == 0 && lane == 0) printf("STAGES iteration=%lld\n", c101 - c100);
  if (lane == 0) {
    unsigned long long g_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    printf("TIMELINE bond %d sm %u entry %llu prologue_ns %llu loop_ns %llu end %llu\n", prob,
           static_cast<unsigned>(__mysmid()), g_entry, g_loop - g_entry, g_end - g_loop, g_end);
    if (prob == 0)
      printf("PROLOGUE_NS bias %llu hamiltonian %llu tables %llu\n", g_marks[0] - g_entry, g_marks[1] - g_marks[0],
             g_marks[2] - g_marks[1]);
  }
#else
  (void)g_entry;
  (void)g_loop;
#endif
  if (lane == 0) {
    if (p.clk) p.clk[2 * prob + 1] = global_ns();
    p.iters[prob] = iters;
    p.converged[prob] = converged;
    p.energy[prob] = e_final;
    p.theta_out[prob] = s.th;
  }
  const int len = converged ? iters + 1 : T + 1;
  for (int k = len + lane; k < p.traj_stride; k += 32) traj[k] = __longlong_as_double(-1LL);
}

// H2 fast path (n = 4, one parameter, 3 circuits x 8 lanes x 2 amplitudes).
// Exchanges per iteration: one shuffle per flip group, a 3-level reduction
// and 3 energy shuffles; the DoubleExcitation partner exchange of the fixed
// input state is done once.
template <bool PES>
__global__ void __launch_bounds__(PES ? kPesThreads : 32, 1) k_h2(SmallParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
  double* bc = reinterpret_cast<double*>(smem_raw + sizeof(Shared));
  const int prob = blockIdx.x;
  unsigned long long g_entry = 0, g_loop = 0;
#ifdef VQF_STAGE_CLOCKS
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
#endif
  if (!prologue<PES>(sh, p, prob, bc, 16)) return;
#ifdef VQF_STAGE_CLOCKS
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_loop));
#endif
  H2Lane L;
  const int lane = threadIdx.x & 31, seg = lane >> 3;
  L.sl = lane & 7;
  L.circ = seg < 3 ? seg : 0;
  L.shift = L.circ == 1 ? kShift : L.circ == 2 ? -kShift : 0.0;
  L.G = sh.n_groups;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const bool on = g < L.G;
    const int f = on ? sh.flip[g] : 0;
    L.fl[g] = f & 7;
    L.fs[g] = f & 8;
    L.o0[g] = on ? sh.tab[g * 16 + L.sl] : make_double2(0.0, 0.0);
    L.o1[g] = on ? sh.tab[g * 16 + 8 + L.sl] : make_double2(0.0, 0.0);
  }
  // basis_state(4, {1,1,0,0}): index 12 = slot 1 of sl 4; partner i ^ 15
  L.in0 = 0.0;
  L.in1 = L.sl == 4 ? 1.0 : 0.0;
  L.q0 = __shfl_xor_sync(0xffffffffu, L.in1, 7, 8);
  L.q1 = __shfl_xor_sync(0xffffffffu, L.in0, 7, 8);
  // PES Hamiltonians (real Jordan-Wigner coefficients, a diagonal group and
  // at most the flip-15 group) run with whole-state lanes: no reduction
  // shuffles on the iteration's critical path
  bool full = PES && L.G >= 1 && L.G <= 2 && sh.flip[0] == 0 && (L.G < 2 || sh.flip[1] == 15);
  if (full)
    for (int g = 0; g < L.G; ++g)
      for (int i = 0; i < 16; ++i) full = full && sh.tab[g * 16 + i].y == 0.0;
  if (full) {
    L.circ = lane < 3 ? lane : 0;
    L.shift = L.circ == 1 ? kShift : L.circ == 2 ? -kShift : 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      L.fo0[i] = sh.tab[i].x;
      L.fo1[i] = L.G == 2 ? sh.tab[16 + i].x : 0.0;
      L.fin[i] = sh.init_state[i];
    }
    h2_optimise<-1>(sh, p, prob, bc, L, g_entry, g_loop);
    return;
  }
  switch (L.G) {  // warp-uniform: one specialised loop per group count
    case 1: h2_optimise<1>(sh, p, prob, bc, L, g_entry, g_loop); break;
    case 2: h2_optimise<2>(sh, p, prob, bc, L, g_entry, g_loop); break;
    case 3: h2_optimise<3>(sh, p, prob, bc, L, g_entry, g_loop); break;
    case 4: h2_optimise<4>(sh, p, prob, bc, L, g_entry, g_loop); break;
    default: h2_optimise<0>(sh, p, prob, bc, L, g_entry, g_loop); break;
  }
}

template <int A, bool PES, bool H2>
__global__ void __launch_bounds__(PES ? kPesThreads : 32) k_vqe_warp(SmallParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
  const int prob = blockIdx.x;
  const int n = p.n_qubits, D = 1 << n, P = p.n_params, NC = 2 * P + 1;
  const int L = D / A;
  const int lgL = __ffs(L) - 1;
  const int lane = threadIdx.x & 31;
  double* bc = reinterpret_cast<double*>(smem_raw + sizeof(Shared));  // [2][T]

  if (!prologue<PES>(sh, p, prob, bc, D)) return;
  int basis = 12;
  if (!H2) {
    if (lane == 0) basis = build_program(sh, p.ansatz_kind, n, p.layers);
    basis = __shfl_sync(0xffffffffu, basis, 0);
  }
  // lane k owns parameter k (and k + 32): theta, m, v in registers
  double th_reg[2], m_reg[2] = {0.0, 0.0}, v_reg[2] = {0.0, 0.0};
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int k = lane + 32 * r;
    th_reg[r] = (k < P && p.init_theta) ? p.init_theta[(size_t)prob * P + k] : 0.0;
    if (k < P) sh.theta[k] = th_reg[r];
  }
  __syncwarp();

  double* traj = p.traj + (size_t)prob * p.traj_stride;
  const int seg = lane / L, segs = 32 / L, sl = lane % L;
  int iters = 0, converged = 0, status = 0;
  double err_val = 0.0;

  for (int iter = 0; iter <= p.max_iterations; ++iter) {
    const bool final_eval = (iter == p.max_iterations);  // vqe.hpp:244-247
    // (1) angles: (cos, sin)(0.5 * (theta_k + {0, +pi/2, -pi/2}))
    for (int idx = lane; idx < 3 * P; idx += 32) {
      const int k = idx / 3, j = idx - 3 * k;
      double t = sh.theta[k];
      if (j == 1) t = t + kShift;
      if (j == 2) t = t - kShift;
      double s, c;
      sincos_short(0.5 * t, &s, &c);
      sh.cs[k][j] = make_double2(c, s);
    }
    __syncwarp();
    // (2) circuits, segs at a time; energies exchanged by shuffles when one
    //     round covers every circuit (the common case), else via smem
    const int nc = final_eval ? 1 : NC;
    double2 e_own = make_double2(0.0, 0.0);
    for (int c0 = 0; c0 < nc; c0 += segs) {
      const int c = c0 + seg;
      double2 amp[A];
      run_circuit<A, H2>(sh, amp, c < nc ? c : 0, sl, L, lgL, basis);
      const double2 e = circuit_energy<A>(sh, amp, sl, L, lgL, D);
      if (nc <= segs) e_own = e;
      else if (sl == 0 && c < nc) sh.energy[c] = e;
    }
    if (nc > segs) __syncwarp();
    auto energy_of = [&](int c) -> double2 {  // warp-uniform c
      return nc <= segs ? shfl2(e_own, c * L) : sh.energy[c];
    };
    // (3) checked_energy + gradient checks in the reference's order
    //     (vqe.hpp:227-238), evaluated redundantly by every lane
    {
      const double2 e0 = energy_of(0);
      if (fabs(e0.y) >= 1e-10) {
        status = kStatusImag;
        err_val = e0.y;
      } else if (!isfinite(e0.x)) {
        status = kStatusNonFinite;
      } else {
        for (int c = 1; c < nc; ++c) {
          const double im = energy_of(c).y;
          if (!status && fabs(im) >= 1e-10) {
            status = kStatusImag;
            err_val = im;
          }
        }
      }
      if (status) {
        if (lane == 0) {
          p.status[prob] = status;
          p.err_val[prob] = err_val;
          p.err_iter[prob] = iter;
          for (int k = 0; k < P; ++k) p.err_theta[(size_t)prob * P + k] = sh.theta[k];
        }
        break;
      }
      if (lane == 0) traj[iter] = e0.x;
    }
    if (final_eval) break;
    // gradient (vqe.hpp:118-124) in the lane that owns the parameter
    double g_reg[2] = {0.0, 0.0};
    double g_inf = 0.0;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (32 * r >= P) break;
      const int k = lane + 32 * r;
      double ep, em;
      if (nc <= segs) {
        const int kk = k < P ? k : 0;
        ep = __shfl_sync(0xffffffffu, e_own.x, ((2 * kk + 1) * L) & 31);
        em = __shfl_sync(0xffffffffu, e_own.x, ((2 * kk + 2) * L) & 31);
      } else {
        ep = k < P ? sh.energy[2 * k + 1].x : 0.0;
        em = k < P ? sh.energy[2 * k + 2].x : 0.0;
      }
      g_reg[r] = 0.5 * (ep - em);
      if (k < P) g_inf = fmax(g_inf, fabs(g_reg[r]));
    }
    for (int o = 1; o < P && o < 32; o <<= 1) g_inf = fmax(g_inf, __shfl_xor_sync(0xffffffffu, g_inf, o));
    g_inf = __shfl_sync(0xffffffffu, g_inf, 0);  // warp-uniform stop decision
    if (p.has_tol && g_inf < p.tol) {
      converged = 1;
      break;
    }
    // (4) adam_step (vqe.hpp:152-174), t = iter + 1, in the owning lane
    const double b1 = bc[2 * iter], b2 = bc[2 * iter + 1];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int k = lane + 32 * r;
      if (k < P) {
        const double g = g_reg[r];
        const double mk = p.beta1 * m_reg[r] + (1.0 - p.beta1) * g;
        const double vk = p.beta2 * v_reg[r] + (1.0 - p.beta2) * g * g;
        const double m_hat = mk * b1;  // b1, b2 = 1 / (1 - beta^t)
        const double v_hat = vk * b2;
        th_reg[r] = th_reg[r] - adam_delta(p.lr, m_hat, v_hat, p.eps);
        m_reg[r] = mk;
        v_reg[r] = vk;
        sh.theta[k] = th_reg[r];
      }
    }
    iters = iter + 1;
    __syncwarp();
  }
  if (status) return;
  if (lane == 0) {
    if (p.clk) p.clk[2 * prob + 1] = global_ns();
    p.iters[prob] = iters;
    p.converged[prob] = converged;
    p.energy[prob] = traj[converged ? iters : p.max_iterations];
  }
  for (int k = lane; k < P; k += 32) p.theta_out[(size_t)prob * P + k] = sh.theta[k];
  // NaN-pad the unused tail of a converged run's trajectory row
  const int len = converged ? iters + 1 : p.max_iterations + 1;
  for (int t = len + lane; t < p.traj_stride; t += 32) traj[t] = __longlong_as_double(-1LL);
}

size_t smem_for(const SmallParams& p) {
  const size_t smem = sizeof(Shared) + 2 * sizeof(double) * (size_t)std::max(p.max_iterations, 1);
  if (smem > 227 * 1024) throw_invalid("small engine: max_iterations too large for the on-chip bias tables");
  return smem;
}

// Raises a kernel's dynamic shared memory limit once per process (the
// attribute is per function, and the driver call costs microseconds on the
// launch path otherwise).
void opt_in_smem(void (*kernel)(SmallParams)) {
  static std::mutex mu;
  static std::vector<std::pair<int, const void*>> done;  // (device, kernel)
  int dev = 0;
  VQF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == dev && d.second == reinterpret_cast<const void*>(kernel)) return;
  VQF_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  done.emplace_back(dev, reinterpret_cast<const void*>(kernel));
}

template <int A, bool PES, bool H2>
void launch_k(const SmallParams& p, uint32_t batch, cudaStream_t stream) {
  const size_t smem = smem_for(p);
  opt_in_smem(k_vqe_warp<A, PES, H2>);
  k_vqe_warp<A, PES, H2><<<batch, PES ? kPesThreads : 32, smem, stream>>>(p);
}

template <bool PES>
void launch_h2(const SmallParams& p, uint32_t batch, cudaStream_t stream) {
  const size_t smem = smem_for(p);
  opt_in_smem(k_h2<PES>);
  k_h2<PES><<<batch, PES ? kPesThreads : 32, smem, stream>>>(p);
}

template <int A>
void launch_a(const SmallParams& p, uint32_t batch, bool pes, cudaStream_t stream) {
  if constexpr (A == 2) {  // the H2 ansatz always lands here (D = 16, NC = 3)
    if (p.ansatz_kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION) {
      if (pes) launch_h2<true>(p, batch, stream);
      else launch_h2<false>(p, batch, stream);
      return;
    }
  }
  // PES mode builds H2 Hamiltonians: only the H2 ansatz reaches it (above),
  // so the generic kernel is instantiated without the chemistry prologue
  if (pes) throw Error(VQF_LOGIC_ERROR, "small engine: PES mode needs the H2 ansatz");
  launch_k<A, false, false>(p, batch, stream);
}

}  // namespace

size_t small_smem_bytes() { return sizeof(Shared); }

// Lanes per circuit L: the largest power of two with NC * L <= 32 and
// L <= D (one circuit round per iteration when it fits); amplitudes per
// lane A = D / L.
int small_amps_per_lane(int n_qubits, int n_params) {
  const int D = 1 << n_qubits, NC = 2 * n_params + 1;
  int L = 1;
  while (L * 2 <= D && NC * L * 2 <= 32) L *= 2;
  return D / L;
}

void launch_vqe_small(const SmallParams& p, uint32_t batch, bool pes, cudaStream_t stream) {
  switch (small_amps_per_lane(p.n_qubits, p.n_params)) {
    case 1: launch_a<1>(p, batch, pes, stream); break;
    case 2: launch_a<2>(p, batch, pes, stream); break;
    case 4: launch_a<4>(p, batch, pes, stream); break;
    case 8: launch_a<8>(p, batch, pes, stream); break;
    case 16: launch_a<16>(p, batch, pes, stream); break;
    default: throw Error(VQF_LOGIC_ERROR, "small engine: unsupported register size");
  }
  VQF_LAUNCHED();
  VQF_CUDA(cudaGetLastError());
}

}  // namespace vqf
