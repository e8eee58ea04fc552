// Shared-memory VQE engine: a whole run_vqe (vqe.hpp:194-254) in ONE
// cooperative launch for registers that fit one CTA's shared memory
// (4 <= n <= 13 complex128, <= 14 complex64; one qubit more with the state in
// an L2-resident global buffer per CTA).
//
// The reference evaluates every Adam iteration as 1 + 2P fresh circuits
// (energy(theta), then E(theta +- pi/2 e_k), vqe.hpp:112-127, :226-243).
// Here CTA c owns circuit c (CTAs loop when 2P + 1 exceeds the co-resident
// grid); its state lives in shared memory for the whole circuit:
//   * permutation gates (CNOT, X) move no data: the engine tracks the frame
//     logical index i = M p ^ c of physical slot p (M an invertible GF(2)
//     matrix, c a bit vector); a CNOT(a -> b) adds row a of M to row b, an X
//     flips a bit of c (compiled on the host, compile_block_program);
//   * RY(theta) on logical bit b pairs physical slots p and p ^ v with
//     v = M^-1 e_b; the slot holding logical bit 0 is the one with
//     parity(row_b(M) & p) ^ c_b = 0.  Rotations that commute (one layer's
//     RYs, same frame) are applied R at a time in registers: a thread loads
//     the 2^R slots base ^ span{v_1..v_R}, rotates, stores back: one shared
//     memory pass per R gates, with per-slot arithmetic bitwise equal to the
//     reference's c*a0 - s*a1 / s*a0 + c*a1 (a logical-1 base negates s);
//   * <psi|H|psi> reads the final frame: the host rewrote every term's
//     masks (flip' = M^-1 flip, yz' = M^T yz, sign (-1)^popc(yz & c)), so
//     the expectation is the usual flip-grouped pair sum over the physical
//     slots, reduced in a fixed order in the CTA;
//   * after every iteration the CTAs meet at a grid barrier; every CTA then
//     reads the 2P + 1 energies (same order), runs the reference's checks,
//     gradient, tolerance test and Adam (vqe.hpp:152-174 with the host's
//     bias corrections 1 - beta^t, IEEE divisions and sqrt: bitwise the
//     reference's update) and continues with identical parameters, so no
//     broadcast is needed.  CTA 0 writes the trajectory and the results.
// Nothing touches HBM on the critical path except 16 bytes per circuit and
// iteration; the launch is latency-bound (a few microseconds per iteration).
#include <algorithm>
#include <cstring>
#include <mutex>

#include "vqe_block.cuh"
#include "vqe_small.cuh"

namespace vqf {

namespace {

constexpr double kShift = 1.5707963267948966;  // std::numbers::pi / 2 (vqe.hpp:115)
constexpr int kBlockThreads = 512;
constexpr uint32_t kBlockSmemCap = 220 * 1024;  // dynamic; the kernel's static arrays take < 1 KB

template <typename T>
struct Amp;
template <>
struct Amp<double> {
  using type = double2;
};
template <>
struct Amp<float> {
  using type = float2;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t insert_zeros(uint32_t k, const uint32_t* piv, int r) {
  // piv ascending: open a zero at each pivot position
  for (int j = 0; j < r; ++j) {
    const uint32_t lo = k & ((1u << piv[j]) - 1u);
    k = ((k ^ lo) << 1) | lo;
  }
  return k;
}

// All CTAs arrive; thread 0 spins on the arrival counter (acquire) until
// `target`.  A 4 s watchdog (or another CTA's abort) sets the abort word and
// releases everyone, so a broken co-residency can never hang the device.
__device__ bool grid_barrier(unsigned* bar, unsigned target) {
  __shared__ int ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    const unsigned long long t0 = global_ns();
    int good = 1;
    while (ld_acquire(bar) < target) {
      if (ld_acquire(bar + 1) != 0u) {
        good = 0;
        break;
      }
      if (global_ns() - t0 > 4000000000ull) {
        atomicExch(bar + 1, 1u);
        good = 0;
        break;
      }
      __nanosleep(20);
    }
    __threadfence();
    ok = good;
  }
  __syncthreads();
  return ok != 0;
}

// Fixed-order CTA sum of one complex value per thread (result in thread 0).
__device__ double2 block_sum(double2 v, double2* scratch) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[w] = v;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; ++i) {
      s.x += scratch[i].x;
      s.y += scratch[i].y;
    }
  return s;
}

// 16 amplitudes per thread (R = 4) need more than the 128 registers a
// 512-thread CTA leaves: those passes run 256 threads x 2 bases.
template <int R>
constexpr int kThreadsOf = R >= 4 ? 256 : kBlockThreads;

// -DVQF_STAGE_CLOCKS: per-stage clock64 stamps of CTA 0, iteration 2,
// printed at exit (scripts/block_stage_clocks.sh)
#ifdef VQF_STAGE_CLOCKS
#define BCLK(k) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && iter == 2) stamp[k] = clock64()
#else
#define BCLK(k)
#endif

// The last CTA out resets the barrier words, so the next launch finds them
// zero without a memset (an aborted launch is reset by the host).
__device__ void block_exit(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(bar + 2, 1u) == gridDim.x - 1) {
      if (atomicAdd(bar + 1, 0u) == 0u) {
        bar[0] = 0u;
        bar[2] = 0u;
        __threadfence();
      }
    }
  }
}

// A team evaluates one circuit at a time.  TEAMS (small registers): teams
// of L = 2^n / 2^R lanes inside ONE CTA, one team per circuit: passes sync
// with __syncwarp, the iteration's exchange is one __syncthreads.  Otherwise
// one team per CTA (a cooperative grid of CTAs, grid barrier per iteration).
template <bool TEAMS>
struct Team {
  int id, count, lane, L;
  __device__ Team(int lanes) {
    if (TEAMS) {
      L = lanes;
      id = threadIdx.x / lanes;
      count = blockDim.x / lanes;
      lane = threadIdx.x % lanes;
    } else {
      L = blockDim.x;
      id = blockIdx.x;
      count = gridDim.x;
      lane = threadIdx.x;
    }
  }
  __device__ void sync() const {
    if (TEAMS) __syncwarp();
    else __syncthreads();
  }
  // fixed-order sum over the team (result in lane 0)
  __device__ double2 sum(double2 v, double2* scratch) const {
    if (TEAMS) {
      for (int o = L >> 1; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
      }
      return v;
    }
    return block_sum(v, scratch);
  }
};

template <typename T, int R, bool TEAMS>
__device__ void vqe_block_body(const BlockParams& p) {
  using A2 = typename Amp<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P = p.P, NC = p.NC, tid = threadIdx.x, nt = blockDim.x;
  const uint32_t D = 1u << p.n;
  const Team<TEAMS> tm(p.team_lanes);
  const int n_slots = TEAMS ? tm.count : 1;  // per-team state / angle slots
  const BlockSmem L(p.n, p.gstate ? 0 : sizeof(A2), P, p.obytes, p.herm ? p.n_terms : 0, p.herm ? p.n_groups : 0,
                    n_slots);
  A2* psi = p.gstate ? static_cast<A2*>(p.gstate) + ((size_t)blockIdx.x << p.n)
                     : reinterpret_cast<A2*>(smem_raw + L.psi) + (TEAMS ? (size_t)tm.id << p.n : 0);
  double* theta = reinterpret_cast<double*>(smem_raw + L.theta);
  double* mom = reinterpret_cast<double*>(smem_raw + L.mom);
  double* vel = reinterpret_cast<double*>(smem_raw + L.vel);
  double2* cs = reinterpret_cast<double2*>(smem_raw + L.cs);  // (cos, sin) per parameter (x3 for TEAMS)
  double2* e_all = reinterpret_cast<double2*>(smem_raw + L.e_all);  // the iteration's 2P + 1 energies
  BlockRTerm* rt = reinterpret_cast<BlockRTerm*>(smem_raw + L.rterms);
  uint32_t* gflip = reinterpret_cast<uint32_t*>(smem_raw + L.gflip);
  uint32_t* goff = reinterpret_cast<uint32_t*>(smem_raw + L.goff);
  __shared__ double2 scratch[kBlockThreads / 32];
  __shared__ double2 e_self;
  __shared__ int stop_flag;
  const int lane = tm.lane, LT = tm.L;

  if (blockIdx.x == 0 && tid == 0 && p.clk) p.clk[0] = global_ns();
  for (int k = tid; k < P; k += nt) {
    theta[k] = p.init_theta ? p.init_theta[k] : 0.0;
    mom[k] = 0.0;
    vel[k] = 0.0;
  }
  const int G = p.n_groups;
  if (p.herm) {
    // real-form Hamiltonian into shared memory, and the diagonal operator
    // O(i) = sum_t a_t (-1)^popc(yz'_t & i) once per launch: every circuit
    // of every iteration reads the same final frame
    for (int t = tid; t < p.n_terms; t += nt) rt[t] = p.rterms[t];
    for (int g = tid; g < G; g += nt) gflip[g] = p.group_flip[g];
    for (int g = tid; g <= G; g += nt) goff[g] = p.group_off[g];
    __syncthreads();
    if (p.obytes) {
      for (uint32_t i = tid; i < D; i += nt) {
        double o = 0.0;
        for (uint32_t t = goff[0]; t < goff[1]; ++t) o += (__popc(rt[t].yz & i) & 1u) ? -rt[t].a : rt[t].a;
        if (p.obytes == 8) reinterpret_cast<double*>(smem_raw + L.otab)[i] = o;
        else reinterpret_cast<float*>(smem_raw + L.otab)[i] = static_cast<float>(o);
      }
    }
  }
  __syncthreads();
  const int n_it = p.max_iterations;
  int iters = 0, converged = 0;
  unsigned arrivals = 0;
#ifdef VQF_STAGE_CLOCKS
  long long stamp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  for (int iter = 0; iter <= n_it; ++iter) {
    BCLK(0);
    if (TEAMS) {  // the iteration's 3P (cos, sin) pairs, shared by every team
      for (int q = tid; q < 3 * P; q += nt) {
        const int k = q / 3, w = q - 3 * k;
        const double a = w == 0 ? theta[k] : w == 1 ? theta[k] + kShift : theta[k] - kShift;
        double sn, cn;
        sincos(0.5 * a, &sn, &cn);
        cs[q] = make_double2(cn, sn);
      }
      __syncthreads();
    }
    const bool final_eval = iter == n_it;
    const int n_circ = final_eval ? 1 : NC;
    double2* E = p.energies + (iter & 1) * NC;
    // TEAMS: every team runs the same number of rounds (spare teams repeat
    // circuit 0 and store nothing), so warp-wide syncs always match
    const int rounds = TEAMS ? (NC + tm.count - 1) / tm.count : 1;
    for (int rd = 0, c0 = tm.id; TEAMS ? rd < rounds : c0 < n_circ; ++rd, c0 += tm.count) {
      const bool mine = c0 < n_circ;
      const int c = mine ? c0 : 0;
      // (cos, sin) of half the circuit's angles (apply_gate, statevector.hpp:157-158)
      const int shifted = c == 0 ? -1 : (c - 1) >> 1;
      tm.sync();
      if (!TEAMS)
        for (int k = lane; k < P; k += LT) {
          double a = theta[k];
          if (k == shifted) a = (c & 1) ? a + kShift : a - kShift;
          double sn, cn;
          sincos(0.5 * a, &sn, &cn);
          cs[k] = make_double2(cn, sn);
        }
      // TEAMS: cs holds (theta, theta + pi/2, theta - pi/2) per parameter,
      // computed once per iteration for the whole CTA
      const int csel = (c & 1) ? 1 : 2;
      for (uint32_t i = lane; i < D; i += LT) psi[i] = A2{T(0), T(0)};
      tm.sync();
      if (lane == 0) psi[block_slot(p.init_index)] = A2{T(1), T(0)};
      tm.sync();
      BCLK(1);
      // rotation passes: thread-owned cosets base ^ span{vec}, R commuting
      // RYs in fp64 registers (complex64 states round once per pass)
      for (int ps = 0; ps < p.n_passes; ++ps) {
        const BlockPass& bp = p.passes[ps];
        uint32_t sv[R], row[R], piv[R];
        int par[R];
        double cj[R], sj[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          sv[j] = bp.svec[j];
          row[j] = bp.row[j];
          piv[j] = bp.piv[j];
          par[j] = bp.param[j];
          const double2 t = par[j] < 0       ? make_double2(1.0, 0.0)
                            : !TEAMS         ? cs[par[j]]
                            : cs[3 * par[j] + (par[j] == shifted ? csel : 0)];
          cj[j] = t.x;
          sj[j] = t.y;
        }
        const uint32_t cb = bp.cbits;
        for (uint32_t b = lane; b < (D >> R); b += LT) {
          const uint32_t base = insert_zeros(b, piv, R);
          const uint32_t sbase = block_slot(base);
          double2 x[1 << R];
#pragma unroll
          for (int m = 0; m < (1 << R); ++m) {
            uint32_t o = sbase;
#pragma unroll
            for (int j = 0; j < R; ++j)
              if ((m >> j) & 1) o ^= sv[j];
            const A2 v = psi[o];
            x[m] = make_double2(v.x, v.y);
          }
#pragma unroll
          for (int j = 0; j < R; ++j) {
            if (par[j] < 0) continue;  // padding vector: no rotation
            // padding vectors are orthogonal to every real row, so the
            // logical bit of wire j flips exactly with m_j: one orientation
            // per coset (a logical-1 base swaps the roles: s -> -s)
            const bool one = ((__popc(row[j] & base) ^ (cb >> j)) & 1u) != 0u;
            const double cc = cj[j], s = one ? -sj[j] : sj[j];
#pragma unroll
            for (int m = 0; m < (1 << R); ++m) {
              if ((m >> j) & 1) continue;
              const double2 t0 = x[m], t1 = x[m | (1 << j)];
              x[m] = make_double2(fma(cc, t0.x, -(s * t1.x)), fma(cc, t0.y, -(s * t1.y)));
              x[m | (1 << j)] = make_double2(fma(s, t0.x, cc * t1.x), fma(s, t0.y, cc * t1.y));
            }
          }
#pragma unroll
          for (int m = 0; m < (1 << R); ++m) {
            uint32_t o = sbase;
#pragma unroll
            for (int j = 0; j < R; ++j)
              if ((m >> j) & 1) o ^= sv[j];
            psi[o] = A2{T(x[m].x), T(x[m].y)};
          }
        }
        tm.sync();
      }
      BCLK(2);
      // expectation (statevector.hpp:217-249) over the final frame
      double2 acc = make_double2(0.0, 0.0);
      if (p.herm) {
        if (p.obytes) {
          for (uint32_t i = lane; i < D; i += LT) {
            const A2 a = psi[block_slot(i)];
            const double o = p.obytes == 8 ? reinterpret_cast<const double*>(smem_raw + L.otab)[i]
                                           : (double)reinterpret_cast<const float*>(smem_raw + L.otab)[i];
            acc.x = fma((double)a.x * (double)a.x + (double)a.y * (double)a.y, o, acc.x);
          }
        } else if (goff[1] > goff[0]) {
          for (uint32_t i = lane; i < D; i += LT) {
            const A2 a = psi[block_slot(i)];
            double o = 0.0;
            for (uint32_t t = goff[0]; t < goff[1]; ++t) o += (__popc(rt[t].yz & i) & 1u) ? -rt[t].a : rt[t].a;
            acc.x = fma((double)a.x * (double)a.x + (double)a.y * (double)a.y, o, acc.x);
          }
        }
        for (int g = 1; g < G; ++g) {
          const uint32_t F = gflip[g], t0 = goff[g], t1 = goff[g + 1], sF = block_slot(F);
          const uint32_t pv = 31 - __clz(F);  // highest flip bit: pair bases stay contiguous
          for (uint32_t k = lane; k < (D >> 1); k += LT) {
            const uint32_t lo = k & ((1u << pv) - 1u);
            const uint32_t i = ((k ^ lo) << 1) | lo, si = block_slot(i);
            const A2 a = psi[si], bb = psi[si ^ sF];
            // w = 2 Re(conj(a) b) or 2 Im(conj(a) b)
            const double wre = 2.0 * fma((double)a.x, (double)bb.x, (double)a.y * (double)bb.y);
            const double wim = 2.0 * fma((double)a.x, (double)bb.y, -((double)a.y * (double)bb.x));
            for (uint32_t t = t0; t < t1; ++t) {
              const BlockRTerm q = rt[t];
              const double w = q.odd ? wim : wre;
              acc.x = fma((__popc(q.yz & i) & 1u) ? -q.a : q.a, w, acc.x);
            }
          }
        }
      } else {
        // general (non-Hermitian) coefficients: complex accumulation, so the
        // reference's imaginary-residue check sees the true residue
        const uint32_t t0 = p.group_off[0], t1 = p.group_off[1];
        if (t1 > t0)
          for (uint32_t i = lane; i < D; i += LT) {
            const A2 a = psi[block_slot(i)];
            const double pr = (double)a.x * (double)a.x + (double)a.y * (double)a.y;
            double ore = 0.0, oim = 0.0;
            for (uint32_t t = t0; t < t1; ++t) {
              const BlockTerm bt = p.terms[t];
              const bool neg = (__popc(bt.yz & i) & 1u) != 0u;
              ore += neg ? -bt.cb_re : bt.cb_re;
              oim += neg ? -bt.cb_im : bt.cb_im;
            }
            acc.x += pr * ore;
            acc.y += pr * oim;
          }
        for (int g = 1; g < G; ++g) {
          const uint32_t F = p.group_flip[g], g0 = p.group_off[g], g1 = p.group_off[g + 1];
          const uint32_t pv = 31 - __clz(F);
          for (uint32_t k = lane; k < (D >> 1); k += LT) {
            const uint32_t lo = k & ((1u << pv) - 1u);
            const uint32_t i = ((k ^ lo) << 1) | lo, j = i ^ F;
            const A2 a = psi[block_slot(i)], bb = psi[block_slot(j)];
            // v = conj(a) b; both directions: cb s(i) (v + sigma conj(v))
            const double vre = (double)a.x * (double)bb.x + (double)a.y * (double)bb.y;
            const double vim = (double)a.x * (double)bb.y - (double)a.y * (double)bb.x;
            for (uint32_t t = g0; t < g1; ++t) {
              const BlockTerm bt = p.terms[t];
              const bool neg = (__popc(bt.yz & i) & 1u) != 0u;
              const bool sig = (__popc(bt.yz & F) & 1u) != 0u;
              // w = 2 Re(v) (sigma = +1) or 2i Im(v) (sigma = -1)
              const double wre = sig ? 0.0 : 2.0 * vre, wim = sig ? 2.0 * vim : 0.0;
              const double cre = bt.cb_re * wre - bt.cb_im * wim, cim = bt.cb_re * wim + bt.cb_im * wre;
              acc.x += neg ? -cre : cre;
              acc.y += neg ? -cim : cim;
            }
          }
        }
      }
      const double2 e = tm.sum(acc, scratch);
      if (lane == 0 && mine) {
        if (final_eval) e_self = e;
        else if (TEAMS) e_all[c] = e;
        else __stcg(&E[c], e);
      }
      BCLK(3);
    }
    if (final_eval) {
      if (blockIdx.x != 0) return;
      __syncthreads();
      if (tid == 0) {
        const double2 e = e_self;
        int st = 0;
        if (fabs(e.y) >= 1e-10) {
          st = kStatusImag;
          *p.err_val = e.y;
        } else if (!isfinite(e.x)) {
          st = kStatusNonFinite;
        }
        if (st) {
          *p.status = st;
          *p.err_iter = n_it;
        } else {
          p.traj[n_it] = e.x;
          *p.energy = e.x;
        }
      }
      break;
    }
    if (TEAMS) {
      __syncthreads();
    } else {
      arrivals += gridDim.x;
      if (!grid_barrier(p.barrier, arrivals)) {
        if (blockIdx.x == 0 && tid == 0) *p.status = kStatusAbort;
        return;
      }
      // the energies come in with one parallel L2 load per thread
      for (int c = tid; c < NC; c += nt) e_all[c] = __ldcg(&E[c]);
      __syncthreads();
    }
    BCLK(4);
    // every CTA: the iteration's checks, gradient, tolerance, Adam.  Warp 0
    // finds the first failing circuit (ballots, in circuit order) and the
    // gradient's infinity norm.
    if (tid < 32) {
      const double2 e0 = e_all[0];
      int st = 0;
      double ev = 0.0;
      if (fabs(e0.y) >= 1e-10) {
        st = kStatusImag;
        ev = e0.y;
      } else if (!isfinite(e0.x)) {
        st = kStatusNonFinite;
      } else {
        for (int cb0 = 1; cb0 < NC; cb0 += 32) {
          const int c = cb0 + tid;
          const double im = c < NC ? e_all[c].y : 0.0;
          const unsigned bad = __ballot_sync(0xffffffffu, fabs(im) >= 1e-10);
          if (bad) {
            st = kStatusImag;
            ev = e_all[cb0 + __ffs(bad) - 1].y;
            break;
          }
        }
      }
      double g_inf = 0.0;
      for (int k = tid; k < P; k += 32) g_inf = fmax(g_inf, fabs(0.5 * (e_all[2 * k + 1].x - e_all[2 * k + 2].x)));
      for (int o = 16; o > 0; o >>= 1) g_inf = fmax(g_inf, __shfl_xor_sync(0xffffffffu, g_inf, o));
      if (tid == 0) {
        if (blockIdx.x == 0) {
          if (st) {
            *p.status = st;
            *p.err_val = ev;
            *p.err_iter = iter;
          } else {
            p.traj[iter] = e0.x;
          }
        }
        stop_flag = st ? 2 : (p.has_tol && g_inf < p.tol) ? 1 : 0;
      }
    }
    __syncthreads();
    if (stop_flag == 2) {
      if (blockIdx.x == 0)
        for (int k = tid; k < P; k += nt) p.err_theta[k] = theta[k];
      return;
    }
    if (stop_flag == 1) {
      converged = 1;
      if (blockIdx.x == 0 && tid == 0) *p.energy = e_all[0].x;
      break;
    }
    BCLK(5);
    // adam_step (vqe.hpp:152-174), t = iter + 1
    const double bc1 = p.bc[2 * iter], bc2 = p.bc[2 * iter + 1];
    for (int k = tid; k < P; k += nt) {
      const double g = 0.5 * (e_all[2 * k + 1].x - e_all[2 * k + 2].x);
      const double mk = p.beta1 * mom[k] + (1.0 - p.beta1) * g;
      const double vk = p.beta2 * vel[k] + (1.0 - p.beta2) * g * g;
      const double m_hat = mk / bc1;
      const double v_hat = vk / bc2;
      theta[k] = theta[k] - p.lr * m_hat / (sqrt(v_hat) + p.eps);
      mom[k] = mk;
      vel[k] = vk;
    }
    iters = iter + 1;
    __syncthreads();
    BCLK(6);
#ifdef VQF_STAGE_CLOCKS
    if (blockIdx.x == 0 && tid == 0 && iter == 2)
      printf("BLOCK_STAGES n=%d teams=%d: sincos+init %lld passes %lld expect %lld exchange %lld checks %lld adam %lld total %lld\n",
             p.n, TEAMS ? 1 : 0, stamp[1] - stamp[0], stamp[2] - stamp[1], stamp[3] - stamp[2], stamp[4] - stamp[3],
             stamp[5] - stamp[4], stamp[6] - stamp[5], stamp[6] - stamp[0]);
#endif
  }
  if (blockIdx.x != 0) return;
  __syncthreads();
  for (int k = tid; k < P; k += nt) p.theta_out[k] = theta[k];
  if (tid == 0) {
    *p.iters = iters;
    *p.converged = converged;
    if (p.clk) p.clk[1] = global_ns();
  }
}

template <typename T, int R, bool TEAMS, int NB>
__global__ void __launch_bounds__(TEAMS ? kBlockThreads : kThreadsOf<R>)
    k_vqe_block(const __grid_constant__ BlockArgsN<NB> a) {
  BlockParams p = a.p;
  if (a.inl) {  // input pointers are offsets into the parameter block
    const auto at = [&](const void* off) { return a.blob + reinterpret_cast<size_t>(off); };
    p.bc = reinterpret_cast<const double*>(at(p.bc));
    p.passes = reinterpret_cast<const BlockPass*>(at(p.passes));
    p.group_flip = reinterpret_cast<const uint32_t*>(at(p.group_flip));
    p.group_off = reinterpret_cast<const uint32_t*>(at(p.group_off));
    p.terms = reinterpret_cast<const BlockTerm*>(at(p.terms));
    p.rterms = reinterpret_cast<const BlockRTerm*>(at(p.rterms));
    if (p.init_theta) p.init_theta = reinterpret_cast<const double*>(at(p.init_theta));
  }
  vqe_block_body<T, R, TEAMS>(p);
  if (!TEAMS) block_exit(p.barrier);
}

// ------------------------------------------------------------- host side
struct Frame {
  uint32_t n;
  std::vector<uint32_t> row;   // row[b]: physical mask whose parity is logical bit b (index bit b)
  std::vector<uint32_t> col;   // col[b]: M^-1 e_b (physical pair vector of logical bit b)
  uint32_t c = 0;
  explicit Frame(uint32_t n_) : n(n_), row(n_), col(n_) {
    for (uint32_t b = 0; b < n; ++b) row[b] = col[b] = 1u << b;
  }
  // CNOT(control bit a, target bit b) on the logical state: M' = C M, c' = C c
  void cnot(uint32_t a, uint32_t b) {
    row[b] ^= row[a];
    if ((c >> a) & 1u) c ^= 1u << b;
    col[a] ^= col[b];  // M'^-1 = M^-1 C
  }
  uint32_t map_flip(uint32_t f) const {  // M^-1 f
    uint32_t o = 0;
    for (uint32_t b = 0; b < n; ++b)
      if ((f >> b) & 1u) o ^= col[b];
    return o;
  }
  uint32_t map_yz(uint32_t yz) const {  // M^T yz
    uint32_t o = 0;
    for (uint32_t b = 0; b < n; ++b)
      if ((yz >> b) & 1u) o ^= row[b];
    return o;
  }
};

// Completes `vec` (independent) to R vectors with unit vectors and picks
// pivots (ascending) such that the span restricted to the pivots is
// bijective.
void finish_pass(BlockPass& bp, uint32_t n, int R) {
  std::vector<uint32_t> red;  // reduced basis, red[i] has pivot piv_i
  std::vector<uint32_t> pv;
  auto reduce = [&](uint32_t v) {
    for (size_t i = 0; i < red.size(); ++i)
      if ((v >> pv[i]) & 1u) v ^= red[i];
    return v;
  };
  // pivot = highest set bit of the reduced vector: thread bases then vary in
  // the low index bits (contiguous shared-memory slots)
  auto add = [&](uint32_t v) {
    const uint32_t w = reduce(v);
    if (w == 0) return false;
    const uint32_t pb = 31u - static_cast<uint32_t>(__builtin_clz(w));
    for (size_t i = 0; i < red.size(); ++i)
      if ((red[i] >> pb) & 1u) red[i] ^= w;
    red.push_back(w);
    pv.push_back(pb);
    return true;
  };
  const int real = bp.r;
  for (int j = 0; j < real; ++j)
    if (!add(bp.vec[j])) throw Error(VQF_LOGIC_ERROR, "block engine: dependent rotation vectors");
  // padding: x' = e_b ^ sum_j (row_j . e_b) vec_j is orthogonal to every
  // real row (row_i . vec_j = delta_ij), so a coset member's logical bits
  // change only with its real rotation bits
  for (uint32_t b = n; b-- > 0 && bp.r < R;) {
    uint32_t x = 1u << b;
    for (int j = 0; j < real; ++j)
      if ((bp.row[j] >> b) & 1u) x ^= bp.vec[j];
    if (add(x)) {
      bp.vec[bp.r] = x;
      bp.row[bp.r] = 0;
      bp.param[bp.r] = -1;
      ++bp.r;
    }
  }
  if (bp.r != R) throw Error(VQF_LOGIC_ERROR, "block engine: register narrower than a pass");
  std::sort(pv.begin(), pv.end());
  for (int j = 0; j < R; ++j) {
    bp.piv[j] = pv[j];
    bp.svec[j] = block_slot(bp.vec[j]);
  }
}

// Teams inside one CTA while 2P + 1 teams fit kTeamThreads threads (n <= 7
// for two HEA layers): R = n - 3 (1..3), so a team is 8 lanes (16 from
// 7 qubits) and the passes stay parallel across lanes.  Otherwise one CTA
// per circuit, R = 3 (R = 4 from 13 qubits: 16 amplitudes per thread).
constexpr uint32_t kTeamThreads = 512;
int team_bits(uint32_t n) { return static_cast<int>(std::min<uint32_t>(3u, std::max<uint32_t>(1u, n - 3))); }
bool use_teams(uint32_t n, uint32_t P) {
  if (n < 4 || n > 7) return false;
  const uint32_t lanes = (1u << n) >> team_bits(n), NC = 2 * P + 1;
  return ((NC * lanes + 31u) & ~31u) <= kTeamThreads;
}
int pass_bits(uint32_t n, bool teams) { return teams ? team_bits(n) : n >= 13 ? 4 : 3; }

}  // namespace

BlockProgram compile_block_program(int32_t kind, uint32_t layers, uint32_t n, const CompiledHam& h, int32_t dtype) {
  if (kind != VQF_ANSATZ_HARDWARE_EFFICIENT) throw_invalid("block engine: hardware-efficient ansatz only");
  if (n < (uint32_t)kBlockMinN || n > (uint32_t)block_max_n(dtype)) throw_invalid("block engine: register width");
  BlockProgram prog;
  prog.n = n;
  prog.gmem = n > static_cast<uint32_t>(block_smem_max_n(dtype));
  prog.teams = !prog.gmem && use_teams(n, layers * n);
  prog.R = static_cast<uint32_t>(pass_bits(n, prog.teams));
  Frame fr(n);
  const auto bit = [&](uint32_t q) { return n - 1 - q; };  // MSB-first (pauli.hpp:225-227)
  int32_t k = 0;
  for (uint32_t layer = 0; layer < layers; ++layer) {
    // RY(theta_k) on wires 0..n-1 (vqe.hpp:84-87): one frame, R per pass
    BlockPass cur{};
    for (uint32_t q = 0; q < n; ++q) {
      const uint32_t b = bit(q);
      cur.vec[cur.r] = fr.col[b];
      cur.row[cur.r] = fr.row[b];
      if ((fr.c >> b) & 1u) cur.cbits |= 1u << cur.r;
      cur.param[cur.r] = k++;
      if (++cur.r == (int32_t)prog.R) {
        finish_pass(cur, n, prog.R);
        prog.passes.push_back(cur);
        cur = BlockPass{};
      }
    }
    if (cur.r > 0) {
      finish_pass(cur, n, prog.R);
      prog.passes.push_back(cur);
    }
    // CNOT(q, q + 1) for q = 0..n-2 (vqe.hpp:88-90): frame only
    for (uint32_t q = 0; q + 1 < n; ++q) fr.cnot(bit(q), bit(q + 1));
  }
  // Hamiltonian in the final frame
  const size_t G = h.group_flip.size();
  prog.group_off.push_back(0);
  for (size_t g = 0; g < G; ++g) {
    prog.group_flip.push_back(fr.map_flip(static_cast<uint32_t>(h.group_flip[g])));
    for (uint32_t t = h.group_offset[g]; t < h.group_offset[g + 1]; ++t) {
      const MaskTerm& m = h.terms[t];
      const uint32_t yz = static_cast<uint32_t>(m.yz);
      const bool neg = (__builtin_popcount(yz & fr.c) & 1) != 0;
      prog.terms.push_back(BlockTerm{fr.map_yz(yz), 0u, neg ? -m.cb_re : m.cb_re, neg ? -m.cb_im : m.cb_im});
    }
    prog.group_off.push_back(static_cast<uint32_t>(prog.terms.size()));
  }
  if (G == 0) {  // no terms at all: an empty diagonal group
    prog.group_flip.push_back(0);
    prog.group_off.push_back(0);
  }
  prog.init_index = 0;
  // real form (BlockRTerm) when every coefficient allows it
  prog.herm = true;
  for (size_t g = 0; g + 1 < prog.group_off.size() && prog.herm; ++g) {
    const uint32_t F = prog.group_flip[g];
    for (uint32_t t = prog.group_off[g]; t < prog.group_off[g + 1]; ++t) {
      const BlockTerm& bt = prog.terms[t];
      const bool odd = (__builtin_popcount(bt.yz & F) & 1) != 0;  // odd Y count: cb purely imaginary
      if (odd ? bt.cb_re != 0.0 : bt.cb_im != 0.0) {
        prog.herm = false;
        break;
      }
      // w = 2 Re v (even) or 2 Im v (odd); cb w = cb_re 2 Re v, or (i cb_im)(2i Im v) = -cb_im 2 Im v
      prog.rterms.push_back(BlockRTerm{bt.yz, odd ? 1u : 0u, odd ? -bt.cb_im : bt.cb_re});
    }
  }
  if (!prog.herm) prog.rterms.clear();
  // diagonal operator table when it fits next to the state
  const uint32_t amp = dtype == VQF_F32 ? 8u : 16u;
  const uint32_t P = layers * n;
  const uint32_t T = static_cast<uint32_t>(prog.terms.size()), Gp = static_cast<uint32_t>(prog.group_flip.size());
  const uint32_t NC = 2 * P + 1;
  if (prog.teams) {
    prog.lanes = (1u << n) >> prog.R;
    prog.threads = (NC * prog.lanes + 31u) & ~31u;
    prog.slots = prog.threads / prog.lanes;
  } else {
    const uint32_t bases = (1u << n) >> prog.R;
    prog.lanes = std::min<uint32_t>(prog.R >= 4 ? 256u : static_cast<uint32_t>(kBlockThreads), std::max<uint32_t>(32u, bases));
    prog.threads = prog.lanes;
    prog.slots = 1;
  }
  const uint32_t Th = prog.herm ? T : 0u, Gh = prog.herm ? Gp : 0u;
  const uint32_t samp = prog.gmem ? 0u : amp;  // state bytes in shared memory
  if (BlockSmem(n, samp, P, 0, Th, Gh, prog.slots).total > kBlockSmemCap)
    throw_invalid("block engine: problem does not fit shared memory");
  prog.obytes = 0;
  if (prog.herm && prog.group_off[1] > prog.group_off[0])
    for (uint32_t ob : {8u, 4u})
      if (BlockSmem(n, samp, P, ob, Th, Gh, prog.slots).total <= kBlockSmemCap) {
        prog.obytes = ob;
        break;
      }
  return prog;
}

size_t block_smem_bytes(const BlockProgram& prog, int32_t dtype, int32_t P) {
  const uint32_t T = prog.herm ? static_cast<uint32_t>(prog.terms.size()) : 0u;
  const uint32_t G = prog.herm ? static_cast<uint32_t>(prog.group_flip.size()) : 0u;
  const uint32_t amp = prog.gmem ? 0u : dtype == VQF_F32 ? 8u : 16u;
  return BlockSmem(prog.n, amp, static_cast<uint32_t>(P), prog.obytes, T, G, prog.slots).total;
}

namespace {

using BlockKernel = const void*;

template <int NB>
BlockKernel pick_kernel(const BlockProgram& prog, bool f32) {
  if (prog.teams) {
    if (prog.R == 1) return f32 ? (BlockKernel)k_vqe_block<float, 1, true, NB> : (BlockKernel)k_vqe_block<double, 1, true, NB>;
    if (prog.R == 2) return f32 ? (BlockKernel)k_vqe_block<float, 2, true, NB> : (BlockKernel)k_vqe_block<double, 2, true, NB>;
    return f32 ? (BlockKernel)k_vqe_block<float, 3, true, NB> : (BlockKernel)k_vqe_block<double, 3, true, NB>;
  }
  if (prog.R == 4) return f32 ? (BlockKernel)k_vqe_block<float, 4, false, NB> : (BlockKernel)k_vqe_block<double, 4, false, NB>;
  return f32 ? (BlockKernel)k_vqe_block<float, 3, false, NB> : (BlockKernel)k_vqe_block<double, 3, false, NB>;
}

// The kernel instance for (storage type, R, launch shape, parameter block),
// with its dynamic shared memory limit raised once per device.
BlockKernel block_kernel(const BlockProgram& prog, int32_t dtype, bool small_args) {
  const bool f32 = dtype == VQF_F32;
  const BlockKernel k = small_args ? pick_kernel<kBlockInlineSmall>(prog, f32) : pick_kernel<kBlockInline>(prog, f32);
  static std::mutex mu;
  static std::vector<std::pair<int, BlockKernel>> done;
  int dev = 0;
  VQF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == dev && d.second == k) return k;
  VQF_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kBlockSmemCap));
  done.emplace_back(dev, k);
  return k;
}

// Co-resident CTAs for (kernel, threads, smem), cached: the occupancy query
// costs microseconds on a path that is itself tens of microseconds.
int max_grid(BlockKernel k, size_t smem, int threads, int device) {
  struct Key {
    BlockKernel k;
    int device, threads;
    size_t smem;
    int cap;
  };
  static std::mutex mu;
  static std::vector<Key> cache;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const Key& e : cache)
      if (e.k == k && e.device == device && e.threads == threads && e.smem == smem) return e.cap;
  }
  int per_sm = 0, sms = 0;
  VQF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem));
  VQF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  std::lock_guard<std::mutex> lock(mu);
  cache.push_back(Key{k, device, threads, smem, per_sm * sms});
  return per_sm * sms;
}

}  // namespace

int block_grid(const BlockProgram& prog, int32_t dtype, int NC, int device) {
  if (prog.teams) return 1;
  const size_t smem = block_smem_bytes(prog, dtype, NC / 2);
  const int cap = max_grid(block_kernel(prog, dtype, false), smem, static_cast<int>(prog.threads), device);
  if (cap < 1) throw Error(VQF_CUDA_ERROR, "block engine: kernel does not fit an SM");
  return std::min(cap, NC);
}

void launch_vqe_block(const BlockArgs& a, size_t used, const BlockProgram& prog, int grid, cudaStream_t stream) {
  const BlockParams& p = a.p;
  const size_t smem = block_smem_bytes(prog, p.dtype, p.P);
  const bool small_args = !a.inl || used <= static_cast<size_t>(kBlockInlineSmall);
  const BlockKernel k = block_kernel(prog, p.dtype, small_args);
  static thread_local BlockArgsN<kBlockInlineSmall> sa;
  void* kargs[1];
  if (small_args) {
    sa.p = a.p;
    sa.inl = a.inl;
    if (a.inl) std::memcpy(sa.blob, a.blob, used);
    kargs[0] = &sa;
  } else {
    kargs[0] = const_cast<BlockArgs*>(&a);
  }
  if (prog.teams) {  // one CTA: an ordinary launch is co-resident by construction
    VQF_CUDA(cudaLaunchKernel(k, dim3(1), dim3(prog.threads), kargs, smem, stream));
  } else {
    VQF_CUDA(cudaLaunchCooperativeKernel(k, dim3(grid), dim3(prog.threads), kargs, smem, stream));
  }
  VQF_LAUNCHED();
}

}  // namespace vqf
