// Register-resident batched VQE engine for small registers (n <= 5) and the
// fused H2 potential-energy-surface kernel.
//
// The reference evaluates each bond serially: per Adam iteration one energy
// plus 2P parameter-shifted energies, each a fresh heap-allocated
// StateVector (vqe.hpp:99-127, :226-243).  Here one CTA owns one problem
// (one bond) for its whole optimisation:
//   * every circuit of an iteration (base + 2P shifts) is simulated at once,
//     D = 2^n lanes per circuit, one amplitude per lane, gates as warp
//     shuffles (no memory traffic at all);
//   * expectation is a per-lane table lookup: the Hamiltonian is folded once
//     into per-flip-group tables O_g(i) = sum_t cb_t (-1)^popc(i & yz_t), and
//     <psi|H|psi> = sum_i sum_g O_g(i) conj(psi_i) psi_{i ^ f_g}, reduced by
//     an xor-butterfly (bitwise identical on every lane, placement
//     independent);
//   * Adam runs on device with host-computed bias-correction tables
//     (bitwise the reference's std::pow, vqe.hpp:161-162);
//   * in PES mode the CTA first builds its bond's Hamiltonian from scratch
//     (STO-3G integrals -> RHF -> Jordan-Wigner, chem.cuh), so a whole PES is
//     ONE launch with 800 bytes of input.
// The path is latency bound (a bond's state is 256 B); nothing here touches
// HBM beyond the outputs.
#include <cmath>

#include "chem.cuh"
#include "vqe_small.cuh"

namespace vqf {

namespace {

constexpr double kShift = 1.5707963267948966;  // std::numbers::pi / 2 (vqe.hpp:115)

__device__ __forceinline__ double2 shfl_xor2(double2 v, int m, int width) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m, width);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, m, width);
  return v;
}

// a' = c a - s b written as the reference does (complex * real, then
// subtract): statevector.hpp:160-163, :195-196.
__device__ __forceinline__ double2 rot_lo(double c, double s, double2 a, double2 b) {
  return make_double2(c * a.x - s * b.x, c * a.y - s * b.y);
}
__device__ __forceinline__ double2 rot_hi(double c, double s, double2 a, double2 b) {
  return make_double2(s * a.x + c * b.x, s * a.y + c * b.y);
}

// Circuit c's angle for parameter j (gradient(), vqe.hpp:118-123).
__device__ __forceinline__ double circuit_angle(const double* theta, int j, int c) {
  double t = theta[j];
  if (c == 2 * j + 1) t = t + kShift;
  if (c == 2 * j + 2) t = t - kShift;
  return t;
}

// prepare_ansatz (vqe.hpp:65-96) for one lane (amplitude index i) of a
// D-lane segment.  All lanes of the warp execute every shuffle.
__device__ double2 run_ansatz(int kind, int n, int layers, const double* theta, int c, int i) {
  const int D = 1 << n;
  double2 amp;
  if (kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION) {
    amp = make_double2(i == 12 ? 1.0 : 0.0, 0.0);  // basis_state(4, {1,1,0,0})
    double s, cc;
    sincos(0.5 * circuit_angle(theta, 0, c), &s, &cc);
    // DoubleExcitation(theta, 0, 1, 2, 3): sel = 1111, |1100> = 12 <-> |0011> = 3
    const double2 partner = shfl_xor2(amp, 15, D);
    if ((i & 15) == 12) amp = rot_lo(cc, s, amp, partner);
    else if ((i & 15) == 3) amp = rot_hi(cc, s, partner, amp);
    return amp;
  }
  amp = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
  int k = 0;
  for (int layer = 0; layer < layers; ++layer) {
    for (int q = 0; q < n; ++q) {
      const int bit = 1 << (n - 1 - q);
      double s, cc;
      sincos(0.5 * circuit_angle(theta, k++, c), &s, &cc);
      const double2 partner = shfl_xor2(amp, bit, D);
      amp = (i & bit) ? rot_hi(cc, s, partner, amp) : rot_lo(cc, s, amp, partner);
    }
    for (int q = 0; q + 1 < n; ++q) {
      const int cb = 1 << (n - 1 - q), tb = 1 << (n - 2 - q);
      const double2 partner = shfl_xor2(amp, tb, D);
      if (i & cb) amp = partner;
    }
  }
  return amp;
}

struct Shared {
  // Hamiltonian tables
  int n_groups;
  int flip[kSmallMaxD];
  double2 tab[kSmallMaxD * kSmallMaxD];  // [group][lane]
  // optimiser state
  double theta[kSmallMaxP], m[kSmallMaxP], v[kSmallMaxP], grad[kSmallMaxP];
  double2 energy[2 * kSmallMaxP + 1];
  int stop, converged, iters;
  // PES-mode scratch
  double prim[1296];
  chem::AoInts ints;
  chem::HfOut hf;
  double C[2][2];
  double mo[16];
  int ckey[chem::kNumContrib];
  double cre[chem::kNumContrib], cim[chem::kNumContrib];
  double kre[256], kim[256];
  int kseen[256];
  int keys[256];
  MaskTerm terms[256];
  int n_terms;
};

// Builds the per-group lane tables from n_terms mask terms in smem.
__device__ void build_tables(Shared& sh, int n) {
  const int D = 1 << n;
  if (threadIdx.x == 0) {
    int G = 0;
    sh.flip[G++] = 0;  // diagonal group first
    for (int t = 0; t < sh.n_terms; ++t) {
      const int f = static_cast<int>(sh.terms[t].flip);
      bool found = false;
      for (int g = 0; g < G; ++g) found |= (sh.flip[g] == f);
      if (!found) sh.flip[G++] = f;
    }
    sh.n_groups = G;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < sh.n_groups * D; idx += blockDim.x) {
    const int g = idx / D, i = idx % D;
    double re = 0.0, im = 0.0;
    for (int t = 0; t < sh.n_terms; ++t) {
      if (static_cast<int>(sh.terms[t].flip) != sh.flip[g]) continue;
      const bool odd = __popcll(static_cast<uint64_t>(i) & sh.terms[t].yz) & 1;
      re += odd ? -sh.terms[t].cb_re : sh.terms[t].cb_re;
      im += odd ? -sh.terms[t].cb_im : sh.terms[t].cb_im;
    }
    sh.tab[g * D + i] = make_double2(re, im);
  }
  __syncthreads();
}

__device__ __forceinline__ double2 lane_energy(const Shared& sh, double2 amp, int i, int D) {
  double2 acc = make_double2(0.0, 0.0);
  for (int g = 0; g < sh.n_groups; ++g) {
    const double2 p = shfl_xor2(amp, sh.flip[g], D);
    // v = conj(amp) * p
    const double vr = amp.x * p.x + amp.y * p.y, vi = amp.x * p.y - amp.y * p.x;
    const double2 o = sh.tab[g * D + i];
    acc.x += o.x * vr - o.y * vi;
    acc.y += o.x * vi + o.y * vr;
  }
  for (int o = D >> 1; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o, D);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o, D);
  }
  return acc;
}

// PES prologue: this CTA's H2 Hamiltonian, left as mask terms in smem.
// Returns a status (0 ok, kStatusScf, kStatusHermitian) in sh.stop.
__device__ void build_h2_device(Shared& sh, const chem::ChemConsts& k, double bond_angstrom, SmallParams& p,
                                int prob) {
  using namespace chem;
  const double d = bond_angstrom * kAngstromToBohr;
  for (int idx = threadIdx.x; idx < 1296; idx += blockDim.x) sh.prim[idx] = eri_term(k, d, idx);
  if (threadIdx.x < 4) one_electron(k, d, threadIdx.x >> 1, threadIdx.x & 1, sh.ints);
  __syncthreads();
  if (threadIdx.x < 16) {
    double s = 0.0;
    for (int r = 0; r < 81; ++r) s += sh.prim[threadIdx.x * 81 + r];
    sh.ints.eri[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    scf(sh.ints, d, sh.hf, sh.C);
    sh.stop = sh.hf.converged ? 0 : kStatusScf;
  }
  __syncthreads();
  if (sh.stop) return;
  if (threadIdx.x < 16) sh.mo[threadIdx.x] = mo_chem(sh.C, sh.ints.eri, threadIdx.x);
  __syncthreads();
  if (threadIdx.x < 16) {
    const int i = threadIdx.x >> 3, j = (threadIdx.x >> 2) & 1, kk = (threadIdx.x >> 1) & 1, l = threadIdx.x & 1;
    sh.hf.eri_mo[threadIdx.x] = sh.mo[((i * 2 + kk) * 2 + j) * 2 + l];  // <ij|kl> = (ik|jl)
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kNumContrib; idx += blockDim.x) {
    int key;
    double re, im;
    if (!jw_contribution(idx, sh.hf.hmo, sh.hf.eri_mo, sh.hf.e_nuc, key, re, im)) key = -1;
    sh.ckey[idx] = key;
    sh.cre[idx] = re;
    sh.cim[idx] = im;
  }
  __syncthreads();
  // Per-string sums in generation order (canonicalize's merge order).
  for (int key = threadIdx.x; key < 256; key += blockDim.x) {
    double re = 0.0, im = 0.0;
    int seen = 0;
    for (int idx = 0; idx < kNumContrib; ++idx) {
      if (sh.ckey[idx] != key) continue;
      if (!seen) {
        re = sh.cre[idx];
        im = sh.cim[idx];
        seen = 1;
      } else {
        re += sh.cre[idx];
        im += sh.cim[idx];
      }
    }
    sh.kre[key] = re;
    sh.kim[key] = im;
    sh.kseen[key] = seen;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // drop |c| < 1e-12, canonical sort, Hermiticity check (pauli.hpp:195-214)
    int* keys = sh.keys;
    int nk = 0;
    for (int key = 0; key < 256; ++key)
      if (sh.kseen[key] && hypot(sh.kre[key], sh.kim[key]) >= 1e-12) keys[nk++] = key;
    for (int a = 1; a < nk; ++a) {
      const int kk = keys[a];
      const uint32_t ok = key_order(kk);
      int b = a;
      while (b > 0 && key_order(keys[b - 1]) > ok) {
        keys[b] = keys[b - 1];
        --b;
      }
      keys[b] = kk;
    }
    sh.n_terms = 0;
    for (int a = 0; a < nk; ++a) {
      const int key = keys[a];
      if (fabs(sh.kim[key]) >= 1e-10) {
        sh.stop = kStatusHermitian;
        p.err_val[prob] = sh.kim[key];
        break;
      }
      const int x = key & 15, z = key >> 4;
      // MSB-first masks: qubit q -> bit (3 - q)
      uint64_t flip = 0, yz = 0;
      for (int q = 0; q < 4; ++q) {
        if ((x >> q) & 1) flip |= uint64_t{1} << (3 - q);
        if ((z >> q) & 1) yz |= uint64_t{1} << (3 - q);
      }
      const int n_y = __popc(x & z);
      const double c = sh.kre[key];  // imaginary part discarded (chem.hpp:465)
      MaskTerm t{flip, yz, 0.0, 0.0};
      switch (n_y & 3) {
        case 0: t.cb_re = c; break;
        case 1: t.cb_im = -c; break;
        case 2: t.cb_re = -c; break;
        default: t.cb_im = c; break;
      }
      sh.terms[sh.n_terms++] = t;
      if (p.ham_keys != nullptr) {
        p.ham_keys[prob * 16 + a] = key;
        p.ham_coeffs[prob * 16 + a] = c;
      }
    }
    if (p.ham_count != nullptr) p.ham_count[prob] = sh.stop ? 0 : sh.n_terms;
    if (p.hf_out != nullptr) {
      p.hf_out[4 * prob + 0] = sh.hf.hf_energy;
      p.hf_out[4 * prob + 1] = sh.hf.e_elec;
      p.hf_out[4 * prob + 2] = sh.hf.e_nuc;
      p.hf_out[4 * prob + 3] = sh.hf.scf_iterations;
    }
  }
  __syncthreads();
}

template <bool PES>
__global__ void __launch_bounds__(PES ? 256 : 1024) k_vqe_small(SmallParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
  const int prob = blockIdx.x;
  const int n = p.n_qubits, D = 1 << n, P = p.n_params, NC = 2 * P + 1;
  const int slot = threadIdx.x / D, lane = threadIdx.x % D, slots = blockDim.x / D;

  if (threadIdx.x == 0) {
    sh.stop = 0;
    sh.converged = 0;
    sh.iters = 0;
  }
  __syncthreads();
  if (PES) {
    if (p.status[prob] != 0) return;  // rejected on the host (bond out of range)
    build_h2_device(sh, p.chem, p.bonds[prob], p, prob);
    if (sh.stop) {
      if (threadIdx.x == 0) p.status[prob] = sh.stop;
      return;
    }
  } else {
    const uint32_t t0 = p.term_off[prob], t1 = p.term_off[prob + 1];
    for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) sh.terms[t - t0] = p.terms[t];
    if (threadIdx.x == 0) sh.n_terms = static_cast<int>(t1 - t0);
    __syncthreads();
  }
  build_tables(sh, n);
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    sh.theta[k] = p.init_theta ? p.init_theta[(size_t)prob * P + k] : 0.0;
    sh.m[k] = 0.0;
    sh.v[k] = 0.0;
  }
  __syncthreads();
  double* traj = p.traj + (size_t)prob * p.traj_stride;

  // Warps whose first circuit slot is past the last circuit skip the round
  // (warp-uniform, so the shuffles of active warps stay convergent).
  const int warp_first_slot = (threadIdx.x & ~31) / D;
  for (int iter = 0; iter < p.max_iterations; ++iter) {
    for (int c0 = 0; c0 < NC; c0 += slots) {
      if (c0 + warp_first_slot >= NC) continue;
      const int c = c0 + slot;
      const double2 amp = run_ansatz(p.ansatz_kind, n, p.layers, sh.theta, c < NC ? c : 0, lane);
      const double2 e = lane_energy(sh, amp, lane, D);
      if (lane == 0 && c < NC) sh.energy[c] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // checked_energy + gradient, in the reference's order (vqe.hpp:227-238)
      const double2 e = sh.energy[0];
      int st = 0;
      double val = 0.0;
      if (fabs(e.y) >= 1e-10) {
        st = kStatusImag;
        val = e.y;
      } else if (!isfinite(e.x)) {
        st = kStatusNonFinite;
      } else {
        for (int c = 1; c < NC && !st; ++c)
          if (fabs(sh.energy[c].y) >= 1e-10) {
            st = kStatusImag;
            val = sh.energy[c].y;
          }
      }
      if (st) {
        sh.stop = st;
        p.status[prob] = st;
        p.err_val[prob] = val;
        p.err_iter[prob] = iter;
        for (int k = 0; k < P; ++k) p.err_theta[(size_t)prob * P + k] = sh.theta[k];
      } else {
        traj[iter] = e.x;
        double g_inf = 0.0;
        for (int k = 0; k < P; ++k) {
          sh.grad[k] = 0.5 * (sh.energy[2 * k + 1].x - sh.energy[2 * k + 2].x);
          g_inf = fmax(g_inf, fabs(sh.grad[k]));
        }
        if (p.has_tol && g_inf < p.tol) {
          sh.stop = 1;
          sh.converged = 1;
        }
      }
    }
    __syncthreads();
    if (sh.stop) break;
    // adam_step (vqe.hpp:152-174) with t = iter + 1
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
      const double g = sh.grad[k];
      const double mk = p.beta1 * sh.m[k] + (1.0 - p.beta1) * g;
      const double vk = p.beta2 * sh.v[k] + (1.0 - p.beta2) * g * g;
      const double m_hat = mk / p.bc1[iter];
      const double v_hat = vk / p.bc2[iter];
      sh.theta[k] = sh.theta[k] - p.lr * m_hat / (sqrt(v_hat) + p.eps);
      sh.m[k] = mk;
      sh.v[k] = vk;
    }
    if (threadIdx.x == 0) sh.iters = iter + 1;
    __syncthreads();
  }

  if (sh.stop > 1) return;  // error recorded
  if (!sh.converged) {
    // final checked_energy (vqe.hpp:244-247)
    if (threadIdx.x < 32) {  // warp 0; every slot in it runs circuit 0
      const double2 amp = run_ansatz(p.ansatz_kind, n, p.layers, sh.theta, 0, lane);
      const double2 e = lane_energy(sh, amp, lane, D);
      if (threadIdx.x == 0) sh.energy[0] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double2 e = sh.energy[0];
      if (fabs(e.y) >= 1e-10) {
        p.status[prob] = kStatusImag;
        p.err_val[prob] = e.y;
        p.err_iter[prob] = p.max_iterations;
      } else if (!isfinite(e.x)) {
        p.status[prob] = kStatusNonFinite;
        p.err_iter[prob] = p.max_iterations;
        for (int k = 0; k < P; ++k) p.err_theta[(size_t)prob * P + k] = sh.theta[k];
      } else {
        traj[p.max_iterations] = e.x;
      }
    }
  }
  if (threadIdx.x == 0 && p.status[prob] == 0) {
    p.iters[prob] = sh.iters;
    p.converged[prob] = sh.converged;
    p.energy[prob] = traj[sh.converged ? sh.iters : p.max_iterations];
  }
  for (int k = threadIdx.x; k < P; k += blockDim.x) p.theta_out[(size_t)prob * P + k] = sh.theta[k];
  // NaN-pad the unused tail of a converged run's trajectory row
  const int len = sh.converged ? sh.iters + 1 : p.max_iterations + 1;
  for (int t = len + threadIdx.x; t < p.traj_stride; t += blockDim.x) traj[t] = __longlong_as_double(-1LL);
}

}  // namespace

size_t small_smem_bytes() { return sizeof(Shared); }

void launch_vqe_small(const SmallParams& p, uint32_t batch, bool pes, cudaStream_t stream) {
  const int D = 1 << p.n_qubits, NC = 2 * p.n_params + 1;
  int threads = ((NC * D + 31) / 32) * 32;
  if (threads > 1024) threads = 1024;
  if (pes) threads = 256;  // chemistry prologue uses 256; H2 needs 3 x 16 lanes
  const size_t smem = sizeof(Shared);
  if (pes) {
    VQF_CUDA(cudaFuncSetAttribute(k_vqe_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_vqe_small<true><<<batch, threads, smem, stream>>>(p);
  } else {
    VQF_CUDA(cudaFuncSetAttribute(k_vqe_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_vqe_small<false><<<batch, threads, smem, stream>>>(p);
  }
  VQF_LAUNCHED();
  VQF_CUDA(cudaGetLastError());
}

}  // namespace vqf
