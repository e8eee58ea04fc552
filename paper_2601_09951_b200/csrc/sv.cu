// State-vector kernels for sm_100a.  All are HBM-bandwidth bound (about
// 0.2 flop/B); the design goal is one coalesced 16-byte load and store per
// touched amplitude, several independent amplitude pairs in flight per
// thread, and deterministic reductions (no floating-point atomics) so that
// results do not depend on launch geometry or GPU count.
//
// Algorithmic bytes per launch (S = 2^n * sizeof(amp)):
//   X / RY / SingleExcitation-free 1q gates : 2S   (every amp read + written)
//   CNOT                                    : S    (control-1 half)
//   DoubleExcitation                        : S/4  (2^(n-3) amps touched)
//   SingleExcitation                        : S    (2^(n-1) amps touched)
//   expectation, per flip group             : S    (read once)
#include <algorithm>
#include <cstring>
#include <mutex>

#include "sv.cuh"
#include "tile.cuh"

namespace vqf {

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;
constexpr int kExpU = 8;  // loads in flight per thread in the expectation passes
constexpr int kRedBlocks = 4 * 148;  // reduction grid: 4 CTAs per SM (148 SMs)

template <typename T>
struct V2;
template <>
struct V2<double> {
  using type = double2;
};
template <>
struct V2<float> {
  using type = float2;
};

__device__ __forceinline__ uint64_t insert_zero(uint64_t k, uint32_t bit) {
  const uint64_t low = k & ((uint64_t{1} << bit) - 1);
  return ((k >> bit) << (bit + 1)) | low;
}

// Inserts zero bits at the (ascending) positions pos[0..m).
template <int M>
__device__ __forceinline__ uint64_t insert_zeros(uint64_t k, const uint32_t* pos) {
#pragma unroll
  for (int i = 0; i < M; ++i) k = insert_zero(k, pos[i]);
  return k;
}

template <typename T>
__device__ __forceinline__ void entry_cs(const GateArgs& g, uint64_t b, T& c, T& s) {
  if (g.cs != nullptr) {
    c = static_cast<T>(g.cs[2 * b]);
    s = static_cast<T>(g.cs[2 * b + 1]);
  } else {
    c = static_cast<T>(g.c);
    s = static_cast<T>(g.s);
  }
}

// ---------------------------------------------------- one-qubit gates
// X and RY on wire bit `bit`: statevector.hpp:150-166 (for_each_pair :124).
// Thread work item = one amplitude pair; kUnroll pairs per thread, strided
// by blockDim so each unrolled step is a fully coalesced warp access.
template <typename T, bool IS_X>
__global__ void __launch_bounds__(kThreads) k_gate1(typename V2<T>::type* __restrict__ a, uint32_t n, uint32_t bit,
                                                    uint64_t total_pairs, GateArgs g) {
  using A = typename V2<T>::type;
  const uint64_t half_log = n - 1;
  const uint64_t base = (uint64_t)blockIdx.x * (kThreads * kUnroll) + threadIdx.x;
  const uint64_t stride_bit = uint64_t{1} << bit;
  A x0[kUnroll], x1[kUnroll];
  uint64_t i0[kUnroll];
  bool ok[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint64_t p = base + (uint64_t)u * kThreads;
    ok[u] = p < total_pairs;
    const uint64_t b = p >> half_log, k = p & ((uint64_t{1} << half_log) - 1);
    i0[u] = (b << n) | insert_zero(k, bit);
    if (ok[u]) {
      x0[u] = a[i0[u]];
      x1[u] = a[i0[u] | stride_bit];
    }
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    if (!ok[u]) continue;
    if (IS_X) {
      a[i0[u]] = x1[u];
      a[i0[u] | stride_bit] = x0[u];
    } else {
      T c, s;
      entry_cs<T>(g, (base + (uint64_t)u * kThreads) >> half_log, c, s);
      A y0, y1;
      y0.x = c * x0[u].x - s * x1[u].x;
      y0.y = c * x0[u].y - s * x1[u].y;
      y1.x = s * x0[u].x + c * x1[u].x;
      y1.y = s * x0[u].y + c * x1[u].y;
      a[i0[u]] = y0;
      a[i0[u] | stride_bit] = y1;
    }
  }
}

// CNOT (statevector.hpp:167-178): only control=1 pairs are enumerated, so
// the kernel touches exactly half the state.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_cnot(typename V2<T>::type* __restrict__ a, uint32_t n, uint32_t pos_lo,
                                                   uint32_t pos_hi, uint64_t cbit, uint64_t tbit,
                                                   uint64_t total) {
  using A = typename V2<T>::type;
  const uint64_t qlog = n - 2;
  const uint64_t base = (uint64_t)blockIdx.x * (kThreads * kUnroll) + threadIdx.x;
  const uint32_t pos[2] = {pos_lo, pos_hi};
  A x0[kUnroll], x1[kUnroll];
  uint64_t i0[kUnroll];
  bool ok[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint64_t p = base + (uint64_t)u * kThreads;
    ok[u] = p < total;
    const uint64_t b = p >> qlog, k = p & ((uint64_t{1} << qlog) - 1);
    i0[u] = (b << n) | insert_zeros<2>(k, pos) | cbit;
    if (ok[u]) {
      x0[u] = a[i0[u]];
      x1[u] = a[i0[u] | tbit];
    }
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    if (!ok[u]) continue;
    a[i0[u]] = x1[u];
    a[i0[u] | tbit] = x0[u];
  }
}

// Givens rotation between the index patterns lo_pat and hi_pat of the
// wires in `pos` (M zero bits inserted).  DoubleExcitation
// (statevector.hpp:179-200): M = 4, |1100> (a) <-> |0011> (b);
// SingleExcitation: M = 2, |10> (a) <-> |01> (b).
//   a' = c a - s b,  b' = s a + c b
template <typename T, int M>
__global__ void __launch_bounds__(kThreads) k_givens(typename V2<T>::type* __restrict__ a, uint32_t n, GateArgs g,
                                                     uint64_t pat_a, uint64_t pat_b, uint64_t total,
                                                     uint32_t p0, uint32_t p1, uint32_t p2, uint32_t p3) {
  using A = typename V2<T>::type;
  const uint64_t qlog = n - M;
  const uint32_t pos[4] = {p0, p1, p2, p3};
  const uint64_t base = (uint64_t)blockIdx.x * (kThreads * kUnroll) + threadIdx.x;
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint64_t p = base + (uint64_t)u * kThreads;
    if (p >= total) continue;
    const uint64_t b = p >> qlog, k = p & ((uint64_t{1} << qlog) - 1);
    const uint64_t r = (b << n) | insert_zeros<M>(k, pos);
    const A x = a[r | pat_a], y = a[r | pat_b];
    T c, s;
    entry_cs<T>(g, b, c, s);
    A xa, yb;
    xa.x = c * x.x - s * y.x;
    xa.y = c * x.y - s * y.y;
    yb.x = s * x.x + c * y.x;
    yb.y = s * x.y + c * y.y;
    a[r | pat_a] = xa;
    a[r | pat_b] = yb;
  }
}

template <typename T>
__global__ void k_set_basis(typename V2<T>::type* a, uint32_t n, uint32_t batch, uint64_t index) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) {
    typename V2<T>::type one;
    one.x = T(1);
    one.y = T(0);
    a[((uint64_t)b << n) | index] = one;
  }
}

// ------------------------------------------------------- reductions
__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Block-wide deterministic sum; result valid in thread 0.
__device__ __forceinline__ double2 block_sum(double2 v) {
  __shared__ double2 sh[kThreads / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < kThreads / 32 ? sh[l] : make_double2(0.0, 0.0);
    v = warp_sum(v);
  }
  __syncthreads();
  return v;
}

__device__ __forceinline__ double parity_sign(uint64_t x) { return (__popcll(x) & 1) ? -1.0 : 1.0; }

// Diagonal group: sum_i |psi_i|^2 * sum_t cb_t (-1)^popc(i & yz_t)
// (statevector.hpp:227-234, all diagonal terms fused into one pass).
// grid = (blocks, batch); partials[(entry * G + group) * blocks + block].
template <typename T>
__global__ void __launch_bounds__(kThreads) k_expect_diag(const typename V2<T>::type* __restrict__ a, uint32_t n,
                                                          const MaskTerm* __restrict__ terms, uint32_t n_terms,
                                                          double* __restrict__ partials, uint32_t G, uint32_t group) {
  __shared__ MaskTerm st[64];
  const uint32_t b = blockIdx.y;
  const uint64_t D = uint64_t{1} << n;
  const typename V2<T>::type* s = a + ((uint64_t)b << n);
  double2 acc = make_double2(0.0, 0.0);
  for (uint32_t t0 = 0; t0 < n_terms; t0 += 64) {
    const uint32_t cnt = min(64u, n_terms - t0);
    __syncthreads();
    if (threadIdx.x < cnt) st[threadIdx.x] = terms[t0 + threadIdx.x];
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < D; i += (uint64_t)gridDim.x * kThreads) {
      const typename V2<T>::type x = s[i];
      const double p = (double)x.x * (double)x.x + (double)x.y * (double)x.y;
      double dre = 0.0, dim = 0.0;
      for (uint32_t t = 0; t < cnt; ++t) {
        const double sg = parity_sign(i & st[t].yz);
        dre += sg * st[t].cb_re;
        dim += sg * st[t].cb_im;
      }
      acc.x += p * dre;
      acc.y += p * dim;
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    const size_t o = ((size_t)b * G + group) * gridDim.x + blockIdx.x;
    partials[2 * o] = acc.x;
    partials[2 * o + 1] = acc.y;
  }
}

// Diagonal group, tiled: the index splits as i = (hi << B) | lo over tiles of
// 2^B contiguous amplitudes, and every Z-string sign factorises as
// (-1)^popc(i & yz) = (-1)^popc(lo & yz_lo) * (-1)^popc(hi & yz_hi).
//   * terms with yz_hi = 0 fold into a per-CTA table L[lo] (built once);
//   * terms with yz_lo = 0 fold into one scalar per tile;
//   * mixed terms stay a per-amplitude loop.
// Per amplitude: one L lookup (shared memory), two adds, |psi|^2 * D, with
// kExpU loads in flight per thread — the pass is HBM-bound instead of
// looping over every Z term per amplitude.
// grid = (blocks, batch); dynamic smem = 2^B double2.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_expect_diag_tiled(
    const typename V2<T>::type* __restrict__ a, uint32_t n, uint32_t B, const MaskTerm* __restrict__ lo_t,
    uint32_t n_lo, const MaskTerm* __restrict__ hi_t, uint32_t n_hi, const MaskTerm* __restrict__ mx_t,
    uint32_t n_mx, double* __restrict__ partials, uint32_t G) {
  extern __shared__ double2 Ltab[];
  __shared__ MaskTerm mx[64];
  const uint32_t b = blockIdx.y;
  const uint32_t tile_amps = 1u << B;
  const uint64_t n_tiles = uint64_t{1} << (n - B);
  const typename V2<T>::type* s = a + ((uint64_t)b << n);
  for (uint32_t lo = threadIdx.x; lo < tile_amps; lo += kThreads) {
    double re = 0.0, im = 0.0;
    for (uint32_t t = 0; t < n_lo; ++t) {
      const double sg = parity_sign(lo & lo_t[t].yz);
      re += sg * lo_t[t].cb_re;
      im += sg * lo_t[t].cb_im;
    }
    Ltab[lo] = make_double2(re, im);
  }
  if (threadIdx.x < n_mx) mx[threadIdx.x] = mx_t[threadIdx.x];
  __syncthreads();
  double2 acc = make_double2(0.0, 0.0);
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    double hre = 0.0, him = 0.0;  // warp-uniform per tile
    for (uint32_t t = 0; t < n_hi; ++t) {
      const double sg = parity_sign(tile & (hi_t[t].yz >> B));
      hre += sg * hi_t[t].cb_re;
      him += sg * hi_t[t].cb_im;
    }
    const uint64_t base = tile << B;
    for (uint32_t lo0 = threadIdx.x; lo0 < tile_amps; lo0 += kThreads * kExpU) {
      typename V2<T>::type x[kExpU];
#pragma unroll
      for (int u = 0; u < kExpU; ++u) {
        const uint32_t lo = lo0 + u * kThreads;
        if (lo < tile_amps) x[u] = s[base | lo];
      }
#pragma unroll
      for (int u = 0; u < kExpU; ++u) {
        const uint32_t lo = lo0 + u * kThreads;
        if (lo >= tile_amps) break;
        const uint64_t i = base | lo;
        const double p = (double)x[u].x * (double)x[u].x + (double)x[u].y * (double)x[u].y;
        const double2 l = Ltab[lo];
        double dre = l.x + hre, dim = l.y + him;
        for (uint32_t t = 0; t < n_mx; ++t) {
          const double sg = parity_sign(i & mx[t].yz);
          dre += sg * mx[t].cb_re;
          dim += sg * mx[t].cb_im;
        }
        acc.x += p * dre;
        acc.y += p * dim;
      }
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    const size_t o = ((size_t)b * G + 0) * gridDim.x + blockIdx.x;
    partials[2 * o] = acc.x;
    partials[2 * o + 1] = acc.y;
  }
}

// Cross term between two states a, b of one register:
//   sum_t cb_t sum_i (-1)^popc(i & yz_t) conj(a_i) b_{i ^ flip_t}
// (the shard-pair contribution of a Pauli term that flips global wires of a
// distributed state, paper_2601_09951_b200/dsv.py).  Terms in shared memory,
// per-block partials, fixed-order final sum.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_expect_cross(const typename V2<T>::type* __restrict__ a,
                                                           const typename V2<T>::type* __restrict__ bvec, uint32_t n,
                                                           const MaskTerm* __restrict__ terms, uint32_t n_terms,
                                                           double* __restrict__ partials) {
  __shared__ MaskTerm st[64];
  const uint64_t D = uint64_t{1} << n;
  double2 acc = make_double2(0.0, 0.0);
  for (uint32_t t0 = 0; t0 < n_terms; t0 += 64) {
    const uint32_t cnt = min(64u, n_terms - t0);
    __syncthreads();
    if (threadIdx.x < cnt) st[threadIdx.x] = terms[t0 + threadIdx.x];
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < D; i += (uint64_t)gridDim.x * kThreads) {
      const typename V2<T>::type x = a[i];
      for (uint32_t t = 0; t < cnt; ++t) {
        const typename V2<T>::type y = bvec[i ^ st[t].flip];
        const double vr = (double)x.x * (double)y.x + (double)x.y * (double)y.y;
        const double vi = (double)x.x * (double)y.y - (double)x.y * (double)y.x;
        const double sg = parity_sign(i & st[t].yz);
        acc.x += sg * (st[t].cb_re * vr - st[t].cb_im * vi);
        acc.y += sg * (st[t].cb_re * vi + st[t].cb_im * vr);
      }
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = acc.x;
    partials[2 * blockIdx.x + 1] = acc.y;
  }
}

// Off-diagonal group with flip mask f (statevector.hpp:235-241): each pair
// (i, j = i ^ f), i with f's top bit clear, is read once.  With
// v = conj(psi_i) psi_j and sigma_t = (-1)^popc(f & yz_t), the two
// contributions of a term are cb_t s_t(i) (v + sigma_t conj(v)), i.e.
// 2 Re(v) for sigma = +1 and 2i Im(v) for sigma = -1.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_expect_flip(const typename V2<T>::type* __restrict__ a, uint32_t n,
                                                          uint64_t flip, uint32_t hb,
                                                          const MaskTerm* __restrict__ terms, uint32_t n_terms,
                                                          double* __restrict__ partials, uint32_t G, uint32_t group) {
  __shared__ MaskTerm st[64];
  __shared__ double sig[64];
  const uint32_t b = blockIdx.y;
  const uint64_t half = uint64_t{1} << (n - 1);
  const typename V2<T>::type* s = a + ((uint64_t)b << n);
  double2 acc = make_double2(0.0, 0.0);
  for (uint32_t t0 = 0; t0 < n_terms; t0 += 64) {
    const uint32_t cnt = min(64u, n_terms - t0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      st[threadIdx.x] = terms[t0 + threadIdx.x];
      sig[threadIdx.x] = parity_sign(flip & st[threadIdx.x].yz);
    }
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    for (uint64_t k0 = (uint64_t)blockIdx.x * kThreads + threadIdx.x; k0 < half; k0 += stride * kExpU) {
      typename V2<T>::type x[kExpU], y[kExpU];
      uint64_t idx[kExpU];
#pragma unroll
      for (int u = 0; u < kExpU; ++u) {  // pairs in flight before arithmetic
        const uint64_t k = k0 + u * stride;
        idx[u] = insert_zero(k, hb);
        if (k < half) {
          x[u] = s[idx[u]];
          y[u] = s[idx[u] ^ flip];
        }
      }
#pragma unroll
      for (int u = 0; u < kExpU; ++u) {
        if (k0 + u * stride >= half) break;
        const uint64_t i = idx[u];
        // v = conj(x) * y
        const double vr = (double)x[u].x * (double)y[u].x + (double)x[u].y * (double)y[u].y;
        const double vi = (double)x[u].x * (double)y[u].y - (double)x[u].y * (double)y[u].x;
        double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
        for (uint32_t t = 0; t < cnt; ++t) {
          const double sg = parity_sign(i & st[t].yz);
          if (sig[t] > 0.0) {
            ar += sg * st[t].cb_re;
            ai += sg * st[t].cb_im;
          } else {
            br += sg * st[t].cb_re;
            bi += sg * st[t].cb_im;
          }
        }
        // A * (2 vr) + B * (2i vi)
        acc.x += 2.0 * (ar * vr - bi * vi);
        acc.y += 2.0 * (ai * vr + br * vi);
      }
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    const size_t o = ((size_t)b * G + group) * gridDim.x + blockIdx.x;
    partials[2 * o] = acc.x;
    partials[2 * o + 1] = acc.y;
  }
}

// Fixed-order final sum per entry: groups in order, blocks in order within
// a group, as a block tree over contiguous partials.
__global__ void __launch_bounds__(kThreads) k_final_sum(const double* __restrict__ partials, uint32_t per_entry,
                                                        double* __restrict__ out) {
  const uint32_t b = blockIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  for (uint32_t j = threadIdx.x; j < per_entry; j += kThreads) {
    acc.x += partials[2 * ((size_t)b * per_entry + j)];
    acc.y += partials[2 * ((size_t)b * per_entry + j) + 1];
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    out[2 * b] = acc.x;
    out[2 * b + 1] = acc.y;
  }
}

uint32_t red_blocks(uint64_t work_items) {
  const uint64_t need = (work_items + kThreads - 1) / kThreads;
  return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(need, kRedBlocks)));
}

template <typename T>
void apply_t(vqf_statevector* sv, const GateArgs& g) {
  using A = typename V2<T>::type;
  A* a = static_cast<A*>(sv->amps);
  const uint32_t n = sv->n_qubits;
  const uint64_t batch = sv->batch;
  const auto bit_of = [n](uint32_t w) { return n - 1 - w; };
  const auto grid_for = [](uint64_t items) {
    return static_cast<unsigned>((items + kThreads * kUnroll - 1) / (kThreads * kUnroll));
  };
  switch (g.kind) {
    case VQF_GATE_PAULI_X:
    case VQF_GATE_RY: {
      const uint64_t total = batch << (n - 1);
      if (g.kind == VQF_GATE_PAULI_X)
        k_gate1<T, true><<<grid_for(total), kThreads, 0, sv->stream>>>(a, n, bit_of(g.wires[0]), total, g);
      else
        k_gate1<T, false><<<grid_for(total), kThreads, 0, sv->stream>>>(a, n, bit_of(g.wires[0]), total, g);
      break;
    }
    case VQF_GATE_CNOT: {
      const uint32_t bc = bit_of(g.wires[0]), bt = bit_of(g.wires[1]);
      const uint64_t total = batch << (n - 2);
      k_cnot<T><<<grid_for(total), kThreads, 0, sv->stream>>>(a, n, std::min(bc, bt), std::max(bc, bt),
                                                               uint64_t{1} << bc, uint64_t{1} << bt, total);
      break;
    }
    case VQF_GATE_DOUBLE_EXCITATION: {
      uint32_t pos[4];
      uint64_t m[4];
      for (int i = 0; i < 4; ++i) {
        pos[i] = bit_of(g.wires[i]);
        m[i] = uint64_t{1} << pos[i];
      }
      std::sort(pos, pos + 4);
      const uint64_t total = batch << (n - 4);
      k_givens<T, 4><<<grid_for(total), kThreads, 0, sv->stream>>>(a, n, g, m[0] | m[1], m[2] | m[3], total,
                                                                   pos[0], pos[1], pos[2], pos[3]);
      break;
    }
    case VQF_GATE_SINGLE_EXCITATION: {
      uint32_t pos[2] = {bit_of(g.wires[0]), bit_of(g.wires[1])};
      const uint64_t m0 = uint64_t{1} << pos[0], m1 = uint64_t{1} << pos[1];
      std::sort(pos, pos + 2);
      const uint64_t total = batch << (n - 2);
      k_givens<T, 2><<<grid_for(total), kThreads, 0, sv->stream>>>(a, n, g, m0, m1, total, pos[0], pos[1], 0, 0);
      break;
    }
    default:
      throw Error(VQF_LOGIC_ERROR, "unknown gate kind");
  }
  VQF_LAUNCHED();
  VQF_CUDA(cudaGetLastError());
}

void ensure_partials(vqf_statevector* sv, size_t doubles) {
  if (sv->partial_cap >= doubles) return;
  VQF_CUDA(cudaSetDevice(sv->device));
  if (sv->partials) VQF_CUDA(cudaFree(sv->partials));
  VQF_CUDA(cudaMalloc(&sv->partials, doubles * sizeof(double)));
  sv->partial_cap = doubles;
}

void ensure_terms(vqf_statevector* sv, size_t bytes) {
  if (sv->terms_cap >= bytes) return;
  if (sv->terms_dev) VQF_CUDA(cudaFree(sv->terms_dev));
  VQF_CUDA(cudaMalloc(&sv->terms_dev, bytes));
  sv->terms_cap = bytes;
}

template <typename T>
void expectation_t(vqf_statevector* sv, const CompiledHam& h, double* dev_out) {
  using A = typename V2<T>::type;
  const A* a = static_cast<const A*>(sv->amps);
  const uint32_t n = sv->n_qubits;
  const uint32_t G = static_cast<uint32_t>(h.group_flip.size());
  const uint32_t nb_diag = red_blocks(uint64_t{1} << n);
  const uint32_t nb_flip = n >= 1 ? red_blocks(uint64_t{1} << (n - 1)) : 1;
  const uint32_t nb = std::max(nb_diag, nb_flip);
  ensure_partials(sv, 2 * (size_t)sv->batch * G * nb);
  VQF_CUDA(cudaMemsetAsync(sv->partials, 0, 2 * sizeof(double) * sv->batch * G * nb, sv->stream));
  // Diagonal group split for the tiled kernel (k_expect_diag_tiled): terms
  // whose Z/Y support is all below / all above the tile width, and mixed.
  const uint32_t B = std::min<uint32_t>(n, 11);  // 2048-amplitude tiles, 32 KB table
  const uint64_t lo_mask = (uint64_t{1} << B) - 1;
  std::vector<MaskTerm> all = h.terms, lo, hi, mx;
  for (uint32_t t = h.group_offset[0]; t < h.group_offset[1]; ++t) {
    const MaskTerm& m = h.terms[t];
    if ((m.yz & ~lo_mask) == 0) lo.push_back(m);
    else if ((m.yz & lo_mask) == 0) hi.push_back(m);
    else mx.push_back(m);
  }
  const bool tiled = mx.size() <= 64;
  const uint32_t o_lo = static_cast<uint32_t>(all.size());
  all.insert(all.end(), lo.begin(), lo.end());
  const uint32_t o_hi = static_cast<uint32_t>(all.size());
  all.insert(all.end(), hi.begin(), hi.end());
  const uint32_t o_mx = static_cast<uint32_t>(all.size());
  all.insert(all.end(), mx.begin(), mx.end());
  ensure_terms(sv, std::max<size_t>(1, all.size()) * sizeof(MaskTerm));
  if (!all.empty())
    VQF_CUDA(cudaMemcpyAsync(sv->terms_dev, all.data(), all.size() * sizeof(MaskTerm), cudaMemcpyHostToDevice,
                             sv->stream));
  const MaskTerm* td = static_cast<const MaskTerm*>(sv->terms_dev);
  for (uint32_t g = 0; g < G; ++g) {
    const uint32_t t0 = h.group_offset[g], cnt = h.group_offset[g + 1] - t0;
    if (cnt == 0) continue;
    if (g == 0 && tiled) {
      k_expect_diag_tiled<T><<<dim3(nb, sv->batch), kThreads, sizeof(double2) << B, sv->stream>>>(
          a, n, B, td + o_lo, static_cast<uint32_t>(lo.size()), td + o_hi, static_cast<uint32_t>(hi.size()),
          td + o_mx, static_cast<uint32_t>(mx.size()), sv->partials, G);
    } else if (g == 0) {
      k_expect_diag<T><<<dim3(nb, sv->batch), kThreads, 0, sv->stream>>>(a, n, td + t0, cnt, sv->partials, G, 0);
    } else {
      const uint64_t f = h.group_flip[g];
      const uint32_t hb = 63 - __builtin_clzll(f);
      k_expect_flip<T><<<dim3(nb, sv->batch), kThreads, 0, sv->stream>>>(a, n, f, hb, td + t0, cnt, sv->partials,
                                                                         G, g);
    }
    VQF_LAUNCHED();
  }
  k_final_sum<<<sv->batch, kThreads, 0, sv->stream>>>(sv->partials, G * nb, dev_out);
  VQF_LAUNCHED();
  VQF_CUDA(cudaGetLastError());
}

}  // namespace

void sv_check_gate(const vqf_statevector* sv, const vqf_gate& g) {
  // statevector.hpp:105-120 check_wires
  uint32_t expected = 0;
  switch (g.kind) {
    case VQF_GATE_PAULI_X:
    case VQF_GATE_RY: expected = 1; break;
    case VQF_GATE_CNOT:
    case VQF_GATE_SINGLE_EXCITATION: expected = 2; break;
    case VQF_GATE_DOUBLE_EXCITATION: expected = 4; break;
    default: throw Error(VQF_LOGIC_ERROR, "unknown gate kind");
  }
  if (g.n_wires != expected) throw_invalid("gate wire count mismatch");
  for (uint32_t i = 0; i < g.n_wires; ++i) {
    if (g.wires[i] >= sv->n_qubits) throw_invalid("gate wire exceeds register size");
    for (uint32_t j = i + 1; j < g.n_wires; ++j)
      if (g.wires[i] == g.wires[j]) throw_invalid("duplicate gate wire");
  }
}

void sv_apply(vqf_statevector* sv, const GateArgs& g) {
  if (sv->dtype == VQF_F64)
    apply_t<double>(sv, g);
  else
    apply_t<float>(sv, g);
}

void sv_reset(vqf_statevector* sv, uint64_t basis_index) {
  VQF_CUDA(cudaMemsetAsync(sv->amps, 0, sv->amp_bytes() * sv->dim() * sv->batch, sv->stream));
  const unsigned blocks = (sv->batch + 127) / 128;
  if (sv->dtype == VQF_F64)
    k_set_basis<double><<<blocks, 128, 0, sv->stream>>>(static_cast<double2*>(sv->amps), sv->n_qubits, sv->batch,
                                                       basis_index);
  else
    k_set_basis<float><<<blocks, 128, 0, sv->stream>>>(static_cast<float2*>(sv->amps), sv->n_qubits, sv->batch,
                                                      basis_index);
  VQF_LAUNCHED();
  VQF_CUDA(cudaGetLastError());
}

void sv_expectation_async(vqf_statevector* sv, const CompiledHam& h, double* dev_out) {
  if (sv->dtype == VQF_F64)
    expectation_t<double>(sv, h, dev_out);
  else
    expectation_t<float>(sv, h, dev_out);
}

void sv_expectation(vqf_statevector* sv, const CompiledHam& h, double* out) {
  sv_expectation_async(sv, h, sv->dev_out);
  VQF_CUDA(cudaMemcpyAsync(sv->host_out, sv->dev_out, 2 * sizeof(double) * sv->batch, cudaMemcpyDeviceToHost,
                           sv->stream));
  VQF_CUDA(cudaStreamSynchronize(sv->stream));
  std::memcpy(out, sv->host_out, 2 * sizeof(double) * sv->batch);
}

void sv_norms(vqf_statevector* sv, double* out) {
  CompiledHam id;
  id.n_qubits = sv->n_qubits;
  id.group_flip = {0};
  id.group_offset = {0, 1};
  id.terms = {MaskTerm{0, 0, 1.0, 0.0}};
  std::vector<double> tmp(2 * sv->batch);
  sv_expectation(sv, id, tmp.data());
  for (uint32_t b = 0; b < sv->batch; ++b) out[b] = std::sqrt(tmp[2 * b]);
}

void retain_pool(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lock(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return;
  cudaMemPool_t pool;
  VQF_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t threshold = UINT64_MAX;
  VQF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  done.push_back(device);
}

void sv_ensure_cs(vqf_statevector* sv, size_t n_doubles) {
  if (sv->cs_cap >= n_doubles) return;
  if (sv->cs_dev) VQF_CUDA(cudaFree(sv->cs_dev));
  VQF_CUDA(cudaMalloc(&sv->cs_dev, n_doubles * sizeof(double)));
  sv->cs_cap = n_doubles;
}

}  // namespace vqf

using namespace vqf;

extern "C" {

int vqf_sv_create(uint32_t n_qubits, uint32_t batch, int32_t dtype, int32_t device, vqf_sv* out) {
  return guarded([&] {
    if (out == nullptr) throw_invalid("null output handle");
    if (n_qubits < 1 || n_qubits > 36) throw_invalid("state vector: n_qubits must be in [1, 36]");
    if (batch < 1) throw_invalid("state vector: batch must be >= 1");
    if (dtype != VQF_F64 && dtype != VQF_F32) throw_invalid("state vector: unknown dtype");
    auto* sv = new vqf_statevector();
    sv->n_qubits = n_qubits;
    sv->batch = batch;
    sv->dtype = dtype;
    sv->device = device;
    try {
      VQF_CUDA(cudaSetDevice(device));
      VQF_CUDA(cudaStreamCreateWithFlags(&sv->own_stream, cudaStreamNonBlocking));
      sv->stream = sv->own_stream;
      // stream-ordered allocation from the device pool, whose release
      // threshold is raised once per device so freed states stay mapped and
      // repeated calls (VQE iterations, scaling widths) reuse HBM instead of
      // paying cudaMalloc page-mapping costs
      retain_pool(device);
      VQF_CUDA(cudaMallocAsync(&sv->amps, sv->amp_bytes() * sv->dim() * batch, sv->stream));
      VQF_CUDA(cudaMallocHost(&sv->host_out, 2 * sizeof(double) * batch));
      VQF_CUDA(cudaMalloc(&sv->dev_out, 2 * sizeof(double) * batch));
      sv_reset(sv, 0);
      VQF_CUDA(cudaStreamSynchronize(sv->stream));
    } catch (...) {
      vqf_sv_destroy(sv);
      throw;
    }
    *out = sv;
  });
}

int vqf_sv_destroy(vqf_sv sv) {
  return guarded([&] {
    if (sv == nullptr) return;
    cudaSetDevice(sv->device);
    if (sv->stream) cudaStreamSynchronize(sv->stream);
    if (sv->own_stream && sv->own_stream != sv->stream) cudaStreamSynchronize(sv->own_stream);
    if (sv->amps) {  // freed on the handle's own stream (a caller stream may be gone)
      cudaFreeAsync(sv->amps, sv->own_stream);
      cudaStreamSynchronize(sv->own_stream);
    }
    if (sv->partials) cudaFree(sv->partials);
    if (sv->terms_dev) cudaFree(sv->terms_dev);
    if (sv->cs_dev) cudaFree(sv->cs_dev);
    if (sv->host_out) cudaFreeHost(sv->host_out);
    if (sv->dev_out) cudaFree(sv->dev_out);
    if (sv->own_stream) cudaStreamDestroy(sv->own_stream);
    delete sv;
  });
}

int vqf_sv_info(vqf_sv sv, uint32_t* n_qubits, uint32_t* batch, int32_t* dtype, int32_t* device) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    if (n_qubits) *n_qubits = sv->n_qubits;
    if (batch) *batch = sv->batch;
    if (dtype) *dtype = sv->dtype;
    if (device) *device = sv->device;
  });
}

int vqf_sv_set_stream(vqf_sv sv, void* cuda_stream) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    VQF_CUDA(cudaSetDevice(sv->device));
    VQF_CUDA(cudaStreamSynchronize(sv->stream));
    sv->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : sv->own_stream;
  });
}

int vqf_sv_reset(vqf_sv sv) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    VQF_CUDA(cudaSetDevice(sv->device));
    sv_reset(sv, 0);
    VQF_CUDA(cudaStreamSynchronize(sv->stream));
  });
}

int vqf_sv_set_basis_state(vqf_sv sv, const int32_t* bits, uint32_t n_bits) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    if (n_bits != sv->n_qubits) throw_invalid("basis_state: bit count != qubit count");
    uint64_t index = 0;
    for (uint32_t q = 0; q < sv->n_qubits; ++q)
      if (bits[q]) index |= qubit_bit(sv->n_qubits, q);
    VQF_CUDA(cudaSetDevice(sv->device));
    sv_reset(sv, index);
    VQF_CUDA(cudaStreamSynchronize(sv->stream));
  });
}

int vqf_sv_upload(vqf_sv sv, const double* amps) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    VQF_CUDA(cudaSetDevice(sv->device));
    const size_t count = sv->dim() * sv->batch;
    if (sv->dtype == VQF_F64) {
      VQF_CUDA(cudaMemcpyAsync(sv->amps, amps, count * 16, cudaMemcpyHostToDevice, sv->stream));
    } else {
      std::vector<float> tmp(2 * count);
      for (size_t i = 0; i < 2 * count; ++i) tmp[i] = static_cast<float>(amps[i]);
      VQF_CUDA(cudaMemcpyAsync(sv->amps, tmp.data(), count * 8, cudaMemcpyHostToDevice, sv->stream));
      VQF_CUDA(cudaStreamSynchronize(sv->stream));
    }
    VQF_CUDA(cudaStreamSynchronize(sv->stream));
  });
}

int vqf_sv_download(vqf_sv sv, double* amps) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    VQF_CUDA(cudaSetDevice(sv->device));
    const size_t count = sv->dim() * sv->batch;
    if (sv->dtype == VQF_F64) {
      VQF_CUDA(cudaMemcpyAsync(amps, sv->amps, count * 16, cudaMemcpyDeviceToHost, sv->stream));
      VQF_CUDA(cudaStreamSynchronize(sv->stream));
    } else {
      std::vector<float> tmp(2 * count);
      VQF_CUDA(cudaMemcpyAsync(tmp.data(), sv->amps, count * 8, cudaMemcpyDeviceToHost, sv->stream));
      VQF_CUDA(cudaStreamSynchronize(sv->stream));
      for (size_t i = 0; i < 2 * count; ++i) amps[i] = tmp[i];
    }
  });
}

int vqf_sv_norm(vqf_sv sv, double* out) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    VQF_CUDA(cudaSetDevice(sv->device));
    sv_norms(sv, out);
  });
}

int vqf_apply_gate(vqf_sv sv, const vqf_gate* gate) { return vqf_apply_circuit(sv, gate, 1); }

int vqf_apply_circuit(vqf_sv sv, const vqf_gate* gates, uint32_t n_gates) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    VQF_CUDA(cudaSetDevice(sv->device));
    for (uint32_t i = 0; i < n_gates; ++i) sv_check_gate(sv, gates[i]);  // all-or-nothing validation
    if (n_gates == 1) {
      const vqf_gate& g = gates[0];
      GateArgs a{g.kind, g.n_wires, {g.wires[0], g.wires[1], g.wires[2], g.wires[3]}, std::cos(0.5 * g.angle),
                 std::sin(0.5 * g.angle), nullptr};
      sv_apply(sv, a);
    } else {  // fused shared-memory tile passes (tile.cu)
      std::vector<TGate> tg(n_gates);
      for (uint32_t i = 0; i < n_gates; ++i) {
        const vqf_gate& g = gates[i];
        tg[i] = TGate{g.kind, g.n_wires, {g.wires[0], g.wires[1], g.wires[2], g.wires[3]}, -1,
                      std::cos(0.5 * g.angle), std::sin(0.5 * g.angle)};
      }
      run_circuit_tiled(sv, tg, nullptr);
    }
    VQF_CUDA(cudaStreamSynchronize(sv->stream));
  });
}

int vqf_expectation_complex(vqf_sv sv, const vqf_hamiltonian* h, double* out) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    if (h == nullptr) throw_invalid("null hamiltonian");
    if (h->n_qubits != sv->n_qubits) throw_invalid("expectation: qubit count mismatch");
    const CompiledHam c = compile_hamiltonian(h);
    VQF_CUDA(cudaSetDevice(sv->device));
    sv_expectation(sv, c, out);
  });
}

int vqf_sv_device_ptr(vqf_sv sv, void** ptr, uint64_t* bytes) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    VQF_CUDA(cudaStreamSynchronize(sv->stream));
    *ptr = sv->amps;
    *bytes = sv->amp_bytes() * sv->dim() * sv->batch;
  });
}

int vqf_cross_expectation(vqf_sv a, vqf_sv b, const vqf_hamiltonian* h, double* out) {
  return guarded([&] {
    if (a == nullptr || b == nullptr || h == nullptr) throw_invalid("null argument");
    if (a->n_qubits != b->n_qubits || h->n_qubits != a->n_qubits || a->dtype != b->dtype || a->device != b->device)
      throw_invalid("cross expectation: states must share register, dtype and device");
    const CompiledHam c = compile_hamiltonian(h);
    VQF_CUDA(cudaSetDevice(a->device));
    VQF_CUDA(cudaStreamSynchronize(b->stream));
    const uint32_t nb = red_blocks(a->dim());
    ensure_partials(a, 2 * (size_t)nb);
    const size_t tb = std::max<size_t>(1, c.terms.size()) * sizeof(MaskTerm);
    ensure_terms(a, tb);
    if (!c.terms.empty())
      VQF_CUDA(cudaMemcpyAsync(a->terms_dev, c.terms.data(), c.terms.size() * sizeof(MaskTerm),
                               cudaMemcpyHostToDevice, a->stream));
    const MaskTerm* td = static_cast<const MaskTerm*>(a->terms_dev);
    const uint32_t nt = static_cast<uint32_t>(c.terms.size());
    if (a->dtype == VQF_F64)
      k_expect_cross<double><<<nb, kThreads, 0, a->stream>>>(static_cast<const double2*>(a->amps),
                                                            static_cast<const double2*>(b->amps), a->n_qubits, td, nt,
                                                            a->partials);
    else
      k_expect_cross<float><<<nb, kThreads, 0, a->stream>>>(static_cast<const float2*>(a->amps),
                                                           static_cast<const float2*>(b->amps), a->n_qubits, td, nt,
                                                           a->partials);
    VQF_LAUNCHED();
    k_final_sum<<<1, kThreads, 0, a->stream>>>(a->partials, nb, a->dev_out);
    VQF_LAUNCHED();
    VQF_CUDA(cudaMemcpyAsync(a->host_out, a->dev_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, a->stream));
    VQF_CUDA(cudaStreamSynchronize(a->stream));
    out[0] = a->host_out[0];
    out[1] = a->host_out[1];
  });
}

int vqf_expectation(vqf_sv sv, const vqf_hamiltonian* h, double* out) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    if (h == nullptr) throw_invalid("null hamiltonian");
    if (h->n_qubits != sv->n_qubits) throw_invalid("expectation: qubit count mismatch");
    const CompiledHam c = compile_hamiltonian(h);
    VQF_CUDA(cudaSetDevice(sv->device));
    std::vector<double> tot(2 * sv->batch);
    sv_expectation(sv, c, tot.data());
    for (uint32_t b = 0; b < sv->batch; ++b) {
      // statevector.hpp:244-247
      if (std::abs(tot[2 * b + 1]) >= 1e-10)
        throw_runtime("expectation has imaginary residue " + fstr(tot[2 * b + 1]));
      out[b] = tot[2 * b];
    }
  });
}

}  // extern "C"
