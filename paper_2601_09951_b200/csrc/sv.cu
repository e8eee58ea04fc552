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
#include <utility>

#include "expect_tile.cuh"
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
    if (ok[u]) {  // L2-only loads: no L1 line fill around sparse sectors
      x0[u] = __ldcg(a + i0[u]);
      x1[u] = __ldcg(a + (i0[u] | tbit));
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
    const A x = __ldcg(a + (r | pat_a)), y = __ldcg(a + (r | pat_b));  // L2-only: sparse sectors
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

// conj(a) b as (re, im) in double.  fp64 states: fp64 products; fp32 states:
// the two products per component in fp32 (one FFMA each, no conversions on
// the operands; ~6e-8 relative, inside the 1e-5 fp32 bar), accumulated by
// the caller in fp64.
__device__ __forceinline__ void conj_mul(double2 a, double2 b, double& re, double& im) {
  re = __fma_rn(a.x, b.x, a.y * b.y);
  im = __fma_rn(a.x, b.y, -(a.y * b.x));
}
__device__ __forceinline__ void conj_mul(float2 a, float2 b, double& re, double& im) {
  re = static_cast<double>(__fmaf_rn(a.x, b.x, a.y * b.y));
  im = static_cast<double>(__fmaf_rn(a.x, b.y, -(a.y * b.x)));
}

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

// Diagonal group, factorised (n >= kDiagB).  Thread t of a 256-thread CTA
// owns the amplitudes lo_u = t + 256 u (u < 8) of every 2048-amplitude tile
// it visits, so with i = (tile << 11) | lo_u each Z-string sign factorises
// into a per-thread constant, a per-u pattern and a per-tile sign:
//   * low terms (Z support below bit 11): the thread's sign for lo_u is fixed
//     across tiles, so it accumulates P_u = sum_tiles |psi|^2 and applies the
//     low terms once at the end;
//   * high terms (support at bit 11 and above): one complex scalar H(tile),
//     evaluated lane-parallel (one term per lane, xor-butterfly sum, identical
//     in every lane) and applied to q = sum_u |psi_u|^2;
//   * mixed terms: sign = parity(((tile << 8) | t) & m) * (-1)^popc(u & v)
//     with m = (yz_hi << 8) | yz[0..8) and v = yz[8..11), so the per-u part
//     is an 8-point Walsh-Hadamard transform W of the thread's |psi_u|^2 and
//     each term costs one parity + one FMA per tile (host packs m into .yz
//     and v into .flip, terms sorted by v).
// Per amplitude that leaves one 16-byte load, |psi|^2 and a few adds: the
// pass is HBM-bound for any number of diagonal terms.  Summation order is
// fixed by (n, grid), so results are deterministic.
constexpr uint32_t kDiagB = 11, kDiagU = 8;
static_assert(kThreads * kDiagU == (1u << kDiagB), "diag tile = CTA x unroll");

struct DiagSplit {
  uint32_t n_lo, n_hi, n_mx;
  uint32_t mx_off[9];  // mixed terms with v = j are [mx_off[j], mx_off[j + 1])
};

template <typename T>
__global__ void __launch_bounds__(kThreads) k_expect_diag_fact(const typename V2<T>::type* __restrict__ a, uint32_t n,
                                                               const MaskTerm* __restrict__ lo_t,
                                                               const MaskTerm* __restrict__ hi_t,
                                                               const MaskTerm* __restrict__ mx_t, const DiagSplit ds,
                                                               double* __restrict__ partials, uint32_t G,
                                                               uint32_t stride) {
  using A = typename V2<T>::type;
  __shared__ MaskTerm sh_hi[64];
  __shared__ MaskTerm sh_mx[64];
  for (uint32_t t = threadIdx.x; t < ds.n_hi; t += kThreads) sh_hi[t] = hi_t[t];
  for (uint32_t t = threadIdx.x; t < ds.n_mx; t += kThreads) sh_mx[t] = mx_t[t];
  __syncthreads();
  const uint32_t b = blockIdx.y, lane = threadIdx.x & 31;
  const uint64_t n_tiles = uint64_t{1} << (n - kDiagB);
  const A* s = a + ((uint64_t)b << n) + threadIdx.x;
  double P[kDiagU];
#pragma unroll
  for (int u = 0; u < (int)kDiagU; ++u) P[u] = 0.0;
  double acc_re = 0.0, acc_im = 0.0;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const A* src = s + (tile << kDiagB);
    A x[kDiagU];
#pragma unroll
    for (int u = 0; u < (int)kDiagU; ++u) x[u] = src[u * kThreads];
    // H(tile) while the loads are in flight
    double hr = 0.0, hi = 0.0;
    if (ds.n_hi) {
      for (uint32_t t = lane; t < ds.n_hi; t += 32) {
        const double sg = parity_sign(tile & (sh_hi[t].yz >> kDiagB));
        hr += sg * sh_hi[t].cb_re;
        hi += sg * sh_hi[t].cb_im;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        hr += __shfl_xor_sync(0xffffffffu, hr, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
      }
    }
    double p[kDiagU];
#pragma unroll
    for (int u = 0; u < (int)kDiagU; ++u) {
      p[u] = (double)x[u].x * (double)x[u].x + (double)x[u].y * (double)x[u].y;
      P[u] += p[u];
    }
    if (ds.n_hi) {
      const double q = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
      acc_re += q * hr;
      acc_im += q * hi;
    }
    if (ds.n_mx) {
      double w[kDiagU];  // w[v] = sum_u (-1)^popc(u & v) p[u]
#pragma unroll
      for (int u = 0; u < (int)kDiagU; ++u) w[u] = p[u];
#pragma unroll
      for (int h = 1; h < (int)kDiagU; h <<= 1)
#pragma unroll
        for (int u = 0; u < (int)kDiagU; ++u)
          if ((u & h) == 0) {
            const double l = w[u], r = w[u | h];
            w[u] = l + r;
            w[u | h] = l - r;
          }
      const uint64_t xt = (tile << 8) | threadIdx.x;
#pragma unroll
      for (int v = 0; v < (int)kDiagU; ++v)
        for (uint32_t t = ds.mx_off[v]; t < ds.mx_off[v + 1]; ++t) {
          const double sw = parity_sign(xt & sh_mx[t].yz) * w[v];
          acc_re += sw * sh_mx[t].cb_re;
          acc_im += sw * sh_mx[t].cb_im;
        }
    }
  }
  // low terms, once per owned lo_u
#pragma unroll
  for (int u = 0; u < (int)kDiagU; ++u) {
    const uint32_t lo = threadIdx.x + u * kThreads;
    double lr = 0.0, li = 0.0;
    for (uint32_t t = 0; t < ds.n_lo; ++t) {
      const double sg = parity_sign(lo & lo_t[t].yz);
      lr += sg * lo_t[t].cb_re;
      li += sg * lo_t[t].cb_im;
    }
    acc_re += P[u] * lr;
    acc_im += P[u] * li;
  }
  const double2 acc = block_sum(make_double2(acc_re, acc_im));
  if (threadIdx.x == 0) {
    const size_t o = ((size_t)b * G + 0) * stride + blockIdx.x;
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
  constexpr int U = kExpU;
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
    for (uint64_t k0 = (uint64_t)blockIdx.x * kThreads + threadIdx.x; k0 < half; k0 += stride * U) {
      typename V2<T>::type x[U], y[U];
      uint64_t idx[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // pairs in flight before arithmetic
        const uint64_t k = k0 + u * stride;
        idx[u] = insert_zero(k, hb);
        if (k < half) {
          x[u] = s[idx[u]];
          y[u] = s[idx[u] ^ flip];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k0 + u * stride >= half) break;
        const uint64_t i = idx[u];
        // v = conj(x) * y
        double vr, vi;
        conj_mul(x[u], y[u], vr, vi);
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

// One flip group whose top flip bit hb is >= 11, factorised like the
// diagonal pass: pair index k = (tile << 11) | lo_u, lo_u = t + 256 u, so the
// pair's index is i = (I(tile) << 11) | lo_u with I(tile) = tile with a zero
// inserted at bit hb - 11, and each term's sign splits into
// parity(((I << 8) | t) & m) (host packs m = (yz >> 11) << 8 | yz[0..8) into
// .yz) times (-1)^popc(u & v), v = yz[8..11) (in .flip bits 0-2; bit 3 set
// when sigma = -1, i.e. odd Y count on the flip).  Per tile a thread forms the
// 8 pair products and their Walsh-Hadamard transforms; each term then costs
// one parity and one FMA per tile instead of work per pair.  Terms sorted by
// v, offsets in DiagSplit::mx_off.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_expect_flip_fact(const typename V2<T>::type* __restrict__ a,
                                                               uint32_t n, uint64_t flip, uint32_t hb,
                                                               const MaskTerm* __restrict__ terms, const DiagSplit ds,
                                                               bool need_im, double* __restrict__ partials,
                                                               uint32_t G, uint32_t group, uint32_t stride) {
  using A = typename V2<T>::type;
  __shared__ MaskTerm st[64];
  for (uint32_t t = threadIdx.x; t < ds.n_mx; t += kThreads) st[t] = terms[t];
  __syncthreads();
  const uint32_t b = blockIdx.y;
  const uint64_t n_tiles = uint64_t{1} << (n - 1 - kDiagB);
  const A* s = a + ((uint64_t)b << n);
  const uint32_t hbt = hb - kDiagB;
  double acc_re = 0.0, acc_im = 0.0;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t I = insert_zero(tile, hbt);
    const uint64_t i0 = (I << kDiagB) | threadIdx.x;
    A x[kDiagU], y[kDiagU];
#pragma unroll
    for (int u = 0; u < (int)kDiagU; ++u) {
      const uint64_t i = i0 + (uint64_t)u * kThreads;
      x[u] = s[i];
      y[u] = s[i ^ flip];
    }
    double wr[kDiagU], wi[kDiagU];
#pragma unroll
    for (int u = 0; u < (int)kDiagU; ++u) conj_mul(x[u], y[u], wr[u], wi[u]);
#pragma unroll
    for (int h = 1; h < (int)kDiagU; h <<= 1)
#pragma unroll
      for (int u = 0; u < (int)kDiagU; ++u)
        if ((u & h) == 0) {
          const double l = wr[u], r = wr[u | h];
          wr[u] = l + r;
          wr[u | h] = l - r;
          if (need_im) {
            const double li = wi[u], ri = wi[u | h];
            wi[u] = li + ri;
            wi[u | h] = li - ri;
          }
        }
    const uint64_t xt = (I << 8) | threadIdx.x;
#pragma unroll
    for (int v = 0; v < (int)kDiagU; ++v)
      for (uint32_t t = ds.mx_off[v]; t < ds.mx_off[v + 1]; ++t) {
        const MaskTerm m = st[t];
        const double sg = parity_sign(xt & m.yz);
        if ((m.flip & 8u) == 0) {  // sigma = +1: cb s 2 Re(v)
          const double w = 2.0 * sg * wr[v];
          acc_re += m.cb_re * w;
          acc_im += m.cb_im * w;
        } else {  // sigma = -1: cb s 2i Im(v)
          const double w = 2.0 * sg * wi[v];
          acc_re -= m.cb_im * w;
          acc_im += m.cb_re * w;
        }
      }
  }
  const double2 acc = block_sum(make_double2(acc_re, acc_im));
  if (threadIdx.x == 0) {
    const size_t o = ((size_t)b * G + group) * stride + blockIdx.x;
    partials[2 * o] = acc.x;
    partials[2 * o + 1] = acc.y;
  }
}

// Several flip groups in one pass.  Each thread holds the 16 amplitudes that
// differ in four "register" index bits R (all >= 5) of one base index whose
// bits 0..4 are the lane, so warp loads stay 512 B contiguous.  A group whose
// flip mask lies inside R u {0..4} pairs amplitudes inside the thread
// (register bits) or across lanes (__shfl_xor on the lane bits): the pass
// reads the state once for all of them instead of once per group.
//
// Per group the thread forms v_k = conj(psi_i) psi_{i ^ f} for its pairs
// (each unordered pair once, from the side where f's top bit is clear; 8
// pairs when f has register bits, else 16 on the lanes whose top flip bit is
// clear).  A term's sign (-1)^popc(i & yz) splits into the base part
// (-1)^popc(base & yz) and a register pattern p over the pair index k (host
// packed into .flip), so each term costs one Walsh sum
// W_p = sum_k (-1)^popc(k & p) v_k with compile-time signs, then
// cb s_base (W + sigma conj W) as in k_expect_flip.
constexpr int kRegBits = 4, kRegAmps = 1 << kRegBits;
constexpr int kMultiMaxGroups = 32, kMultiMaxTerms = 128;

struct MultiPass {
  uint32_t rb[kRegBits];                // register bits, ascending, all >= 5
  uint32_t n_groups;
  uint32_t goff[kMultiMaxGroups + 1];   // group j's terms: [goff[j], goff[j + 1])
  uint64_t flip[kMultiMaxGroups];
  uint32_t im_groups;  // bit j: group j has a term with sigma = -1 (needs Im v)
};

// index bits of register slot r (r compile time after unrolling)
__device__ __forceinline__ uint64_t reg_offset(int r, const uint64_t (&rb)[kRegBits]) {
  uint64_t m = 0;
#pragma unroll
  for (int j = 0; j < kRegBits; ++j)
    if (r & (1 << j)) m |= rb[j];
  return m;
}

// x with its sign flipped when bit is set (xor on the sign bit: no select,
// no multiply)
__device__ __forceinline__ double flip_sign(double x, uint32_t bit) {
  return __hiloint2double(__double2hiint(x) ^ static_cast<int>(bit << 31), __double2loint(x));
}

__device__ __forceinline__ float flip_sign(float x, uint32_t bit) {
  return __int_as_float(__float_as_int(x) ^ static_cast<int>(bit << 31));
}

// conj(a) b in the amplitude precision (the multi-group pass keeps fp32
// states' pair products and Walsh sums in fp32: 8 terms, ~1e-7 relative)
__device__ __forceinline__ void conj_mul_native(double2 a, double2 b, double& re, double& im) { conj_mul(a, b, re, im); }
__device__ __forceinline__ void conj_mul_native(float2 a, float2 b, float& re, float& im) {
  re = __fmaf_rn(a.x, b.x, a.y * b.y);
  im = __fmaf_rn(a.x, b.y, -(a.y * b.x));
}

// W_p = sum_k (-1)^popc(k & p) v_k over NP pairs; p = 0 (no Z/Y on the
// register bits, e.g. every TFIM term) is a plain sum
template <int NP, typename VT>
__device__ __forceinline__ double walsh(const VT (&v)[NP], uint32_t p) {
  VT w = VT(0);
  if (p == 0) {
#pragma unroll
    for (int k = 0; k < NP; ++k) w += v[k];
  } else {
#pragma unroll
    for (int k = 0; k < NP; ++k) w += flip_sign(v[k], __popc(k & p) & 1u);
  }
  return static_cast<double>(w);
}

// The terms of one group from its 8 pair products v_k: each term adds
// cb s_base (W + sigma conj W) (k_expect_flip's pair formula summed over k).
// `neg` flips s_base for the lanes of a lane-pair group that hold the side-1
// amplitudes (see multi_group_lane).
template <typename VT>
__device__ __forceinline__ void multi_terms(const VT (&vr)[kRegAmps / 2], const VT (&vi)[kRegAmps / 2],
                                            bool need_im, uint64_t base, bool side, const MaskTerm* st,
                                            const double* sig, uint32_t t0, uint32_t t1, double& acc_re,
                                            double& acc_im) {
  for (uint32_t t = t0; t < t1; ++t) {
    const MaskTerm m = st[t];
    const uint32_t pk = static_cast<uint32_t>(m.flip) & (kRegAmps / 2 - 1);
    double sb = parity_sign(base & m.yz);
    if (side && ((sig[t] < 0.0) != (((m.flip >> (kRegBits - 1)) & 1u) != 0))) sb = -sb;
    if (sig[t] > 0.0) {  // cb s (W + conj W) = cb s 2 Re W
      const double w = 2.0 * sb * walsh<kRegAmps / 2>(vr, pk);
      acc_re += m.cb_re * w;
      acc_im += m.cb_im * w;
    } else if (need_im) {  // cb s (W - conj W) = cb s 2i Im W
      const double w = 2.0 * sb * walsh<kRegAmps / 2>(vi, pk);
      acc_re -= m.cb_im * w;
      acc_im += m.cb_re * w;
    }
  }
}

// A group with register flip pattern FR != 0 (compile time: partners are
// fixed registers; f's top bit is a register bit, so the pairs are the 8
// slots with that bit clear) and lane pattern fl (partner lane via
// __shfl_xor, every lane joins).
template <int FR, typename A>
__device__ __forceinline__ void multi_group(const A (&x)[kRegAmps], uint32_t fl, bool need_im, uint64_t base,
                                            const MaskTerm* st, const double* sig, uint32_t t0, uint32_t t1,
                                            double& acc_re, double& acc_im) {
  constexpr int top = 31 - __builtin_clz((unsigned)FR);
  using VT = decltype(A{}.x);
  VT vr[kRegAmps / 2], vi[kRegAmps / 2];
  int k = 0;
#pragma unroll
  for (int r = 0; r < kRegAmps; ++r) {
    if ((r >> top) & 1) continue;
    A y = x[r ^ FR];
    if (fl) {
      y.x = __shfl_xor_sync(0xffffffffu, y.x, fl);
      y.y = __shfl_xor_sync(0xffffffffu, y.y, fl);
    }
    conj_mul_native(x[r], y, vr[k], vi[k]);
    ++k;
  }
  multi_terms(vr, vi, need_im, base, false, st, sig, t0, t1, acc_re, acc_im);
}

// Lane-only flip (FR = 0): the lane whose top flip bit is clear ("side 0")
// takes the pairs of slots 0..7, its partner ("side 1") those of slots
// 8..15; one shuffle per slot serves both (each sends what the other needs).
// v_k is always conj(side-0 amplitude) * side-1 amplitude, and side-1 lanes
// evaluate the side-0 sign: s(base ^ fl) = s(base) sigma (f = fl), times the
// pattern's bit 3 for slots k + 8.
template <typename A>
__device__ __forceinline__ void multi_group_lane(const A (&x)[kRegAmps], uint32_t fl, bool side, bool need_im,
                                                 uint64_t base, const MaskTerm* st, const double* sig, uint32_t t0,
                                                 uint32_t t1, double& acc_re, double& acc_im) {
  using VT = decltype(A{}.x);
  VT vr[kRegAmps / 2], vi[kRegAmps / 2];
#pragma unroll
  for (int k = 0; k < kRegAmps / 2; ++k) {
    const A own = side ? x[k + kRegAmps / 2] : x[k];
    A y = side ? x[k] : x[k + kRegAmps / 2];
    y.x = __shfl_xor_sync(0xffffffffu, y.x, fl);
    y.y = __shfl_xor_sync(0xffffffffu, y.y, fl);
    VT ur, u;
    conj_mul_native(own, y, ur, u);
    vr[k] = ur;
    vi[k] = flip_sign(u, side ? 1u : 0u);
  }
  multi_terms(vr, vi, need_im, base, side, st, sig, t0, t1, acc_re, acc_im);
}

template <typename A, int... FR>
__device__ __forceinline__ void multi_dispatch(uint32_t fr, std::integer_sequence<int, FR...>,
                                               const A (&x)[kRegAmps], uint32_t fl, bool need_im, uint64_t base,
                                               const MaskTerm* st, const double* sig, uint32_t t0, uint32_t t1,
                                               double& acc_re, double& acc_im) {
  ((fr == (uint32_t)(FR + 1) ? multi_group<FR + 1>(x, fl, need_im, base, st, sig, t0, t1, acc_re, acc_im) : void()),
   ...);
}

// grid = (blocks, batch); partials[(entry * G + slot) * stride + block].
template <typename T>
__global__ void __launch_bounds__(kThreads, 2) k_expect_multi(const typename V2<T>::type* __restrict__ a, uint32_t n,
                                                              const MaskTerm* __restrict__ terms, const MultiPass mp,
                                                              double* __restrict__ partials, uint32_t G,
                                                              uint32_t slot, uint32_t stride) {
  using A = typename V2<T>::type;
  __shared__ MaskTerm st[kMultiMaxTerms];
  __shared__ double sig[kMultiMaxTerms];
  for (uint32_t j = 0; j < mp.n_groups; ++j)
    for (uint32_t t = mp.goff[j] + threadIdx.x; t < mp.goff[j + 1]; t += kThreads) {
      st[t] = terms[t];
      sig[t] = parity_sign(mp.flip[j] & terms[t].yz);
    }
  __syncthreads();
  const uint32_t b = blockIdx.y, lane = threadIdx.x & 31;
  const uint64_t n_bases = uint64_t{1} << (n - kRegBits);
  const A* s = a + ((uint64_t)b << n);
  uint64_t rmask[kRegBits];
#pragma unroll
  for (int j = 0; j < kRegBits; ++j) rmask[j] = uint64_t{1} << mp.rb[j];
  double acc_re = 0.0, acc_im = 0.0;
  const uint64_t stride_k = (uint64_t)gridDim.x * kThreads;
  for (uint64_t k = (uint64_t)blockIdx.x * kThreads + threadIdx.x; k < n_bases; k += stride_k) {
    uint64_t base = k;
#pragma unroll
    for (int j = 0; j < kRegBits; ++j) base = insert_zero(base, mp.rb[j]);
    A x[kRegAmps];
#pragma unroll
    for (int r = 0; r < kRegAmps; ++r) x[r] = s[base | reg_offset(r, rmask)];
    for (uint32_t g = 0; g < mp.n_groups; ++g) {
      const uint64_t f = mp.flip[g];
      const uint32_t fl = static_cast<uint32_t>(f & 31u);
      uint32_t fr = 0;
#pragma unroll
      for (int j = 0; j < kRegBits; ++j)
        if ((f >> mp.rb[j]) & 1u) fr |= 1u << j;
      const bool need_im = (mp.im_groups >> g) & 1u;  // any term with sigma = -1
      if (fr) {
        multi_dispatch(fr, std::make_integer_sequence<int, kRegAmps - 1>{}, x, fl, need_im, base, st, sig,
                       mp.goff[g], mp.goff[g + 1], acc_re, acc_im);
      } else {
        const bool side = ((lane >> (31 - __clz(fl))) & 1u) != 0;
        multi_group_lane(x, fl, side, need_im, base, st, sig, mp.goff[g], mp.goff[g + 1], acc_re, acc_im);
      }
    }
  }
  const double2 acc = block_sum(make_double2(acc_re, acc_im));
  if (threadIdx.x == 0) {
    const size_t idx = ((size_t)b * G + slot) * stride + blockIdx.x;
    partials[2 * idx] = acc.x;
    partials[2 * idx + 1] = acc.y;
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

// Host-side plan of one expectation: which kernel reads the state for each
// flip group, and the packed term array every kernel indexes into.
//   diagonal group : k_expect_diag_fact (n >= 11, <= 64 high / mixed terms),
//                    else k_expect_diag_tiled (<= 64 mixed), else k_expect_diag
//   flip groups    : packed into k_expect_multi passes when their flip bits
//                    above bit 4 number <= 4 (first fit in group order), else
//                    one k_expect_flip pass each
struct MultiLaunch {
  MultiPass mp{};
  uint64_t rset = 0;
  uint32_t first_group = 0, term_base = 0;
  std::vector<uint32_t> groups;
};

struct ExpPlan {
  enum DiagMode { DIAG_NONE, DIAG_FACT, DIAG_TILED, DIAG_PLAIN } diag = DIAG_NONE;
  std::vector<MaskTerm> all;  // h.terms, then per-kernel repacked term lists
  uint32_t B = 0, o_lo = 0, o_hi = 0, o_mx = 0, n_lo = 0, n_hi = 0, n_mx = 0;  // tiled split
  DiagSplit ds{};
  uint32_t o_flo = 0, o_fhi = 0, o_fmx = 0;  // factorised split
  std::vector<MultiLaunch> multi;
  std::vector<uint32_t> single;  // flip groups read by their own k_expect_flip pass
  struct FactFlip {
    uint32_t group, term_base;
    DiagSplit ds;
    bool need_im;
  };
  std::vector<FactFlip> fact;  // single groups on k_expect_flip_fact (top flip bit >= 11)
  std::vector<ExpTileParams> tiles;  // single-bit flip groups on k_expect_tile passes (expect_tile.cu)
  uint32_t state_passes() const {
    return (diag != DIAG_NONE ? 1u : 0u) +
           static_cast<uint32_t>(multi.size() + single.size() + fact.size() + tiles.size());
  }
};

ExpPlan plan_expectation(const CompiledHam& h, uint32_t n, int32_t dtype = VQF_F64) {
  ExpPlan pl;
  const uint32_t G = static_cast<uint32_t>(h.group_flip.size());
  std::vector<char> on_tiles;
  pl.tiles = plan_expect_tiles(h, n, dtype, on_tiles);
  pl.all = h.terms;
  // a small real diagonal group rides along in one tile pass
  const bool diag_folded = fold_diag_into_tiles(pl.tiles, h, dtype);
  if (!diag_folded && G > 0 && h.group_offset[1] > h.group_offset[0]) {
    // tiled split: support all below / all above the 2048-amplitude tile, mixed
    pl.B = std::min<uint32_t>(n, 11);
    const uint64_t lo_mask = (uint64_t{1} << pl.B) - 1;
    std::vector<MaskTerm> lo, hi, mx;
    for (uint32_t t = h.group_offset[0]; t < h.group_offset[1]; ++t) {
      const MaskTerm& m = h.terms[t];
      if ((m.yz & ~lo_mask) == 0) lo.push_back(m);
      else if ((m.yz & lo_mask) == 0) hi.push_back(m);
      else mx.push_back(m);
    }
    pl.o_lo = static_cast<uint32_t>(pl.all.size());
    pl.all.insert(pl.all.end(), lo.begin(), lo.end());
    pl.o_hi = static_cast<uint32_t>(pl.all.size());
    pl.all.insert(pl.all.end(), hi.begin(), hi.end());
    pl.o_mx = static_cast<uint32_t>(pl.all.size());
    pl.all.insert(pl.all.end(), mx.begin(), mx.end());
    pl.n_lo = static_cast<uint32_t>(lo.size());
    pl.n_hi = static_cast<uint32_t>(hi.size());
    pl.n_mx = static_cast<uint32_t>(mx.size());
    pl.diag = mx.size() <= 64 ? ExpPlan::DIAG_TILED : ExpPlan::DIAG_PLAIN;
    // factorised split: mixed terms re-packed as {flip = v, yz = (yz_hi << 8) | yz[0..8)}, sorted by v
    if (n >= kDiagB) {
      const uint64_t fmask = (uint64_t{1} << kDiagB) - 1;
      std::vector<MaskTerm> f_lo, f_hi, f_mx;
      for (uint32_t t = h.group_offset[0]; t < h.group_offset[1]; ++t) {
        const MaskTerm& m = h.terms[t];
        if ((m.yz & ~fmask) == 0) f_lo.push_back(m);
        else if ((m.yz & fmask) == 0) f_hi.push_back(m);
        else f_mx.push_back(MaskTerm{(m.yz >> 8) & 7, ((m.yz >> kDiagB) << 8) | (m.yz & 0xff), m.cb_re, m.cb_im});
      }
      if (f_hi.size() <= 64 && f_mx.size() <= 64) {
        std::stable_sort(f_mx.begin(), f_mx.end(),
                         [](const MaskTerm& x, const MaskTerm& y) { return x.flip < y.flip; });
        pl.ds.n_lo = static_cast<uint32_t>(f_lo.size());
        pl.ds.n_hi = static_cast<uint32_t>(f_hi.size());
        pl.ds.n_mx = static_cast<uint32_t>(f_mx.size());
        for (uint32_t v = 0, j = 0; v <= 8; ++v) {
          while (j < f_mx.size() && f_mx[j].flip < v) ++j;
          pl.ds.mx_off[v] = j;
        }
        pl.o_flo = static_cast<uint32_t>(pl.all.size());
        pl.all.insert(pl.all.end(), f_lo.begin(), f_lo.end());
        pl.o_fhi = static_cast<uint32_t>(pl.all.size());
        pl.all.insert(pl.all.end(), f_hi.begin(), f_hi.end());
        pl.o_fmx = static_cast<uint32_t>(pl.all.size());
        pl.all.insert(pl.all.end(), f_mx.begin(), f_mx.end());
        pl.diag = ExpPlan::DIAG_FACT;
      }
    }
  }
  for (uint32_t g = 1; g < G; ++g) {
    const uint32_t cnt = h.group_offset[g + 1] - h.group_offset[g];
    if (cnt == 0 || on_tiles[g]) continue;
    const uint64_t out = h.group_flip[g] & ~uint64_t{31};
    if (n < 5 + kRegBits || cnt > (uint32_t)kMultiMaxTerms || __builtin_popcountll(out) > kRegBits) {
      pl.single.push_back(g);
      continue;
    }
    MultiLaunch* dst = nullptr;
    for (MultiLaunch& ml : pl.multi) {
      uint32_t terms = 0;
      for (uint32_t q : ml.groups) terms += h.group_offset[q + 1] - h.group_offset[q];
      if (__builtin_popcountll(ml.rset | out) <= kRegBits && ml.groups.size() < (size_t)kMultiMaxGroups &&
          terms + cnt <= (uint32_t)kMultiMaxTerms) {
        dst = &ml;
        break;
      }
    }
    if (dst == nullptr) {
      pl.multi.emplace_back();
      dst = &pl.multi.back();
      dst->first_group = g;
    }
    dst->rset |= out;
    dst->groups.push_back(g);
  }
  // single groups with a high top flip bit: factorised pass
  if (n >= kDiagB + 2) {
    std::vector<uint32_t> keep;
    for (const uint32_t g : pl.single) {
      const uint64_t f = h.group_flip[g];
      const uint32_t hb = 63 - __builtin_clzll(f), cnt = h.group_offset[g + 1] - h.group_offset[g];
      if (hb < kDiagB || cnt > 64) {
        keep.push_back(g);
        continue;
      }
      ExpPlan::FactFlip ff{};
      ff.group = g;
      std::vector<MaskTerm> ts;
      for (uint32_t t = h.group_offset[g]; t < h.group_offset[g + 1]; ++t) {
        const MaskTerm& m = h.terms[t];
        const bool neg = __builtin_popcountll(f & m.yz) & 1;
        ff.need_im = ff.need_im || neg;
        ts.push_back(MaskTerm{((m.yz >> 8) & 7) | (neg ? 8u : 0u), ((m.yz >> kDiagB) << 8) | (m.yz & 0xff), m.cb_re,
                              m.cb_im});
      }
      std::stable_sort(ts.begin(), ts.end(), [](const MaskTerm& x, const MaskTerm& y) { return (x.flip & 7) < (y.flip & 7); });
      ff.ds.n_mx = static_cast<uint32_t>(ts.size());
      for (uint32_t v = 0, j = 0; v <= 8; ++v) {
        while (j < ts.size() && (ts[j].flip & 7) < v) ++j;
        ff.ds.mx_off[v] = j;
      }
      ff.term_base = static_cast<uint32_t>(pl.all.size());
      pl.all.insert(pl.all.end(), ts.begin(), ts.end());
      pl.fact.push_back(ff);
    }
    pl.single = keep;
  }
  for (MultiLaunch& ml : pl.multi) {
    for (uint32_t bit = 5; bit < n && __builtin_popcountll(ml.rset) < kRegBits; ++bit) ml.rset |= uint64_t{1} << bit;
    uint32_t j = 0;
    for (uint32_t bit = 5; bit < n; ++bit)
      if ((ml.rset >> bit) & 1u) ml.mp.rb[j++] = bit;
    ml.term_base = static_cast<uint32_t>(pl.all.size());
    ml.mp.n_groups = static_cast<uint32_t>(ml.groups.size());
    ml.mp.goff[0] = 0;
    for (uint32_t q = 0; q < ml.groups.size(); ++q) {
      const uint32_t g = ml.groups[q];
      const uint64_t f = h.group_flip[g];
      ml.mp.flip[q] = f;
      uint32_t fr = 0;
      for (uint32_t j = 0; j < (uint32_t)kRegBits; ++j)
        if ((f >> ml.mp.rb[j]) & 1u) fr |= 1u << j;
      const uint32_t top = fr ? 31u - __builtin_clz(fr) : 0u;
      for (uint32_t t = h.group_offset[g]; t < h.group_offset[g + 1]; ++t) {
        // yz on the register bits as a pattern over the pair index k: all
        // four bits when the pairs are lane pairs, else the three bits left
        // after removing f's top register bit (always clear on the pair side)
        MaskTerm m = h.terms[t];
        uint32_t p = 0;
        for (uint32_t j = 0; j < (uint32_t)kRegBits; ++j)
          if ((m.yz >> ml.mp.rb[j]) & 1u) p |= 1u << j;
        if (fr) p = (p & ((1u << top) - 1)) | ((p >> (top + 1)) << top);
        m.flip = p;  // (base has zeros on R, so popc(base & yz) skips the register part)
        if (__builtin_popcountll(f & m.yz) & 1) ml.mp.im_groups |= 1u << q;
        pl.all.push_back(m);
      }
      ml.mp.goff[q + 1] = static_cast<uint32_t>(pl.all.size()) - ml.term_base;
    }
  }
  return pl;
}

template <typename K>
uint32_t resident_grid(K kernel, uint32_t cap, uint64_t need) {
  // one resident wave: grid = SMs x CTAs per SM (no tail), capped by the
  // partial-sum stride and by the work
  int occ = 0, dev = 0, sms = 148;
  VQF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0));
  VQF_CUDA(cudaGetDevice(&dev));
  VQF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return static_cast<uint32_t>(
      std::max<uint64_t>(1, std::min<uint64_t>({(uint64_t)cap, need, (uint64_t)std::max(occ, 1) * sms})));
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
  const ExpPlan pl = plan_expectation(h, n, sv->dtype);
  ensure_terms(sv, std::max<size_t>(1, pl.all.size()) * sizeof(MaskTerm));
  if (!pl.all.empty())
    VQF_CUDA(cudaMemcpyAsync(sv->terms_dev, pl.all.data(), pl.all.size() * sizeof(MaskTerm), cudaMemcpyHostToDevice,
                             sv->stream));
  const MaskTerm* td = static_cast<const MaskTerm*>(sv->terms_dev);
  const dim3 grid(nb, sv->batch);
  switch (pl.diag) {
    case ExpPlan::DIAG_FACT: {
      static thread_local uint32_t nbf = 0, nbf_n = 0;
      if (nbf_n != n) {
        nbf = resident_grid(k_expect_diag_fact<T>, nb, uint64_t{1} << (n - kDiagB));
        nbf_n = n;
      }
      k_expect_diag_fact<T><<<dim3(nbf, sv->batch), kThreads, 0, sv->stream>>>(
          a, n, td + pl.o_flo, td + pl.o_fhi, td + pl.o_fmx, pl.ds, sv->partials, G, nb);
      VQF_LAUNCHED();
      break;
    }
    case ExpPlan::DIAG_TILED:
      k_expect_diag_tiled<T><<<grid, kThreads, sizeof(double2) << pl.B, sv->stream>>>(
          a, n, pl.B, td + pl.o_lo, pl.n_lo, td + pl.o_hi, pl.n_hi, td + pl.o_mx, pl.n_mx, sv->partials, G);
      VQF_LAUNCHED();
      break;
    case ExpPlan::DIAG_PLAIN:
      k_expect_diag<T><<<grid, kThreads, 0, sv->stream>>>(a, n, td + h.group_offset[0],
                                                          h.group_offset[1] - h.group_offset[0], sv->partials, G, 0);
      VQF_LAUNCHED();
      break;
    case ExpPlan::DIAG_NONE: break;
  }
  launch_expect_tiles(sv, pl.tiles, sv->partials, G, nb);
  for (const uint32_t g : pl.single) {
    const uint32_t t0 = h.group_offset[g], cnt = h.group_offset[g + 1] - t0;
    const uint64_t f = h.group_flip[g];
    const uint32_t hb = 63 - __builtin_clzll(f);
    k_expect_flip<T><<<grid, kThreads, 0, sv->stream>>>(a, n, f, hb, td + t0, cnt, sv->partials, G, g);
    VQF_LAUNCHED();
  }
  if (!pl.fact.empty()) {
    static thread_local uint32_t nbff = 0, nbff_n = 0;
    if (nbff_n != n) {
      nbff = resident_grid(k_expect_flip_fact<T>, nb, uint64_t{1} << (n - 1 - kDiagB));
      nbff_n = n;
    }
    for (const ExpPlan::FactFlip& ff : pl.fact) {
      const uint64_t f = h.group_flip[ff.group];
      const uint32_t hb = 63 - __builtin_clzll(f);
      k_expect_flip_fact<T><<<dim3(nbff, sv->batch), kThreads, 0, sv->stream>>>(
          a, n, f, hb, td + ff.term_base, ff.ds, ff.need_im, sv->partials, G, ff.group, nb);
      VQF_LAUNCHED();
    }
  }
  if (!pl.multi.empty()) {
    static thread_local uint32_t nbm = 0, nbm_n = 0;
    if (nbm_n != n) {
      nbm = resident_grid(k_expect_multi<T>, nb, ((uint64_t{1} << (n - kRegBits)) + kThreads - 1) / kThreads);
      nbm_n = n;
    }
    for (const MultiLaunch& ml : pl.multi) {
      k_expect_multi<T><<<dim3(nbm, sv->batch), kThreads, 0, sv->stream>>>(a, n, td + ml.term_base, ml.mp,
                                                                            sv->partials, G, ml.first_group, nb);
      VQF_LAUNCHED();
    }
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

// Handle resources (stream, pinned / device result words, reduction and
// term scratch) are recycled per device: creating a state handle then costs
// one pool allocation instead of cudaStreamCreate + cudaMallocHost +
// cudaMalloc (and their synchronising frees), whose latency spikes made
// repeated VQE runs jittery.
struct SvAux {
  cudaStream_t stream = nullptr;
  double* host_out = nullptr;
  double* dev_out = nullptr;
  size_t out_cap = 0;  // doubles
  double* partials = nullptr;
  size_t partial_cap = 0;
  void* terms_dev = nullptr;
  size_t terms_cap = 0;
  double* cs_dev = nullptr;
  size_t cs_cap = 0;
};
constexpr size_t kAuxKeep = 16;

std::mutex& aux_mutex() {
  static std::mutex mu;
  return mu;
}
std::vector<std::pair<int, SvAux>>& aux_pool() {
  static std::vector<std::pair<int, SvAux>> pool;
  return pool;
}

void aux_release(const SvAux& a) {
  if (a.partials) cudaFree(a.partials);
  if (a.terms_dev) cudaFree(a.terms_dev);
  if (a.cs_dev) cudaFree(a.cs_dev);
  if (a.host_out) cudaFreeHost(a.host_out);
  if (a.dev_out) cudaFree(a.dev_out);
  if (a.stream) cudaStreamDestroy(a.stream);
}

void sv_take_aux(vqf_statevector* sv) {
  SvAux a;
  bool found = false;
  {
    std::lock_guard<std::mutex> lock(aux_mutex());
    auto& pool = aux_pool();
    for (size_t i = pool.size(); i-- > 0;)
      if (pool[i].first == sv->device) {
        a = pool[i].second;
        pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(i));
        found = true;
        break;
      }
  }
  if (!found) VQF_CUDA(cudaStreamCreateWithFlags(&a.stream, cudaStreamNonBlocking));
  const size_t need = 2 * static_cast<size_t>(sv->batch);
  if (a.out_cap < need) {
    if (a.host_out) VQF_CUDA(cudaFreeHost(a.host_out));
    if (a.dev_out) VQF_CUDA(cudaFree(a.dev_out));
    a.host_out = nullptr;
    a.dev_out = nullptr;
    const size_t cap = std::max<size_t>(need, 256);
    VQF_CUDA(cudaMallocHost(&a.host_out, cap * sizeof(double)));
    VQF_CUDA(cudaMalloc(&a.dev_out, cap * sizeof(double)));
    a.out_cap = cap;
  }
  sv->own_stream = a.stream;
  sv->host_out = a.host_out;
  sv->dev_out = a.dev_out;
  sv->out_cap = a.out_cap;
  sv->partials = a.partials;
  sv->partial_cap = a.partial_cap;
  sv->terms_dev = a.terms_dev;
  sv->terms_cap = a.terms_cap;
  sv->cs_dev = a.cs_dev;
  sv->cs_cap = a.cs_cap;
}

void sv_return_aux(vqf_statevector* sv) {
  SvAux a;
  a.stream = sv->own_stream;
  a.host_out = sv->host_out;
  a.dev_out = sv->dev_out;
  a.out_cap = sv->out_cap;
  a.partials = sv->partials;
  a.partial_cap = sv->partial_cap;
  a.terms_dev = sv->terms_dev;
  a.terms_cap = sv->terms_cap;
  a.cs_dev = sv->cs_dev;
  a.cs_cap = sv->cs_cap;
  {
    std::lock_guard<std::mutex> lock(aux_mutex());
    auto& pool = aux_pool();
    size_t mine = 0;
    for (const auto& e : pool) mine += e.first == sv->device;
    if (mine < kAuxKeep) {
      pool.emplace_back(sv->device, a);
      return;
    }
  }
  aux_release(a);
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
      sv_take_aux(sv);
      sv->stream = sv->own_stream;
      // stream-ordered allocation from the device pool, whose release
      // threshold is raised once per device so freed states stay mapped and
      // repeated calls (VQE iterations, scaling widths) reuse HBM instead of
      // paying cudaMalloc page-mapping costs
      retain_pool(device);
      VQF_CUDA(cudaMallocAsync(&sv->amps, sv->amp_bytes() * sv->dim() * batch, sv->stream));
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
    if (sv->own_stream) sv_return_aux(sv);  // scratch, result words and stream are recycled
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

int vqf_circuit_plan(uint32_t n_qubits, int32_t dtype, const vqf_gate* gates, uint32_t n_gates, uint32_t* passes,
                     uint32_t* fused_ops) {
  return guarded([&] {
    if (n_qubits < 1 || n_qubits > 36) throw_invalid("circuit plan: n_qubits must be in [1, 36]");
    if (dtype != VQF_F64 && dtype != VQF_F32) throw_invalid("circuit plan: unknown dtype");
    vqf_statevector probe;
    probe.n_qubits = n_qubits;
    for (uint32_t i = 0; i < n_gates; ++i) sv_check_gate(&probe, gates[i]);
    uint32_t p = n_gates, f = 0;
    if (n_gates > 1) {
      std::vector<TGate> tg(n_gates);
      for (uint32_t i = 0; i < n_gates; ++i) {
        const vqf_gate& g = gates[i];
        tg[i] = TGate{g.kind, g.n_wires, {g.wires[0], g.wires[1], g.wires[2], g.wires[3]}, -1, 1.0, 0.0};
      }
      plan_tile_counts(n_qubits, dtype, tg, &p, &f);
    }
    if (passes) *passes = p;
    if (fused_ops) *fused_ops = f;
  });
}

int vqf_expectation_plan(const vqf_hamiltonian* h, uint32_t* state_passes, uint32_t* flip_groups,
                         uint32_t* multi_passes) {
  return vqf_expectation_plan_ex(h, VQF_F64, state_passes, flip_groups, multi_passes);
}

int vqf_expectation_plan_ex(const vqf_hamiltonian* h, int32_t dtype, uint32_t* state_passes, uint32_t* flip_groups,
                            uint32_t* multi_passes) {
  return guarded([&] {
    if (h == nullptr) throw_invalid("null hamiltonian");
    if (dtype != VQF_F64 && dtype != VQF_F32) throw_invalid("expectation plan: unknown dtype");
    const CompiledHam c = compile_hamiltonian(h);
    const ExpPlan pl = plan_expectation(c, h->n_qubits, dtype);
    uint32_t groups = 0;
    for (size_t g = 1; g < c.group_flip.size(); ++g) groups += c.group_offset[g + 1] > c.group_offset[g] ? 1 : 0;
    if (state_passes) *state_passes = pl.state_passes();
    if (flip_groups) *flip_groups = groups;
    if (multi_passes) *multi_passes = static_cast<uint32_t>(pl.multi.size() + pl.tiles.size());
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
