// Adjoint-differentiation gradient for the HBM engine (wide registers).
//
// The reference differentiates with the two-term parameter shift
// (vqe.hpp:112-127): 2P extra circuits per iteration.  For the
// hardware-efficient ansatz at 26 qubits that is 105 full circuits per
// iteration.  The adjoint method gets the same gradient (analytically equal
// for these single-frequency gates; numerically equal to ~1e-15) from:
//   forward   psi = U_L ... U_1 |init>                     (existing kernels)
//   k_apply_ham  lambda = H psi, E = <psi|lambda>          (one tiled pass)
//   backward  for k = L..1:  psi <- U_k^dag psi;
//             if U_k has parameter j:  g_j = 2 Re <lambda| dU_k/dtheta |psi>;
//             lambda <- U_k^dag lambda
// A parameterised backward step is one kernel (k_adj_givens): it reads and
// writes both vectors once (4S) and reduces the derivative inner product
// deterministically into per-block partials.  Up to four consecutive RYs on
// distinct wires share one such pass (k_adj_ry_multi), and runs of X / CNOT
// gates are un-applied to each vector by the fused tile path (permutation
// passes, tile.cu).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "adjoint.cuh"
#include "tile.cuh"

namespace vqf {

namespace {

constexpr int kThreads = 256;
constexpr int kU = 4;
constexpr int kBlocks = 4 * 148;
constexpr uint32_t kTileBits = 11;
constexpr int kMaxGroups = 256;
constexpr int kMaxTerms = 1024;

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

__device__ __forceinline__ double parity_sign(uint64_t x) { return (__popcll(x) & 1) ? -1.0 : 1.0; }

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;
}

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

// lambda = H psi and <psi|lambda>, one pass over 2^B-amplitude tiles.
// Per amplitude i: lambda_i = D(i) psi_i + sum_g O_g(i) psi_{i ^ f_g}, with
// D from the tiled diagonal split and O_g(i) = sum_t cb_t (-1)^popc(i & yz_t).
template <typename T>
__global__ void __launch_bounds__(kThreads) k_apply_ham(const typename V2<T>::type* __restrict__ psi,
                                                        typename V2<T>::type* __restrict__ lam, uint32_t n,
                                                        uint32_t B, HamDevC h, double* __restrict__ partials) {
  using A = typename V2<T>::type;
  extern __shared__ double2 Ltab[];
  __shared__ MaskTerm mx[64];
  const uint32_t tile_amps = 1u << B;
  const uint64_t n_tiles = uint64_t{1} << (n - B);
  for (uint32_t lo = threadIdx.x; lo < tile_amps; lo += kThreads) {
    double re = 0.0, im = 0.0;
    for (uint32_t t = 0; t < h.n_lo; ++t) {
      const double sg = parity_sign(lo & h.lo_t[t].yz);
      re += sg * h.lo_t[t].cb_re;
      im += sg * h.lo_t[t].cb_im;
    }
    Ltab[lo] = make_double2(re, im);
  }
  if (threadIdx.x < h.n_mx) mx[threadIdx.x] = h.mx_t[threadIdx.x];
  __syncthreads();
  double2 acc = make_double2(0.0, 0.0);
  __shared__ double2 ohi[kMaxGroups];  // per flip group: its tile-constant operator part
  __shared__ uint64_t sflip[kMaxGroups];
  __shared__ uint32_t sgoff[kMaxGroups + 1], sghi[kMaxGroups];
  for (uint32_t g = threadIdx.x; g <= h.n_groups; g += kThreads) {
    sgoff[g] = h.group_off[g];
    if (g < h.n_groups) {
      sflip[g] = h.flips[g];
      sghi[g] = h.group_hi[g];
    }
  }
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    double hre = 0.0, him = 0.0;
    for (uint32_t t = 0; t < h.n_hi; ++t) {
      const double sg = parity_sign(tile & (h.hi_t[t].yz >> B));
      hre += sg * h.hi_t[t].cb_re;
      him += sg * h.hi_t[t].cb_im;
    }
    // terms whose Z/Y support lies at or above the tile bits have one sign
    // per tile: sum them once per group here, not per amplitude
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < h.n_groups; g += kThreads) {
      double re = 0.0, im = 0.0;
      const uint32_t t0 = h.group_off[g];
      for (uint32_t t = t0; t < t0 + h.group_hi[g]; ++t) {
        const double sg = parity_sign(tile & (h.terms[t].yz >> B));
        re += sg * h.terms[t].cb_re;
        im += sg * h.terms[t].cb_im;
      }
      ohi[g] = make_double2(re, im);
    }
    __syncthreads();
    const uint64_t base = tile << B;
    for (uint32_t lo0 = threadIdx.x; lo0 < tile_amps; lo0 += kThreads * kU) {
      A x[kU];
      double2 l[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t lo = lo0 + u * kThreads;
        if (lo < tile_amps) x[u] = psi[base | lo];
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t lo = lo0 + u * kThreads;
        const uint64_t i = base | lo;
        double dre = 0.0, dim = 0.0;
        if (lo < tile_amps) {
          const double2 lt = Ltab[lo];
          dre = lt.x + hre;
          dim = lt.y + him;
          for (uint32_t t = 0; t < h.n_mx; ++t) {
            const double sg = parity_sign(i & mx[t].yz);
            dre += sg * mx[t].cb_re;
            dim += sg * mx[t].cb_im;
          }
        }
        l[u] = make_double2(dre * (double)x[u].x - dim * (double)x[u].y, dre * (double)x[u].y + dim * (double)x[u].x);
      }
      for (uint32_t g = 0; g < h.n_groups; ++g) {
        const uint64_t f = sflip[g];
        A y[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint32_t lo = lo0 + u * kThreads;
          if (lo < tile_amps) y[u] = psi[(base | lo) ^ f];
        }
        const double2 oc = ohi[g];
        const uint32_t t_lo = sgoff[g] + sghi[g], t_end = sgoff[g + 1];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const uint64_t i = base | (lo0 + u * kThreads);
          double ore = oc.x, oim = oc.y;
          for (uint32_t t = t_lo; t < t_end; ++t) {
            const double sg = parity_sign(i & h.terms[t].yz);
            ore += sg * h.terms[t].cb_re;
            oim += sg * h.terms[t].cb_im;
          }
          // l += O y (fused multiply-adds)
          l[u].x = __fma_rn(ore, (double)y[u].x, __fma_rn(-oim, (double)y[u].y, l[u].x));
          l[u].y = __fma_rn(ore, (double)y[u].y, __fma_rn(oim, (double)y[u].x, l[u].y));
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t lo = lo0 + u * kThreads;
        if (lo >= tile_amps) break;
        A out;
        out.x = static_cast<T>(l[u].x);
        out.y = static_cast<T>(l[u].y);
        lam[base | lo] = out;
        // <psi|lambda> += conj(psi_i) lambda_i
        acc.x += (double)x[u].x * l[u].x + (double)x[u].y * l[u].y;
        acc.y += (double)x[u].x * l[u].y - (double)x[u].y * l[u].x;
      }
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = acc.x;
    partials[2 * blockIdx.x + 1] = acc.y;
  }
}

// One backward step of a Givens-type parameterised gate G(theta) =
// [[c, -s], [s, c]] on amplitude pairs (r | pat_a, r | pat_b), r = index with
// M zero bits inserted at pos[] (RY: M = 1, pat_a = 0, pat_b = bit;
// DoubleExcitation: M = 4, |1100> / |0011>; SingleExcitation: M = 2).
//   psi'  = G^dag psi                       (psi_{k-1})
//   g    += Re( conj(l_a) mu_a + conj(l_b) mu_b ),  mu = (dG/dtheta) psi'
//   lam'  = G^dag lam
// dG/dtheta = 1/2 [[-s, -c], [c, -s]].  Per-block partials of g.
template <typename T, int M>
__global__ void __launch_bounds__(kThreads) k_adj_givens(typename V2<T>::type* __restrict__ psi,
                                                         typename V2<T>::type* __restrict__ lam, uint32_t n,
                                                         uint64_t pat_a, uint64_t pat_b, uint64_t total, uint32_t p0,
                                                         uint32_t p1, uint32_t p2, uint32_t p3, double c, double s,
                                                         double* __restrict__ partials) {
  using A = typename V2<T>::type;
  const uint32_t pos[4] = {p0, p1, p2, p3};
  const T ct = static_cast<T>(c), st = static_cast<T>(s);
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t k0 = (uint64_t)blockIdx.x * kThreads + threadIdx.x; k0 < total; k0 += stride * kU) {
    A a[kU], b[kU], la[kU], lb[kU];
    uint64_t r[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t k = k0 + u * stride;
      uint64_t x = k;
#pragma unroll
      for (int m = 0; m < M; ++m) x = insert_zero(x, pos[m]);
      r[u] = x;
      if (k < total) {
        a[u] = psi[x | pat_a];
        b[u] = psi[x | pat_b];
        la[u] = lam[x | pat_a];
        lb[u] = lam[x | pat_b];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (k0 + u * stride >= total) break;
      // psi' = G^dag psi: a' = c a + s b, b' = -s a + c b
      A pa, pb;  // (fused multiply-adds throughout)
      pa.x = fma(ct, a[u].x, st * b[u].x);
      pa.y = fma(ct, a[u].y, st * b[u].y);
      pb.x = fma(ct, b[u].x, -(st * a[u].x));
      pb.y = fma(ct, b[u].y, -(st * a[u].y));
      // mu = dG psi' = 1/2 (-s a' - c b', c a' - s b')
      const double mar = fma(-s, (double)pa.x, -(c * (double)pb.x)), mai = fma(-s, (double)pa.y, -(c * (double)pb.y));
      const double mbr = fma(c, (double)pa.x, -(s * (double)pb.x)), mbi = fma(c, (double)pa.y, -(s * (double)pb.y));
      acc = fma(0.5 * (double)la[u].x, mar, fma(0.5 * (double)la[u].y, mai,
            fma(0.5 * (double)lb[u].x, mbr, fma(0.5 * (double)lb[u].y, mbi, acc))));
      A qa, qb;
      qa.x = fma(ct, la[u].x, st * lb[u].x);
      qa.y = fma(ct, la[u].y, st * lb[u].y);
      qb.x = fma(ct, lb[u].x, -(st * la[u].x));
      qb.y = fma(ct, lb[u].y, -(st * la[u].y));
      psi[r[u] | pat_a] = pa;
      psi[r[u] | pat_b] = pb;
      lam[r[u] | pat_a] = qa;
      lam[r[u] | pat_b] = qb;
    }
  }
  const double2 t = block_sum(make_double2(acc, 0.0));
  if (threadIdx.x == 0) partials[blockIdx.x] = t.x;
}

// K consecutive RY gates on distinct wires (they commute), un-applied in
// one pass over both vectors.  Each thread holds the 2^K amplitudes of psi
// and lambda that differ in the K gate bits (slot bit j <-> gate j, so every
// pair is a fixed pair of registers) and runs k_adj_givens' step for gate
// 0, 1, ..., K-1 in turn: psi' = G^dag psi, g_j += Re<lambda| dG psi'>,
// lambda' = G^dag lambda.  Per-block partials per gate.
struct RyGroup {
  uint32_t bit[4];
  double c[4], s[4];
  double* part[4];  // gate j's per-block partial row
};

template <typename T, int K>
__global__ void __launch_bounds__(kThreads) k_adj_ry_multi(typename V2<T>::type* __restrict__ psi,
                                                           typename V2<T>::type* __restrict__ lam, uint32_t n,
                                                           const RyGroup gr) {
  using A = typename V2<T>::type;
  constexpr int D = 1 << K;
  uint32_t pos[K];
#pragma unroll
  for (int j = 0; j < K; ++j) pos[j] = gr.bit[j];
  // ascending insertion order for the base index
  uint32_t asc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) asc[j] = pos[j];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = i + 1; j < K; ++j)
      if (asc[j] < asc[i]) {
        const uint32_t t = asc[i];
        asc[i] = asc[j];
        asc[j] = t;
      }
  uint64_t off[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    uint64_t o = 0;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (r & (1 << j)) o |= uint64_t{1} << pos[j];
    off[r] = o;
  }
  double acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0.0;
  const uint64_t total = uint64_t{1} << (n - K);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t k = (uint64_t)blockIdx.x * kThreads + threadIdx.x; k < total; k += stride) {
    uint64_t base = k;
#pragma unroll
    for (int j = 0; j < K; ++j) base = insert_zero(base, asc[j]);
    A a[D], l[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      a[r] = psi[base | off[r]];
      l[r] = lam[base | off[r]];
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const double c = gr.c[j], sn = gr.s[j];
      const T ct = static_cast<T>(c), st = static_cast<T>(sn);
#pragma unroll
      for (int r = 0; r < D; ++r) {
        if (r & (1 << j)) continue;
        A& x = a[r];
        A& y = a[r | (1 << j)];
        A& lx = l[r];
        A& ly = l[r | (1 << j)];
        A pa, pb;  // psi' = G^dag psi (fused multiply-adds throughout)
        pa.x = fma(ct, x.x, st * y.x);
        pa.y = fma(ct, x.y, st * y.y);
        pb.x = fma(ct, y.x, -(st * x.x));
        pb.y = fma(ct, y.y, -(st * x.y));
        // mu = dG psi' = 1/2 (-s a' - c b', c a' - s b'); g += Re<lambda|mu>
        const double mar = fma(-sn, (double)pa.x, -(c * (double)pb.x)), mai = fma(-sn, (double)pa.y, -(c * (double)pb.y));
        const double mbr = fma(c, (double)pa.x, -(sn * (double)pb.x)), mbi = fma(c, (double)pa.y, -(sn * (double)pb.y));
        acc[j] = fma(0.5 * (double)lx.x, mar, fma(0.5 * (double)lx.y, mai,
                 fma(0.5 * (double)ly.x, mbr, fma(0.5 * (double)ly.y, mbi, acc[j]))));
        A qa, qb;  // lambda' = G^dag lambda
        qa.x = fma(ct, lx.x, st * ly.x);
        qa.y = fma(ct, lx.y, st * ly.y);
        qb.x = fma(ct, ly.x, -(st * lx.x));
        qb.y = fma(ct, ly.y, -(st * lx.y));
        x = pa;
        y = pb;
        lx = qa;
        ly = qb;
      }
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      psi[base | off[r]] = a[r];
      lam[base | off[r]] = l[r];
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double2 t = block_sum(make_double2(acc[j], 0.0));
    if (threadIdx.x == 0) gr.part[j][blockIdx.x] = t.x;
  }
}

// The same backward step for RYs when the vectors sit in a GF(2) frame
// (logical index i = M p ^ c of physical slot p): the backward sweep
// un-applies CNOT / X chains by updating the frame instead of moving data
// (the gradient's inner products do not care where amplitudes sit).  RY on
// logical bit b pairs slots p and p ^ vec (vec = M^-1 e_b); the slot holding
// logical 0 is the one with parity(row & p) ^ cbit = 0, one orientation per
// coset (vec_i . row_j = delta_ij), so a logical-1 base just swaps the pair.
struct RyFrameGroup {
  uint64_t vec[4], row[4];
  uint32_t piv[4];  // ascending pivot bits of span{vec}
  uint32_t cbits;
  double c[4], s[4];
  double* part[4];
};

template <typename T, int K>
__global__ void __launch_bounds__(kThreads) k_adj_ry_frame(typename V2<T>::type* __restrict__ psi,
                                                           typename V2<T>::type* __restrict__ lam, uint32_t n,
                                                           const RyFrameGroup gr) {
  using A = typename V2<T>::type;
  constexpr int D = 1 << K;
  uint64_t off[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    uint64_t o = 0;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (r & (1 << j)) o ^= gr.vec[j];
    off[r] = o;
  }
  double acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0.0;
  const uint64_t total = uint64_t{1} << (n - K);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t k = (uint64_t)blockIdx.x * kThreads + threadIdx.x; k < total; k += stride) {
    uint64_t base = k;
#pragma unroll
    for (int j = 0; j < K; ++j) base = insert_zero(base, gr.piv[j]);
    A a[D], l[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      a[r] = psi[base ^ off[r]];
      l[r] = lam[base ^ off[r]];
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const bool one = ((__popcll(gr.row[j] & base) ^ (gr.cbits >> j)) & 1u) != 0u;
      const double c = gr.c[j], sn = gr.s[j];
      const T ct = static_cast<T>(c), st = static_cast<T>(sn);
#pragma unroll
      for (int r = 0; r < D; ++r) {
        if (r & (1 << j)) continue;
        // logical (0, 1) members of the pair
        const A x = one ? a[r | (1 << j)] : a[r], y = one ? a[r] : a[r | (1 << j)];
        const A lx = one ? l[r | (1 << j)] : l[r], ly = one ? l[r] : l[r | (1 << j)];
        A pa, pb;  // psi' = G^dag psi
        pa.x = fma(ct, x.x, st * y.x);
        pa.y = fma(ct, x.y, st * y.y);
        pb.x = fma(ct, y.x, -(st * x.x));
        pb.y = fma(ct, y.y, -(st * x.y));
        const double mar = fma(-sn, (double)pa.x, -(c * (double)pb.x)), mai = fma(-sn, (double)pa.y, -(c * (double)pb.y));
        const double mbr = fma(c, (double)pa.x, -(sn * (double)pb.x)), mbi = fma(c, (double)pa.y, -(sn * (double)pb.y));
        acc[j] = fma(0.5 * (double)lx.x, mar, fma(0.5 * (double)lx.y, mai,
                 fma(0.5 * (double)ly.x, mbr, fma(0.5 * (double)ly.y, mbi, acc[j]))));
        A qa, qb;  // lambda' = G^dag lambda
        qa.x = fma(ct, lx.x, st * ly.x);
        qa.y = fma(ct, lx.y, st * ly.y);
        qb.x = fma(ct, ly.x, -(st * lx.x));
        qb.y = fma(ct, ly.y, -(st * lx.y));
        a[r] = one ? pb : pa;
        a[r | (1 << j)] = one ? pa : pb;
        l[r] = one ? qb : qa;
        l[r | (1 << j)] = one ? qa : qb;
      }
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      psi[base ^ off[r]] = a[r];
      lam[base ^ off[r]] = l[r];
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double2 t = block_sum(make_double2(acc[j], 0.0));
    if (threadIdx.x == 0) gr.part[j][blockIdx.x] = t.x;
  }
}

// Host frame of the backward sweep (logical i = M p ^ c): rows of M (bit
// b's parity mask over physical bits) and columns of M^-1 (bit b's pair
// vector).
struct SweepFrame {
  uint32_t n;
  std::vector<uint64_t> row, col;
  uint64_t c = 0;
  explicit SweepFrame(uint32_t n_) : n(n_), row(n_), col(n_) {
    for (uint32_t b = 0; b < n; ++b) row[b] = col[b] = uint64_t{1} << b;
  }
  void cnot(uint32_t a, uint32_t b) {  // control bit a, target bit b
    row[b] ^= row[a];
    if ((c >> a) & 1u) c ^= uint64_t{1} << b;
    col[a] ^= col[b];
  }
  void x(uint32_t b) { c ^= uint64_t{1} << b; }
};

// pivots (highest set bits after reduction, ascending) of independent vectors
void frame_pivots(const uint64_t* v, int k, uint32_t* piv) {
  std::vector<uint64_t> red;
  std::vector<uint32_t> pv;
  for (int j = 0; j < k; ++j) {
    uint64_t w = v[j];
    for (size_t i = 0; i < red.size(); ++i)
      if ((w >> pv[i]) & 1u) w ^= red[i];
    if (w == 0) throw Error(VQF_LOGIC_ERROR, "adjoint frame: dependent pair vectors");
    const uint32_t pb = 63u - static_cast<uint32_t>(__builtin_clzll(w));
    for (size_t i = 0; i < red.size(); ++i)
      if ((red[i] >> pb) & 1u) red[i] ^= w;
    red.push_back(w);
    pv.push_back(pb);
  }
  std::sort(pv.begin(), pv.end());
  for (int j = 0; j < k; ++j) piv[j] = pv[j];
}

// Self-inverse CNOT on both vectors in one pass.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_adj_cnot(typename V2<T>::type* __restrict__ psi,
                                                       typename V2<T>::type* __restrict__ lam, uint32_t n,
                                                       uint32_t pos_lo, uint32_t pos_hi, uint64_t cbit, uint64_t tbit,
                                                       uint64_t total) {
  using A = typename V2<T>::type;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t k0 = (uint64_t)blockIdx.x * kThreads + threadIdx.x; k0 < total; k0 += stride * kU) {
    A a[kU], b[kU], la[kU], lb[kU];
    uint64_t r[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t k = k0 + u * stride;
      r[u] = insert_zero(insert_zero(k, pos_lo), pos_hi) | cbit;
      if (k < total) {
        a[u] = psi[r[u]];
        b[u] = psi[r[u] | tbit];
        la[u] = lam[r[u]];
        lb[u] = lam[r[u] | tbit];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (k0 + u * stride >= total) break;
      psi[r[u]] = b[u];
      psi[r[u] | tbit] = a[u];
      lam[r[u]] = lb[u];
      lam[r[u] | tbit] = la[u];
    }
  }
}

// Fixed-order sums of per-block partials: out[j] = sum_b partials[j * nb + b]
// for the P gradient rows (scaled by 2) and the energy row (complex).
__global__ void k_adj_finish(const double* __restrict__ gpart, uint32_t P, uint32_t nb,
                             const double* __restrict__ epart, uint32_t ne, double* __restrict__ out) {
  const uint32_t j = blockIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  if (j < P) {
    for (uint32_t b = threadIdx.x; b < nb; b += kThreads) acc.x += gpart[(size_t)j * nb + b];
  } else {
    for (uint32_t b = threadIdx.x; b < ne; b += kThreads) {
      acc.x += epart[2 * b];
      acc.y += epart[2 * b + 1];
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    if (j < P) out[j] = 2.0 * acc.x;
    else {
      out[P] = acc.x;
      out[P + 1] = acc.y;
    }
  }
}

template <typename T>
void run_t(AdjointPlan& pl, const std::vector<AdjGate>& prog, const std::vector<double>& theta, double* e_out,
           double* grad_out) {
  using A = typename V2<T>::type;
  vqf_statevector* sv = pl.psi;
  A* psi = static_cast<A*>(pl.psi->amps);
  A* lam = static_cast<A*>(pl.lam->amps);
  const uint32_t n = sv->n_qubits;
  cudaStream_t st = sv->stream;
  const auto grid_for = [](uint64_t items) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((items + kThreads * kU - 1) / (kThreads * kU), kBlocks)));
  };
  // lambda = H psi, E = <psi|lambda>
  const uint32_t B = pl.tile_bits;
  k_apply_ham<T><<<pl.nb_ham, kThreads, sizeof(double2) << B, st>>>(psi, lam, n, B, pl.hd, pl.epart);
  VQF_LAUNCHED();
  // backward sweep.  Programs of RYs, CNOTs and Xs (the hardware-efficient
  // ansatz) run in a GF(2) frame: CNOT / X chains only update the frame and
  // every RY group is one frame-aware two-vector pass (no permutation passes
  // over psi and lambda); other programs move the data.
  bool frame_ok = !std::getenv("VQF_ADJ_NO_FRAME");
  for (const AdjGate& g : prog)
    frame_ok = frame_ok && ((g.kind == VQF_GATE_RY && g.param >= 0) || (g.kind == VQF_GATE_CNOT && g.param < 0) ||
                            (g.kind == VQF_GATE_PAULI_X && g.param < 0));
  if (frame_ok) {
    SweepFrame fr(n);
    const auto bit_of = [n](uint32_t w) { return n - 1 - w; };
    for (size_t gi = prog.size(); gi-- > 0;) {
      const AdjGate& g = prog[gi];
      if (g.kind == VQF_GATE_CNOT) {
        fr.cnot(bit_of(g.wires[0]), bit_of(g.wires[1]));
        continue;
      }
      if (g.kind == VQF_GATE_PAULI_X) {
        fr.x(bit_of(g.wires[0]));
        continue;
      }
      size_t cnt = 1;  // consecutive RYs on distinct wires (they commute)
      while (cnt < 4 && gi >= cnt && prog[gi - cnt].kind == VQF_GATE_RY) {
        bool distinct = true;
        for (size_t q = 0; q < cnt; ++q) distinct = distinct && prog[gi - cnt].wires[0] != prog[gi - q].wires[0];
        if (!distinct) break;
        ++cnt;
      }
      RyFrameGroup gr{};
      for (size_t q = 0; q < cnt; ++q) {  // gate q of the group = prog[gi - q] (backward order)
        const AdjGate& h = prog[gi - q];
        const uint32_t b = bit_of(h.wires[0]);
        const double th = theta[h.param];
        gr.vec[q] = fr.col[b];
        gr.row[q] = fr.row[b];
        if ((fr.c >> b) & 1u) gr.cbits |= 1u << q;
        gr.c[q] = std::cos(0.5 * th);
        gr.s[q] = std::sin(0.5 * th);
        gr.part[q] = pl.gpart + (size_t)h.param * pl.nb;
      }
      frame_pivots(gr.vec, static_cast<int>(cnt), gr.piv);
      switch (cnt) {
        case 1: k_adj_ry_frame<T, 1><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, gr); break;
        case 2: k_adj_ry_frame<T, 2><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, gr); break;
        case 3: k_adj_ry_frame<T, 3><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, gr); break;
        default: k_adj_ry_frame<T, 4><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, gr); break;
      }
      VQF_LAUNCHED();
      gi -= cnt - 1;
    }
  }
  for (size_t gi = frame_ok ? 0 : prog.size(); gi-- > 0;) {
    const AdjGate& g = prog[gi];
    const auto bit_of = [n](uint32_t w) { return n - 1 - w; };
    // a run of >= 2 parameter-free self-inverse gates (CNOT / X chains) is
    // un-applied to both vectors by the fused tile path: one pass per vector
    // for the run instead of one two-vector pass per gate
    size_t run0 = gi + 1;
    while (run0 > 0 && prog[run0 - 1].param < 0 &&
           (prog[run0 - 1].kind == VQF_GATE_CNOT || prog[run0 - 1].kind == VQF_GATE_PAULI_X))
      --run0;
    if (gi + 1 - run0 >= 2) {
      std::vector<TGate> inv;
      for (size_t k = gi + 1; k-- > run0;) {  // reversed: (G_m ... G_1)^dag = G_1 ... G_m for self-inverse G
        const AdjGate& q = prog[k];
        inv.push_back(TGate{q.kind, q.kind == VQF_GATE_CNOT ? 2u : 1u, {q.wires[0], q.wires[1], 0, 0}, -1, 1.0, 0.0});
      }
      run_circuit_tiled(pl.psi, inv, nullptr);
      cudaStream_t own = pl.lam->stream;  // keep every launch of the sweep on psi's stream
      pl.lam->stream = st;
      run_circuit_tiled(pl.lam, inv, nullptr);
      pl.lam->stream = own;
      gi = run0;
      continue;
    }
    // up to three consecutive RYs on distinct wires (they commute): one
    // two-vector pass for the group instead of one per gate
    if (g.kind == VQF_GATE_RY && g.param >= 0) {
      size_t cnt = 1;
      while (cnt < 4 && gi >= cnt && prog[gi - cnt].kind == VQF_GATE_RY && prog[gi - cnt].param >= 0) {
        bool distinct = true;
        for (size_t q = 0; q < cnt; ++q) distinct = distinct && prog[gi - cnt].wires[0] != prog[gi - q].wires[0];
        if (!distinct) break;
        ++cnt;
      }
      if (cnt >= 2) {
        RyGroup gr{};
        for (size_t q = 0; q < cnt; ++q) {  // gate q of the group = prog[gi - q] (backward order)
          const AdjGate& h = prog[gi - q];
          const double th = theta[h.param];
          gr.bit[q] = bit_of(h.wires[0]);
          gr.c[q] = std::cos(0.5 * th);
          gr.s[q] = std::sin(0.5 * th);
          gr.part[q] = pl.gpart + (size_t)h.param * pl.nb;
        }
        if (cnt == 2) k_adj_ry_multi<T, 2><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, gr);
        else if (cnt == 3) k_adj_ry_multi<T, 3><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, gr);
        else k_adj_ry_multi<T, 4><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, gr);
        VQF_LAUNCHED();
        gi -= cnt - 1;
        continue;
      }
    }
    if (g.kind == VQF_GATE_CNOT) {
      const uint32_t bc = bit_of(g.wires[0]), bt = bit_of(g.wires[1]);
      const uint64_t total = uint64_t{1} << (n - 2);
      k_adj_cnot<T><<<grid_for(total), kThreads, 0, st>>>(psi, lam, n, std::min(bc, bt), std::max(bc, bt),
                                                           uint64_t{1} << bc, uint64_t{1} << bt, total);
    } else {
      const double th = theta[g.param];
      const double c = std::cos(0.5 * th), s = std::sin(0.5 * th);
      double* gp = pl.gpart + (size_t)g.param * pl.nb;
      if (g.kind == VQF_GATE_RY) {
        const uint32_t b = bit_of(g.wires[0]);
        const uint64_t total = uint64_t{1} << (n - 1);
        k_adj_givens<T, 1><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, 0, uint64_t{1} << b, total, b, 0, 0, 0, c, s, gp);
      } else if (g.kind == VQF_GATE_DOUBLE_EXCITATION) {
        uint32_t pos[4];
        uint64_t m[4];
        for (int i = 0; i < 4; ++i) {
          pos[i] = bit_of(g.wires[i]);
          m[i] = uint64_t{1} << pos[i];
        }
        std::sort(pos, pos + 4);
        const uint64_t total = uint64_t{1} << (n - 4);
        k_adj_givens<T, 4><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, m[0] | m[1], m[2] | m[3], total, pos[0], pos[1],
                                                       pos[2], pos[3], c, s, gp);
      } else {  // SingleExcitation
        uint32_t pos[2] = {bit_of(g.wires[0]), bit_of(g.wires[1])};
        const uint64_t m0 = uint64_t{1} << pos[0], m1 = uint64_t{1} << pos[1];
        std::sort(pos, pos + 2);
        const uint64_t total = uint64_t{1} << (n - 2);
        k_adj_givens<T, 2><<<pl.nb, kThreads, 0, st>>>(psi, lam, n, m0, m1, total, pos[0], pos[1], 0, 0, c, s, gp);
      }
    }
    VQF_LAUNCHED();
  }
  const uint32_t P = pl.P;
  k_adj_finish<<<P + 1, kThreads, 0, st>>>(pl.gpart, P, pl.nb, pl.epart, pl.nb_ham, pl.dout);
  VQF_LAUNCHED();
  VQF_CUDA(cudaMemcpyAsync(pl.hout, pl.dout, (P + 2) * sizeof(double), cudaMemcpyDeviceToHost, st));
  VQF_CUDA(cudaStreamSynchronize(st));
  VQF_CUDA(cudaGetLastError());
  std::memcpy(grad_out, pl.hout, P * sizeof(double));
  e_out[0] = pl.hout[P];
  e_out[1] = pl.hout[P + 1];
}

}  // namespace

bool AdjointPlan::supports(const CompiledHam& h, uint32_t n_qubits) {
  const uint32_t tb = std::min<uint32_t>(n_qubits, kTileBits);
  const uint64_t lo_mask = (uint64_t{1} << tb) - 1;
  uint32_t mixed = 0;
  for (uint32_t t = h.group_offset[0]; t < h.group_offset[1]; ++t)
    mixed += (h.terms[t].yz & ~lo_mask) != 0 && (h.terms[t].yz & lo_mask) != 0;
  const size_t groups = h.group_offset.size() >= 2 ? h.group_offset.size() - 2 : 0;
  const size_t off_terms = h.group_offset.empty() ? 0 : h.group_offset.back() - h.group_offset[1];
  return mixed <= 64 && groups <= kMaxGroups && off_terms <= kMaxTerms;
}

void AdjointPlan::init(vqf_statevector* psi_, vqf_statevector* lam_, const CompiledHam& h, uint32_t n_params) {
  psi = psi_;
  lam = lam_;
  P = n_params;
  const uint32_t n = psi->n_qubits;
  tile_bits = std::min<uint32_t>(n, kTileBits);
  nb = kBlocks;
  nb_ham = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t{1} << (n - tile_bits), kBlocks)));
  // Hamiltonian tables: diagonal split + off-diagonal groups
  const uint64_t lo_mask = (uint64_t{1} << tile_bits) - 1;
  std::vector<MaskTerm> lo, hi, mx, off;
  std::vector<uint64_t> flips;
  std::vector<uint32_t> goff{0};
  for (uint32_t t = h.group_offset[0]; t < h.group_offset[1]; ++t) {
    const MaskTerm& m = h.terms[t];
    if ((m.yz & ~lo_mask) == 0) lo.push_back(m);
    else if ((m.yz & lo_mask) == 0) hi.push_back(m);
    else mx.push_back(m);
  }
  if (mx.size() > 64)
    throw_invalid("adjoint gradient: " + std::to_string(mx.size()) +
                  " diagonal terms straddle the tile boundary (limit 64; use parameter shift)");
  std::vector<uint32_t> ghi;
  for (size_t g = 1; g + 1 < h.group_offset.size(); ++g) {
    flips.push_back(h.group_flip[g]);
    uint32_t nh = 0;
    for (uint32_t t = h.group_offset[g]; t < h.group_offset[g + 1]; ++t)  // tile-constant terms first
      if ((h.terms[t].yz & lo_mask) == 0) {
        off.push_back(h.terms[t]);
        ++nh;
      }
    for (uint32_t t = h.group_offset[g]; t < h.group_offset[g + 1]; ++t)
      if ((h.terms[t].yz & lo_mask) != 0) off.push_back(h.terms[t]);
    ghi.push_back(nh);
    goff.push_back(static_cast<uint32_t>(off.size()));
  }
  if (flips.size() > kMaxGroups || off.size() > kMaxTerms)
    throw_invalid("adjoint gradient: " + std::to_string(flips.size()) + " flip groups / " + std::to_string(off.size()) +
                  " off-diagonal terms exceed the tables (" + std::to_string(kMaxGroups) + " / " +
                  std::to_string(kMaxTerms) + "; use parameter shift)");
  std::vector<unsigned char> blob;
  auto put = [&](const void* p, size_t bytes) {
    const size_t at = (blob.size() + 15) & ~size_t{15};
    blob.resize(at + std::max<size_t>(bytes, 16));
    if (bytes) std::memcpy(blob.data() + at, p, bytes);
    return at;
  };
  const size_t o_lo = put(lo.data(), lo.size() * sizeof(MaskTerm));
  const size_t o_hi = put(hi.data(), hi.size() * sizeof(MaskTerm));
  const size_t o_mx = put(mx.data(), mx.size() * sizeof(MaskTerm));
  const size_t o_fl = put(flips.data(), flips.size() * sizeof(uint64_t));
  const size_t o_go = put(goff.data(), goff.size() * sizeof(uint32_t));
  const size_t o_te = put(off.data(), off.size() * sizeof(MaskTerm));
  const size_t o_gh = put(ghi.data(), ghi.size() * sizeof(uint32_t));
  const size_t o_gp = put(nullptr, 0);
  blob.resize(o_gp);
  const size_t bytes = o_gp + sizeof(double) * ((size_t)P * nb + 2 * (size_t)nb_ham + P + 2);
  VQF_CUDA(cudaSetDevice(psi->device));
  // stream-ordered pool allocation (no device-wide synchronisation on the
  // free); the small pinned result block is cached per thread
  free_stream = psi->own_stream;
  VQF_CUDA(cudaMallocAsync(&dev, bytes, free_stream));
  VQF_CUDA(cudaMemcpyAsync(dev, blob.data(), blob.size(), cudaMemcpyHostToDevice, free_stream));
  VQF_CUDA(cudaStreamSynchronize(free_stream));
  {
    thread_local double* pin = nullptr;
    thread_local size_t pin_cap = 0;
    if (pin_cap < P + 2) {
      if (pin) VQF_CUDA(cudaFreeHost(pin));
      pin = nullptr;
      pin_cap = std::max<size_t>(P + 2, 256);
      VQF_CUDA(cudaMallocHost(&pin, sizeof(double) * pin_cap));
    }
    hout = pin;
  }
  auto* d = static_cast<unsigned char*>(dev);
  hd = HamDevC{reinterpret_cast<const MaskTerm*>(d + o_lo), reinterpret_cast<const MaskTerm*>(d + o_hi),
               reinterpret_cast<const MaskTerm*>(d + o_mx), static_cast<uint32_t>(lo.size()),
               static_cast<uint32_t>(hi.size()), static_cast<uint32_t>(mx.size()),
               reinterpret_cast<const uint64_t*>(d + o_fl), reinterpret_cast<const uint32_t*>(d + o_go),
               reinterpret_cast<const uint32_t*>(d + o_gh), reinterpret_cast<const MaskTerm*>(d + o_te),
               static_cast<uint32_t>(flips.size())};
  gpart = reinterpret_cast<double*>(d + o_gp);
  epart = gpart + (size_t)P * nb;
  dout = epart + 2 * (size_t)nb_ham;
  const int smem = static_cast<int>(sizeof(double2) << tile_bits);
  VQF_CUDA(cudaFuncSetAttribute(k_apply_ham<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  VQF_CUDA(cudaFuncSetAttribute(k_apply_ham<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  VQF_CUDA(cudaMemsetAsync(gpart, 0, sizeof(double) * (size_t)P * nb, psi->stream));
}

AdjointPlan::~AdjointPlan() {
  if (dev) cudaFreeAsync(dev, free_stream);
}

void AdjointPlan::run(const std::vector<AdjGate>& prog, const std::vector<double>& theta, double* e_out,
                      double* grad_out) {
  VQF_CUDA(cudaSetDevice(psi->device));
  if (psi->dtype == VQF_F64)
    run_t<double>(*this, prog, theta, e_out, grad_out);
  else
    run_t<float>(*this, prog, theta, e_out, grad_out);
}

}  // namespace vqf
