// Gate fusion through shared-memory tiles.
//
// A pass works on "gathered tiles": 2^B contiguous low-index amplitudes
// (512 B runs) times 2^k chosen high index bits h_0..h_{k-1} (B + k = 11
// local bits for fp64, 32 KB).  Runs arrive by TMA tensor loads with the
// 128 B swizzle; three consumer groups per CTA each own a two-stage ring and
// a named barrier.  Every gate of the pass whose wires map into the local
// bits is merged into fused ops of <= 3 bits (4 with a DoubleExcitation);
// each op is one real 2^m x 2^m matrix composed per CTA and applied to the
// thread's amplitudes in registers (fp64 3-bit ops on the FP64 tensor cores,
// mma.sync m8n8k4).  X / CNOT-only passes are an affine map of the local
// index applied in the write-back.  One HBM read + write of the state per
// pass instead of per gate.
//
// The host scheduler walks the circuit's dependency DAG (gates sharing a wire
// keep their order; gates on disjoint wires commute) and, among ready gates
// that fit, takes the one adding the fewest new high bits (then sharing the
// most): for the hardware-efficient ansatz the CNOT chain advances five
// wires per pass.
//
// Composed matrices (and FMA / MMA accumulation) change rounding only:
// amplitudes agree with the per-gate kernels to ~1e-16 (tests/).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "tile.cuh"

namespace vqf {

namespace {

constexpr int kMaxOps = 64;        // TileParams stays under the 4 KB kernel-parameter limit
constexpr int kMaxHigh = 6;
constexpr int kTileBlocks = 148;   // persistent: one CTA per SM
// four single-buffered consumer groups (128 KB of tiles): a group loads its
// next tile after writing back the current one while the other three
// compute; measured against 3 groups x 2 stages (the previous default, 192
// KB), 5 x 1 and 6 x 1 (scripts/ab_variants.sh: HEA(2) n = 30 80.5 vs 84.2,
// 89.2, 121.5 ms)
#ifndef VQF_TILE_GROUPS
#define VQF_TILE_GROUPS 4
#endif
#ifndef VQF_TILE_STAGES
#define VQF_TILE_STAGES 1
#endif
#ifndef VQF_TILE_LB
#define VQF_TILE_LB 11  // fp64 tile = 2^11 amplitudes (32 KB); fp32 one bit more
#endif
#ifndef VQF_TILE_NT
#define VQF_TILE_NT 128
#endif
constexpr int kGroups = VQF_TILE_GROUPS;  // consumer groups per CTA
constexpr int kNT = VQF_TILE_NT;          // threads per group (half of it for 4-bit fused ops in fp64)
constexpr int kStages = VQF_TILE_STAGES;  // TMA ring depth per group (32 KB tiles)
constexpr int kMaxFuse = 4;        // local bits of one fused op (16 amplitudes per thread)
constexpr uint32_t kMatElems = 2560;
constexpr int kDq = 4;  // item groups per step of the tensor-core fused op
constexpr uint32_t kNoMma = 1u << 31;  // TileFop::ipos: run this op on the FMA path  // composed fused-op matrices per pass (20 KB of fp64)
// fp64 passes run 512 threads with fused ops of <= 3 bits (8 amplitudes in
// registers, <= 128 registers), or 256 threads when a DoubleExcitation needs
// a 4-bit op; fp32 always 512 threads x <= 4 bits

// One gate inside a fused op: pairs (r | A, r | B) of the op's 2^m register
// slots, for every r with the bits of A | B clear; ROT: a' = c a - s b,
// b' = s a + c b (statevector.hpp:160-163, :195-196), else swap.
//   X / RY on slot bit j : A = 0,        B = 1 << j
//   CNOT (c, t)          : A = C,        B = C | T
//   SingleExcitation     : A = 1 << w0,  B = 1 << w1
//   DoubleExcitation     : A = w0 | w1,  B = w2 | w3
struct TileSub {
  uint32_t code;  // (rot << 8) | (A << 4) | B
  int32_t param;  // per-entry (c, s) index or -1
  double c, s;
};

// A fused op: m <= 4 local bit positions (ascending, 8 bits each) and its
// gates [sub0, sub0 + n_sub).  Each thread loads the 2^m amplitudes of one
// work item into registers, applies all the gates, and stores them back:
// one shared-memory round trip per op instead of per gate.
struct TileFop {
  uint32_t m, pos, sub0, n_sub, uoff;  // uoff: the op's matrix in the composed-matrix area
  // tensor-core ops: the two free local bits that enumerate the four items of
  // an MMA column group (chosen on the host against shared-memory bank
  // conflicts; 0 = the lowest free bits), 5 bits each
  uint32_t ipos;
};

struct TileParams {
  uint32_t n, B, k, n_fops, batch;
  uint32_t hb[kMaxHigh];  // global bit of local bit B + j, ascending
  const double* cs;
  // Permutation-only pass (every gate X / CNOT): no fused ops; the tile is
  // written back as out[L] = in[F(L)] with F(L) = c ^ xor of col[b] over
  // the set bits b of L (an affine map over GF(2) on the local index).
  uint32_t perm_only, perm_c;
  uint32_t perm_col[16];
  TileFop fops[kMaxOps];
  TileSub subs[kMaxOps];
};

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

__device__ __forceinline__ uint64_t insert_zero64(uint64_t k, uint32_t bit) {
  const uint64_t low = k & ((uint64_t{1} << bit) - 1);
  return ((k >> bit) << (bit + 1)) | low;
}

// ---- TMA helpers (sm_90+ PTX; SASS: UTMALDG / SYNCS)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// one 4 KB run (box {128 B, 32 rows, 1}) of the state, 128 B-swizzled into
// shared memory; completion counted on the mbarrier
__device__ __forceinline__ void tma_load_run(void* dst, const CUtensorMap* map, int32_t row, int32_t entry,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(0), "r"(row), "r"(entry), "r"(smem_addr(bar))
      : "memory");
}

// Shared-memory slot of local amplitude L under the TMA 128 B swizzle: the
// 16-byte chunk index (bits 4..6 of the byte offset) is xor-ed with the
// 128-byte row index mod 8 (bits 7..9), so amplitudes one row apart land in
// different banks.
template <typename T>
__device__ __forceinline__ uint32_t swz(uint32_t L) {
  if (sizeof(T) == 8) return L ^ ((L >> 3) & 7u);        // 16 B amplitude = one chunk
  return L ^ (((L >> 4) & 7u) << 1);                     // 8 B amplitude: chunk = L >> 1
}

// Global start index of run j (0 <= j < 2^k) of tile `tile`.
__device__ __forceinline__ uint64_t run_start(const TileParams& p, uint64_t tile, uint32_t j) {
  uint64_t base = tile << p.B;
  for (uint32_t m = 0; m < p.k; ++m) base = insert_zero64(base, p.hb[m]);
  for (uint32_t m = 0; m < p.k; ++m) base |= (uint64_t)((j >> m) & 1u) << p.hb[m];
  return base;
}

// Every gate here is a real orthogonal map on its pairs, so a fused op is
// one real 2^m x 2^m matrix U (row-major, in shared memory) composed once
// per CTA from its gates and the CTA's batch entry angles: start from the
// identity and apply each gate to the rows of every column.  The angles are
// staged in shared memory first (one parallel round of global loads instead
// of a dependent L2 round trip per gate) and each thread composes one
// (op, column) pair, so the serial chain is one op's gates: batched states
// launch a CTA set per entry and pay this once per (CTA, entry).
template <typename T>
__device__ void compose_fops(const TileParams& p, T* U) {
  __shared__ double2 sc[kMaxOps];
  uint32_t n_subs = 0;
  for (uint32_t o = 0; o < p.n_fops; ++o) n_subs = max(n_subs, p.fops[o].sub0 + p.fops[o].n_sub);
  for (uint32_t q = threadIdx.x; q < n_subs; q += blockDim.x) {
    const TileSub& g = p.subs[q];
    double2 v = make_double2(g.c, g.s);
    if (g.param >= 0) v = *reinterpret_cast<const double2*>(p.cs + 2 * ((size_t)g.param * p.batch + blockIdx.y));
    sc[q] = v;
  }
  __syncthreads();
  for (uint32_t w = threadIdx.x;; w += blockDim.x) {
    uint32_t o = 0, col = w;
    while (o < p.n_fops && col >= (1u << p.fops[o].m)) col -= 1u << p.fops[o].m, ++o;
    if (o >= p.n_fops) break;
    const TileFop& f = p.fops[o];
    const uint32_t d = 1u << f.m;
    T* u = U + f.uoff;
    for (uint32_t r = 0; r < d; ++r) u[r * d + col] = r == col ? T(1) : T(0);
    for (uint32_t q = 0; q < f.n_sub; ++q) {
      const TileSub& g = p.subs[f.sub0 + q];
      const double c = sc[f.sub0 + q].x, sn = sc[f.sub0 + q].y;
      const uint32_t A = (g.code >> 4) & 15u, B = g.code & 15u, S = A | B;
      for (uint32_t r = 0; r < d; ++r) {
        if (r & S) continue;
        const T x = u[(r | A) * d + col], y = u[(r | B) * d + col];
        if (g.code >> 8) {  // a' = c a - s b, b' = s a + c b (statevector.hpp:160-163, :195-196)
          u[(r | A) * d + col] = static_cast<T>(c) * x - static_cast<T>(sn) * y;
          u[(r | B) * d + col] = static_cast<T>(sn) * x + static_cast<T>(c) * y;
        } else {
          u[(r | A) * d + col] = y;
          u[(r | B) * d + col] = x;
        }
      }
    }
  }
}

// One fused op over the whole tile: work item w -> base with zeros at the
// op's bits; 2^M amplitudes in registers, y = U x with U broadcast from
// shared memory.  The swizzle is xor-linear and base / slot offsets have
// disjoint bits, so slot addresses are swz(base) ^ swz(offset).
template <int M, typename T, int NT>
__device__ __forceinline__ void run_fop(typename V2<T>::type* t, uint32_t NL, const TileFop& f, const T* U,
                                        uint32_t gt) {
  using A = typename V2<T>::type;
  constexpr int D = 1 << M;
  uint32_t pos[M];
#pragma unroll
  for (int j = 0; j < M; ++j) pos[j] = (f.pos >> (8 * j)) & 0xffu;
  uint32_t sd[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    uint32_t d = 0;
#pragma unroll
    for (int j = 0; j < M; ++j)
      if (r & (1 << j)) d |= 1u << pos[j];
    sd[r] = swz<T>(d);
  }
  const T* u = U + f.uoff;
  const uint32_t items = NL >> M;
  const auto base_of = [&](uint32_t w) {
    uint32_t base = w;
#pragma unroll
    for (int j = 0; j < M; ++j) base = ((base >> pos[j]) << (pos[j] + 1)) | (base & ((1u << pos[j]) - 1));
    return swz<T>(base);
  };
  using P2 = typename V2<T>::type;
  if constexpr (M == 3 && sizeof(T) == 8) {
    if (f.ipos != kNoMma && items >= 4 * NT / 32 * kDq) {
      // fp64 tensor cores: Y (8 slots x 2 columns per item) = U (8 x 8) X as
      // mma.sync m8n8k4 f64 over groups of four items (eight real columns:
      // item-major, re / im).  Fragments (PTX m8n8k4 .f64, g = lane / 4,
      // t = lane % 4): A[g][t] -> U[g][k0 + t]; B[t][g] -> X[k0 + t][col g] =
      // component (g & 1) of slot k0 + t of item g / 2; D[g][2t + i] ->
      // component i of slot g of item t.  One warp instruction does 256
      // FMAs; kDq item groups per step keep loads and MMAs in flight.
      const uint32_t lane = gt & 31u, g = lane >> 2, tq = lane & 3u;
      const double a_lo = u[g * 8 + tq], a_hi = u[g * 8 + 4 + tq];
      const double* td = reinterpret_cast<const double*>(t);
      // item 4q + i = base(4q) | base(i) for i < 4 (disjoint bits) and the
      // swizzle is xor-linear, so the per-lane parts are fixed per op and
      // each item group costs one (warp-uniform) base computation
      // item 4q + i: i on the two chosen free bits c1, c2, q on the other
      // free bits (ascending): base = ins2(q) | dep2(i), both swizzled apart
      const uint32_t c1 = f.ipos & 31u, c2 = (f.ipos >> 5) & 31u;
      const auto dep2 = [&](uint32_t i) { return swz<T>(((i & 1u) << c1) | (((i >> 1) & 1u) << c2)); };
      uint32_t p5[M + 2];  // zero-insertion positions for q: op bits + c1, c2, ascending
      {
        uint32_t all[M + 2];
#pragma unroll
        for (int j = 0; j < M; ++j) all[j] = pos[j];
        all[M] = c1;
        all[M + 1] = c2;
#pragma unroll
        for (int i = 0; i < M + 2; ++i)
#pragma unroll
          for (int j = i + 1; j < M + 2; ++j)
            if (all[j] < all[i]) {
              const uint32_t tmp = all[i];
              all[i] = all[j];
              all[j] = tmp;
            }
#pragma unroll
        for (int j = 0; j < M + 2; ++j) p5[j] = all[j];
      }
      const auto ins2 = [&](uint32_t q) {
        uint32_t b = q;
#pragma unroll
        for (int j = 0; j < M + 2; ++j) b = ((b >> p5[j]) << (p5[j] + 1)) | (b & ((1u << p5[j]) - 1));
        return swz<T>(b);
      };
      const uint32_t in_lo = 2 * (dep2(g >> 1) ^ sd[tq]) + (g & 1u);
      const uint32_t in_hi = 2 * (dep2(g >> 1) ^ sd[4 + tq]) + (g & 1u);
      const uint32_t out_off = dep2(tq) ^ sd[g];
      const uint32_t groups = items >> 2, wstride = NT / 32;
      // groups q0 + d (q0 a multiple of kDq): base(4 (q0 + d)) =
      // base(4 q0) | base(4 d), so one base per step plus fixed offsets
      uint32_t offd[kDq];
#pragma unroll
      for (int d = 0; d < kDq; ++d) offd[d] = ins2(d);
      for (uint32_t q0 = (gt >> 5) * kDq; q0 < groups; q0 += wstride * kDq) {
        double b_lo[kDq], b_hi[kDq], c0[kDq], c1[kDq];
        uint32_t sb_out[kDq];
        const uint32_t sbq = ins2(q0);
#pragma unroll
        for (int d = 0; d < kDq; ++d) {
          const uint32_t sb4 = sbq ^ offd[d];
          sb_out[d] = sb4 ^ out_off;
          b_lo[d] = td[(2 * sb4) ^ in_lo];
          b_hi[d] = td[(2 * sb4) ^ in_hi];
          c0[d] = 0.0;
          c1[d] = 0.0;
        }
#pragma unroll
        for (int d = 0; d < kDq; ++d)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(c0[d]), "+d"(c1[d])
                       : "d"(a_lo), "d"(b_lo[d]));
#pragma unroll
        for (int d = 0; d < kDq; ++d)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(c0[d]), "+d"(c1[d])
                       : "d"(a_hi), "d"(b_hi[d]));
#pragma unroll
        for (int d = 0; d < kDq; ++d) {
          A y;
          y.x = c0[d];
          y.y = c1[d];
          t[sb_out[d]] = y;
        }
      }
      return;
    }
  }
  if constexpr (M <= 3) {
    // two work items per step: both items' loads in flight together and each
    // 16-byte matrix-row load feeds both (the tile has 2 x NT items for m = 3)
    for (uint32_t w = gt; w < items; w += 2 * NT) {
      const bool two = w + NT < items;
      const uint32_t sb0 = base_of(w), sb1 = two ? base_of(w + NT) : sb0;
      A x0[D], x1[D];
#pragma unroll
      for (int r = 0; r < D; ++r) {
        x0[r] = t[sb0 ^ sd[r]];
        x1[r] = t[sb1 ^ sd[r]];
      }
#pragma unroll
      for (int r = 0; r < D; ++r) {
        A a0, a1, b0, b1;  // item 0 / item 1, even / odd columns
        a0.x = a0.y = a1.x = a1.y = b0.x = b0.y = b1.x = b1.y = T(0);
        if constexpr (D == 1) {
          a0.x = u[0] * x0[0].x;
          a0.y = u[0] * x0[0].y;
          b0.x = u[0] * x1[0].x;
          b0.y = u[0] * x1[0].y;
        } else {
          const P2* row = reinterpret_cast<const P2*>(u + r * D);
#pragma unroll
          for (int c = 0; c < D; c += 2) {
            const P2 m = row[c / 2];
            a0.x = fma(m.x, x0[c].x, a0.x);
            a0.y = fma(m.x, x0[c].y, a0.y);
            a1.x = fma(m.y, x0[c + 1].x, a1.x);
            a1.y = fma(m.y, x0[c + 1].y, a1.y);
            b0.x = fma(m.x, x1[c].x, b0.x);
            b0.y = fma(m.x, x1[c].y, b0.y);
            b1.x = fma(m.y, x1[c + 1].x, b1.x);
            b1.y = fma(m.y, x1[c + 1].y, b1.y);
          }
        }
        A y0, y1;
        y0.x = a0.x + a1.x;
        y0.y = a0.y + a1.y;
        y1.x = b0.x + b1.x;
        y1.y = b0.y + b1.y;
        t[sb0 ^ sd[r]] = y0;
        if (two) t[sb1 ^ sd[r]] = y1;
      }
    }
  } else {
    for (uint32_t w = gt; w < items; w += NT) {
      const uint32_t sb = base_of(w);
      A x[D];
#pragma unroll
      for (int r = 0; r < D; ++r) x[r] = t[sb ^ sd[r]];
#pragma unroll
      for (int r = 0; r < D; ++r) {
        // row r of U as 16-byte broadcast loads; two accumulation chains per
        // component (even / odd columns) halve the dependent-FMA depth
        A y0, y1;
        y0.x = y0.y = y1.x = y1.y = T(0);
        const P2* row = reinterpret_cast<const P2*>(u + r * D);
#pragma unroll
        for (int c = 0; c < D; c += 2) {
          const P2 m = row[c / 2];
          y0.x = fma(m.x, x[c].x, y0.x);
          y0.y = fma(m.x, x[c].y, y0.y);
          y1.x = fma(m.y, x[c + 1].x, y1.x);
          y1.y = fma(m.y, x[c + 1].y, y1.y);
        }
        A y;
        y.x = y0.x + y1.x;
        y.y = y0.y + y1.y;
        t[sb ^ sd[r]] = y;
      }
    }
  }
}

// Named barrier over the NT threads of one consumer group (ids 1, 2; 0 is
// __syncthreads).
template <int NT>
__device__ __forceinline__ void group_sync(uint32_t group) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "r"(NT) : "memory");
}

// Persistent tile kernel.  The CTA runs two independent consumer groups of
// NT threads; group g takes every other tile of the CTA's sequence, with its
// own kStages-deep TMA ring (lane 0 of the group's first warp arms the
// stage's mbarrier with the tile's bytes, its lanes issue the 2^k runs as
// TMA tensor loads, 128 B swizzle) and its own named barrier, so one group's
// barrier waits and shared-memory phases overlap the other group's work.
// Each tile: the pass's fused ops (y = U x on 2^m amplitudes per thread),
// then coalesced 16-byte stores back to HBM.
template <typename T, int NT, int MAXM, bool PERM>
__global__ void __launch_bounds__(kGroups * NT, 1)
    k_tile(typename V2<T>::type* __restrict__ a, const __grid_constant__ CUtensorMap map, const TileParams p) {
  using A = typename V2<T>::type;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 128 B swizzle atoms are 1024 B: align the rings (the launch adds 1 KB
  // slack); indexing smem_raw keeps the pointer in the shared window (LDS/STS)
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const uint32_t LB = p.B + p.k, NL = 1u << LB;
  const uint32_t run_amps = 1u << p.B, n_runs = 1u << p.k;
  const uint32_t tile_bytes = NL * sizeof(A), run_bytes = run_amps * sizeof(A);
  const uint32_t amps_per_row = 128 / sizeof(A);
  const uint32_t group = threadIdx.x / NT, gt = threadIdx.x % NT;
  unsigned char* ring = smem + (size_t)group * kStages * tile_bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kGroups * kStages * (size_t)tile_bytes) + group * kStages;
  T* U = reinterpret_cast<T*>(smem + kGroups * kStages * (size_t)tile_bytes + 256);  // composed fused-op matrices
  __shared__ uint64_t run_off_all[kGroups][1 << kMaxHigh];
  uint64_t* run_off = run_off_all[group];
  A* s = a + ((uint64_t)blockIdx.y << p.n);
  const uint64_t n_tiles = uint64_t{1} << (p.n - LB);
  if (gt == 0) {
    if (group == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
    for (int st = 0; st < kStages; ++st) mbar_init(&bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (!PERM) compose_fops<T>(p, U);
  // permutation-only pass: F as two 64-entry tables (bits 0-5, bits 6-11)
  __shared__ uint16_t ftab[PERM ? 2 : 1][64];
  if constexpr (PERM)
    for (uint32_t e = threadIdx.x; e < 128; e += blockDim.x) {
      const uint32_t half = e >> 6, j = e & 63u;
      uint32_t v = 0;
      for (uint32_t b = 0; b < 6; ++b)
        if ((j >> b) & 1u) v ^= p.perm_col[6 * half + b];
      ftab[half][j] = static_cast<uint16_t>(v);
    }
  __syncthreads();
  const auto stage_buf = [&](int st) { return reinterpret_cast<A*>(ring + (size_t)st * tile_bytes); };
  const auto issue_load = [&](uint64_t tile, int st) {
    const uint32_t lane = gt;
    if (lane == 0) mbar_expect_tx(&bar[st], tile_bytes);
    unsigned char* dst = reinterpret_cast<unsigned char*>(stage_buf(st));
    for (uint32_t j = lane; j < n_runs; j += 32)
      tma_load_run(dst + (size_t)j * run_bytes, &map, static_cast<int32_t>(run_start(p, tile, j) / amps_per_row),
                   static_cast<int32_t>(blockIdx.y), &bar[st]);
  };
  // the group's tiles: blockIdx.x + (kGroups i + group) * gridDim.x
  const uint64_t step = kGroups * (uint64_t)gridDim.x;
  const uint64_t first = blockIdx.x + (uint64_t)group * gridDim.x;
  if (gt < 32)
    for (int st = 0; st < kStages - 1; ++st) {
      const uint64_t t0 = first + (uint64_t)st * step;
      if (t0 < n_tiles) issue_load(t0, st);
    }
  uint64_t tile = first;
  for (uint32_t it = 0; tile < n_tiles; tile += step, ++it) {
    const int cur = it % kStages;
    const uint64_t ahead = tile + (uint64_t)(kStages - 1) * step;
    // that stage's previous tile was written back before the group barrier
    // that closed the previous iteration
    if (gt < 32 && ahead < n_tiles) issue_load(ahead, (it + kStages - 1) % kStages);
    mbar_wait(&bar[cur], (it / kStages) & 1u);
    A* t = stage_buf(cur);
    for (uint32_t o = 0; o < (PERM ? 0u : p.n_fops); ++o) {
      const TileFop f = p.fops[o];
      switch (f.m) {
        case 1: run_fop<1, T, NT>(t, NL, f, U, gt); break;
        case 2: run_fop<2, T, NT>(t, NL, f, U, gt); break;
        case 3: run_fop<3, T, NT>(t, NL, f, U, gt); break;
        default:
          if constexpr (MAXM >= 4) run_fop<4, T, NT>(t, NL, f, U, gt);
          break;
      }
      group_sync<NT>(group);
    }
    // write-back: coalesced 16-byte stores, consecutive threads along a run
    for (uint32_t j = gt; j < n_runs; j += NT) run_off[j] = run_start(p, tile, j);
    group_sync<NT>(group);
    const uint32_t low_mask = run_amps - 1;
    if constexpr (PERM) {
#pragma unroll 4
      for (uint32_t li = gt; li < NL; li += NT) {
        const uint32_t src = p.perm_c ^ ftab[0][li & 63u] ^ ftab[1][li >> 6];
        s[run_off[li >> p.B] | (li & low_mask)] = t[swz<T>(src)];
      }
    } else {
#pragma unroll 4
      for (uint32_t li = gt; li < NL; li += NT) s[run_off[li >> p.B] | (li & low_mask)] = t[swz<T>(li)];
    }
    group_sync<NT>(group);  // buffer free for the stage's next TMA load
  }
}

// dst[e] = src for e < m (one read of the source, m writes): entries of a
// batch joining the shared prefix of a circuit family.
template <typename A>
__global__ void k_broadcast(const A* __restrict__ src, A* __restrict__ dst, uint32_t m, uint64_t dim) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < dim; i += (uint64_t)gridDim.x * blockDim.x) {
    const A v = src[i];
    for (uint32_t e = 0; e < m; ++e) dst[e * dim + i] = v;
  }
}

struct Pass {
  std::vector<uint32_t> hbits;  // ascending global bits
  std::vector<int> gates;
};

// Local bit budget: 64 KB of shared memory per tile (kStages tiles resident).
void tile_shape(uint32_t n, int32_t dtype, uint32_t& B, uint32_t& kmax) {
  // 32 KB tiles (two groups x kStages per CTA) in runs of 512 B (one TMA box
  // of 4 rows x 128 B): B = 5 (fp64) / 6 (fp32), leaving 6 gathered high bits
  const uint32_t LB = dtype == VQF_F64 ? VQF_TILE_LB : VQF_TILE_LB + 1;
  B = std::min<uint32_t>(n, LB - kMaxHigh);
  kmax = std::min<uint32_t>(LB - B, n - B);
}

std::vector<Pass> schedule(uint32_t n, uint32_t B, uint32_t kmax, const std::vector<TGate>& gates) {
  const size_t G = gates.size();
  std::vector<std::vector<int>> preds(G);
  std::vector<int> last(64, -1);
  for (size_t i = 0; i < G; ++i) {
    for (uint32_t w = 0; w < gates[i].n_wires; ++w) {
      const int l = last[gates[i].wires[w]];
      if (l >= 0 && std::find(preds[i].begin(), preds[i].end(), l) == preds[i].end()) preds[i].push_back(l);
      last[gates[i].wires[w]] = static_cast<int>(i);
    }
  }
  const auto high_bits = [&](const TGate& g) {
    std::vector<uint32_t> hb;
    for (uint32_t w = 0; w < g.n_wires; ++w) {
      const uint32_t b = n - 1 - g.wires[w];
      if (b >= B) hb.push_back(b);
    }
    return hb;
  };
  std::vector<char> done(G, 0);
  size_t remaining = G;
  std::vector<Pass> passes;
  while (remaining) {
    Pass pass;
    bool added = true;
    // greedy: among ready gates that fit, take the one adding the fewest new
    // high bits, then sharing the most bits with the pass, then the earliest
    // (keeps a CNOT chain advancing instead of letting independent RYs claim
    // the bit budget)
    while (added && pass.gates.size() < static_cast<size_t>(kMaxOps)) {
      added = false;
      int best = -1, best_new = 1 << 20, best_share = -1;
      for (size_t i = 0; i < G; ++i) {
        if (done[i]) continue;
        bool ready = true;
        for (int pr : preds[i]) ready = ready && done[pr];
        if (!ready) continue;
        int fresh = 0, share = 0;
        for (uint32_t b : high_bits(gates[i])) {
          if (std::find(pass.hbits.begin(), pass.hbits.end(), b) == pass.hbits.end()) ++fresh;
          else ++share;
        }
        if (pass.hbits.size() + fresh > kmax) continue;
        if (fresh < best_new || (fresh == best_new && share > best_share)) {
          best = static_cast<int>(i);
          best_new = fresh;
          best_share = share;
        }
      }
      if (best >= 0) {
        for (uint32_t b : high_bits(gates[best]))
          if (std::find(pass.hbits.begin(), pass.hbits.end(), b) == pass.hbits.end()) pass.hbits.push_back(b);
        pass.gates.push_back(best);
        done[best] = 1;
        --remaining;
        added = true;
      }
    }
    if (pass.gates.empty()) {
      // a gate with more high wires than the tile has room for: the driver
      // runs it with the single-gate kernel (empty hbits marks that)
      for (size_t i = 0; i < G; ++i) {
        if (done[i]) continue;
        bool ready = true;
        for (int pr : preds[i]) ready = ready && done[pr];
        if (!ready) continue;
        pass.gates.push_back(static_cast<int>(i));
        pass.hbits = {0xffffffffu};
        done[i] = 1;
        --remaining;
        break;
      }
    }
    // a pass that needed fewer high bits still moves full tiles: pad with
    // spectator bits (lowest free ones, so neighbouring runs are adjacent in
    // HBM) -- a 2^8-amplitude tile spends its time in barriers and TMA
    // issue, not on its bytes
    if (pass.hbits.empty() || pass.hbits[0] != 0xffffffffu)
      for (uint32_t b = B; b < n && pass.hbits.size() < kmax; ++b)
        if (std::find(pass.hbits.begin(), pass.hbits.end(), b) == pass.hbits.end()) pass.hbits.push_back(b);
    std::sort(pass.hbits.begin(), pass.hbits.end());
    passes.push_back(std::move(pass));
  }
  return passes;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (fn == nullptr) throw Error(VQF_CUDA_ERROR, "CUDA: cuTensorMapEncodeTiled unavailable");
  return fn;
}

// The state as a 3-d tensor {128 B row, rows, batch entry}; box = one run of
// 2^B amplitudes (<= 32 rows), 128 B swizzle.
CUtensorMap state_map(const vqf_statevector* sv, uint32_t run_bytes) {
  const bool f64 = sv->dtype == VQF_F64;
  const uint64_t amp = f64 ? 16 : 8;
  const cuuint64_t dims[3] = {f64 ? 16u : 32u, (sv->dim() * amp) / 128, sv->batch};
  const cuuint64_t strides[2] = {128, sv->dim() * amp};
  const cuuint32_t box[3] = {f64 ? 16u : 32u, run_bytes / 128, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap m;
  const CUresult r = encode_fn()(&m, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                 sv->amps, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(VQF_CUDA_ERROR, "CUDA: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

// Gate -> (local bits, code over those bits) for the fused-op merge.
struct LocalGate {
  uint32_t bits;  // local bit mask
  uint32_t rot, ma, mb;  // pair patterns as local bit masks
  int32_t param;
  double c, s;
};

uint32_t compress(uint32_t mask, const uint32_t* pos, uint32_t m) {
  uint32_t out = 0;
  for (uint32_t j = 0; j < m; ++j)
    if ((mask >> pos[j]) & 1u) out |= 1u << j;
  return out;
}

// Kernel parameters of one pass: the gates mapped to local bits and merged
// into fused ops.
// Gates [first, *next) of the pass go into this launch: the composed
// matrices must fit kMatElems, otherwise the pass is split into several
// launches over the same tiles.
TileParams build_params(uint32_t n, uint32_t batch, uint32_t B, const std::vector<TGate>& gates, const Pass& pass,
                        const double* cs_dev, uint32_t fuse_bits, size_t first, size_t* next) {
  TileParams p{};
  p.n = n;
  p.B = B;
  p.k = static_cast<uint32_t>(pass.hbits.size());
  p.batch = batch;
  p.cs = cs_dev;
  for (uint32_t j = 0; j < p.k; ++j) p.hb[j] = pass.hbits[j];
  const auto local = [&](uint32_t wire) -> uint32_t {
    const uint32_t b = n - 1 - wire;
    if (b < B) return b;
    for (uint32_t j = 0; j < p.k; ++j)
      if (p.hb[j] == b) return B + j;
    throw Error(VQF_LOGIC_ERROR, "tile scheduler: wire outside the pass");
  };
  std::vector<LocalGate> lg;
  for (int gi : pass.gates) {
    const TGate& g = gates[gi];
    LocalGate o{};
    o.param = g.param;
    o.c = g.c;
    o.s = g.s;
    uint32_t lb[4];
    for (uint32_t w = 0; w < g.n_wires; ++w) {
      lb[w] = local(g.wires[w]);
      o.bits |= 1u << lb[w];
    }
    switch (g.kind) {
      case VQF_GATE_PAULI_X:
      case VQF_GATE_RY:
        o.rot = g.kind == VQF_GATE_RY;
        o.ma = 0;
        o.mb = 1u << lb[0];
        break;
      case VQF_GATE_CNOT:
        o.rot = 0;
        o.ma = 1u << lb[0];
        o.mb = (1u << lb[0]) | (1u << lb[1]);
        break;
      case VQF_GATE_DOUBLE_EXCITATION:
        o.rot = 1;
        o.ma = (1u << lb[0]) | (1u << lb[1]);  // |1100>
        o.mb = (1u << lb[2]) | (1u << lb[3]);  // |0011>
        break;
      case VQF_GATE_SINGLE_EXCITATION:
        o.rot = 1;
        o.ma = 1u << lb[0];  // |10>
        o.mb = 1u << lb[1];  // |01>
        break;
      default:
        throw Error(VQF_LOGIC_ERROR, "unknown gate kind");
    }
    lg.push_back(o);
  }
  // a pass of X / CNOT gates only is an affine index map F on the local
  // bits: out[L] = in[F(L)] with F = f_1 o ... o f_m (gate 1 first in the
  // circuit, so f_m acts on L first); applied in the write-back
  bool perm = first == 0;
  for (const LocalGate& o : lg) perm = perm && !o.rot;
  if (perm) {
    const auto F = [&](uint32_t x) {
      for (size_t q = lg.size(); q-- > 0;) {
        const LocalGate& o = lg[q];
        if (o.ma == 0) x ^= o.mb;                                            // X: mb = target bit
        else if (x & o.ma) x ^= o.mb ^ o.ma;                                 // CNOT: ma = control, mb = control | target
      }
      return x;
    };
    const uint32_t LB = B + p.k;
    p.perm_only = 1;
    p.perm_c = F(0);
    for (uint32_t b = 0; b < 16; ++b) p.perm_col[b] = b < LB ? (F(1u << b) ^ p.perm_c) : 0u;
    *next = lg.size();
    return p;
  }
  // merge consecutive gates (the pass order respects the circuit's DAG)
  // while their local bits fit one fused op
  size_t i = first;
  uint32_t uoff = 0;
  while (i < lg.size()) {
    uint32_t u = lg[i].bits;
    bool wide = fuse_bits == kMaxFuse || __builtin_popcount(u) == 4;
    size_t j = i + 1;
    while (j < lg.size()) {
      const bool w2 = wide || __builtin_popcount(lg[j].bits) == 4;
      if (__builtin_popcount(u | lg[j].bits) > (w2 ? kMaxFuse : fuse_bits)) break;
      wide = w2;
      u |= lg[j++].bits;
    }
    TileFop f{};
    uint32_t pos[kMaxFuse], m = 0;
    for (uint32_t b = 0; b < 32; ++b)
      if ((u >> b) & 1u) pos[m++] = b;
    f.m = m;
    if (uoff + (1u << (2 * m)) > kMatElems) break;  // matrix area full: the rest goes to the next launch
    f.uoff = uoff;
    uoff += 1u << (2 * m);
    for (uint32_t q = 0; q < m; ++q) f.pos |= pos[q] << (8 * q);
    f.sub0 = p.n_fops == 0 ? 0 : p.fops[p.n_fops - 1].sub0 + p.fops[p.n_fops - 1].n_sub;
    for (size_t q = i; q < j; ++q) {
      TileSub& t = p.subs[f.sub0 + f.n_sub++];
      t.code = (lg[q].rot << 8) | (compress(lg[q].ma, pos, m) << 4) | compress(lg[q].mb, pos, m);
      t.param = lg[q].param;
      t.c = lg[q].c;
      t.s = lg[q].s;
    }
    p.fops[p.n_fops++] = f;
    i = j;
  }
  *next = i;
  return p;
}

// Item bits of a tensor-core op: the two free local bits c1 < c2 whose
// shared-memory bank pattern for the MMA fragments (B loads of both
// k-chunks: 4 slots x 4 items x re/im per warp access; D stores: 8 slots x 4
// items) has the fewest lanes per bank, under the 128 B swizzle.
uint32_t choose_item_bits(const TileFop& f, uint32_t LB) {
  uint32_t pos[3], used = 0;
  for (uint32_t j = 0; j < 3; ++j) {
    pos[j] = (f.pos >> (8 * j)) & 0xffu;
    used |= 1u << pos[j];
  }
  const auto swz8 = [](uint32_t L) { return (L ^ (L >> 3)) & 7u; };
  const auto dep = [&](uint32_t k) {
    uint32_t d = 0;
    for (uint32_t j = 0; j < 3; ++j)
      if ((k >> j) & 1u) d |= 1u << pos[j];
    return d;
  };
  uint32_t best = 0, best_score = ~0u;
  for (uint32_t c1 = 0; c1 < LB; ++c1) {
    if ((used >> c1) & 1u) continue;
    for (uint32_t c2 = c1 + 1; c2 < LB; ++c2) {
      if ((used >> c2) & 1u) continue;
      const auto dep2 = [&](uint32_t i) { return ((i & 1u) << c1) | (((i >> 1) & 1u) << c2); };
      // 8-byte B loads are served per half-warp (16 lanes, bank pair = (amp
      // mod 8, re/im)), 16-byte D stores per quarter-warp (8 lanes, amp mod
      // 8): the score adds the worst lane count per bank in each phase
      uint32_t score = 0;
      for (uint32_t chunk = 0; chunk < 2; ++chunk)
        for (uint32_t half = 0; half < 2; ++half) {
          uint32_t cnt[16] = {};
          for (uint32_t lane = 16 * half; lane < 16 * half + 16; ++lane) {
            const uint32_t g = lane >> 2, tq = lane & 3u;
            cnt[swz8(dep2(g >> 1) | dep(4 * chunk + tq)) * 2 + (g & 1u)]++;
          }
          score += *std::max_element(cnt, cnt + 16);
        }
      for (uint32_t quarter = 0; quarter < 4; ++quarter) {
        uint32_t cnt[8] = {};
        for (uint32_t lane = 8 * quarter; lane < 8 * quarter + 8; ++lane) cnt[swz8(dep2(lane & 3u) | dep(lane >> 2))]++;
        score += *std::max_element(cnt, cnt + 8);
      }
      if (score < best_score) {
        best_score = score;
        best = c1 | (c2 << 5);
      }
    }
  }
  // ops whose slot bits all lie above the swizzle's reach (index bits >= 6)
  // put several MMA lanes on one bank whatever the item bits; they take the
  // FMA path, which spreads lanes over items instead
  return best_score <= 12 ? best : kNoMma;
}

template <typename T>
void launch_pass(vqf_statevector* sv, const std::vector<TGate>& gates, const Pass& pass, uint32_t B,
                 const double* cs_dev, uint32_t active = 0) {
  // active: batch entries [0, active) take the pass (0 = all)
  if (active == 0) active = sv->batch;
  const uint32_t n = sv->n_qubits;
  for (size_t first = 0, next = 0; first < pass.gates.size(); first = next) {
  TileParams p = build_params(n, sv->batch, B, gates, pass, cs_dev, sizeof(T) == 8 ? 3 : 4, first, &next);
  bool wide = false;
  for (uint32_t o = 0; o < p.n_fops; ++o) wide = wide || p.fops[o].m == 4;
  const uint32_t LB = B + p.k;
  if (sizeof(T) == 8)
    for (uint32_t o = 0; o < p.n_fops; ++o)
      if (p.fops[o].m == 3) p.fops[o].ipos = choose_item_bits(p.fops[o], LB);
  const uint64_t n_tiles = uint64_t{1} << (n - LB);
  // persistent over one entry's tiles; a batched state launches a CTA set
  // per entry, so give each group >= 16 tiles there to amortise the CTA
  // prologue (matrix composition, ring fill) over enough traffic
  uint64_t gx = std::min<uint64_t>(n_tiles, kTileBlocks);
  if (active > 1) gx = std::max<uint64_t>(1, std::min<uint64_t>(gx, n_tiles / (kGroups * 16)));
  const unsigned grid = static_cast<unsigned>(gx);
  const uint32_t run_bytes = static_cast<uint32_t>(sizeof(typename V2<T>::type) << B);
  // the encoded map is cached per (state allocation, run size)
  static thread_local std::vector<std::pair<std::pair<const void*, uint64_t>, CUtensorMap>> maps;
  const auto key = std::make_pair(static_cast<const void*>(sv->amps),
                                  (uint64_t)run_bytes | ((uint64_t)n << 32) | ((uint64_t)sv->batch << 40) |
                                      ((uint64_t)sv->dtype << 62));
  const CUtensorMap* map = nullptr;
  for (auto& e : maps)
    if (e.first == key) map = &e.second;
  if (map == nullptr) {
    if (maps.size() > 16) maps.erase(maps.begin());
    maps.emplace_back(key, state_map(sv, run_bytes));
    map = &maps.back().second;
  }
  const size_t smem = kGroups * kStages * (sizeof(typename V2<T>::type) << LB) + 256 + kMatElems * sizeof(T) + 1024;  // rings + mbarriers + matrices + align
  auto* amps = static_cast<typename V2<T>::type*>(sv->amps);
  if (p.perm_only)
    k_tile<T, kNT, 1, true><<<dim3(grid, active), kGroups * kNT, smem, sv->stream>>>(amps, *map, p);
  else if (sizeof(T) == 4 || !wide)
    k_tile<T, kNT, sizeof(T) == 4 ? 4 : 3, false><<<dim3(grid, active), kGroups * kNT, smem, sv->stream>>>(amps, *map, p);
  else
    k_tile<T, kNT / 2, 4, false><<<dim3(grid, active), kGroups * kNT / 2, smem, sv->stream>>>(amps, *map, p);
  VQF_LAUNCHED();
  }
}

}  // namespace

std::vector<int> plan_tile_passes(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates) {
  uint32_t B, kmax;
  tile_shape(n_qubits, dtype, B, kmax);
  std::vector<int> out;
  for (const Pass& p : schedule(n_qubits, B, kmax, gates)) out.push_back(static_cast<int>(p.gates.size()));
  return out;
}

void plan_tile_counts(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates, uint32_t* passes,
                      uint32_t* fused_ops) {
  uint32_t B, kmax;
  tile_shape(n_qubits, dtype, B, kmax);
  const std::vector<Pass> ps = schedule(n_qubits, B, kmax, gates);
  uint32_t fops = 0, launches = 0;
  for (const Pass& p : ps) {
    if (!p.hbits.empty() && p.hbits[0] == 0xffffffffu) {
      ++launches;
      continue;
    }
    for (size_t first = 0, next = 0; first < p.gates.size(); first = next, ++launches) {
      const TileParams tp = build_params(n_qubits, 1, B, gates, p, nullptr, dtype == VQF_F64 ? 3 : 4, first, &next);
      fops += tp.n_fops;
      if (std::getenv("VQF_TILE_DEBUG")) {
        std::fprintf(stderr, "launch %u: k=%u hb=", launches, tp.k);
        for (uint32_t j = 0; j < tp.k; ++j) std::fprintf(stderr, "%u,", tp.hb[j]);
        std::fprintf(stderr, " perm=%u fops=%u:", tp.perm_only, tp.n_fops);
        for (uint32_t o = 0; o < tp.n_fops; ++o) {
          const uint32_t ip = tp.fops[o].m == 3 && dtype == VQF_F64 ? choose_item_bits(tp.fops[o], B + tp.k) : 0;
          std::fprintf(stderr, " m%u/%u[%x]%s", tp.fops[o].m, tp.fops[o].n_sub, tp.fops[o].pos,
                       ip == kNoMma ? "F" : "");
        }
        std::fprintf(stderr, "\n");
      }
    }
  }
  *passes = launches;
  *fused_ops = fops;
}

namespace {
void ensure_tile_attrs(const vqf_statevector* sv) {
  static thread_local int opted = -1;
  if (opted != sv->device) {
    const int bytes = kGroups * kStages * (16 << VQF_TILE_LB) + 256 + kMatElems * 8 + 1024;
    VQF_CUDA(cudaFuncSetAttribute(k_tile<double, kNT, 3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    VQF_CUDA(cudaFuncSetAttribute(k_tile<double, kNT / 2, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    VQF_CUDA(cudaFuncSetAttribute(k_tile<float, kNT, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    VQF_CUDA(cudaFuncSetAttribute(k_tile<double, kNT, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    VQF_CUDA(cudaFuncSetAttribute(k_tile<float, kNT, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    opted = sv->device;
  }
}
}  // namespace

int run_circuit_tiled(vqf_statevector* sv, const std::vector<TGate>& gates, const double* cs_dev) {
  if (gates.empty()) return 0;
  const uint32_t n = sv->n_qubits;
  uint32_t B, kmax;
  tile_shape(n, sv->dtype, B, kmax);
  ensure_tile_attrs(sv);
  const std::vector<Pass> passes = schedule(n, B, kmax, gates);
  const bool tiny = (sv->amp_bytes() << B) < 128;  // 2-3 qubits: a run is below one 128 B row
  for (const Pass& pass : passes) {
    if (tiny) {
      for (int gi : pass.gates) {
        const TGate& g = gates[gi];
        GateArgs ga{g.kind, g.n_wires, {g.wires[0], g.wires[1], g.wires[2], g.wires[3]}, g.c, g.s,
                    g.param >= 0 ? cs_dev + 2 * (size_t)g.param * sv->batch : nullptr};
        sv_apply(sv, ga);
      }
      continue;
    }
    if (!pass.hbits.empty() && pass.hbits[0] == 0xffffffffu) {
      const TGate& g = gates[pass.gates[0]];
      GateArgs ga{g.kind, g.n_wires, {g.wires[0], g.wires[1], g.wires[2], g.wires[3]}, g.c, g.s,
                  g.param >= 0 ? cs_dev + 2 * (size_t)g.param * sv->batch : nullptr};
      sv_apply(sv, ga);
      continue;
    }
    if (sv->dtype == VQF_F64)
      launch_pass<double>(sv, gates, pass, B, cs_dev);
    else
      launch_pass<float>(sv, gates, pass, B, cs_dev);
  }
  VQF_CUDA(cudaGetLastError());
  return static_cast<int>(passes.size());
}

std::vector<int> tile_param_first_pass(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates,
                                       uint32_t n_params) {
  uint32_t B, kmax;
  tile_shape(n_qubits, dtype, B, kmax);
  const uint32_t amp = dtype == VQF_F64 ? 16 : 8;
  if ((amp << B) < 128 || gates.empty()) return {};  // tiny registers: per-gate path
  const std::vector<Pass> passes = schedule(n_qubits, B, kmax, gates);
  std::vector<int> first(n_params, -1);
  for (size_t p = 0; p < passes.size(); ++p) {
    if (!passes[p].hbits.empty() && passes[p].hbits[0] == 0xffffffffu) return {};  // single-gate fallback pass
    for (int gi : passes[p].gates) {
      const int32_t j = gates[gi].param;
      if (j >= 0 && (uint32_t)j < n_params && first[j] < 0) first[j] = static_cast<int>(p);
    }
  }
  return first;
}

int run_circuit_tiled_shared(vqf_statevector* sv, const std::vector<TGate>& gates, const double* cs_dev,
                             const std::vector<uint32_t>& join) {
  const uint32_t n = sv->n_qubits;
  uint32_t B, kmax;
  tile_shape(n, sv->dtype, B, kmax);
  if (join.size() != sv->batch) throw Error(VQF_LOGIC_ERROR, "shared-prefix circuit: one join pass per entry");
  for (size_t e = 1; e < join.size(); ++e)
    if (join[e] < join[e - 1]) throw Error(VQF_LOGIC_ERROR, "shared-prefix circuit: join passes must not decrease");
  ensure_tile_attrs(sv);
  const std::vector<Pass> passes = schedule(n, B, kmax, gates);
  const uint64_t dim = sv->dim();
  uint32_t active = 0;
  while (active < sv->batch && join[active] == 0) ++active;
  // entries [active, upto) take entry 0's state after the passes so far
  const auto join_up_to = [&](uint64_t upto) {
    if (upto <= active) return;
    const uint32_t m = static_cast<uint32_t>(upto - active);
    if (sv->dtype == VQF_F64) {
      auto* a = static_cast<double2*>(sv->amps);
      k_broadcast<double2><<<kTileBlocks * 8, 256, 0, sv->stream>>>(a, a + active * dim, m, dim);
    } else {
      auto* a = static_cast<float2*>(sv->amps);
      k_broadcast<float2><<<kTileBlocks * 8, 256, 0, sv->stream>>>(a, a + active * dim, m, dim);
    }
    VQF_LAUNCHED();
    active = static_cast<uint32_t>(upto);
  };
  for (size_t p = 0; p < passes.size(); ++p) {
    uint32_t next = active;
    while (next < sv->batch && join[next] <= p) ++next;
    join_up_to(next);
    if (sv->dtype == VQF_F64)
      launch_pass<double>(sv, gates, passes[p], B, cs_dev, active);
    else
      launch_pass<float>(sv, gates, passes[p], B, cs_dev, active);
  }
  join_up_to(sv->batch);  // entries differing in no gate: entry 0's final state
  VQF_CUDA(cudaGetLastError());
  return static_cast<int>(passes.size());
}

}  // namespace vqf
