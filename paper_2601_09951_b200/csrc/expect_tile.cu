// Multi-group expectation passes over gathered TMA tiles.
//
// expectation (statevector.hpp:217-249) = sum over flip groups of
//   sum_t cb_t sum_i (-1)^popc(i & yz_t) conj(psi_i) psi_{i ^ flip}.
// A flip group whose flip is ONE index bit q (TFIM's X_q, and any X_q / Y_q
// string dressed with Z's) pairs amplitudes that differ in bit q only.  A
// tile pass reads the state once as gathered tiles -- 2^B contiguous
// amplitudes (one 128-byte row) times the 2^k values of a window of
// contiguous bits [h, h + k), ONE 4-d TMA box per tile (tma::window_map) --
// and
// evaluates every group whose bit is local to the tile: up to kExpPhases
// register phases, each holding 2^4 amplitudes per thread whose local index
// differs in 4 register bits, one flip group per register bit.  TFIM at
// n = 30 needs 4 such passes (plus the diagonal pass) instead of one pass per
// group.
//
// Per pair (i with bit q clear, j = i ^ 2^q) and term t, v = conj(psi_i)
// psi_j; both directions together give cb_t s_t(i) (v + sigma_t conj(v)) with
// sigma_t = (-1)^[q in yz_t]: 2 Re(v) or 2i Im(v) (the same split as
// k_expect_flip in sv.cu).  s_t(i) factorises into the parity of the thread's
// base index (register bits zero; tile and thread bits) and a 16-bit sign
// mask over the register slots, precomputed on the host.  Each thread keeps
// one fp64 accumulator per (phase, slot, term) across all its tiles; at the
// end the CTA reduces them in a fixed order and writes one complex partial
// per group -- deterministic, no floating-point atomics.
//
// Algorithmic bytes: S per pass (read only).
#include <algorithm>

#include "expect_tile.cuh"
#include "tma.cuh"

namespace vqf {

namespace {

using namespace tma;

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

// consumer groups per CTA (fp64 3 x 128 threads, fp32 2 x 256 threads) and
// tile buffers per group (fp64 1, fp32 2: 227 KB with the accumulators;
// fp64 2 x 2 measured 7 % slower than 3 x 1)
#ifndef VQF_EXP_GROUPS64
#define VQF_EXP_GROUPS64 3
#endif
#ifndef VQF_EXP_BUFS64
#define VQF_EXP_BUFS64 1
#endif
#ifndef VQF_EXP_GROUPS32
#define VQF_EXP_GROUPS32 2
#endif
#ifndef VQF_EXP_BUFS32
#define VQF_EXP_BUFS32 2
#endif
template <typename T>
constexpr int kEGroupsOf = sizeof(T) == 8 ? VQF_EXP_GROUPS64 : VQF_EXP_GROUPS32;
template <typename T>
constexpr int kEBufsOf = sizeof(T) == 8 ? VQF_EXP_BUFS64 : VQF_EXP_BUFS32;
constexpr int kAcc = kExpPhases * kExpSlots * kExpTerms;
constexpr int kEBlocks = 148;
template <typename T>
constexpr int kELB = sizeof(T) == 8 ? 11 : 12;  // 32 KB tiles
template <typename T>
constexpr int kEB = sizeof(T) == 8 ? 3 : 4;  // runs of 128 B
constexpr int kER = kExpSlots;               // register bits per phase


template <typename T, int LB, bool DIAG>
__global__ void __launch_bounds__(kEGroupsOf<T> << (LB - kER), 1)
    k_expect_tile(const __grid_constant__ CUtensorMap map, const __grid_constant__ ExpTileParams p,
                  double* __restrict__ partials) {
  using A = typename V2<T>::type;
  constexpr int kEGroups = kEGroupsOf<T>, kBufs = kEBufsOf<T>;
  constexpr uint32_t NT = 1u << (LB - kER), NL = 1u << LB, NR = 1u << kER;
  constexpr uint32_t tile_bytes = NL * sizeof(A);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const uint32_t group = threadIdx.x / NT, gt = threadIdx.x % NT;
  // the group's ring of kBufs tile buffers and their mbarriers (1 KB gap)
  A* const ring = reinterpret_cast<A*>(smem + (size_t)group * kBufs * tile_bytes);
  uint64_t* const bars = reinterpret_cast<uint64_t*>(smem + kEGroups * kBufs * (size_t)tile_bytes) + group * kBufs;
  const uint64_t n_tiles = uint64_t{1} << (p.n - p.B - p.k);
  const uint32_t mid_bits = p.h - p.B;
  const uint64_t top_per_entry = uint64_t{1} << (p.n - p.h - p.k);
  if (gt == 0) {
    if (group == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
    for (int b = 0; b < kBufs; ++b) mbar_init(&bars[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // tile T of the entry: mid = low (h - B) bits of T, top = the rest
  const uint64_t step = kEGroups * (uint64_t)gridDim.x;
  // the group's i-th tile goes to buffer i % kBufs
  const auto issue_load = [&](uint64_t tile, int b) {
    if (gt == 0) {
      mbar_expect_tx(&bars[b], tile_bytes);
      tma_load_window(ring + (size_t)b * NL, &map, static_cast<int32_t>(tile & ((uint64_t{1} << mid_bits) - 1)),
                      static_cast<int32_t>((tile >> mid_bits) + blockIdx.y * top_per_entry), &bars[b]);
    }
  };
  const uint64_t first = blockIdx.x + (uint64_t)group * gridDim.x;
  for (int b = 0; b < kBufs; ++b)
    if (first + b * step < n_tiles) issue_load(first + b * step, b);
  // one fp64 accumulator per (phase, slot, term) and thread, slot-major in
  // shared memory behind the tiles (consecutive threads, consecutive words)
  const uint32_t nthr = blockDim.x;
  double* acc = reinterpret_cast<double*>(smem + kEGroups * kBufs * (size_t)tile_bytes + 1024);
  for (uint32_t q = 0; q < (uint32_t)kAcc; ++q) acc[q * nthr + threadIdx.x] = 0.0;
  // folded diagonal group: sign of Z string t on the thread's amplitude r is
  // parity(tile base) ^ parity(thread part) ^ parity(r & v_t); the thread
  // parts are fixed (phase 0's layout), the tile parts come from one ballot
  uint32_t thr_sig = 0;
  double acc_diag = 0.0;
  uint64_t my_dmask = 0;  // lane q < n_diag: string q's Z mask (tile parities by ballot)
  if constexpr (DIAG) {
    if ((threadIdx.x & 31u) < p.n_diag) my_dmask = p.dmask[threadIdx.x & 31u];
    uint32_t bl = 0;
    for (int j = 0; j < LB - kER; ++j)
      if ((gt >> j) & 1u) bl ^= p.ph[0].tb_l[j];
    const uint64_t ti = ((uint64_t)(bl >> p.B) << p.h) | (bl & ((1u << p.B) - 1));
    for (uint32_t q = 0; q < p.n_diag; ++q)
      if (__popcll(ti & p.dmask[q]) & 1) thr_sig |= 1u << q;
  }
  // Slot metadata, constant over the pass, hoisted out of the tile loop: bit
  // s = ph * kExpSlots + j of live / xtype / sig0 = the slot has terms / is
  // one X-type term (smask 0) / that term's sigma.  Term signs split as
  // parity(i & yz) = parity(g0 & yz) ^ parity(thread part & yz): the thread
  // parts are fixed (thr_par, bit s * kExpTerms + k), the tile part comes
  // from one ballot per tile (lane s * kExpTerms + k holds that term's yz).
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t live = 0, xtype = 0, sig0 = 0, thr_par = 0;
  uint64_t my_yz = 0;
  // (the slot masks read kernel parameters only: CTA-uniform, so the slot
  // tests below can run on the uniform datapath)
  for (uint32_t ph = 0; ph < p.n_phases; ++ph)
    for (int j = 0; j < kExpSlots; ++j) {
      const ExpSlot& S = p.ph[ph].slot[j];
      const uint32_t sl = ph * kExpSlots + j;
      if (S.n_terms) live |= 1u << sl;
      if (S.n_terms == 1 && S.smask[0] == 0) xtype |= 1u << sl;
      if (S.sigma[0]) sig0 |= 1u << sl;
    }
  for (uint32_t ph = 0; ph < p.n_phases; ++ph) {
    uint32_t bl = 0;
    for (int j = 0; j < LB - kER; ++j)
      if ((gt >> j) & 1u) bl ^= p.ph[ph].tb_l[j];
    const uint64_t tpart = ((uint64_t)(bl >> p.B) << p.h) | (bl & ((1u << p.B) - 1));
    for (int j = 0; j < kExpSlots; ++j) {
      const ExpSlot& S = p.ph[ph].slot[j];
      const uint32_t sl = ph * kExpSlots + j;
      for (uint32_t k = 0; k < S.n_terms && k < (uint32_t)kExpTerms; ++k) {
        const uint32_t ti = sl * kExpTerms + k;
        if (__popcll(tpart & S.yz[k]) & 1) thr_par |= 1u << ti;
        if (lane == ti) my_yz = S.yz[k];
      }
    }
  }
  static_assert(kExpPhases * kExpSlots * kExpTerms <= 32, "term signs in one ballot");
  // first-term accumulators of every (phase, slot) in registers across the
  // tiles (the phase loop is unrolled), written to shared memory at the end;
  // the folded-diagonal pass (more registers live) keeps them in shared
  // memory, loaded and stored once per phase
  constexpr bool kRegAcc = !DIAG;
  double ra[kExpPhases][kExpSlots];
#pragma unroll
  for (int ph = 0; ph < kExpPhases; ++ph)
#pragma unroll
    for (int j = 0; j < kExpSlots; ++j) ra[ph][j] = 0.0;
  uint64_t tile = first;
  for (uint32_t it = 0; tile < n_tiles; tile += step, ++it) {
    const int buf = static_cast<int>(it % kBufs);
    const A* t = ring + (size_t)buf * NL;
    mbar_wait(&bars[buf], (it / kBufs) & 1u);
    // global index of the tile's local index 0: (top << (h + k)) | (mid << B)
    const uint64_t g0 = ((tile >> mid_bits) << (p.h + p.k)) | ((tile & ((uint64_t{1} << mid_bits) - 1)) << p.B);
    const uint32_t neg = __ballot_sync(0xffffffffu, __popcll(g0 & my_yz) & 1) ^ thr_par;
#pragma unroll
    for (int ph = 0; ph < kExpPhases; ++ph) {
      if (ph >= (int)p.n_phases) break;
      const ExpPhase& P = p.ph[ph];
      uint32_t base_s = 0;
#pragma unroll
      for (int j = 0; j < LB - kER; ++j)
        if ((gt >> j) & 1u) base_s ^= P.tb_s[j];
      uint32_t rv[kER];
#pragma unroll
      for (int j = 0; j < kER; ++j) rv[j] = P.rv_s[j];
      A x[NR];
#pragma unroll
      for (uint32_t r = 0; r < NR; ++r) {
        uint32_t o = base_s;
#pragma unroll
        for (int j = 0; j < kER; ++j)
          if (r & (1u << j)) o ^= rv[j];
        x[r] = t[o];
      }
      if (ph + 1 == (int)p.n_phases) {
        // every thread has read the tile: refill its buffer kBufs tiles ahead
        group_sync<NT>(group);
        if (tile + kBufs * step < n_tiles) issue_load(tile + kBufs * step, buf);
      }
      if (DIAG && ph == 0) {
        const bool tb = __popcll(g0 & my_dmask) & 1;
        const uint32_t sig = __ballot_sync(0xffffffffu, tb) ^ thr_sig;
        // w[v] = sum_r (-1)^popc(r & v) |x_r|^2 (Walsh-Hadamard over the slots)
        double w[NR];
#pragma unroll
        for (uint32_t r = 0; r < NR; ++r) {
          const double re = static_cast<double>(x[r].x), im = static_cast<double>(x[r].y);
          w[r] = fma(re, re, im * im);
        }
#pragma unroll
        for (uint32_t hh = 1; hh < NR; hh <<= 1)
#pragma unroll
          for (uint32_t u = 0; u < NR; ++u)
            if (!(u & hh)) {
              const double l = w[u], r = w[u | hh];
              w[u] = l + r;
              w[u | hh] = l - r;
            }
        double d = 0.0;
#pragma unroll
        for (uint32_t v = 0; v < NR; ++v) {
          if (!((p.v_live >> v) & 1u)) continue;  // uniform
          const uint32_t m = p.dq1[v];
          d = fma(p.dc1[v] * static_cast<double>(__popc(m) - 2 * __popc(sig & m)), w[v], d);
        }
        for (uint32_t e = 0; e < p.n_ov; ++e) {  // further classes (none for TFIM)
          const uint32_t m = p.ov_dq[e], ve = p.ov_v[e];
          double wv = w[0];
#pragma unroll
          for (uint32_t u = 1; u < NR; ++u) wv = ve == u ? w[u] : wv;
          d = fma(p.ov_dc[e] * static_cast<double>(__popc(m) - 2 * __popc(sig & m)), wv, d);
        }
        acc_diag += d;
      }
      double* const acc_ph = acc + (size_t)(ph * kExpSlots * kExpTerms) * nthr + threadIdx.x;
      double a0s[kExpSlots];
      if constexpr (!kRegAcc)
#pragma unroll
        for (int j = 0; j < kExpSlots; ++j) a0s[j] = acc_ph[(size_t)(j * kExpTerms) * nthr];
      double (&a0)[kExpSlots] = kRegAcc ? ra[ph] : a0s;
#pragma unroll
      for (int j = 0; j < kExpSlots; ++j) {
        const uint32_t sl = ph * kExpSlots + j;
        if (!((live >> sl) & 1u)) continue;
        if ((xtype >> sl) & 1u) {
          // one term without Y / Z on the register bits (TFIM's X_q): the
          // pair sum is FMA chains over Re(v) or Im(v), 2 ops per pair (fp64:
          // four independent chains for latency; fp32 measured faster with one)
          constexpr uint32_t kCh = sizeof(T) == 8 ? 4 : 1;
          T pc[4] = {T(0), T(0), T(0), T(0)};
          if ((sig0 >> sl) & 1u) {
#pragma unroll
            for (uint32_t r = 0, q = 0; r < NR; ++r) {
              if (r & (1u << j)) continue;
              const A a = x[r], b = x[r | (1u << j)];
              pc[q % kCh] = fma(a.x, b.y, pc[q % kCh]);
              pc[q % kCh] = fma(-a.y, b.x, pc[q % kCh]);
              ++q;
            }
          } else {
#pragma unroll
            for (uint32_t r = 0, q = 0; r < NR; ++r) {
              if (r & (1u << j)) continue;
              const A a = x[r], b = x[r | (1u << j)];
              pc[q % kCh] = fma(a.x, b.x, pc[q % kCh]);
              pc[q % kCh] = fma(a.y, b.y, pc[q % kCh]);
              ++q;
            }
          }
          const T part = (pc[0] + pc[1]) + (pc[2] + pc[3]);
          const double pd = static_cast<double>(part);
          a0[j] += ((neg >> (sl * kExpTerms)) & 1u) ? -pd : pd;
          continue;
        }
        const ExpSlot& S = P.slot[j];
        // pair products and the per-term sums over the thread's 8 pairs in
        // the storage precision (complex64 states: fp32, one conversion per
        // term instead of two per pair), accumulated across tiles in fp64
        T re[NR / 2], im[NR / 2];
#pragma unroll
        for (uint32_t r = 0, q = 0; r < NR; ++r) {
          if (r & (1u << j)) continue;
          const A a = x[r], b = x[r | (1u << j)];
          re[q] = fma(a.x, b.x, a.y * b.y);
          im[q] = fma(a.x, b.y, -(a.y * b.x));
          ++q;
        }
#pragma unroll
        for (int k = 0; k < kExpTerms; ++k) {
          if (k >= (int)S.n_terms) break;
          const uint32_t sm = S.smask[k];
          const bool use_im = S.sigma[k] != 0;
          T part = T(0);
#pragma unroll
          for (uint32_t r = 0, q = 0; r < NR; ++r) {
            if (r & (1u << j)) continue;
            const T v = use_im ? im[q] : re[q];
            part += ((sm >> r) & 1u) ? -v : v;
            ++q;
          }
          const double pd = static_cast<double>(part);
          const double sd = ((neg >> (sl * kExpTerms + k)) & 1u) ? -pd : pd;
          if (k == 0) a0[j] += sd;
          else acc_ph[(size_t)(j * kExpTerms + k) * nthr] += sd;
        }
      }
      if constexpr (!kRegAcc)
#pragma unroll
        for (int j = 0; j < kExpSlots; ++j) acc_ph[(size_t)(j * kExpTerms) * nthr] = a0s[j];
    }
  }
  if constexpr (kRegAcc)
#pragma unroll
  for (int ph = 0; ph < kExpPhases; ++ph)
#pragma unroll
    for (int j = 0; j < kExpSlots; ++j) acc[(size_t)((ph * kExpSlots + j) * kExpTerms) * nthr + threadIdx.x] = ra[ph][j];
  // fixed-order CTA reduction of the accumulators
  __shared__ double diag_warp[32];
  if constexpr (DIAG) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc_diag += __shfl_xor_sync(0xffffffffu, acc_diag, o);
    if ((threadIdx.x & 31u) == 0) diag_warp[threadIdx.x >> 5] = acc_diag;
  }
  __syncthreads();
  if (DIAG && threadIdx.x == 0) {
    double sd = 0.0;
    for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) sd += diag_warp[w];
    const size_t idx = ((size_t)blockIdx.y * p.G + 0) * p.nb + blockIdx.x;
    partials[2 * idx] = sd;
    partials[2 * idx + 1] = 0.0;
  }
  const double* red = acc;
  __shared__ double term_sum[kAcc];
  if (threadIdx.x < (uint32_t)kAcc) {
    double s = 0.0;
    for (uint32_t q = 0; q < nthr; ++q) s += red[threadIdx.x * nthr + q];
    term_sum[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x < (uint32_t)(kExpPhases * kExpSlots)) {
    const uint32_t ph = threadIdx.x / kExpSlots, j = threadIdx.x % kExpSlots;
    if (ph < p.n_phases) {
      const ExpSlot& S = p.ph[ph].slot[j];
      if (S.n_terms) {
        double er = 0.0, ei = 0.0;
        for (uint32_t k = 0; k < S.n_terms; ++k) {
          const double v = 2.0 * term_sum[(ph * kExpSlots + j) * kExpTerms + k];
          if (S.sigma[k]) {  // cb * (i v)
            er -= S.cb_im[k] * v;
            ei += S.cb_re[k] * v;
          } else {  // cb * v
            er += S.cb_re[k] * v;
            ei += S.cb_im[k] * v;
          }
        }
        const size_t idx = ((size_t)blockIdx.y * p.G + S.group) * p.nb + blockIdx.x;
        partials[2 * idx] = er;
        partials[2 * idx + 1] = ei;
      }
    }
  }
}

template <typename T>
size_t exp_smem_bytes() {
  constexpr int LB = kELB<T>;
  constexpr int kEGroups = kEGroupsOf<T>;
  const size_t tiles = kEGroups * kEBufsOf<T> * (sizeof(typename V2<T>::type) << LB);
  const size_t accs = sizeof(double) * kAcc * (kEGroups << (LB - kER));
  return 1024 + tiles + 1024 + accs;  // align slack, tiles, mbarriers (in the 1 KB gap), accumulators
}

uint32_t bank_of_local(bool f64, uint32_t L) {
  return f64 ? (tma::swz<double>(L) & 7u) : (tma::swz<float>(L) & 15u);
}

uint32_t rank_gf2(std::vector<uint32_t> v) {
  uint32_t rank = 0;
  for (uint32_t bit = 0; bit < 32; ++bit) {
    size_t piv = v.size();
    for (size_t i = rank; i < v.size(); ++i)
      if ((v[i] >> bit) & 1u) {
        piv = i;
        break;
      }
    if (piv == v.size()) continue;
    std::swap(v[rank], v[piv]);
    for (size_t i = 0; i < v.size(); ++i)
      if (i != rank && ((v[i] >> bit) & 1u)) v[i] ^= v[rank];
    ++rank;
  }
  return rank;
}

}  // namespace

std::vector<ExpTileParams> plan_expect_tiles(const CompiledHam& h, uint32_t n, int32_t dtype,
                                             std::vector<char>& taken) {
  const bool f64 = dtype == VQF_F64;
  const uint32_t LB = f64 ? kELB<double> : kELB<float>;
  const uint32_t B = f64 ? kEB<double> : kEB<float>;
  const uint32_t K = LB - B;
  const uint32_t G = static_cast<uint32_t>(h.group_flip.size());
  taken.assign(G, 0);
  std::vector<ExpTileParams> out;
  if (n < LB || std::getenv("VQF_NO_EXPECT_TILES")) return out;
  // candidate groups by flip bit
  std::vector<std::pair<uint32_t, uint32_t>> cand;  // (bit, group)
  for (uint32_t g = 1; g < G; ++g) {
    const uint64_t f = h.group_flip[g];
    const uint32_t cnt = h.group_offset[g + 1] - h.group_offset[g];
    if (cnt == 0 || cnt > (uint32_t)kExpTerms || __builtin_popcountll(f) != 1) continue;
    cand.emplace_back(static_cast<uint32_t>(__builtin_ctzll(f)), g);
  }
  // a pass needs at least two groups to beat the per-group kernels
  if (cand.size() < 2) return out;
  std::sort(cand.begin(), cand.end());
  const uint32_t cap = kExpPhases * kExpSlots;
  size_t next = 0;
  while (next < cand.size()) {
    // window [hw, hw + K): from the lowest uncovered group bit (>= B), kept
    // inside the register; groups below B ride along in every pass
    const uint32_t lo = std::max<uint32_t>(B, cand[next].first);
    const uint32_t hw = std::min<uint32_t>(lo, n - K);
    std::vector<std::pair<uint32_t, uint32_t>> mine;
    while (next < cand.size() && mine.size() < cap) {
      const uint32_t bit = cand[next].first;
      if (bit >= B && (bit < hw || bit >= hw + K)) break;
      mine.push_back(cand[next++]);
    }
    if (mine.size() < 2 && !out.empty()) break;  // a lone leftover: the per-group kernels
    const auto local = [&](uint32_t bit) -> uint32_t {
      if (bit < B) return bit;
      if (bit >= hw && bit < hw + K) return B + bit - hw;
      throw Error(VQF_LOGIC_ERROR, "expectation tile: bit outside the pass");
    };
    const auto global_of = [&](uint32_t lb) { return lb < B ? lb : hw + lb - B; };
    ExpTileParams p{};
    p.n = n;
    p.B = B;
    p.k = K;
    p.h = hw;
    for (size_t c0 = 0; c0 < mine.size(); c0 += kExpSlots) {
      ExpPhase& P = p.ph[p.n_phases++];
      uint32_t regs[kExpSlots], used = 0;
      size_t m = std::min<size_t>(kExpSlots, mine.size() - c0);
      for (size_t q = 0; q < m; ++q) {
        regs[q] = local(mine[c0 + q].first);
        used |= 1u << regs[q];
      }
      for (int b = static_cast<int>(LB) - 1; b >= 0 && m < (size_t)kExpSlots; --b)
        if (!((used >> b) & 1u)) {
          regs[m++] = static_cast<uint32_t>(b);
          used |= 1u << b;
        }
      // thread bits: lanes of one shared-memory wavefront on distinct banks
      std::vector<uint32_t> fr;
      for (uint32_t b = 0; b < LB; ++b)
        if (!((used >> b) & 1u)) fr.push_back(b);
      const uint32_t q = f64 ? 3 : 4;
      std::vector<uint32_t> best;
      uint32_t best_rank = 0;
      for (uint32_t mask = 0; mask < (1u << fr.size()); ++mask) {
        if (static_cast<uint32_t>(__builtin_popcount(mask)) != q) continue;
        std::vector<uint32_t> pick, vecs;
        for (size_t i = 0; i < fr.size(); ++i)
          if ((mask >> i) & 1u) {
            pick.push_back(fr[i]);
            vecs.push_back(bank_of_local(f64, 1u << fr[i]));
          }
        const uint32_t r = rank_gf2(vecs);
        if (best.empty() || r > best_rank) {
          best = pick;
          best_rank = r;
        }
      }
      std::vector<uint32_t> tb = best;
      for (uint32_t b : fr)
        if (std::find(tb.begin(), tb.end(), b) == tb.end()) tb.push_back(b);
      for (size_t j = 0; j < tb.size(); ++j) {
        P.tb_s[j] = static_cast<uint16_t>(f64 ? tma::swz<double>(1u << tb[j]) : tma::swz<float>(1u << tb[j]));
        P.tb_l[j] = static_cast<uint16_t>(1u << tb[j]);
      }
      for (uint32_t j = 0; j < (uint32_t)kExpSlots; ++j) {
        P.rv_s[j] = static_cast<uint16_t>(f64 ? tma::swz<double>(1u << regs[j]) : tma::swz<float>(1u << regs[j]));
        p.reg_gbit[p.n_phases - 1][j] = static_cast<uint8_t>(global_of(regs[j]));
      }
      for (size_t s = 0; s < std::min<size_t>(kExpSlots, mine.size() - c0); ++s) {
        const uint32_t g = mine[c0 + s].second;
        ExpSlot& S = P.slot[s];
        S.group = g;
        S.n_terms = h.group_offset[g + 1] - h.group_offset[g];
        const uint64_t f = h.group_flip[g];
        for (uint32_t k = 0; k < S.n_terms; ++k) {
          const MaskTerm& mt = h.terms[h.group_offset[g] + k];
          S.cb_re[k] = mt.cb_re;
          S.cb_im[k] = mt.cb_im;
          S.sigma[k] = __builtin_popcountll(f & mt.yz) & 1;
          // register-slot part of yz: slot j's local bit regs[j] -> global bit
          uint32_t ysl = 0;
          for (uint32_t j = 0; j < (uint32_t)kExpSlots; ++j) {
            const uint32_t gb = global_of(regs[j]);
            if ((mt.yz >> gb) & 1u) ysl |= 1u << j;
          }
          uint32_t sm = 0;
          for (uint32_t r = 0; r < 16; ++r)
            if (__builtin_popcount(r & ysl) & 1) sm |= 1u << r;
          S.smask[k] = sm;
          // the thread's base index has zeros on the register bits, so the
          // full mask gives the tile / thread parity
          S.yz[k] = mt.yz;
        }
        taken[g] = 1;
      }
    }
    out.push_back(p);
  }
  return out;
}

bool fold_diag_into_tiles(std::vector<ExpTileParams>& passes, const CompiledHam& h, int32_t dtype) {
  if ((dtype != VQF_F64 && std::getenv("VQF_NO_DIAG_FOLD32")) || passes.empty() || h.group_flip.empty() || h.group_flip[0] != 0 ||
      std::getenv("VQF_NO_DIAG_FOLD"))
    return false;
  const uint32_t t0 = h.group_offset[0], t1 = h.group_offset[1];
  if (t1 <= t0 || t1 - t0 > (uint32_t)kExpDiag) return false;
  for (uint32_t t = t0; t < t1; ++t)
    if (h.terms[t].cb_im != 0.0) return false;
  // the pass with the fewest register phases (the last one among equals)
  size_t best = 0;
  for (size_t i = 0; i < passes.size(); ++i)
    if (passes[i].n_phases <= passes[best].n_phases) best = i;
  ExpTileParams& p = passes[best];
  std::vector<std::pair<uint32_t, uint32_t>> byv;  // (register pattern, term)
  for (uint32_t t = t0; t < t1; ++t) {
    uint32_t v = 0;
    for (uint32_t j = 0; j < (uint32_t)kExpSlots; ++j)
      if ((h.terms[t].yz >> p.reg_gbit[0][j]) & 1u) v |= 1u << j;
    byv.emplace_back(v, t);
  }
  std::stable_sort(byv.begin(), byv.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  p.n_diag = t1 - t0;
  for (size_t q = 0; q < byv.size(); ++q) p.dmask[q] = h.terms[byv[q].second].yz;
  // classes of equal (v, coefficient), in order of first appearance per v:
  // the first at index v, the others in the overflow list
  p.v_live = 0;
  p.n_ov = 0;
  for (uint32_t v = 0, q = 0; v < 16; ++v) {
    p.dq1[v] = 0;
    p.dc1[v] = 0.0;
    const uint32_t ov0 = p.n_ov;
    for (; q < byv.size() && byv[q].first == v; ++q) {
      const double c = h.terms[byv[q].second].cb_re;
      if (!((p.v_live >> v) & 1u) || p.dc1[v] == c) {
        p.v_live |= 1u << v;
        p.dc1[v] = c;
        p.dq1[v] |= 1u << q;
        continue;
      }
      uint32_t e = ov0;
      while (e < p.n_ov && p.ov_dc[e] != c) ++e;
      if (e == p.n_ov) {
        p.ov_dc[e] = c;
        p.ov_v[e] = v;
        p.ov_dq[e] = 0;
        ++p.n_ov;
      }
      p.ov_dq[e] |= 1u << q;
    }
  }
  return true;
}

namespace {
template <typename T>
void launch_t(vqf_statevector* sv, std::vector<ExpTileParams>& passes, double* partials, uint32_t G, uint32_t nb) {
  constexpr int LB = kELB<T>;
  static thread_local int opted = -1;
  if (opted != sv->device) {
    VQF_CUDA(cudaFuncSetAttribute(k_expect_tile<T, LB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(exp_smem_bytes<T>())));
    VQF_CUDA(cudaFuncSetAttribute(k_expect_tile<T, LB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(exp_smem_bytes<T>())));
    opted = sv->device;
  }
  const uint64_t n_tiles = uint64_t{1} << (sv->n_qubits - LB);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>({n_tiles, (uint64_t)kEBlocks, (uint64_t)nb}));
  for (ExpTileParams& p : passes) {
    p.G = G;
    p.nb = nb;
    const CUtensorMap* map = tma::cached_window_map(sv, p.h, p.k);
    const dim3 g(grid, sv->batch);
    const unsigned threads = kEGroupsOf<T> << (LB - kER);
    if (p.n_diag) k_expect_tile<T, LB, true><<<g, threads, exp_smem_bytes<T>(), sv->stream>>>(*map, p, partials);
    else k_expect_tile<T, LB, false><<<g, threads, exp_smem_bytes<T>(), sv->stream>>>(*map, p, partials);
    VQF_LAUNCHED();
  }
}
}  // namespace

void launch_expect_tiles(vqf_statevector* sv, std::vector<ExpTileParams> passes, double* partials, uint32_t G,
                         uint32_t nb) {
  if (passes.empty()) return;
  if (sv->dtype == VQF_F64)
    launch_t<double>(sv, passes, partials, G, nb);
  else
    launch_t<float>(sv, passes, partials, G, nb);
}

}  // namespace vqf
