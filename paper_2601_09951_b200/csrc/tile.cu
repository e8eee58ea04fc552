// Gate fusion through shared-memory tiles, gates applied in registers.
//
// A pass works on "gathered tiles": 2^B contiguous low-index amplitudes
// (512 B runs) times 2^k chosen high index bits h_0..h_{k-1}, LB = B + k
// local bits (fp64: LB = 11, 32 KB; fp32: LB = 12, 32 KB).  Runs arrive by
// TMA tensor loads (128 B swizzle, completion on an mbarrier) and leave by
// TMA tensor stores (cp.async.bulk.tensor shared -> global): one HBM read and
// one write of the state per pass, whatever the number of gates in it.
//
// Inside a tile the pass's gates run as a sequence of PHASES.  In a phase
// every thread of the consumer group holds 2^R amplitudes in registers
// (R = 4 for fp64, 5 for fp32): the amplitudes whose local index differs in
// the phase's R register bits.  Rotations (RY / SingleExcitation /
// DoubleExcitation, statevector.hpp:156-200) run on those registers as a
// branch-free sequence of STEPS: a SingleExcitation on register slots (0, 1),
// a DoubleExcitation on slots 0..3, then one RY on every slot, each with its
// (cos, sin) from a per-CTA table whose entry 0 is the identity (1, 0); the
// host puts the excitations' wires on those fixed slots.  The register code
// is therefore static: no per-gate dispatch, no register shuffling.
//
// Permutation gates (X, CNOT) never move data inside a tile: they are
// affine maps over GF(2) of the local index, composed on the host into the
// FRAME F of the tile (logical amplitude L sits at shared-memory slot
// swz(F(L))).  A phase loads and stores its registers through F (in place);
// the last phase stores through the map that leaves the tile in plain order
// for the TMA store.  Between phases the tile goes through shared memory once
// (one group barrier).  The host chooses each phase's register bits (the
// rotations it can take in dependency order) and its thread bits so that the
// lanes of one shared-memory wavefront hit distinct bank groups.
//
// Passes of X / CNOT only are an affine map of the local index applied in
// the write-back (no register phases).
//
// The host scheduler walks the circuit's dependency DAG (gates sharing a wire
// keep their order; gates on disjoint wires commute) and, among ready gates
// that fit, takes the one adding the fewest new high bits (then sharing the
// most): for the hardware-efficient ansatz the CNOT chain advances five wires
// per pass.  Reordering commuting rotations changes rounding only (~1e-16;
// tests/ compare with the reference at 1e-12).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "tile.cuh"
#include "tma.cuh"

namespace vqf {

namespace tma {
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

const CUtensorMap* cached_state_map(const vqf_statevector* sv, uint32_t run_bytes) {
  static thread_local std::vector<std::pair<std::pair<const void*, uint64_t>, CUtensorMap>> maps;
  const auto key = std::make_pair(static_cast<const void*>(sv->amps),
                                  (uint64_t)run_bytes | ((uint64_t)sv->n_qubits << 32) | ((uint64_t)sv->batch << 40) |
                                      ((uint64_t)sv->dtype << 62));
  for (auto& e : maps)
    if (e.first == key) return &e.second;
  if (maps.size() > 16) maps.erase(maps.begin());
  maps.emplace_back(key, state_map(sv, run_bytes));
  return &maps.back().second;
}
// Window map: the state as {128 B row, mid, window, top x batch} for a tile
// made of the B low bits (one 128 B row) and the k contiguous bits [h, h + k):
// dims {elements per row, 2^(h - B), 2^k, 2^(n - h - k) * batch}, box
// {elements per row, 1, 2^k, 1}, so one TMA instruction moves a whole tile.
CUtensorMap window_map(const vqf_statevector* sv, uint32_t h, uint32_t k) {
  const bool f64 = sv->dtype == VQF_F64;
  const uint64_t amp = f64 ? 16 : 8, per_row = 128 / amp;
  const uint32_t B = f64 ? 3 : 4;
  const uint32_t n = sv->n_qubits;
  if (h < B || h + k > n || k > 8) throw Error(VQF_LOGIC_ERROR, "window map: bad window");
  const cuuint64_t dims[4] = {f64 ? 16u : 32u, uint64_t{1} << (h - B), uint64_t{1} << k,
                              (uint64_t{1} << (n - h - k)) * sv->batch};
  const cuuint64_t strides[3] = {128, (uint64_t{1} << h) * amp, (uint64_t{1} << (h + k)) * amp};
  const cuuint32_t box[4] = {f64 ? 16u : 32u, 1, 1u << k, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  (void)per_row;
  CUtensorMap m;
  const CUresult r = encode_fn()(&m, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                                 sv->amps, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(VQF_CUDA_ERROR, "CUDA: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

const CUtensorMap* cached_window_map(const vqf_statevector* sv, uint32_t h, uint32_t k) {
  static thread_local std::vector<std::pair<std::pair<const void*, uint64_t>, CUtensorMap>> maps;
  const auto key = std::make_pair(static_cast<const void*>(sv->amps),
                                  (uint64_t)h | ((uint64_t)k << 8) | ((uint64_t)sv->n_qubits << 16) |
                                      ((uint64_t)sv->batch << 24) | ((uint64_t)sv->dtype << 62));
  for (auto& e : maps)
    if (e.first == key) return &e.second;
  if (maps.size() > 64) maps.erase(maps.begin());
  maps.emplace_back(key, window_map(sv, h, k));
  return &maps.back().second;
}
CUtensorMap tile_map(const vqf_statevector* sv, uint32_t B, uint32_t h, uint32_t k) {
  const bool f64 = sv->dtype == VQF_F64;
  const uint64_t amp = f64 ? 16 : 8;
  const uint32_t rb = f64 ? 3 : 4;  // bits of one 128 B row
  const uint32_t n = sv->n_qubits;
  if (B < rb || h < B || h + k > n || k > 8 || (1u << (B - rb + k)) > 256)
    throw Error(VQF_LOGIC_ERROR, "tile map: bad window");
  const cuuint64_t dims[5] = {f64 ? 16u : 32u, uint64_t{1} << (B - rb), uint64_t{1} << (h - B), uint64_t{1} << k,
                              (uint64_t{1} << (n - h - k)) * sv->batch};
  const cuuint64_t strides[4] = {128, (uint64_t{1} << B) * amp, (uint64_t{1} << h) * amp,
                                 (uint64_t{1} << (h + k)) * amp};
  const cuuint32_t box[5] = {f64 ? 16u : 32u, 1u << (B - rb), 1, 1u << k, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUtensorMap m;
  const CUresult r = encode_fn()(&m, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
                                 sv->amps, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(VQF_CUDA_ERROR, "CUDA: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

const CUtensorMap* cached_tile_map(const vqf_statevector* sv, uint32_t B, uint32_t h, uint32_t k) {
  static thread_local std::vector<std::pair<std::pair<const void*, uint64_t>, CUtensorMap>> maps;
  const auto key = std::make_pair(static_cast<const void*>(sv->amps),
                                  (uint64_t)h | ((uint64_t)k << 8) | ((uint64_t)B << 12) | ((uint64_t)sv->n_qubits << 16) |
                                      ((uint64_t)sv->batch << 24) | ((uint64_t)sv->dtype << 62));
  for (auto& e : maps)
    if (e.first == key) return &e.second;
  if (maps.size() > 64) maps.erase(maps.begin());
  maps.emplace_back(key, tile_map(sv, B, h, k));
  return &maps.back().second;
}
}  // namespace tma

namespace {

using namespace tma;

constexpr int kMaxRot = 72;     // (cos, sin) entries per launch (kernel parameters stay < 4 KB)
constexpr int kMaxSteps = 56;   // register steps per launch
constexpr int kMaxPhases = 12;  // register phases per launch
constexpr size_t kPhaseRot = 20;  // rotations per phase (bounds its steps and table entries)
#ifndef VQF_TILE_MAX_HIGH
#define VQF_TILE_MAX_HIGH 7
#endif
constexpr int kMaxHigh = VQF_TILE_MAX_HIGH;
constexpr int kTileBlocks = 148;  // persistent: one CTA per SM
#ifndef VQF_TILE_GROUPS
#define VQF_TILE_GROUPS 4  // independent consumer groups per CTA (128 threads each)
#endif
#ifndef VQF_TILE_STAGES
#define VQF_TILE_STAGES 1  // tile buffers per group
#endif
#ifndef VQF_TILE_LB
#define VQF_TILE_LB 11  // fp64 tile = 2^11 amplitudes (32 KB); fp32 one bit more
#endif
#ifndef VQF_TILE_GROUPS32
#define VQF_TILE_GROUPS32 4  // fp32: 128-thread groups (32 amplitudes per thread over 2^12-amplitude tiles)
#endif
#ifndef VQF_TILE_R32
#define VQF_TILE_R32 5
#endif
constexpr int kStages = VQF_TILE_STAGES;
#ifndef VQF_TILE_LB32
#define VQF_TILE_LB32 (VQF_TILE_LB + 1)
#endif
constexpr int kLB64 = VQF_TILE_LB, kLB32 = VQF_TILE_LB32;
constexpr int kR64 = 4, kR32 = VQF_TILE_R32;  // register bits per phase (16 / 32 amplitudes per thread)
// consumer groups per CTA: 4 x 128 threads (<= 128 registers each); measured for fp32 against
// 2 x 256 threads with 16 registers of amplitudes (scripts/build_variant.sh): 24.5 vs 33.6 ms per n = 30 layer
template <typename T>
constexpr int kGroupsOf = sizeof(T) == 8 ? VQF_TILE_GROUPS : VQF_TILE_GROUPS32;
#ifndef VQF_TILE_SLOTS
#define VQF_TILE_SLOTS 4  // tile buffers per CTA, shared round-robin by the groups
#endif
// A CTA's tiles i = 0, 1, ... use slot i % kSlots; group g takes i = g mod
// G.  Whoever finishes reading tile i out of its slot loads tile i + kSlots
// into it, so kSlots - G tiles are always in flight ahead of the groups.
// measured (scripts/ring_check.sh, n = 30 HEA layer, with the issued[]
// guard below): 6 slots 32.2 ms fp64 / 23.0 ms fp32 vs 4 slots 32.6 / 22.6 ms,
// so the default keeps one slot per group
template <typename T>
constexpr int kSlotsOf = VQF_TILE_SLOTS > kGroupsOf<T> * kStages ? VQF_TILE_SLOTS : kGroupsOf<T> * kStages;
constexpr int kB = 5;              // run = 2^5 amplitudes: 512 B fp64 (one TMA box of 4 x 128 B rows)

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

// ------------------------------------------------------- register steps
// One step over the thread's 2^R register slots x[r], applied in this order:
//   SingleExcitation: pairs (r|1, r|2) for r with slot bits 0, 1 clear
//   DoubleExcitation: pairs (r|3, r|12) for r with slot bits 0..3 clear
//   RY on slot j = 0..R-1: pairs (r, r|2^j) for r with slot bit j clear
// each a Givens rotation a' = c a - s b, b' = s a + c b on the pair (a, b)
// (statevector.hpp:160-163, :195-196) with (c, s) from the CTA's table;
// index 0 = (1, 0) = identity.
struct TileStep {
  int16_t se, de;  // table indices of the excitations (0: none)
  int16_t ry[5];   // per slot (0: none)
  uint16_t flags;  // bit 0: has SingleExcitation, bit 1: has DoubleExcitation
};

template <typename P, typename T>
__device__ __forceinline__ void givens(P& a, P& b, T c, T s) {
  const P u = a, v = b;
  a.x = fma(c, u.x, -s * v.x);
  a.y = fma(c, u.y, -s * v.y);
  b.x = fma(s, u.x, c * v.x);
  b.y = fma(s, u.y, c * v.y);
}

// Factored RY steps (fp32): every Givens rotation scales both outputs by the
// same factor, so a slot's RY runs as
//   |c| >= |s|: a' = u - k v, b' = v + k u   (k = s / c, factor c)
//   else      : a' = k u - v, b' = u + k v   (k = c / s, factor s)
// -- 2 FMAs per amplitude component instead of a multiply and an FMA -- and
// the product of the factors, equal for all the thread's amplitudes, is
// applied once at the end of the phase.  rk[q] = k (in the state's
// precision), rform[q] = the branch, and the kernel prologue multiplies each
// phase's factors once per CTA (pscale); entry 0 = (k 0, factor 1): identity,
// exact.  fp64 keeps the direct form (the factored one spills there and
// measured 6 % slower).
#ifndef VQF_TILE_FACTORED32
#define VQF_TILE_FACTORED32 1
#endif
template <typename T>
constexpr bool kFactored = sizeof(T) == 4 && VQF_TILE_FACTORED32;

// VQF_TILE_SKIP_ID=1 skips slots without an RY in the step (table entry 0)
// on a uniform branch instead of rotating them by the identity (exact either
// way).  Measured (scripts/ab_tile.sh, HEA layer): fp32 n = 30 15.46 vs
// 14.86-15.03 ms, n = 28 4.08 vs 3.94-4.11 ms, fp64 equal -- the fp32 pass is
// not bound by the rotation FMAs, and the branch costs the LB = 12 instance
// registers (152 B of spills vs 68 B), so the default keeps the identities.
#ifndef VQF_TILE_SKIP_ID
#define VQF_TILE_SKIP_ID 0
#endif
constexpr bool kSkipIdentity = VQF_TILE_SKIP_ID;

template <int R, typename P, typename T>
__device__ __forceinline__ void run_step(P (&x)[1 << R], const TileStep& st, const double2* rcs, const T* sk,
                                         uint32_t fm) {
  constexpr int NR = 1 << R;
  if (st.flags & 1u) {
    const double2 v = rcs[st.se];
#pragma unroll
    for (int r = 0; r < NR; r += 4) givens(x[r | 1], x[r | 2], static_cast<T>(v.x), static_cast<T>(v.y));
  }
  if (st.flags & 2u) {
    const double2 v = rcs[st.de];
#pragma unroll
    for (int r = 0; r < NR; r += 16) givens(x[r | 3], x[r | 12], static_cast<T>(v.x), static_cast<T>(v.y));
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (kSkipIdentity && st.ry[j] == 0) continue;  // CTA-uniform: no divergence
    if constexpr (kFactored<T>) {
      const T k = sk[j];  // the step's slot-j k and form, gathered in the prologue
      if (!((fm >> j) & 1u)) {
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if (!(r & (1 << j))) {
            P& a = x[r];
            P& b = x[r | (1 << j)];
            const P u = a;
            a.x = fma(-k, b.x, u.x);
            a.y = fma(-k, b.y, u.y);
            b.x = fma(k, u.x, b.x);
            b.y = fma(k, u.y, b.y);
          }
      } else {
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if (!(r & (1 << j))) {
            P& a = x[r];
            P& b = x[r | (1 << j)];
            const P u = a;
            a.x = fma(k, u.x, -b.x);
            a.y = fma(k, u.y, -b.y);
            b.x = fma(k, b.x, u.x);
            b.y = fma(k, b.y, u.y);
          }
      }
    } else {
      const double2 v = rcs[st.ry[j]];
      const T c = static_cast<T>(v.x), sn = static_cast<T>(v.y);
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (!(r & (1 << j))) givens(x[r], x[r | (1 << j)], c, sn);
    }
  }
}

// ------------------------------------------------------------ parameters
// One register phase: steps [step0, step0 + n_steps).  Thread bit j of the
// group's thread index selects the shared-memory slot offset ld_tb[j],
// register slot bit j the offset ld_r[j], and ld_c is the constant part: the
// swizzled images of the frame's affine map are xor-linear, so an
// amplitude's slot is ld_c ^ (xor of its bits' offsets).  Stores use the st_*
// offsets (equal to the loads' except when the phase re-lays the tile out).
struct TilePhase {
  uint16_t step0, n_steps;
  uint16_t ld_c, st_c;
  uint16_t ld_tb[9], ld_r[5];
  uint16_t st_tb[9], st_r[5];
  uint16_t relayout;
  // last phase only: store straight to HBM from the registers.  st_* then
  // hold the UNswizzled store map (local index of the register in the
  // plain tile); the lanes are local bits 0..4, so a warp's store covers one
  // 512-byte run.
  uint16_t direct;
};

struct TileParams {
  uint32_t n, B, k, batch, n_phases;
  uint32_t merge;  // hb[0..merge) = B, B+1, ...: 2^merge adjacent runs move as one TMA box
  uint32_t win;    // 1: hb is one window [hb[0], hb[0] + k) and the map a tile map: one box per tile
  uint32_t hb[kMaxHigh];  // global bit of local bit B + j, ascending
  const double* cs;       // per-entry (cos, sin) table: cs[2 (param * batch + entry)]
  // Permutation-only pass (every gate X / CNOT): the tile is written back as
  // out[L] = in[F(L)] with F(L) = c ^ xor of col[b] over the set bits b of L
  // (an affine map over GF(2) on the local index).
  uint32_t perm_only, perm_c;
  uint32_t perm_col[16];
  uint32_t n_rot;              // (cos, sin) table entries; entry 0 = (1, 0)
  int32_t rot_param[kMaxRot];  // >= 0: per-entry table row; < 0: (rot_c, rot_s)
  double rot_c[kMaxRot], rot_s[kMaxRot];
  uint8_t rot_neg[kMaxRot];    // 1: negated angle (an excitation with its pair roles swapped)
  TilePhase ph[kMaxPhases];
  TileStep steps[kMaxSteps];
};
static_assert(sizeof(TileParams) <= 4096, "kernel parameter limit");

// Global start index of run j (0 <= j < 2^k) of tile `tile`.
__device__ __forceinline__ uint64_t run_start(const TileParams& p, uint64_t tile, uint32_t j) {
  if (p.win) {  // gathered bits = the window [h, h + k): closed form
    const uint32_t h = p.hb[0], mid = h - p.B;
    return ((tile >> mid) << (h + p.k)) | ((tile & ((uint64_t{1} << mid) - 1)) << p.B) | ((uint64_t)j << h);
  }
  uint64_t base = tile << p.B;
  for (uint32_t m = 0; m < p.k; ++m) base = insert_zero64(base, p.hb[m]);
  for (uint32_t m = 0; m < p.k; ++m) base |= (uint64_t)((j >> m) & 1u) << p.hb[m];
  return base;
}

// One register phase on the tile t: load the thread's 2^R amplitudes through
// the frame, run the phase's steps in registers, store them back.
// Direct last phase: after the loads (one group barrier: the buffer is then
// free) `refill` issues the group's next TMA loads into it, so the next tile
// streams in while this one computes and stores.
template <typename T, int R, int LB, int NT, typename Refill>
__device__ __forceinline__ void run_phase(typename V2<T>::type* t, const TilePhase& ph, const TileStep* steps,
                                          const double2* rcs, const T* sk, const uint32_t* sform, T pscale,
                                          uint32_t gt, uint32_t group,
                                          typename V2<T>::type* s, const uint64_t* run_off, uint32_t B,
                                          Refill&& refill) {
  using A = typename V2<T>::type;
  constexpr int NR = 1 << R;
  const auto slots = [&](const uint16_t* tb, const uint16_t* rv, uint32_t c, uint32_t (&off)[NR]) {
    uint32_t base = c;
#pragma unroll
    for (int j = 0; j < LB - R; ++j)
      if ((gt >> j) & 1u) base ^= tb[j];
    uint32_t r_off[R];
#pragma unroll
    for (int j = 0; j < R; ++j) r_off[j] = rv[j];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      uint32_t o = base;
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (r & (1 << j)) o ^= r_off[j];
      off[r] = o;
    }
  };
  uint32_t off[NR];
  slots(ph.ld_tb, ph.ld_r, ph.ld_c, off);
  A x[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) x[r] = t[off[r]];
  const bool direct = ph.direct != 0;
  if (direct || ph.relayout) {
    group_sync<NT>(group);  // every slot read before any is overwritten / refilled
    slots(ph.st_tb, ph.st_r, ph.st_c, off);
    if (direct) refill();
  }
  const uint32_t n_steps = ph.n_steps, step0 = ph.step0;
  const T scale = pscale;  // product of the phase's factors (kernel prologue)
  for (uint32_t q = step0; q < step0 + n_steps; ++q)
    run_step<R, A, T>(x, steps[q], rcs, sk + (size_t)q * R, kFactored<T> ? sform[q] : 0u);
  if constexpr (kFactored<T>) {
    if (n_steps != 0)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        x[r].x *= scale;
        x[r].y *= scale;
      }
  }
  if (direct) {
    const uint32_t low = (1u << B) - 1;
#pragma unroll
    for (int r = 0; r < NR; ++r) s[run_off[off[r] >> B] | (off[r] & low)] = x[r];
  } else {
#pragma unroll
    for (int r = 0; r < NR; ++r) t[off[r]] = x[r];
  }
}

// Persistent tile kernel: G consumer groups of NT = 2^(LB - R) threads, each
// with S tile buffers; group g takes every G-th tile of the CTA's sequence.
// Per tile: wait for its TMA loads, run the register phases (a group barrier
// after each), then the group's first warp issues the TMA stores of the
// runs, waits until they have read the buffer and refills it with the
// group's tile S steps ahead.  Permutation passes write back with 16-byte
// stores through the affine index map instead.
template <typename T, int R, int LB, bool PERM>
__global__ void __launch_bounds__(kGroupsOf<T> << (LB - R), 1)
    k_tile(typename V2<T>::type* __restrict__ a, const __grid_constant__ CUtensorMap map,
           const __grid_constant__ TileParams p) {
  using A = typename V2<T>::type;
  constexpr int kGroups = kGroupsOf<T>;
  constexpr uint32_t NT = 1u << (LB - R), NL = 1u << LB;
  constexpr uint32_t tile_bytes = NL * sizeof(A);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 128 B swizzle atoms are 1024 B: align the rings (the launch adds 1 KB
  // slack); indexing smem_raw keeps the pointer in the shared window
  unsigned char* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const uint32_t run_amps = 1u << p.B, n_runs = 1u << p.k;
  const uint32_t run_bytes = run_amps * sizeof(A);
  constexpr uint32_t amps_per_row = 128 / sizeof(A);
  const uint32_t group = threadIdx.x / NT, gt = threadIdx.x % NT;
  constexpr int kSlots = kSlotsOf<T>;
  unsigned char* ring = smem;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kSlots * (size_t)tile_bytes);
  __shared__ double2 rcs[kMaxRot];
  __shared__ T rk[kFactored<T> ? kMaxRot : 1];          // factored form: k per rotation
  __shared__ double rfac[kFactored<T> ? kMaxRot : 1];    // and its factor
  __shared__ T pscale[kFactored<T> ? kMaxPhases : 1];    // product of a phase's factors
  __shared__ T sk[kFactored<T> ? kMaxSteps * R : 1];     // k of step q, slot j at q * R + j
  __shared__ uint32_t sform[kFactored<T> ? kMaxSteps : 1];  // bit j: slot j's form
  __shared__ uint8_t rform[kFactored<T> ? kMaxRot : 1];
  __shared__ uint16_t ftab[PERM ? 2 : 1][64];
  // run starts of the group's current tile (double-buffered: a fast thread
  // fills the next tile's while slow ones still store the current one)
  __shared__ uint64_t run_off_all[kGroups][2][1 << kMaxHigh];
  const int32_t entry = static_cast<int32_t>(blockIdx.y);
  A* s = a + ((uint64_t)blockIdx.y << p.n);
  const uint64_t n_tiles = uint64_t{1} << (p.n - p.B - p.k);
  if (gt == 0) {
    if (group == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
    if (group == 0)
      for (int st = 0; st < kSlots; ++st) mbar_init(&bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (PERM) {
    for (uint32_t e = threadIdx.x; e < 128; e += blockDim.x) {
      const uint32_t half = e >> 6, j = e & 63u;
      uint32_t v = 0;
      for (uint32_t b = 0; b < 6; ++b)
        if ((j >> b) & 1u) v ^= p.perm_col[6 * half + b];
      ftab[half][j] = static_cast<uint16_t>(v);
    }
  } else {
    // the pass's rotation angles for this batch entry, one parallel round of
    // loads
    for (uint32_t q = threadIdx.x; q < p.n_rot; q += blockDim.x) {
      double2 v = make_double2(p.rot_c[q], p.rot_s[q]);
      if (p.rot_param[q] >= 0)
        v = *reinterpret_cast<const double2*>(p.cs + 2 * ((size_t)p.rot_param[q] * p.batch + blockIdx.y));
      if (p.rot_neg[q]) v.y = -v.y;
      rcs[q] = v;
      if constexpr (kFactored<T>) {
        const bool by_c = fabs(v.x) >= fabs(v.y);
        rk[q] = static_cast<T>(by_c ? v.y / v.x : v.x / v.y);
        rfac[q] = by_c ? v.x : v.y;
        rform[q] = by_c ? 0 : 1;
      }
    }
    if constexpr (kFactored<T>) {
      // each phase's factors multiplied once per CTA, in the order the steps
      // used to apply them (step by step, slot by slot)
      __syncthreads();
      for (uint32_t ph = threadIdx.x; ph < p.n_phases; ph += blockDim.x) {
        T sc = T(1);
        for (uint32_t q = p.ph[ph].step0; q < p.ph[ph].step0 + p.ph[ph].n_steps; ++q)
          for (int j = 0; j < R; ++j) sc *= static_cast<T>(rfac[p.steps[q].ry[j]]);
        pscale[ph] = sc;
      }
      for (uint32_t e = threadIdx.x; e < (uint32_t)(kMaxSteps * R); e += blockDim.x)
        sk[e] = rk[p.steps[e / R].ry[e % R]];
      for (uint32_t q = threadIdx.x; q < (uint32_t)kMaxSteps; q += blockDim.x) {
        uint32_t fm = 0;
        for (int j = 0; j < R; ++j) fm |= (uint32_t)rform[p.steps[q].ry[j]] << j;
        sform[q] = fm;
      }
    }
  }
  __syncthreads();
  // issued[s] = CTA tile index whose load the slot's pending mbarrier phase
  // belongs to: with more slots than groups a fast group could otherwise
  // reach a slot two phases ahead of a slow refiller and mistake the parity
  // of an older phase for its own (ABA)
  __shared__ volatile uint32_t issued[8];
  static_assert(kSlotsOf<T> <= 8, "tile ring: at most 8 slots");
  const auto stage_buf = [&](int st) { return reinterpret_cast<A*>(ring + (size_t)st * tile_bytes); };
  // tile map coordinates (p.win): mid = the tile's bits below the window,
  // top = the rest, batch entries stacked above
  const uint32_t mid_bits = p.win ? p.hb[0] - p.B : 0;
  const auto win_mid = [&](uint64_t tile) { return static_cast<int32_t>(tile & ((uint64_t{1} << mid_bits) - 1)); };
  const auto win_top = [&](uint64_t tile) {
    return static_cast<int32_t>((tile >> mid_bits) + ((uint64_t)entry << (p.n - p.hb[0] - p.k)));
  };
  const auto issue_load = [&](uint64_t tile, int st) {
    const uint32_t lane = gt;
    if (lane == 0) {
      mbar_expect_tx(&bar[st], tile_bytes);
      issued[st] = static_cast<uint32_t>((tile - blockIdx.x) / gridDim.x);
    }
    unsigned char* dst = reinterpret_cast<unsigned char*>(stage_buf(st));
    if (p.win) {
      if (lane == 0) tma_load_tile(dst, &map, win_mid(tile), win_top(tile), &bar[st]);
      return;
    }
    for (uint32_t j = lane; j < (n_runs >> p.merge); j += 32)
      tma_load_run(dst + ((size_t)j << p.merge) * run_bytes, &map,
                   static_cast<int32_t>(run_start(p, tile, j << p.merge) / amps_per_row), entry, &bar[st]);
  };
  // the CTA's tiles: tile(i) = blockIdx.x + i * gridDim.x; group g takes
  // i = g, g + G, ...; tile i sits in slot i % kSlots
  const uint64_t step = kGroups * (uint64_t)gridDim.x;
  const uint64_t first = blockIdx.x + (uint64_t)group * gridDim.x;
  if (group == 0 && gt < 32)
    for (int st = 0; st < kSlots; ++st) {
      const uint64_t t0 = blockIdx.x + (uint64_t)st * gridDim.x;
      if (t0 < n_tiles) issue_load(t0, st);
    }
  __syncthreads();  // the initial loads are issued before any group waits on a refill chain
  uint64_t tile = first;
  const bool direct = !PERM && p.ph[p.n_phases - 1].direct != 0;
  for (uint32_t i = group; tile < n_tiles; tile += step, i += kGroups) {
    const uint32_t it = i / kGroups;  // the group's own tile count
    const int cur = static_cast<int>(i % kSlots);
    const uint64_t ahead = tile + (uint64_t)kSlots * gridDim.x;  // tile i + kSlots, same slot
    if (kSlots > kGroups)
      while (issued[cur] != i) {
      }
    mbar_wait(&bar[cur], (i / kSlots) & 1u);
    A* t = stage_buf(cur);
    uint64_t* run_off = run_off_all[group][it & 1u];
    if (PERM || direct)
      for (uint32_t j = gt; j < n_runs; j += NT) run_off[j] = run_start(p, tile, j);
    if constexpr (PERM) {
      // read the whole tile through the index map into registers, free the
      // buffer for the next load, then 16-byte stores along the runs
      constexpr uint32_t U = NL / NT;
      A v[U];
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) {
        const uint32_t li = gt + u * NT;
        v[u] = t[swz<T>(p.perm_c ^ ftab[0][li & 63u] ^ ftab[1][li >> 6])];
      }
      group_sync<NT>(group);
      if (gt < 32 && ahead < n_tiles) issue_load(ahead, cur);
      const uint32_t low_mask = run_amps - 1;
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) {
        const uint32_t li = gt + u * NT;
        s[run_off[li >> p.B] | (li & low_mask)] = v[u];
      }
    } else {
      const auto refill = [&] {
        if (gt < 32 && ahead < n_tiles) issue_load(ahead, cur);
      };
      for (uint32_t ph = 0; ph < p.n_phases; ++ph) {
        run_phase<T, R, LB, NT>(t, p.ph[ph], p.steps, rcs, sk, sform, kFactored<T> ? pscale[ph] : T(1), gt, group, s,
                                run_off, p.B, refill);
        if (ph + 1 == p.n_phases) {
          if (direct) break;
          fence_proxy_async();  // generic-proxy stores -> TMA store reads
        }
        group_sync<NT>(group);
      }
      if (!direct && gt < 32) {
        if (p.win) {
          if (gt == 0) tma_store_tile(t, &map, win_mid(tile), win_top(tile));
        } else {
          for (uint32_t j = gt; j < (n_runs >> p.merge); j += 32)
            tma_store_run(reinterpret_cast<unsigned char*>(t) + ((size_t)j << p.merge) * run_bytes, &map,
                          static_cast<int32_t>(run_start(p, tile, j << p.merge) / amps_per_row), entry);
        }
        bulk_commit();
        bulk_wait_read();  // this lane's stores have read the buffer
        __syncwarp();
        if (ahead < n_tiles) issue_load(ahead, cur);
      }
    }
  }
  if constexpr (!PERM)
    if (gt < 32) bulk_wait_all();
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

// --------------------------------------------------------------- host side
struct Pass {
  std::vector<uint32_t> hbits;  // ascending global bits
  std::vector<int> gates;
};

int tile_lb(int32_t dtype) { return dtype == VQF_F64 ? kLB64 : kLB32; }
int tile_r(int32_t dtype) { return dtype == VQF_F64 ? kR64 : kR32; }

// Tile geometry: runs of 2^B amplitudes, up to kmax gathered high bits;
// registers narrower than the full tile use one tile of their own width
// (down to R + 5 local bits: one warp per consumer group).
void tile_shape(uint32_t n, int32_t dtype, uint32_t& B, uint32_t& kmax) {
  const uint32_t LB = std::min<uint32_t>(n, static_cast<uint32_t>(tile_lb(dtype)));
  B = std::min<uint32_t>(n, kB);
  kmax = LB - B;
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
    while (added) {
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
      // runs it with the single-gate kernel (hbits = {~0} marks that)
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

// Gate -> (local bits, pair pattern over those bits).
struct LocalGate {
  uint32_t bits;         // local bit mask
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

// The pass's gates mapped to local bits (local bit b < B: global bit b;
// local bit B + j: global bit hb[j]).
std::vector<LocalGate> local_gates(uint32_t n, uint32_t B, const std::vector<uint32_t>& hb,
                                   const std::vector<TGate>& gates, const Pass& pass) {
  const auto local = [&](uint32_t wire) -> uint32_t {
    const uint32_t b = n - 1 - wire;
    if (b < B) return b;
    for (size_t j = 0; j < hb.size(); ++j)
      if (hb[j] == b) return B + static_cast<uint32_t>(j);
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
  return lg;
}

// Affine map over GF(2) of the LB-bit local index: L -> c ^ (xor of col[b]
// over the set bits b of L).
struct Affine {
  uint32_t c = 0;
  uint32_t col[16] = {};
  static Affine identity(uint32_t LB) {
    Affine a;
    for (uint32_t b = 0; b < LB; ++b) a.col[b] = 1u << b;
    return a;
  }
  uint32_t lin(uint32_t L) const {
    uint32_t v = 0;
    for (uint32_t b = 0; b < 16; ++b)
      if ((L >> b) & 1u) v ^= col[b];
    return v;
  }
  uint32_t operator()(uint32_t L) const { return c ^ lin(L); }
};

Affine compose(const Affine& f, const Affine& g, uint32_t LB) {  // f o g
  Affine h;
  h.c = f(g.c);
  for (uint32_t b = 0; b < LB; ++b) h.col[b] = f.lin(g.col[b]);
  return h;
}

Affine inverse(const Affine& f, uint32_t LB) {
  std::vector<uint32_t> inv(size_t{1} << LB);
  for (uint32_t L = 0; L < (1u << LB); ++L) inv[f(L)] = L;
  Affine g;
  g.c = inv[0];
  for (uint32_t b = 0; b < LB; ++b) g.col[b] = inv[1u << b] ^ g.c;
  return g;
}

// X / CNOT as the index permutation they apply (self-inverse): X on bit t
// flips it; CNOT (control c, target t) flips t where c is set.
Affine perm_of(const LocalGate& g, uint32_t LB) {
  Affine a = Affine::identity(LB);
  if (g.ma == 0) a.c = g.mb;                          // X: mb = target bit
  else a.col[__builtin_ctz(g.ma)] ^= g.mb ^ g.ma;     // CNOT: ma = control, mb = control | target
  return a;
}

// A phase as planned on the host.
struct PhasePlan {
  Affine load;                 // frame at the phase start (in-place phases store through it too)
  Affine store;                // store map (differs only when the phase re-lays the tile out)
  uint32_t slot_bit[5] = {};   // local bit of register slot j
  std::vector<TileStep> steps;
  std::vector<int> step_gate_rot;  // per rotation added: local gate index (for the angle table)
};

// Slot kinds fixed by an excitation in the phase.
enum : int { kFixNone = 0, kFixSE = 1, kFixDE = 2 };

// Register phases of one launch: walk the gates in pass order; a phase
// takes every rotation whose bits fit its R register bits (excitations on
// the fixed slots) and that depends on no gate left for a later phase; a
// permutation is taken into the frame after the phase's rotations unless a
// skipped gate precedes it, and then blocks the rotations on its bits.  The
// gates done after any number of phases are therefore closed under
// predecessors.  Returns false when the launch's tables are full (the caller
// continues with the remaining gates in a new launch).
struct PassPlan {
  std::vector<PhasePlan> phases;
  std::vector<int> rot_gate;  // table entry k >= 1 -> local gate index
  Affine end_frame;
};

PassPlan plan_launch(const std::vector<LocalGate>& lg, std::vector<char>& done, uint32_t LB, uint32_t R) {
  PassPlan out;
  Affine F = Affine::identity(LB);
  size_t n_steps = 0;
  const auto remaining = [&] {
    for (char d : done)
      if (!d) return true;
    return false;
  };
  while (remaining()) {
    PhasePlan ph;
    ph.load = F;
    uint32_t regs = 0, blocked = 0, perm_bits = 0;
    int fix = kFixNone;
    uint32_t fix_a = 0, fix_b = 0;  // excitation's A / B local masks
    std::vector<int> rots;          // rotations taken, in order
    std::vector<int> perms;         // permutations taken, in order
    std::vector<int> signs;         // per rotation: +1, or -1 for an excitation with A / B swapped
    for (size_t i = 0; i < lg.size(); ++i) {
      if (done[i]) continue;
      const LocalGate& g = lg[i];
      if (g.bits & blocked) {
        blocked |= g.bits;
        continue;
      }
      if (!g.rot) {
        perms.push_back(static_cast<int>(i));
        perm_bits |= g.bits;
        done[i] = 1;
        continue;
      }
      bool ok = (g.bits & perm_bits) == 0 &&
                static_cast<uint32_t>(__builtin_popcount(regs | g.bits)) <= R;
      int sign = 1;
      const int kind = g.ma == 0 ? kFixNone : (__builtin_popcount(g.ma) == 1 ? kFixSE : kFixDE);
      if (ok && kind != kFixNone) {
        if (fix == kFixNone) {
          fix = kind;
          fix_a = g.ma;
          fix_b = g.mb;
        } else if (fix == kind && fix_a == g.ma && fix_b == g.mb) {
        } else if (fix == kind && fix_a == g.mb && fix_b == g.ma) {
          sign = -1;  // the same rotation with the pair's roles swapped: angle -> -angle
        } else {
          ok = false;
        }
      }
      if (ok && rots.size() >= kPhaseRot) ok = false;
      if (!ok) {
        blocked |= g.bits;
        continue;
      }
      regs |= g.bits;
      rots.push_back(static_cast<int>(i));
      signs.push_back(sign);
      done[i] = 1;
    }
    if (rots.empty()) {  // only permutations were free: fold them into the frame
      for (int q : perms) F = compose(F, perm_of(lg[q], LB), LB);
      continue;
    }
    // register slots: the excitation's wires first (SE: A -> 0, B -> 1;
    // DE: A -> 0, 1, B -> 2, 3), then the other rotation bits, then padding
    uint32_t used = 0, m = 0;
    const auto put = [&](uint32_t b) {
      if (!((used >> b) & 1u)) {
        ph.slot_bit[m++] = b;
        used |= 1u << b;
      }
    };
    if (fix != kFixNone) {
      for (uint32_t b = 0; b < LB; ++b)
        if ((fix_a >> b) & 1u) put(b);
      for (uint32_t b = 0; b < LB; ++b)
        if ((fix_b >> b) & 1u) put(b);
    }
    for (uint32_t b = 0; b < LB; ++b)
      if ((regs >> b) & 1u) put(b);
    for (int b = static_cast<int>(LB) - 1; b >= 0 && m < R; --b) put(static_cast<uint32_t>(b));
    const auto slot_of = [&](uint32_t b) {
      for (uint32_t j = 0; j < R; ++j)
        if (ph.slot_bit[j] == b) return static_cast<int>(j);
      return -1;
    };
    // steps: excitation, then one RY per slot; a gate that cannot follow
    // the step's content in that order opens a new step
    TileStep cur{};
    bool open = false;
    const auto flush = [&] {
      if (open) ph.steps.push_back(cur);
      cur = TileStep{};
      open = false;
    };
    for (size_t q = 0; q < rots.size(); ++q) {
      const LocalGate& g = lg[rots[q]];
      out.rot_gate.push_back(signs[q] * (rots[q] + 1));  // entry index = rot_gate.size(); sign = angle sign
      const int16_t entry = static_cast<int16_t>(out.rot_gate.size());
      if (g.ma == 0) {  // RY
        const int j = slot_of(__builtin_ctz(g.mb));
        if (open && cur.ry[j] != 0) flush();
        cur.ry[j] = entry;
      } else if (__builtin_popcount(g.ma) == 1) {  // SingleExcitation on slots (0, 1)
        bool any_ry = false;
        for (int j = 0; j < 5; ++j) any_ry = any_ry || cur.ry[j] != 0;
        if (open && (cur.flags != 0 || any_ry)) flush();
        cur.se = entry;
        cur.flags |= 1u;
      } else {  // DoubleExcitation on slots 0..3
        bool any_ry = false;
        for (int j = 0; j < 5; ++j) any_ry = any_ry || cur.ry[j] != 0;
        if (open && ((cur.flags & 2u) || any_ry)) flush();
        cur.de = entry;
        cur.flags |= 2u;
      }
      open = true;
    }
    flush();
    n_steps += ph.steps.size();
    for (int q : perms) F = compose(F, perm_of(lg[q], LB), LB);
    ph.store = ph.load;
    out.phases.push_back(std::move(ph));
    if (out.phases.size() == kMaxPhases || n_steps + kPhaseRot > kMaxSteps ||
        out.rot_gate.size() + 1 + kPhaseRot > kMaxRot)
      break;
  }
  // the permutations taken after the last phase: its stores leave the tile
  // in plain order, i.e. logical L of its frame at F_end^-1 (F_last (L))
  out.end_frame = F;
  if (!out.phases.empty()) {
    PhasePlan& last = out.phases.back();
    last.store = compose(inverse(F, LB), last.load, LB);
  }
  return out;
}

// Bank-group vector of shared-memory slot offset v (fp64: the 16-byte chunk
// of a 128-byte line, 3 bits; fp32: the 8-byte unit, 4 bits).
uint32_t bank_of(bool f64, uint32_t v) { return f64 ? (v & 7u) : (v & 15u); }

uint32_t gf2_rank(std::vector<uint32_t> v) {
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

// Thread bits of a phase: the LB - R non-register local bits, ordered so that
// the lanes of one shared-memory wavefront (8 lanes x 16 B fp64, 16 lanes x
// 8 B fp32) cover as many bank groups as possible through the load and the
// store maps.
template <typename T>
std::vector<uint32_t> thread_bits(const PhasePlan& ph, uint32_t R, uint32_t LB) {
  const bool f64 = sizeof(T) == 8;
  uint32_t regs = 0;
  for (uint32_t j = 0; j < R; ++j) regs |= 1u << ph.slot_bit[j];
  std::vector<uint32_t> free_bits;
  for (uint32_t b = 0; b < LB; ++b)
    if (!((regs >> b) & 1u)) free_bits.push_back(b);
  const uint32_t q = std::min<uint32_t>(f64 ? 3 : 4, static_cast<uint32_t>(free_bits.size()));
  std::vector<uint32_t> best;
  uint32_t best_score = 0;
  const size_t m = free_bits.size();
  for (uint32_t mask = 0; mask < (1u << m); ++mask) {
    if (static_cast<uint32_t>(__builtin_popcount(mask)) != q) continue;
    std::vector<uint32_t> pick, vl, vs;
    for (size_t i = 0; i < m; ++i)
      if ((mask >> i) & 1u) {
        pick.push_back(free_bits[i]);
        vl.push_back(bank_of(f64, swz<T>(ph.load.col[free_bits[i]])));
        vs.push_back(bank_of(f64, swz<T>(ph.store.col[free_bits[i]])));
      }
    const uint32_t score = 2 * gf2_rank(vl) + gf2_rank(vs);
    if (best.empty() || score > best_score) {
      best = pick;
      best_score = score;
    }
  }
  std::vector<uint32_t> out = best;
  for (uint32_t b : free_bits)
    if (std::find(out.begin(), out.end(), b) == out.end()) out.push_back(b);
  return out;
}

// Launch parameters for the pass; one launch per chunk of phases that fits
// the parameter tables.
template <typename T>
std::vector<TileParams> build_launches(uint32_t n, uint32_t batch, uint32_t B, const std::vector<TGate>& gates,
                                       const Pass& pass, const double* cs_dev) {
  const uint32_t LB = B + static_cast<uint32_t>(pass.hbits.size());
  const uint32_t R = sizeof(T) == 8 ? kR64 : kR32;
  TileParams base{};
  base.n = n;
  base.B = B;
  base.k = static_cast<uint32_t>(pass.hbits.size());
  base.batch = batch;
  base.cs = cs_dev;
  for (uint32_t j = 0; j < base.k; ++j) base.hb[j] = pass.hbits[j];
  const std::vector<LocalGate> lg = local_gates(n, B, pass.hbits, gates, pass);
  // a pass of X / CNOT gates only is an affine index map F on the local
  // bits: out[L] = in[F(L)] with F = f_1 o ... o f_m (gate 1 first in the
  // circuit, so f_m acts on L first); applied in the write-back
  bool perm = true;
  for (const LocalGate& o : lg) perm = perm && !o.rot;
  if (perm) {
    Affine F = Affine::identity(LB);
    for (const LocalGate& o : lg) F = compose(F, perm_of(o, LB), LB);
    TileParams p = base;
    p.perm_only = 1;
    p.perm_c = F.c;
    for (uint32_t b = 0; b < 16; ++b) p.perm_col[b] = b < LB ? F.col[b] : 0u;
    return {p};
  }
  std::vector<TileParams> out;
  std::vector<char> done(lg.size(), 0);
  const auto left = [&] {
    for (char d : done)
      if (!d) return true;
    return false;
  };
  while (left()) {
    const PassPlan plan = plan_launch(lg, done, LB, R);
    if (plan.phases.empty()) {
      // only permutations were left for this launch: one pure re-layout
      TileParams p = base;
      p.perm_only = 1;
      p.perm_c = plan.end_frame.c;
      for (uint32_t b = 0; b < 16; ++b) p.perm_col[b] = b < LB ? plan.end_frame.col[b] : 0u;
      out.push_back(p);
      continue;
    }
    TileParams p = base;
    p.n_rot = static_cast<uint32_t>(plan.rot_gate.size()) + 1;
    p.rot_param[0] = -1;
    p.rot_c[0] = 1.0;
    p.rot_s[0] = 0.0;
    for (size_t k = 0; k < plan.rot_gate.size(); ++k) {
      const int code = plan.rot_gate[k];
      const LocalGate& g = lg[std::abs(code) - 1];
      p.rot_param[k + 1] = g.param;
      p.rot_c[k + 1] = g.c;
      p.rot_s[k + 1] = g.s;
      p.rot_neg[k + 1] = code < 0 ? 1 : 0;  // (c, s) -> (c, -s)
    }
    uint32_t n_steps = 0;
    for (size_t pi = 0; pi < plan.phases.size(); ++pi) {
      const PhasePlan& ph = plan.phases[pi];
      TilePhase& tp = p.ph[p.n_phases++];
      // the launch's last phase stores straight to HBM when its lanes can be
      // the run bits 0..B-1 (no register slot there) and the store map keeps
      // those bits among themselves (a warp then writes one run)
      bool direct = pi + 1 == plan.phases.size() && !std::getenv("VQF_TILE_NO_DIRECT");
      for (uint32_t j = 0; j < R; ++j) direct = direct && ph.slot_bit[j] >= B;
      for (uint32_t b = 0; b < B; ++b) direct = direct && (ph.store.col[b] >> B) == 0;
      std::vector<uint32_t> tb;
      if (direct) {
        for (uint32_t b = 0; b < LB; ++b) {
          bool reg = false;
          for (uint32_t j = 0; j < R; ++j) reg = reg || ph.slot_bit[j] == b;
          if (!reg) tb.push_back(b);
        }
      } else {
        tb = thread_bits<T>(ph, R, LB);
      }
      const auto st_map = [&](uint32_t v) { return static_cast<uint16_t>(direct ? v : swz<T>(v)); };
      tp.direct = direct ? 1 : 0;
      tp.ld_c = static_cast<uint16_t>(swz<T>(ph.load.c));
      tp.st_c = st_map(ph.store.c);
      for (size_t j = 0; j < tb.size(); ++j) {
        tp.ld_tb[j] = static_cast<uint16_t>(swz<T>(ph.load.col[tb[j]]));
        tp.st_tb[j] = st_map(ph.store.col[tb[j]]);
      }
      bool same = ph.load.c == ph.store.c;
      for (uint32_t j = 0; j < R; ++j) {
        tp.ld_r[j] = static_cast<uint16_t>(swz<T>(ph.load.col[ph.slot_bit[j]]));
        tp.st_r[j] = st_map(ph.store.col[ph.slot_bit[j]]);
      }
      for (uint32_t b = 0; b < LB; ++b) same = same && ph.load.col[b] == ph.store.col[b];
      tp.relayout = same || direct ? 0 : 1;
      tp.step0 = static_cast<uint16_t>(n_steps);
      tp.n_steps = static_cast<uint16_t>(ph.steps.size());
      for (const TileStep& st : ph.steps) p.steps[n_steps++] = st;
    }
    out.push_back(p);
  }
  return out;
}

template <typename T>
void launch_pass(vqf_statevector* sv, const std::vector<TGate>& gates, const Pass& pass, uint32_t B,
                 const double* cs_dev, uint32_t active = 0) {
  // active: batch entries [0, active) take the pass (0 = all)
  if (active == 0) active = sv->batch;
  const uint32_t n = sv->n_qubits;
  constexpr int R = sizeof(T) == 8 ? kR64 : kR32;
  const uint32_t LB = B + static_cast<uint32_t>(pass.hbits.size());
  const uint64_t n_tiles = uint64_t{1} << (n - LB);
  // persistent over one entry's tiles; a batched state launches a CTA set
  // per entry, so give each group >= 16 tiles there to amortise the CTA
  // prologue over enough traffic
  uint64_t gx = std::min<uint64_t>(n_tiles, kTileBlocks);
  constexpr int kGroups = kGroupsOf<T>;
  if (active > 1) gx = std::max<uint64_t>(1, std::min<uint64_t>(gx, n_tiles / (kGroups * 16)));
  const unsigned grid = static_cast<unsigned>(gx);
  const uint32_t run_bytes = static_cast<uint32_t>(sizeof(typename V2<T>::type) << B);
  // high bits B, B+1, ... (spectator padding usually starts there) make
  // adjacent runs: one TMA box of 2^merge runs instead of 2^merge boxes
  uint32_t merge = 0;
  while (merge < pass.hbits.size() && pass.hbits[merge] == B + merge && (run_bytes << (merge + 1)) <= 32768u) ++merge;
  if (sizeof(T) == 8 || std::getenv("VQF_TILE_NO_MERGE")) merge = 0;  // measured: fp32 +10%, fp64 -1.4%
  // a pass whose gathered bits form one window moves each tile as one 5-d box
  bool win = !pass.hbits.empty() && pass.hbits[0] >= B && !std::getenv("VQF_TILE_NO_WINDOW");
  for (size_t m = 1; win && m < pass.hbits.size(); ++m) win = pass.hbits[m] == pass.hbits[0] + m;
  if (win) merge = 0;
  const CUtensorMap* map = win ? tma::cached_tile_map(sv, B, pass.hbits[0], static_cast<uint32_t>(pass.hbits.size()))
                               : tma::cached_state_map(sv, run_bytes << merge);
  const size_t smem = kSlotsOf<T> * (sizeof(typename V2<T>::type) << LB) + 8 * kSlotsOf<T> + 1024;
  auto* amps = static_cast<typename V2<T>::type*>(sv->amps);
  for (TileParams& p : build_launches<T>(n, sv->batch, B, gates, pass, cs_dev)) {
    p.merge = merge;
    p.win = win ? 1u : 0u;
    const dim3 g(grid, active);
    const unsigned threads = kGroups << (LB - R);
    constexpr int LBmax = sizeof(T) == 8 ? kLB64 : kLB32;
    switch (LBmax - static_cast<int>(LB)) {
      case 0:
        if (p.perm_only) k_tile<T, R, LBmax, true><<<g, threads, smem, sv->stream>>>(amps, *map, p);
        else k_tile<T, R, LBmax, false><<<g, threads, smem, sv->stream>>>(amps, *map, p);
        break;
      case 1:
        if (p.perm_only) k_tile<T, R, LBmax - 1, true><<<g, threads, smem, sv->stream>>>(amps, *map, p);
        else k_tile<T, R, LBmax - 1, false><<<g, threads, smem, sv->stream>>>(amps, *map, p);
        break;
      case 2:
        if (p.perm_only) k_tile<T, R, LBmax - 2, true><<<g, threads, smem, sv->stream>>>(amps, *map, p);
        else k_tile<T, R, LBmax - 2, false><<<g, threads, smem, sv->stream>>>(amps, *map, p);
        break;
      default:
        throw Error(VQF_LOGIC_ERROR, "tile pass: unsupported tile width");
    }
    VQF_LAUNCHED();
  }
}

template <typename T, int R, int LB>
void opt_in_smem() {
  constexpr int kGroups = kGroupsOf<T>;
  const int bytes = kSlotsOf<T> * (static_cast<int>(sizeof(T)) * 2 << LB) + 8 * kSlotsOf<T> + 1024;
  VQF_CUDA(cudaFuncSetAttribute(k_tile<T, R, LB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  VQF_CUDA(cudaFuncSetAttribute(k_tile<T, R, LB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void ensure_tile_attrs(const vqf_statevector* sv) {
  static thread_local int opted = -1;
  if (opted != sv->device) {
    opt_in_smem<double, kR64, kLB64>();
    opt_in_smem<double, kR64, kLB64 - 1>();
    opt_in_smem<double, kR64, kLB64 - 2>();
    opt_in_smem<float, kR32, kLB32>();
    opt_in_smem<float, kR32, kLB32 - 1>();
    opt_in_smem<float, kR32, kLB32 - 2>();
    opted = sv->device;
  }
}

// Registers below the narrowest instantiated tile (full width - 2 bits, at
// least one warp per group) take one launch per gate.
bool tile_too_small(uint32_t n, int32_t dtype) {
  return n < static_cast<uint32_t>(std::max(tile_lb(dtype) - 2, tile_r(dtype) + 5));
}

void apply_single(vqf_statevector* sv, const TGate& g, const double* cs_dev) {
  GateArgs ga{g.kind, g.n_wires, {g.wires[0], g.wires[1], g.wires[2], g.wires[3]}, g.c, g.s,
              g.param >= 0 ? cs_dev + 2 * (size_t)g.param * sv->batch : nullptr};
  sv_apply(sv, ga);
}

}  // namespace

std::vector<int> plan_tile_passes(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates) {
  if (tile_too_small(n_qubits, dtype)) return std::vector<int>(gates.size(), 1);
  uint32_t B, kmax;
  tile_shape(n_qubits, dtype, B, kmax);
  std::vector<int> out;
  for (const Pass& p : schedule(n_qubits, B, kmax, gates)) out.push_back(static_cast<int>(p.gates.size()));
  return out;
}

void plan_tile_counts(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates, uint32_t* passes,
                      uint32_t* fused_ops) {
  if (tile_too_small(n_qubits, dtype)) {
    *passes = static_cast<uint32_t>(gates.size());
    *fused_ops = 0;
    return;
  }
  uint32_t B, kmax;
  tile_shape(n_qubits, dtype, B, kmax);
  const std::vector<Pass> ps = schedule(n_qubits, B, kmax, gates);
  uint32_t phases = 0, launches = 0;
  for (const Pass& p : ps) {
    if (!p.hbits.empty() && p.hbits[0] == 0xffffffffu) {
      ++launches;
      continue;
    }
    const std::vector<TileParams> ls = dtype == VQF_F64 ? build_launches<double>(n_qubits, 1, B, gates, p, nullptr)
                                                        : build_launches<float>(n_qubits, 1, B, gates, p, nullptr);
    for (const TileParams& tp : ls) {
      phases += tp.n_phases;
      if (std::getenv("VQF_TILE_DEBUG")) {
        std::fprintf(stderr, "launch %u: k=%u hb=", launches, tp.k);
        for (uint32_t j = 0; j < tp.k; ++j) std::fprintf(stderr, "%u,", tp.hb[j]);
        std::fprintf(stderr, " perm=%u phases=%u:", tp.perm_only, tp.n_phases);
        for (uint32_t q = 0; q < tp.n_phases; ++q)
          std::fprintf(stderr, " %u%s%s", tp.ph[q].n_steps, tp.ph[q].relayout ? "*" : "", tp.ph[q].direct ? "d" : "");
        std::fprintf(stderr, "\n");
      }
      ++launches;
    }
  }
  *passes = launches;
  *fused_ops = phases;
}

int run_circuit_tiled(vqf_statevector* sv, const std::vector<TGate>& gates, const double* cs_dev) {
  if (gates.empty()) return 0;
  const uint32_t n = sv->n_qubits;
  if (tile_too_small(n, sv->dtype)) {
    for (const TGate& g : gates) apply_single(sv, g, cs_dev);
    return static_cast<int>(gates.size());
  }
  uint32_t B, kmax;
  tile_shape(n, sv->dtype, B, kmax);
  ensure_tile_attrs(sv);
  const std::vector<Pass> passes = schedule(n, B, kmax, gates);
  for (const Pass& pass : passes) {
    if (!pass.hbits.empty() && pass.hbits[0] == 0xffffffffu) {
      apply_single(sv, gates[pass.gates[0]], cs_dev);
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
  if (tile_too_small(n_qubits, dtype) || gates.empty()) return {};  // per-gate path
  uint32_t B, kmax;
  tile_shape(n_qubits, dtype, B, kmax);
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
  if (tile_too_small(n, sv->dtype)) throw Error(VQF_LOGIC_ERROR, "shared-prefix circuit: register below tile size");
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
    if (!passes[p].hbits.empty() && passes[p].hbits[0] == 0xffffffffu)
      throw Error(VQF_LOGIC_ERROR, "shared-prefix circuit: single-gate pass");
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
