// Gate fusion through shared-memory tiles.
//
// A pass works on "gathered tiles": 2^B contiguous low-index amplitudes
// (coalesced HBM transfers) times 2^k chosen high index bits h_0..h_{k-1}
// (B + k local bits = 64 KB of shared memory).  The CTA loads a tile, applies
// every gate of the pass whose wires map into its local bits — gates become
// shared-memory passes between __syncthreads — and writes it back: one HBM
// read + write of the state per pass instead of per gate.
//
// The host scheduler walks the circuit's dependency DAG (gates sharing a wire
// keep their order; gates on disjoint wires commute) and greedily packs ready
// gates into a pass while the union of their high bits fits in k.  For the
// hardware-efficient ansatz every RY on a low wire rides along in every pass,
// and the CNOT chain advances k - 1 wires per pass.
//
// Per-gate arithmetic is exactly that of the single-gate kernels (sv.cu);
// commuting gates may be applied in a different order, so amplitudes agree
// with the unfused path to rounding (~1e-16).
#include <algorithm>

#include "tile.cuh"

namespace vqf {

namespace {

constexpr int kTileThreads = 1024;  // one persistent CTA per SM, 8 warps per SMSP
constexpr int kMaxOps = 64;  // TileParams stays under the 4 KB kernel-parameter limit
constexpr int kMaxHigh = 6;
constexpr int kTileBlocks = 148;  // persistent: one CTA per SM
constexpr int kStages = 3;       // TMA ring depth (3 x 64 KB)

enum : int32_t { OP_SWAP = 0, OP_ROT = 1 };

struct TileOp {
  int32_t mode;   // OP_SWAP (X, CNOT) or OP_ROT (RY, DE, SE)
  int32_t param;  // per-entry (c, s) index or -1
  uint32_t ma, mb;  // local index patterns of the two amplitudes of a pair
  uint32_t pos;   // local bit positions, 8 bits each, ascending
  uint32_t npos;
  double c, s;
};

struct TileParams {
  uint32_t n, B, k, n_ops, batch;
  uint32_t hb[kMaxHigh];  // global bit of local bit B + j, ascending
  const double* cs;
  TileOp ops[kMaxOps];
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

// ---- TMA bulk-copy helpers (sm_90+ PTX; SASS: UBLKCP / SYNCS)
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
// global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// shared -> global, tracked by bulk groups
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Inserts zero bits at the op's (ascending) local bit positions; npos is
// 1, 2 or 4 so every case is a fixed shift/mask sequence.
__device__ __forceinline__ uint32_t ins0(uint32_t r, uint32_t b) { return ((r >> b) << (b + 1)) | (r & ((1u << b) - 1)); }
__device__ __forceinline__ uint32_t spread(uint32_t r, const TileOp& op) {
  r = ins0(r, op.pos & 0xffu);
  if (op.npos == 1) return r;
  r = ins0(r, (op.pos >> 8) & 0xffu);
  if (op.npos == 2) return r;
  r = ins0(r, (op.pos >> 16) & 0xffu);
  return ins0(r, (op.pos >> 24) & 0xffu);
}

// Global start index of run j (0 <= j < 2^k) of tile `tile`.
__device__ __forceinline__ uint64_t run_start(const TileParams& p, uint64_t tile, uint32_t j) {
  uint64_t base = tile << p.B;
  for (uint32_t m = 0; m < p.k; ++m) base = insert_zero64(base, p.hb[m]);
  for (uint32_t m = 0; m < p.k; ++m) base |= (uint64_t)((j >> m) & 1u) << p.hb[m];
  return base;
}

// Persistent tile kernel with a kStages-deep TMA ring.  Thread 0 is the
// copy engine: it keeps kStages - 1 tiles in flight, issuing the 2^k
// contiguous 2^B-amplitude runs of each as TMA bulk copies (one mbarrier per
// stage, expect_tx = tile bytes), while all threads apply the pass's gates to
// the current tile in shared memory; the tile then leaves as bulk stores.
template <typename T>
__global__ void __launch_bounds__(kTileThreads, 1) k_tile(typename V2<T>::type* __restrict__ a, const TileParams p) {
  using A = typename V2<T>::type;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t LB = p.B + p.k, NL = 1u << LB;
  const uint32_t run_amps = 1u << p.B, n_runs = 1u << p.k;
  const uint32_t tile_bytes = NL * sizeof(A), run_bytes = run_amps * sizeof(A);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + kStages * (size_t)tile_bytes);
  __shared__ uint64_t run_off[1 << kMaxHigh];
  A* s = a + ((uint64_t)blockIdx.y << p.n);
  const uint64_t n_tiles = uint64_t{1} << (p.n - LB);
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) mbar_init(&bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const auto stage_buf = [&](int st) { return reinterpret_cast<A*>(smem_raw + (size_t)st * tile_bytes); };
  // warp 0 issues a tile: lane 0 arms the stage's mbarrier with the tile's
  // byte count, lane j copies run j (the arm and the copies may land in any
  // order: the phase needs both the arrival and the bytes)
  const auto issue_load = [&](uint64_t tile, int st) {
    const uint32_t lane = threadIdx.x;
    if (lane == 0) mbar_expect_tx(&bar[st], tile_bytes);
    A* dst = stage_buf(st);
    for (uint32_t j = lane; j < n_runs; j += 32)
      bulk_g2s(dst + (size_t)j * run_amps, s + run_start(p, tile, j), run_bytes, &bar[st]);
  };
  if (threadIdx.x < 32)
    for (int st = 0; st < kStages - 1; ++st) {
      const uint64_t t0 = blockIdx.x + (uint64_t)st * gridDim.x;
      if (t0 < n_tiles) issue_load(t0, st);
    }
  uint64_t tile = blockIdx.x;
  for (uint32_t it = 0; tile < n_tiles; tile += gridDim.x, ++it) {
    const int cur = it % kStages;
    const uint64_t ahead = tile + (uint64_t)(kStages - 1) * gridDim.x;
    // that stage's previous tile was written back (and the buffer released)
    // before the __syncthreads that closed the previous iteration
    if (threadIdx.x < 32 && ahead < n_tiles) issue_load(ahead, (it + kStages - 1) % kStages);
    mbar_wait(&bar[cur], (it / kStages) & 1u);
    A* t = stage_buf(cur);
    for (uint32_t o = 0; o < p.n_ops; ++o) {
      const TileOp op = p.ops[o];
      T c = static_cast<T>(op.c), sn = static_cast<T>(op.s);
      if (op.param >= 0) {
        const double* cs = p.cs + 2 * ((size_t)op.param * p.batch + blockIdx.y);
        c = static_cast<T>(cs[0]);
        sn = static_cast<T>(cs[1]);
      }
      const uint32_t npairs = NL >> op.npos;
      // two pairs per thread per step, all four shared-memory loads issued
      // before any arithmetic (pairs of one op never overlap)
      for (uint32_t q0 = threadIdx.x; q0 < npairs; q0 += 2 * kTileThreads) {
        uint32_t ia[2], ib[2];
        A x[2], y[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t r = spread(q0 + u * kTileThreads, op);
          ia[u] = r | op.ma;
          ib[u] = r | op.mb;
          if (q0 + u * kTileThreads < npairs) {
            x[u] = t[ia[u]];
            y[u] = t[ib[u]];
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (q0 + u * kTileThreads >= npairs) break;
          if (op.mode == OP_SWAP) {
            t[ia[u]] = y[u];
            t[ib[u]] = x[u];
          } else {  // a' = c a - s b, b' = s a + c b (statevector.hpp:160-163, :195-196)
            A xa, yb;
            xa.x = c * x[u].x - sn * y[u].x;
            xa.y = c * x[u].y - sn * y[u].y;
            yb.x = sn * x[u].x + c * y[u].x;
            yb.y = sn * x[u].y + c * y[u].y;
            t[ia[u]] = xa;
            t[ib[u]] = yb;
          }
        }
      }
      __syncthreads();
    }
    // write-back: coalesced 16-byte stores, consecutive threads along a run
    if (threadIdx.x < n_runs) run_off[threadIdx.x] = run_start(p, tile, threadIdx.x);
    __syncthreads();
    const uint32_t low_mask = run_amps - 1;
    for (uint32_t li = threadIdx.x; li < NL; li += kTileThreads) s[run_off[li >> p.B] | (li & low_mask)] = t[li];
    __syncthreads();  // buffer free for the stage's next TMA load
  }
}

struct Pass {
  std::vector<uint32_t> hbits;  // ascending global bits
  std::vector<int> gates;
};

// Local bit budget: 64 KB of shared memory per tile (kStages tiles resident).
void tile_shape(uint32_t n, int32_t dtype, uint32_t& B, uint32_t& kmax) {
  const uint32_t LB = dtype == VQF_F64 ? 12 : 13;
  if (n <= LB) {
    B = n;
    kmax = 0;
    return;
  }
  B = std::max<uint32_t>(LB - kMaxHigh + 2, 7);  // >= 2 KB contiguous runs (fp64: B = 8)
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
    while (added && pass.gates.size() < static_cast<size_t>(kMaxOps)) {
      added = false;
      for (size_t i = 0; i < G; ++i) {
        if (done[i]) continue;
        bool ready = true;
        for (int pr : preds[i]) ready = ready && done[pr];
        if (!ready) continue;
        std::vector<uint32_t> u = pass.hbits;
        for (uint32_t b : high_bits(gates[i]))
          if (std::find(u.begin(), u.end(), b) == u.end()) u.push_back(b);
        if (u.size() > kmax) continue;
        pass.hbits = u;
        pass.gates.push_back(static_cast<int>(i));
        done[i] = 1;
        --remaining;
        added = true;
        break;  // rescan from the first gate: readiness changed
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
    std::sort(pass.hbits.begin(), pass.hbits.end());
    passes.push_back(std::move(pass));
  }
  return passes;
}

template <typename T>
void launch_pass(vqf_statevector* sv, const std::vector<TGate>& gates, const Pass& pass, uint32_t B,
                 const double* cs_dev) {
  const uint32_t n = sv->n_qubits;
  TileParams p{};
  p.n = n;
  p.B = B;
  p.k = static_cast<uint32_t>(pass.hbits.size());
  p.batch = sv->batch;
  p.cs = cs_dev;
  for (uint32_t j = 0; j < p.k; ++j) p.hb[j] = pass.hbits[j];
  const auto local = [&](uint32_t wire) -> uint32_t {
    const uint32_t b = n - 1 - wire;
    if (b < B) return b;
    for (uint32_t j = 0; j < p.k; ++j)
      if (p.hb[j] == b) return B + j;
    throw Error(VQF_LOGIC_ERROR, "tile scheduler: wire outside the pass");
  };
  for (int gi : pass.gates) {
    const TGate& g = gates[gi];
    TileOp op{};
    op.param = g.param;
    op.c = g.c;
    op.s = g.s;
    uint32_t lb[4];
    for (uint32_t w = 0; w < g.n_wires; ++w) lb[w] = local(g.wires[w]);
    switch (g.kind) {
      case VQF_GATE_PAULI_X:
      case VQF_GATE_RY:
        op.mode = g.kind == VQF_GATE_PAULI_X ? OP_SWAP : OP_ROT;
        op.ma = 0;
        op.mb = 1u << lb[0];
        break;
      case VQF_GATE_CNOT:
        op.mode = OP_SWAP;
        op.ma = 1u << lb[0];
        op.mb = (1u << lb[0]) | (1u << lb[1]);
        break;
      case VQF_GATE_DOUBLE_EXCITATION:
        op.mode = OP_ROT;
        op.ma = (1u << lb[0]) | (1u << lb[1]);  // |1100>
        op.mb = (1u << lb[2]) | (1u << lb[3]);  // |0011>
        break;
      case VQF_GATE_SINGLE_EXCITATION:
        op.mode = OP_ROT;
        op.ma = 1u << lb[0];  // |10>
        op.mb = 1u << lb[1];  // |01>
        break;
      default:
        throw Error(VQF_LOGIC_ERROR, "unknown gate kind");
    }
    std::sort(lb, lb + g.n_wires);
    op.npos = g.n_wires;
    op.pos = 0;
    for (uint32_t w = 0; w < g.n_wires; ++w) op.pos |= lb[w] << (8 * w);
    p.ops[p.n_ops++] = op;
  }
  const uint32_t LB = B + p.k;
  const uint64_t n_tiles = uint64_t{1} << (n - LB);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n_tiles, kTileBlocks));
  const size_t smem = kStages * (sizeof(typename V2<T>::type) << LB) + 8 * kStages;  // ring + mbarriers
  k_tile<T><<<dim3(grid, sv->batch), kTileThreads, smem, sv->stream>>>(static_cast<typename V2<T>::type*>(sv->amps), p);
  VQF_LAUNCHED();
}

}  // namespace

std::vector<int> plan_tile_passes(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates) {
  uint32_t B, kmax;
  tile_shape(n_qubits, dtype, B, kmax);
  std::vector<int> out;
  for (const Pass& p : schedule(n_qubits, B, kmax, gates)) out.push_back(static_cast<int>(p.gates.size()));
  return out;
}

int run_circuit_tiled(vqf_statevector* sv, const std::vector<TGate>& gates, const double* cs_dev) {
  if (gates.empty()) return 0;
  const uint32_t n = sv->n_qubits;
  uint32_t B, kmax;
  tile_shape(n, sv->dtype, B, kmax);
  static thread_local int opted = -1;
  if (opted != sv->device) {
    VQF_CUDA(cudaFuncSetAttribute(k_tile<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * 64 * 1024 + 8 * kStages));
    VQF_CUDA(cudaFuncSetAttribute(k_tile<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * 64 * 1024 + 8 * kStages));
    opted = sv->device;
  }
  const std::vector<Pass> passes = schedule(n, B, kmax, gates);
  for (const Pass& pass : passes) {
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

}  // namespace vqf
