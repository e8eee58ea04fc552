// TMA (cp.async.bulk.tensor) and mbarrier helpers shared by the tiled
// kernels (tile.cu: fused gate passes; expect_tile.cu: multi-group
// expectation passes).  SASS: UTMALDG / UTMASTG / SYNCS.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "sv.cuh"

namespace vqf {
namespace tma {

__device__ __forceinline__ uint64_t insert_zero64(uint64_t k, uint32_t bit) {
  const uint64_t low = k & ((uint64_t{1} << bit) - 1);
  return ((k >> bit) << (bit + 1)) | low;
}

// ---- TMA / mbarrier helpers (SASS: UTMALDG / UTMASTG / SYNCS)
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
// one run (box {128 B, rows, 1}) of the state, 128 B-swizzled into shared
// memory; completion counted on the mbarrier
__device__ __forceinline__ void tma_load_run(void* dst, const CUtensorMap* map, int32_t row, int32_t entry,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(0), "r"(row), "r"(entry), "r"(smem_addr(bar))
      : "memory");
}
// the reverse: one run from shared memory (un-swizzled by the map) to HBM
__device__ __forceinline__ void tma_store_run(const void* src, const CUtensorMap* map, int32_t row, int32_t entry) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map), "r"(0),
               "r"(row), "r"(entry), "r"(smem_addr(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Shared-memory slot of local amplitude L under the TMA 128 B swizzle: the
// 16-byte chunk index (bits 4..6 of the byte offset) is xor-ed with the
// 128-byte row index mod 8 (bits 7..9).  Linear over GF(2).
template <typename T>
__host__ __device__ __forceinline__ uint32_t swz(uint32_t L) {
  if (sizeof(T) == 8) return L ^ ((L >> 3) & 7u);   // 16 B amplitude = one chunk
  return L ^ (((L >> 4) & 7u) << 1);                 // 8 B amplitude: chunk = L >> 1
}

// Named barrier over the NT threads of one consumer group (id 0 is
// __syncthreads).
template <int NT>
__device__ __forceinline__ void group_sync(uint32_t group) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "r"(NT) : "memory");
}


// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();

// The state as a 3-d tensor {128 B row, rows, batch entry}; box = one run of
// run_bytes (<= 32 rows), 128 B swizzle.  Loads and stores share it.
CUtensorMap state_map(const vqf_statevector* sv, uint32_t run_bytes);

// Cached per (allocation, run size, shape) on the calling thread.
const CUtensorMap* cached_state_map(const vqf_statevector* sv, uint32_t run_bytes);

// Window map of a tile = B low bits (one 128 B row; B = 3 fp64, 4 fp32) x the
// contiguous bits [h, h + k): one TMA box per tile (cached per thread).
CUtensorMap window_map(const vqf_statevector* sv, uint32_t h, uint32_t k);
const CUtensorMap* cached_window_map(const vqf_statevector* sv, uint32_t h, uint32_t k);

// One tile of a window map: coordinates {0, mid, 0, top}.
__device__ __forceinline__ void tma_load_window(void* dst, const CUtensorMap* map, int32_t mid, int32_t top,
                                                uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(0), "r"(mid), "r"(0), "r"(top), "r"(smem_addr(bar))
      : "memory");
}

// Tile map of a fused pass whose gathered bits are one window [h, h + k):
// the state as {128 B row, run rows, mid, window, top x batch} with runs of
// 2^B amplitudes (B >= the row's bits), so ONE 5-d box moves the whole tile
// (2^(B + k) amplitudes, the run-by-run smem image: run w at w * run bytes).
CUtensorMap tile_map(const vqf_statevector* sv, uint32_t B, uint32_t h, uint32_t k);
const CUtensorMap* cached_tile_map(const vqf_statevector* sv, uint32_t B, uint32_t h, uint32_t k);

// One tile of a tile map: coordinates {0, 0, mid, 0, top}.
__device__ __forceinline__ void tma_load_tile(void* dst, const CUtensorMap* map, int32_t mid, int32_t top,
                                              uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(0), "r"(0), "r"(mid), "r"(0), "r"(top), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_tile(const void* src, const CUtensorMap* map, int32_t mid, int32_t top) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(map),
               "r"(0), "r"(0), "r"(mid), "r"(0), "r"(top), "r"(smem_addr(src))
               : "memory");
}

}  // namespace tma
}  // namespace vqf
