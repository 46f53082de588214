// sof_tma.cuh — TMA (cp.async.bulk.tensor) staging of Gaussian records for sm_100a.
//
// The opacity-evaluation kernels stream a tile's Gaussian list — an INDEX list into
// the per-view record array (tiles.hpp:88-92 keeps lists of indices) — through
// shared memory. The records are gathered with the sm_100a TMA row gather
// (`tile::gather4`: four 128-B rows of a 2D tensor per instruction, completion
// counted on an mbarrier), double-buffered so the next chunk lands while the
// current one is evaluated. The record array is described by a 2D tensor map of
// {16 x 8 B columns, n rows}, box {16, 1}.
#pragma once

#include <cuda.h>
#include <cstdint>

namespace sofk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make barrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

// a tensor map in global memory written by the host before the launch
__device__ __forceinline__ void tma_fence_acquire(const CUtensorMap* tmap) {
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(tmap))
               : "memory");
}

// Four rows (r0..r3) of the tensor map's 2D tensor, columns [0, box0), into
// consecutive rows at dst; completion (4 x row bytes) is signalled on bar.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tmap, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

// Warp-level issue of one chunk of up to 32 record rows: lane l holds the row index
// of entry l (lanes >= cnt are ignored). Rows are gathered four at a time; a partial
// last group repeats the chunk's last row (those slots are never read). All 32 lanes
// of the calling warp must be converged.
__device__ __forceinline__ void tma_issue_rows(void* dst, const CUtensorMap* tmap, int my_row, int cnt,
                                               uint64_t* bar, uint32_t row_bytes) {
  const int lane = threadIdx.x & 31;
  const int row = __shfl_sync(0xffffffffu, my_row, lane < cnt ? lane : cnt - 1);
  const int n4 = (cnt + 3) >> 2;
  if (lane == 0) mbar_arrive_expect_tx(bar, uint32_t(n4) * 4u * row_bytes);
  __syncwarp();
  const int q = lane & 7;
  const int r0 = __shfl_sync(0xffffffffu, row, 4 * q);
  const int r1 = __shfl_sync(0xffffffffu, row, 4 * q + 1);
  const int r2 = __shfl_sync(0xffffffffu, row, 4 * q + 2);
  const int r3 = __shfl_sync(0xffffffffu, row, 4 * q + 3);
  if (lane < n4) tma_gather4(static_cast<char*>(dst) + size_t(lane) * 4 * row_bytes, tmap, r0, r1, r2, r3, bar);
}

}  // namespace sofk

// Host: a {16 x 8 B, rows} tensor map over a record array (128-B rows).
int sof_make_row_tmap(CUtensorMap* out, const void* base, int64_t rows);
