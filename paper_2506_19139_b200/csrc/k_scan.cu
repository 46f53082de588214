// k_scan.cu — hand-written device-wide exclusive prefix sums (no CUB).
//
// Three passes over 2048-element blocks: per-block totals, one CTA scanning the totals,
// then each block's local scan plus its offset. The output has n + 1 entries (the last
// one is the total), which is the CSR offset layout every caller wants. Reads the input
// twice and writes the output once: HBM-bound for large n, a few microseconds of launch
// latency for small n.
#include <cuda_runtime.h>

#include "sof_internal.h"

namespace sofk {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanBlock = kScanThreads * kScanItems;  // elements per block

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, v, s);
    if (lane >= s) v += u;
  }
  return v;
}

// Exclusive scan of one value per thread across the CTA (blockDim.x == kScanThreads);
// returns the CTA total through *total.
template <typename T>
__device__ __forceinline__ T cta_excl_scan(T v, T* total) {
  __shared__ T warp_sum[kScanThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const T inc = warp_incl_scan(v);
  if (lane == 31) warp_sum[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = (lane < kScanThreads / 32) ? warp_sum[lane] : T(0);
    s = warp_incl_scan(s);
    if (lane < kScanThreads / 32) warp_sum[lane] = s;
  }
  __syncthreads();
  const T before = (w > 0) ? warp_sum[w - 1] : T(0);
  *total = warp_sum[kScanThreads / 32 - 1];
  __syncthreads();  // warp_sum is reused by the next call
  return before + inc - v;
}

template <typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads) k_scan_block_sums(int64_t n, const In* __restrict__ in,
                                                                  Out* __restrict__ bsum) {
  const int64_t b0 = int64_t(blockIdx.x) * kScanBlock;
  Out s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = b0 + k * kScanThreads + threadIdx.x;  // coalesced
    if (i < n) s += Out(in[i]);
  }
  Out total;
  (void)cta_excl_scan(s, &total);
  if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

// one CTA: exclusive scan of the block totals in place (any count)
template <typename Out>
__global__ void __launch_bounds__(kScanThreads) k_scan_totals(int64_t nb, Out* bsum) {
  Out carry = 0;
  for (int64_t base = 0; base < nb; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    const Out v = (i < nb) ? bsum[i] : Out(0);
    Out total;
    const Out ex = cta_excl_scan(v, &total);
    if (i < nb) bsum[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) bsum[nb] = carry;
}

template <typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(int64_t n, const In* __restrict__ in,
                                                             const Out* __restrict__ boff, Out* __restrict__ out,
                                                             int64_t nb) {
  // thread t scans its kScanItems consecutive elements (loaded through shared memory so
  // the global accesses stay coalesced)
  __shared__ Out tile[kScanBlock];
  const int64_t b0 = int64_t(blockIdx.x) * kScanBlock;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = b0 + k * kScanThreads + threadIdx.x;
    tile[k * kScanThreads + threadIdx.x] = (i < n) ? Out(in[i]) : Out(0);
  }
  __syncthreads();
  Out local[kScanItems];
  Out s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    local[k] = s;
    s += tile[threadIdx.x * kScanItems + k];
  }
  Out total;
  const Out ex = cta_excl_scan(s, &total) + boff[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) tile[threadIdx.x * kScanItems + k] = ex + local[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = b0 + k * kScanThreads + threadIdx.x;
    if (i < n) out[i] = tile[k * kScanThreads + threadIdx.x];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = boff[nb];
}

template <typename In, typename Out>
static void scan_impl(sof_ctx* c, const In* in, Out* out, int64_t n, cudaStream_t st) {
  if (n <= 0) {
    SOF_CUDA(cudaMemsetAsync(out, 0, sizeof(Out), st));
    return;
  }
  const int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  c->scan_tmp.ensure(size_t(nb + 1) * sizeof(Out));
  Out* bsum = reinterpret_cast<Out*>(c->scan_tmp.p);
  k_scan_block_sums<In, Out><<<unsigned(nb), kScanThreads, 0, st>>>(n, in, bsum);
  k_scan_totals<Out><<<1, kScanThreads, 0, st>>>(nb, bsum);
  k_scan_apply<In, Out><<<unsigned(nb), kScanThreads, 0, st>>>(n, in, bsum, out, nb);
  c->launches += 3;
  SOF_CUDA(cudaGetLastError());
}

void scan_u32_i64(sof_ctx* c, const uint32_t* in, int64_t* out, int64_t n) { scan_impl(c, in, out, n, c->stream); }
void scan_i32_i32(sof_ctx* c, const int32_t* in, int32_t* out, int64_t n) { scan_impl(c, in, out, n, c->stream); }
void scan_i64_i64(sof_ctx* c, const int64_t* in, int64_t* out, int64_t n) { scan_impl(c, in, out, n, c->stream); }

}  // namespace sofk
