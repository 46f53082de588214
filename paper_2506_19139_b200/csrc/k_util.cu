// k_util.cu — device-side input validation, stream-event timing, pinned host
// registration and the FP64-pipe peak probe used as the roofline denominator of
// the FP64 opacity-evaluation kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/sof_cuda.h"
#include "sof_internal.h"
#include "sof_tma.cuh"

#include <cudaTypedefs.h>

// Tensor map of a 128-B-row record array for the TMA row gather (sof_tma.cuh). The
// driver entry point is resolved once through the runtime (no -lcuda link).
int sof_make_row_tmap(CUtensorMap* out, const void* base, int64_t rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return -1;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {16, cuuint64_t(std::max<int64_t>(rows, 1))};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {16, 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -int(r);
}

namespace sofk {

// Tet index range check, one 16-B tet per load, one flag write per warp at most.
__global__ void k_check_tets(int64_t nt, const int4* __restrict__ tets, int32_t bound, int32_t* bad) {
  bool b = false;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nt; t += int64_t(gridDim.x) * blockDim.x) {
    const int4 q = tets[t];
    b |= (unsigned(q.x) >= unsigned(bound)) | (unsigned(q.y) >= unsigned(bound)) | (unsigned(q.z) >= unsigned(bound)) |
         (unsigned(q.w) >= unsigned(bound));
  }
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
}

// Each thread runs 8 independent DFMA chains; 2 FLOP per DFMA.
__global__ void k_fp64_peak(int iters, double seed, double* sink) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, b = 1e-7;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, b);
    a1 = fma(a1, m, b);
    a2 = fma(a2, m, b);
    a3 = fma(a3, m, b);
    a4 = fma(a4, m, b);
    a5 = fma(a5, m, b);
    a6 = fma(a6, m, b);
    a7 = fma(a7, m, b);
  }
  const double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (r == 12345.678) sink[0] = r;  // keep the chains live
}

__global__ void k_fill_f64(int64_t n, double* p, double v) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_zero_words(int64_t n4, uint32_t* p4, int64_t n1, uint8_t* tail) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n4) p4[i] = 0u;
  if (i < n1) tail[i] = 0;
}

// cudaMemsetAsync(p, 0, bytes) as a kernel: memsets may be executed by a copy engine
// and then queue behind a large asynchronous upload (sof_set_tets_async).
void zero_async(sof_ctx* c, void* p, int64_t bytes) {
  if (bytes <= 0) return;
  const bool aligned = (reinterpret_cast<uintptr_t>(p) & 3) == 0;
  const int64_t n4 = aligned ? bytes / 4 : 0, n1 = bytes - 4 * n4;
  uint8_t* tail = static_cast<uint8_t*>(p) + 4 * n4;
  const int64_t n = std::max(n4, n1);
  k_zero_words<<<grid_for(n, 256), 256, 0, c->stream>>>(n4, static_cast<uint32_t*>(p), n1, tail);
  SOF_LAUNCHED(c);
}

void fill_f64(sof_ctx* c, double* p, int64_t n, double v) {
  if (n <= 0) return;
  k_fill_f64<<<grid_for(n, 256), 256, 0, c->stream>>>(n, p, v);
  SOF_LAUNCHED(c);
}

int prof_mark(sof_ctx* c) {
  if (!c->time_eval) return -1;
  if (c->evnext == c->evpool.size()) {
    cudaEvent_t e;
    SOF_CUDA(cudaEventCreate(&e));
    c->evpool.push_back(e);
  }
  SOF_CUDA(cudaEventRecord(c->evpool[c->evnext], c->stream));
  return int(c->evnext++);
}

void prof_span(sof_ctx* c, int a, int b, int kind) {
  if (a < 0 || b < 0) return;
  c->span_a.push_back(a);
  c->span_b.push_back(b);
  c->span_k.push_back(kind);
}

void prof_collect(sof_ctx* c, double* ms) {
  for (int k = 0; k < kProfKinds; ++k) ms[k] = 0.0;
  if (c->evnext) SOF_CUDA(cudaEventSynchronize(c->evpool[c->evnext - 1]));
  for (size_t i = 0; i < c->span_a.size(); ++i) {
    float x = 0.f;
    SOF_CUDA(cudaEventElapsedTime(&x, c->evpool[c->span_a[i]], c->evpool[c->span_b[i]]));
    ms[c->span_k[i]] += x;
  }
  c->span_a.clear();
  c->span_b.clear();
  c->span_k.clear();
  c->evnext = 0;
}

void check_tet_indices(sof_ctx* c, cudaStream_t st, int64_t nt, const int32_t* tets_dev, int64_t nv,
                       int32_t* bad) {
  k_check_tets<<<std::min<int64_t>(grid_for(nt, 256), 148 * 16), 256, 0, st>>>(
      nt, reinterpret_cast<const int4*>(tets_dev), int32_t(nv), bad);
  SOF_LAUNCHED(c);
}

void pump_upload(sof_ctx* c, int64_t max_bytes) {
  if (!c->tets_pending || !c->up_src || c->up_done >= c->up_bytes) return;
  const int64_t n = std::min(max_bytes, c->up_bytes - c->up_done);
  SOF_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(c->tt.p) + c->up_done, c->up_src + c->up_done, size_t(n),
                           cudaMemcpyHostToDevice, c->stream_copy));
  c->up_done += n;
  if (c->up_done == c->up_bytes) {
    if (c->nt > 0) check_tet_indices(c, c->stream_copy, c->nt, c->tt.p, c->up_nv, c->tets_bad.p);
    SOF_CUDA(cudaEventRecord(c->tets_ev, c->stream_copy));
    c->up_src = nullptr;
  }
}

void tets_ready(sof_ctx* c) {
  if (!c->tets_pending) return;
  if (c->up_src) pump_upload(c, c->up_bytes - c->up_done);
  const auto t0 = std::chrono::steady_clock::now();
  const bool was_done = cudaEventQuery(c->tets_ev) == cudaSuccess;
  SOF_CUDA(cudaEventSynchronize(c->tets_ev));
  if (std::getenv("SOF_DEBUG_TETS"))
    std::fprintf(stderr, "tets_ready: copy %s, waited %.2f ms\n", was_done ? "done" : "pending",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  int32_t bad = 0;
  SOF_CUDA(cudaMemcpy(&bad, c->tets_bad.p, sizeof bad, cudaMemcpyDeviceToHost));
  c->tets_pending = false;
  if (bad) {
    c->has_tets = false;
    throw InvalidArg("tet vertex index out of range");
  }
}

}  // namespace sofk

using namespace sofk;

extern "C" {

int sof_validate_tets_dev(sof_ctx* c, int64_t nt, const int32_t* tets_dev, int64_t nv) {
  if (!c) return SOF_E_INVALID;
  if (nt > 0 && (!tets_dev || (reinterpret_cast<uintptr_t>(tets_dev) & 15))) {
    c->err = "tets_dev must be a 16-byte aligned device array of 4 * nt indices";
    return SOF_E_INVALID;
  }
  try {
    DBuf<int32_t>& bad = c->ms.nsel;
    bad.ensure(1);
    zero_async(c, bad.p, 4);
    if (nt > 0) {
      k_check_tets<<<std::min<int64_t>(grid_for(nt, 256), 148 * 16), 256, 0, c->stream>>>(
          nt, reinterpret_cast<const int4*>(tets_dev), int32_t(nv), bad.p);
      SOF_LAUNCHED(c);
    }
    return read_scalar(c, bad.p) ? SOF_E_INVALID : SOF_OK;
  } catch (const std::exception& e) {
    c->err = e.what();
    return SOF_E_CUDA;
  }
}

int sof_event_record(sof_ctx* c, int slot) {
  if (!c || slot < 0 || slot >= 8) return SOF_E_INVALID;
  if (!c->user_ev[slot] && cudaEventCreate(&c->user_ev[slot]) != cudaSuccess) return SOF_E_CUDA;
  return cudaEventRecord(c->user_ev[slot], c->stream) == cudaSuccess ? SOF_OK : SOF_E_CUDA;
}

int sof_event_elapsed(sof_ctx* c, int a, int b, float* ms) {
  if (!c || !ms || a < 0 || b < 0 || a >= 8 || b >= 8 || !c->user_ev[a] || !c->user_ev[b])
    return SOF_E_INVALID;
  if (cudaEventSynchronize(c->user_ev[b]) != cudaSuccess) return SOF_E_CUDA;
  return cudaEventElapsedTime(ms, c->user_ev[a], c->user_ev[b]) == cudaSuccess ? SOF_OK : SOF_E_CUDA;
}

int sof_stream_wait(sof_ctx* c, void* stream) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    SOF_CUDA(cudaEventRecord(c->interop_ev, static_cast<cudaStream_t>(stream)));
    SOF_CUDA(cudaStreamWaitEvent(c->stream, c->interop_ev, 0));
  });
}

int sof_get_stream(sof_ctx* c, void** stream) {
  if (!c || !stream) return SOF_E_INVALID;
  *stream = c->stream;
  return SOF_OK;
}

int sof_sync(sof_ctx* c) {
  if (!c) return SOF_E_INVALID;
  return cudaStreamSynchronize(c->stream) == cudaSuccess ? SOF_OK : SOF_E_CUDA;
}

int sof_host_register(void* ptr, size_t bytes) {
  if (!ptr || !bytes) return SOF_E_INVALID;
  return cudaHostRegister(ptr, bytes, cudaHostRegisterDefault) == cudaSuccess ? SOF_OK : SOF_E_CUDA;
}

int sof_host_unregister(void* ptr) {
  if (!ptr) return SOF_E_INVALID;
  return cudaHostUnregister(ptr) == cudaSuccess ? SOF_OK : SOF_E_CUDA;
}

int sof_fp64_peak(sof_ctx* c, double* tflops) {
  if (!c || !tflops) return SOF_E_INVALID;
  try {
    SOF_CUDA(cudaSetDevice(c->device));
    int sms = 0;
    SOF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    DBuf<double> sink;
    sink.ensure(1);
    const int iters = 1 << 14, threads = 256, blocks = sms * 8;
    cudaEvent_t a, b;
    SOF_CUDA(cudaEventCreate(&a));
    SOF_CUDA(cudaEventCreate(&b));
    k_fp64_peak<<<blocks, threads, 0, c->stream>>>(iters, 1.0, sink.p);  // warm-up
    SOF_LAUNCHED(c);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      SOF_CUDA(cudaEventRecord(a, c->stream));
      k_fp64_peak<<<blocks, threads, 0, c->stream>>>(iters, 1.0 + r, sink.p);
      SOF_LAUNCHED(c);
      SOF_CUDA(cudaEventRecord(b, c->stream));
      SOF_CUDA(cudaEventSynchronize(b));
      float ms = 0.f;
      SOF_CUDA(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8.0 * double(iters) * threads * double(blocks);
    *tflops = flops / (best * 1e-3) / 1e12;
    return SOF_OK;
  } catch (const std::exception& e) {
    c->err = e.what();
    return SOF_E_CUDA;
  }
}

}  // extern "C"
