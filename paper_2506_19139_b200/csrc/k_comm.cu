// k_comm.cu — the library-owned multi-GPU meshing step.
//
// One process per GPU; each process's sof_ctx owns a communicator (sof_comm_init) and
// sof_extract then runs the view-sharded / tet-sharded protocol entirely on the
// library stream — no host round trip per collective, no caller-side plumbing:
//
//   label   views split into contiguous ranges; each rank labels its range with local
//           pruning; r* = allreduce MIN of (exterior_r ? r : R) is the first exterior
//           rank; ranks after r* mask their minima to +inf (the sequential reference never
//           evaluates those views, field_eval.hpp:147); allreduce MIN of the minima is the
//           sequential min. Without pruning: MIN of the minima, MAX of the flags.
//   march   tets split into contiguous ranges (marching_tets.hpp:29-84 per range); edge and
//           triangle lists all-gathered in rank order and merged into the whole-grid
//           first-appearance numbering (march_merge, k_mesh.cu).
//   refine  per iteration: every rank classifies all midpoints against its views;
//           allreduce MAX of the exterior flags; identical bracket updates everywhere
//           (marching_tets.hpp:94-114).
//   weld    replicated (assemble_mesh, mesh.hpp:36-79).
//
// Every merge is exact, so the mesh equals the single-GPU (and the reference's) mesh bit
// for bit. Collectives: NCCL over NVLink (the library resolves libnccl.so.2 at run time:
// the copy a host framework already loaded, else the system one). A second, in-process
// communicator (sof_comm_init_local) joins several contexts of one process — driven from
// one host thread each — through device-side reductions, so the protocol code above runs
// unchanged with 2..N ranks on one GPU in the tests; it never makes a kernel wait on
// another rank's kernel (every exchange is host-synchronised).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "../../include/sof_cuda.h"
#include "sof_internal.h"

namespace sofk {

enum CommType { kF64 = 0, kI32 = 1, kU8 = 2, kI64 = 3 };
enum CommOp { kMin = 0, kMax = 1 };

inline size_t type_size(int t) { return t == kF64 || t == kI64 ? 8 : t == kI32 ? 4 : 1; }

struct Comm {
  int rank = 0, size = 1;
  Comm() = default;
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  virtual ~Comm() = default;
  virtual const char* kind() const = 0;
  // in place, on stream st
  virtual void allreduce(void* buf, size_t count, int type, int op, cudaStream_t st) = 0;
  // recv[r * bytes, (r + 1) * bytes) = rank r's send, on stream st
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
};

// ---- NCCL ------------------------------------------------------------------------------------

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string err;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // a host framework's copy
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
             api.GetErrorString;
    if (!api.ok) api.err = "libnccl.so.2 lacks an expected symbol";
  });
  return api;
}

#define SOF_NCCL(call)                                                                          \
  do {                                                                                          \
    const ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess) throw ::sofk::NcclError(std::string("NCCL: ") + nccl().GetErrorString(r_)); \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  const char* kind() const override { return "nccl"; }
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  static ncclDataType_t dt(int t) {
    return t == kF64 ? ncclFloat64 : t == kI32 ? ncclInt32 : t == kI64 ? ncclInt64 : ncclUint8;
  }
  void allreduce(void* buf, size_t count, int type, int op, cudaStream_t st) override {
    if (count == 0) return;
    SOF_NCCL(nccl().AllReduce(buf, buf, count, dt(type), op == kMin ? ncclMin : ncclMax, comm, st));
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    if (bytes == 0) return;
    SOF_NCCL(nccl().AllGather(send, recv, bytes, ncclUint8, comm, st));
  }
};

// ---- in-process communicator (several contexts of one process, one host thread each) -----------

template <typename T>
__global__ void k_reduce_ptrs(T* const* __restrict__ bufs, int n, int64_t count, int op) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    T v = bufs[0][i];
    for (int r = 1; r < n; ++r) {
      const T u = bufs[r][i];
      v = (op == kMin) ? (u < v ? u : v) : (v < u ? u : v);
    }
    for (int r = 0; r < n; ++r) bufs[r][i] = v;
  }
}

struct LocalGroup {
  int size = 0;
  int device = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<void*> a, b;  // per-rank buffers of the current exchange
  cudaStream_t st = nullptr;
  void** dptrs = nullptr;  // device copy of a
  std::string err;
  int refs = 0;
  ~LocalGroup() {
    if (dptrs) cudaFree(dptrs);
    if (st) cudaStreamDestroy(st);
  }
};

struct LocalComm : Comm {
  std::shared_ptr<LocalGroup> g;
  const char* kind() const override { return "local"; }
  // every rank: its stream is drained, its pointers posted; the last arriving rank runs
  // the exchange on the group's stream and releases the others
  template <typename F>
  void exchange(void* a, void* b, cudaStream_t st, F&& work) {
    SOF_CUDA(cudaStreamSynchronize(st));
    std::unique_lock<std::mutex> lk(g->m);
    const uint64_t my = g->gen;
    g->a[rank] = a;
    g->b[rank] = b;
    if (++g->arrived == g->size) {
      try {
        work();
        SOF_CUDA(cudaStreamSynchronize(g->st));
      } catch (const std::exception& e) {
        g->err = e.what();
      }
      g->arrived = 0;
      ++g->gen;
      g->cv.notify_all();
    } else if (!g->cv.wait_for(lk, std::chrono::seconds(600), [&] { return g->gen != my; })) {
      throw std::runtime_error("local communicator: a rank did not reach the exchange");
    }
    if (!g->err.empty()) throw std::runtime_error("local communicator: " + g->err);
  }
  void allreduce(void* buf, size_t count, int type, int op, cudaStream_t st) override {
    exchange(buf, nullptr, st, [&] {
      SOF_CUDA(cudaMemcpyAsync(g->dptrs, g->a.data(), sizeof(void*) * g->size, cudaMemcpyHostToDevice, g->st));
      if (count == 0) return;
      const unsigned grid = unsigned(std::min<size_t>((count + 255) / 256, 4096));
      if (type == kF64)
        k_reduce_ptrs<double><<<grid, 256, 0, g->st>>>(reinterpret_cast<double* const*>(g->dptrs), g->size,
                                                      int64_t(count), op);
      else if (type == kI32)
        k_reduce_ptrs<int32_t><<<grid, 256, 0, g->st>>>(reinterpret_cast<int32_t* const*>(g->dptrs), g->size,
                                                       int64_t(count), op);
      else if (type == kI64)
        k_reduce_ptrs<int64_t><<<grid, 256, 0, g->st>>>(reinterpret_cast<int64_t* const*>(g->dptrs), g->size,
                                                       int64_t(count), op);
      else
        k_reduce_ptrs<uint8_t><<<grid, 256, 0, g->st>>>(reinterpret_cast<uint8_t* const*>(g->dptrs), g->size,
                                                       int64_t(count), op);
      SOF_CUDA(cudaGetLastError());
    });
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    exchange(const_cast<void*>(send), recv, st, [&] {
      if (bytes == 0) return;
      for (int d = 0; d < g->size; ++d)
        for (int r = 0; r < g->size; ++r)
          SOF_CUDA(cudaMemcpyAsync(static_cast<char*>(g->b[d]) + r * bytes, g->a[r], bytes,
                                   cudaMemcpyDeviceToDevice, g->st));
    });
  }
};

void comm_destroy(sof_ctx* c) {
  delete c->comm;
  c->comm = nullptr;
}

// ---- the sharded extraction ----------------------------------------------------------------------

__global__ void k_ext_rank2(int64_t n, const uint8_t* __restrict__ ext, int rank, int world, int32_t* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = ext[i] ? rank : world;
}

__global__ void k_mask_min2(int64_t n, const int32_t* __restrict__ rstar, int rank, double* m) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n && rank > rstar[i]) m[i] = INFINITY;
}

__global__ void k_finalize_sharded2(int64_t n, const double* __restrict__ m, const int32_t* __restrict__ rstar,
                                    int world, double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double v = m[i];
  out[i] = (rstar[i] < world) ? ((0.49999999 < v) ? 0.49999999 : v) : v;  // field_eval.hpp:175
}

// label -> march -> refine -> weld over this rank's views / tets (see the file comment).
void extract_sharded(sof_ctx* c, const sof_extract_opts& o, int vb, int ve, uint64_t* cl, uint64_t* cr,
                     cudaEvent_t* ev) {
  Comm& comm = *c->comm;
  const int R = comm.size, r = comm.rank;
  const int v0 = vb + int(int64_t(ve - vb) * r / R), v1 = vb + int(int64_t(ve - vb) * (r + 1) / R);
  const int64_t nv = c->nv;
  cudaStream_t st = c->stream;
  const bool prune = (o.strategies & SOF_PRUNE) != 0;
  // label
  fill_f64(c, c->min_op.p, nv, 1.0);
  zero_async(c, c->ext.p, nv);
  eval_views(c, v0, v1, nv, c->tv.p, o.strategies, o.tile_size, true, kModeLabel, c->min_op.p, c->ext.p, nullptr,
             nullptr, nullptr, cl);
  c->shard_i32.ensure(std::max<int64_t>(nv, 1));
  int32_t* rstar = c->shard_i32.p;
  const unsigned g = grid_for(std::max<int64_t>(nv, 1), 256);
  if (prune) {
    k_ext_rank2<<<g, 256, 0, st>>>(nv, c->ext.p, r, R, rstar);
    SOF_LAUNCHED(c);
    comm.allreduce(rstar, nv, kI32, kMin, st);
    k_mask_min2<<<g, 256, 0, st>>>(nv, rstar, r, c->min_op.p);
    SOF_LAUNCHED(c);
    comm.allreduce(c->min_op.p, nv, kF64, kMin, st);
  } else {
    comm.allreduce(c->min_op.p, nv, kF64, kMin, st);
    comm.allreduce(c->ext.p, nv, kU8, kMax, st);
    k_ext_rank2<<<g, 256, 0, st>>>(nv, c->ext.p, 0, R, rstar);
    SOF_LAUNCHED(c);
  }
  k_finalize_sharded2<<<g, 256, 0, st>>>(nv, c->min_op.p, rstar, R, c->grid_opacity.p);
  SOF_LAUNCHED(c);
  c->grid_n = nv;
  SOF_CUDA(cudaEventRecord(ev[1], st));
  // march over this rank's tets, gathered and merged in rank order
  tets_ready(c);
  const int64_t t0 = c->nt * r / R, t1 = c->nt * (r + 1) / R;
  march_range(c, c->grid_opacity.p, t0, t1);
  c->shard_i64.ensure(2 * (R + 1));
  int64_t* cnt_dev = c->shard_i64.p;  // [0, 2): mine, [2, 2 + 2R): everyone's
  const int64_t mine[2] = {c->n_edges, c->n_march_tris};
  SOF_CUDA(cudaMemcpyAsync(cnt_dev, mine, sizeof mine, cudaMemcpyHostToDevice, st));
  comm.allgather(cnt_dev, cnt_dev + 2, 2 * sizeof(int64_t), st);
  std::vector<int64_t> cnt(2 * R);
  SOF_CUDA(cudaMemcpyAsync(cnt.data(), cnt_dev + 2, sizeof(int64_t) * 2 * R, cudaMemcpyDeviceToHost, st));
  SOF_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> ecount(R), tcount(R);
  int64_t me = 1, mt = 1, se = 0, stt = 0;
  for (int k = 0; k < R; ++k) {
    ecount[k] = cnt[2 * k];
    tcount[k] = cnt[2 * k + 1];
    me = std::max(me, ecount[k]);
    mt = std::max(mt, tcount[k]);
    se += ecount[k];
    stt += tcount[k];
  }
  // padded per-rank blocks (collectives have no gatherv), then compacted in rank order
  DBuf<int32_t>& send = c->shard_send;
  DBuf<int32_t>& recv = c->shard_recv;
  DBuf<int32_t>& all = c->shard_all;
  const int64_t blk = 2 * me + 3 * mt;  // int32 per rank: edges then triangles
  send.ensure(blk);
  recv.ensure(blk * R);
  all.ensure(std::max<int64_t>(2 * se + 3 * stt, 1));
  if (c->n_edges > 0)
    SOF_CUDA(cudaMemcpyAsync(send.p, c->r_edges.p, sizeof(int32_t) * 2 * c->n_edges, cudaMemcpyDeviceToDevice, st));
  if (c->n_march_tris > 0)
    SOF_CUDA(cudaMemcpyAsync(send.p + 2 * me, c->r_tris.p, sizeof(int32_t) * 3 * c->n_march_tris,
                             cudaMemcpyDeviceToDevice, st));
  comm.allgather(send.p, recv.p, sizeof(int32_t) * blk, st);
  int32_t* edges_all = all.p;
  int32_t* tris_all = all.p + 2 * se;
  for (int k = 0, eo = 0, to = 0; k < R; ++k) {
    if (ecount[k] > 0)
      SOF_CUDA(cudaMemcpyAsync(edges_all + eo, recv.p + k * blk, sizeof(int32_t) * 2 * ecount[k],
                               cudaMemcpyDeviceToDevice, st));
    if (tcount[k] > 0)
      SOF_CUDA(cudaMemcpyAsync(tris_all + to, recv.p + k * blk + 2 * me, sizeof(int32_t) * 3 * tcount[k],
                               cudaMemcpyDeviceToDevice, st));
    eo += int(2 * ecount[k]);
    to += int(3 * tcount[k]);
  }
  march_merge(c, c->grid_opacity.p, R, ecount.data(), edges_all, tcount.data(), tris_all);
  SOF_CUDA(cudaEventRecord(ev[2], st));
  // refine: classify against this rank's views, MAX-merge the flags every iteration
  const int64_t ne = c->n_edges;
  if (o.refine_iterations > 0 && ne > 0) {
    refine_init(c, ne, c->r_edges.p);
    bisect_cache_views(c, v0, v1, ne, c->r_edges.p, o.strategies, o.tile_size);
    for (int it = 0; it < o.refine_iterations; ++it) {
      refine_mid(c, ne, c->ms.rext.p);
      eval_views(c, v0, v1, ne, c->ms.mid.p, o.strategies, o.tile_size, true, kModeClassify, nullptr, c->ms.rext.p,
                 nullptr, nullptr, nullptr, cr);
      comm.allreduce(c->ms.rext.p, ne, kU8, kMax, st);
      refine_update(c, ne, c->ms.rext.p);
    }
    refine_final(c, ne, c->r_everts.p);
  }
  SOF_CUDA(cudaEventRecord(ev[3], st));
  const double* res = nullptr;
  if (o.compute_residuals) {  // value_at = min over views: this rank's views, MIN-reduced
    double* val = level_set_values(c, o, v0, v1);
    comm.allreduce(val, c->n_edges, kF64, kMin, st);
    res = residuals_from_values(c, val);
  }
  assemble(c, c->n_edges, c->r_everts.p, c->n_march_tris, c->r_tris.p, o.weld_eps, o.min_area, res);
}

}  // namespace sofk

using namespace sofk;

extern "C" {

int sof_comm_unique_id(void* id_out) {
  if (!id_out) return SOF_E_INVALID;
  NcclApi& api = nccl();
  if (!api.ok) return SOF_E_NCCL;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return SOF_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == SOF_COMM_ID_BYTES, "NCCL unique id size");
  std::memcpy(id_out, &id, sizeof id);
  return SOF_OK;
}

int sof_comm_init(sof_ctx* c, const void* id, int nranks, int rank) {
  if (!c || !id || nranks < 1 || rank < 0 || rank >= nranks) return SOF_E_INVALID;
  try {
    SOF_CUDA(cudaSetDevice(c->device));
    NcclApi& api = nccl();
    if (!api.ok) {
      c->err = api.err;
      return SOF_E_NCCL;
    }
    comm_destroy(c);
    auto* nc = new NcclComm;
    nc->rank = rank;
    nc->size = nranks;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    const ncclResult_t r = api.CommInitRank(&nc->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      c->err = std::string("ncclCommInitRank: ") + api.GetErrorString(r);
      nc->comm = nullptr;
      delete nc;
      return SOF_E_NCCL;
    }
    c->comm = nc;
    return SOF_OK;
  } catch (const std::exception& e) {
    c->err = e.what();
    return SOF_E_CUDA;
  }
}

int sof_comm_init_local(sof_ctx* const* ctxs, int n) {
  if (!ctxs || n < 1) return SOF_E_INVALID;
  for (int k = 0; k < n; ++k)
    if (!ctxs[k] || ctxs[k]->device != ctxs[0]->device) return SOF_E_INVALID;
  try {
    SOF_CUDA(cudaSetDevice(ctxs[0]->device));
    auto g = std::make_shared<LocalGroup>();
    g->size = n;
    g->device = ctxs[0]->device;
    g->a.assign(n, nullptr);
    g->b.assign(n, nullptr);
    SOF_CUDA(cudaStreamCreateWithFlags(&g->st, cudaStreamNonBlocking));
    SOF_CUDA(cudaMalloc(&g->dptrs, sizeof(void*) * n));
    for (int k = 0; k < n; ++k) {
      comm_destroy(ctxs[k]);
      auto* lc = new LocalComm;
      lc->rank = k;
      lc->size = n;
      lc->g = g;
      ctxs[k]->comm = lc;
    }
    return SOF_OK;
  } catch (const std::exception& e) {
    ctxs[0]->err = e.what();
    return SOF_E_CUDA;
  }
}

int sof_comm_info(const sof_ctx* c, int* nranks, int* rank) {
  if (!c) return SOF_E_INVALID;
  if (nranks) *nranks = c->comm ? c->comm->size : 1;
  if (rank) *rank = c->comm ? c->comm->rank : 0;
  return c->comm ? (std::strcmp(c->comm->kind(), "nccl") == 0 ? 1 : 2) : 0;
}

int sof_comm_destroy(sof_ctx* c) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] { comm_destroy(c); });
}

}  // extern "C"
