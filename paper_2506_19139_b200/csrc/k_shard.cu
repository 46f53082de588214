// k_shard.cu — device primitives of the view-sharded meshing step (one process per
// GPU, views split into contiguous ranges, collectives by the caller over NCCL).
//
// The label pass must reproduce the SEQUENTIAL reference (field_eval.hpp:145-176)
// exactly even though each rank only sees its own views. With pruning, a vertex's
// final value is the min over the views up to (and including) the first view in
// which it becomes exterior; views after that are skipped. Rank r runs its range
// with local pruning and reports (exterior_r, min_r). The first exterior rank r* is
// an all-reduce MIN of (exterior_r ? r : R); ranks after r* drop out (+inf) and an
// all-reduce MIN of the masked minima gives exactly the sequential min. The bisection
// is classification-only: an all-reduce MAX of the exterior flags per iteration.
#include <cuda_runtime.h>

#include "../../include/sof_cuda.h"
#include "sof_internal.h"

namespace sofk {

__global__ void k_ext_rank(int64_t n, const uint8_t* __restrict__ ext, int rank, int world,
                           int32_t* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = ext[i] ? rank : world;
}

__global__ void k_mask_min(int64_t n, const int32_t* __restrict__ rstar, int rank, double* m) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n && rank > rstar[i]) m[i] = INFINITY;
}

__global__ void k_finalize_sharded(int64_t n, const double* __restrict__ m,
                                   const int32_t* __restrict__ rstar, int world, double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double v = m[i];
  out[i] = (rstar[i] < world) ? ((0.49999999 < v) ? 0.49999999 : v) : v;  // field_eval.hpp:175
}

template <typename F>
int guarded(sof_ctx* c, F&& f) {
  if (!c) return SOF_E_INVALID;
  try {
    SOF_CUDA(cudaSetDevice(c->device));
    f();
    SOF_CUDA(cudaStreamSynchronize(c->stream));
    return SOF_OK;
  } catch (const InvalidArg& e) {
    c->err = e.what();
    return SOF_E_INVALID;
  } catch (const StateError& e) {
    c->err = e.what();
    return SOF_E_STATE;
  } catch (const OomError& e) {
    c->err = e.what();
    return SOF_E_OOM;
  } catch (const std::exception& e) {
    c->err = e.what();
    return SOF_E_CUDA;
  }
}

}  // namespace sofk

using namespace sofk;

extern "C" {

int sof_tets_vertices_dev(sof_ctx* c, const double** xyz_dev, int64_t* nv) {
  if (!c || !xyz_dev) return SOF_E_INVALID;
  if (!c->has_tets) return SOF_E_STATE;
  *xyz_dev = c->tv.p;
  if (nv) *nv = c->nv;
  return SOF_OK;
}

int sof_shard_ext_rank_dev(sof_ctx* c, int64_t n, const uint8_t* ext_dev, int rank, int world,
                           int32_t* out_dev) {
  return guarded(c, [&] {
    if (n <= 0) return;
    k_ext_rank<<<grid_for(n, 256), 256, 0, c->stream>>>(n, ext_dev, rank, world, out_dev);
    SOF_LAUNCHED(c);
  });
}

int sof_shard_mask_min_dev(sof_ctx* c, int64_t n, const int32_t* rstar_dev, int rank,
                           double* min_dev) {
  return guarded(c, [&] {
    if (n <= 0) return;
    k_mask_min<<<grid_for(n, 256), 256, 0, c->stream>>>(n, rstar_dev, rank, min_dev);
    SOF_LAUNCHED(c);
  });
}

int sof_shard_finalize_dev(sof_ctx* c, int64_t n, const double* min_dev, const int32_t* rstar_dev,
                           int world) {
  return guarded(c, [&] {
    if (!c->has_tets || n != c->nv) throw InvalidArg("finalize needs one value per resident vertex");
    c->grid_opacity.ensure(std::max<int64_t>(n, 1));
    if (n > 0) {
      k_finalize_sharded<<<grid_for(n, 256), 256, 0, c->stream>>>(n, min_dev, rstar_dev, world,
                                                                   c->grid_opacity.p);
      SOF_LAUNCHED(c);
    }
    c->grid_n = n;
  });
}

int sof_march_resident(sof_ctx* c, int64_t* n_edges, int64_t* n_tris) {
  return guarded(c, [&] {
    if (!c->has_tets || c->grid_n != c->nv) throw StateError("no label result for the resident tets");
    march(c, c->grid_opacity.p);
    if (n_edges) *n_edges = c->n_edges;
    if (n_tris) *n_tris = c->n_march_tris;
  });
}

int sof_march_range_resident(sof_ctx* c, int64_t t0, int64_t t1, int64_t* n_edges, int64_t* n_tris) {
  return guarded(c, [&] {
    if (!c->has_tets || c->grid_n != c->nv) throw StateError("no label result for the resident tets");
    march_range(c, c->grid_opacity.p, t0, t1);
    if (n_edges) *n_edges = c->n_edges;
    if (n_tris) *n_tris = c->n_march_tris;
  });
}

int sof_march_result_copy_dev(sof_ctx* c, int32_t* edges_dst, int32_t* tris_dst) {
  return guarded(c, [&] {
    if (c->n_edges < 0) throw StateError("no marching result");
    if (edges_dst && c->n_edges > 0)
      SOF_CUDA(cudaMemcpyAsync(edges_dst, c->r_edges.p, sizeof(int32_t) * 2 * c->n_edges, cudaMemcpyDeviceToDevice,
                               c->stream));
    if (tris_dst && c->n_march_tris > 0)
      SOF_CUDA(cudaMemcpyAsync(tris_dst, c->r_tris.p, sizeof(int32_t) * 3 * c->n_march_tris,
                               cudaMemcpyDeviceToDevice, c->stream));
    SOF_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int sof_march_merge_dev(sof_ctx* c, int world, const int64_t* edge_counts, const int32_t* edges_dev,
                        const int64_t* tri_counts, const int32_t* tris_dev, int64_t* n_edges, int64_t* n_tris) {
  return guarded(c, [&] {
    if (!edge_counts || !tri_counts) throw InvalidArg("null shard counts");
    if (!c->has_tets || c->grid_n != c->nv) throw StateError("no label result for the resident tets");
    march_merge(c, c->grid_opacity.p, world, edge_counts, edges_dev, tri_counts, tris_dev);
    if (n_edges) *n_edges = c->n_edges;
    if (n_tris) *n_tris = c->n_march_tris;
  });
}

int sof_refine_phase_dev(sof_ctx* c, int phase, uint8_t* ext_dev, int v0, int v1, int strategies,
                         int tile_size, uint64_t* counters) {
  return guarded(c, [&] {
    if (c->n_edges < 0) throw StateError("no marching result");
    const int64_t ne = c->n_edges;
    switch (phase) {
      case 0:
        refine_init(c, ne, c->r_edges.p);
        bisect_cache_views(c, v0, v1, ne, c->r_edges.p, strategies, tile_size);
        break;
      case 1:
        refine_mid(c, ne, ext_dev);
        if (ne > 0)
          eval_views(c, v0, v1, ne, c->ms.mid.p, strategies, tile_size, true, kModeClassify,
                     nullptr, ext_dev, nullptr, nullptr, nullptr, counters);
        break;
      case 2: refine_update(c, ne, ext_dev); break;
      case 3: refine_final(c, ne, c->r_everts.p); break;
      default: throw InvalidArg("refine phase must be 0..3");
    }
  });
}

int sof_assemble_resident(sof_ctx* c, double weld_eps, double min_area, int64_t* nv, int64_t* nt) {
  return guarded(c, [&] {
    if (c->n_edges < 0) throw StateError("no marching result");
    assemble(c, c->n_edges, c->r_everts.p, c->n_march_tris, c->r_tris.p, weld_eps, min_area);
    if (nv) *nv = c->mesh_nv;
    if (nt) *nt = c->mesh_nt;
  });
}

}  // extern "C"
