// capi.cu — the extern "C" boundary of libsof_cuda.so (include/sof_cuda.h).
//
// Marshals host arrays to the device, validates arguments the way the reference
// does (exceptions -> status codes + sof_last_error), and sequences the stages in
// k_field.cu / k_mesh.cu / k_render.cu. No compute happens on the host.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/sof_cuda.h"
#include "sof_internal.h"

using namespace sofk;

namespace {

template <typename T>
void upload(sof_ctx* c, DBuf<T>& dst, const T* src, size_t count) {
  dst.ensure(std::max<size_t>(count, 1));
  if (count) SOF_CUDA(cudaMemcpyAsync(dst.p, src, sizeof(T) * count, cudaMemcpyHostToDevice, c->stream));
}

template <typename T>
void download(sof_ctx* c, T* dst, const T* src, size_t count) {
  if (count && dst)
    SOF_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * count, cudaMemcpyDeviceToHost, c->stream));
}

void sync(sof_ctx* c) { SOF_CUDA(cudaStreamSynchronize(c->stream)); }

void need_views(sof_ctx* c) {
  if (!c->has_scene) throw StateError("no scene: call sof_set_scene first");
  if (c->cams.empty()) throw StateError("no views: call sof_set_views first");
}

void check_points(int64_t n, const double* xyz) {
  if (n < 0) throw InvalidArg("negative point count");
  if (n > 0 && !xyz) throw InvalidArg("null point array");
  if (n >= (int64_t(1) << 31)) throw InvalidArg("more than 2^31 points per call");
}

}  // namespace

extern "C" {

int sof_version(void) { return 1; }

const char* sof_last_error(const sof_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t sof_kernel_launches(const sof_ctx* ctx) { return ctx ? ctx->launches : 0; }

int64_t sof_scene_size(const sof_ctx* ctx) { return ctx && ctx->has_scene ? ctx->n : -1; }

int sof_ctx_create(int device, sof_ctx** out) {
  if (!out) return SOF_E_INVALID;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    (void)cudaGetLastError();
    return SOF_E_CUDA;
  }
  if (device < 0 || device >= count) return SOF_E_INVALID;
  auto* c = new (std::nothrow) sof_ctx;
  if (!c) return SOF_E_OOM;
  c->device = device;
  const int st = guard(c, [&] {
    SOF_CUDA(cudaSetDevice(device));
    SOF_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    SOF_CUDA(cudaEventCreate(&c->ev0));
    SOF_CUDA(cudaEventCreate(&c->ev1));
    {
      // the prep lane (per-view records + binning for the next view) runs at the highest
      // priority: its CTAs are dispatched ahead of the evaluation's pending CTAs, so the
      // next view's lists are ready before the current evaluation drains
      int lo = 0, hi = 0;
      SOF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const int prio = std::getenv("SOF_PREP_PRIORITY_OFF") ? lo : hi;
      SOF_CUDA(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, prio));
    }
    SOF_CUDA(cudaStreamCreateWithFlags(&c->stream_copy, cudaStreamNonBlocking));
    SOF_CUDA(cudaEventCreateWithFlags(&c->tets_ev, cudaEventDisableTiming));
    SOF_CUDA(cudaEventCreateWithFlags(&c->interop_ev, cudaEventDisableTiming));
    SOF_CUDA(cudaMallocHost(&c->pinned_scalar, 8 * sizeof(uint64_t)));
    for (auto& e : c->prep_ev) SOF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : c->eval_ev) SOF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    size_t free_b = 0, total_b = 0;
    SOF_CUDA(cudaMemGetInfo(&free_b, &total_b));
    // per-view record / binding caches may take up to half of the free HBM
    c->cache_budget = free_b / 2;
  });
  if (st != SOF_OK) {
    delete c;
    return st;
  }
  *out = c;
  return SOF_OK;
}

void sof_ctx_destroy(sof_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  sofk::comm_destroy(ctx);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  for (auto e : ctx->prep_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->eval_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->evpool) cudaEventDestroy(e);
  for (auto e : ctx->user_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->stream2) {
    cudaStreamSynchronize(ctx->stream2);
    cudaStreamDestroy(ctx->stream2);
  }
  if (ctx->stream_copy) {
    cudaStreamSynchronize(ctx->stream_copy);
    cudaStreamDestroy(ctx->stream_copy);
  }
  if (ctx->tets_ev) cudaEventDestroy(ctx->tets_ev);
  if (ctx->interop_ev) cudaEventDestroy(ctx->interop_ev);
  if (ctx->pinned_scalar) cudaFreeHost(ctx->pinned_scalar);
  cudaStream_t s = ctx->stream;
  delete ctx;
  if (s) cudaStreamDestroy(s);
}

int sof_set_scene(sof_ctx* c, int64_t n, const double* pos, const double* scale,
                  const double* rot, const double* opacity, const double* dc,
                  double filter_scale) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (n < 0 || (n > 0 && (!pos || !scale || !rot || !opacity)))
      throw InvalidArg("invalid scene arrays");
    c->n = n;
    c->filter_scale = filter_scale;
    upload(c, c->pos, pos, 3 * n);
    upload(c, c->scale, scale, 3 * n);
    upload(c, c->rot, rot, 4 * n);
    upload(c, c->opa, opacity, n);
    if (dc) upload(c, c->dc, dc, 3 * n);
    else {
      c->dc.ensure(std::max<int64_t>(3 * n, 1));
      zero_async(c, c->dc.p, int64_t(sizeof(double)) * 3 * n);
    }
    // precompute() rejects non-finite parameters (precompute.hpp:60-63); checked on the
    // device, read back with the upload's synchronisation. A rejected scene leaves none.
    c->d_scalar.ensure(4);
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(c->d_scalar.p);
    zero_async(c, bad, sizeof(unsigned long long));
    scene_check_finite(c, bad);
    scene_prep(c);
    invalidate_view_caches(c);
    SOF_CUDA(cudaMemcpyAsync(c->pinned_scalar, bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (c->pinned_scalar[0] != 0) {
      c->n = 0;
      c->has_scene = false;
      throw InvalidArg("non-finite Gaussian parameters");
    }
    c->has_scene = true;
  });
}

int sof_set_views(sof_ctx* c, int v, const double* R, const double* t, const double* intr,
                  const int32_t* wh, const double* nearfar) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (v < 0 || (v > 0 && (!R || !t || !intr || !wh))) throw InvalidArg("invalid camera arrays");
    (void)nearfar;  // near/far are carried by Camera but unused on this path
    // validated into a temporary: a rejected camera leaves the previous set (and its
    // cached per-view records / bindings) untouched
    std::vector<Cam> cams(v);
    for (int k = 0; k < v; ++k) {
      Cam& cam = cams[k];
      for (int i = 0; i < 9; ++i) cam.R[i] = R[9 * k + i];
      for (int i = 0; i < 3; ++i) cam.t[i] = t[3 * k + i];
      cam.fx = intr[4 * k];
      cam.fy = intr[4 * k + 1];
      cam.cx = intr[4 * k + 2];
      cam.cy = intr[4 * k + 3];
      cam.w = wh[2 * k];
      cam.h = wh[2 * k + 1];
      if (cam.w <= 0 || cam.h <= 0) throw InvalidArg("camera resolution must be positive");
      // Camera::center() = -R^T t, evaluated as (-R^T) * t (camera.hpp:20)
      for (int i = 0; i < 3; ++i)
        cam.center[i] = (-cam.R[i]) * cam.t[0] + (-cam.R[3 + i]) * cam.t[1] + (-cam.R[6 + i]) * cam.t[2];
    }
    c->cams.swap(cams);
    invalidate_view_caches(c);
  });
}

int sof_set_tets(sof_ctx* c, int64_t nv, const double* xyz, int64_t nt, const int32_t* tets) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    check_points(nv, xyz);
    if (nt < 0 || (nt > 0 && !tets)) throw InvalidArg("invalid tet array");
    if (c->tets_pending) SOF_CUDA(cudaStreamSynchronize(c->stream_copy));
    c->tets_pending = false;
    c->up_src = nullptr;  // a not yet issued async upload is dropped
    upload(c, c->tv, xyz, 3 * nv);
    upload(c, c->tt, tets, 4 * nt);
    c->has_tets = false;
    // index range check on the device (4 * nt indices would cost seconds on the host)
    if (sof_validate_tets_dev(c, nt, c->tt.p, nv) != SOF_OK)
      throw InvalidArg("tet vertex index out of range");
    c->nv = nv;
    c->nt = nt;
    c->has_tets = true;
    sync(c);
  });
}

int sof_set_cache_budget(sof_ctx* c, int64_t bytes) {
  if (!c || bytes < 0) return SOF_E_INVALID;
  return guard(c, [&] {
    c->cache_budget = size_t(bytes);
    invalidate_view_caches(c);
  });
}

int sof_set_tets_async(sof_ctx* c, int64_t nv, const double* xyz, int64_t nt, const int32_t* tets) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    check_points(nv, xyz);
    if (nt < 0 || (nt > 0 && !tets)) throw InvalidArg("invalid tet array");
    if (nv > INT32_MAX) throw InvalidArg("too many vertices for int32 tet indices");
    if (c->tets_pending) SOF_CUDA(cudaStreamSynchronize(c->stream_copy));
    upload(c, c->tv, xyz, 3 * nv);
    // the tets travel on the copy stream while the label pass (which needs only the
    // vertices) runs; march waits for them (tets_ready)
    SOF_CUDA(cudaStreamSynchronize(c->stream));  // c->tt may still be read by earlier work
    c->tt.ensure(std::max<int64_t>(4 * nt, 1));
    c->tets_bad.ensure(1);
    SOF_CUDA(cudaMemsetAsync(c->tets_bad.p, 0, sizeof(int32_t), c->stream_copy));
    c->up_src = reinterpret_cast<const char*>(tets);
    c->up_bytes = int64_t(sizeof(int32_t)) * 4 * nt;
    c->up_done = 0;
    c->up_nv = nv;
    c->tets_pending = true;
    c->nt = nt;
    pump_upload(c, kUploadChunk);  // the rest is fed by the label pass / tets_ready
    c->nv = nv;
    c->has_tets = true;
  });
}

int sof_precompute_view(sof_ctx* c, int view, double* out13) {
  if (!c || !out13) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    const Rec* rec = view_records(c, view);
    std::vector<Rec> hr(c->n);
    std::vector<GaussStatic> hg(c->n);
    download(c, hr.data(), rec, c->n);
    download(c, hg.data(), c->gstat.p, c->n);
    sync(c);
    for (int64_t i = 0; i < c->n; ++i) {
      double* o = out13 + 13 * i;
      for (int k = 0; k < 6; ++k) o[k] = hr[i].ic[k];
      for (int k = 0; k < 3; ++k) o[6 + k] = hr[i].b[k];
      o[9] = hr[i].c;
      o[10] = hg[i].E;
      o[11] = hr[i].zmin;
      o[12] = hr[i].op;
    }
  });
}

int sof_tile_binding(sof_ctx* c, int view, int tile_size, int64_t* n_tiles, int64_t* n_entries) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
    if (tile_size <= 0) throw InvalidArg("tile_size must be positive");
    const Binding& b = view_binding(c, view, tile_size);
    c->bind_tiles = int64_t(b.tiles_x) * b.tiles_y;
    c->bind_entries = b.entries;
    c->last_binding_view = view;
    // keep a copy for sof_copy_result (the binding may live in the scratch slot)
    c->goff.ensure(c->bind_tiles + 1);
    SOF_CUDA(cudaMemcpyAsync(c->goff.p, b.off.p, sizeof(int64_t) * (c->bind_tiles + 1),
                             cudaMemcpyDeviceToDevice, c->stream));
    c->eval_in.ensure(std::max<int64_t>(b.entries, 1));
    if (b.entries)
      SOF_CUDA(cudaMemcpyAsync(c->eval_in.p, b.ent.p, sizeof(int32_t) * b.entries,
                               cudaMemcpyDeviceToDevice, c->stream));
    sync(c);
    if (n_tiles) *n_tiles = c->bind_tiles;
    if (n_entries) *n_entries = c->bind_entries;
  });
}

int sof_live_binding_stats(sof_ctx* c, int view, int tile_size, int64_t* stats) {
  if (!c || !stats) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
    if (tile_size <= 0) throw InvalidArg("tile_size must be positive");
    const Binding& b = view_binding(c, view, tile_size, true);
    stats[0] = b.entries;
    stats[1] = b.nb;
    stats[2] = b.nx;
    sync(c);
  });
}

int sof_schedule_points(sof_ctx* c, int view, int64_t n, const double* xyz, int tile_size,
                        int64_t* n_sched, int64_t* n_blocks, int32_t* tile_assignment,
                        int32_t* order, int32_t* key_tile, double* key_depth,
                        int32_t* block_ranges, int32_t* block_to_tile) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (c->cams.empty()) throw StateError("no views: call sof_set_views first");
    check_points(n, xyz);
    if (tile_size <= 0) throw InvalidArg("tile_size must be positive");
    upload(c, c->pts, xyz, 3 * n);
    std::vector<int32_t> ta(n), ord, kt, br, bt;
    std::vector<double> kd;
    schedule_points_exact(c, view, n, c->pts.p, tile_size, ta.data(), ord, kt, kd, br, bt);
    if (n_sched) *n_sched = int64_t(ord.size());
    if (n_blocks) *n_blocks = int64_t(bt.size());
    if (tile_assignment) std::copy(ta.begin(), ta.end(), tile_assignment);
    if (order) std::copy(ord.begin(), ord.end(), order);
    if (key_tile) std::copy(kt.begin(), kt.end(), key_tile);
    if (key_depth) std::copy(kd.begin(), kd.end(), key_depth);
    if (block_ranges) std::copy(br.begin(), br.end(), block_ranges);
    if (block_to_tile) std::copy(bt.begin(), bt.end(), block_to_tile);
  });
}

int sof_view_opacity(sof_ctx* c, int view, int64_t n, const double* xyz, int strategies,
                     int tile_size, int classify_mode, double* o, uint8_t* observed,
                     uint8_t* complete, uint64_t* counters) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    check_points(n, xyz);
    if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
    upload(c, c->pts, xyz, 3 * n);
    c->o_view.ensure(std::max<int64_t>(n, 1));
    c->observed.ensure(std::max<int64_t>(n, 1));
    c->complete.ensure(std::max<int64_t>(n, 1));
    eval_views(c, view, view + 1, n, c->pts.p, strategies, tile_size, classify_mode != 0,
               kModeView, nullptr, nullptr, c->o_view.p, c->observed.p, c->complete.p, counters);
    download(c, o, c->o_view.p, n);
    download(c, observed, c->observed.p, n);
    download(c, complete, c->complete.p, n);
    sync(c);
  });
}

int sof_classify_points(sof_ctx* c, int64_t n, const double* xyz, int strategies, int tile_size,
                        uint8_t* interior, uint64_t* counters) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    check_points(n, xyz);
    upload(c, c->pts, xyz, 3 * n);
    c->ext.ensure(std::max<int64_t>(n, 1));
    zero_async(c, c->ext.p, n);
    eval_views(c, 0, int(c->cams.size()), n, c->pts.p, strategies, tile_size, true, kModeClassify,
               nullptr, c->ext.p, nullptr, nullptr, nullptr, counters);
    std::vector<uint8_t> ext(n);
    download(c, ext.data(), c->ext.p, n);
    sync(c);
    for (int64_t i = 0; i < n; ++i) interior[i] = !ext[i];
  });
}

int sof_value_at(sof_ctx* c, int64_t n, const double* xyz, int strategies, int tile_size,
                 double* out, uint64_t* counters) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    check_points(n, xyz);
    upload(c, c->pts, xyz, 3 * n);
    c->min_op.ensure(std::max<int64_t>(n, 1));
    fill_f64(c, c->min_op.p, n, 1.0);

    eval_views(c, 0, int(c->cams.size()), n, c->pts.p, strategies, tile_size, false, kModeValue,
               c->min_op.p, nullptr, nullptr, nullptr, nullptr, counters);
    download(c, out, c->min_op.p, n);
    sync(c);
  });
}

int sof_label_grid(sof_ctx* c, int64_t nv, const double* xyz, int strategies, int tile_size,
                   int classify_mode, double* opacity, uint64_t* counters) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    check_points(nv, xyz);
    upload(c, c->pts, xyz, 3 * nv);
    c->min_op.ensure(std::max<int64_t>(nv, 1));
    c->ext.ensure(std::max<int64_t>(nv, 1));
    c->grid_opacity.ensure(std::max<int64_t>(nv, 1));
    fill_f64(c, c->min_op.p, nv, 1.0);

    zero_async(c, c->ext.p, nv);
    eval_views(c, 0, int(c->cams.size()), nv, c->pts.p, strategies, tile_size, classify_mode != 0,
               kModeLabel, c->min_op.p, c->ext.p, nullptr, nullptr, nullptr, counters);
    finalize_label(c, nv, c->min_op.p, c->ext.p, c->grid_opacity.p);
    c->grid_n = nv;
    download(c, opacity, c->grid_opacity.p, nv);
    sync(c);
  });
}

int sof_label_views_dev(sof_ctx* c, int v0, int v1, int64_t n, const double* xyz_dev,
                        int strategies, int tile_size, int classify_mode,
                        double* min_opacity_dev, uint8_t* exterior_dev, uint64_t* counters) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    check_points(n, xyz_dev);
    eval_views(c, v0, v1, n, xyz_dev, strategies, tile_size, classify_mode != 0, kModeLabel,
               min_opacity_dev, exterior_dev, nullptr, nullptr, nullptr, counters);
    sync(c);
  });
}

int sof_classify_views_dev(sof_ctx* c, int v0, int v1, int64_t n, const double* xyz_dev,
                           int strategies, int tile_size, uint8_t* exterior_dev,
                           uint64_t* counters) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    check_points(n, xyz_dev);
    eval_views(c, v0, v1, n, xyz_dev, strategies, tile_size, true, kModeClassify, nullptr,
               exterior_dev, nullptr, nullptr, nullptr, counters);
    sync(c);
  });
}

int sof_marching_tets(sof_ctx* c, const double* opacity, int64_t* n_edges, int64_t* n_tris) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (!c->has_tets) throw StateError("no tets: call sof_set_tets first");
    const double* opa_dev = nullptr;
    if (opacity) {
      upload(c, c->grid_opacity, opacity, c->nv);
      c->grid_n = c->nv;
      opa_dev = c->grid_opacity.p;
    } else {
      if (c->grid_n != c->nv) throw StateError("no label result for the resident tets");
      opa_dev = c->grid_opacity.p;
    }
    march(c, opa_dev);
    sync(c);
    if (n_edges) *n_edges = c->n_edges;
    if (n_tris) *n_tris = c->n_march_tris;
  });
}

int sof_refine(sof_ctx* c, int64_t ne, const int32_t* edges, double* verts, int iterations,
               int strategies, int tile_size, uint64_t* counters) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    need_views(c);
    if (!c->has_tets) throw StateError("no tets: call sof_set_tets first");
    if (ne < 0 || (ne > 0 && (!edges || !verts))) throw InvalidArg("invalid edge arrays");
    for (int64_t i = 0; i < 2 * ne; ++i)
      if (edges[i] < 0 || edges[i] >= c->nv) throw InvalidArg("edge vertex index out of range");
    DBuf<int32_t> de;
    DBuf<double> dv;
    upload(c, de, edges, 2 * ne);
    upload(c, dv, verts, 3 * ne);
    refine(c, ne, de.p, dv.p, iterations, strategies, tile_size, 0, int(c->cams.size()), counters);
    download(c, verts, dv.p, 3 * ne);
    sync(c);
  });
}

int sof_assemble(sof_ctx* c, int64_t nverts, const double* verts, int64_t ntris,
                 const int32_t* tris, double weld_eps, double min_area, int64_t* out_verts,
                 int64_t* out_tris) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (nverts < 0 || ntris < 0 || (nverts && !verts) || (ntris && !tris))
      throw InvalidArg("invalid mesh arrays");
    for (int64_t i = 0; i < 3 * ntris; ++i)
      if (tris[i] < 0 || tris[i] >= nverts) throw InvalidArg("triangle index out of range");
    if (!(weld_eps > 0.0)) throw InvalidArg("weld_eps must be positive");
    DBuf<double> dv;
    DBuf<int32_t> dt;
    upload(c, dv, verts, 3 * nverts);
    upload(c, dt, tris, 3 * ntris);
    assemble(c, nverts, dv.p, ntris, dt.p, weld_eps, min_area);
    sync(c);
    if (out_verts) *out_verts = c->mesh_nv;
    if (out_tris) *out_tris = c->mesh_nt;
  });
}

int sof_assemble_residuals(sof_ctx* c, int64_t nverts, const double* verts, const double* residuals,
                           int64_t ntris, const int32_t* tris, double weld_eps, double min_area, int64_t* out_verts,
                           int64_t* out_tris) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (nverts < 0 || ntris < 0 || (nverts && !verts) || (ntris && !tris))
      throw InvalidArg("invalid mesh arrays");
    for (int64_t i = 0; i < 3 * ntris; ++i)
      if (tris[i] < 0 || tris[i] >= nverts) throw InvalidArg("triangle index out of range");
    if (!(weld_eps > 0.0)) throw InvalidArg("weld_eps must be positive");
    DBuf<double> dv, dr;
    DBuf<int32_t> dt;
    upload(c, dv, verts, 3 * nverts);
    upload(c, dt, tris, 3 * ntris);
    if (residuals) upload(c, dr, residuals, nverts);
    assemble(c, nverts, dv.p, ntris, dt.p, weld_eps, min_area, residuals ? dr.p : nullptr);
    sync(c);
    if (out_verts) *out_verts = c->mesh_nv;
    if (out_tris) *out_tris = c->mesh_nt;
  });
}

int sof_set_eval_path(sof_ctx* c, int path) {
  if (!c || path < 0 || path > 1) return SOF_E_INVALID;
  if (c->eval_path != path) {
    c->eval_path = path;
    sofk::invalidate_view_caches(c);  // the record layout per view depends on the path
  }
  return SOF_OK;
}

int sof_set_staging(sof_ctx* c, int mode) {
  if (!c || mode < 0 || mode > 1) return SOF_E_INVALID;
  c->staging = mode;
  return SOF_OK;
}

void sof_extract_opts_default(sof_extract_opts* o) {
  if (!o) return;
  o->strategies = SOF_ALL_STRATEGIES;
  o->tile_size = 16;
  o->refine_iterations = 8;
  o->weld_eps = 1e-7;
  o->min_area = 1e-14;
  o->view_begin = -1;
  o->view_end = -1;
  o->profile = 0;
  o->compute_residuals = 0;
}

int sof_extract(sof_ctx* c, const sof_extract_opts* opts, sof_extract_stats* stats) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    const bool dbg = std::getenv("SOF_DEBUG_HOST") != nullptr;
    const auto h0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
      if (dbg)
        std::fprintf(stderr, "  extract %-10s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
    };
    need_views(c);
    if (!c->has_tets) throw StateError("no tets: call sof_set_tets first");
    sof_extract_opts o;
    sof_extract_opts_default(&o);
    if (opts) o = *opts;
    int v0 = o.view_begin, v1 = o.view_end;
    if (v0 < 0 || v1 < 0) {
      v0 = 0;
      v1 = int(c->cams.size());
    }
    sof_extract_stats st;
    std::memset(&st, 0, sizeof st);
    mark_views_stale(c);  // per-view records / bindings are rebuilt inside every extract
    const int64_t launches0 = c->launches;
    c->eval_launches = 0;
    c->exact_evals = 0;
    c->contrib_evals = 0;
    c->scanned_evals = 0;
    c->host_ms[0] = c->host_ms[1] = 0.0;
    c->time_eval = stats != nullptr && o.profile != 0;
    if (c->time_eval) {
      double drop[kProfKinds];
      prof_collect(c, drop);  // reset the event pool
    }
    cudaEvent_t e[5];
    for (auto& x : e) SOF_CUDA(cudaEventCreate(&x));
    const int64_t nv = c->nv;
    c->min_op.ensure(std::max<int64_t>(nv, 1));
    c->ext.ensure(std::max<int64_t>(nv, 1));
    c->grid_opacity.ensure(std::max<int64_t>(nv, 1));
    SOF_CUDA(cudaEventRecord(e[0], c->stream));
    mark("start");
    uint64_t cl[2] = {0, 0}, cr[2] = {0, 0};
    if (c->comm) {
      // multi-GPU: this rank's share of the views and tets, collectives on the stream
      extract_sharded(c, o, v0, v1, cl, cr, e);
      mark("sharded");
    } else {
      // label_grid (extract.hpp:59-61): classification mode, views in order
      fill_f64(c, c->min_op.p, nv, 1.0);
      zero_async(c, c->ext.p, nv);
      eval_views(c, v0, v1, nv, c->tv.p, o.strategies, o.tile_size, true, kModeLabel, c->min_op.p,
                 c->ext.p, nullptr, nullptr, nullptr, cl);
      finalize_label(c, nv, c->min_op.p, c->ext.p, c->grid_opacity.p);
      c->grid_n = nv;
      SOF_CUDA(cudaEventRecord(e[1], c->stream));
      mark("label");
      march(c, c->grid_opacity.p);
      SOF_CUDA(cudaEventRecord(e[2], c->stream));
      mark("march");
      refine(c, c->n_edges, c->r_edges.p, c->r_everts.p, o.refine_iterations, o.strategies,
             o.tile_size, v0, v1, cr);
      SOF_CUDA(cudaEventRecord(e[3], c->stream));
      mark("refine");
      const double* res = o.compute_residuals ? level_set_residuals(c, o, v0, v1) : nullptr;
      assemble(c, c->n_edges, c->r_everts.p, c->n_march_tris, c->r_tris.p, o.weld_eps, o.min_area, res);
    }
    SOF_CUDA(cudaEventRecord(e[4], c->stream));
    SOF_CUDA(cudaEventSynchronize(e[4]));
    mark("weld");
    float ms[4];
    for (int k = 0; k < 4; ++k) SOF_CUDA(cudaEventElapsedTime(&ms[k], e[k], e[k + 1]));
    for (auto& x : e) cudaEventDestroy(x);
    c->time_eval = false;
    st.crossing_edges = c->n_edges;
    st.march_triangles = c->n_march_tris;
    st.mesh_vertices = c->mesh_nv;
    st.mesh_triangles = c->mesh_nt;
    st.label_pairs = cl[0];
    st.refine_pairs = cr[0];
    st.pairs = cl[0] + cr[0];
    st.point_view_evals = cl[1] + cr[1];
    st.ms_label = ms[0];
    st.ms_march = ms[1];
    st.ms_refine = ms[2];
    st.ms_weld = ms[3];
    double pms[kProfKinds] = {0.0};
    if (o.profile) prof_collect(c, pms);
    st.ms_eval_kernel = pms[kProfEval];
    st.ms_prep = pms[kProfPrep];
    st.exact_pairs = c->exact_evals;
    st.contrib_pairs = c->contrib_evals;
    st.scanned_pairs = c->scanned_evals;
    st.host_ms_prep = c->host_ms[0];
    st.host_ms_sched = c->host_ms[1];
    st.ms_sched = pms[kProfSched];
    st.eval_launches = c->eval_launches;
    st.kernel_launches = c->launches - launches0;
    if (stats) *stats = st;
  });
}

int sof_seed_points(sof_ctx* c, int variant, int cutoff, double filter_scale, int64_t* n_out) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (!c->has_scene) throw StateError("no scene: call sof_set_scene first");
    if (variant < 0 || variant > 2 || cutoff < 0 || cutoff > 1) throw InvalidArg("invalid seed options");
    seed_points(c, variant, cutoff, filter_scale);
    sync(c);
    if (n_out) *n_out = c->n_seeds;
  });
}

int64_t sof_result_count(const sof_ctx* c, int kind) {
  if (!c) return -1;
  switch (kind) {
    case SOF_R_EDGES: return c->n_edges < 0 ? -1 : 2 * c->n_edges;
    case SOF_R_EDGE_VERTS: return c->n_edges < 0 ? -1 : 3 * c->n_edges;
    case SOF_R_TRIANGLES: return c->n_march_tris < 0 ? -1 : 3 * c->n_march_tris;
    case SOF_R_MESH_VERTS: return c->mesh_nv < 0 ? -1 : 3 * c->mesh_nv;
    case SOF_R_MESH_TRIS: return c->mesh_nt < 0 ? -1 : 3 * c->mesh_nt;
    case SOF_R_GRID_OPACITY: return c->grid_n;
    case SOF_R_TILE_OFFSETS: return c->bind_tiles < 0 ? -1 : c->bind_tiles + 1;
    case SOF_R_TILE_ENTRIES: return c->bind_entries;
    case SOF_R_SEEDS: return c->n_seeds < 0 ? -1 : 3 * c->n_seeds;
    case SOF_R_SEED_PROVENANCE: return c->n_seeds;
    case SOF_R_MESH_RESIDUALS: return c->mesh_nres;
    case SOF_R_TETS: return int64_t(c->delaunay_tets.size());
    case SOF_R_CONTRIB_INDEX: return c->n_contrib;
    case SOF_R_CONTRIB_VALUES: return c->n_contrib < 0 ? -1 : 6 * c->n_contrib;
    default: return -1;
  }
}

int sof_copy_result(sof_ctx* c, int kind, void* dst) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    const int64_t cnt = sof_result_count(c, kind);
    if (cnt < 0) throw StateError("no result of that kind");
    if (cnt == 0) return;
    if (!dst) throw InvalidArg("null destination");
    switch (kind) {
      case SOF_R_EDGES: download(c, (int32_t*)dst, c->r_edges.p, cnt); break;
      case SOF_R_EDGE_VERTS: download(c, (double*)dst, c->r_everts.p, cnt); break;
      case SOF_R_TRIANGLES: download(c, (int32_t*)dst, c->r_tris.p, cnt); break;
      case SOF_R_MESH_VERTS: download(c, (double*)dst, c->m_verts.p, cnt); break;
      case SOF_R_MESH_TRIS: download(c, (int32_t*)dst, c->m_tris.p, cnt); break;
      case SOF_R_GRID_OPACITY: download(c, (double*)dst, c->grid_opacity.p, cnt); break;
      case SOF_R_TILE_OFFSETS: download(c, (int64_t*)dst, c->goff.p, cnt); break;
      case SOF_R_TILE_ENTRIES: download(c, (int32_t*)dst, c->eval_in.p, cnt); break;
      case SOF_R_SEEDS: download(c, (double*)dst, c->seeds.p, cnt); break;
      case SOF_R_SEED_PROVENANCE: download(c, (uint8_t*)dst, c->seed_prov.p, cnt); break;
      case SOF_R_MESH_RESIDUALS: download(c, (double*)dst, c->m_res.p, cnt); break;
      case SOF_R_TETS: std::memcpy(dst, c->delaunay_tets.data(), sizeof(int32_t) * cnt); break;
      case SOF_R_CONTRIB_INDEX: download(c, (int32_t*)dst, c->ct_idx.p, cnt); break;
      case SOF_R_CONTRIB_VALUES: download(c, (double*)dst, c->ct_val.p, cnt); break;
    }
    sync(c);
  });
}

}  // extern "C"
