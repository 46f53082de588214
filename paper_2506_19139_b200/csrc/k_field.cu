// k_field.cu — per-view preprocessing (K0/K1), Gaussian tile binning (K2), point
// scheduling (K3) and the opacity-field evaluation kernel (K4), FP64 parity path.
//
// Reference path replaced: ViewSet::build / precompute (opacity_field.hpp:26-34,
// precompute.hpp:57-87), build_tile_binding (tiles.hpp:94-146), schedule_points
// (tiles.hpp:29-84) and FieldEvaluator::view_opacity / classify_point / value_at /
// label_grid (field_eval.hpp:59-176). Compiled with --fmad=false: every FP64
// expression is the reference's, so values and decisions are bit-identical.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sof_internal.h"
#include "sof_tma.cuh"

namespace sofk {

// threads (= points) per evaluation CTA; the schedule cuts tiles into blocks of this size
#ifndef SOF_EVAL_THREADS
#define SOF_EVAL_THREADS 128
#endif
constexpr int kEvalThreads = SOF_EVAL_THREADS;

// ---- helpers ------------------------------------------------------------------------------

int bits_for(uint64_t max_value) {
  int b = 1;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b;
}

void sort_pairs_u64(sof_ctx* c, const uint64_t* kin, uint64_t* kout, const int32_t* vin,
                    int32_t* vout, int64_t n, int end_bit) {
  if (n <= 0) return;
  size_t bytes = 0;
  SOF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0, end_bit,
                                           c->stream));
  c->cub_tmp.ensure(bytes);
  SOF_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, bytes, kin, kout, vin, vout, n, 0,
                                           end_bit, c->stream));
  c->launches += 2 + (end_bit + 7) / 8;
}

void sort_pairs_u32(sof_ctx* c, const uint32_t* kin, uint32_t* kout, const int32_t* vin,
                    int32_t* vout, int64_t n, int end_bit) {
  if (n <= 0) return;
  size_t bytes = 0;
  SOF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0, end_bit,
                                           c->stream));
  c->cub_tmp.ensure(bytes);
  SOF_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, bytes, kin, kout, vin, vout, n, 0,
                                           end_bit, c->stream));
  c->launches += 2 + (end_bit + 7) / 8;
}

void exclusive_scan_u32_to_i64(sof_ctx* c, const uint32_t* in, int64_t* out, int64_t n) {
  if (n <= 0) return;
  size_t bytes = 0;
  SOF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, c->stream));
  c->cub_tmp.ensure(bytes);
  SOF_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, bytes, in, out, n, c->stream));
  c->launches += 2;
}

void exclusive_scan_i32(sof_ctx* c, const int32_t* in, int32_t* out, int64_t n) {
  if (n <= 0) return;
  size_t bytes = 0;
  SOF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, c->stream));
  c->cub_tmp.ensure(bytes);
  SOF_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, bytes, in, out, n, c->stream));
  c->launches += 2;
}

// ---- K0 / K1: preprocessing ------------------------------------------------------------------

__global__ void k_gauss_static(int64_t n, const double* __restrict__ pos,
                               const double* __restrict__ scale, const double* __restrict__ rot,
                               const double* __restrict__ opa, double fs, GaussStatic* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  GaussStatic g;
  gauss_static(pos + 3 * i, scale + 3 * i, rot + 4 * i, opa[i], fs, g);
  out[i] = g;
}

__global__ void k_view_rec(int64_t n, const GaussStatic* __restrict__ g, Cam cam, Rec* out,
                           RecF* outf) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  Rec r;
  gauss_view(g[i], cam, r);
  out[i] = r;
  if (outf) outf[i] = make_recf(r);
}

// Live bindings: Gaussians the reference lists in every tile (their box crosses the
// camera plane, tiles.hpp:116-126) are COUNTED through one sorted per-view list
// (Binding::nb/bkey/bidx) instead of being listed everywhere. kCountBehind: behind the
// camera (gauss_behind), listed nowhere; kCountCross: listed only in the tiles whose
// points it may reach (cross_tile_live); Binding::xpos marks those entries so the
// evaluation does not count them twice.
constexpr uint8_t kCountBehind = 1, kCountCross = 2;

// cross_tile_count out of line (rare; keeps the rect kernels' register count)
__device__ __noinline__ uint32_t cross_tile_count_ni(const Rec* __restrict__ r, int ts, int tiles_x, int tiles_y) {
  return cross_tile_count(*r, ts, tiles_x, tiles_y);
}

// Per-view binning inputs of k_tile_rect, produced by the record kernel in the same
// pass over GaussStatic when the binding of the view is built right away.
struct RectOut {
  int ts, tiles_x, tiles_y;
  int4* rect;
  uint32_t* cnt;
  uint64_t* zkey;
  int32_t* idx;
  bool live_only;   // leave dead Gaussians (op < 1/255) out of the lists (see Binding::live)
  uint8_t* behind;  // live_only: 1 for gauss_behind Gaussians (counted, not listed)
  unsigned long long* nflag;  // live_only: number of nonzero count flags (the count list's size)
};

// warp-aggregated increment of *ctr for the lanes with f set
__device__ __forceinline__ void count_flags(unsigned long long* ctr, bool f) {
  const unsigned m = __ballot_sync(__activemask(), f);
  if (m && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(ctr, (unsigned long long)__popc(m));
}

// k_view_rec + k_tile_rect in one pass (one GaussStatic read per Gaussian and view).
#ifndef SOF_REC_MINB
#define SOF_REC_MINB 1
#endif
__global__ void __launch_bounds__(128, SOF_REC_MINB) k_view_rec_rect(int64_t n, const GaussStatic* __restrict__ g,
                                                                     Cam cam, Rec* out, RectOut ro) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i > n) return;
  if (i == n) {  // sentinel for the exclusive scan over n + 1 counts
    ro.cnt[n] = 0;
    return;
  }
  const GaussStatic gs = g[i];
  Rec r;
  gauss_view(gs, cam, r);
  out[i] = r;
  int tx0, tx1, ty0, ty1;
  uint32_t count = 0;
  const bool live = ro.live_only && r.op >= kMinAlpha;
  const bool behind = live && gauss_behind(gs, cam, r.c);
  bool crosses = false;
  if (!(ro.live_only && (r.op < kMinAlpha || behind)) &&
      tile_rect(gs, cam, ro.ts, ro.tiles_x, ro.tiles_y, tx0, tx1, ty0, ty1, &crosses)) {
    count = (live && crosses) ? cross_tile_count_ni(out + i, ro.ts, ro.tiles_x, ro.tiles_y)
                              : uint32_t(tx1 - tx0 + 1) * uint32_t(ty1 - ty0 + 1);
    ro.rect[i] = make_int4(tx0, tx1, ty0, ty1);
  }
  if (ro.live_only) {
    const uint8_t f = behind ? kCountBehind : (live && crosses) ? kCountCross : 0;
    ro.behind[i] = f;
    count_flags(ro.nflag, f != 0);
  }
  ro.cnt[i] = count;
  ro.zkey[i] = double_key(r.zmin);
  ro.idx[i] = int32_t(i);
}

// precompute() rejects non-finite parameters (precompute.hpp:60-63): checked on the
// device (a host loop over the arrays cost ~10 ms per 3M Gaussians of the e2e step)
__global__ void k_check_finite(int64_t n, const double* __restrict__ pos, const double* __restrict__ scale,
                               const double* __restrict__ opa, unsigned long long* bad) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  bool ok = true;
  if (i < n) {
    ok = isfinite(opa[i]);
    for (int k = 0; k < 3; ++k) ok = ok && isfinite(pos[3 * i + k]) && isfinite(scale[3 * i + k]);
  }
  if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1ull);
}

void scene_check_finite(sof_ctx* c, unsigned long long* bad) {
  if (c->n == 0) return;
  k_check_finite<<<grid_for(c->n, 256), 256, 0, c->stream>>>(c->n, c->pos.p, c->scale.p, c->opa.p, bad);
  SOF_LAUNCHED(c);
}

void scene_prep(sof_ctx* c) {
  c->gstat.ensure(c->n);
  if (c->n == 0) return;
  k_gauss_static<<<grid_for(c->n, 128), 128, 0, c->stream>>>(
      c->n, c->pos.p, c->scale.p, c->rot.p, c->opa.p, c->filter_scale, c->gstat.p);
  SOF_LAUNCHED(c);
}

// Marks every per-view cache stale but keeps the allocations (each meshing step
// recomputes its per-view records and bindings; nothing is carried across calls).
void mark_views_stale(sof_ctx* c) {
  c->rec_valid.assign(c->cams.size(), 0);
  for (auto& b : c->bindings) b.view = -1;
  for (int k = 0; k < 2; ++k) {
    c->bind_scratch[k].view = -1;
    c->scratch_view[k] = -1;
  }
  c->cache_bytes = 0;
  c->view_cache_off = false;
}

// New scene or cameras: drop the cached per-view state. Buffers are kept (grow-only)
// unless the number of views changes, so repeated uploads do not re-allocate HBM.
void invalidate_view_caches(sof_ctx* c) {
  if (c->recs.size() != c->cams.size()) {
    c->recs.clear();
    c->recfs.clear();
    c->bindings.clear();
    c->recs.resize(c->cams.size());
    c->recfs.resize(c->cams.size());
    c->bindings.resize(c->cams.size());
  }
  mark_views_stale(c);
}

// Records of `view` (cached for the step when the budget allows). With ro, a fresh
// computation also writes the binning inputs (returns true in *rect_done).
static const Rec* view_records_impl(sof_ctx* c, int view, const RectOut* ro, bool* rect_done) {
  if (rect_done) *rect_done = false;
  if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
  if (c->rec_valid[view] == 1) return c->recs[view].p;
  if (c->rec_valid[view] == 2) {  // a truncated bisection cache: not the full records
    c->rec_valid[view] = 0;
    c->bindings[view].view = -1;
  }
  const int sel = c->scratch_sel;
  if (c->scratch_view[sel] == view) return c->rec_scratch[sel].p;
  const bool with_f = c->eval_path == 0;  // float filter records only for the FP32 path
  const size_t bytes = size_t(c->n) * (sizeof(Rec) + (with_f ? sizeof(RecF) : 0));
  DBuf<Rec>* dst = &c->rec_scratch[sel];
  DBuf<RecF>* dstf = &c->recf_scratch[sel];
  c->scratch_view[sel] = view;
  if (!c->view_cache_off && c->cache_bytes + bytes <= c->cache_budget) {
    c->scratch_view[sel] = -1;
    dst = &c->recs[view];
    dstf = &c->recfs[view];
    c->cache_bytes += bytes;
    c->rec_valid[view] = 1;
  }
  dst->ensure(std::max<int64_t>(c->n, 1));
  if (with_f) dstf->ensure(std::max<int64_t>(c->n, 1));
  if (c->n > 0 && ro && !with_f) {
    k_view_rec_rect<<<grid_for(c->n + 1, 128), 128, 0, c->stream>>>(c->n, c->gstat.p, c->cams[view], dst->p, *ro);
    SOF_LAUNCHED(c);
    *rect_done = true;
  } else if (c->n > 0) {
    k_view_rec<<<grid_for(c->n, 128), 128, 0, c->stream>>>(c->n, c->gstat.p, c->cams[view],
                                                            dst->p, with_f ? dstf->p : nullptr);
    SOF_LAUNCHED(c);
  }
  return dst->p;
}

const Rec* view_records(sof_ctx* c, int view) { return view_records_impl(c, view, nullptr, nullptr); }

// Float filter records of `view`, valid after view_records(c, view).
const RecF* view_recf(sof_ctx* c, int view) {
  if (c->rec_valid[view] == 1) return c->recfs[view].p;
  return c->recf_scratch[c->scratch_view[0] == view ? 0 : 1].p;
}

// ---- K2: Gaussian tile binning ------------------------------------------------------------------

__global__ void k_tile_rect(int64_t n, const GaussStatic* __restrict__ g,
                            const Rec* __restrict__ rec, Cam cam, int ts, int tiles_x, int tiles_y,
                            bool live_only, int4* rect, uint32_t* cnt, uint64_t* zkey, int32_t* idx,
                            uint8_t* behind_out, unsigned long long* nflag) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i > n) return;
  if (i == n) {  // sentinel for the exclusive scan over n + 1 counts
    cnt[n] = 0;
    return;
  }
  int tx0, tx1, ty0, ty1;
  uint32_t count = 0;
  const bool live = live_only && rec[i].op >= kMinAlpha;
  const bool behind = live && gauss_behind(g[i], cam, rec[i].c);
  bool crosses = false;
  if (!(live_only && (rec[i].op < kMinAlpha || behind)) &&
      tile_rect(g[i], cam, ts, tiles_x, tiles_y, tx0, tx1, ty0, ty1, &crosses)) {
    count = (live && crosses) ? cross_tile_count_ni(rec + i, ts, tiles_x, tiles_y)
                              : uint32_t(tx1 - tx0 + 1) * uint32_t(ty1 - ty0 + 1);
    rect[i] = make_int4(tx0, tx1, ty0, ty1);
  }
  if (live_only) {
    const uint8_t f = behind ? kCountBehind : (live && crosses) ? kCountCross : 0;
    behind_out[i] = f;
    count_flags(nflag, f != 0);
  }
  cnt[i] = count;
  zkey[i] = double_key(rec[i].zmin);
  idx[i] = int32_t(i);
}

__global__ void k_gather_counts(int64_t n, const int32_t* __restrict__ order,
                                const uint32_t* __restrict__ cnt, uint32_t* out) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r > n) return;
  out[r] = (r == n) ? 0u : cnt[order[r]];
}

// One thread per Gaussian (in (min_z, index) order) emits its (tile, gaussian)
// entries; Gaussians covering many tiles (rare) hand the tail to their warp.
// Live crossing Gaussians (gflag kCountCross) emit only their cross_tile_live tiles, one
// warp per Gaussian scanning the screen row by row (compacted with ballots, so the
// entries come out in row-major tile order as the count in the rect kernel assumed).
__device__ __forceinline__ void emit_cross_warp(const Rec& r, int32_t g, int64_t o, int ts, int tiles_x, int tiles_y,
                                                uint32_t* keys, int32_t* vals) {
  const int lane = threadIdx.x & 31;
  for (int ty = 0; ty < tiles_y; ++ty) {
    if (!cross_row_live(r, ts, tiles_x, ty)) continue;
    for (int tx0 = 0; tx0 < tiles_x; tx0 += 32) {
      const int tx = tx0 + lane;
      const bool pass = tx < tiles_x && cross_tile_live(r, ts, tx, ty);
      const unsigned m = __ballot_sync(0xffffffffu, pass);
      if (pass) {
        const int64_t q = o + __popc(m & ((1u << lane) - 1u));
        keys[q] = uint32_t(ty * tiles_x + tx);
        vals[q] = g;
      }
      o += __popc(m);
    }
  }
}

__global__ void k_emit_entries(int64_t n, const int32_t* __restrict__ order,
                               const int4* __restrict__ rect, const uint32_t* __restrict__ cnt,
                               const int64_t* __restrict__ off, int tiles_x, uint32_t* keys,
                               int32_t* vals, const uint8_t* __restrict__ gflag) {
  constexpr uint32_t kOwn = 16;  // entries written by the owning thread
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int32_t g = -1;
  uint32_t count = 0;
  int4 rc = make_int4(0, 0, 0, 0);
  int64_t base = 0;
  bool cross = false;
  if (r < n) {
    g = order[r];
    count = cnt[g];
    if (count) {
      rc = rect[g];
      base = off[r];
      cross = gflag && gflag[g] == kCountCross;  // emitted by k_emit_cross
    }
  }
  if (cross) count = 0;
  {  // row-major walk of the first kOwn tiles of the rectangle (no divisions)
    const uint32_t own = min(count, kOwn);
    int tx = rc.x, ty = rc.z;
    for (uint32_t k = 0; k < own; ++k) {
      keys[base + k] = uint32_t(ty * tiles_x + tx);
      vals[base + k] = g;
      if (++tx > rc.y) {
        tx = rc.x;
        ++ty;
      }
    }
  }
  // large footprints: the warp writes the remaining entries cooperatively
  unsigned big = __ballot_sync(0xffffffffu, count > kOwn);
  while (big) {
    const int src = __ffs(big) - 1;
    big &= big - 1;
    const uint32_t bc = __shfl_sync(0xffffffffu, count, src);
    const int32_t bg = __shfl_sync(0xffffffffu, g, src);
    const int bx = __shfl_sync(0xffffffffu, rc.x, src), by = __shfl_sync(0xffffffffu, rc.y, src);
    const int bz = __shfl_sync(0xffffffffu, rc.z, src);
    const int64_t bb = __shfl_sync(0xffffffffu, base, src);
    const int bw = by - bx + 1;
    for (uint32_t k = kOwn + lane; k < bc; k += 32) {
      const int ty = bz + int(k / bw), tx = bx + int(k % bw);
      keys[bb + k] = uint32_t(ty * tiles_x + tx);
      vals[bb + k] = bg;
    }
  }
}

// The live crossing Gaussians' entries (the slots k_emit_entries left to it).
__global__ void k_emit_cross(int64_t n, const int32_t* __restrict__ order, const uint32_t* __restrict__ cnt,
                             const int64_t* __restrict__ off, const uint8_t* __restrict__ gflag,
                             const Rec* __restrict__ rec, int ts, int tiles_x, int tiles_y, uint32_t* keys,
                             int32_t* vals) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  int32_t g = -1;
  bool cross = false;
  if (r < n) {
    g = order[r];
    cross = cnt[g] != 0 && gflag[g] == kCountCross;
  }
  unsigned xb = __ballot_sync(0xffffffffu, cross);
  while (xb) {
    const int src = __ffs(xb) - 1;
    xb &= xb - 1;
    const int32_t bg = __shfl_sync(0xffffffffu, g, src);
    const int64_t rr = __shfl_sync(0xffffffffu, r, src);
    emit_cross_warp(rec[bg], bg, off[rr], ts, tiles_x, tiles_y, keys, vals);
  }
}

// starts[t] = first position with key >= t, for t in [0, nseg]; keys sorted ascending.
template <typename K, int SHIFT>
__global__ void k_segment_starts(int64_t m, const K* __restrict__ keys, int64_t nseg,
                                 int64_t* starts) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j > m) return;
  const int64_t k = (j < m) ? int64_t(uint64_t(keys[j]) >> SHIFT) : nseg;
  const int64_t prev = (j > 0) ? int64_t(uint64_t(keys[j - 1]) >> SHIFT) : -1;
  for (int64_t t = prev + 1; t <= k; ++t) starts[t] = j;
}

static void build_binding_tail(sof_ctx* c, int view, int ts, Binding& b, int64_t M, int64_t T,
                               int tiles_x, int tiles_y);

static void build_binding(sof_ctx* c, int view, int ts, bool live, Binding& b, bool charge) {
  b.trunc = false;
  const Cam& cam = c->cams[view];
  const int tiles_x = (cam.w + ts - 1) / ts, tiles_y = (cam.h + ts - 1) / ts;
  const int64_t T = int64_t(tiles_x) * tiles_y;
  const int64_t n = c->n;
  b.live = live;
  if (n == 0) {
    view_records(c, view);
    build_binding_tail(c, view, ts, b, 0, T, tiles_x, tiles_y);
    return;
  }
  c->rect.ensure(n);
  c->gcount.ensure(n + 1);
  c->zkey_in.ensure(n);
  c->zkey_out.ensure(n);
  c->gidx_in.ensure(n);
  c->gidx_out.ensure(n);
  c->goff.ensure(n + 1);
  c->gbehind.ensure(n);
  c->bin_scalar.ensure(4);  // [0] visible count, [1] tie-run overflow, [2] count flags
  zero_async(c, c->bin_scalar.p, 4 * sizeof(int64_t));
  unsigned long long* nflag = reinterpret_cast<unsigned long long*>(c->bin_scalar.p + 2);
  const RectOut ro{ts, tiles_x, tiles_y, c->rect.p, c->gcount.p, c->zkey_in.p, c->gidx_in.p, live, c->gbehind.p,
                   nflag};
  bool rect_done = false;
  const Rec* rec = view_records_impl(c, view, &ro, &rect_done);
  if (!rect_done) {
    k_tile_rect<<<grid_for(n + 1, 128), 128, 0, c->stream>>>(n, c->gstat.p, rec, cam, ts, tiles_x,
                                                              tiles_y, live, c->rect.p, c->gcount.p,
                                                              c->zkey_in.p, c->gidx_in.p, c->gbehind.p, nflag);
    SOF_LAUNCHED(c);
  }
  bin_by_key(c, view, ts, tiles_x, tiles_y, b, charge);
}

__global__ void k_gather_keys(int64_t n, const int32_t* __restrict__ perm, const uint64_t* __restrict__ src,
                              uint64_t* dst) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j < n) dst[j] = src[perm[j]];
}

// Bisection-cache binning (bisect_cache_views): a Gaussian enters tile t only when
// t is reachable by a crossing-edge segment and its min_z <= zmax(t) (ordered keys),
// i.e. exactly the entries of the full list's prefix that the bisection can read.
__device__ __forceinline__ bool tile_wanted(const unsigned long long* zmax, int64_t t, unsigned long long zk) {
  return zmax[t] >= zk;  // zmax 0: no segment reaches t (every key is >= 1)
}

// (live crossing Gaussians: only their cross_tile_live tiles, as k_emit_entries; in their
// own kernels, so the common path keeps its register count)
__device__ __forceinline__ uint32_t filtered_cross_count(const Rec* __restrict__ rp, int4 rc,
                                                      const unsigned long long* __restrict__ zmax, int tiles_x,
                                                      unsigned long long zk, int ts) {
  const Rec r = *rp;
  uint32_t k = 0;
  for (int ty = rc.z; ty <= rc.w; ++ty) {
    if (!cross_row_live(r, ts, tiles_x, ty)) continue;
    for (int tx = rc.x; tx <= rc.y; ++tx)
      k += tile_wanted(zmax, int64_t(ty) * tiles_x + tx, zk) && cross_tile_live(r, ts, tx, ty);
  }
  return k;
}

__device__ __forceinline__ void filtered_cross_emit(const Rec* __restrict__ rp, int32_t g, int4 rc, int64_t o,
                                                 const unsigned long long* __restrict__ zmax, int tiles_x,
                                                 unsigned long long zk, int ts, uint32_t* keys, int32_t* vals) {
  const Rec r = *rp;
  for (int ty = rc.z; ty <= rc.w; ++ty) {
    if (!cross_row_live(r, ts, tiles_x, ty)) continue;
    for (int tx = rc.x; tx <= rc.y; ++tx) {
      const int64_t t = int64_t(ty) * tiles_x + tx;
      if (tile_wanted(zmax, t, zk) && cross_tile_live(r, ts, tx, ty)) {
        keys[o] = uint32_t(t);
        vals[o] = g;
        ++o;
      }
    }
  }
}

__global__ void k_filter_counts(int64_t n, const int4* __restrict__ rect, const uint64_t* __restrict__ zkey,
                                const unsigned long long* __restrict__ zmax, int tiles_x, uint32_t* cnt,
                                const uint8_t* __restrict__ gflag, const Rec* __restrict__ rec, int ts) {
  const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (g >= n || cnt[g] == 0) return;
  const int4 rc = rect[g];
  const unsigned long long zk = zkey[g];
  if (gflag && gflag[g] == kCountCross) return;  // k_filter_counts_cross
  uint32_t k = 0;
  for (int ty = rc.z; ty <= rc.w; ++ty)
    for (int tx = rc.x; tx <= rc.y; ++tx) k += tile_wanted(zmax, int64_t(ty) * tiles_x + tx, zk);
  cnt[g] = k;
}

__global__ void k_emit_filtered(int64_t n, const int32_t* __restrict__ order, const int4* __restrict__ rect,
                                const int64_t* __restrict__ off, const uint64_t* __restrict__ zkey,
                                const unsigned long long* __restrict__ zmax, int tiles_x, uint32_t* keys,
                                int32_t* vals, const uint8_t* __restrict__ gflag, const Rec* __restrict__ rec,
                                int ts) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  const int32_t g = order[r];
  const int4 rc = rect[g];
  const unsigned long long zk = zkey[g];
  int64_t o = off[r];
  if (gflag && gflag[g] == kCountCross) return;  // k_emit_filtered_cross
  for (int ty = rc.z; ty <= rc.w; ++ty)
    for (int tx = rc.x; tx <= rc.y; ++tx) {
      const int64_t t = int64_t(ty) * tiles_x + tx;
      if (tile_wanted(zmax, t, zk)) {
        keys[o] = uint32_t(t);
        vals[o] = g;
        ++o;
      }
    }
}

__global__ void k_filter_counts_cross(int64_t n, const int4* __restrict__ rect, const uint64_t* __restrict__ zkey,
                                      const unsigned long long* __restrict__ zmax, int tiles_x, uint32_t* cnt,
                                      const uint8_t* __restrict__ gflag, const Rec* __restrict__ rec, int ts) {
  const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (g >= n || cnt[g] == 0 || gflag[g] != kCountCross) return;
  cnt[g] = filtered_cross_count(rec + g, rect[g], zmax, tiles_x, zkey[g], ts);
}

__global__ void k_emit_filtered_cross(int64_t n, const int32_t* __restrict__ order, const int4* __restrict__ rect,
                                      const int64_t* __restrict__ off, const uint64_t* __restrict__ zkey,
                                      const unsigned long long* __restrict__ zmax, int tiles_x, uint32_t* keys,
                                      int32_t* vals, const uint8_t* __restrict__ gflag, const Rec* __restrict__ rec,
                                      int ts) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  const int32_t g = order[r];
  if (gflag[g] != kCountCross) return;
  filtered_cross_emit(rec + g, g, rect[g], off[r], zmax, tiles_x, zkey[g], ts, keys, vals);
}

// Positions i in [0, M) of a tile-list array whose entry is a kCountCross Gaussian
// (flag[ent[i]]), ascending: PASS 0 counts per block of kSelBlock, PASS 1 writes.
constexpr int kSelBlock = 1024;
template <int PASS>
__global__ void __launch_bounds__(256) k_cross_sel(int64_t M, const int32_t* __restrict__ ent,
                                                   const uint8_t* __restrict__ flag, int64_t* cnt,
                                                   const int64_t* __restrict__ off, int64_t* out) {
  __shared__ int wsum[8];
  const int64_t b0 = int64_t(blockIdx.x) * kSelBlock;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t base = PASS ? off[blockIdx.x] : 0;
  int total = 0;
  for (int rr = 0; rr < kSelBlock / 256; ++rr) {
    const int64_t i = b0 + rr * 256 + threadIdx.x;
    const bool p = i < M && flag[ent[i]] == kCountCross;
    if (PASS == 0) {
      total += __syncthreads_count(p);
      continue;
    }
    const unsigned m = __ballot_sync(0xffffffffu, p);
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    int pre = 0, all = 0;
    for (int k = 0; k < 8; ++k) {
      pre += (k < w) ? wsum[k] : 0;
      all += wsum[k];
    }
    if (p) out[base + pre + __popc(m & ((1u << lane) - 1u))] = i;
    base += all;
    __syncthreads();
  }
  if (PASS == 0 && threadIdx.x == 0) cnt[blockIdx.x] = total;
}

// (key, 2 index) of the counted Gaussians (Binding::bidx holds 2 g: see count_pairs)
__global__ void k_count_list_init(int64_t nb, const int32_t* __restrict__ sel, const uint64_t* __restrict__ zkey,
                                  uint64_t* key, int32_t* idx2) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= nb) return;
  key[j] = zkey[sel[j]];
  idx2[j] = 2 * sel[j];
}

struct HasTiles {
  const uint32_t* cnt;
  __device__ bool operator()(int32_t i) const { return cnt[i] != 0; }
};

// 32-bit order key of a sort key: the double behind the 64-bit key rounded toward
// -inf to float (monotone, so x < y implies f(x) <= f(y)), -0 folded onto +0.
__global__ void k_float_keys(int64_t m, const int32_t* __restrict__ idx, const uint64_t* __restrict__ zkey,
                             uint32_t* fkey) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= m) return;
  float f = __double2float_rd(key_double(zkey[idx[j]]));
  if (f == 0.0f) f = 0.0f;
  const uint32_t u = __float_as_uint(f);
  fkey[j] = (u >> 31) ? ~u : (u | 0x80000000u);
}

// Runs of equal float keys (in index order after the stable sort) are re-sorted by the
// full 64-bit key, index breaking ties: the result is the (key, index) order. A run
// longer than kTieRun sets *overflow (the caller then sorts by the 64-bit keys).
constexpr int kTieRun = 32;
__global__ void k_fix_ties(int64_t m, const uint32_t* __restrict__ fk, int32_t* idx,
                           const uint64_t* __restrict__ zkey, int* overflow) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const uint32_t f = (j < m) ? fk[j] : 0u;
  // neighbours through the warp (one load per element); the warp's edge lanes load theirs
  uint32_t prev = __shfl_up_sync(0xffffffffu, f, 1), next = __shfl_down_sync(0xffffffffu, f, 1);
  if (j >= m) return;
  if (lane == 0) prev = (j > 0) ? fk[j - 1] : ~f;
  if (lane == 31 || j + 1 >= m) next = (j + 1 < m) ? fk[j + 1] : ~f;
  if ((j > 0 && prev == f) || j + 1 >= m || next != f) return;  // head of a run >= 2 only
  int64_t e = j + 1;
  while (e < m && fk[e] == f) {
    if (++e - j > kTieRun) {
      atomicExch(overflow, 1);
      return;
    }
  }
  const int L = int(e - j);
  uint64_t kk[kTieRun];
  int32_t ii[kTieRun];
  for (int q = 0; q < L; ++q) {
    ii[q] = idx[j + q];
    kk[q] = zkey[ii[q]];
  }
  for (int q = 1; q < L; ++q) {  // insertion sort; indices ascend already, so key ties keep them
    const uint64_t k = kk[q];
    const int32_t i = ii[q];
    int r = q - 1;
    while (r >= 0 && kk[r] > k) {
      kk[r + 1] = kk[r];
      ii[r + 1] = ii[r];
      --r;
    }
    kk[r + 1] = k;
    ii[r + 1] = i;
  }
  for (int q = 0; q < L; ++q) idx[j + q] = ii[q];
}

// Second half of a binning: the Gaussians with at least one tile (the others emit
// nothing) in (zkey_in, index) order, their (tile, gaussian) entries emitted in that
// order, and a stable sort by tile gives per-tile lists ordered by (key, index).
// Inputs: c->rect, c->gcount[n + 1] (0 sentinel), c->zkey_in filled by a rect kernel.
//
// The (key, index) sort: the visible Gaussians are compacted in index order, sorted
// stably by a 32-bit float rounding of the key (4 radix passes instead of 8), and runs
// of equal float keys are then re-sorted by the full key (k_fix_ties); runs longer than
// kTieRun (never seen in practice) fall back to the 64-bit sort.
void bin_by_key(sof_ctx* c, int view, int ts, int tiles_x, int tiles_y, Binding& b,
                bool charge_cache) {
  const int64_t T = int64_t(tiles_x) * tiles_y;
  const int64_t n = c->n;
  if (c->bin_zmax) {  // bisection-cache binning: only the reachable (tile, depth) entries
    k_filter_counts<<<grid_for(n, 256), 256, 0, c->stream>>>(n, c->rect.p, c->zkey_in.p, c->bin_zmax, tiles_x,
                                                             c->gcount.p, b.live ? c->gbehind.p : nullptr,
                                                             nullptr, ts);
    SOF_LAUNCHED(c);
    if (b.live) {
      k_filter_counts_cross<<<grid_for(n, 256), 256, 0, c->stream>>>(n, c->rect.p, c->zkey_in.p, c->bin_zmax,
                                                                     tiles_x, c->gcount.p, c->gbehind.p,
                                                                     view_records(c, view), ts);
      SOF_LAUNCHED(c);
    }
  }
  // visible Gaussians in index order -> gidx_in[0, m)
  {
    size_t bytes = 0;
    thrust::counting_iterator<int32_t> it(0);
    HasTiles pred{c->gcount.p};
    SOF_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, c->gidx_in.p, c->bin_scalar.p, n, pred, c->stream));
    c->cub_tmp.ensure(bytes);
    SOF_CUDA(cub::DeviceSelect::If(c->cub_tmp.p, bytes, it, c->gidx_in.p, c->bin_scalar.p, n, pred, c->stream));
    c->launches += 2;
  }
  const int64_t m = read_scalar(c, c->bin_scalar.p);
  c->bin_m = m;
  if (m > 0) {
    uint32_t* fk_in = reinterpret_cast<uint32_t*>(c->zkey_out.p);  // zkey_out: 2 x n u32 of scratch
    uint32_t* fk_out = fk_in + n;
    k_float_keys<<<grid_for(m, 256), 256, 0, c->stream>>>(m, c->gidx_in.p, c->zkey_in.p, fk_in);
    SOF_LAUNCHED(c);
    sort_pairs_u32(c, fk_in, fk_out, c->gidx_in.p, c->gidx_out.p, m, 32);
    k_fix_ties<<<grid_for(m, 256), 256, 0, c->stream>>>(m, fk_out, c->gidx_out.p, c->zkey_in.p,
                                                         reinterpret_cast<int*>(c->bin_scalar.p + 1));
    SOF_LAUNCHED(c);
  }
  c->ekey_in.ensure(m + 1);
  auto offsets = [&]() {
    k_gather_counts<<<grid_for(m + 1, 256), 256, 0, c->stream>>>(m, c->gidx_out.p, c->gcount.p, c->ekey_in.p);
    SOF_LAUNCHED(c);
    exclusive_scan_u32_to_i64(c, c->ekey_in.p, c->goff.p, m + 1);
  };
  offsets();
  // one read-back for the entry count, the tie-run overflow flag and the count-list size
  int64_t M = 0, nflag_h = 0;
  int overflow = 0;
  SOF_CUDA(cudaMemcpyAsync(c->pinned_scalar, c->goff.p + m, 8, cudaMemcpyDeviceToHost, c->stream));
  SOF_CUDA(cudaMemcpyAsync(c->pinned_scalar + 1, c->bin_scalar.p + 1, 8, cudaMemcpyDeviceToHost, c->stream));
  SOF_CUDA(cudaMemcpyAsync(c->pinned_scalar + 2, c->bin_scalar.p + 2, 8, cudaMemcpyDeviceToHost, c->stream));
  SOF_CUDA(cudaStreamSynchronize(c->stream));
  std::memcpy(&M, c->pinned_scalar, 8);
  std::memcpy(&overflow, c->pinned_scalar + 1, sizeof(int));
  std::memcpy(&nflag_h, c->pinned_scalar + 2, 8);
  if (m > 0 && overflow) {  // a long tie run (never seen in practice): the full 64-bit sort
    c->zkey_aux.ensure(m);
    k_gather_keys<<<grid_for(m, 256), 256, 0, c->stream>>>(m, c->gidx_in.p, c->zkey_in.p, c->zkey_aux.p);
    SOF_LAUNCHED(c);
    sort_pairs_u64(c, c->zkey_aux.p, c->zkey_out.p, c->gidx_in.p, c->gidx_out.p, m, 64);
    offsets();
    M = read_scalar(c, c->goff.p + m);
  }
  c->bin_nflag = nflag_h;
  if (charge_cache && &b != &c->bind_scratch[0] && &b != &c->bind_scratch[1]) {
    // keep the list resident for the rest of the step if the cache budget allows
    const size_t bytes = size_t(M) * 4 + size_t(T + 1) * 8;
    if (c->view_cache_off || c->cache_bytes + bytes > c->cache_budget) {
      c->bind_scratch[c->scratch_sel].live = b.live;
      c->bind_scratch[c->scratch_sel].trunc = false;
      build_binding_tail(c, view, ts, c->bind_scratch[c->scratch_sel], M, T, tiles_x, tiles_y);
      return;
    }
    c->cache_bytes += bytes;
  }
  build_binding_tail(c, view, ts, b, M, T, tiles_x, tiles_y);
}

// Binding::xpos: the list positions of b.ent[0, M) holding kCountCross Gaussians
// (flag indexed by the entry: Gaussian ids, or rows of a truncated binding).
static void cross_positions(sof_ctx* c, Binding& b, int64_t M, const uint8_t* flag) {
  const int64_t nblk = (M + kSelBlock - 1) / kSelBlock;
  c->sel_cnt.ensure(nblk + 1);
  c->sel_off.ensure(nblk + 1);
  k_cross_sel<0><<<unsigned(nblk), 256, 0, c->stream>>>(M, b.ent.p, flag, c->sel_cnt.p, nullptr, nullptr);
  SOF_LAUNCHED(c);
  scan_i64_i64(c, c->sel_cnt.p, c->sel_off.p, nblk);
  const int64_t X = read_scalar(c, c->sel_off.p + nblk);
  b.nx = X;
  if (X == 0) return;
  b.xpos.ensure(X);
  k_cross_sel<1><<<unsigned(nblk), 256, 0, c->stream>>>(M, b.ent.p, flag, nullptr, c->sel_off.p, b.xpos.p);
  SOF_LAUNCHED(c);
}

static void build_binding_tail(sof_ctx* c, int view, int ts, Binding& b, int64_t M, int64_t T,
                               int tiles_x, int tiles_y) {

  // (on the binding that is served: the view's cache or a scratch slot)
  b.nb = 0;
  b.nx = 0;
  if (b.live && c->n > 0 && c->bin_nflag > 0) {  // the counted Gaussians: (min_z key, index) order, index
                                                 // order kept on ties
    size_t bytes = 0;
    thrust::counting_iterator<int32_t> it(0);
    const uint8_t* flags = c->gbehind.p;
    const int64_t n = c->n;
    c->zkey_aux.ensure(n);
    int32_t* sel = reinterpret_cast<int32_t*>(c->zkey_aux.p);  // n int32 of scratch
    SOF_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, sel, c->bin_scalar.p + 1, n, c->stream));
    c->cub_tmp.ensure(bytes);
    SOF_CUDA(cub::DeviceSelect::Flagged(c->cub_tmp.p, bytes, it, flags, sel, c->bin_scalar.p + 1, n, c->stream));
    c->launches += 2;
    const int64_t nb = read_scalar(c, c->bin_scalar.p + 1);
    b.nb = nb;
    if (nb > 0) {
      b.bkey.ensure(2 * nb);
      b.bidx.ensure(2 * nb);
      k_count_list_init<<<grid_for(nb, 256), 256, 0, c->stream>>>(nb, sel, c->zkey_in.p, b.bkey.p + nb,
                                                                   b.bidx.p + nb);
      SOF_LAUNCHED(c);
      sort_pairs_u64(c, b.bkey.p + nb, b.bkey.p, b.bidx.p + nb, b.bidx.p, nb, 64);  // stable: index order on ties
    }
  }
  const int64_t n = c->n;
  b.view = view;
  b.tile_size = ts;
  b.tiles_x = tiles_x;
  b.tiles_y = tiles_y;
  if (M > INT32_MAX) throw InvalidArg("a view's tile lists exceed 2^31 entries");
  b.off.ensure(T + 1);
  b.entries = M;
  b.ent.ensure(std::max<int64_t>(M, 1));
  if (M > 0) {
    c->ekey_in.ensure(M);
    c->ekey_out.ensure(M);
    c->eval_in.ensure(M);
    const uint8_t* gflag = b.live ? c->gbehind.p : nullptr;
    const Rec* rec = view_records(c, view);
    if (c->bin_zmax) {
      k_emit_filtered<<<grid_for(c->bin_m, 256), 256, 0, c->stream>>>(c->bin_m, c->gidx_out.p, c->rect.p, c->goff.p,
                                                                       c->zkey_in.p, c->bin_zmax, tiles_x,
                                                                       c->ekey_in.p, c->eval_in.p, gflag, nullptr, ts);
      if (gflag && b.nb > 0) {
        k_emit_filtered_cross<<<grid_for(c->bin_m, 256), 256, 0, c->stream>>>(
            c->bin_m, c->gidx_out.p, c->rect.p, c->goff.p, c->zkey_in.p, c->bin_zmax, tiles_x, c->ekey_in.p,
            c->eval_in.p, gflag, rec, ts);
        SOF_LAUNCHED(c);
      }
    } else
    {
      k_emit_entries<<<grid_for(c->bin_m, 256), 256, 0, c->stream>>>(c->bin_m, c->gidx_out.p, c->rect.p, c->gcount.p,
                                                                      c->goff.p, tiles_x, c->ekey_in.p, c->eval_in.p,
                                                                      b.nb > 0 ? gflag : nullptr);
      if (gflag && b.nb > 0) {
        k_emit_cross<<<grid_for(c->bin_m, 256), 256, 0, c->stream>>>(c->bin_m, c->gidx_out.p, c->gcount.p, c->goff.p,
                                                                      gflag, rec, ts, tiles_x, tiles_y, c->ekey_in.p,
                                                                      c->eval_in.p);
        SOF_LAUNCHED(c);
      }
    }
    SOF_LAUNCHED(c);
    // stable sort by tile keeps the (min_z, index) order inside every tile list
    sort_pairs_u32(c, c->ekey_in.p, c->ekey_out.p, c->eval_in.p, b.ent.p, M, bits_for(T));
    if (b.nb > 0) cross_positions(c, b, M, c->gbehind.p);
  }
  k_segment_starts<uint32_t, 0><<<grid_for(M + 1, 256), 256, 0, c->stream>>>(M, c->ekey_out.p, T,
                                                                             b.off.p);
  SOF_LAUNCHED(c);
}

const Binding& view_binding(sof_ctx* c, int view, int tile_size, bool live) {
  Binding& cached = c->bindings[view];
  if (cached.view == view && cached.tile_size == tile_size && cached.live == live && !cached.trunc) return cached;
  if (cached.trunc) {  // a truncated bisection cache is rebuilt as a full binding
    cached.view = -1;
    cached.trunc = false;
    if (c->rec_valid[view] == 2) c->rec_valid[view] = 0;
  }
  for (int k = 0; k < 2; ++k)
    if (c->bind_scratch[k].view == view && c->bind_scratch[k].tile_size == tile_size &&
        c->bind_scratch[k].live == live)
      return c->bind_scratch[k];
  // builds into the per-view slot (kept for the rest of the step) or, past the
  // cache budget, into the scratch slot; a resident binding of this view with other
  // parameters is rebuilt in place (its bytes are already charged to the budget)
  const bool resident = cached.view == view;
  build_binding(c, view, tile_size, live, cached, !resident);
  return (cached.view == view) ? cached : c->bind_scratch[c->scratch_sel];
}

// ---- K3: point scheduling ------------------------------------------------------------------------
//
// Points are grouped by tile with a counting sort (histogram, scan over the T
// tiles, scatter), then cut into blocks of <= 256 points of one tile
// (tiles.hpp:61-82). Everything stays on the device: no host synchronisation per
// view. Order inside a tile is arbitrary; it cannot change any result because
// every (point, view) evaluation is independent (field_eval.hpp:146-154).

// Warp-aggregated atomicAdd on a per-bin counter (all 32 lanes call it). Candidates
// arrive in index order, so equal bins mostly form runs of adjacent lanes: each run
// is reserved with one atomic by its first lane (shuffle + ballot only; no
// match.any, whose ADU throughput capped the scheduling kernels). Returns the slot
// of this lane among the lanes of its run that hit `bin`, offset by the run's base.
__device__ __forceinline__ int warp_tile_add(int* counters, int bin, bool valid) {
  constexpr unsigned kAll = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int k = valid ? bin : -1;
  const int prev = __shfl_up_sync(kAll, k, 1);
  const unsigned bnd = __ballot_sync(kAll, lane == 0 || prev != k);  // run starts
  const unsigned upto = (2u << lane) - 1u;                            // lanes <= this one
  const int leader = 31 - __clz(bnd & upto);
  int base = 0;
  if (valid && leader == lane) {
    const unsigned after = bnd & ~upto;
    const int end = after ? __ffs(after) - 1 : 32;
    base = atomicAdd(counters + k, end - lane);
  }
  base = __shfl_sync(kAll, base, leader);
  return base + (lane - leader);
}

// Per point: tile of the view (-1 when pruned or unobserved), histogram per tile.
// Candidates are all points (cand == nullptr) or a compacted list of the points not
// yet pruned; tile_of is indexed by candidate slot. S bins per tile: 16 (4x4 pixel
// cells) or 1.
// TS: the tile size when it is the default 16 (shifts and masks instead of integer
// divisions by a runtime value), 0 for any other tile size.
#ifndef SOF_SCHED_PTS
#define SOF_SCHED_PTS 1
#endif
constexpr int kSchedPts = SOF_SCHED_PTS;  // points per thread (loads of all issued first)
template <int TS>
__global__ void k_sched_tile(int64_t n, const int32_t* __restrict__ cand,
                             const double* __restrict__ xyz, Cam cam, int ts, int tiles_x,
                             bool single_bin, int S, const uint8_t* __restrict__ skip, int32_t* tile_of,
                             int* tile_cnt) {
  const int64_t k0 = blockIdx.x * int64_t(blockDim.x) * kSchedPts + threadIdx.x;
  double px[kSchedPts], py[kSchedPts], pz[kSchedPts];
  bool live[kSchedPts];
#pragma unroll
  for (int j = 0; j < kSchedPts; ++j) {
    const int64_t k = k0 + int64_t(j) * blockDim.x;
    live[j] = false;
    px[j] = py[j] = pz[j] = 0.0;
    if (k < n) {
      const int64_t i = cand ? cand[k] : k;
      if (!(skip && skip[i])) {
        live[j] = true;
        px[j] = xyz[3 * i];
        py[j] = xyz[3 * i + 1];
        pz[j] = xyz[3 * i + 2];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kSchedPts; ++j) {
    const int64_t k = k0 + int64_t(j) * blockDim.x;
    int tile = -1;
    if (live[j]) {
      const PointTile pt = point_tile<TS>(cam, px[j], py[j], pz[j], ts, tiles_x);
      // bin = tile x (4x4 cell of pixels inside the tile): points of one cell are
      // adjacent, so a warp covers a compact screen region (coherent conic culls)
      if (pt.tile >= 0) {
        if (single_bin) {
          tile = 0;
        } else if (S != 16) {
          tile = pt.tile;
        } else if (TS == 16) {  // px, py >= 0 here, so shifts are the divisions
          tile = pt.tile * 16 + ((((int)pt.py) & 15) >> 2) * 4 + ((((int)pt.px) & 15) >> 2);
        } else {
          const int cs = (ts + 3) / 4;
          tile = pt.tile * 16 + (((int)pt.py % ts) / cs) * 4 + ((int)pt.px % ts) / cs;
        }
      }
    }
    if (k < n) tile_of[k] = tile;
    warp_tile_add(tile_cnt, tile, tile >= 0);
  }
}

struct NotPruned {
  const uint8_t* ext;
  __device__ bool operator()(int32_t i) const { return ext[i] == 0; }
};

// Scatter pass: kScatterItems warp-contiguous groups of 32 candidates per warp, so
// that each warp keeps several slot-reserving atomics in flight (the returned base is
// a long round trip; one item per thread left this kernel latency-bound).
#ifndef SOF_SCATTER_ITEMS
#define SOF_SCATTER_ITEMS 4
#endif
constexpr int kScatterItems = SOF_SCATTER_ITEMS;
__global__ void k_sched_scatter(int64_t n, const int32_t* __restrict__ cand,
                                const int32_t* __restrict__ tile_of,
                                const int* __restrict__ tile_off, int* tile_cur, int32_t* order) {
  constexpr unsigned kAll = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t k0 = w * (32 * kScatterItems) + lane;
  int tile[kScatterItems], base[kScatterItems], leader[kScatterItems], off[kScatterItems];
  for (int q = 0; q < kScatterItems; ++q) {
    const int64_t k = k0 + 32 * q;
    tile[q] = (k < n) ? tile_of[k] : -1;
  }
  for (int q = 0; q < kScatterItems; ++q) {  // reserve: one atomic per run of equal bins
    const int t = tile[q];
    const int prev = __shfl_up_sync(kAll, t, 1);
    const unsigned bnd = __ballot_sync(kAll, lane == 0 || prev != t);
    const unsigned upto = (2u << lane) - 1u;
    leader[q] = 31 - __clz(bnd & upto);
    base[q] = 0;
    if (t >= 0 && leader[q] == lane) {
      const unsigned after = bnd & ~upto;
      const int end = after ? __ffs(after) - 1 : 32;
      base[q] = atomicAdd(tile_cur + t, end - lane);
    }
    off[q] = (t >= 0) ? tile_off[t] : 0;
  }
  for (int q = 0; q < kScatterItems; ++q) {
    const int b = __shfl_sync(kAll, base[q], leader[q]);
    if (tile[q] >= 0) {
      const int64_t k = k0 + 32 * q;
      order[off[q] + b + (lane - leader[q])] = cand ? cand[k] : int32_t(k);
    }
  }
}

// One thread per tile: blocks per tile; an exclusive scan of these gives block ids.
// tile_off indexes bins; tile t spans bins [t S, (t + 1) S)
__global__ void k_block_counts(int T, int S, const int* __restrict__ tile_off, int* blk_cnt) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > T) return;
  blk_cnt[t] = (t == T) ? 0
                        : (tile_off[int64_t(t + 1) * S] - tile_off[int64_t(t) * S] + kEvalThreads - 1) /
                              kEvalThreads;
}

// Block descriptors {first point, end point, tile, 0}; with the tile lists' offsets
// (loff) {first point, end point, list begin, list end}, so the evaluation kernel
// reads its list bounds without a dependent load (lists hold < 2^31 entries).
__global__ void k_block_fill(int T, int S, const int* __restrict__ tile_off,
                             const int* __restrict__ blk_off, const int64_t* __restrict__ loff, int4* blocks,
                             int64_t* nblocks) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) *nblocks = blk_off[T];
  if (t >= T) return;
  const int b0 = blk_off[t], b1 = blk_off[t + 1];
  const int p0 = tile_off[int64_t(t) * S], p1 = tile_off[int64_t(t + 1) * S];
  const int z = loff ? int(loff[t]) : t, w = loff ? int(loff[t + 1]) : 0;
  for (int b = b0; b < b1; ++b) {
    const int s = p0 + (b - b0) * kEvalThreads;
    blocks[b] = make_int4(s, min(s + kEvalThreads, p1), z, w);
  }
}

// ---- K4: opacity evaluation ----------------------------------------------------------------------

#ifndef SOF_EVAL_CHUNK
#define SOF_EVAL_CHUNK 32
#endif
// strategies bit set by eval_views when the schedule was built one view ahead: the
// evaluation re-reads the pruned flag of each scheduled point
constexpr int kRecheckPruned = 1 << 8;
constexpr int kChunk = SOF_EVAL_CHUNK;  // Gaussian records staged in shared memory per step
// CTAs per SM the register budget is set for: the label launch at 9 (56 registers;
// 682 vs 689 ms per C3 label pass at 10 / 48 registers, 691 at 8), the grouped bisection
// at 11 (refine 69.6 ms; 71.3 at 10, 75 at 9, 69.7 at 12)
#ifndef SOF_EVAL_MINB
#define SOF_EVAL_MINB 9
#endif
#ifndef SOF_GROUP_MINB
#define SOF_GROUP_MINB 11
#endif
// Instrumentation counters of k_eval (pairs evaluated in FP64 / contributing): they
// cost registers in the hot loop, so they are compiled in only on request
// (-DSOF_EVAL_STATS=1); the reference's pair counters are always exact.
#ifndef SOF_EVAL_STATS
#define SOF_EVAL_STATS 0
#endif

// Streams a live-only tile list (lp[0, len)) through shared memory in chunks of kChunk
// records and runs eval_chunk(rec*, cnt) -> pairs on each, until every thread of the
// CTA is done. STAGE selects the staging; both give identical results (A/B on C3 in
// DESIGN.md §4):
//   0 (default): every thread copies 16 B of the chunk (index load + record load),
//     two barriers per chunk; srec[0] only;
//   1 (sof_set_staging): TMA row gather — warp 0 issues tile::gather4 over the index
//     list (sof_tma.cuh) into an mbarrier double buffer one chunk ahead, one barrier
//     per chunk. +4% kernel time on C3: the loads were never the bottleneck, and the
//     issue (a uniform-register waterfall over 8 gathers) serialises on warp 0.
// Also measured and dropped: per-lane 1D cp.async.bulk copies (+14%), a register
// double buffer (+6%; with 4 CTAs/SM +8%).
template <int STAGE, typename F>
__device__ __forceinline__ unsigned stream_list(const int32_t* __restrict__ lp, int len, const Rec* __restrict__ recs,
                                                const CUtensorMap* tmap, Rec (*srec)[kChunk], uint64_t* s_bar,
                                                bool& done, F&& eval_chunk) {
  const int nchunks = (len + kChunk - 1) / kChunk;
  auto chunk_cnt = [&](int k) { return min(kChunk, len - k * kChunk); };
  unsigned pairs = 0;
  if constexpr (STAGE == 1) {
    static_assert(kChunk <= 32, "TMA staging issues one row per lane of warp 0");
    const bool warp0 = threadIdx.x < 32;
    auto chunk_row = [&](int k) {  // this lane's list entry of chunk k (0 past the end)
      const int e = k * kChunk + int(threadIdx.x & 31);
      return e < len ? lp[e] : 0;
    };
    if (threadIdx.x == 0) {
      mbar_init(&s_bar[0], 1);
      mbar_init(&s_bar[1], 1);
      mbar_fence_init();
    }
    __syncthreads();
    int next_row = 0;  // warp 0: list entry of chunk k + 1 held one chunk ahead
    if (warp0 && nchunks > 0) {
      tma_issue_rows(srec[0], tmap, chunk_row(0), chunk_cnt(0), &s_bar[0], sizeof(Rec));
      next_row = chunk_row(1);
    }
    int k = 0;
    for (; k < nchunks; ++k) {
      // all threads are past chunk k - 1: its buffer may be refilled with chunk k + 1
      if (!__syncthreads_or(!done)) break;
      if (warp0 && k + 1 < nchunks) {
        tma_issue_rows(srec[(k + 1) & 1], tmap, next_row, chunk_cnt(k + 1), &s_bar[(k + 1) & 1], sizeof(Rec));
        next_row = chunk_row(k + 2);
      }
      if (done) continue;
      mbar_wait(&s_bar[k & 1], (k >> 1) & 1);
      pairs += eval_chunk(srec[k & 1], chunk_cnt(k));
    }
    // early exit: chunk k was issued but never waited on; the CTA's shared memory must
    // not be released while the copy is in flight
    if (k < nchunks && threadIdx.x == 0) mbar_wait(&s_bar[k & 1], (k >> 1) & 1);
  } else {
    for (int k = 0; k < nchunks; ++k) {
      if (!__syncthreads_or(!done)) break;
      const int cnt = chunk_cnt(k);
      for (int q8 = threadIdx.x; q8 < cnt * kRecV2; q8 += blockDim.x) {
        const int r = q8 / kRecV2, q = q8 % kRecV2;
        reinterpret_cast<double2*>(&srec[0][r])[q] =
            __ldg(reinterpret_cast<const double2*>(recs + lp[k * kChunk + r]) + q);
      }
      __syncthreads();
      if (!done) pairs += eval_chunk(srec[0], cnt);
    }
  }
  return pairs;
}

// The min-z break of a chunk (field_eval.hpp:90-93): records are sorted by min_z, so
// the scan of a chunk stops at the first record with min_z > z_point. One FP64 compare
// against the chunk's last record rules the break out for the whole chunk; otherwise a
// binary search finds it. The loop then runs up to that index without per-record min_z
// tests (same pairs, same break, fewer instructions on the culled path).
__device__ __forceinline__ int chunk_limit(const Rec* rp, int cnt, double zp, bool& brk) {
  brk = false;
  if (cnt <= 0 || !(rp[cnt - 1].zmin > zp)) return cnt;
  int lo = 0, hi = cnt - 1;  // the first index with min_z > zp lies in [lo, hi]
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rp[mid].zmin > zp)
      hi = mid;
    else
      lo = mid + 1;
  }
  brk = true;
  return lo;
}

// The reference loop (field_eval.hpp:86-108) over one staged chunk of a live-only,
// min_z-sorted list: records up to the chunk's break are culled by the screen-space conic
// or evaluated exactly by eval_one (which returns true on the early stop). Returns the
// pairs counted; sets done at the min-z break or the early stop. SOF_PAIR_CULL tests two
// records' conics per step (both culled: one branch for the pair).
#ifndef SOF_PAIR_CULL
#define SOF_PAIR_CULL 1
#endif
// stop: the chunk position of the record at which the early stop happened (else -1).
// QUAD: four conics per step first (the grouped bisection: 73 -> 71 ms per C3 step; the
// label launch is faster with two, 688 vs 696 ms)
template <bool QUAD = false, typename F>
__device__ __forceinline__ unsigned scan_chunk(const Rec* rp, int cnt, double zp, float cu, float cv, float cuu,
                                               float cvv, float cuv, bool& done, int& stop, F&& eval_one) {
  bool brk;
  const int lim = chunk_limit(rp, cnt, zp, brk);
  int e = 0;
  if constexpr (QUAD) {
    for (; e + 3 < lim; e += 4) {
      const bool cs[4] = {conic_culls(rp[e], cu, cv, cuu, cvv, cuv), conic_culls(rp[e + 1], cu, cv, cuu, cvv, cuv),
                          conic_culls(rp[e + 2], cu, cv, cuu, cvv, cuv), conic_culls(rp[e + 3], cu, cv, cuu, cvv, cuv)};
      if (cs[0] && cs[1] && cs[2] && cs[3]) continue;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (!cs[u] && eval_one(rp[e + u])) {
          done = true;
          stop = e + u;
          return unsigned(e + u + 1);
        }
    }
  }
#if SOF_PAIR_CULL
  for (; e + 1 < lim; e += 2) {
    const bool c0 = conic_culls(rp[e], cu, cv, cuu, cvv, cuv);
    const bool c1 = conic_culls(rp[e + 1], cu, cv, cuu, cvv, cuv);
    if (c0 && c1) continue;
    if (!c0 && eval_one(rp[e])) {
      done = true;
      stop = e;
      return unsigned(e + 1);
    }
    if (!c1 && eval_one(rp[e + 1])) {
      done = true;
      stop = e + 1;
      return unsigned(e + 2);
    }
  }
#endif
  for (; e < lim; ++e) {
    if (conic_culls(rp[e], cu, cv, cuu, cvv, cuv)) continue;  // alpha < 1/255 for sure
    if (eval_one(rp[e])) {
      done = true;
      stop = e;
      return unsigned(e + 1);  // this pair was counted
    }
  }
  if (brk) done = true;  // the record at lim ends the sorted scan (not counted)
  return unsigned(lim);
}

// The view's counted Gaussians (Binding::nb: behind the camera, or crossing its plane),
// sorted by (min_z key, index), and the list positions of the crossing ones that are
// listed in some tiles (Binding::xpos).
struct Behind {
  const uint64_t* key;
  const int32_t* idx;  // 2 g (2 row / 2 row - 1 in a truncated binding)
  int64_t n;
  const int64_t* xpos;
  int64_t nx;
};

// Pairs the reference counts for a point whose scan of the listed entries processed the
// positions [l0, l0 + P) of its tile list, beyond those P. The reference's list holds
// every counted Gaussian; its scan processes them in (min_z, index) order up to the early
// stop at the listed entry (stop_key, stop_cmp = 2 * its index/row) inclusive, or else up
// to the min-z break: all with min_z <= z_point (field_eval.hpp:86-108). Listed crossing
// entries among the processed positions are already in P and are taken off again.
__device__ __forceinline__ int count_pairs(const Behind& bh, bool stopped, uint64_t stop_key, int32_t stop_cmp,
                                           double zp, int64_t l0, unsigned P) {
  int add = 0;
  if (bh.n > 0) {
    const uint64_t K = stopped ? stop_key : double_key(zp);
    const int32_t I = stopped ? stop_cmp : INT_MAX;
    int64_t lo = 0, hi = bh.n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const uint64_t k = __ldg(bh.key + mid);
      if (k < K || (k == K && __ldg(bh.idx + mid) <= I)) lo = mid + 1;
      else hi = mid;
    }
    add = int(lo);
  }
  if (bh.nx > 0 && P > 0) {
    auto lower = [&](int64_t x) {
      int64_t lo = 0, hi = bh.nx;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(bh.xpos + mid) < x) lo = mid + 1;
        else hi = mid;
      }
      return lo;
    };
    add -= int(lower(l0 + P) - lower(l0));
  }
  return add;
}

// One CTA = one schedule block (<= 256 points of one tile). The block's Gaussian
// list is streamed through shared memory in chunks; every thread runs the exact
// view_opacity loop (field_eval.hpp:86-108) for its point.
//
// FAST (tile lists + min-z + dead cull, the default strategies): the lists are
// live-only (Binding::live), so the loop has no per-record strategy tests, and the
// chunks are gathered by TMA (tile::gather4 over the index list, sof_tma.cuh) into a
// double buffer: warp 0 issues chunk k + 1 right after the barrier that frees its
// buffer, and the CTA evaluates chunk k meanwhile. One barrier per chunk (it also
// detects the all-done early exit).
template <int MODE, bool TILED, bool FAST, int STAGE = 0>
__global__ void __launch_bounds__(kEvalThreads, SOF_EVAL_MINB) k_eval(
    const int4* __restrict__ blocks, const int64_t* __restrict__ nblocks,
    const int32_t* __restrict__ pidx, const double* __restrict__ xyz, Cam cam, int ts,
    int tiles_x, const int64_t* __restrict__ loff, const int32_t* __restrict__ lent,
    int64_t n_gauss, const Rec* __restrict__ recs, int strategies, int classify, double* min_op,
    uint8_t* ext, double* o_out, uint8_t* obs_out, uint8_t* comp_out,
    unsigned long long* pairs_counter, const __grid_constant__ CUtensorMap tmap, Behind bh) {
  static_assert(!FAST || TILED, "the fast loop relies on min_z-sorted tile lists");
  __shared__ __align__(128) Rec srec[STAGE == 1 ? 2 : 1][kChunk];
  __shared__ __align__(16) double s_exp[128];  // sof_exp's table (shared-memory latency)
  __shared__ __align__(8) uint64_t s_bar[2];
  const int64_t b = blockIdx.x;
  if (b >= *nblocks) return;
  const int4 blk = blocks[b];
  const int j = blk.x + int(threadIdx.x);
  bool active = j < blk.y;
  int i = 0;
  PointRay pr;
  pr.observed = false;
  double m_prev = 0.0;  // min_op[i], loaded up front so its latency hides behind the loop
  if (active) {
    i = pidx[j];
    if (MODE == kModeLabel || MODE == kModeValue) m_prev = min_op[i];
    // the schedule is built one view ahead (eval_views): a point the previous view's
    // evaluation pruned may still be listed; the reference skips it (field_eval.hpp:147)
    const bool pruned = (MODE == kModeLabel || MODE == kModeClassify) && (strategies & kRecheckPruned) && ext[i];
    pr = point_ray(cam, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], ts, tiles_x);
    active = !pruned;
  }
  int64_t l0 = 0, l1 = n_gauss;
  if (TILED) {  // list bounds carried by the block descriptor (k_block_fill)
    l0 = blk.z;
    l1 = blk.w;
  }
  (void)loff;
  const bool dead_cull = strategies & 16, use_min_z = strategies & 2;
  const bool early = classify && (strategies & 4);
  const float cu = float(pr.px), cv = float(pr.py);
  const float cuu = cu * cu, cvv = cv * cv, cuv = cu * cv;
  double survive = 1.0;
  bool complete = true;
  bool done = !active;
  unsigned pairs = 0, exact = 0, contrib = 0, scanned = 0;
  for (int q = threadIdx.x; q < 128; q += blockDim.x) s_exp[q] = kSofExpTabDev[q];
  if constexpr (FAST) {
    const int32_t* lp = lent + l0;
    const int len = int(l1 - l0);  // tile lists hold < 2^31 entries
    // the exact reference loop over one staged chunk; returns the pairs it counted
    auto eval_one = [&](const Rec& r) {
      if (SOF_EVAL_STATS) ++exact;
      const double alpha = pair_alpha(r, pr.d, pr.t, SofExpSmem{smem_u32(s_exp)});
      if (alpha == 0.0) return false;
      if (SOF_EVAL_STATS) ++contrib;
      survive *= 1.0 - alpha;
      if (early && 1.0 - survive > 0.5) {
        complete = false;
        return true;
      }
      return false;
    };
    int chunk_no = 0, stop = -1;
    uint64_t stop_key = 0;
    int32_t stop_idx = -1;
    auto eval_chunk = [&](const Rec* rp, int cnt) {
      const unsigned p = scan_chunk(rp, cnt, pr.zp, cu, cv, cuu, cvv, cuv, done, stop, eval_one);
      if (stop >= 0 && bh.n > 0 && stop_idx < 0) {  // where the early stop happened, for count_pairs
        stop_key = double_key(rp[stop].zmin);
        stop_idx = 2 * lp[chunk_no * kChunk + stop];
      }
      ++chunk_no;
      return p;
    };
    pairs += stream_list<STAGE>(lp, len, recs, &tmap, srec, s_bar, done, eval_chunk);
    scanned = pairs;
    if (active) pairs += count_pairs(bh, stop >= 0, stop_key, stop_idx, pr.zp, l0, pairs);
  } else {
    for (int64_t base = l0; base < l1; base += kChunk) {
      if (!__syncthreads_or(!done)) break;
      const int cnt = int(std::min<int64_t>(kChunk, l1 - base));
      for (int k = threadIdx.x; k < cnt * kRecV2; k += blockDim.x) {
        const int r = k / kRecV2, q = k % kRecV2;
        const int64_t g = TILED ? int64_t(lent[base + r]) : base + r;
        reinterpret_cast<double2*>(&srec[0][r])[q] = __ldg(reinterpret_cast<const double2*>(recs + g) + q);
      }
      __syncthreads();
      if (done) continue;
      for (int k = 0; k < cnt; ++k) {
        const Rec& r = srec[0][k];
        if (dead_cull && r.op < kMinAlpha) continue;
        if (use_min_z && r.zmin > pr.zp) {
          if (TILED) {  // list sorted by min_z (field_eval.hpp:91)
            done = true;
            break;
          }
          continue;
        }
        ++pairs;
        if (conic_culls(r, cu, cv, cuu, cvv, cuv)) continue;  // alpha < 1/255 for sure
        if (SOF_EVAL_STATS) ++exact;
        const double alpha = pair_alpha(r, pr.d, pr.t, SofExpSmem{smem_u32(s_exp)});
        if (alpha == 0.0) continue;
        if (SOF_EVAL_STATS) ++contrib;
        survive *= 1.0 - alpha;
        if (early && 1.0 - survive > 0.5) {
          complete = false;
          done = true;
          break;
        }
      }
    }
  }
  if (active) {
    const double o = 1.0 - survive;
    if (MODE == kModeLabel || MODE == kModeValue) {
      min_op[i] = (o < m_prev) ? o : m_prev;
      if (MODE == kModeLabel && complete && o < 0.5) ext[i] = 1;
    } else if (MODE == kModeClassify) {
      if (complete && o < 0.5) ext[i] = 1;
    } else {
      o_out[i] = o;
      obs_out[i] = 1;
      comp_out[i] = complete;
    }
  }
  // pairs counter: warp reduce, one atomic per warp
  // pairs, point_view_evals, FP64 evals, contributing evals
  unsigned long long p = pairs, q = active, e = exact, w = contrib;
  for (int s = 16; s > 0; s >>= 1) {
    w += __shfl_down_sync(0xffffffffu, w, s);
    p += __shfl_down_sync(0xffffffffu, p, s);
    q += __shfl_down_sync(0xffffffffu, q, s);
    e += __shfl_down_sync(0xffffffffu, e, s);
  }
  if ((threadIdx.x & 31) == 0) {
    if (p) atomicAdd(pairs_counter, p);
    if (q) atomicAdd(pairs_counter + 1, q);
    if (e) atomicAdd(pairs_counter + 2, e);
    if (w) atomicAdd(pairs_counter + 3, w);
  }
  if (FAST && bh.n > 0) {  // views with counted Gaussians: the list entries actually scanned
    unsigned long long sc = scanned;
    for (int s = 16; s > 0; s >>= 1) sc += __shfl_down_sync(0xffffffffu, sc, s);
    if ((threadIdx.x & 31) == 0 && sc) atomicAdd(pairs_counter + 4, sc);
  }
}

// FP32-filtered evaluation: same semantics and bit-identical results as k_eval.
// Per chunk of kChunkF records staged in shared memory (float copies), every
// thread scans the chunk in FP32 and queues the pairs the certified filter
// cannot skip (RecF, sof_device.cuh); the queue is then replayed in list order
// with the exact FP64 pair arithmetic (pair_alpha) reading the FP64 record from
// global memory. The survive product, early stop and min-z break are exact, and
// the reference's pair counter is reproduced from per-pair ordinals.
constexpr int kChunkF = 64;

template <int MODE, bool TILED>
__global__ void __launch_bounds__(256) k_eval_f32(
    const int4* __restrict__ blocks, const int64_t* __restrict__ nblocks,
    const int32_t* __restrict__ pidx, const double* __restrict__ xyz, Cam cam, int ts,
    int tiles_x, const int64_t* __restrict__ loff, const int32_t* __restrict__ lent,
    int64_t n_gauss, const Rec* __restrict__ recs, const RecF* __restrict__ recf, int strategies,
    int classify, double* min_op, uint8_t* ext, double* o_out, uint8_t* obs_out,
    uint8_t* comp_out, unsigned long long* counters) {
  __shared__ __align__(16) RecF sf[kChunkF];
  __shared__ int32_t sg[kChunkF];
  __shared__ uint8_t qk[kChunkF][256];  // queued record (chunk index) per thread
  __shared__ uint8_t qo[kChunkF][256];  // pair ordinal of the queued record in the chunk
  const int64_t b = blockIdx.x;
  if (b >= *nblocks) return;
  const int4 blk = blocks[b];
  const int tid = threadIdx.x;
  const int j = blk.x + tid;
  bool active = j < blk.y;
  int i = 0;
  PointRay pr;
  pr.observed = false;
  pr.zp = 0.0;
  pr.t = 1.0;
  pr.d[0] = pr.d[1] = pr.d[2] = 0.0;
  if (active) {
    i = pidx[j];
    // schedule built one view ahead: skip points pruned since (as k_eval)
    if ((MODE == kModeLabel || MODE == kModeClassify) && (strategies & kRecheckPruned) && ext[i])
      active = false;
    else
      pr = point_ray(cam, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], ts, tiles_x);
  }
  // per-point float monomials of the ray direction (abc_cached precompute.hpp:39-45)
  const float x = float(pr.d[0]), y = float(pr.d[1]), z = float(pr.d[2]);
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
  const float tf = float(pr.t);
  const float zpf = __double2float_rn(pr.zp);
  int64_t l0 = 0, l1 = n_gauss;
  if (TILED) {
    l0 = blk.z;
    l1 = blk.w;
  }
  (void)loff;
  const bool dead_cull = strategies & 16, use_min_z = strategies & 2;
  const bool early = classify && (strategies & 4);
  double survive = 1.0;
  bool complete = true;
  bool done = !active;
  unsigned pairs = 0, exact_evals = 0;
  for (int64_t base = l0; base < l1; base += kChunkF) {
    if (!__syncthreads_or(!done)) break;
    const int cnt = int(min(int64_t(kChunkF), l1 - base));
    for (int k = tid; k < cnt * 4; k += blockDim.x) {
      const int r = k >> 2, q = k & 3;
      const int32_t g = TILED ? lent[base + r] : int32_t(base + r);
      reinterpret_cast<float4*>(&sf[r])[q] = __ldg(reinterpret_cast<const float4*>(recf + g) + q);
      if (q == 0) sg[r] = g;
    }
    __syncthreads();
    if (!done) {
      int qn = 0, np = 0;
      bool brk = false;
      for (int k = 0; k < cnt; ++k) {
        const RecF& r = sf[k];
        if (dead_cull && (r.flags & 1u)) continue;
        if (use_min_z) {
          // exact `min_z > z_point`: float compare, FP64 only on a float tie
          const bool gt = (r.zmin > zpf) || (r.zmin == zpf && __ldg(&recs[sg[k]].zmin) > pr.zp);
          if (gt) {
            if (TILED) {  // list sorted by min_z (field_eval.hpp:91)
              brk = true;
              break;
            }
            continue;
          }
        }
        ++np;
        const float bb = fmaf(r.b2[0], x, fmaf(r.b2[1], y, r.b2[2] * z));
        if (bb >= r.kb) continue;  // b_fp64 >= 0: te <= 0, skipped by the reference
        const float a = fmaf(r.ic[0], xx, fmaf(r.ic[1], yy, fmaf(r.ic[2], zz,
                        fmaf(r.ic[3], xy, fmaf(r.ic[4], xz, r.ic[5] * yz)))));
        bool need = !(a > r.ka);
        if (!need) {
          const float ra = __frcp_rn(a);
          const float tst = -0.5f * bb * ra;
          const float te = fminf(tst, tf);
          const float g = fmaf(fmaf(a, te, bb), te, r.c);
          // |g_f - g_fp64| <= ka te^2 + kb |te| + kc + kb^2 / a (the last term bounds the
          // second-order effect of the t* error, a (dt*)^2 <= db^2 / (4a))
          const float s = fmaf(r.ka, te * te, fmaf(r.kb, fabsf(te) + r.kb * ra, r.kc));
          need = !(g - s > r.gthr);  // otherwise alpha_fp64 < 1/255 for sure
        }
        if (need) {
          qk[qn][tid] = uint8_t(k);
          qo[qn][tid] = uint8_t(np);
          ++qn;
        }
      }
      // exact replay of the queued pairs, in list order
      int stop = -1;
      for (int q = 0; q < qn; ++q) {
        const int k = qk[q][tid];
        const Rec r = recs[sg[k]];
        ++exact_evals;
        const double alpha = pair_alpha(r, pr.d, pr.t);
        if (alpha == 0.0) continue;
        survive *= 1.0 - alpha;
        if (early && 1.0 - survive > 0.5) {
          complete = false;
          stop = qo[q][tid];
          break;
        }
      }
      if (stop >= 0) {
        pairs += unsigned(stop);
        done = true;
      } else {
        pairs += unsigned(np);
        if (brk) done = true;
      }
    }
  }
  if (active) {
    const double o = 1.0 - survive;
    if (MODE == kModeLabel || MODE == kModeValue) {
      const double m = min_op[i];
      min_op[i] = (o < m) ? o : m;
      if (MODE == kModeLabel && complete && o < 0.5) ext[i] = 1;
    } else if (MODE == kModeClassify) {
      if (complete && o < 0.5) ext[i] = 1;
    } else {
      o_out[i] = o;
      obs_out[i] = 1;
      comp_out[i] = complete;
    }
  }
  unsigned long long p = pairs, q = active, e = exact_evals;
  for (int s = 16; s > 0; s >>= 1) {
    p += __shfl_down_sync(0xffffffffu, p, s);
    q += __shfl_down_sync(0xffffffffu, q, s);
    e += __shfl_down_sync(0xffffffffu, e, s);
  }
  if ((threadIdx.x & 31) == 0) {
    if (p) atomicAdd(counters, p);
    if (q) atomicAdd(counters + 1, q);
    if (e) atomicAdd(counters + 2, e);
  }
}

__global__ void k_fill_view_outputs(int64_t n, double* o, uint8_t* obs, uint8_t* comp) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  o[i] = 1.0;
  obs[i] = 0;
  comp[i] = 1;
}

// ---- grouped classification (binary_search_refine's classify_point over many views) ---------------
//
// The bisection classifies the same midpoints against every view (field_eval.hpp:114-125).
// Per view the schedule + evaluation is only ~100 us of work, so per-view launches were
// dominated by launch overhead. Here a group of up to kGroupViews views is scheduled and
// evaluated at once: bins are (view, tile), every (midpoint, view) item is evaluated
// exactly as k_eval does, and k_group_fixup then applies the reference's per-point view
// order: views are visited in order and, under prune, the first exterior view ends the
// visit (field_eval.hpp:121), so later items of that point neither count pairs nor
// matter. Items evaluated after a point's first exterior view are wasted work only
// (a few percent: interior midpoints are evaluated in every view anyway).

#ifndef SOF_GROUP_VIEWS
#define SOF_GROUP_VIEWS 32
#endif
constexpr int kGroupViews = SOF_GROUP_VIEWS;  // views scheduled and evaluated per grouped launch

struct GroupTables {
  int g0, G;
  int64_t bin_base[kGroupViews + 1];  // first bin of each view of the group
};

template <int TS>  // 16: the default tile size as a compile-time constant (see k_sched_tile)
__global__ void k_sched_group(int64_t n, const double* __restrict__ xyz, const Cam* __restrict__ cams, int ts,
                              GroupTables gt, const uint8_t* __restrict__ skip, int32_t* item_bin, int* bin_cnt) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const bool live = k < n && !(skip && skip[k]);
  double x0 = 0.0, x1 = 0.0, x2 = 0.0;
  if (live) {
    x0 = xyz[3 * k];
    x1 = xyz[3 * k + 1];
    x2 = xyz[3 * k + 2];
  }
  for (int j = 0; j < gt.G; ++j) {
    int bin = -1;
    if (live) {
      const Cam& cam = cams[gt.g0 + j];
      const int tiles_x = (TS == 16) ? (cam.w + 15) >> 4 : (cam.w + ts - 1) / ts;
      const PointTile pt = point_tile<TS>(cam, x0, x1, x2, ts, tiles_x);
      if (pt.tile >= 0) bin = int(gt.bin_base[j]) + pt.tile;
    }
    if (k < n) item_bin[int64_t(j) * n + k] = bin;
    warp_tile_add(bin_cnt, bin, bin >= 0);
  }
}

__global__ void k_scatter_group(int64_t n, int G, const int32_t* __restrict__ item_bin,
                                const int* __restrict__ bin_off, int* bin_cur, int32_t* order) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  for (int j = 0; j < G; ++j) {
    const int bin = (k < n) ? item_bin[int64_t(j) * n + k] : -1;
    const int slot = warp_tile_add(bin_cur, bin, bin >= 0);
    if (bin >= 0) order[bin_off[bin] + slot] = int32_t(int64_t(j) * n + k);
  }
}

// k_eval's fast loop (default strategies, classify mode) over the items of a group:
// block.z is a (view, tile) bin; the view's camera, records and tile lists come from
// device tables. Writes the per-item pair count and exterior flag.
template <int STAGE>
__global__ void __launch_bounds__(kEvalThreads, SOF_GROUP_MINB) k_eval_group(
    const int4* __restrict__ blocks, const int64_t* __restrict__ nblocks, const int32_t* __restrict__ items,
    int64_t n, const double* __restrict__ xyz, const Cam* __restrict__ cams, int ts, GroupTables gt,
    const int64_t* const* __restrict__ loffs, const int32_t* const* __restrict__ lents,
    const Rec* const* __restrict__ recs_v, const CUtensorMap* __restrict__ tmaps, bool early,
    uint32_t* item_pairs, uint8_t* item_ext,
    unsigned long long* counters, const uint64_t* const* __restrict__ bkeys,
    const int32_t* const* __restrict__ bidxs, const int64_t* __restrict__ nbeh,
    const int64_t* const* __restrict__ xposs, const int64_t* __restrict__ nxs) {
  __shared__ __align__(128) Rec srec[STAGE == 1 ? 2 : 1][kChunk];
  __shared__ __align__(16) double s_exp[128];
  __shared__ __align__(8) uint64_t s_bar[2];
  const int64_t b = blockIdx.x;
  if (b >= *nblocks) return;
  const int4 blk = blocks[b];
  int j = 0;
  while (j + 1 < gt.G && gt.bin_base[j + 1] <= blk.z) ++j;
  const int v = gt.g0 + j;
  const int tile = blk.z - int(gt.bin_base[j]);
  const Cam cam = cams[v];
  const CUtensorMap* tmap = tmaps + v;
  const Rec* recs = recs_v[v];
  const int32_t* __restrict__ lent = lents[v];
  const int tiles_x = (cam.w + ts - 1) / ts;
  const int p = blk.x + int(threadIdx.x);
  const bool active = p < blk.y;
  int64_t item = 0, k = 0;
  PointRay pr;
  pr.observed = false;
  pr.zp = 0.0;
  if (active) {
    item = items[p];
    k = item - int64_t(j) * n;
    pr = point_ray(cam, xyz[3 * k], xyz[3 * k + 1], xyz[3 * k + 2], ts, tiles_x);
  }
  const int64_t l0 = loffs[v][tile], l1 = loffs[v][tile + 1];
  const float cu = float(pr.px), cv = float(pr.py);
  const float cuu = cu * cu, cvv = cv * cv, cuv = cu * cv;
  double survive = 1.0;
  bool complete = true;
  bool done = !active;
  unsigned pairs = 0, exact = 0, contrib = 0;
  for (int q = threadIdx.x; q < 128; q += blockDim.x) s_exp[q] = kSofExpTabDev[q];
  // k_eval's fast loop over the live-only list (stream_list); with TMA staging the
  // tensor maps live in global memory, written by a host copy before the launch
  if (STAGE == 1 && threadIdx.x < 32) tma_fence_acquire(tmap);
  auto eval_one = [&](const Rec& r) {
    if (SOF_EVAL_STATS) ++exact;
    const double alpha = pair_alpha(r, pr.d, pr.t, SofExpSmem{smem_u32(s_exp)});
    if (alpha == 0.0) return false;
    if (SOF_EVAL_STATS) ++contrib;
    survive *= 1.0 - alpha;
    if (early && 1.0 - survive > 0.5) {
      complete = false;
      return true;
    }
    return false;
  };
  const Behind bh{bkeys[v], bidxs[v], nbeh[v], xposs[v], nxs[v]};
  const int32_t* lp = lent + l0;
  int chunk_no = 0, stop = -1;
  uint64_t stop_key = 0;
  int32_t stop_idx = -1;
  auto eval_chunk = [&](const Rec* rp, int cnt) {
    const unsigned p = scan_chunk<true>(rp, cnt, pr.zp, cu, cv, cuu, cvv, cuv, done, stop, eval_one);
    if (stop >= 0 && bh.n > 0 && stop_idx < 0) {
      stop_key = double_key(rp[stop].zmin);
      stop_idx = 2 * lp[chunk_no * kChunk + stop];
    }
    ++chunk_no;
    return p;
  };
  pairs += stream_list<STAGE>(lp, int(l1 - l0), recs, tmap, srec, s_bar, done, eval_chunk);
  unsigned long long sc = pairs;
  if (active) pairs += count_pairs(bh, stop >= 0, stop_key, stop_idx, pr.zp, l0, pairs);
  if (active) {
    item_pairs[item] = pairs;
    item_ext[item] = (complete && 1.0 - survive < 0.5) ? 1 : 0;
  }
  if (bh.n > 0) {  // views with counted Gaussians: the list entries actually scanned
    for (int s = 16; s > 0; s >>= 1) sc += __shfl_down_sync(0xffffffffu, sc, s);
    if ((threadIdx.x & 31) == 0 && sc) atomicAdd(counters + 4, sc);
  }
  if (SOF_EVAL_STATS) {
    unsigned long long e = exact, w = contrib;
    for (int s = 16; s > 0; s >>= 1) {
      e += __shfl_down_sync(0xffffffffu, e, s);
      w += __shfl_down_sync(0xffffffffu, w, s);
    }
    if ((threadIdx.x & 31) == 0) {
      if (e) atomicAdd(counters + 2, e);
      if (w) atomicAdd(counters + 3, w);
    }
  }
}

// The reference's view order per midpoint: counters of every observed view up to the
// first exterior one (all of them without prune), exterior = any.
__global__ void k_group_fixup(int64_t n, int G, bool prune, const int32_t* __restrict__ item_bin,
                              const uint32_t* __restrict__ item_pairs, const uint8_t* __restrict__ item_ext,
                              uint8_t* ext, unsigned long long* counters) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  unsigned long long pairs = 0, pve = 0;
  if (k < n && !(prune && ext[k])) {
    bool ex = false;
    for (int j = 0; j < G; ++j) {
      const int64_t it = int64_t(j) * n + k;
      if (item_bin[it] < 0) continue;  // not observed (or skipped)
      ++pve;
      pairs += item_pairs[it];
      if (item_ext[it]) {
        ex = true;
        if (prune) break;
      }
    }
    if (ex) ext[k] = 1;
  }
  for (int s = 16; s > 0; s >>= 1) {
    pairs += __shfl_down_sync(0xffffffffu, pairs, s);
    pve += __shfl_down_sync(0xffffffffu, pve, s);
  }
  if ((threadIdx.x & 31) == 0) {
    if (pairs) atomicAdd(counters, pairs);
    if (pve) atomicAdd(counters + 1, pve);
  }
}

// Bisection classification of n points (ext[k] = exterior) over views [v0, v1) in
// groups; false when the grouped path does not apply (then eval_views runs per view).
static bool view_resident(const sof_ctx* c, int v, int tile_size) {
  const Binding& b = c->bindings[v];
  return c->rec_valid[v] && b.view == v && b.tile_size == tile_size && b.live;
}

static bool classify_grouped_run(sof_ctx* c, int v0, int v1, int64_t n, const double* xyz, int strategies,
                                 int tile_size, uint8_t* ext, uint64_t* counters_host);

// Classification over views [v0, v1) in view order: maximal runs of views whose records
// and live tile lists are resident go through the grouped kernels, the other views
// (past the cache budget) through the per-view path. Processing stays in view order, so
// pruning and the counters follow the reference's sequential visit (field_eval.hpp:114-125).
static bool classify_grouped(sof_ctx* c, int v0, int v1, int64_t n, const double* xyz, int strategies,
                             int tile_size, uint8_t* ext, uint64_t* counters_host) {
  if (c->eval_path != 1 || (strategies & 19) != 19 || n <= 0 || v1 <= v0) return false;
  if (std::getenv("SOF_NO_GROUPED")) return false;
  bool run = false;  // at least two consecutive resident views
  for (int v = v0; v + 1 < v1 && !run; ++v) run = view_resident(c, v, tile_size) && view_resident(c, v + 1, tile_size);
  if (!run) return false;
  for (int v = v0; v < v1;) {
    int e = v;
    while (e < v1 && view_resident(c, e, tile_size)) ++e;
    if (e > v && classify_grouped_run(c, v, e, n, xyz, strategies, tile_size, ext, counters_host)) {
      v = e;
      continue;
    }
    const int stop = (e > v) ? e : v + 1;  // a run the grouped path declined, or one view
    for (; v < stop; ++v)
      eval_views(c, v, v + 1, n, xyz, strategies, tile_size, true, kModeClassify, nullptr, ext, nullptr, nullptr,
                 nullptr, counters_host);
  }
  return true;
}

static bool classify_grouped_run(sof_ctx* c, int v0, int v1, int64_t n, const double* xyz, int strategies,
                                 int tile_size, uint8_t* ext, uint64_t* counters_host) {
  const int V = int(c->cams.size());
  const int G = std::min(kGroupViews, v1 - v0);
  if (int64_t(G) * n >= (int64_t(1) << 31)) return false;
  std::vector<const void*> ptrs(6 * size_t(V), nullptr);
  std::vector<int64_t> nbeh(2 * size_t(V), 0);  // [V] counted Gaussians, [V] listed crossing positions
  for (int v = v0; v < v1; ++v) {
    const Binding& bd = c->bindings[v];
    ptrs[v] = bd.off.p;
    ptrs[V + v] = bd.ent.p;
    ptrs[2 * V + v] = c->recs[v].p;
    ptrs[3 * V + v] = bd.nb ? bd.bkey.p : nullptr;
    ptrs[4 * V + v] = bd.nb ? bd.bidx.p : nullptr;
    ptrs[5 * V + v] = bd.nx ? bd.xpos.p : nullptr;
    nbeh[v] = bd.nb;
    nbeh[V + v] = bd.nx;
  }
  GroupScratch& g = c->grp;
  g.cams.ensure(V);
  g.ptrs.ensure(6 * V);
  g.nbeh.ensure(2 * V);
  SOF_CUDA(cudaMemcpyAsync(g.cams.p, c->cams.data(), sizeof(Cam) * V, cudaMemcpyHostToDevice, c->stream));
  SOF_CUDA(cudaMemcpyAsync(g.ptrs.p, ptrs.data(), sizeof(void*) * 6 * V, cudaMemcpyHostToDevice, c->stream));
  SOF_CUDA(cudaMemcpyAsync(g.nbeh.p, nbeh.data(), sizeof(int64_t) * 2 * V, cudaMemcpyHostToDevice, c->stream));
  if (c->staging == 1) {  // TMA staging: one tensor map per view's record array
    std::vector<CUtensorMap> tmaps(static_cast<size_t>(V));
    std::memset(tmaps.data(), 0, sizeof(CUtensorMap) * size_t(V));
    for (int v = v0; v < v1; ++v)
      if (sof_make_row_tmap(&tmaps[v], c->recs[v].p, c->bindings[v].trunc ? c->bindings[v].rows : c->n) != 0)
        throw StateError("cuTensorMapEncodeTiled failed for the records");
    g.tmaps.ensure(V);
    SOF_CUDA(cudaMemcpyAsync(g.tmaps.p, tmaps.data(), sizeof(CUtensorMap) * V, cudaMemcpyHostToDevice, c->stream));
  }
  g.item_bin.ensure(int64_t(G) * n);
  g.item_pairs.ensure(int64_t(G) * n);
  g.item_ext.ensure(int64_t(G) * n);
  g.order.ensure(int64_t(G) * n);
  c->d_counters.ensure(5);
  c->d_scalar.ensure(4);
  zero_async(c, c->d_counters.p, int64_t(sizeof(unsigned long long)) * 5);
  const bool prune = strategies & 8, early = strategies & 4;
  const int64_t* const* loffs = reinterpret_cast<const int64_t* const*>(g.ptrs.p);
  const int32_t* const* lents = reinterpret_cast<const int32_t* const*>(g.ptrs.p + V);
  const Rec* const* recs = reinterpret_cast<const Rec* const*>(g.ptrs.p + 2 * V);
  const uint64_t* const* bkeys = reinterpret_cast<const uint64_t* const*>(g.ptrs.p + 3 * V);
  const int32_t* const* bidxs = reinterpret_cast<const int32_t* const*>(g.ptrs.p + 4 * V);
  const int64_t* const* xposs = reinterpret_cast<const int64_t* const*>(g.ptrs.p + 5 * V);
  for (int g0 = v0; g0 < v1; g0 += G) {
    GroupTables gt;
    gt.g0 = g0;
    gt.G = std::min(G, v1 - g0);
    gt.bin_base[0] = 0;
    for (int j = 0; j < gt.G; ++j) {
      const Cam& cam = c->cams[g0 + j];
      const int64_t T = int64_t((cam.w + tile_size - 1) / tile_size) * ((cam.h + tile_size - 1) / tile_size);
      gt.bin_base[j + 1] = gt.bin_base[j] + T;
    }
    const int64_t NB = gt.bin_base[gt.G];
    PointSchedule& s = c->sched;
    s.tile_cnt.ensure(2 * (NB + 1));
    s.tile_off.ensure(NB + 1);
    s.blk_cnt.ensure(NB + 1);
    s.blk_off.ensure(NB + 1);
    zero_async(c, s.tile_cnt.p, int64_t(sizeof(int)) * 2 * (NB + 1));
    int* cur = s.tile_cnt.p + (NB + 1);
    const uint8_t* skip = prune ? ext : nullptr;
    if (tile_size == 16)
      k_sched_group<16><<<grid_for(n, 256), 256, 0, c->stream>>>(n, xyz, g.cams.p, tile_size, gt, skip, g.item_bin.p,
                                                           s.tile_cnt.p);
    else
      k_sched_group<0><<<grid_for(n, 256), 256, 0, c->stream>>>(n, xyz, g.cams.p, tile_size, gt, skip, g.item_bin.p,
                                                           s.tile_cnt.p);
    SOF_LAUNCHED(c);
    exclusive_scan_i32(c, s.tile_cnt.p, s.tile_off.p, NB + 1);
    k_scatter_group<<<grid_for(n, 256), 256, 0, c->stream>>>(n, gt.G, g.item_bin.p, s.tile_off.p, cur, g.order.p);
    SOF_LAUNCHED(c);
    k_block_counts<<<grid_for(NB + 1, 256), 256, 0, c->stream>>>(int(NB), 1, s.tile_off.p, s.blk_cnt.p);
    SOF_LAUNCHED(c);
    exclusive_scan_i32(c, s.blk_cnt.p, s.blk_off.p, NB + 1);
    const int64_t grid = (int64_t(gt.G) * n + kEvalThreads - 1) / kEvalThreads + NB;
    s.blocks.ensure(grid);
    k_block_fill<<<grid_for(NB + 1, 256), 256, 0, c->stream>>>(int(NB), 1, s.tile_off.p, s.blk_off.p, nullptr,
                                                               s.blocks.p,
                                                               c->d_scalar.p);
    SOF_LAUNCHED(c);
    const int e0 = prof_mark(c);
    if (c->staging == 1)
      k_eval_group<1><<<unsigned(grid), kEvalThreads, 0, c->stream>>>(s.blocks.p, c->d_scalar.p, g.order.p, n, xyz, g.cams.p,
                                                             tile_size, gt, loffs, lents, recs, g.tmaps.p, early,
                                                             g.item_pairs.p, g.item_ext.p, c->d_counters.p, bkeys,
                                                             bidxs, g.nbeh.p, xposs, g.nbeh.p + V);
    else
      k_eval_group<0><<<unsigned(grid), kEvalThreads, 0, c->stream>>>(s.blocks.p, c->d_scalar.p, g.order.p, n, xyz, g.cams.p,
                                                             tile_size, gt, loffs, lents, recs, nullptr, early,
                                                             g.item_pairs.p, g.item_ext.p, c->d_counters.p, bkeys,
                                                             bidxs, g.nbeh.p, xposs, g.nbeh.p + V);
    SOF_LAUNCHED(c);
    prof_span(c, e0, prof_mark(c), kProfEval);
    c->eval_launches++;
    k_group_fixup<<<grid_for(n, 256), 256, 0, c->stream>>>(n, gt.G, prune, g.item_bin.p, g.item_pairs.p,
                                                           g.item_ext.p, ext, c->d_counters.p);
    SOF_LAUNCHED(c);
  }
  if (counters_host) {
    unsigned long long h[5];
    SOF_CUDA(cudaMemcpyAsync(h, c->d_counters.p, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    SOF_CUDA(cudaStreamSynchronize(c->stream));
    counters_host[0] += h[0];
    counters_host[1] += h[1];
    c->exact_evals += h[2];
    c->contrib_evals += h[3];
    c->scanned_evals += h[4];
  }
  return true;
}

// The FP64 fast loop of k_eval: tile lists + min-z + dead cull (the default strategies).
static bool fast_loop(const sof_ctx* c, int strategies) {
  return c->eval_path == 1 && (strategies & 19) == 19;
}

// ---- bisection cache for views past the record budget -----------------------------------------
//
// binary_search_refine (marching_tets.hpp:94-114) classifies midpoints that always lie on
// their crossing edge's segment [p_in, p_out]. In a view, such a point's list scan
// stops at the first entry with min_z > its view depth (field_eval.hpp:90-93), so tile
// t only ever reads the prefix of its list with min_z <= zmax(t), zmax(t) = the largest
// endpoint depth over the segments whose projection can reach tile t. For views whose
// records and lists did not fit the cache during the label pass, the lists are built
// once, truncated to those prefixes (a midpoint's scan over the prefix makes exactly
// the reference's pairs, breaks and early stops: the entry after the prefix has
// min_z > zmax(t) >= the point's depth), and their records compacted — small enough to
// stay resident for all iterations, so the grouped kernels serve every view instead of
// re-binning a view per iteration.

// per tile: ordered key of the largest depth a midpoint in the tile can have (0: none)
__global__ void k_segment_zmax(int64_t ne, const int32_t* __restrict__ edges, const double* __restrict__ xyz,
                               Cam cam, int ts, int tiles_x, int tiles_y, unsigned long long* zmax,
                               int* bail) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= ne) return;
  const int32_t a = edges[2 * e], b = edges[2 * e + 1];
  double z[2], px[2], py[2];
  const int32_t v[2] = {a, b};
  for (int q = 0; q < 2; ++q) {
    const double x0 = xyz[3 * v[q]], x1 = xyz[3 * v[q] + 1], x2 = xyz[3 * v[q] + 2];
    z[q] = to_view_c(cam, 2, x0, x1, x2);
    if (z[q] > 1e-6) {
      px[q] = cam.fx * to_view_c(cam, 0, x0, x1, x2) / z[q] + cam.cx;
      py[q] = cam.fy * to_view_c(cam, 1, x0, x1, x2) / z[q] + cam.cy;
    }
  }
  if (z[0] <= 0.0 && z[1] <= 0.0) return;  // the whole segment is behind: never observed
  if (z[0] <= 1e-6 || z[1] <= 1e-6) {       // crosses (or touches) the camera plane
    atomicExch(bail, 1);
    return;
  }
  // tile box of the projected segment, dilated by one tile against rounding of the
  // midpoints' own projections
  const double lo_x = fmin(px[0], px[1]), hi_x = fmax(px[0], px[1]);
  const double lo_y = fmin(py[0], py[1]), hi_y = fmax(py[0], py[1]);
  if (hi_x < -double(ts) || hi_y < -double(ts) || lo_x > double(cam.w + ts) || lo_y > double(cam.h + ts)) return;
  const int tx0 = max(0, int(floor(fmax(lo_x, -2.0 * ts) / ts)) - 1);
  const int ty0 = max(0, int(floor(fmax(lo_y, -2.0 * ts) / ts)) - 1);
  const int tx1 = min(tiles_x - 1, int(floor(fmin(hi_x, double(cam.w + 2 * ts)) / ts)) + 1);
  const int ty1 = min(tiles_y - 1, int(floor(fmin(hi_y, double(cam.h + 2 * ts)) / ts)) + 1);
  if (int64_t(tx1 - tx0 + 1) * (ty1 - ty0 + 1) > 4096) {  // a long screen segment: keep the full lists
    atomicExch(bail, 1);
    return;
  }
  const double zm = fmax(z[0], z[1]);
  const unsigned long long key = double_key(zm + 1e-9 * (1.0 + zm));
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) atomicMax(zmax + int64_t(ty) * tiles_x + tx, key);
}

// per tile: length of the list prefix with min_z <= zmax(t) (lists sorted by (min_z, index))
__global__ void k_trunc_len(int64_t T, const int64_t* __restrict__ off, const int32_t* __restrict__ ent,
                            const Rec* __restrict__ rec, const unsigned long long* __restrict__ zmax,
                            int64_t* len) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t > T) return;
  if (t == T) {
    len[T] = 0;
    return;
  }
  const unsigned long long zk = zmax[t];
  int64_t lo = off[t], hi = off[t + 1];
  if (zk == 0) {
    len[t] = 0;
    return;
  }
  const double zm = key_double(zk);
  const int64_t l0 = lo;
  while (lo < hi) {  // first entry with min_z > zm
    const int64_t mid = lo + (hi - lo) / 2;
    if (rec[ent[mid]].zmin > zm)
      hi = mid;
    else
      lo = mid + 1;
  }
  len[t] = lo - l0;
}

// one warp per tile: mark the Gaussians of the kept prefixes
__global__ void k_trunc_mark(int64_t T, const int64_t* __restrict__ off, const int32_t* __restrict__ ent,
                             const int64_t* __restrict__ len, uint8_t* used) {
  const int64_t t = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const int64_t b = off[t], L = len[t];
  for (int64_t k = lane; k < L; k += 32) used[ent[b + k]] = 1;
}

// compact row of every used Gaussian; copy its record and its count flag
__global__ void k_trunc_rows(int64_t n, const uint8_t* __restrict__ used, const int32_t* __restrict__ pos,
                             const Rec* __restrict__ rec, Rec* out, const uint8_t* __restrict__ gflag,
                             uint8_t* rflag) {
  const int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (g >= n || !used[g]) return;
  out[pos[g]] = rec[g];
  rflag[pos[g]] = gflag[g];
}

// one warp per tile: the kept prefix, entries remapped to compact rows
__global__ void k_trunc_emit(int64_t T, const int64_t* __restrict__ off, const int32_t* __restrict__ ent,
                             const int64_t* __restrict__ toff, const int32_t* __restrict__ pos, int32_t* out) {
  const int64_t t = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const int64_t b = off[t], ob = toff[t], L = toff[t + 1] - ob;
  for (int64_t k = lane; k < L; k += 32) out[ob + k] = pos[ent[b + k]];
}

// count-list indices (2 g) in row space: 2 row for a Gaussian with a row, 2 pos - 1
// (between the rows before and after it) otherwise, so that comparing with 2 row(stop)
// orders exactly as comparing Gaussian indices (rows keep the Gaussian order)
__global__ void k_rows_of(int64_t nb, const int32_t* __restrict__ gidx2, const int32_t* __restrict__ pos,
                          const uint8_t* __restrict__ used, int32_t* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= nb) return;
  const int32_t g = gidx2[i] >> 1;
  out[i] = used[g] ? 2 * pos[g] : 2 * pos[g] - 1;
}

__global__ void k_u8_to_i32_f(int64_t n, const uint8_t* __restrict__ a, int32_t* b) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j < n) b[j] = a[j];
}

void bisect_cache_views(sof_ctx* c, int v0, int v1, int64_t ne, const int32_t* edges, int strategies,
                        int tile_size) {
  if (!fast_loop(c, strategies) || ne <= 0 || c->n <= 0 || std::getenv("SOF_NO_BISECT_CACHE")) return;
  if (!c->has_tets) return;
  const int64_t n = c->n;
  BisectScratch& bs = c->bis;  // kept across calls (no per-refine allocations)
  DBuf<unsigned long long>& zmax = bs.zmax;
  DBuf<int64_t>&len = bs.len, &toff = bs.toff;
  DBuf<uint8_t>& used = bs.used;
  DBuf<int32_t>&flag = bs.flag, &pos = bs.pos;
  DBuf<int>& bail = bs.bail;
  size_t free_b = size_t(-1);
  const bool dbg = std::getenv("SOF_DEBUG_HOST") != nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  int n_res = 0, n_trunc = 0, n_bail = 0, n_alias = 0;
  double ph[4] = {0, 0, 0, 0};  // debug: host ms in zmax, binning, truncation, memory check
  auto tick = [&]() { return std::chrono::steady_clock::now(); };
  auto ms_since = [&](std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(tick() - t).count();
  };
  struct Report {  // debug summary on every exit path
    bool on;
    const int *res, *trunc, *bail, *alias;
    std::chrono::steady_clock::time_point t0;
    const double* ph;
    ~Report() {
      if (on)
        std::fprintf(stderr,
                     "bisect_cache_views: resident %d truncated %d bailed %d full %d, %.1f ms (zmax %.1f, binning %.1f, "
                     "truncation %.1f, memory %.1f)\n",
                     *res, *trunc, *bail, *alias,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), ph[0],
                     ph[1], ph[2], ph[3]);
    }
  } report{dbg, &n_res, &n_trunc, &n_bail, &n_alias, h0, ph};
  // the views built here get truncated caches; their full records go to the scratch slot
  // (caching them in full would take the memory the truncated caches of later views need)
  struct CacheOff {
    sof_ctx* c;
    bool prev;
    ~CacheOff() { c->view_cache_off = prev; }
  } cache_off{c, c->view_cache_off};
  c->view_cache_off = true;
  for (int v = v0; v < v1; ++v) {
    if (view_resident(c, v, tile_size)) {
      ++n_res;
      continue;
    }
    const Cam& cam = c->cams[v];
    const int tiles_x = (cam.w + tile_size - 1) / tile_size, tiles_y = (cam.h + tile_size - 1) / tile_size;
    const int64_t T = int64_t(tiles_x) * tiles_y;
    // tiles and depths the midpoints can reach (needs no records)
    auto t0 = tick();
    zmax.ensure(T);
    bail.ensure(1);
    zero_async(c, zmax.p, sizeof(unsigned long long) * T);
    zero_async(c, bail.p, sizeof(int));
    k_segment_zmax<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, edges, c->tv.p, cam, tile_size, tiles_x, tiles_y,
                                                             zmax.p, bail.p);
    SOF_LAUNCHED(c);
    const bool bailed = read_scalar(c, bail.p);
    ph[0] += ms_since(t0);
    t0 = tick();
    if (bailed) {  // this view keeps the per-view path
      ++n_bail;
      continue;
    }
    // the view's records and its lists restricted to the reachable (tile, depth)
    // entries, built in the scratch slot, then compacted below
    Binding& full = c->bind_scratch[c->scratch_sel];
    c->bin_zmax = zmax.p;
    try {
      build_binding(c, v, tile_size, true, full, false);
    } catch (...) {
      c->bin_zmax = nullptr;
      full.view = -1;
      throw;
    }
    c->bin_zmax = nullptr;
    full.view = -1;  // a filtered binding is never served as the view's lists
    const Rec* rec = view_records(c, v);
    if (dbg) SOF_CUDA(cudaStreamSynchronize(c->stream));
    ph[1] += ms_since(t0);
    t0 = tick();
    // the budget had room after all: the records are cached in full (the per-view path
    // serves the view); never truncate into the buffers being read
    if (rec == c->recs[v].p) {
      ++n_alias;
      continue;
    }
    len.ensure(T + 1);
    toff.ensure(T + 1);
    k_trunc_len<<<grid_for(T + 1, 256), 256, 0, c->stream>>>(T, full.off.p, full.ent.p, rec, zmax.p, len.p);
    SOF_LAUNCHED(c);
    {
      size_t bytes = 0;
      SOF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, len.p, toff.p, T + 1, c->stream));
      c->cub_tmp.ensure(bytes);
      SOF_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, bytes, len.p, toff.p, T + 1, c->stream));
      c->launches += 2;
    }
    used.ensure(n);
    zero_async(c, used.p, n);
    k_trunc_mark<<<grid_for(T * 32, 256), 256, 0, c->stream>>>(T, full.off.p, full.ent.p, len.p, used.p);
    SOF_LAUNCHED(c);
    flag.ensure(n + 1);
    pos.ensure(n + 1);
    k_u8_to_i32_f<<<grid_for(n, 256), 256, 0, c->stream>>>(n, used.p, flag.p);
    SOF_LAUNCHED(c);
    zero_async(c, flag.p + n, sizeof(int32_t));
    exclusive_scan_i32(c, flag.p, pos.p, n + 1);
    const int64_t L = read_scalar(c, toff.p + T);
    const int64_t R = read_scalar(c, pos.p + n);
    ph[2] += ms_since(t0);
    t0 = tick();
    // room for it? (the full caches of the resident views stay; leave headroom). Free
    // memory is queried once per call and tracked across the views' new allocations.
    if (free_b == size_t(-1)) {
      size_t total_b = 0;
      SOF_CUDA(cudaMemGetInfo(&free_b, &total_b));
    }
    // DBuf::ensure over-allocates by 1/8; the per-view path that serves the views past
    // this point needs headroom for the buffers it may still grow
    const size_t need = (size_t(R) * sizeof(Rec) + size_t(L) * 4 + size_t(T + 1) * 8 +
                         size_t(full.nb) * 12 + size_t(full.nx) * 8) * 9 / 8 + (size_t(1) << 22);
    const size_t headroom = (size_t(2) << 30) + size_t(n) * 64;
    Binding& b = c->bindings[v];
    const size_t have = c->recs[v].bytes() + b.ent.bytes() + b.off.bytes() + b.bkey.bytes() + b.bidx.bytes() +
                        b.xpos.bytes();
    // the view's buffers from an earlier step already hold this cache: nothing is
    // allocated (every later step of the same scene takes this path)
    const bool in_place = c->recs[v].cap >= size_t(std::max<int64_t>(R, 1)) &&
                          b.ent.cap >= size_t(std::max<int64_t>(L, 1)) && b.off.cap >= size_t(T + 1) &&
                          (full.nb == 0 || (b.bkey.cap >= size_t(full.nb) && b.bidx.cap >= size_t(full.nb)));
    if (!in_place && need > have) {
      if (need - have + headroom > free_b) {  // out of memory: per-view path from here
        if (std::getenv("SOF_DEBUG_HOST"))
          std::fprintf(stderr, "bisect_cache_views: out of memory at view %d (free %.1f GB, need %.2f GB)\n", v,
                       free_b / 1e9, need / 1e9);
        break;
      }
      free_b -= need;  // upper bound of what the ensures below allocate
    }
    c->recs[v].ensure(std::max<int64_t>(R, 1));
    ph[3] += ms_since(t0);
    t0 = tick();
    bs.rflag.ensure(std::max<int64_t>(R, 1));
    k_trunc_rows<<<grid_for(n, 256), 256, 0, c->stream>>>(n, used.p, pos.p, rec, c->recs[v].p, c->gbehind.p,
                                                          bs.rflag.p);
    SOF_LAUNCHED(c);
    b.off.ensure(T + 1);
    SOF_CUDA(cudaMemcpyAsync(b.off.p, toff.p, sizeof(int64_t) * (T + 1), cudaMemcpyDeviceToDevice, c->stream));
    b.ent.ensure(std::max<int64_t>(L, 1));
    k_trunc_emit<<<grid_for(T * 32, 256), 256, 0, c->stream>>>(T, full.off.p, full.ent.p, toff.p, pos.p, b.ent.p);
    SOF_LAUNCHED(c);
    // the counted Gaussians, their indices in row space (k_rows_of), and the positions of
    // the listed crossing ones in the truncated lists
    b.nb = full.nb;
    b.nx = 0;
    if (b.nb > 0) {
      b.bkey.ensure(b.nb);
      b.bidx.ensure(b.nb);
      SOF_CUDA(cudaMemcpyAsync(b.bkey.p, full.bkey.p, sizeof(uint64_t) * b.nb, cudaMemcpyDeviceToDevice, c->stream));
      k_rows_of<<<grid_for(b.nb, 256), 256, 0, c->stream>>>(b.nb, full.bidx.p, pos.p, used.p, b.bidx.p);
      SOF_LAUNCHED(c);
      if (L > 0) cross_positions(c, b, L, bs.rflag.p);
    }
    b.view = v;
    b.tile_size = tile_size;
    b.tiles_x = tiles_x;
    b.tiles_y = tiles_y;
    b.live = true;
    b.trunc = true;
    b.rows = R;
    b.entries = L;
    c->rec_valid[v] = 2;
    ++n_trunc;
    SOF_CUDA(cudaStreamSynchronize(c->stream));  // the scratch slot is reused by the next view
    ph[2] += ms_since(t0);
  }
}

template <int MODE>
static void launch_eval(sof_ctx* c, bool tiled, int64_t grid, const int32_t* pidx,
                        const double* xyz, const Cam& cam, int ts, int tiles_x, const Binding* bd,
                        const Rec* rec, int strategies, bool classify, double* min_op,
                        uint8_t* ext, double* o_out, uint8_t* obs, uint8_t* comp) {
  if (grid <= 0) return;
  const int64_t* nb = c->sched.nblocks.p;
  unsigned long long* pc = c->d_counters.p;
  const int e0 = prof_mark(c);
  const RecF* recf = view_recf(c, int(&cam - c->cams.data()));
  if (c->eval_path == 0) {
    if (tiled)
      k_eval_f32<MODE, true><<<unsigned(grid), kEvalThreads, 0, c->stream>>>(
          c->sched.blocks.p, nb, pidx, xyz, cam, ts, tiles_x, bd->off.p, bd->ent.p, c->n, rec, recf,
          strategies, classify, min_op, ext, o_out, obs, comp, pc);
    else
      k_eval_f32<MODE, false><<<unsigned(grid), kEvalThreads, 0, c->stream>>>(
          c->sched.blocks.p, nb, pidx, xyz, cam, ts, tiles_x, nullptr, nullptr, c->n, rec, recf,
          strategies, classify, min_op, ext, o_out, obs, comp, pc);
  } else if (fast_loop(c, strategies)) {  // live-only lists, TMA-gathered records
    if (!bd->live) throw StateError("internal: the fast evaluation loop needs live-only tile lists");
    const Behind bh{bd->bkey.p, bd->bidx.p, bd->nb, bd->xpos.p, bd->nx};
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof tmap);
    if (c->staging == 1) {
      if (sof_make_row_tmap(&tmap, rec, c->n) != 0) throw StateError("cuTensorMapEncodeTiled failed for the records");
      k_eval<MODE, true, true, 1><<<unsigned(grid), kEvalThreads, 0, c->stream>>>(
          c->sched.blocks.p, nb, pidx, xyz, cam, ts, tiles_x, bd->off.p, bd->ent.p, c->n, rec,
          strategies, classify, min_op, ext, o_out, obs, comp, pc, tmap, bh);
    } else {
      k_eval<MODE, true, true, 0><<<unsigned(grid), kEvalThreads, 0, c->stream>>>(
          c->sched.blocks.p, nb, pidx, xyz, cam, ts, tiles_x, bd->off.p, bd->ent.p, c->n, rec,
          strategies, classify, min_op, ext, o_out, obs, comp, pc, tmap, bh);
    }
  } else {
    CUtensorMap none;
    std::memset(&none, 0, sizeof none);
    if (tiled)
      k_eval<MODE, true, false><<<unsigned(grid), kEvalThreads, 0, c->stream>>>(
          c->sched.blocks.p, nb, pidx, xyz, cam, ts, tiles_x, bd->off.p, bd->ent.p, c->n, rec,
          strategies, classify, min_op, ext, o_out, obs, comp, pc, none, Behind{nullptr, nullptr, 0, nullptr, 0});
    else
      k_eval<MODE, false, false><<<unsigned(grid), kEvalThreads, 0, c->stream>>>(
          c->sched.blocks.p, nb, pidx, xyz, cam, ts, tiles_x, nullptr, nullptr, c->n, rec,
          strategies, classify, min_op, ext, o_out, obs, comp, pc, none, Behind{nullptr, nullptr, 0, nullptr, 0});
  }
  SOF_LAUNCHED(c);
  prof_span(c, e0, prof_mark(c), kProfEval);
  c->eval_launches++;
}

void eval_views(sof_ctx* c, int v0, int v1, int64_t n, const double* xyz, int strategies,
                int tile_size, bool classify_mode, EvalMode mode, double* min_op, uint8_t* ext,
                double* o_out, uint8_t* obs_out, uint8_t* comp_out, uint64_t* counters_host) {
  if (!c->has_scene) throw StateError("no scene: call sof_set_scene first");
  if (v0 < 0 || v1 > int(c->cams.size()) || v0 > v1) throw InvalidArg("view range out of bounds");
  if (tile_size <= 0) throw InvalidArg("tile_size must be positive");
  // the five EvalStrategies toggles only (field_eval.hpp:14-20); higher bits are
  // internal kernel flags (kRecheckPruned) and never come from the caller
  if (strategies & ~int(SOF_ALL_STRATEGIES)) throw InvalidArg("strategies mask has bits outside 0..31");
  const bool tiled = strategies & 1;
  const bool prune = strategies & 8;
  // the FP64 fast loop (tile lists + min-z + dead cull) runs on live-only lists
  const bool live_lists = fast_loop(c, strategies);
  // A label pass uses each view once; its full per-view caches only serve the bisection
  // afterwards. When fewer than a quarter of the views' records would fit the budget
  // (C5: 65 of 500), cache none: the memory then holds the bisection's truncated caches
  // (0.59 GB instead of 1.4 GB per view on C5), so fewer views are re-binned per iteration.
  // The decision holds until the caches are marked stale (the next step): the bisection's
  // per-view path must not fill the memory its truncated caches hold either.
  if (mode == kModeLabel && !std::getenv("SOF_LABEL_CACHE_ALWAYS")) {
    const double per_view = double(n > 0 ? c->n : 0) * double(sizeof(Rec));
    const double views = double(v1 - v0);
    c->view_cache_off = per_view > 0.0 && double(c->cache_budget) < 0.25 * views * per_view;
  }
  if (mode == kModeClassify &&
      classify_grouped(c, v0, v1, n, xyz, strategies, tile_size, ext, counters_host))
    return;
  c->d_counters.ensure(5);
  c->d_scalar.ensure(4);
  zero_async(c, c->d_counters.p, int64_t(sizeof(unsigned long long)) * 5);
  PointSchedule& s = c->sched;
  if (mode == kModeView && n > 0) {
    k_fill_view_outputs<<<grid_for(n, 256), 256, 0, c->stream>>>(n, o_out, obs_out, comp_out);
    SOF_LAUNCHED(c);
  }
  // Per-view preprocessing (K1 records + K2 tile binding + K3 point schedule) runs on
  // the prep lane (second stream, own CUB scratch), one view ahead of the evaluation:
  // the host issues view v's evaluation, then prepares view v + 1 (its one size
  // readback blocks only the host) while the GPU evaluates view v.
  int64_t ncand = n;      // candidate points of the next view
  bool use_list = false;  // candidates = s.active[0, ncand) instead of all points
  const Rec* prep_rec[2] = {nullptr, nullptr};
  const Binding* prep_bd[2] = {nullptr, nullptr};
  const uint8_t* skip = (prune && (mode == kModeLabel || mode == kModeClassify)) ? ext : nullptr;
  // SOF_SCHED_LOOKAHEAD: build view v + 1's schedule on the prep lane during view v's
  // evaluation (off the critical path; the evaluation then re-checks the pruned flags).
  // Default off: 1.3% faster per C3 step, but the evaluation kernel then shares the SMs
  // with the scheduler for its whole span.
  const bool lookahead = std::getenv("SOF_SCHED_LOOKAHEAD") != nullptr;
  // kRecheckPruned relies on ext only ever going 0 -> 1 while K3 for view v + 1 reads it
  // on the prep lane and view v's K4 writes it: a stale 0 is re-checked inside K4
  const int eval_strategies = strategies | ((lookahead && skip) ? kRecheckPruned : 0);
  int64_t sched_grid[2] = {0, 0};  // evaluation grid of the schedule built for view pv
  auto sched_view = [&](int pv) {
    const Cam& cam = c->cams[pv];
    const int tiles_x = (cam.w + tile_size - 1) / tile_size;
    const int tiles_y = (cam.h + tile_size - 1) / tile_size;
    const int T = tiled ? tiles_x * tiles_y : 1;
    const int p1 = prof_mark(c);
    const auto h1 = std::chrono::steady_clock::now();
    // K3: group the active, observed points of this view by tile (no host sync). The
    // pruned flags may still change under the previous view's evaluation: a point
    // pruned after this pass is skipped by the evaluation kernel itself.
    s.tile_of.ensure(n);
    s.order.ensure(n);
    s.nblocks.ensure(1);
    // bins per tile: 4x4-pixel cells when points are dense enough to fill them (label
    // grids), else whole tiles (bisection midpoints)
    const int S = (tiled && ncand >= 1024 * int64_t(T)) ? 16 : 1;
    const int64_t NB = int64_t(T) * S;
    s.tile_cnt.ensure(2 * (NB + 1));
    s.tile_off.ensure(NB + 1);
    s.blk_cnt.ensure(T + 1);
    s.blk_off.ensure(T + 1);
    zero_async(c, s.tile_cnt.p, int64_t(sizeof(int)) * 2 * (NB + 1));
    int* tile_cur = s.tile_cnt.p + (NB + 1);
    const int32_t* cand = use_list ? s.active.p : nullptr;
    if (tile_size == 16)
      k_sched_tile<16><<<grid_for((ncand + kSchedPts - 1) / kSchedPts, 256), 256, 0, c->stream>>>(ncand, cand, xyz, cam, tile_size, tiles_x,
                                                                    !tiled, S, skip, s.tile_of.p, s.tile_cnt.p);
    else
      k_sched_tile<0><<<grid_for((ncand + kSchedPts - 1) / kSchedPts, 256), 256, 0, c->stream>>>(ncand, cand, xyz, cam, tile_size, tiles_x,
                                                                   !tiled, S, skip, s.tile_of.p, s.tile_cnt.p);
    SOF_LAUNCHED(c);
    exclusive_scan_i32(c, s.tile_cnt.p, s.tile_off.p, NB + 1);
    k_sched_scatter<<<grid_for((ncand + kScatterItems - 1) / kScatterItems, 256), 256, 0, c->stream>>>(
        ncand, cand, s.tile_of.p, s.tile_off.p, tile_cur, s.order.p);
    SOF_LAUNCHED(c);
    k_block_counts<<<grid_for(T + 1, 256), 256, 0, c->stream>>>(T, S, s.tile_off.p, s.blk_cnt.p);
    SOF_LAUNCHED(c);
    exclusive_scan_i32(c, s.blk_cnt.p, s.blk_off.p, T + 1);
    const int64_t grid = (ncand + kEvalThreads - 1) / kEvalThreads + T;
    s.blocks.ensure(grid);
    k_block_fill<<<grid_for(T + 1, 256), 256, 0, c->stream>>>(T, S, s.tile_off.p, s.blk_off.p,
                                                               tiled ? prep_bd[pv & 1]->off.p : nullptr, s.blocks.p,
                                                               s.nblocks.p);
    SOF_LAUNCHED(c);
    sched_grid[pv & 1] = grid;
    prof_span(c, p1, prof_mark(c), kProfSched);
    c->host_ms[1] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h1).count();
  };
  auto swap_lane = [&]() {  // the prep lane's stream and scratch (CUB, the hand-written scans, k_cross_sel)
    std::swap(c->stream, c->stream2);
    c->cub_tmp.swap(c->cub_tmp2);
    c->scan_tmp.swap(c->scan_tmp2);
    c->sel_cnt.swap(c->sel_cnt2);
    c->sel_off.swap(c->sel_off2);
  };
  auto prep_view = [&](int pv) {
    swap_lane();
    c->scratch_sel = pv & 1;
    try {
      // scratch slot pv & 1 may still hold the records / tile lists of view pv - 2 (past
      // the cache budget): wait until its evaluation on the main stream is done
      SOF_CUDA(cudaStreamWaitEvent(c->stream, c->eval_ev[pv & 1], 0));
      const int p0 = prof_mark(c);
      // binding first: it computes the records in the same pass as the tile rectangles
      prep_bd[pv & 1] = tiled ? &view_binding(c, pv, tile_size, live_lists) : nullptr;
      prep_rec[pv & 1] = view_records(c, pv);
      prof_span(c, p0, prof_mark(c), kProfPrep);
      // K3 for view pv into the other schedule buffers (view pv - 1's evaluation reads
      // the current ones); pv - 2's evaluation, which read them, is done (event above)
      if (lookahead) {
        s.swap_view_buffers(c->sched_alt);
        sched_view(pv);
      }
      SOF_CUDA(cudaEventRecord(c->prep_ev[pv & 1], c->stream));
    } catch (...) {
      swap_lane();
      throw;
    }
    swap_lane();
  };
  const bool dbg = std::getenv("SOF_DEBUG_HOST") != nullptr;
  const auto hd0 = std::chrono::steady_clock::now();
  for (int v = v0; v < v1 && n > 0; ++v) {
    if (dbg && (v - v0 < 3 || v + 1 == v1))
      std::fprintf(stderr, "    view %3d issued at %8.2f ms ncand %lld list %d\n", v,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hd0).count(),
                   (long long)ncand, int(use_list));
    const Cam& cam = c->cams[v];
    const int tiles_x = (cam.w + tile_size - 1) / tile_size;
    const auto h0 = std::chrono::steady_clock::now();
    if (v == v0) {
      // the prep lane's first two views reuse buffers of earlier main-stream work
      SOF_CUDA(cudaEventRecord(c->eval_ev[0], c->stream));
      SOF_CUDA(cudaEventRecord(c->eval_ev[1], c->stream));
      prep_view(v);
    }
    // the records, binding and schedule of view v were prepared on the prep lane
    // (during view v - 1's evaluation)
    SOF_CUDA(cudaStreamWaitEvent(c->stream, c->prep_ev[v & 1], 0));
    c->host_ms[0] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    if (!lookahead) sched_view(v);  // on the main stream, after view v - 1's evaluation

    const Rec* rec = prep_rec[v & 1];
    const Binding* bd = prep_bd[v & 1];
    const int64_t grid = sched_grid[v & 1];
    const int32_t* pidx = s.order.p;
    switch (mode) {
      case kModeLabel:
        launch_eval<kModeLabel>(c, tiled, grid, pidx, xyz, cam, tile_size, tiles_x, bd, rec,
                                eval_strategies, classify_mode, min_op, ext, o_out, obs_out, comp_out);
        break;
      case kModeClassify:
        launch_eval<kModeClassify>(c, tiled, grid, pidx, xyz, cam, tile_size, tiles_x, bd, rec,
                                   eval_strategies, true, min_op, ext, o_out, obs_out, comp_out);
        break;
      case kModeView:
        launch_eval<kModeView>(c, tiled, grid, pidx, xyz, cam, tile_size, tiles_x, bd, rec,
                               eval_strategies, classify_mode, min_op, ext, o_out, obs_out, comp_out);
        break;
      case kModeValue:
        launch_eval<kModeValue>(c, tiled, grid, pidx, xyz, cam, tile_size, tiles_x, bd, rec,
                                eval_strategies, false, min_op, ext, o_out, obs_out, comp_out);
        break;
    }
    SOF_CUDA(cudaEventRecord(c->eval_ev[v & 1], c->stream));
    // drop pruned points from the candidate list now and then (the reference skips them,
    // field_eval.hpp:147); the list shrinks fast over the first views
    const int done_views = v - v0 + 1;
    pump_upload(c, kUploadChunk);  // a pending tets upload advances one chunk per view
    if (skip && v + 1 < v1 && (done_views <= 4 || done_views % 16 == 0)) {
      s.active2.ensure(std::max<int64_t>(ncand, 1));
      s.nsel.ensure(1);
      size_t bytes = 0;
      NotPruned pred{ext};
      if (use_list) {
        SOF_CUDA(cub::DeviceSelect::If(nullptr, bytes, s.active.p, s.active2.p, s.nsel.p, ncand, pred, c->stream));
        c->cub_tmp.ensure(bytes);
        SOF_CUDA(cub::DeviceSelect::If(c->cub_tmp.p, bytes, s.active.p, s.active2.p, s.nsel.p, ncand, pred,
                                       c->stream));
      } else {
        thrust::counting_iterator<int32_t> it(0);
        SOF_CUDA(cub::DeviceSelect::If(nullptr, bytes, it, s.active2.p, s.nsel.p, ncand, pred, c->stream));
        c->cub_tmp.ensure(bytes);
        SOF_CUDA(cub::DeviceSelect::If(c->cub_tmp.p, bytes, it, s.active2.p, s.nsel.p, ncand, pred, c->stream));
      }
      c->launches += 2;
      s.active.swap(s.active2);
      ncand = read_scalar(c, s.nsel.p);
      use_list = true;
      if (ncand == 0) break;  // every point is pruned: the remaining views skip them all
    }
    if (v + 1 < v1) {
      const auto h3 = std::chrono::steady_clock::now();
      prep_view(v + 1);
      c->host_ms[0] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h3).count();
    }
  }
  if (dbg)
    std::fprintf(stderr, "    all views issued at %8.2f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hd0).count());
  if (counters_host) {
    unsigned long long h[5];
    SOF_CUDA(cudaMemcpyAsync(h, c->d_counters.p, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    SOF_CUDA(cudaStreamSynchronize(c->stream));
    counters_host[0] += h[0];
    counters_host[1] += h[1];
    c->exact_evals += h[2];
    c->contrib_evals += h[3];
    c->scanned_evals += h[4];
  }
}

// label_grid's final write (field_eval.hpp:173-175)
__global__ void k_finalize_label(int64_t n, const double* __restrict__ m,
                                 const uint8_t* __restrict__ ext, double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double v = m[i];
  out[i] = ext[i] ? ((0.49999999 < v) ? 0.49999999 : v) : v;
}

void finalize_label(sof_ctx* c, int64_t n, const double* min_op, const uint8_t* ext, double* out) {
  if (n <= 0) return;
  k_finalize_label<<<grid_for(n, 256), 256, 0, c->stream>>>(n, min_op, ext, out);
  SOF_LAUNCHED(c);
}

// ---- exact schedule_points (API / parity; tiles.hpp:29-84) -------------------------------------

__global__ void k_sched_exact(int64_t n, const double* __restrict__ xyz, Cam cam, int ts,
                              int tiles_x, int32_t* tile_assign, uint64_t* dkey, int32_t* idx) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  // tiles.hpp:46-51: observe test without the t >= 1e-12 rule of view_opacity
  const double x0 = xyz[3 * i], x1 = xyz[3 * i + 1], x2 = xyz[3 * i + 2];
  const double vx = to_view_c(cam, 0, x0, x1, x2);
  const double vy = to_view_c(cam, 1, x0, x1, x2);
  const double vz = to_view_c(cam, 2, x0, x1, x2);
  int tile = -1;
  if (vz > 0.0) {
    const double px = cam.fx * vx / vz + cam.cx;
    const double py = cam.fy * vy / vz + cam.cy;
    if (!(px < 0.0 || px >= cam.w || py < 0.0 || py >= cam.h))
      tile = (int)py / ts * tiles_x + (int)px / ts;
  }
  tile_assign[i] = tile;
  dkey[i] = double_key(vz);
  idx[i] = int32_t(i);
}

void schedule_points_exact(sof_ctx* c, int view, int64_t n, const double* xyz, int ts,
                           int32_t* tile_assignment, std::vector<int32_t>& order,
                           std::vector<int32_t>& key_tile, std::vector<double>& key_depth,
                           std::vector<int32_t>& block_ranges,
                           std::vector<int32_t>& block_to_tile) {
  if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
  const Cam& cam = c->cams[view];
  const int tiles_x = (cam.w + ts - 1) / ts, tiles_y = (cam.h + ts - 1) / ts;
  order.clear();
  key_tile.clear();
  key_depth.clear();
  block_ranges.clear();
  block_to_tile.clear();
  if (n == 0) return;
  DBuf<int32_t> tile, tile_sorted;
  DBuf<uint64_t> k1, k2;
  DBuf<int32_t> i1, i2;
  tile.ensure(n);
  tile_sorted.ensure(n);
  k1.ensure(n);
  k2.ensure(n);
  i1.ensure(n);
  i2.ensure(n);
  k_sched_exact<<<grid_for(n, 256), 256, 0, c->stream>>>(n, xyz, cam, ts, tiles_x, tile.p, k1.p,
                                                          i1.p);
  SOF_LAUNCHED(c);
  // (tile, depth, point): sort by depth (stable on index), then stably by tile
  sort_pairs_u64(c, k1.p, k2.p, i1.p, i2.p, n, 64);
  std::vector<int32_t> h_tile(n), h_ord(n);
  std::vector<uint64_t> h_dk(n);
  SOF_CUDA(cudaMemcpyAsync(tile_assignment, tile.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                           c->stream));
  SOF_CUDA(cudaMemcpyAsync(h_ord.data(), i2.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                           c->stream));
  SOF_CUDA(cudaStreamSynchronize(c->stream));
  // stable counting pass by tile on the host side (the API path is not hot)
  const int64_t T = int64_t(tiles_x) * tiles_y;
  std::vector<int64_t> cnt(T + 1, 0);
  for (int64_t r = 0; r < n; ++r) {
    const int t = tile_assignment[h_ord[r]];
    if (t >= 0) cnt[t + 1]++;
  }
  for (int64_t t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
  const int64_t m = cnt[T];
  order.assign(m, 0);
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (int64_t r = 0; r < n; ++r) {
    const int32_t p = h_ord[r];
    const int t = tile_assignment[p];
    if (t >= 0) order[pos[t]++] = p;
  }
  // depths in double from the host copy of the points is not available here; recompute
  std::vector<double> h_xyz(3 * n);
  SOF_CUDA(cudaMemcpy(h_xyz.data(), xyz, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
  key_tile.resize(m);
  key_depth.resize(m);
  for (int64_t k = 0; k < m; ++k) {
    const int32_t p = order[k];
    key_tile[k] = tile_assignment[p];
    key_depth[k] = to_view_c(cam, 2, h_xyz[3 * p], h_xyz[3 * p + 1], h_xyz[3 * p + 2]);
  }
  for (int64_t t = 0; t < T; ++t) {
    const int64_t b0 = cnt[t], b1 = cnt[t + 1];
    for (int64_t b = b0; b < b1; b += kBlockPoints) {
      block_ranges.push_back(int32_t(b));
      block_ranges.push_back(int32_t(std::min<int64_t>(b + kBlockPoints, b1)));
      block_to_tile.push_back(int32_t(t));
    }
  }
}

}  // namespace sofk
