// sof_internal.h — context, device buffers and stage entry points shared by the
// translation units of libsof_cuda.so. Not part of the public ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sof_cuda.h"
#include "sof_device.cuh"

namespace sofk {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OomError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Comm;  // k_comm.cu: the context's communicator (NCCL, or in-process for tests)

#define SOF_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      if (e_ == cudaErrorMemoryAllocation) {                                               \
        (void)cudaGetLastError();                                                          \
        throw ::sofk::OomError(std::string("CUDA out of memory at ") + __FILE__ + ":" +   \
                               std::to_string(__LINE__));                                  \
      }                                                                                    \
      throw ::sofk::CudaError(std::string(cudaGetErrorString(e_)) + " at " + __FILE__ +   \
                              ":" + std::to_string(__LINE__));                             \
    }                                                                                      \
  } while (0)

// Grow-only device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  size_t n = 0;    // logical size
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), cap(o.cap), n(o.n) { o.p = nullptr; o.cap = o.n = 0; }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  T* ensure(size_t count) {
    if (count > cap) {
      if (p) SOF_CUDA(cudaFree(p));
      p = nullptr;
      cap = 0;
      const size_t want = count + count / 8 + 16;
      const cudaError_t e = cudaMalloc(&p, want * sizeof(T));
      if (e == cudaErrorMemoryAllocation) {
        (void)cudaGetLastError();
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        throw ::sofk::OomError("CUDA out of memory: a " + std::to_string(want * sizeof(T) >> 20) +
                               " MiB buffer with " + std::to_string(fr >> 20) + " MiB free");
      }
      SOF_CUDA(e);
      cap = want;
    }
    n = count;
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = n = 0;
  }
  void swap(DBuf& o) noexcept {
    std::swap(p, o.p);
    std::swap(cap, o.cap);
    std::swap(n, o.n);
  }
  size_t bytes() const { return cap * sizeof(T); }
};

// Per-view Gaussian tile lists (TileBinding tiles.hpp:88-92) resident on the device.
struct Binding {
  int view = -1, tile_size = 0, tiles_x = 0, tiles_y = 0;
  // live-only lists: dead Gaussians (op < 1/255) left out. With dead cull + min-z on
  // (the default strategies) the reference skips them before the pair counter and the
  // min-z break (field_eval.hpp:89-93), so these lists give identical results and
  // counters; the exact reference lists (tiles.hpp:134-144) have live = false.
  bool live = false;
  // bisection cache (bisect_cache_views): every list truncated to the depths the
  // bisection midpoints can reach, entries are rows of a compact record array
  bool trunc = false;
  int64_t rows = 0;  // compact record rows (trunc only)
  int64_t entries = 0;
  DBuf<int64_t> off;  // [T + 1]
  DBuf<int32_t> ent;  // [entries], per tile sorted by (min_z, index)
  // live lists only: the gauss_behind Gaussians (sof_device.cuh), which the reference
  // lists in every tile ahead of everything else and which never contribute: left out of
  // the lists, sorted by (min_z key, index) here, and counted by the evaluation
  // Since round 2 the list also holds the live Gaussians whose box crosses the camera
  // plane (listed by the reference in every tile): they are listed only in the tiles
  // whose points they may reach (cross_tile_live), at the list positions xpos.
  int64_t nb = 0;
  DBuf<uint64_t> bkey;  // double_key(min_z)
  DBuf<int32_t> bidx;   // 2 g (a truncated binding: 2 row, or 2 row - 1 between rows)
  int64_t nx = 0;
  DBuf<int64_t> xpos;   // ascending positions in ent of listed crossing Gaussians
};

// Scratch of the per-view point schedule (schedule_points tiles.hpp:29-84).
struct PointSchedule {
  DBuf<int32_t> tile_of;     // [n] tile of each point in this view, -1 if inactive
  DBuf<int32_t> order;       // [n] point indices grouped by tile
  DBuf<int> tile_cnt;        // [2(T + 1)] histogram | scatter cursors
  DBuf<int> tile_off, blk_cnt, blk_off;  // [T + 1]
  DBuf<int4> blocks;         // {start, end, tile, 0}
  DBuf<int32_t> active, active2, nsel;  // candidate points (not pruned), compacted
  DBuf<int64_t> nblocks;                // [1] block count (read by the evaluation kernel)
  // the per-view buffers (not the candidate lists): the schedule of view v + 1 is built
  // on the prep lane while view v's evaluation reads the other set
  void swap_view_buffers(PointSchedule& o) noexcept {
    tile_of.swap(o.tile_of);
    order.swap(o.order);
    tile_cnt.swap(o.tile_cnt);
    tile_off.swap(o.tile_off);
    blk_cnt.swap(o.blk_cnt);
    blk_off.swap(o.blk_off);
    blocks.swap(o.blocks);
    nblocks.swap(o.nblocks);
  }
};

// Persistent (grow-only) scratch of the mesher stages: no allocation in steady state.
struct MeshScratch {
  DBuf<uint8_t> crossing, first_u8;
  DBuf<int32_t> ctets, nsel;
  DBuf<unsigned long long> packed, off;
  DBuf<uint64_t> okey, skey;
  DBuf<int32_t> opos, spos, oin, oout, tri_occ, tri_tet, head, run_incl, is_first, eid, run_eid,
      occ_edge;
  DBuf<double> pin, pout, mid;  // bisection brackets
  DBuf<uint8_t> rext;
  DBuf<uint64_t> kx, ky, kz, k1, k2;  // weld
  DBuf<int32_t> p0, p1, whead, wrun, wrun_first, first_of, wfirst, nid, rt, keep, pos;
  DBuf<double> seed_pts, seed_cpts;       // seed candidates / valid ones in order
  DBuf<uint8_t> seed_prov, seed_cprov;
  DBuf<int32_t> seed_valid, seed_pos;
};

// Render spill pool (k_render.cu): keys / values double-buffered for the segmented sort.
// Grouped bisection classification (k_field.cu classify_grouped).
struct GroupScratch {
  DBuf<Cam> cams;                 // [V]
  DBuf<const void*> ptrs;         // [5V] per-view tile offsets, tile entries, records, behind keys / indices
  DBuf<int64_t> nbeh;             // [V] behind counts
  DBuf<CUtensorMap> tmaps;        // [V] TMA descriptors of the per-view record arrays
  DBuf<int32_t> item_bin, order;  // [G n]
  DBuf<uint32_t> item_pairs;      // [G n]
  DBuf<uint8_t> item_ext;         // [G n]
};

// Scratch of bisect_cache_views (per-tile zmax, truncated list offsets, row maps).
struct BisectScratch {
  DBuf<unsigned long long> zmax;
  DBuf<int64_t> len, toff;
  DBuf<uint8_t> used, rflag;  // rflag: count flag (k_field.cu kCountCross) per compact row
  DBuf<int32_t> flag, pos;
  DBuf<int> bail;
};

// Sorted rasterizer scratch (k_render.cu): per-view render binning, per-pixel slices of
// contributions and their sorted order.
struct RenderScratch {
  DBuf<int4> rect;                // [n] tile rectangle per Gaussian
  DBuf<uint32_t> gcnt;            // [n] tiles per Gaussian
  DBuf<uint32_t> tile_cnt;        // [T] entries per tile (histogram) | scatter cursors
  DBuf<int64_t> tile_off;         // [T + 1]
  DBuf<int32_t> ent;              // [entries] Gaussian ids grouped by tile (any order inside)
  DBuf<int32_t> big;              // Gaussians (binning) / pixels (sort) handled cooperatively
  DBuf<int32_t> big_cnt;          // [4] counts of those lists
  DBuf<uint32_t> pcnt;            // [T * 256] per-pixel bound (conic-passing records)
  DBuf<uint32_t> ncon;            // [T * 256] per-pixel contributions
  DBuf<int64_t> poff;             // [T * 256 + 1] slice offsets (tile-major pixel order)
  DBuf<int64_t> band_off;         // [T + 1] slice offset of each tile's first pixel
  DBuf<char> ent16;               // per contribution: REnt {t*, list position, Gaussian index}
  bool attr_set = false;          // k_rsort_big's dynamic shared-memory limit set
  DBuf<char> rrec;                // [n] per-view render records (k_render.cu RRec, 128 B)
  DBuf<char> ent16b;              // window mode: the resorted slices (REnt)
  DBuf<uint64_t> tmask;           // [n] tiles of a small rectangle the cull leaves (k_rrect)
  DBuf<double> zc;                // window mode: [n] view-space centre depth (arrival order)
};

enum ProfKind { kProfEval = 0, kProfPrep = 1, kProfSched = 2, kProfKinds = 4 };

enum EvalMode { kModeLabel = 0, kModeClassify = 1, kModeView = 2, kModeValue = 3 };

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
};

}  // namespace sofk

struct sof_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;

  // scene
  int64_t n = 0;
  double filter_scale = 0.0;
  bool has_scene = false;
  sofk::DBuf<double> pos, scale, rot, opa, dc;
  sofk::DBuf<sofk::GaussStatic> gstat;

  // views
  std::vector<sofk::Cam> cams;

  // per-view record cache: recs[v] valid when rec_valid[v]
  std::vector<sofk::DBuf<sofk::Rec>> recs;
  std::vector<char> rec_valid;
  std::vector<sofk::Binding> bindings;  // per view (cache keyed by tile size)
  size_t cache_budget = size_t(96) << 30;  // bytes of HBM the per-view caches may use
  size_t cache_bytes = 0;
  // set for a label pass whose views' full caches would mostly not fit the budget: the
  // pass then caches none (each view is used once there) and leaves the memory to the
  // bisection's truncated caches (k_field.cu, eval_views)
  bool view_cache_off = false;
  std::vector<sofk::DBuf<sofk::RecF>> recfs;
  // past the cache budget, per-view state goes to one of two scratch slots (ping-pong:
  // view v + 1 is prepared on the prep stream while view v is evaluated)
  sofk::DBuf<sofk::Rec> rec_scratch[2];
  sofk::DBuf<sofk::RecF> recf_scratch[2];
  sofk::Binding bind_scratch[2];
  int scratch_view[2] = {-1, -1};
  int scratch_sel = 0;
  int eval_path = 1;                      // 0: FP32 filter + exact FP64 replay, 1: FP64 only
  int staging = 0;                        // fast-loop record staging: 0 plain loads, 1 TMA gather4
  uint64_t exact_evals = 0;               // pairs that took the FP64 path (instrumentation)
  uint64_t contrib_evals = 0;             // ... of which contributed (alpha >= 1/255)
  uint64_t scanned_evals = 0;             // list entries the evaluation kernels scanned (their work)
  double host_ms[4] = {0, 0, 0, 0};       // host time in per-view prep / scheduling (instrumentation)

  // prep lane: a second stream (+ its own CUB scratch) for per-view preprocessing
  cudaStream_t stream2 = nullptr;
  cudaEvent_t eval_ev[2] = {nullptr, nullptr};  // end of the eval of views of parity 0 / 1
  cudaStream_t stream_copy = nullptr;     // sof_set_tets_async: tet upload + index check
  uint64_t* pinned_scalar = nullptr;      // [8] pinned host slots for small read-backs
  cudaEvent_t tets_ev = nullptr;          // ... recorded after them
  cudaEvent_t interop_ev = nullptr;       // sof_stream_wait: an event on the caller's stream
  bool tets_pending = false;              // march must wait for tets_ev and check the flag
  // the pending upload, fed to the copy engine in chunks (pump_upload) so that the
  // memsets CUB issues on the same engine never queue behind gigabytes
  const char* up_src = nullptr;
  int64_t up_bytes = 0, up_done = 0, up_nv = 0;
  sofk::DBuf<int32_t> tets_bad;
  sofk::DBuf<char> cub_tmp2;
  cudaEvent_t prep_ev[2] = {nullptr, nullptr};

  // binning scratch
  sofk::DBuf<int4> rect;
  sofk::DBuf<uint32_t> gcount;
  sofk::DBuf<uint8_t> gbehind;     // per Gaussian: gauss_behind (live bindings)
  sofk::DBuf<uint64_t> zkey_in, zkey_out, zkey_aux;
  sofk::DBuf<char> loss_buf;       // batched training-loss inputs / outputs (k_loss.cu)
  sofk::DBuf<int64_t> bin_scalar;  // [4] selected count | tie-run overflow flag | count flags
  int64_t bin_nflag = 0;           // count flags of the binding being built (host copy)
  int64_t bin_m = 0;               // Gaussians with tiles in the current binning
  const unsigned long long* bin_zmax = nullptr;  // bisection-cache binning filter (per tile)
  sofk::BisectScratch bis;
  sofk::DBuf<int32_t> gidx_in, gidx_out;
  sofk::DBuf<int64_t> goff;
  sofk::DBuf<uint32_t> ekey_in, ekey_out;
  sofk::DBuf<int32_t> eval_in;

  sofk::PointSchedule sched;
  sofk::PointSchedule sched_alt;          // second set of per-view schedule buffers
  sofk::MeshScratch ms;
  sofk::RenderScratch rs;
  sofk::GroupScratch grp;
  sofk::DBuf<double> seeds;               // build_seed_points result
  sofk::DBuf<uint8_t> seed_prov;
  int64_t n_seeds = -1;                 // spill pool of k-buffer-overflow pixels
  sofk::DBuf<double> r_out;               // depth, opacity, rgb(3), t_final per pixel
  sofk::DBuf<unsigned long long> r_stats;
  sofk::DBuf<double> r_normal, r_depth_in;  // normal_from_depth output / uploaded depth
  sofk::DBuf<uint8_t> r_valid;
  sofk::DBuf<char> r_query;                 // gaussian_normal queries
  sofk::DBuf<unsigned char> io_bytes;       // scene PLY payload / encoded records
  int r_view = -1;                          // view whose render is in r_out
  int64_t r_bands = 0;                      // tile bands of the last render
  int64_t r_Q = 0;                          // tile-major pixel slots of the last render
  int64_t render_pool = int64_t(24) << 30;  // scratch budget of one render band (bytes)
  int64_t r_window = 0;                     // 0: exact (t*, index) order; K > 0: K-slot windowed resort
  sofk::DBuf<int32_t> ct_idx;               // sof_collect_contributions: gaussian_index per contribution
  sofk::DBuf<double> ct_val;                // ... and (t*, alpha, a, b, c, opacity)
  int64_t n_contrib = -1;
  sofk::DBuf<char> cub_tmp;
  sofk::DBuf<char> scan_tmp;                 // block totals of the hand-written scans (k_scan.cu)
  sofk::DBuf<int64_t> sel_cnt, sel_off;      // compaction block counts / offsets (k_sort.cu, k_cross_sel)
  // the prep lane's own copies (swapped in while it issues work on stream2)
  sofk::DBuf<char> scan_tmp2;
  sofk::DBuf<int64_t> sel_cnt2, sel_off2;
  sofk::DBuf<unsigned long long> d_counters;  // [0] pairs
  sofk::Comm* comm = nullptr;                 // multi-GPU: owned communicator (sof_comm_init)
  sofk::DBuf<int32_t> shard_i32, shard_send, shard_recv, shard_all;  // sharded-step scratch
  sofk::DBuf<int64_t> shard_i64;
  sofk::DBuf<int64_t> d_scalar;               // small device scalars

  // tets
  int64_t nv = 0, nt = 0;
  bool has_tets = false;
  sofk::DBuf<double> tv;
  sofk::DBuf<int32_t> tt;

  // generic point buffers
  sofk::DBuf<double> pts;
  sofk::DBuf<double> min_op, o_view;
  sofk::DBuf<uint8_t> ext, observed, complete;

  // mesher results
  int64_t n_edges = -1, n_march_tris = -1, mesh_nv = -1, mesh_nt = -1, grid_n = -1;
  int64_t mesh_nres = -1;                // residuals of the last weld (-1: none)
  std::vector<int32_t> delaunay_tets;    // sof_tetrahedralize result (host, 4 per tet)
  sofk::DBuf<char> dl_buf;               // device Delaunay: points, tets (x2), cavity, faces
  sofk::DBuf<double> m_res, res_in;      // welded / pre-weld residuals
  sofk::DBuf<double> grid_opacity;
  sofk::DBuf<int32_t> r_edges, r_tris, m_tris;
  sofk::DBuf<double> r_everts, m_verts;
  int64_t bind_tiles = -1, bind_entries = -1;
  int last_binding_view = -1;

  // instrumentation
  double eval_ms = 0.0;
  int64_t eval_launches = 0;
  bool time_eval = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t user_ev[8] = {};
  // event pool for sync-free phase timing (only while time_eval is set)
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  std::vector<int> span_a, span_b, span_k;
};

namespace sofk {

// ---- k_field.cu -------------------------------------------------------------------------
void scene_prep(sof_ctx* c);
void scene_check_finite(sof_ctx* c, unsigned long long* bad);
const Rec* view_records(sof_ctx* c, int view);
const RecF* view_recf(sof_ctx* c, int view);
const Binding& view_binding(sof_ctx* c, int view, int tile_size, bool live = false);
void bin_by_key(sof_ctx* c, int view, int ts, int tiles_x, int tiles_y, Binding& b,
                bool charge_cache);
void invalidate_view_caches(sof_ctx* c);
void mark_views_stale(sof_ctx* c);
// Evaluates points xyz_dev[n] against views [v0, v1) in order (field_eval.hpp:59-176).
void eval_views(sof_ctx* c, int v0, int v1, int64_t n, const double* xyz_dev, int strategies,
                int tile_size, bool classify_mode, EvalMode mode, double* min_op, uint8_t* ext,
                double* o_out, uint8_t* observed_out, uint8_t* complete_out,
                uint64_t* counters_host);
void finalize_label(sof_ctx* c, int64_t n, const double* min_op, const uint8_t* ext, double* out);
void schedule_points_exact(sof_ctx* c, int view, int64_t n, const double* xyz_dev, int tile_size,
                           int32_t* tile_assignment, std::vector<int32_t>& order,
                           std::vector<int32_t>& key_tile, std::vector<double>& key_depth,
                           std::vector<int32_t>& block_ranges, std::vector<int32_t>& block_to_tile);

// ---- k_mesh.cu --------------------------------------------------------------------------
// Makes asynchronously uploaded tets usable on c->stream (waits, checks the index flag).
void tets_ready(sof_ctx* c);
// Issues up to max_bytes more of a pending sof_set_tets_async upload.
void pump_upload(sof_ctx* c, int64_t max_bytes);
constexpr int64_t kUploadChunk = int64_t(64) << 20;
void check_tet_indices(sof_ctx* c, cudaStream_t st, int64_t nt, const int32_t* tets_dev, int64_t nv, int32_t* bad);
void bisect_cache_views(sof_ctx* c, int v0, int v1, int64_t ne, const int32_t* edges_dev, int strategies,
                        int tile_size);
void march(sof_ctx* c, const double* opacity_dev);
void march_range(sof_ctx* c, const double* opacity_dev, int64_t t0, int64_t t1);
void march_merge(sof_ctx* c, const double* opacity_dev, int world, const int64_t* ecount, const int32_t* edges_all,
                 const int64_t* tcount, const int32_t* tris_all);
void refine(sof_ctx* c, int64_t ne, const int32_t* edges_dev, double* verts_dev, int iterations,
            int strategies, int tile_size, int v0, int v1, uint64_t* counters);
void refine_init(sof_ctx* c, int64_t ne, const int32_t* edges_dev);
void refine_mid(sof_ctx* c, int64_t ne, uint8_t* ext_dev);
void refine_update(sof_ctx* c, int64_t ne, const uint8_t* ext_dev);
void refine_final(sof_ctx* c, int64_t ne, double* verts_dev);
int64_t dedup_first(sof_ctx* c, int64_t n, const double* v, double inv);
// extract_mesh's residuals (extract.hpp:65-72): naive value_at at the refined vertices over
// views [v0, v1), then |value - 0.5|; pointers into c->res_in
double* level_set_values(sof_ctx* c, const sof_extract_opts& o, int v0, int v1);
double* residuals_from_values(sof_ctx* c, const double* values);
double* level_set_residuals(sof_ctx* c, const sof_extract_opts& o, int v0, int v1);
void seed_points(sof_ctx* c, int variant, int cutoff, double filter_scale);
void assemble(sof_ctx* c, int64_t nverts, const double* verts_dev, int64_t ntris,
              const int32_t* tris_dev, double weld_eps, double min_area, const double* residuals_dev = nullptr);

// ---- k_comm.cu ----------------------------------------------------------------------------
void comm_destroy(sof_ctx* c);
// the view- / tet-sharded label -> march -> refine -> weld with c->comm (records ev[1..3])
void extract_sharded(sof_ctx* c, const sof_extract_opts& o, int vb, int ve, uint64_t* cl, uint64_t* cr,
                     cudaEvent_t* ev);

// ---- k_util.cu: phase timing -------------------------------------------------------------
void zero_async(sof_ctx* c, void* p, int64_t bytes);
void fill_f64(sof_ctx* c, double* p, int64_t n, double v);
int prof_mark(sof_ctx* c);                              // -1 when not profiling
void prof_span(sof_ctx* c, int a, int b, int kind);
void prof_collect(sof_ctx* c, double* ms_by_kind);      // syncs, sums, resets

// ---- helpers ----------------------------------------------------------------------------
inline unsigned grid_for(int64_t n, int block) { return unsigned((n + block - 1) / block); }
void sort_pairs_u64(sof_ctx* c, const uint64_t* kin, uint64_t* kout, const int32_t* vin,
                    int32_t* vout, int64_t n, int end_bit);
void sort_pairs_u32(sof_ctx* c, const uint32_t* kin, uint32_t* kout, const int32_t* vin,
                    int32_t* vout, int64_t n, int end_bit);
void exclusive_scan_u32_to_i64(sof_ctx* c, const uint32_t* in, int64_t* out, int64_t n);
void exclusive_scan_i32(sof_ctx* c, const int32_t* in, int32_t* out, int64_t n);
// hand-written scans (k_scan.cu) on c->stream: out[0..n] exclusive, out[n] = total
void scan_u32_i64(sof_ctx* c, const uint32_t* in, int64_t* out, int64_t n);
void scan_i32_i32(sof_ctx* c, const int32_t* in, int32_t* out, int64_t n);
void scan_i64_i64(sof_ctx* c, const int64_t* in, int64_t* out, int64_t n);
int bits_for(uint64_t max_value);
template <typename T>
inline T read_scalar(sof_ctx* c, const T* dev) {
  // through a pinned slot: a pageable read-back is staged by the driver and can queue
  // behind a large asynchronous upload (sof_set_tets_async)
  static_assert(sizeof(T) <= sizeof(c->pinned_scalar[0]), "scalar too large");
  SOF_CUDA(cudaMemcpyAsync(c->pinned_scalar, dev, sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  SOF_CUDA(cudaStreamSynchronize(c->stream));
  T h;
  std::memcpy(&h, c->pinned_scalar, sizeof(T));
  return h;
}
#define SOF_LAUNCHED(c)              \
  do {                               \
    (c)->launches++;                 \
    SOF_CUDA(cudaGetLastError());    \
  } while (0)

}  // namespace sofk

namespace sofk {
// Runs f and maps exceptions to the C-ABI status codes (message in sof_last_error).
template <typename F>
inline int guard(sof_ctx* c, F&& f) {
  try {
    if (c) SOF_CUDA(cudaSetDevice(c->device));
    f();
    return SOF_OK;
  } catch (const InvalidArg& e) {
    if (c) c->err = e.what();
    return SOF_E_INVALID;
  } catch (const std::invalid_argument& e) {
    if (c) c->err = e.what();
    return SOF_E_INVALID;
  } catch (const StateError& e) {
    if (c) c->err = e.what();
    return SOF_E_STATE;
  } catch (const OomError& e) {
    if (c) c->err = e.what();
    return SOF_E_OOM;
  } catch (const NcclError& e) {
    if (c) c->err = e.what();
    return SOF_E_NCCL;
  } catch (const CudaError& e) {
    if (c) c->err = e.what();
    return SOF_E_CUDA;
  } catch (const std::bad_alloc&) {
    if (c) c->err = "host allocation failed";
    return SOF_E_OOM;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return SOF_E_RUNTIME;
  }
}

}  // namespace sofk

