/* sof_cuda.h — C-ABI of libsof_cuda.so, the B200-native SOF hot path.
 *
 * This is the drop-in boundary for the sorted opacity-field evaluator, the
 * Marching-Tetrahedra mesher and the sorted rasterizer of arXiv 2506.19139.
 * The reference (/root/reference/proj/include/sof, header-only C++20, CPU) has
 * no FFI of its own; every entry point below names the reference function it
 * replaces (file:line under proj/include/sof/). The C++ host API in
 * include/sof_b200/*.hpp and the Python package paper_2506_19139_b200 both call
 * only these functions.
 *
 * Conventions
 *   - plain pointers and sizes, no C++ or torch types; host pointers unless the
 *     name ends in _dev (device pointers on the context's GPU);
 *   - every function returns an int status: SOF_OK (0) or a negative SOF_E_*;
 *     sof_last_error(ctx) returns the message (e.g. "non-finite Gaussian
 *     parameters", precompute.hpp:60-63);
 *   - arrays: scene pos[3n], scale[3n], rot_wxyz[4n], opacity[n], dc[3n] (activated
 *     values, GaussianPrimitive gaussian.hpp:12-18); cameras R[9V] row-major
 *     world-to-view, t[3V], intr[4V] = {fx, fy, cx, cy}, wh[2V] = {width, height},
 *     nearfar[2V] (Camera camera.hpp:10-21); points xyz[3n]; tets int32[4nt];
 *   - strategies: bit mask of SOF_TILE_SCHEDULING ... SOF_DEAD_CULL
 *     (EvalStrategies field_eval.hpp:14-23);
 *   - counters: uint64[2] = {pairs, point_view_evals} accumulated into by the call
 *     (EvalCounters field_eval.hpp:25-29, exact reference semantics);
 *   - a context owns one GPU and all device memory; use it from one host thread
 *     at a time; variable-size results stay on the device until copied out with
 *     sof_copy_result.
 */
#ifndef SOF_CUDA_H
#define SOF_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SOF_OK = 0,
  SOF_E_INVALID = -1, /* bad argument: std::invalid_argument in the reference */
  SOF_E_CUDA = -2,    /* CUDA runtime error */
  SOF_E_NCCL = -3,    /* collective error */
  SOF_E_OOM = -4,     /* device allocation failed */
  SOF_E_STATE = -5,   /* missing scene / views / tets, or no result of that kind */
  SOF_E_RUNTIME = -6  /* std::runtime_error in the reference (e.g. "no live Gaussians") */
};

enum {
  SOF_TILE_SCHEDULING = 1,
  SOF_MIN_Z = 2,
  SOF_EARLY_STOP = 4,
  SOF_PRUNE = 8,
  SOF_DEAD_CULL = 16,
  SOF_ALL_STRATEGIES = 31 /* EvalStrategies::all(), field_eval.hpp:22 */
};

enum { SOF_DEPTH_MEDIAN = 0, SOF_DEPTH_EXACT = 1 }; /* DepthMode opacity_field.hpp:199 */

/* result kinds for sof_result_count / sof_copy_result */
enum {
  SOF_R_EDGES = 1,         /* int32[2E]  CrossingEdge{inside, outside} (marching_tets.hpp:16-19) */
  SOF_R_EDGE_VERTS = 2,    /* f64[3E]    MarchingResult::vertices (lerp, then refined) */
  SOF_R_TRIANGLES = 3,     /* int32[3T]  MarchingResult::triangles */
  SOF_R_MESH_VERTS = 4,    /* f64[3V]    Mesh::vertices after assemble_mesh */
  SOF_R_MESH_TRIS = 5,     /* int32[3T]  Mesh::triangles after assemble_mesh */
  SOF_R_GRID_OPACITY = 6,  /* f64[nv]    TetGrid::opacity after label_grid */
  SOF_R_TILE_OFFSETS = 7,  /* int64[T+1] per-tile list offsets of the last binding */
  SOF_R_TILE_ENTRIES = 8,  /* int32[M]   per-tile Gaussian lists (TileBinding, tiles.hpp:88-92) */
  SOF_R_SEEDS = 9,         /* f64[3S]    SeedPointSet::points (seed_points.hpp:24-27) */
  SOF_R_SEED_PROVENANCE = 10, /* uint8[S] SeedPointSet::provenance: 0 centre, 1 bound corner */
  SOF_R_MESH_RESIDUALS = 11,  /* f64[V] Mesh::residuals (mesh.hpp:16), when computed */
  SOF_R_TETS = 12,            /* int32[4T] the tets of the last sof_tetrahedralize */
  SOF_R_CONTRIB_INDEX = 13,   /* int32[C] RayContribution::gaussian_index of sof_collect_contributions */
  SOF_R_CONTRIB_VALUES = 14   /* f64[6C] (t_star, alpha, a, b, c, opacity) per contribution */
};

typedef struct sof_ctx sof_ctx;

/* Options of the fused label -> march -> refine -> weld pipeline
 * (ExtractOptions extract.hpp:12-20 minus the seed/Delaunay producer). */
typedef struct sof_extract_opts {
  int strategies;        /* default SOF_ALL_STRATEGIES */
  int tile_size;         /* default 16 (kDefaultTileSize tiles.hpp:14) */
  int refine_iterations; /* default 8 */
  double weld_eps;       /* default 1e-7 (mesh.hpp:38) */
  double min_area;       /* default 1e-14 (mesh.hpp:38) */
  int view_begin;        /* views [view_begin, view_end) of this rank; -1/-1 = all */
  int view_end;
  int profile;           /* 1: per-kernel device timings (ms_eval_kernel, ms_prep, ...); adds
                            two events per launch and a host-side collection; default 0 */
  int compute_residuals; /* ExtractOptions::compute_residuals (extract.hpp:19,65-72): per mesh
                            vertex |value_at - 0.5| with naive strategies, carried through the
                            weld (result SOF_R_MESH_RESIDUALS); default 0 */
} sof_extract_opts;

/* Per-stage statistics (ExtractStats extract.hpp:22-33) plus device timings. */
typedef struct sof_extract_stats {
  int64_t crossing_edges;
  int64_t march_triangles;
  int64_t mesh_vertices;
  int64_t mesh_triangles;
  uint64_t pairs;            /* label + refine, reference `pairs` semantics */
  uint64_t point_view_evals;
  uint64_t label_pairs;
  uint64_t refine_pairs;
  double ms_label;           /* device time per stage (CUDA events) */
  double ms_march;
  double ms_refine;
  double ms_weld;
  double ms_eval_kernel;     /* summed duration of the opacity-eval kernel launches */
  int64_t eval_launches;     /* number of opacity-eval kernel launches */
  int64_t kernel_launches;   /* all kernels launched by the call */
  double ms_prep;            /* per-view records + Gaussian tile binning (K1, K2) */
  double ms_sched;           /* per-view point scheduling (K3) */
  uint64_t exact_pairs;      /* pairs past the screen-space cull (FP64); 0 unless built with SOF_EVAL_STATS */
  double host_ms_prep;       /* host time spent issuing per-view prep (incl. its one sync) */
  double host_ms_sched;      /* host time spent issuing per-view scheduling */
  uint64_t contrib_pairs;    /* FP64-evaluated pairs with alpha >= 1/255; 0 unless SOF_EVAL_STATS */
  uint64_t scanned_pairs;    /* list entries the evaluation kernels scanned in views that have Gaussians
                                counted without listing (behind / crossing the camera plane), which
                                `pairs` includes; 0 when no view has any */
} sof_extract_stats;

/* ---- context --------------------------------------------------------------- */
int sof_ctx_create(int device, sof_ctx** out);
void sof_ctx_destroy(sof_ctx* ctx);
const char* sof_last_error(const sof_ctx* ctx);
int sof_version(void);
/* number of kernels launched on this context so far (instrumentation) */
int64_t sof_kernel_launches(const sof_ctx* ctx);
/* Gaussians of the resident scene; -1 before sof_set_scene. */
int64_t sof_scene_size(const sof_ctx* ctx);

/* ---- inputs ----------------------------------------------------------------- */
/* Replaces the scene half of ViewSet::build (opacity_field.hpp:26-34) and the
 * view-independent half of precompute (precompute.hpp:57-78): uploads the
 * Gaussians and computes Sigma^-1, the filtered opacity and E on the device.
 * Non-finite positions, scales or opacities are rejected as precompute does
 * (precompute.hpp:60-63: "non-finite Gaussian parameters"); the check runs on the
 * device after the upload, so a rejected call leaves the context without a scene. */
int sof_set_scene(sof_ctx* ctx, int64_t n, const double* pos, const double* scale,
                  const double* rot_wxyz, const double* opacity, const double* dc,
                  double filter_scale);
/* The cameras of the ViewSet. Per-view preprocessing runs lazily on the device. */
int sof_set_views(sof_ctx* ctx, int v, const double* R, const double* t, const double* intr,
                  const int32_t* wh, const double* nearfar);
/* The tetra input (TetGrid delaunay.hpp:14-18: vertices + tetrahedra), resident on the device. */
int sof_set_tets(sof_ctx* ctx, int64_t nv, const double* xyz, int64_t nt, const int32_t* tets);
/* As sof_set_tets, but the tets upload (and their index check) runs on a copy stream
 * while the next label pass, which needs only the vertices, computes; the marching
 * stage waits for it. `tets` must stay valid and unchanged until the next sof_extract /
 * sof_marching_tets returns (pinned memory for the copy to overlap). An out-of-range
 * index is reported by that call (SOF_E_INVALID). */
int sof_set_tets_async(sof_ctx* ctx, int64_t nv, const double* xyz, int64_t nt, const int32_t* tets);
/* HBM the per-view records and tile lists of one step may keep resident (default: half
 * of the free memory at sof_ctx_create). Views past the budget are rebuilt when used,
 * in two scratch slots. */
int sof_set_cache_budget(sof_ctx* ctx, int64_t bytes);

/* ---- per-view preprocessing and binning (parity / inspection) -------------------- */
/* PrecomputedGaussian per Gaussian for one view (precompute.hpp:21-28): 13 doubles
 * {inv_cov[6], b_vec[3], c_scalar, tight_bound, min_z, filtered_opacity}. */
int sof_precompute_view(sof_ctx* ctx, int view, double* out13);
/* build_tile_binding (tiles.hpp:94-146) for one view; lists stay on the device
 * (SOF_R_TILE_OFFSETS / SOF_R_TILE_ENTRIES). */
int sof_tile_binding(sof_ctx* ctx, int view, int tile_size, int64_t* n_tiles, int64_t* n_entries);
/* The evaluation's live-only binding of `view` (dead Gaussians left out): stats[3] =
 * {list entries, Gaussians counted instead of listed in every tile (behind the camera or
 * crossing its plane, tiles.hpp:116-126), listed entries of crossing Gaussians}. */
int sof_live_binding_stats(sof_ctx* ctx, int view, int tile_size, int64_t* stats);
/* schedule_points (tiles.hpp:29-84) for one view, exact (tile, depth, point) order.
 * tile_assignment[n]; order/key_tile/key_depth[n_sched]; block_ranges[2*n_blocks],
 * block_to_tile[n_blocks]. Pass NULL outputs to get the counts first. */
int sof_schedule_points(sof_ctx* ctx, int view, int64_t n, const double* xyz, int tile_size,
                        int64_t* n_sched, int64_t* n_blocks, int32_t* tile_assignment,
                        int32_t* order, int32_t* key_tile, double* key_depth,
                        int32_t* block_ranges, int32_t* block_to_tile);

/* ---- opacity field (FieldEvaluator field_eval.hpp:39-198) --------------------------- */
/* view_opacity (field_eval.hpp:59-111) for n points against one view. */
int sof_view_opacity(sof_ctx* ctx, int view, int64_t n, const double* xyz, int strategies,
                     int tile_size, int classify_mode, double* o, uint8_t* observed,
                     uint8_t* complete, uint64_t* counters);
/* classify_point (field_eval.hpp:114-125), batched. interior[n]. */
int sof_classify_points(sof_ctx* ctx, int64_t n, const double* xyz, int strategies, int tile_size,
                        uint8_t* interior, uint64_t* counters);
/* value_at (field_eval.hpp:128-136), batched (classification mode off). */
int sof_value_at(sof_ctx* ctx, int64_t n, const double* xyz, int strategies, int tile_size,
                 double* out, uint64_t* counters);
/* label_grid (field_eval.hpp:140-176): grid.opacity for nv vertices. */
int sof_label_grid(sof_ctx* ctx, int64_t nv, const double* xyz, int strategies, int tile_size,
                   int classify_mode, double* opacity, uint64_t* counters);

/* Device-resident, view-range building blocks for view-sharded multi-GPU runs:
 * label views [v0, v1) with pruning state carried across them. min_opacity and
 * exterior are read and updated in place (initialise to 1.0 / 0). */
int sof_label_views_dev(sof_ctx* ctx, int v0, int v1, int64_t n, const double* xyz_dev,
                        int strategies, int tile_size, int classify_mode,
                        double* min_opacity_dev, uint8_t* exterior_dev, uint64_t* counters);
/* classification of n points against views [v0, v1): exterior_dev |= exterior. */
int sof_classify_views_dev(sof_ctx* ctx, int v0, int v1, int64_t n, const double* xyz_dev,
                           int strategies, int tile_size, uint8_t* exterior_dev,
                           uint64_t* counters);

/* ---- view-sharded meshing primitives (one process per GPU; the caller runs the
 * collectives, see paper_2506_19139_b200/sharded.py) ------------------------------------ */
/* device pointer of the resident tetra vertices (xyz_dev[3 nv]) */
int sof_tets_vertices_dev(sof_ctx* ctx, const double** xyz_dev, int64_t* nv);
/* out[i] = exterior[i] ? rank : world — all-reduce MIN gives the first exterior rank */
int sof_shard_ext_rank_dev(sof_ctx* ctx, int64_t n, const uint8_t* exterior_dev, int rank,
                           int world, int32_t* out_dev);
/* min_opacity[i] = +inf where rank > first_exterior_rank[i] (views after the first
 * exterior view are pruned in the sequential reference, field_eval.hpp:147) */
int sof_shard_mask_min_dev(sof_ctx* ctx, int64_t n, const int32_t* first_ext_rank_dev, int rank,
                           double* min_opacity_dev);
/* label_grid's final write (field_eval.hpp:173-175) into the resident grid opacity */
int sof_shard_finalize_dev(sof_ctx* ctx, int64_t n, const double* min_opacity_dev,
                           const int32_t* first_ext_rank_dev, int world);
/* marching_tets over the resident tets and grid opacity (results stay resident) */
int sof_march_resident(sof_ctx* ctx, int64_t* n_edges, int64_t* n_tris);
/* Tet-sharded march (one shard of marching_tets, marching_tets.hpp:29-84): the
 * resident labels marched over the tet range [t0, t1) only; edges are numbered in
 * first appearance within the range and the triangles reference them. */
int sof_march_range_resident(sof_ctx* ctx, int64_t t0, int64_t t1, int64_t* n_edges, int64_t* n_tris);
/* Copies the current march result into caller device buffers: edges [2E] (inside,
 * outside vertex id), triangles [3T] (edge ids). */
int sof_march_result_copy_dev(sof_ctx* ctx, int32_t* edges_dst, int32_t* tris_dst);
/* Merge of `world` shard results gathered on this device in shard order (shard r =
 * the r-th contiguous tet range): edges_dev = the shards' edge lists concatenated,
 * tris_dev = their triangles (shard-local edge ids) concatenated. Produces the
 * whole-grid marching_tets result (same edge numbering, triangles and winding) as
 * the resident march result. */
int sof_march_merge_dev(sof_ctx* ctx, int world, const int64_t* edge_counts, const int32_t* edges_dev,
                        const int64_t* tri_counts, const int32_t* tris_dev, int64_t* n_edges, int64_t* n_tris);
/* one phase of binary_search_refine over the resident crossing edges:
 * 0 init brackets, 1 midpoints + classify against views [v0, v1) into exterior_dev
 * (cleared first), 2 update brackets from exterior_dev, 3 write the final vertices */
int sof_refine_phase_dev(sof_ctx* ctx, int phase, uint8_t* exterior_dev, int v0, int v1,
                         int strategies, int tile_size, uint64_t* counters);
/* assemble_mesh over the resident refined vertices / triangles */
int sof_assemble_resident(sof_ctx* ctx, double weld_eps, double min_area, int64_t* n_verts,
                          int64_t* n_tris);

/* ---- mesher ------------------------------------------------------------------------- */
/* marching_tets (marching_tets.hpp:29-84) over the resident tets with the given vertex
 * opacities (host array, nv entries; NULL = use the last label result).
 * Results: SOF_R_EDGES, SOF_R_EDGE_VERTS, SOF_R_TRIANGLES. */
int sof_marching_tets(sof_ctx* ctx, const double* opacity, int64_t* n_edges, int64_t* n_tris);
/* binary_search_refine (marching_tets.hpp:94-114) with classify_point as the interior
 * test, run as `iterations` batched device passes over all crossing edges. edges[2E]
 * and verts[3E] are host arrays; verts is updated in place. Grid vertices come from
 * the resident tets. */
int sof_refine(sof_ctx* ctx, int64_t n_edges, const int32_t* edges, double* verts,
               int iterations, int strategies, int tile_size, uint64_t* counters);
/* assemble_mesh (mesh.hpp:36-79). Results: SOF_R_MESH_VERTS, SOF_R_MESH_TRIS. */
int sof_assemble(sof_ctx* ctx, int64_t n_verts, const double* verts, int64_t n_tris,
                 const int32_t* tris, double weld_eps, double min_area, int64_t* out_verts,
                 int64_t* out_tris);
/* assemble_mesh with its residual passthrough (mesh.hpp:36-79, :66): residuals[nverts]
 * (nullable) are carried to the welded vertices (first appearance); result kind
 * SOF_R_MESH_RESIDUALS. */
int sof_assemble_residuals(sof_ctx* ctx, int64_t nverts, const double* verts, const double* residuals,
                           int64_t ntris, const int32_t* tris, double weld_eps, double min_area,
                           int64_t* out_verts, int64_t* out_tris);
/* extract_mesh's label -> march -> refine -> assemble (extract.hpp:59-78) over the
 * resident scene, views and tets, entirely on the device. */
int sof_extract(sof_ctx* ctx, const sof_extract_opts* opts, sof_extract_stats* stats);
void sof_extract_opts_default(sof_extract_opts* opts);

/* ---- utilities ---------------------------------------------------------------------- */
/* device-side check that 0 <= tets_dev[i] < nv for all 4*nt indices (tets_dev: a
 * 16-byte aligned device array, as cudaMalloc returns; SOF_E_INVALID when it is not or an
 * index is out of range) */
int sof_validate_tets_dev(sof_ctx* ctx, int64_t nt, const int32_t* tets_dev, int64_t nv);
/* CUDA events on the context's stream (slots 0..7) for device-side timing */
int sof_event_record(sof_ctx* ctx, int slot);
int sof_event_elapsed(sof_ctx* ctx, int slot_a, int slot_b, float* ms);
int sof_sync(sof_ctx* ctx);
/* Stream interop (no host synchronisation): sof_stream_wait orders the context's stream
 * after all work enqueued so far on `stream` (a cudaStream_t of the caller, e.g. the
 * stream that filled a buffer the library reads next); sof_get_stream returns the
 * context's stream (cudaStream_t) for the opposite direction. */
int sof_stream_wait(sof_ctx* ctx, void* stream);
int sof_get_stream(sof_ctx* ctx, void** stream);
/* page-lock host buffers so uploads run at full link bandwidth */
int sof_host_register(void* ptr, size_t bytes);
int sof_host_unregister(void* ptr);
/* measured FP64 FMA-pipe throughput (TFLOP/s, 2 FLOP per DFMA): the roofline
 * denominator of the FP64 opacity-evaluation kernel */
int sof_fp64_peak(sof_ctx* ctx, double* tflops);

/* opacity-evaluation kernel: 0 = certified FP32 filter + exact FP64 replay,
 * 1 = FP64 for every pair (default). Both produce bit-identical results and counters. */
int sof_set_eval_path(sof_ctx* ctx, int path);

/* record staging of the FP64 fast loop (default strategies): 0 = every thread loads
 * 16 B of the chunk (default, fastest on B200), 1 = TMA row gather (cp.async.bulk.tensor
 * tile::gather4 over the tile's index list into an mbarrier double buffer). Identical
 * results; an sm_100a implementation choice (the reference has no equivalent). */
int sof_set_staging(sof_ctx* ctx, int mode);

/* ---- multi-GPU: a communicator owned by the context -------------
 * One process per GPU. Rank 0 draws a unique id (an ncclUniqueId, 128 bytes), every rank
 * receives it out of band (e.g. torch.distributed's broadcast) and calls sof_comm_init on
 * its context. From then on sof_extract runs the sharded meshing step on the library
 * stream: views split over the ranks for the label pass and the bisection (MIN / MAX
 * all-reduces merge them exactly), tets split for Marching Tetrahedra (all-gathered
 * edge / triangle lists merged into the whole-grid numbering), weld replicated; every rank
 * ends with the same mesh, identical to the single-GPU one. Counters in the stats are the
 * rank's own. NCCL is resolved at run time (libnccl.so.2); SOF_E_NCCL when absent. */
#define SOF_COMM_ID_BYTES 128
int sof_comm_unique_id(void* id_out /* SOF_COMM_ID_BYTES */);
int sof_comm_init(sof_ctx* ctx, const void* id /* from rank 0's sof_comm_unique_id */, int nranks, int rank);
/* Joins n contexts of ONE process (same device) into an in-process communicator whose
 * collectives are device-side reductions between the contexts' buffers. Each context must
 * then be driven from its own host thread (the collectives rendezvous on the host). For
 * testing the sharded protocol with several ranks where only one GPU exists. */
int sof_comm_init_local(sof_ctx* const* ctxs, int n);
/* nranks / rank of the context (1 / 0 without a communicator); returns 0 = none,
 * 1 = NCCL, 2 = in-process, <0 on error. */
int sof_comm_info(const sof_ctx* ctx, int* nranks, int* rank);
int sof_comm_destroy(sof_ctx* ctx);

/* ---- the tetra-input producer ------------------------------------ */
/* delaunay_tetrahedralize (delaunay.hpp:52-142) of n points (host array) on the device:
 * the reference's incremental Bowyer-Watson in its insertion sequence (same enclosing
 * tetrahedron, in-circumsphere slack, cavity re-closing order and arithmetic), each
 * insertion parallel inside one persistent cooperative kernel, so the tet list — and the
 * mesh numbering MT derives from it — is the reference's. O(n^2) work like the reference:
 * seed sets up to ~10^5 points. *n_tets = T; tets via sof_copy_result(SOF_R_TETS).
 * Errors: "need at least 4 points", "degenerate (coplanar) point set". */
int sof_tetrahedralize(sof_ctx* ctx, int64_t n, const double* pts, int64_t* n_tets);

/* ---- results ------------------------------------------------------------------------ */
int64_t sof_result_count(const sof_ctx* ctx, int kind); /* elements (not bytes); <0 if none */
int sof_copy_result(sof_ctx* ctx, int kind, void* host_dst);

/* ---- sorted rasterizer -------------------------------------------------------------- */
/* render_depth_map (render.hpp:26-51) plus render_pixel's colour / final
 * transmittance / accumulated opacity (opacity_field.hpp:192-219) for one view, with the
 * exact per-pixel (t*, index) sort of collect_contributions (opacity_field.hpp:39-61);
 * every output bit-identical. Outputs [h*w] row-major (rgb [h*w*3]); any may be NULL.
 * stats (nullable) uint64[4] = {tested (pixel, list entry) pairs, contributions, pixels
 * with more than 256 contributions (CTA-wide sort), exact-depth fallbacks}. */
int sof_render_view(sof_ctx* ctx, int view, int depth_mode, int tile_size, double* depth,
                    double* opacity, double* rgb, double* t_final, uint64_t* stats);

/* sof_render_view over views [first_view, first_view + n_views), outputs concatenated in
 * view order (view v's pixels start after the w*h pixels of the views before it); each
 * output nullable. */
int sof_render_views(sof_ctx* ctx, int first_view, int n_views, int depth_mode, double* rgb, double* depth,
                     double* opacity, double* t_final);
/* Per-pixel contribution counts [h*w] of the last sof_render_view of `view` (the length
 * of each pixel's collect_contributions list, opacity_field.hpp:39-61). SOF_E_STATE if
 * that view was not the last one rendered. */
int sof_render_counts(sof_ctx* ctx, int view, uint32_t* counts);

/* Per-pixel resort of sof_render_view. 0 (default): the exact (t*, index) order of
 * collect_contributions (opacity_field.hpp:39-61). K > 0: the K-slot window of
 * windowed_resort (opacity_field.hpp:66-91) applied to each pixel's contributions in
 * arrival order = ascending view-space centre depth (ties by index) -- the streaming
 * k-buffer approximation; libstdc++'s tie order is reproduced (stl_order.cuh). */
int sof_set_render_window(sof_ctx* ctx, int64_t window);

/* collect_contributions (opacity_field.hpp:39-61) for n_rays rays of `view` given by
 * their unit directions dirs[3 n_rays] (the reference reads only ray.direction: the
 * cache is relative to the camera centre). offsets_out[n_rays + 1] (host) receives the
 * list offsets; the lists, each sorted by (t*, index), are the results
 * SOF_R_CONTRIB_INDEX / SOF_R_CONTRIB_VALUES. Every Gaussian is tested (no tiles), on
 * the device. */
int sof_collect_contributions(sof_ctx* ctx, int view, int64_t n_rays, const double* dirs, int64_t* offsets_out);

/* windowed_resort (opacity_field.hpp:66-91) of n_lists arrival-ordered lists (host
 * arrays: offsets[n_lists + 1], t_star[offsets[n_lists]]): order_out[k] is the input
 * position (into t_star) of the element the reference puts at output slot k, ties
 * included. One device thread per list. */
int sof_windowed_resort(sof_ctx* ctx, int64_t n_lists, const int64_t* offsets, const double* t_star,
                        int64_t window, int64_t* order_out);

/* render_pixel (opacity_field.hpp:201-219) of n_lists given contribution lists (host:
 * offsets[n_lists + 1], index[C], values[6C] as SOF_R_CONTRIB_VALUES) with the DC colours
 * dc[3 n_gauss] of `gaussians` (NULL: the resident scene's): color[3 n_lists], depth,
 * accumulated_opacity, t_final [n_lists] (each nullable). One device thread per list. */
int sof_render_pixel(sof_ctx* ctx, int64_t n_lists, const int64_t* offsets, const int32_t* index,
                     const double* values, int64_t n_gauss, const double* dc, int depth_mode, double* color,
                     double* depth, double* acc_opacity, double* t_final);

/* Scratch budget (bytes) of one render band: a frame whose per-pixel contribution slices
 * (16 B per candidate) exceed it is rendered in bands of tiles. 0 restores the default
 * (24 GiB). An sm_100a implementation knob; results do not depend on it. */
int sof_set_render_pool(sof_ctx* ctx, int64_t bytes);

/* normal_from_depth (render.hpp:60-88) of the depth map of the last sof_render_view
 * call for `view`, computed from the device-resident depth (no round trip; the `sof
 * render` CLI pairs the two, sof_cli.cpp:122-125). normal [h*w*3] (zero where
 * invalid), valid [h*w]; either may be NULL. SOF_E_STATE if that view was not the
 * last one rendered. */
int sof_render_normals(sof_ctx* ctx, int view, double* normal, uint8_t* valid);

/* normal_from_depth (render.hpp:60-88) of a caller-supplied depth map [h*w] (NaN = no
 * surface, core.hpp:24-26) with view's camera. */
int sof_normal_from_depth(sof_ctx* ctx, int view, const double* depth, double* normal,
                          uint8_t* valid);

/* gaussian_normal (render.hpp:93-107) for m queries: Gaussian gidx[k] of the scene, ray
 * (origin[3k..], dir[3k..]) at parameter t[k] -> out[3k..]. */
int sof_gaussian_normals(sof_ctx* ctx, int64_t m, const int32_t* gidx, const double* origin,
                         const double* dir, const double* t, double* out);

/* ---- seed points (seed_points.hpp), the producer of the tetra input ------------------ */
enum { SOF_SEED_STP = 0, SOF_SEED_THREE_SIGMA = 1, SOF_SEED_STRETCHED_SIGMA = 2 }; /* BoundingVariant */
enum { SOF_SEED_CUT_NONE = 0, SOF_SEED_CUT_DEAD = 1 };                             /* SeedCutoff */
/* build_seed_points (seed_points.hpp:41-87) over the context's scene: Gaussian centres
 * plus the 8 oriented bounding-box corners, deduplicated on the 1e-9 grid in insertion
 * order, on the device. *n_out = seeds; results SOF_R_SEEDS / SOF_R_SEED_PROVENANCE.
 * "no live Gaussians" (SOF_E_RUNTIME) when nothing survives. */
int sof_seed_points(sof_ctx* ctx, int variant, int cutoff, double filter_scale, int64_t* n_out);

/* ---- scene files (io_scene.hpp) ---------------------------------------------------- */
/* parse_scene (io_scene.hpp:54-134): binary little-endian splatting PLY (x y z,
 * scale_0..2 log, rot_0..3 wxyz, opacity logit, f_dc_0..2; other properties skipped by
 * name) decoded and activated on the device straight into the context's scene, as
 * sof_set_scene would set it (filter_scale as there). *n_out = Gaussians. Errors carry
 * the reference's messages ("scene contains no Gaussians", "big-endian PLY is not
 * supported", "missing required property: ...", "truncated PLY payload", "degenerate
 * rotation quaternion", "non-finite value after activation", "malformed PLY header..."). */
int sof_load_scene_ply(sof_ctx* ctx, const char* path, double filter_scale, int64_t* n_out);

/* The context's scene as GaussianPrimitive fields (SoA; any pointer may be NULL). */
int sof_get_scene(sof_ctx* ctx, double* pos, double* scale, double* rot_wxyz, double* opacity, double* dc);

/* write_scene (io_scene.hpp:138-181) of the context's scene: inverse activations on
 * the device, float32 records; byte-identical to the reference writer. */
int sof_write_scene_ply(sof_ctx* ctx, const char* path);


/* ---- training losses (losses.hpp) --------------------------------------
 * Batched over rays: ray r owns samples [off[r], off[r + 1]) (off[0] = 0, nrays + 1
 * entries). One call evaluates the reference's per-ray function for every ray with the
 * same operation order (per-ray losses and per-sample gradients bit-identical). Host
 * buffers in and out. */
/* distortion_loss (losses.hpp:54-107): loss[nrays], d_alpha / d_t [S] (d_alpha only
 * when attach_w) */
int sof_distortion_loss(sof_ctx* ctx, int64_t nrays, const int64_t* off, const double* alpha, const double* t,
                        double near_plane, double far_plane, int attach_w, double* loss, double* d_alpha,
                        double* d_t);
/* extent_loss (losses.hpp:152-179): loss / skipped per ray, gradients per sample */
int sof_extent_loss(sof_ctx* ctx, int64_t nrays, const int64_t* off, const double* w, const double* a,
                    const double* b, const double* c, const double* bound, double near_plane, double far_plane,
                    double* loss, int32_t* skipped, double* d_a, double* d_b, double* d_c, double* d_w);
/* depth_normal_loss (losses.hpp:119-133): normals [3S], pixel_normals [3 nrays] */
int sof_depth_normal_loss(sof_ctx* ctx, int64_t nrays, const int64_t* off, const double* w, const double* normals,
                          const double* pixel_normals, double* loss, double* d_w, double* d_n);
/* opacity_supervision_loss (losses.hpp:195-229): contribs = 6 doubles per sample in the
 * ray's sorted order (t*, alpha, a, b, c, opacity); depth per ray (NaN = no surface) */
int sof_opacity_supervision_loss(sof_ctx* ctx, int64_t nrays, const int64_t* off, const double* contribs,
                                 const double* depth, double* loss, double* field_value, uint8_t* defined,
                                 double* d_alpha);
/* normal_smoothness_loss (losses.hpp:247-293): row-major W x H maps, xyz / rgb triples;
 * per_channel selects ImageGradientMode::kPerChannel */
int sof_normal_smoothness_loss(sof_ctx* ctx, int width, int height, const double* normals, const uint8_t* valid,
                               const double* image, int per_channel, double* loss, int64_t* pixels_used,
                               double* d_normal);
/* l1_rgb_loss (losses.hpp:305-312) over `pixels` rgb triples */
int sof_l1_rgb_loss(sof_ctx* ctx, int64_t pixels, const double* rendered, const double* reference, double* loss);

#ifdef __cplusplus
}
#endif

#endif /* SOF_CUDA_H */
