/* sof_oracle.h — C restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * Plain C11, scalar, single-threaded. Each function restates one reference
 * function (cited file:line under /root/reference/proj/include/sof/) with the
 * same double-precision operation order, the Eigen-API semantics pinned in
 * oracle/eigen_shim/Eigen/Dense, and the framework's sof_exp/sof_log. It is
 * pinned against the reference compiled in place (oracle/_ref) and the golden
 * fixtures in tests/golden/. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may call it, and only as the checker.
 *
 * Arrays: scene pos[3n] scale[3n] rot_wxyz[4n] opacity[n] dc[3n]; cameras
 * R[9V] t[3V] intr[4V] wh[2V]; strategies mask 1 tile 2 min_z 4 early_stop
 * 8 prune 16 dead_cull; counters[2] = {pairs, point_view_evals} (accumulated).
 */
#ifndef SOF_ORACLE_H
#define SOF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sofo_scene {
  int64_t n;
  const double *pos, *scale, *rot, *opacity, *dc;
  double filter_scale;
} sofo_scene;

typedef struct sofo_cams {
  int v;
  const double *R, *t, *intr;
  const int32_t* wh;
} sofo_cams;

/* PrecomputedGaussian for all Gaussians and one view: 13 doubles each
 * {inv_cov[6], b_vec[3], c, tight_bound, min_z, filtered_opacity} (precompute.hpp:57-78). */
void sofo_precompute(const sofo_scene* s, const sofo_cams* c, int view, double* out13);

/* build_tile_binding (tiles.hpp:94-146): offsets[T+1]; entries (capacity cap) ;
 * returns the number of entries (or -needed when cap is too small). */
int64_t sofo_tile_binding(const sofo_scene* s, const sofo_cams* c, int view, int tile_size,
                          int64_t* offsets, int32_t* entries, int64_t cap);

/* FieldEvaluator::view_opacity (field_eval.hpp:59-111) for n points. */
void sofo_view_opacity(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                       int view, int64_t n, const double* xyz, int classify_mode, double* o,
                       uint8_t* observed, uint8_t* complete, uint64_t* counters);

/* label_grid (field_eval.hpp:140-176). */
void sofo_label_grid(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                     int64_t nv, const double* xyz, int classify_mode, double* opacity,
                     uint64_t* counters);

/* label_grid's per-view loop (field_eval.hpp:145-172) over the given cameras with
 * caller-owned state (min_opacity in/out, exterior in/out), without the final write. */
void sofo_label_state(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                      int64_t nv, const double* xyz, int classify_mode, double* min_opacity,
                      uint8_t* exterior, uint64_t* counters);

/* classify_point (field_eval.hpp:114-125) and value_at (:128-136), batched. */
void sofo_classify_points(const sofo_scene* s, const sofo_cams* c, int strategies,
                          int tile_size, int64_t n, const double* xyz, uint8_t* interior,
                          uint64_t* counters);
void sofo_value_at(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                   int64_t n, const double* xyz, double* out, uint64_t* counters);

/* marching_tets (marching_tets.hpp:29-84). Capacities: edges/verts 4*nt, tris 2*nt.
 * Returns edges count; *n_tris receives the triangle count. */
int64_t sofo_marching_tets(int64_t nv, const double* xyz, int64_t nt, const int32_t* tets,
                           const double* opacity, int32_t* edges, double* verts, int32_t* tris,
                           int64_t* n_tris);

/* binary_search_refine (marching_tets.hpp:94-114) with classify_point as interior test. */
void sofo_refine(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                 const double* grid_xyz, int64_t ne, const int32_t* edges, double* verts,
                 int iterations, uint64_t* counters);

/* assemble_mesh (mesh.hpp:36-79). Outputs sized like the inputs; returns the vertex
 * count, *out_ntris the triangle count. */
int64_t sofo_assemble(int64_t nverts, const double* verts, int64_t ntris, const int32_t* tris,
                      double weld_eps, double min_area, double* out_verts, int32_t* out_tris,
                      int64_t* out_ntris);

/* render_pixel over collect_contributions for one pixel (opacity_field.hpp:39-61, 132-166,
 * 201-219); out[6] = {r, g, b, depth (NaN none), accumulated opacity, T_final};
 * returns the contribution count. */
int64_t sofo_render_pixel(const sofo_scene* s, const sofo_cams* c, int view, int px, int py,
                          int exact_depth, double* out6);

#ifdef __cplusplus
}
#endif

#endif
