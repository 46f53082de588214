// extern "C" wrapper over the UNMODIFIED reference headers (TEST INFRASTRUCTURE).
//
// Compiled in place from /root/reference/proj/include (see oracle/Makefile) into
// oracle/_ref/libsof_ref.so. Only tests/, __graft_entry__.smoke() and bench.py's
// reference / cpu_baseline legs load it — as the checker or the timed CPU
// baseline, never as part of the product path. Every entry point forwards to
// the reference function named in its comment; the only code here is marshalling
// between flat arrays and the reference's Eigen/STL types.
//
// Array conventions (shared with the product C-ABI, include/sof_cuda.h):
//   scene:   pos[3n], scale[3n], rot_wxyz[4n], opacity[n], dc[3n]
//   cameras: R[9V] row-major world-to-view, t[3V], intr[4V] = fx,fy,cx,cy,
//            wh[2V] = width,height, nearfar[2V]
//   strategies mask: 1 tile_scheduling, 2 min_z, 4 early_stop, 8 prune, 16 dead_cull
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "sof/bench.hpp"
#include "sof/extract.hpp"
#include "sof/io_camera.hpp"
#include "sof/io_maps.hpp"
#include "sof/io_mesh.hpp"
#include "sof/io_scene.hpp"
#include "sof/losses.hpp"
#include "sof/render.hpp"
#include "test_util.hpp"

using namespace sof;

namespace {

std::vector<GaussianPrimitive> to_scene(int n, const double* pos, const double* scale,
                                        const double* rot, const double* opa, const double* dc) {
  std::vector<GaussianPrimitive> g(n);
  for (int i = 0; i < n; ++i) {
    g[i].position = Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
    g[i].scale = Vec3(scale[3 * i], scale[3 * i + 1], scale[3 * i + 2]);
    g[i].rotation = Quat(rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]);
    g[i].opacity = opa[i];
    if (dc) g[i].dc_color = Vec3(dc[3 * i], dc[3 * i + 1], dc[3 * i + 2]);
  }
  return g;
}

std::vector<Camera> to_cams(int v, const double* R, const double* t, const double* intr,
                            const int* wh, const double* nf) {
  std::vector<Camera> c(v);
  for (int k = 0; k < v; ++k) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) c[k].rotation(i, j) = R[9 * k + 3 * i + j];
    c[k].translation = Vec3(t[3 * k], t[3 * k + 1], t[3 * k + 2]);
    c[k].fx = intr[4 * k];
    c[k].fy = intr[4 * k + 1];
    c[k].cx = intr[4 * k + 2];
    c[k].cy = intr[4 * k + 3];
    c[k].width = wh[2 * k];
    c[k].height = wh[2 * k + 1];
    if (nf) {
      c[k].near = nf[2 * k];
      c[k].far = nf[2 * k + 1];
    }
  }
  return c;
}

void from_scene(const std::vector<GaussianPrimitive>& g, double* pos, double* scale, double* rot,
                double* opa, double* dc) {
  for (size_t i = 0; i < g.size(); ++i) {
    for (int k = 0; k < 3; ++k) {
      pos[3 * i + k] = g[i].position(k);
      scale[3 * i + k] = g[i].scale(k);
      dc[3 * i + k] = g[i].dc_color(k);
    }
    rot[4 * i] = g[i].rotation.w();
    rot[4 * i + 1] = g[i].rotation.x();
    rot[4 * i + 2] = g[i].rotation.y();
    rot[4 * i + 3] = g[i].rotation.z();
    opa[i] = g[i].opacity;
  }
}

void from_cams(const std::vector<Camera>& c, double* R, double* t, double* intr, int* wh,
               double* nf) {
  for (size_t k = 0; k < c.size(); ++k) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) R[9 * k + 3 * i + j] = c[k].rotation(i, j);
    for (int i = 0; i < 3; ++i) t[3 * k + i] = c[k].translation(i);
    intr[4 * k] = c[k].fx;
    intr[4 * k + 1] = c[k].fy;
    intr[4 * k + 2] = c[k].cx;
    intr[4 * k + 3] = c[k].cy;
    wh[2 * k] = c[k].width;
    wh[2 * k + 1] = c[k].height;
    nf[2 * k] = c[k].near;
    nf[2 * k + 1] = c[k].far;
  }
}

EvalStrategies to_strategies(int mask) {
  EvalStrategies s;
  s.tile_scheduling = mask & 1;
  s.min_z = mask & 2;
  s.early_stop = mask & 4;
  s.prune = mask & 8;
  s.dead_cull = mask & 16;
  return s;
}

std::vector<Vec3> to_points(long n, const double* xyz) {
  std::vector<Vec3> p(n);
  for (long i = 0; i < n; ++i) p[i] = Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
  return p;
}

// Variable-size results: named byte arrays fetched by the caller.
struct Bag {
  std::map<std::string, std::vector<char>> arrays;
  template <typename T>
  void put(const std::string& k, const std::vector<T>& v) {
    auto& a = arrays[k];
    a.resize(v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(a.data(), v.data(), a.size());
  }
  void put_vec3(const std::string& k, const std::vector<Vec3>& v) {
    std::vector<double> f(3 * v.size());
    for (size_t i = 0; i < v.size(); ++i)
      for (int c = 0; c < 3; ++c) f[3 * i + c] = v[i](c);
    put(k, f);
  }
};

thread_local std::string g_err;

}  // namespace

struct sofref_ctx {
  std::vector<GaussianPrimitive> gaussians;
  ViewSet views;
  double filter_scale = 0.0;
};

struct sofref_eval {
  sofref_ctx* ctx;
  std::unique_ptr<FieldEvaluator> eval;
};

extern "C" {

const char* sofref_last_error() { return g_err.c_str(); }

double sofref_exp_probe(double x) { return std::exp(x); }
double sofref_log_probe(double x) { return std::log(x); }

// ---- fixtures from the reference's own tests/test_util.hpp -------------------

/// tu::random_scene(std::mt19937(seed), count, extent)  (test_util.hpp:22-40)
void sofref_random_scene(unsigned seed, int count, double extent, double* pos, double* scale,
                         double* rot, double* opa, double* dc) {
  std::mt19937 rng(seed);
  from_scene(tu::random_scene(rng, count, extent), pos, scale, rot, opa, dc);
}

/// tu::shell_scene (test_util.hpp:43-61)
void sofref_shell_scene(int count, double radius, double scale_v, double opacity, double* pos,
                        double* scale, double* rot, double* opa, double* dc) {
  from_scene(tu::shell_scene(count, radius, scale_v, opacity), pos, scale, rot, opa, dc);
}

/// tu::orbit_cameras (test_util.hpp:72-84)
void sofref_orbit_cameras(int count, double dist, double extent, int res, double* R, double* t,
                          double* intr, int* wh, double* nf) {
  from_cams(tu::orbit_cameras(count, dist, extent, res), R, t, intr, wh, nf);
}

/// tu::axis_cameras (test_util.hpp:87-92)
void sofref_axis_cameras(double dist, double extent, int res, double* R, double* t, double* intr,
                         int* wh, double* nf) {
  from_cams(tu::axis_cameras(dist, extent, res), R, t, intr, wh, nf);
}

/// look_at (camera.hpp:62-79)
void sofref_look_at(const double* eye, const double* target, const double* up, double fx,
                    double fy, int w, int h, double* R, double* t, double* intr, int* wh,
                    double* nf) {
  from_cams({look_at(Vec3(eye[0], eye[1], eye[2]), Vec3(target[0], target[1], target[2]),
                     Vec3(up[0], up[1], up[2]), fx, fy, w, h)},
            R, t, intr, wh, nf);
}

// ---- result bags --------------------------------------------------------------

long sofref_bag_size(void* bag, const char* key) {
  auto* b = static_cast<Bag*>(bag);
  auto it = b->arrays.find(key);
  return it == b->arrays.end() ? -1 : long(it->second.size());
}
void sofref_bag_copy(void* bag, const char* key, void* dst) {
  auto* b = static_cast<Bag*>(bag);
  auto it = b->arrays.find(key);
  if (it != b->arrays.end() && !it->second.empty())
    std::memcpy(dst, it->second.data(), it->second.size());
}
void sofref_bag_free(void* bag) { delete static_cast<Bag*>(bag); }

// ---- scene / view context -------------------------------------------------------

/// ViewSet::build (opacity_field.hpp:26-34) over the given scene and cameras.
sofref_ctx* sofref_create(int n, const double* pos, const double* scale, const double* rot,
                          const double* opa, const double* dc, int v, const double* R,
                          const double* t, const double* intr, const int* wh, const double* nf,
                          double filter_scale, int z_mode) {
  try {
    auto* c = new sofref_ctx;
    c->gaussians = to_scene(n, pos, scale, rot, opa, dc);
    c->filter_scale = filter_scale;
    c->views = ViewSet::build(c->gaussians, to_cams(v, R, t, intr, wh, nf), filter_scale,
                              z_mode ? ZExtentMode::kEigenvalue : ZExtentMode::kDiagonal);
    return c;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void sofref_destroy(sofref_ctx* c) { delete c; }

/// PrecomputedGaussian fields per (view, gaussian): inv_cov[6], b_vec[3],
/// c_scalar, tight_bound, min_z, filtered_opacity  (precompute.hpp:21-28)
void sofref_precompute_dump(const sofref_ctx* c, double* out) {
  size_t k = 0;
  for (const auto& cache : c->views.caches)
    for (const auto& pc : cache) {
      for (int i = 0; i < 6; ++i) out[k++] = pc.inv_cov[i];
      for (int i = 0; i < 3; ++i) out[k++] = pc.b_vec(i);
      out[k++] = pc.c_scalar;
      out[k++] = pc.tight_bound;
      out[k++] = pc.min_z;
      out[k++] = pc.filtered_opacity;
    }
}

/// build_tile_binding (tiles.hpp:94-146) for one view -> bag{offsets:int64[T+1], entries:int32}
void* sofref_tile_binding(const sofref_ctx* c, int view, int tile_size) {
  const TileBinding b =
      build_tile_binding(c->gaussians, c->views.caches[view], c->views.cameras[view], tile_size);
  auto* bag = new Bag;
  std::vector<int64_t> off(1, 0);
  std::vector<int32_t> ent;
  for (const auto& l : b.gaussians_per_tile) {
    ent.insert(ent.end(), l.begin(), l.end());
    off.push_back(int64_t(ent.size()));
  }
  bag->put("offsets", off);
  bag->put("entries", ent);
  bag->put("dims", std::vector<int32_t>{b.tiles_x, b.tiles_y});
  return bag;
}

/// schedule_points (tiles.hpp:29-84) for one view
void* sofref_schedule_points(const sofref_ctx* c, int view, long n, const double* xyz,
                             int tile_size) {
  const TileSchedule s = schedule_points(to_points(n, xyz), c->views.cameras[view], tile_size);
  auto* bag = new Bag;
  bag->put("tile_assignment", s.tile_assignment);
  bag->put("order", s.order);
  std::vector<int32_t> kt;
  std::vector<double> kd;
  for (const auto& [t, d] : s.sorted_keys) {
    kt.push_back(t);
    kd.push_back(d);
  }
  bag->put("key_tile", kt);
  bag->put("key_depth", kd);
  bag->put("block_counts", s.block_counts);
  bag->put("block_to_tile", s.block_to_tile);
  std::vector<int32_t> br;
  for (const auto& [b, e] : s.block_ranges) {
    br.push_back(b);
    br.push_back(e);
  }
  bag->put("block_ranges", br);
  return bag;
}

// ---- field evaluator --------------------------------------------------------------

/// FieldEvaluator(gaussians, views, strategies, tile_size) (field_eval.hpp:41-52)
sofref_eval* sofref_eval_create(sofref_ctx* c, int strategies, int tile_size) {
  auto* e = new sofref_eval;
  e->ctx = c;
  e->eval = std::make_unique<FieldEvaluator>(c->gaussians, c->views, to_strategies(strategies),
                                             tile_size);
  return e;
}
void sofref_eval_destroy(sofref_eval* e) { delete e; }
void sofref_eval_counters(const sofref_eval* e, uint64_t* out) {
  const EvalCounters c = e->eval->counters();
  out[0] = c.pairs;
  out[1] = c.point_view_evals;
}
void sofref_eval_reset_counters(const sofref_eval* e) { e->eval->reset_counters(); }

/// FieldEvaluator::view_opacity (field_eval.hpp:59-111) per point
void sofref_view_opacity(const sofref_eval* e, int view, long n, const double* xyz,
                         int classify_mode, double* o, uint8_t* observed, uint8_t* complete) {
  for (long i = 0; i < n; ++i) {
    bool ob = false, co = true;
    o[i] = e->eval->view_opacity(view, Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]),
                                 classify_mode != 0, ob, co);
    observed[i] = ob;
    complete[i] = co;
  }
}

/// FieldEvaluator::classify_point (field_eval.hpp:114-125)
void sofref_classify_points(const sofref_eval* e, long n, const double* xyz, uint8_t* interior) {
  for (long i = 0; i < n; ++i)
    interior[i] = e->eval->classify_point(Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]));
}

/// FieldEvaluator::value_at (field_eval.hpp:128-136)
void sofref_value_at(const sofref_eval* e, long n, const double* xyz, double* out) {
  for (long i = 0; i < n; ++i)
    out[i] = e->eval->value_at(Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]));
}

/// opacity_at_point (opacity_field.hpp:112-123)
void sofref_opacity_at_point(const sofref_ctx* c, long n, const double* xyz, double* out) {
  for (long i = 0; i < n; ++i)
    out[i] = opacity_at_point(c->views, Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]));
}

/// FieldEvaluator::label_grid (field_eval.hpp:140-176); threads = 0 -> serial
void sofref_label_grid(const sofref_eval* e, long nv, const double* xyz, int classify_mode,
                       int threads, double* out_opacity) {
  TetGrid grid;
  grid.vertices = to_points(nv, xyz);
  std::unique_ptr<ThreadPool> pool;
  if (threads > 0) pool = std::make_unique<ThreadPool>(unsigned(threads));
  e->eval->label_grid(grid, classify_mode != 0, pool.get());
  std::memcpy(out_opacity, grid.opacity.data(), sizeof(double) * nv);
}

// ---- mesher -------------------------------------------------------------------------

/// marching_tets (marching_tets.hpp:29-84) -> bag{edges:int32[2E], vertices:f64[3E], triangles:int32[3T]}
void* sofref_marching_tets(long nv, const double* xyz, long nt, const int32_t* tets,
                           const double* opacity) {
  TetGrid grid;
  grid.vertices = to_points(nv, xyz);
  grid.tetrahedra.resize(nt);
  for (long i = 0; i < nt; ++i)
    for (int k = 0; k < 4; ++k) grid.tetrahedra[i][k] = tets[4 * i + k];
  grid.opacity.assign(opacity, opacity + nv);
  const MarchingResult m = marching_tets(grid);
  auto* bag = new Bag;
  std::vector<int32_t> ed;
  for (const auto& e : m.edges) {
    ed.push_back(e.inside);
    ed.push_back(e.outside);
  }
  std::vector<int32_t> tr;
  for (const auto& t : m.triangles) tr.insert(tr.end(), t.begin(), t.end());
  bag->put("edges", ed);
  bag->put_vec3("vertices", m.vertices);
  bag->put("triangles", tr);
  return bag;
}

/// binary_search_refine (marching_tets.hpp:94-114) with eval.classify_point as
/// the interior callback (extract.hpp:66-68). vertices[3E] are updated in place.
void sofref_refine(const sofref_eval* e, long nv, const double* xyz, long ne, const int32_t* edges,
                   double* vertices, int iterations) {
  TetGrid grid;
  grid.vertices = to_points(nv, xyz);
  MarchingResult m;
  m.edges.resize(ne);
  for (long i = 0; i < ne; ++i) m.edges[i] = {edges[2 * i], edges[2 * i + 1]};
  m.vertices = to_points(ne, vertices);
  binary_search_refine(
      m, grid, [&](const Vec3& x) { return e->eval->classify_point(x); }, iterations);
  for (long i = 0; i < ne; ++i)
    for (int c = 0; c < 3; ++c) vertices[3 * i + c] = m.vertices[i](c);
}

/// assemble_mesh (mesh.hpp:36-79) -> bag{vertices:f64[3V], triangles:int32[3T], residuals}
void* sofref_assemble(long nverts, const double* verts, long ntris, const int32_t* tris,
                      const double* residuals, double weld_eps, double min_area) {
  std::vector<std::array<int, 3>> t(ntris);
  for (long i = 0; i < ntris; ++i) t[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
  std::vector<double> res;
  if (residuals) res.assign(residuals, residuals + nverts);
  const Mesh m = assemble_mesh(to_points(nverts, verts), t, residuals ? &res : nullptr, weld_eps,
                               min_area);
  auto* bag = new Bag;
  bag->put_vec3("vertices", m.vertices);
  std::vector<int32_t> tr;
  for (const auto& x : m.triangles) tr.insert(tr.end(), x.begin(), x.end());
  bag->put("triangles", tr);
  bag->put("residuals", m.residuals);
  return bag;
}

/// extract_mesh stages label -> march -> refine -> assemble (extract.hpp:59-78) on a
/// GIVEN tetra grid (seeds and Delaunay are the out-of-scope producer). Timings in
/// seconds: [label, march, refine, assemble]; counters [pairs, point_view_evals].
void* sofref_extract_tetgrid(sofref_ctx* c, long nv, const double* xyz, long nt,
                             const int32_t* tets, int strategies, int tile_size, int iterations,
                             int threads) {
  using clock = std::chrono::steady_clock;
  auto secs = [](clock::time_point a, clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  };
  TetGrid grid;
  grid.vertices = to_points(nv, xyz);
  grid.tetrahedra.resize(nt);
  for (long i = 0; i < nt; ++i)
    for (int k = 0; k < 4; ++k) grid.tetrahedra[i][k] = tets[4 * i + k];
  std::unique_ptr<ThreadPool> pool;
  if (threads > 0) pool = std::make_unique<ThreadPool>(unsigned(threads));
  const auto t0 = clock::now();
  FieldEvaluator eval(c->gaussians, c->views, to_strategies(strategies), tile_size);
  grid.opacity.assign(grid.vertices.size(), 1.0);
  eval.label_grid(grid, true, pool.get());
  const auto t1 = clock::now();
  MarchingResult march = marching_tets(grid);
  const auto t2 = clock::now();
  binary_search_refine(
      march, grid, [&](const Vec3& x) { return eval.classify_point(x); }, iterations);
  const auto t3 = clock::now();
  const Mesh mesh = assemble_mesh(march.vertices, march.triangles, nullptr);
  const auto t4 = clock::now();
  auto* bag = new Bag;
  bag->put("grid_opacity", grid.opacity);
  std::vector<int32_t> ed;
  for (const auto& e : march.edges) {
    ed.push_back(e.inside);
    ed.push_back(e.outside);
  }
  bag->put("edges", ed);
  bag->put_vec3("refined", march.vertices);
  std::vector<int32_t> rt;
  for (const auto& x : march.triangles) rt.insert(rt.end(), x.begin(), x.end());
  bag->put("march_triangles", rt);
  bag->put_vec3("vertices", mesh.vertices);
  std::vector<int32_t> tr;
  for (const auto& x : mesh.triangles) tr.insert(tr.end(), x.begin(), x.end());
  bag->put("triangles", tr);
  const EvalCounters cnt = eval.counters();
  bag->put("counters", std::vector<uint64_t>{cnt.pairs, cnt.point_view_evals});
  bag->put("seconds", std::vector<double>{secs(t0, t1), secs(t1, t2), secs(t2, t3), secs(t3, t4)});
  return bag;
}

/// build_seed_points + delaunay_tetrahedralize (seed_points.hpp:41-87, delaunay.hpp:52-142):
/// the reference's own tetra-input producer, for small scenes.
/// delaunay_tetrahedralize (delaunay.hpp:52-142) of arbitrary points -> bag{tets:int32}
void* sofref_delaunay(long n, const double* xyz) {
  try {
    std::vector<Vec3> pts(size_t(std::max(n, 0L)));
    for (long i = 0; i < n; ++i) pts[size_t(i)] = Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    const TetGrid grid = delaunay_tetrahedralize(pts);
    auto* bag = new Bag;
    std::vector<int32_t> tt;
    for (const auto& x : grid.tetrahedra) tt.insert(tt.end(), x.begin(), x.end());
    bag->put("tets", tt);
    return bag;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* sofref_seed_delaunay(const sofref_ctx* c, int bounding, int cutoff) {
  try {
    const SeedPointSet seeds = build_seed_points(c->gaussians, BoundingVariant(bounding),
                                                 SeedCutoff(cutoff), c->filter_scale);
    const TetGrid grid = delaunay_tetrahedralize(seeds.points);
    auto* bag = new Bag;
    bag->put_vec3("vertices", grid.vertices);
    std::vector<int32_t> tt;
    for (const auto& x : grid.tetrahedra) tt.insert(tt.end(), x.begin(), x.end());
    bag->put("tets", tt);
    return bag;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// build_seed_points (seed_points.hpp:41-87) -> bag{points f64[3S], provenance u8[S]} or NULL
void* sofref_seed_points(const sofref_ctx* c, int bounding, int cutoff, double filter_scale) {
  try {
    const SeedPointSet seeds =
        build_seed_points(c->gaussians, BoundingVariant(bounding), SeedCutoff(cutoff), filter_scale);
    auto* bag = new Bag;
    bag->put_vec3("points", seeds.points);
    std::vector<uint8_t> prov;
    for (auto p : seeds.provenance) prov.push_back(uint8_t(p));
    bag->put("provenance", prov);
    return bag;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// extract_mesh (extract.hpp:35-86), the full reference pipeline incl. seeds + Delaunay.
void* sofref_extract_full(sofref_ctx* c, int strategies, int tile_size, int iterations,
                          int threads) {
  try {
    ExtractOptions opt;
    opt.strategies = to_strategies(strategies);
    opt.tile_size = tile_size;
    opt.refine_iterations = iterations;
    opt.filter_scale = c->filter_scale;
    std::unique_ptr<ThreadPool> pool;
    if (threads > 0) pool = std::make_unique<ThreadPool>(unsigned(threads));
    ExtractStats st;
    const Mesh mesh = extract_mesh(c->gaussians, c->views, opt, &st, pool.get());
    auto* bag = new Bag;
    bag->put_vec3("vertices", mesh.vertices);
    std::vector<int32_t> tr;
    for (const auto& x : mesh.triangles) tr.insert(tr.end(), x.begin(), x.end());
    bag->put("triangles", tr);
    bag->put("counters", std::vector<uint64_t>{st.counters.pairs, st.counters.point_view_evals});
    return bag;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// write_mesh_ply (io_mesh.hpp:55-73)
int sofref_write_mesh_ply(long nverts, const double* verts, long ntris, const int32_t* tris,
                          const char* path) {
  try {
    Mesh m;
    m.vertices = to_points(nverts, verts);
    m.triangles.resize(ntris);
    for (long i = 0; i < ntris; ++i) m.triangles[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    write_mesh_ply(m, path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

/// write_mesh_obj (io_mesh.hpp:19-29)
int sofref_write_mesh_obj(long nverts, const double* verts, long ntris, const int32_t* tris, const char* path) {
  try {
    Mesh m;
    m.vertices = to_points(nverts, verts);
    m.triangles.resize(ntris);
    for (long i = 0; i < ntris; ++i) m.triangles[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    write_mesh_obj(m, path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

/// save_cameras (io_camera.hpp:65-87)
int sofref_save_cameras(int v, const double* R, const double* t, const double* intr, const int* wh,
                        const double* nf, const char* path) {
  try {
    save_cameras(to_cams(v, R, t, intr, wh, nf), path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

/// load_cameras (io_camera.hpp:17-63): the camera count (arrays filled when it fits `cap`),
/// or -1 with the reference's message.
int sofref_load_cameras(const char* path, int cap, double* R, double* t, double* intr, int* wh,
                        double* nf) {
  try {
    const auto c = load_cameras(path);
    if ((int)c.size() <= cap) from_cams(c, R, t, intr, wh, nf);
    return (int)c.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

/// read_mesh_ply (io_mesh.hpp:75-113) -> bag{vertices f64, triangles int32} or NULL (message in last_error)
void* sofref_read_mesh_ply(const char* path) {
  try {
    const Mesh m = read_mesh_ply(path);
    auto* bag = new Bag;
    std::vector<double> v;
    std::vector<int32_t> t;
    for (const auto& p : m.vertices)
      for (int k = 0; k < 3; ++k) v.push_back(p(k));
    for (const auto& f : m.triangles)
      for (int k = 0; k < 3; ++k) t.push_back(f[k]);
    bag->put("vertices", v);
    bag->put("triangles", t);
    return bag;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// parse_scene (io_scene.hpp:54-134) -> bag{pos, scale, rot (wxyz), opacity, dc} or NULL
void* sofref_parse_scene(const char* path) {
  try {
    const SceneFile sf = parse_scene(path);
    auto* bag = new Bag;
    std::vector<double> pos, scale, rot, op, dc;
    for (const auto& g : sf.gaussians) {
      for (int k = 0; k < 3; ++k) {
        pos.push_back(g.position(k));
        scale.push_back(g.scale(k));
        dc.push_back(g.dc_color(k));
      }
      rot.push_back(g.rotation.w());
      rot.push_back(g.rotation.x());
      rot.push_back(g.rotation.y());
      rot.push_back(g.rotation.z());
      op.push_back(g.opacity);
    }
    bag->put("pos", pos);
    bag->put("scale", scale);
    bag->put("rot", rot);
    bag->put("opacity", op);
    bag->put("dc", dc);
    return bag;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// write_scene (io_scene.hpp:138-181)
int sofref_write_scene(int n, const double* pos, const double* scale, const double* rot, const double* opa,
                       const double* dc, const char* path) {
  try {
    write_scene(to_scene(n, pos, scale, rot, opa, dc), path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---- render -------------------------------------------------------------------------

/// render_depth_map (render.hpp:26-51) for one view. depth/opacity: [h*w] row-major.
/// rows restricts to [row0, row1) (others untouched); threads 0 -> serial.
void sofref_render_depth_map(const sofref_ctx* c, int view, int exact, int row0, int row1,
                             int threads, double* depth, double* opacity) {
  const Camera& cam = c->views.cameras[view];
  const auto& cache = c->views.caches[view];
  const DepthMode mode = exact ? DepthMode::kExact : DepthMode::kMedian;
  auto render_row = [&](int y) {
    // identical body to render.hpp:33-43
    for (int x = 0; x < cam.width; ++x) {
      const Ray ray = ray_through_pixel(cam, x + 0.5, y + 0.5);
      const auto contribs = collect_contributions(cache, ray);
      double d = kNoSurface, o = 0.0;
      if (mode == DepthMode::kMedian) {
        if (auto m = median_depth(contribs)) d = *m;
      } else {
        if (auto m = exact_depth(contribs)) d = m->t;
      }
      if (!is_no_surface(d)) o = opacity_along_ray(contribs, d);
      depth[size_t(y) * cam.width + x] = d;
      opacity[size_t(y) * cam.width + x] = o;
    }
  };
  if (row0 == 0 && row1 == cam.height) {
    // the reference entry point itself
    std::unique_ptr<ThreadPool> pool;
    if (threads > 0) pool = std::make_unique<ThreadPool>(unsigned(threads));
    const DepthMap m = render_depth_map(cache, cam, mode, pool.get());
    std::memcpy(depth, m.depth.data.data(), sizeof(double) * m.depth.data.size());
    std::memcpy(opacity, m.opacity.data.data(), sizeof(double) * m.opacity.data.size());
    return;
  }
  if (threads > 0) {
    ThreadPool pool{unsigned(threads)};
    pool.parallel_for(row0, row1, render_row);
  } else {
    for (int y = row0; y < row1; ++y) render_row(y);
  }
}

/// collect_contributions + render_pixel (opacity_field.hpp:39-61, 201-219) for a list of
/// pixels (px, py integer indices; ray through the pixel centre as render.hpp:33).
/// out: color[3n], depth[n], acc_opacity[n], t_final[n], n_contrib[n]
void sofref_render_pixels(const sofref_ctx* c, int view, int exact, long n, const int32_t* pix,
                          double* color, double* depth, double* acc, double* tfinal,
                          int32_t* ncontrib) {
  const Camera& cam = c->views.cameras[view];
  const auto& cache = c->views.caches[view];
  for (long i = 0; i < n; ++i) {
    const Ray ray = ray_through_pixel(cam, pix[2 * i] + 0.5, pix[2 * i + 1] + 0.5);
    const auto contribs = collect_contributions(cache, ray);
    const PixelOutputs p =
        render_pixel(contribs, c->gaussians, exact ? DepthMode::kExact : DepthMode::kMedian);
    for (int k = 0; k < 3; ++k) color[3 * i + k] = p.color(k);
    depth[i] = p.depth;
    acc[i] = p.accumulated_opacity;
    tfinal[i] = p.transmittance_final;
    ncontrib[i] = int32_t(contribs.size());
  }
}

/// The K-window resort render mode: per pixel collect_contributions, re-ordered into
/// arrival order by view-space centre depth (ties by index; a strict total order, so any
/// sort gives it), then windowed_resort(window) (opacity_field.hpp:66-91) and render_pixel.
void sofref_render_pixels_windowed(const sofref_ctx* c, int view, int exact, long window, long n,
                                   const int32_t* pix, double* color, double* depth, double* acc,
                                   double* tfinal, int32_t* ncontrib) {
  const Camera& cam = c->views.cameras[view];
  const auto& cache = c->views.caches[view];
  std::vector<double> zc(c->gaussians.size());
  for (size_t i = 0; i < zc.size(); ++i) zc[i] = cam.to_view(c->gaussians[i].position).z();
  for (long i = 0; i < n; ++i) {
    const Ray ray = ray_through_pixel(cam, pix[2 * i] + 0.5, pix[2 * i + 1] + 0.5);
    auto contribs = collect_contributions(cache, ray);
    std::sort(contribs.begin(), contribs.end(), [&](const RayContribution& l, const RayContribution& r) {
      const double a = zc[size_t(l.gaussian_index)], b = zc[size_t(r.gaussian_index)];
      return a < b || (a == b && l.gaussian_index < r.gaussian_index);
    });
    contribs = windowed_resort(std::move(contribs), size_t(window));
    const PixelOutputs p =
        render_pixel(contribs, c->gaussians, exact ? DepthMode::kExact : DepthMode::kMedian);
    for (int k = 0; k < 3; ++k) color[3 * i + k] = p.color(k);
    depth[i] = p.depth;
    acc[i] = p.accumulated_opacity;
    tfinal[i] = p.transmittance_final;
    ncontrib[i] = int32_t(contribs.size());
  }
}

/// windowed_resort (opacity_field.hpp:66-91) of one list given (t*, index) in arrival order;
/// out_idx[n] = the gaussian_index sequence it returns.
void sofref_windowed_resort(long n, const double* t, const int32_t* idx, long window, int32_t* out_idx) {
  std::vector<RayContribution> in(size_t(std::max(n, 0L)));
  for (long i = 0; i < n; ++i) {
    in[size_t(i)].t_star = t[i];
    in[size_t(i)].gaussian_index = idx[i];
  }
  const auto out = windowed_resort(std::move(in), size_t(window));
  for (size_t i = 0; i < out.size(); ++i) out_idx[i] = out[i].gaussian_index;
}

/// render_pixel (opacity_field.hpp:201-219) of given contribution lists:
/// vals = 6 doubles per contribution (t*, alpha, a, b, c, opacity).
void sofref_render_pixel_lists(const sofref_ctx* c, int exact, long nl, const int64_t* off, const int32_t* idx,
                               const double* vals, double* color, double* depth, double* acc, double* tfinal) {
  for (long l = 0; l < nl; ++l) {
    std::vector<RayContribution> rc;
    for (int64_t k = off[l]; k < off[l + 1]; ++k) {
      RayContribution r;
      r.gaussian_index = idx[k];
      r.t_star = vals[6 * k];
      r.alpha = vals[6 * k + 1];
      r.a = vals[6 * k + 2];
      r.b = vals[6 * k + 3];
      r.c = vals[6 * k + 4];
      r.opacity = vals[6 * k + 5];
      rc.push_back(r);
    }
    const PixelOutputs p = render_pixel(rc, c->gaussians, exact ? DepthMode::kExact : DepthMode::kMedian);
    for (int k = 0; k < 3; ++k) color[3 * l + k] = p.color(k);
    depth[l] = p.depth;
    acc[l] = p.accumulated_opacity;
    tfinal[l] = p.transmittance_final;
  }
}

/// normal_from_depth (render.hpp:60-88) of a [h*w] depth map for view's camera.
/// out: normal[3*h*w] (zero where invalid), valid[h*w]
void sofref_normal_from_depth(const sofref_ctx* c, int view, const double* depth, double* normal,
                              uint8_t* valid) {
  const Camera& cam = c->views.cameras[view];
  Grid2D<double> g(cam.width, cam.height, 0.0);
  std::memcpy(g.data.data(), depth, sizeof(double) * g.data.size());
  const NormalMap nm = normal_from_depth(g, cam);
  for (size_t i = 0; i < nm.normal.data.size(); ++i) {
    for (int k = 0; k < 3; ++k) normal[3 * i + k] = nm.normal.data[i](k);
    valid[i] = nm.valid.data[i];
  }
}

/// gaussian_normal (render.hpp:93-107) for m (gaussian, ray origin, ray direction, t)
void sofref_gaussian_normals(const sofref_ctx* c, long m, const int32_t* gidx, const double* o,
                             const double* d, const double* t, double* out) {
  for (long k = 0; k < m; ++k) {
    const Ray ray{Vec3(o[3 * k], o[3 * k + 1], o[3 * k + 2]), Vec3(d[3 * k], d[3 * k + 1], d[3 * k + 2])};
    const Vec3 n = gaussian_normal(c->gaussians[gidx[k]], ray, t[k]);
    for (int i = 0; i < 3; ++i) out[3 * k + i] = n(i);
  }
}

/// The reference `sof render` per-view output (sof_cli.cpp:122-130): render_depth_map,
/// normal_from_depth, and the two float maps written by write_float_map.
void sofref_render_maps(const sofref_ctx* c, int view, int exact, int threads, const char* depth_path,
                        const char* normal_path) {
  const Camera& cam = c->views.cameras[view];
  std::unique_ptr<ThreadPool> pool;
  if (threads > 0) pool = std::make_unique<ThreadPool>(unsigned(threads));
  const DepthMap dm = render_depth_map(c->views.caches[view], cam,
                                       exact ? DepthMode::kExact : DepthMode::kMedian, pool.get());
  const NormalMap nm = normal_from_depth(dm.depth, cam);
  write_float_map(depth_to_map(dm), depth_path);
  write_float_map(normals_to_map(nm), normal_path);
}

/// write_float_map (io_maps.hpp:30-38) of a raw float buffer; 0 on success, 1 on throw
int sofref_write_float_map(int w, int h, int ch, const float* data, const char* path) {
  FloatMap m;
  m.width = w;
  m.height = h;
  m.channels = ch;
  m.data.assign(data, data + size_t(std::max(w, 0)) * std::max(h, 0) * std::max(ch, 0));
  try {
    write_float_map(m, path);
  } catch (...) {
    return 1;
  }
  return 0;
}

/// collect_contributions (opacity_field.hpp:39-61) for one pixel ->
/// bag{index:int32, t_star/alpha/a/b/c/opacity: f64}
void* sofref_collect_contributions(const sofref_ctx* c, int view, int px, int py) {
  const Camera& cam = c->views.cameras[view];
  const Ray ray = ray_through_pixel(cam, px + 0.5, py + 0.5);
  const auto contribs = collect_contributions(c->views.caches[view], ray);
  auto* bag = new Bag;
  std::vector<int32_t> idx;
  std::vector<double> ts, al, a, b, cc, op;
  for (const auto& rc : contribs) {
    idx.push_back(rc.gaussian_index);
    ts.push_back(rc.t_star);
    al.push_back(rc.alpha);
    a.push_back(rc.a);
    b.push_back(rc.b);
    cc.push_back(rc.c);
    op.push_back(rc.opacity);
  }
  bag->put("index", idx);
  bag->put("t_star", ts);
  bag->put("alpha", al);
  bag->put("a", a);
  bag->put("b", b);
  bag->put("c", cc);
  bag->put("opacity", op);
  return bag;
}


// ---- training losses (losses.hpp), one reference call per ray / image ---------

void sofref_distortion_loss(long nrays, const int64_t* off, const double* alpha, const double* t, double near_plane,
                            double far_plane, int attach_w, double* loss, double* d_alpha, double* d_t) {
  for (long r = 0; r < nrays; ++r) {
    std::vector<DistortionSample> s;
    for (int64_t i = off[r]; i < off[r + 1]; ++i) s.push_back({alpha[i], t[i]});
    const auto out = distortion_loss(s, near_plane, far_plane, attach_w != 0);
    loss[r] = out.loss;
    for (size_t k = 0; k < s.size(); ++k) {
      d_t[off[r] + k] = out.d_t[k];
      if (attach_w) d_alpha[off[r] + k] = out.d_alpha[k];
    }
  }
}

void sofref_extent_loss(long nrays, const int64_t* off, const double* w, const double* a, const double* b,
                        const double* c, const double* bound, double near_plane, double far_plane, double* loss,
                        int32_t* skipped, double* d_a, double* d_b, double* d_c, double* d_w) {
  for (long r = 0; r < nrays; ++r) {
    std::vector<ExtentSample> s;
    for (int64_t i = off[r]; i < off[r + 1]; ++i) s.push_back({w[i], a[i], b[i], c[i], bound[i]});
    const auto out = extent_loss(s, near_plane, far_plane);
    loss[r] = out.loss;
    skipped[r] = out.skipped;
    for (size_t k = 0; k < s.size(); ++k) {
      d_a[off[r] + k] = out.d_a[k];
      d_b[off[r] + k] = out.d_b[k];
      d_c[off[r] + k] = out.d_c[k];
      d_w[off[r] + k] = out.d_w[k];
    }
  }
}

void sofref_depth_normal_loss(long nrays, const int64_t* off, const double* w, const double* normals,
                              const double* pixel_normals, double* loss, double* d_w, double* d_n) {
  for (long r = 0; r < nrays; ++r) {
    std::vector<double> ws;
    std::vector<Vec3> ns;
    for (int64_t i = off[r]; i < off[r + 1]; ++i) {
      ws.push_back(w[i]);
      ns.push_back(Vec3(normals[3 * i], normals[3 * i + 1], normals[3 * i + 2]));
    }
    const Vec3 pn(pixel_normals[3 * r], pixel_normals[3 * r + 1], pixel_normals[3 * r + 2]);
    const auto out = depth_normal_loss(ws, ns, pn);
    loss[r] = out.loss;
    for (size_t k = 0; k < ws.size(); ++k) {
      d_w[off[r] + k] = out.d_w[k];
      for (int q = 0; q < 3; ++q) d_n[3 * (off[r] + k) + q] = out.d_n[k](q);
    }
  }
}

void sofref_opacity_supervision_loss(long nrays, const int64_t* off, const double* contribs, const double* depth,
                                     double* loss, double* field, uint8_t* defined, double* d_alpha) {
  for (long r = 0; r < nrays; ++r) {
    std::vector<RayContribution> cs;
    for (int64_t i = off[r]; i < off[r + 1]; ++i) {
      RayContribution rc;
      rc.gaussian_index = int(i - off[r]);
      rc.t_star = contribs[6 * i];
      rc.alpha = contribs[6 * i + 1];
      rc.a = contribs[6 * i + 2];
      rc.b = contribs[6 * i + 3];
      rc.c = contribs[6 * i + 4];
      rc.opacity = contribs[6 * i + 5];
      cs.push_back(rc);
    }
    const auto out = opacity_supervision_loss(cs, depth[r]);
    loss[r] = out.loss;
    field[r] = out.field_value;
    defined[r] = out.defined ? 1 : 0;
    for (size_t k = 0; k < cs.size(); ++k) d_alpha[off[r] + k] = out.defined ? out.d_alpha[k] : 0.0;
  }
}

void sofref_normal_smoothness_loss(int width, int height, const double* normals, const uint8_t* valid,
                                   const double* image, int per_channel, double* loss, int64_t* used,
                                   double* d_normal) {
  NormalMap nm;
  nm.normal = Grid2D<Vec3>(width, height, Vec3::Zero());
  nm.valid = Grid2D<unsigned char>(width, height, 0);
  Grid2D<Vec3> img(width, height, Vec3::Zero());
  for (size_t p = 0; p < size_t(width) * height; ++p) {
    nm.normal.data[p] = Vec3(normals[3 * p], normals[3 * p + 1], normals[3 * p + 2]);
    nm.valid.data[p] = valid[p];
    img.data[p] = Vec3(image[3 * p], image[3 * p + 1], image[3 * p + 2]);
  }
  const auto out = normal_smoothness_loss(nm, img, per_channel ? ImageGradientMode::kPerChannel
                                                               : ImageGradientMode::kLuminance);
  *loss = out.loss;
  *used = out.pixels_used;
  for (size_t p = 0; p < size_t(width) * height; ++p)
    for (int q = 0; q < 3; ++q) d_normal[3 * p + q] = out.d_normal.data[p](q);
}

double sofref_l1_rgb_loss(long pixels, const double* a, const double* b) {
  Grid2D<Vec3> ga(int(pixels), 1, Vec3::Zero()), gb(int(pixels), 1, Vec3::Zero());
  for (long p = 0; p < pixels; ++p) {
    ga.data[p] = Vec3(a[3 * p], a[3 * p + 1], a[3 * p + 2]);
    gb.data[p] = Vec3(b[3 * p], b[3 * p + 1], b[3 * p + 2]);
  }
  return l1_rgb_loss(ga, gb);
}

}  // extern "C"
