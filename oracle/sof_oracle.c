/* sof_oracle.c — C restatement of the SOF hot path (TEST INFRASTRUCTURE).
 *
 * See sof_oracle.h. Build: gcc -std=c11 -O2 -ffp-contract=off (oracle/Makefile).
 * Every floating-point expression keeps the reference's C++ evaluation order
 * (left-associative sums, no contraction) and the Eigen-API semantics pinned in
 * oracle/eigen_shim/Eigen/Dense; exp/log are sof_exp/sof_log
 * (paper_2506_19139_b200/csrc/sof_math.h), which oracle/ref_interpose.cpp also
 * routes the compiled reference through. Pinned by tests/test_oracle_cpu.py.
 */
#include "sof_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_2506_19139_b200/csrc/sof_math.h"

#define K_MIN_ALPHA (1.0 / 255.0) /* core.hpp:18 */
#define K_MAX_ALPHA 0.999         /* core.hpp:22 */
#define K_MIN_SCALE 1e-8          /* gaussian.hpp:20 */

typedef struct {
  double R[9], t[3], fx, fy, cx, cy, center[3];
  int w, h;
} Cam;

/* PrecomputedGaussian (precompute.hpp:21-28) */
typedef struct {
  double ic[6], b[3], c, E, zmin, op;
} PC;

/* Camera fields (camera.hpp:10-21); center() = (-R^T) t (camera.hpp:20) */
static Cam load_cam(const sofo_cams* c, int v) {
  Cam m;
  memcpy(m.R, c->R + 9 * v, sizeof m.R);
  memcpy(m.t, c->t + 3 * v, sizeof m.t);
  m.fx = c->intr[4 * v];
  m.fy = c->intr[4 * v + 1];
  m.cx = c->intr[4 * v + 2];
  m.cy = c->intr[4 * v + 3];
  m.w = c->wh[2 * v];
  m.h = c->wh[2 * v + 1];
  for (int i = 0; i < 3; ++i)
    m.center[i] = (-m.R[i]) * m.t[0] + (-m.R[3 + i]) * m.t[1] + (-m.R[6 + i]) * m.t[2];
  return m;
}

/* Camera::to_view (camera.hpp:19), component i */
static double to_view(const Cam* m, int i, const double* x) {
  return m->R[3 * i] * x[0] + m->R[3 * i + 1] * x[1] + m->R[3 * i + 2] * x[2] + m->t[i];
}

/* Quaternion::toRotationMatrix (Eigen), q = (w, x, y, z) */
static void rotation(const double* q, double* r) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  r[0] = 1.0 - (tyy + tzz);
  r[1] = txy - twz;
  r[2] = txz + twy;
  r[3] = txy + twz;
  r[4] = 1.0 - (txx + tzz);
  r[5] = tyz - twx;
  r[6] = txz - twy;
  r[7] = tyz + twx;
  r[8] = 1.0 - (txx + tyy);
}

/* (r * diag(d)) * r^T with Eigen's diagonal product and row-times-column sums */
static void r_d_rt(const double* r, const double* d, double* out) {
  double m[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[3 * i + j] = r[3 * i + j] * d[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      out[3 * i + j] = m[3 * i] * r[3 * j] + m[3 * i + 1] * r[3 * j + 1] + m[3 * i + 2] * r[3 * j + 2];
}

/* Matrix3d::determinant (Eigen bruteforce_det3) */
static double det3(const double* m) {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}

/* precompute (precompute.hpp:57-78) with covariance (gaussian.hpp:23-26),
 * filtered_opacity (gaussian.hpp:67-73), tight_bound (gaussian.hpp:60-64) and
 * z_extent_sigma kDiagonal (precompute.hpp:49-55). */
static void precompute_one(const sofo_scene* s, int64_t i, const Cam* cam, PC* pc) {
  const double* p = s->pos + 3 * i;
  const double* sc = s->scale + 3 * i;
  double r[9], inv_cov[9], cov[9];
  rotation(s->rot + 4 * i, r);
  double d[3];
  for (int k = 0; k < 3; ++k) {
    const double sk = sc[k] < K_MIN_SCALE ? K_MIN_SCALE : sc[k]; /* cwiseMax(kMinScale) */
    d[k] = 1.0 / (sk * sk);
  }
  r_d_rt(r, d, inv_cov);
  pc->ic[0] = inv_cov[0];
  pc->ic[1] = inv_cov[1];
  pc->ic[2] = inv_cov[2];
  pc->ic[3] = inv_cov[4];
  pc->ic[4] = inv_cov[5];
  pc->ic[5] = inv_cov[8];
  double delta[3];
  for (int k = 0; k < 3; ++k) delta[k] = cam->center[k] - p[k];
  for (int k = 0; k < 3; ++k)
    pc->b[k] = inv_cov[3 * k] * delta[0] + inv_cov[3 * k + 1] * delta[1] + inv_cov[3 * k + 2] * delta[2];
  pc->c = delta[0] * pc->b[0] + delta[1] * pc->b[1] + delta[2] * pc->b[2];
  const double s2[3] = {sc[0] * sc[0], sc[1] * sc[1], sc[2] * sc[2]};
  r_d_rt(r, s2, cov);
  if (s->filter_scale <= 0.0) {
    pc->op = s->opacity[i];
  } else {
    double cf[9];
    for (int k = 0; k < 9; ++k) cf[k] = cov[k] + s->filter_scale * ((k % 4 == 0) ? 1.0 : 0.0);
    pc->op = s->opacity[i] * sqrt(det3(cov) / det3(cf));
  }
  if (pc->op < K_MIN_ALPHA) {
    pc->E = 0.0;
  } else {
    const double v = 2.0 * sof_log(255.0 * pc->op);
    pc->E = sqrt(v < 0.0 ? 0.0 : v);
  }
  double wc[3];
  for (int j = 0; j < 3; ++j) wc[j] = cam->R[6] * cov[j] + cam->R[7] * cov[3 + j] + cam->R[8] * cov[6 + j];
  const double czz = wc[0] * cam->R[6] + wc[1] * cam->R[7] + wc[2] * cam->R[8];
  pc->zmin = to_view(cam, 2, p) - pc->E * sqrt(czz);
}

void sofo_precompute(const sofo_scene* s, const sofo_cams* c, int view, double* out13) {
  const Cam cam = load_cam(c, view);
  for (int64_t i = 0; i < s->n; ++i) {
    PC pc;
    precompute_one(s, i, &cam, &pc);
    double* o = out13 + 13 * i;
    memcpy(o, pc.ic, 6 * sizeof(double));
    memcpy(o + 6, pc.b, 3 * sizeof(double));
    o[9] = pc.c;
    o[10] = pc.E;
    o[11] = pc.zmin;
    o[12] = pc.op;
  }
}

/* ---- tile binding (tiles.hpp:94-146) ------------------------------------------------ */

/* int(x) as the x86-64 reference binary computes it (cvttsd2si) */
static int x86_int(double x) {
  return (x >= -2147483648.0 && x < 2147483648.0) ? (int)x : (int)0x80000000;
}

static const PC* g_sort_pc; /* comparator context (single-threaded oracle) */

static int cmp_minz(const void* a, const void* b) {
  const int l = *(const int32_t*)a, r = *(const int32_t*)b;
  const double zl = g_sort_pc[l].zmin, zr = g_sort_pc[r].zmin;
  if (zl != zr) return zl < zr ? -1 : 1;
  return (l > r) - (l < r);
}

typedef struct {
  int tiles_x, tiles_y, tile_size;
  int64_t* off;
  int32_t* ent;
} Binding;

static int rect_of(const sofo_scene* s, int64_t gi, const PC* pc, const Cam* cam, int ts, int tiles_x,
                   int tiles_y, int* tx0, int* tx1, int* ty0, int* ty1) {
  const double r = pc->E;
  if (r <= 0.0) return 0;
  double rot[9];
  rotation(s->rot + 4 * gi, rot);
  const double* p = s->pos + 3 * gi;
  const double* sc = s->scale + 3 * gi;
  double min_x = 1e300, max_x = -1e300, min_y = 1e300, max_y = -1e300;
  int crosses = 0;
  for (int mask = 0; mask < 8; ++mask) {
    const double l[3] = {r * sc[0] * (double)((mask & 1) ? 1 : -1),
                         r * sc[1] * (double)((mask & 2) ? 1 : -1),
                         r * sc[2] * (double)((mask & 4) ? 1 : -1)};
    double w[3];
    for (int k = 0; k < 3; ++k) w[k] = p[k] + (rot[3 * k] * l[0] + rot[3 * k + 1] * l[1] + rot[3 * k + 2] * l[2]);
    const double vx = to_view(cam, 0, w), vy = to_view(cam, 1, w), vz = to_view(cam, 2, w);
    if (vz <= 1e-9) {
      crosses = 1;
      break;
    }
    const double px = cam->fx * vx / vz + cam->cx, py = cam->fy * vy / vz + cam->cy;
    if (px < min_x) min_x = px;
    if (max_x < px) max_x = px;
    if (py < min_y) min_y = py;
    if (max_y < py) max_y = py;
  }
  *tx0 = 0;
  *tx1 = tiles_x - 1;
  *ty0 = 0;
  *ty1 = tiles_y - 1;
  if (!crosses) {
    int a = x86_int(floor(min_x)) / ts;
    *tx0 = a > 0 ? a : 0;
    a = x86_int(floor(max_x)) / ts;
    *tx1 = a < tiles_x - 1 ? a : tiles_x - 1;
    a = x86_int(floor(min_y)) / ts;
    *ty0 = a > 0 ? a : 0;
    a = x86_int(floor(max_y)) / ts;
    *ty1 = a < tiles_y - 1 ? a : tiles_y - 1;
    if (max_x < 0.0 || min_x >= cam->w || max_y < 0.0 || min_y >= cam->h) return 0;
  }
  return 1;
}

static Binding make_binding(const sofo_scene* s, const PC* pcs, const Cam* cam, int ts) {
  Binding b;
  b.tile_size = ts;
  b.tiles_x = (cam->w + ts - 1) / ts;
  b.tiles_y = (cam->h + ts - 1) / ts;
  const int64_t T = (int64_t)b.tiles_x * b.tiles_y;
  b.off = calloc((size_t)T + 1, sizeof(int64_t));
  int64_t* cnt = calloc((size_t)T + 1, sizeof(int64_t));
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t gi = 0; gi < s->n; ++gi) {
      int tx0, tx1, ty0, ty1;
      if (!rect_of(s, gi, &pcs[gi], cam, ts, b.tiles_x, b.tiles_y, &tx0, &tx1, &ty0, &ty1)) continue;
      for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
          const int64_t t = (int64_t)ty * b.tiles_x + tx;
          if (pass == 0) b.off[t + 1]++;
          else b.ent[cnt[t]++] = (int32_t)gi;
        }
    }
    if (pass == 0) {
      for (int64_t t = 0; t < T; ++t) b.off[t + 1] += b.off[t];
      b.ent = malloc(sizeof(int32_t) * (size_t)(b.off[T] + 1));
      for (int64_t t = 0; t < T; ++t) cnt[t] = b.off[t];
    }
  }
  free(cnt);
  g_sort_pc = pcs;
  for (int64_t t = 0; t < T; ++t)
    qsort(b.ent + b.off[t], (size_t)(b.off[t + 1] - b.off[t]), sizeof(int32_t), cmp_minz);
  return b;
}

int64_t sofo_tile_binding(const sofo_scene* s, const sofo_cams* c, int view, int tile_size,
                          int64_t* offsets, int32_t* entries, int64_t cap) {
  const Cam cam = load_cam(c, view);
  PC* pcs = malloc(sizeof(PC) * (size_t)(s->n + 1));
  for (int64_t i = 0; i < s->n; ++i) precompute_one(s, i, &cam, &pcs[i]);
  Binding b = make_binding(s, pcs, &cam, tile_size);
  const int64_t T = (int64_t)b.tiles_x * b.tiles_y;
  const int64_t m = b.off[T];
  memcpy(offsets, b.off, sizeof(int64_t) * (size_t)(T + 1));
  if (m <= cap && entries) memcpy(entries, b.ent, sizeof(int32_t) * (size_t)m);
  free(b.off);
  free(b.ent);
  free(pcs);
  return m <= cap ? m : -m;
}

/* ---- the field evaluator (field_eval.hpp:39-198) ----------------------------------- */

typedef struct {
  const sofo_scene* s;
  int nviews, strategies, tile_size;
  Cam* cams;
  PC** pcs;       /* per view */
  Binding* bind;  /* per view, when tile scheduling */
} Eval;

static Eval eval_make(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size) {
  Eval e;
  e.s = s;
  e.nviews = c->v;
  e.strategies = strategies;
  e.tile_size = tile_size;
  e.cams = malloc(sizeof(Cam) * (size_t)(c->v + 1));
  e.pcs = malloc(sizeof(PC*) * (size_t)(c->v + 1));
  e.bind = (strategies & 1) ? malloc(sizeof(Binding) * (size_t)(c->v + 1)) : NULL;
  for (int v = 0; v < c->v; ++v) {
    e.cams[v] = load_cam(c, v);
    e.pcs[v] = malloc(sizeof(PC) * (size_t)(s->n + 1));
    for (int64_t i = 0; i < s->n; ++i) precompute_one(s, i, &e.cams[v], &e.pcs[v][i]);
    if (e.bind) e.bind[v] = make_binding(s, e.pcs[v], &e.cams[v], tile_size);
  }
  return e;
}

static void eval_free(Eval* e) {
  for (int v = 0; v < e->nviews; ++v) {
    free(e->pcs[v]);
    if (e->bind) {
      free(e->bind[v].off);
      free(e->bind[v].ent);
    }
  }
  free(e->pcs);
  free(e->cams);
  free(e->bind);
}

/* view_opacity (field_eval.hpp:59-111) */
static double view_opacity(const Eval* e, int v, const double* x, int classify, int* observed,
                           int* complete, uint64_t* counters) {
  const Cam* cam = &e->cams[v];
  *complete = 1;
  /* Camera::observes (camera.hpp:29-33) */
  const double vx = to_view(cam, 0, x), vy = to_view(cam, 1, x), vz = to_view(cam, 2, x);
  *observed = 0;
  if (!(vz <= 0.0)) {
    const double px = cam->fx * vx / vz + cam->cx, py = cam->fy * vy / vz + cam->cy;
    *observed = px >= 0.0 && px < cam->w && py >= 0.0 && py < cam->h;
  }
  if (!*observed) return 1.0;
  /* ray_through_point (camera.hpp:52-59) */
  double d[3];
  for (int k = 0; k < 3; ++k) d[k] = x[k] - cam->center[k];
  const double t = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  if (t < 1e-12) {
    *observed = 0;
    return 1.0;
  }
  for (int k = 0; k < 3; ++k) d[k] = d[k] / t;
  const double z_point = vz;
  counters[1] += 1;
  const PC* cache = e->pcs[v];
  const int32_t* list = NULL;
  int64_t count = e->s->n;
  if (e->strategies & 1) {
    const double px = cam->fx * vx / vz + cam->cx, py = cam->fy * vy / vz + cam->cy;
    const Binding* b = &e->bind[v];
    const int tile = (int)py / e->tile_size * b->tiles_x + (int)px / e->tile_size;
    list = b->ent + b->off[tile];
    count = b->off[tile + 1] - b->off[tile];
  }
  double survive = 1.0;
  uint64_t pairs = 0;
  for (int64_t k = 0; k < count; ++k) {
    const PC* pc = &cache[list ? list[k] : k];
    if ((e->strategies & 16) && pc->op < K_MIN_ALPHA) continue;
    if ((e->strategies & 2) && pc->zmin > z_point) {
      if (list) break;
      continue;
    }
    ++pairs;
    /* abc_cached (precompute.hpp:39-45), peak_t, eval_1d (gaussian.hpp:47-52) */
    const double X = d[0], Y = d[1], Z = d[2];
    const double a = pc->ic[0] * X * X + pc->ic[3] * Y * Y + pc->ic[5] * Z * Z +
                     2.0 * (pc->ic[1] * X * Y + pc->ic[2] * X * Z + pc->ic[4] * Y * Z);
    const double b = 2.0 * (X * pc->b[0] + Y * pc->b[1] + Z * pc->b[2]);
    const double t_star = -b / (2.0 * a);
    const double te = t < t_star ? t : t_star;
    if (te <= 0.0) continue;
    double alpha = pc->op * sof_exp(-0.5 * ((a * te + b) * te + pc->c));
    if (alpha < K_MIN_ALPHA) continue;
    alpha = K_MAX_ALPHA < alpha ? K_MAX_ALPHA : alpha;
    survive *= 1.0 - alpha;
    if (classify && (e->strategies & 4) && 1.0 - survive > 0.5) {
      *complete = 0;
      break;
    }
  }
  counters[0] += pairs;
  return 1.0 - survive;
}

void sofo_view_opacity(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                       int view, int64_t n, const double* xyz, int classify_mode, double* o,
                       uint8_t* observed, uint8_t* complete, uint64_t* counters) {
  Eval e = eval_make(s, c, strategies, tile_size);
  for (int64_t i = 0; i < n; ++i) {
    int ob, co;
    o[i] = view_opacity(&e, view, xyz + 3 * i, classify_mode, &ob, &co, counters);
    observed[i] = (uint8_t)ob;
    complete[i] = (uint8_t)co;
  }
  eval_free(&e);
}

/* label_grid (field_eval.hpp:140-176): views sequential, pruning state carried */
void sofo_label_grid(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                     int64_t nv, const double* xyz, int classify_mode, double* opacity,
                     uint64_t* counters) {
  Eval e = eval_make(s, c, strategies, tile_size);
  double* min_op = malloc(sizeof(double) * (size_t)(nv + 1));
  uint8_t* ext = calloc((size_t)nv + 1, 1);
  for (int64_t i = 0; i < nv; ++i) min_op[i] = 1.0;
  for (int v = 0; v < c->v; ++v)
    for (int64_t i = 0; i < nv; ++i) {
      if ((strategies & 8) && ext[i]) continue;
      int ob, co;
      const double o = view_opacity(&e, v, xyz + 3 * i, classify_mode, &ob, &co, counters);
      if (!ob) continue;
      min_op[i] = o < min_op[i] ? o : min_op[i];
      if (co && o < 0.5) ext[i] = 1;
    }
  for (int64_t i = 0; i < nv; ++i)
    opacity[i] = ext[i] ? (0.49999999 < min_op[i] ? 0.49999999 : min_op[i]) : min_op[i];
  free(min_op);
  free(ext);
  eval_free(&e);
}

void sofo_label_state(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                      int64_t nv, const double* xyz, int classify_mode, double* min_op,
                      uint8_t* ext, uint64_t* counters) {
  Eval e = eval_make(s, c, strategies, tile_size);
  for (int v = 0; v < c->v; ++v)
    for (int64_t i = 0; i < nv; ++i) {
      if ((strategies & 8) && ext[i]) continue;
      int ob, co;
      const double o = view_opacity(&e, v, xyz + 3 * i, classify_mode, &ob, &co, counters);
      if (!ob) continue;
      min_op[i] = o < min_op[i] ? o : min_op[i];
      if (co && o < 0.5) ext[i] = 1;
    }
  eval_free(&e);
}

/* classify_point (field_eval.hpp:114-125) */
static int classify_point(const Eval* e, const double* x, uint64_t* counters) {
  int interior = 1;
  for (int v = 0; v < e->nviews; ++v) {
    int ob, co;
    const double o = view_opacity(e, v, x, 1, &ob, &co, counters);
    if (ob && co && o < 0.5) {
      interior = 0;
      if (e->strategies & 8) break;
    }
  }
  return interior;
}

void sofo_classify_points(const sofo_scene* s, const sofo_cams* c, int strategies,
                          int tile_size, int64_t n, const double* xyz, uint8_t* interior,
                          uint64_t* counters) {
  Eval e = eval_make(s, c, strategies, tile_size);
  for (int64_t i = 0; i < n; ++i) interior[i] = (uint8_t)classify_point(&e, xyz + 3 * i, counters);
  eval_free(&e);
}

/* value_at (field_eval.hpp:128-136) */
void sofo_value_at(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                   int64_t n, const double* xyz, double* out, uint64_t* counters) {
  Eval e = eval_make(s, c, strategies, tile_size);
  for (int64_t i = 0; i < n; ++i) {
    double r = 1.0;
    for (int v = 0; v < c->v; ++v) {
      int ob, co;
      const double o = view_opacity(&e, v, xyz + 3 * i, 0, &ob, &co, counters);
      if (ob) r = o < r ? o : r;
    }
    out[i] = r;
  }
  eval_free(&e);
}

/* ---- hash map u64 -> int64 (open addressing) ---------------------------------------------- */

typedef struct {
  uint64_t* key;
  int64_t* val;
  uint8_t* used;
  uint64_t mask;
} Map;

static Map map_make(int64_t want) {
  uint64_t cap = 16;
  while (cap < (uint64_t)want * 2 + 16) cap <<= 1;
  Map m = {calloc(cap, 8), calloc(cap, 8), calloc(cap, 1), cap - 1};
  return m;
}
static void map_free(Map* m) {
  free(m->key);
  free(m->val);
  free(m->used);
}
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
/* returns the slot; *inserted = 1 when the key was new (value set to v) */
static int64_t map_emplace(Map* m, uint64_t k, uint64_t h, int64_t v, int* inserted) {
  uint64_t i = h & m->mask;
  while (m->used[i]) {
    if (m->key[i] == k) {
      *inserted = 0;
      return m->val[i];
    }
    i = (i + 1) & m->mask;
  }
  m->used[i] = 1;
  m->key[i] = k;
  m->val[i] = v;
  *inserted = 1;
  return v;
}

/* ---- marching_tets (marching_tets.hpp:29-84) -------------------------------------------- */

typedef struct {
  Map slots;
  int64_t nv, n_edges, n_tris;
  const double *xyz, *opa;
  int32_t *edges, *tris;
  double* verts;
} March;

/* edge_vertex (marching_tets.hpp:32-44) */
static int32_t edge_vertex(March* M, int32_t vi_in, int32_t vi_out) {
  const uint64_t key = ((uint64_t)(uint32_t)vi_in << 32) | (uint32_t)vi_out;
  int ins;
  const int64_t slot = map_emplace(&M->slots, key, mix64(key), M->n_edges, &ins);
  if (ins) {
    const int64_t e = M->n_edges++;
    M->edges[2 * e] = vi_in;
    M->edges[2 * e + 1] = vi_out;
    const double oi = M->opa[vi_in], oo = M->opa[vi_out];
    const double s = (0.5 - oi) / (oo - oi);
    for (int k = 0; k < 3; ++k) {
      const double pi = M->xyz[3 * vi_in + k], po = M->xyz[3 * vi_out + k];
      M->verts[3 * e + k] = pi + s * (po - pi);
    }
  }
  return (int32_t)slot;
}

/* emit (marching_tets.hpp:45-52) */
static void emit(March* M, int32_t e0, int32_t e1, int32_t e2, const double* ref) {
  const double *a = M->verts + 3 * e0, *b = M->verts + 3 * e1, *c = M->verts + 3 * e2;
  const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  const double w[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const double n[3] = {u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]};
  double g[3];
  for (int k = 0; k < 3; ++k) g[k] = (a[k] + b[k] + c[k]) / 3.0 - ref[k];
  int32_t* t = M->tris + 3 * M->n_tris++;
  t[0] = e0;
  if (n[0] * g[0] + n[1] * g[1] + n[2] * g[2] >= 0.0) {
    t[1] = e1;
    t[2] = e2;
  } else {
    t[1] = e2;
    t[2] = e1;
  }
}

int64_t sofo_marching_tets(int64_t nv, const double* xyz, int64_t nt, const int32_t* tets,
                           const double* opacity, int32_t* edges, double* verts, int32_t* tris,
                           int64_t* n_tris) {
  March M = {map_make(4 * nt + 16), nv, 0, 0, xyz, opacity, edges, tris, verts};
  for (int64_t ti = 0; ti < nt; ++ti) {
    const int32_t* tet = tets + 4 * ti;
    int32_t in[4], out[4];
    int ni = 0, no = 0;
    for (int k = 0; k < 4; ++k) {
      if (opacity[tet[k]] >= 0.5) in[ni++] = tet[k];
      else out[no++] = tet[k];
    }
    if (ni == 0 || ni == 4) continue;
    double ref[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < ni; ++k)
      for (int q = 0; q < 3; ++q) ref[q] = ref[q] + xyz[3 * in[k] + q];
    for (int q = 0; q < 3; ++q) ref[q] = ref[q] / (double)ni;
    if (ni == 1) {
      /* emit(edge_vertex(i0,o0), edge_vertex(i0,o1), edge_vertex(i0,o2), ref): the
       * reference binary (GCC, x86-64) evaluates these arguments right to left */
      const int32_t e2 = edge_vertex(&M, in[0], out[2]);
      const int32_t e1 = edge_vertex(&M, in[0], out[1]);
      const int32_t e0 = edge_vertex(&M, in[0], out[0]);
      emit(&M, e0, e1, e2, ref);
    } else if (ni == 3) {
      const int32_t e2 = edge_vertex(&M, in[2], out[0]);
      const int32_t e1 = edge_vertex(&M, in[1], out[0]);
      const int32_t e0 = edge_vertex(&M, in[0], out[0]);
      emit(&M, e0, e1, e2, ref);
    } else {
      const int32_t ac = edge_vertex(&M, in[0], out[0]);
      const int32_t ad = edge_vertex(&M, in[0], out[1]);
      const int32_t bd = edge_vertex(&M, in[1], out[1]);
      const int32_t bc = edge_vertex(&M, in[1], out[0]);
      emit(&M, ac, ad, bd, ref);
      emit(&M, ac, bd, bc, ref);
    }
  }
  map_free(&M.slots);
  *n_tris = M.n_tris;
  return M.n_edges;
}

/* ---- binary_search_refine (marching_tets.hpp:94-114) ------------------------------------- */

void sofo_refine(const sofo_scene* s, const sofo_cams* c, int strategies, int tile_size,
                 const double* grid_xyz, int64_t ne, const int32_t* edges, double* verts,
                 int iterations, uint64_t* counters) {
  if (iterations <= 0) return;
  Eval e = eval_make(s, c, strategies, tile_size);
  for (int64_t k = 0; k < ne; ++k) {
    double pin[3], pout[3];
    memcpy(pin, grid_xyz + 3 * edges[2 * k], sizeof pin);
    memcpy(pout, grid_xyz + 3 * edges[2 * k + 1], sizeof pout);
    for (int it = 0; it < iterations; ++it) {
      double mid[3];
      for (int q = 0; q < 3; ++q) mid[q] = 0.5 * (pin[q] + pout[q]);
      memcpy(classify_point(&e, mid, counters) ? pin : pout, mid, sizeof mid);
    }
    for (int q = 0; q < 3; ++q) verts[3 * k + q] = 0.5 * (pin[q] + pout[q]);
  }
  eval_free(&e);
}

/* ---- assemble_mesh (mesh.hpp:36-79) ----------------------------------------------------- */

int64_t sofo_assemble(int64_t nverts, const double* verts, int64_t ntris, const int32_t* tris,
                      double weld_eps, double min_area, double* out_verts, int32_t* out_tris,
                      int64_t* out_ntris) {
  /* key triple -> slot; collisions of the 64-bit mix are resolved by a full compare */
  int64_t* keys = malloc(sizeof(int64_t) * 3 * (size_t)(nverts + 1));
  int32_t* remap = malloc(sizeof(int32_t) * (size_t)(nverts + 1));
  uint64_t cap = 16;
  while (cap < (uint64_t)nverts * 2 + 16) cap <<= 1;
  int64_t* table = malloc(sizeof(int64_t) * cap);
  for (uint64_t i = 0; i < cap; ++i) table[i] = -1;
  const double inv = 1.0 / weld_eps;
  int64_t nout = 0;
  for (int64_t i = 0; i < nverts; ++i) {
    int64_t* k = keys + 3 * i;
    for (int q = 0; q < 3; ++q) k[q] = (int64_t)llround(verts[3 * i + q] * inv);
    uint64_t h = 1469598103934665603ull;
    for (int q = 0; q < 3; ++q) h = (h ^ (uint64_t)k[q]) * 1099511628211ull;
    uint64_t slot = mix64(h) & (cap - 1);
    int32_t found = -1;
    while (table[slot] >= 0) {
      const int64_t* o = keys + 3 * table[slot];
      if (o[0] == k[0] && o[1] == k[1] && o[2] == k[2]) {
        found = remap[table[slot]];
        break;
      }
      slot = (slot + 1) & (cap - 1);
    }
    if (found < 0) {
      table[slot] = i;
      found = (int32_t)nout;
      memcpy(out_verts + 3 * nout, verts + 3 * i, 3 * sizeof(double));
      ++nout;
    }
    remap[i] = found;
  }
  int64_t nt = 0;
  for (int64_t t = 0; t < ntris; ++t) {
    const int32_t r[3] = {remap[tris[3 * t]], remap[tris[3 * t + 1]], remap[tris[3 * t + 2]]};
    if (r[0] == r[1] || r[1] == r[2] || r[0] == r[2]) continue;
    const double *a = out_verts + 3 * r[0], *b = out_verts + 3 * r[1], *c = out_verts + 3 * r[2];
    const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    const double w[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    const double n[3] = {u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]};
    if (0.5 * sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]) <= min_area) continue;
    memcpy(out_tris + 3 * nt, r, sizeof r);
    ++nt;
  }
  free(keys);
  free(remap);
  free(table);
  *out_ntris = nt;
  return nout;
}

/* ---- render_pixel (opacity_field.hpp:39-61, 95-166, 192-219) ------------------------------ */

typedef struct {
  int idx;
  double t_star, alpha, a, b, c, op;
} Contrib;

static int cmp_contrib(const void* x, const void* y) {
  const Contrib *l = x, *r = y;
  if (l->t_star != r->t_star) return l->t_star < r->t_star ? -1 : 1;
  return (l->idx > r->idx) - (l->idx < r->idx);
}

static double alpha_at(const Contrib* rc, double t) {
  const double te = t < rc->t_star ? t : rc->t_star;
  if (te <= 0.0) return 0.0;
  const double a = rc->op * sof_exp(-0.5 * ((rc->a * te + rc->b) * te + rc->c));
  if (a < K_MIN_ALPHA) return 0.0;
  return K_MAX_ALPHA < a ? K_MAX_ALPHA : a;
}

int64_t sofo_render_pixel(const sofo_scene* s, const sofo_cams* c, int view, int px, int py,
                          int exact_depth, double* out6) {
  const Cam cam = load_cam(c, view);
  /* ray_through_pixel (camera.hpp:42-48): normalize(R^T d_view) */
  const double dv[3] = {((px + 0.5) - cam.cx) / cam.fx, ((py + 0.5) - cam.cy) / cam.fy, 1.0};
  double d[3];
  for (int i = 0; i < 3; ++i) d[i] = cam.R[i] * dv[0] + cam.R[3 + i] * dv[1] + cam.R[6 + i] * dv[2];
  const double sq = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
  if (sq > 0.0) {
    const double nrm = sqrt(sq);
    for (int i = 0; i < 3; ++i) d[i] = d[i] / nrm;
  }
  Contrib* list = malloc(sizeof(Contrib) * (size_t)(s->n + 1));
  int64_t m = 0;
  for (int64_t i = 0; i < s->n; ++i) {
    PC pc;
    precompute_one(s, i, &cam, &pc);
    if (pc.op < K_MIN_ALPHA) continue;
    Contrib rc;
    rc.a = pc.ic[0] * d[0] * d[0] + pc.ic[3] * d[1] * d[1] + pc.ic[5] * d[2] * d[2] +
           2.0 * (pc.ic[1] * d[0] * d[1] + pc.ic[2] * d[0] * d[2] + pc.ic[4] * d[1] * d[2]);
    rc.b = 2.0 * (d[0] * pc.b[0] + d[1] * pc.b[1] + d[2] * pc.b[2]);
    rc.c = pc.c;
    /* peak_value (gaussian.hpp:54-56) */
    const double alpha = pc.op * sof_exp(-0.5 * (rc.c - rc.b * rc.b / (4.0 * rc.a)));
    if (alpha < K_MIN_ALPHA) continue;
    rc.idx = (int)i;
    rc.t_star = -rc.b / (2.0 * rc.a);
    if (rc.t_star <= 0.0) continue;
    rc.alpha = K_MAX_ALPHA < alpha ? K_MAX_ALPHA : alpha;
    rc.op = pc.op;
    list[m++] = rc;
  }
  qsort(list, (size_t)m, sizeof(Contrib), cmp_contrib);
  double color[3] = {0.0, 0.0, 0.0}, T = 1.0;
  for (int64_t k = 0; k < m; ++k) {
    const double* dc = s->dc + 3 * list[k].idx;
    for (int q = 0; q < 3; ++q) color[q] = color[q] + dc[q] * list[k].alpha * T;
    T *= 1.0 - list[k].alpha;
  }
  double depth = NAN;
  /* find_median (opacity_field.hpp:132-142) */
  double Tm = 1.0;
  for (int64_t k = 0; k < m; ++k) {
    const double next = Tm * (1.0 - list[k].alpha);
    if (Tm > 0.5 && next < 0.5) {
      depth = list[k].t_star;
      if (exact_depth) { /* exact_depth (opacity_field.hpp:157-166) */
        const Contrib* rc = &list[k];
        const double lt = 2.0 * sof_log((Tm - 0.5) / (Tm * rc->op));
        const double disc = rc->b * rc->b - 4.0 * rc->a * (rc->c + lt);
        if (!(disc < 0.0)) depth = list[k].t_star - sqrt(disc) / (2.0 * rc->a);
      }
      break;
    }
    Tm = next;
  }
  double acc = 0.0;
  if (!isnan(depth)) {
    double tr = 1.0;
    for (int64_t k = 0; k < m; ++k) tr *= 1.0 - alpha_at(&list[k], depth);
    acc = 1.0 - tr;
  }
  out6[0] = color[0];
  out6[1] = color[1];
  out6[2] = color[2];
  out6[3] = depth;
  out6[4] = acc;
  out6[5] = T;
  free(list);
  return m;
}
