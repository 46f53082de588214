// delaunay.cu — the tetra-input producer of extract_mesh: the
// incremental Bowyer-Watson tetrahedralization of delaunay.hpp:52-142 on the device.
//
// The reference inserts the seeds one at a time and scans every live tet per insertion;
// MT numbers its edges in the order of the resulting tet list, so a parallel Delaunay --
// same tet set, another order -- would change the mesh's vertex numbering. The device
// keeps the reference's sequence and parallelises inside each insertion, in one
// persistent cooperative kernel (grid-wide barriers between the phases):
//   A  every block tests its contiguous range of the tet array against the new point
//      (strict in-circumsphere test with the reference's 1e-12 / 1e-30 slack, dead tets
//      skipped) and counts the hits;
//   B  blocks with hits write them, in array order, at their offset in the cavity list
//      (the sum of the earlier blocks' counts) and retire those tets;
//   C  block 0 expands the cavity into its faces (4 per bad tet, in the reference's
//      order), keeps the faces met exactly once, and appends the new tets in face order
//      (orientation fix, circumsphere, degenerate slivers dropped), computed in parallel
//      and placed by an ordered prefix;
//   D  now and then, an order-preserving compaction of the live tets (it changes no
//      result: the discovery order depends only on the live tets' relative order).
// The arithmetic is the Eigen-API shim's the reference is pinned to (oracle/eigen_shim:
// row-0 determinant expansion, partial-pivot LU, left-to-right sums; --fmad=false), so
// the tet list equals the reference's exactly. O(n^2) like the reference: meant for
// seed sets of up to ~10^5 points (the reference's own limit).
#include <cooperative_groups.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <vector>

#include "../../include/sof_cuda.h"
#include "sof_internal.h"

namespace cg = cooperative_groups;

namespace sofk {
namespace {

struct V3 {
  double x, y, z;
};
__host__ __device__ inline V3 sub(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ inline double sqn(const V3& a) { return a.x * a.x + a.y * a.y + a.z * a.z; }

// rows r0, r1, r2 (Mat3 with m.row(i) = ...): det by expansion along row 0
__host__ __device__ inline double det3_rows(const V3& r0, const V3& r1, const V3& r2) {
  const double m[3][3] = {{r0.x, r0.y, r0.z}, {r1.x, r1.y, r1.z}, {r2.x, r2.y, r2.z}};
  const double h0 = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]);
  const double h1 = m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]);
  const double h2 = m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
  return h0 - h1 + h2;
}

// Mat3::partialPivLu().solve(rhs)
__host__ __device__ inline V3 lu_solve(const V3& r0, const V3& r1, const V3& r2, const V3& rhs) {
  double lu[3][3] = {{r0.x, r0.y, r0.z}, {r1.x, r1.y, r1.z}, {r2.x, r2.y, r2.z}};
  int perm[3] = {0, 1, 2};
  for (int k = 0; k < 3; ++k) {
    int piv = k;
    for (int i = k + 1; i < 3; ++i)
      if (fabs(lu[i][k]) > fabs(lu[piv][k])) piv = i;
    if (piv != k) {
      for (int c = 0; c < 3; ++c) {
        const double t = lu[k][c];
        lu[k][c] = lu[piv][c];
        lu[piv][c] = t;
      }
      const int t = perm[k];
      perm[k] = perm[piv];
      perm[piv] = t;
    }
    for (int i = k + 1; i < 3; ++i) {
      const double f = lu[k][k] != 0.0 ? lu[i][k] / lu[k][k] : 0.0;
      lu[i][k] = f;
      for (int c = k + 1; c < 3; ++c) lu[i][c] = lu[i][c] - f * lu[k][c];
    }
  }
  const double b[3] = {rhs.x, rhs.y, rhs.z};
  double y[3], x[3];
  for (int i = 0; i < 3; ++i) {
    double s = b[perm[i]];
    for (int k = 0; k < i; ++k) s = s - lu[i][k] * y[k];
    y[i] = s;
  }
  for (int i = 2; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 3; ++k) s = s - lu[i][k] * x[k];
    x[i] = s / lu[i][i];
  }
  return {x[0], x[1], x[2]};
}

// circumsphere (delaunay.hpp:30-47); false for (near-)degenerate tets
__host__ __device__ inline bool sphere(const V3& p0, const V3& p1, const V3& p2, const V3& p3, V3& c,
                                       double& r2) {
  const V3 a = sub(p1, p0), b = sub(p2, p0), d = sub(p3, p0);
  const double det = det3_rows(a, b, d);
  const double vals[9] = {a.x, a.y, a.z, b.x, b.y, b.z, d.x, d.y, d.z};
  double scale = 0.0;
  for (int k = 0; k < 9; ++k) scale = fmax(scale, fabs(vals[k]));
  if (fabs(det) < 1e-14 * scale * scale * scale) return false;
  const V3 rhs{0.5 * (sqn(p1) - sqn(p0)), 0.5 * (sqn(p2) - sqn(p0)), 0.5 * (sqn(p3) - sqn(p0))};
  c = lu_solve(a, b, d, rhs);
  r2 = sqn(sub(c, p0));
  return true;
}

constexpr int kDlThreads = 256;

struct DlState {           // device-resident control words
  int64_t T;               // tets in the array (live and retired)
  int64_t live;            // live tets
  int64_t nbad;            // cavity size of the current insertion
  int error;               // 1: capacity exceeded
  int sel;                 // which of the two tet buffers is current
};

struct DlBuffers {
  const V3* verts;         // n + 4 (the enclosing tetrahedron's corners last)
  int4* tv[2];             // tet vertices (ping-pong for the compaction)
  double4* ts[2];          // circumcentre xyz, radius^2
  uint8_t* alive[2];
  int64_t cap;             // tet capacity per buffer
  int64_t* bad;            // cavity list (tet indices, array order)
  int64_t* bcount;         // per-block counts
  int3* faces;             // 4 per cavity tet
  int32_t* keep;           // per face: 1 = new tet
  int4* nv;                // per face: the new tet (after the orientation fix)
  double4* ns;             // per face: its circumsphere
  int64_t fcap;            // face capacity
  DlState* st;
};

// the new tet of face (f0, f1, f2) around point a (add_tet, delaunay.hpp:75-86)
__device__ bool make_tet(const V3* V, int a, int b, int c, int d, int4& v, double4& s) {
  if (det3_rows(sub(V[b], V[a]), sub(V[c], V[a]), sub(V[d], V[a])) < 0) {
    const int t = c;
    c = d;
    d = t;
  }
  v = make_int4(a, b, c, d);
  V3 cc;
  double r2;
  if (!sphere(V[a], V[b], V[c], V[d], cc, r2)) return false;
  s = make_double4(cc.x, cc.y, cc.z, r2);
  return true;
}

__device__ __forceinline__ bool same_face(int3 a, int3 b) {
  // sorted-triple equality (the reference compares std::sort-ed copies)
  auto sort3 = [](int3 f) {
    int x = f.x, y = f.y, z = f.z, t;
    if (y < x) t = x, x = y, y = t;
    if (z < y) t = y, y = z, z = t;
    if (y < x) t = x, x = y, y = t;
    return make_int3(x, y, z);
  };
  const int3 p = sort3(a), q = sort3(b);
  return p.x == q.x && p.y == q.y && p.z == q.z;
}

// block-wide exclusive scan of one int per thread (kDlThreads threads)
__device__ int block_excl_scan(int v, int* smem, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) smem[w] = inc;
  __syncthreads();
  int before = 0;
  total = 0;
  for (int k = 0; k < kDlThreads / 32; ++k) {
    before += (k < w) ? smem[k] : 0;
    total += smem[k];
  }
  __syncthreads();
  return before + inc - v;
}

__global__ void __launch_bounds__(kDlThreads) k_delaunay(int64_t n, DlBuffers B) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int s_scan[kDlThreads / 32];
  __shared__ int64_t s_off;
  const int nb = gridDim.x, b = blockIdx.x, t = threadIdx.x;
  DlState* st = B.st;
  for (int64_t pi = 0; pi < n; ++pi) {
    const V3 p = B.verts[pi];
    const int sel = *(volatile int*)&st->sel;
    const int64_t T = *(volatile int64_t*)&st->T;
    const int4* tv = B.tv[sel];
    const double4* ts = B.ts[sel];
    uint8_t* alive = B.alive[sel];
    // A: this block's contiguous range, tested in rounds of kDlThreads (array order)
    const int64_t per = (T + nb - 1) / nb;
    const int64_t lo = int64_t(b) * per, hi = min(T, lo + per);
    int cnt = 0;
    for (int64_t ti = lo + t; ti < hi; ti += kDlThreads) {
      if (!alive[ti]) continue;
      const double4 s = ts[ti];
      const V3 d = sub(p, V3{s.x, s.y, s.z});
      if (sqn(d) < s.w * (1.0 - 1e-12) - 1e-30) ++cnt;
    }
    int tot;
    (void)block_excl_scan(cnt, s_scan, tot);
    if (t == 0) B.bcount[b] = tot;
    grid.sync();
    // B: the hits in array order at this block's offset; retire them
    if (t == 0) {
      int64_t off = 0, all = 0;
      for (int k = 0; k < nb; ++k) {
        off += (k < b) ? B.bcount[k] : 0;
        all += B.bcount[k];
      }
      s_off = off;
      if (b == 0) st->nbad = all;
    }
    __syncthreads();
    if (B.bcount[b] > 0) {
      int64_t off = s_off;
      for (int64_t r0 = lo; r0 < hi; r0 += kDlThreads) {
        const int64_t ti = r0 + t;
        bool hit = false;
        if (ti < hi && alive[ti]) {
          const double4 s = ts[ti];
          const V3 d = sub(p, V3{s.x, s.y, s.z});
          hit = sqn(d) < s.w * (1.0 - 1e-12) - 1e-30;
        }
        int rt;
        const int ex = block_excl_scan(hit ? 1 : 0, s_scan, rt);
        if (hit) B.bad[off + ex] = ti;
        off += rt;
      }
      __syncthreads();
      for (int64_t k = s_off + t; k < off; k += kDlThreads) alive[B.bad[k]] = 0;
    }
    grid.sync();
    // C: cavity walls -> new tets (block 0)
    if (b == 0) {
      const int64_t nbad = st->nbad;
      const int64_t F = 4 * nbad;
      if (F > B.fcap) {
        if (t == 0) st->error = 1;
      } else {
        for (int64_t k = t; k < nbad; k += kDlThreads) {
          const int4 v = tv[B.bad[k]];
          B.faces[4 * k + 0] = make_int3(v.x, v.y, v.z);
          B.faces[4 * k + 1] = make_int3(v.x, v.y, v.w);
          B.faces[4 * k + 2] = make_int3(v.x, v.z, v.w);
          B.faces[4 * k + 3] = make_int3(v.y, v.z, v.w);
        }
        __syncthreads();
        for (int64_t i = t; i < F; i += kDlThreads) {
          const int3 f = B.faces[i];
          bool unique = true;
          for (int64_t j = 0; j < F && unique; ++j)
            if (j != i && same_face(f, B.faces[j])) unique = false;
          int keep = 0;
          if (unique) {
            int4 v;
            double4 s;
            if (make_tet(B.verts, int(pi), f.x, f.y, f.z, v, s)) {
              B.nv[i] = v;
              B.ns[i] = s;
              keep = 1;
            }
          }
          B.keep[i] = keep;
        }
        __syncthreads();
        // ordered append behind the current end
        int64_t end = T;
        for (int64_t r0 = 0; r0 < F; r0 += kDlThreads) {
          const int64_t i = r0 + t;
          const int k = (i < F) ? B.keep[i] : 0;
          int rt;
          const int ex = block_excl_scan(k, s_scan, rt);
          if (k) {
            const int64_t dst = end + ex;
            if (dst < B.cap) {
              B.tv[sel][dst] = B.nv[i];
              B.ts[sel][dst] = B.ns[i];
              B.alive[sel][dst] = 1;
            }
          }
          end += rt;
        }
        if (t == 0) {
          if (end > B.cap) st->error = 1;
          st->T = min(end, B.cap);
          st->live = st->live - nbad + (end - T);
        }
      }
    }
    grid.sync();
    if (*(volatile int*)&st->error) return;
    // D: keep the scan near the live count once retired tets outnumber the live ones (the
    // reference compacts past 4 n + 1024 entries; where is immaterial: compaction keeps
    // the live tets' relative order), or before the array could overflow
    const int64_t T2 = *(volatile int64_t*)&st->T, L2 = *(volatile int64_t*)&st->live;
    if (T2 - L2 > max(L2, int64_t(65536)) || T2 > B.cap - B.fcap) {
      const int64_t per2 = (T2 + nb - 1) / nb;
      const int64_t lo2 = int64_t(b) * per2, hi2 = min(T2, lo2 + per2);
      int c2 = 0;
      for (int64_t ti = lo2 + t; ti < hi2; ti += kDlThreads) c2 += B.alive[sel][ti] ? 1 : 0;
      int tot2;
      (void)block_excl_scan(c2, s_scan, tot2);
      if (t == 0) B.bcount[b] = tot2;
      grid.sync();
      if (t == 0) {
        int64_t off = 0, all = 0;
        for (int k = 0; k < nb; ++k) {
          off += (k < b) ? B.bcount[k] : 0;
          all += B.bcount[k];
        }
        s_off = off;
        if (b == 0) {
          st->T = all;
          st->live = all;
        }
      }
      __syncthreads();
      int64_t off = s_off;
      for (int64_t r0 = lo2; r0 < hi2; r0 += kDlThreads) {
        const int64_t ti = r0 + t;
        const bool a = ti < hi2 && B.alive[sel][ti];
        int rt;
        const int ex = block_excl_scan(a ? 1 : 0, s_scan, rt);
        if (a) {
          B.tv[sel ^ 1][off + ex] = B.tv[sel][ti];
          B.ts[sel ^ 1][off + ex] = B.ts[sel][ti];
          B.alive[sel ^ 1][off + ex] = 1;
        }
        off += rt;
      }
      grid.sync();
      if (b == 0 && t == 0) st->sel = sel ^ 1;
      grid.sync();
    }
  }
}

}  // namespace

// One run with the given capacity multiplier; false when a cavity or the tet array
// outgrew its capacity (the caller retries larger).
static bool delaunay_run(sof_ctx* c, const double* pts, int64_t n, int64_t mult,
                         std::vector<std::array<int, 4>>& out) {
  if (n < 4) throw InvalidArg("need at least 4 points");
  // the enclosing tetrahedron (delaunay.hpp:55-67), set up on the host
  std::vector<V3> v(size_t(n) + 4);
  for (int64_t i = 0; i < n; ++i) v[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  V3 lo = v[0], hi = v[0];
  for (int64_t i = 0; i < n; ++i) {
    lo = {std::min(lo.x, v[i].x), std::min(lo.y, v[i].y), std::min(lo.z, v[i].z)};
    hi = {std::max(hi.x, v[i].x), std::max(hi.y, v[i].y), std::max(hi.z, v[i].z)};
  }
  const V3 ctr{0.5 * (lo.x + hi.x), 0.5 * (lo.y + hi.y), 0.5 * (lo.z + hi.z)};
  const double radius = std::max(0.5 * std::sqrt(sqn(sub(hi, lo))), 1.0);
  const double big = 1e4 * radius;
  const V3 corner[4] = {{0.0, 0.0, 3 * big}, {-2 * big, -big, -big}, {2 * big, -big, -big}, {0.0, 2 * big, -big}};
  for (int k = 0; k < 4; ++k) v[n + k] = {ctr.x + corner[k].x, ctr.y + corner[k].y, ctr.z + corner[k].z};
  // the first tet (its orientation fix and circumsphere as add_tet)
  int a = int(n), b = int(n + 1), cc = int(n + 2), d = int(n + 3);
  if (det3_rows(sub(v[b], v[a]), sub(v[cc], v[a]), sub(v[d], v[a])) < 0) std::swap(cc, d);
  V3 c0;
  double r20;
  const bool ok0 = sphere(v[a], v[b], v[cc], v[d], c0, r20);

  // ~6.5 n live tets for random points, retired ones and one insertion's growth; degenerate
  // sets (the reference's slivers leave holes) can need more: mult grows on retry
  const int64_t cap = (16 * n + 262144) * mult;
  const int64_t fcap = 65536 * mult;
  DBuf<char>& m = c->dl_buf;
  const size_t bytes = sizeof(V3) * (n + 4) + 2 * cap * (sizeof(int4) + sizeof(double4) + 1) + cap * 8 +
                       4096 * 8 + fcap * (sizeof(int3) + 4 + sizeof(int4) + sizeof(double4)) + sizeof(DlState) + 4096;
  m.ensure(bytes);
  char* p = m.p;
  auto take = [&](size_t sz) {
    char* r = p;
    p += (sz + 255) & ~size_t(255);
    return r;
  };
  DlBuffers B;
  V3* dverts = reinterpret_cast<V3*>(take(sizeof(V3) * (n + 4)));
  B.verts = dverts;
  for (int k = 0; k < 2; ++k) {
    B.tv[k] = reinterpret_cast<int4*>(take(cap * sizeof(int4)));
    B.ts[k] = reinterpret_cast<double4*>(take(cap * sizeof(double4)));
    B.alive[k] = reinterpret_cast<uint8_t*>(take(cap));
  }
  B.cap = cap;
  B.bad = reinterpret_cast<int64_t*>(take(cap * 8));
  B.bcount = reinterpret_cast<int64_t*>(take(4096 * 8));
  B.faces = reinterpret_cast<int3*>(take(fcap * sizeof(int3)));
  B.keep = reinterpret_cast<int32_t*>(take(fcap * 4));
  B.nv = reinterpret_cast<int4*>(take(fcap * sizeof(int4)));
  B.ns = reinterpret_cast<double4*>(take(fcap * sizeof(double4)));
  B.fcap = fcap;
  B.st = reinterpret_cast<DlState*>(take(sizeof(DlState)));
  cudaStream_t s = c->stream;
  SOF_CUDA(cudaMemcpyAsync(dverts, v.data(), sizeof(V3) * (n + 4), cudaMemcpyHostToDevice, s));
  DlState st0{ok0 ? 1 : 0, ok0 ? 1 : 0, 0, 0, 0};
  SOF_CUDA(cudaMemcpyAsync(B.st, &st0, sizeof st0, cudaMemcpyHostToDevice, s));
  if (ok0) {
    const int4 tv0 = make_int4(a, b, cc, d);
    const double4 ts0 = make_double4(c0.x, c0.y, c0.z, r20);
    const uint8_t one = 1;
    SOF_CUDA(cudaMemcpyAsync(B.tv[0], &tv0, sizeof tv0, cudaMemcpyHostToDevice, s));
    SOF_CUDA(cudaMemcpyAsync(B.ts[0], &ts0, sizeof ts0, cudaMemcpyHostToDevice, s));
    SOF_CUDA(cudaMemcpyAsync(B.alive[0], &one, 1, cudaMemcpyHostToDevice, s));
  }
  // one co-resident grid: every block takes part in every barrier
  int dev = 0, sms = 0, per_sm = 0;
  SOF_CUDA(cudaGetDevice(&dev));
  SOF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SOF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_delaunay, kDlThreads, 0));
  const int grid = std::max(1, std::min(sms * std::max(per_sm, 1), 4096));
  int64_t nn = n;
  void* args[] = {&nn, &B};
  SOF_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_delaunay), grid, kDlThreads, args, 0, s));
  SOF_LAUNCHED(c);
  DlState st;
  SOF_CUDA(cudaMemcpyAsync(&st, B.st, sizeof st, cudaMemcpyDeviceToHost, s));
  SOF_CUDA(cudaStreamSynchronize(s));
  if (st.error) return false;
  std::vector<int4> tv(size_t(st.T));
  std::vector<uint8_t> al(size_t(st.T));
  if (st.T > 0) {
    SOF_CUDA(cudaMemcpyAsync(tv.data(), B.tv[st.sel], sizeof(int4) * st.T, cudaMemcpyDeviceToHost, s));
    SOF_CUDA(cudaMemcpyAsync(al.data(), B.alive[st.sel], st.T, cudaMemcpyDeviceToHost, s));
    SOF_CUDA(cudaStreamSynchronize(s));
  }
  out.clear();  // live tets without enclosing-tetrahedron corners, in order
  for (int64_t i = 0; i < st.T; ++i) {
    const int4 q = tv[size_t(i)];
    if (al[size_t(i)] && q.x < n && q.y < n && q.z < n && q.w < n) out.push_back({q.x, q.y, q.z, q.w});
  }
  return true;
}

std::vector<std::array<int, 4>> delaunay_device(sof_ctx* c, const double* pts, int64_t n) {
  if (n < 4) throw InvalidArg("need at least 4 points");
  std::vector<std::array<int, 4>> out;
  bool ok = false;
  for (int64_t mult = 1; !ok && mult <= 64; mult *= 4) {
    size_t free_b = 0, total_b = 0;
    SOF_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double need = double((16 * n + 262144) * mult) * 2 * (sizeof(int4) + sizeof(double4) + 1) +
                        double(65536 * mult) * 64;
    if (mult > 1 && need > 0.8 * double(free_b + c->dl_buf.bytes())) break;
    ok = delaunay_run(c, pts, n, mult, out);
  }
  if (!ok) throw StateError("device Delaunay: the tet array outgrew the device memory");
  if (out.empty()) throw InvalidArg("degenerate (coplanar) point set");
  return out;
}

}  // namespace sofk

using namespace sofk;

extern "C" int sof_tetrahedralize(sof_ctx* c, int64_t n, const double* pts, int64_t* n_tets) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (n < 0 || (n > 0 && !pts)) throw InvalidArg("invalid point array");
    if (n >= (int64_t(1) << 31) - 8) throw InvalidArg("more than 2^31 points");
    const std::vector<std::array<int, 4>> t = delaunay_device(c, pts, n);
    c->delaunay_tets.assign(reinterpret_cast<const int32_t*>(t.data()),
                            reinterpret_cast<const int32_t*>(t.data()) + 4 * t.size());
    if (n_tets) *n_tets = int64_t(t.size());
  });
}
