// delaunay.cu — the tetra-input producer of extract_mesh: incremental
// Bowyer-Watson tetrahedralization with the semantics of delaunay.hpp:52-142, on the host.
//
// Why the host: the reference inserts the seeds one at a time and scans every live tet
// per insertion; MT numbers its edges in the order of the resulting tet list, so a
// parallel (GPU) Delaunay — same tet set, another order — would change the mesh's vertex
// numbering. This restatement reproduces the reference's tet list exactly: the same
// enclosing tetrahedron, the same strict in-circumsphere test with its 1e-12 / 1e-30 slack,
// cavity walls (faces met once) re-closed in the order the cavity tets were found, the
// same orientation fix and degeneracy threshold, and the arithmetic of the Eigen-API the
// reference is pinned to (oracle/eigen_shim: row-0 determinant expansion, partial-pivot
// LU, left-to-right sums). It is a host stage of the producer, not of the hot path
// (label -> march -> refine -> weld stay on the device).
#include <algorithm>
#include <array>
#include <cmath>
#include <stdexcept>
#include <unordered_map>
#include <vector>

#include "../../include/sof_cuda.h"
#include "sof_internal.h"

namespace sofk {
namespace {

struct V3 {
  double x, y, z;
};
inline V3 sub(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double sqn(const V3& a) { return a.x * a.x + a.y * a.y + a.z * a.z; }

// rows r0, r1, r2 (Mat3 with m.row(i) = ...): det by expansion along row 0
inline double det3_rows(const V3& r0, const V3& r1, const V3& r2) {
  const double m[3][3] = {{r0.x, r0.y, r0.z}, {r1.x, r1.y, r1.z}, {r2.x, r2.y, r2.z}};
  auto h = [&](int a, int b, int c) { return m[0][a] * (m[1][b] * m[2][c] - m[1][c] * m[2][b]); };
  return h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
}

// Mat3::partialPivLu().solve(rhs)
inline V3 lu_solve(const V3& r0, const V3& r1, const V3& r2, const V3& rhs) {
  double lu[3][3] = {{r0.x, r0.y, r0.z}, {r1.x, r1.y, r1.z}, {r2.x, r2.y, r2.z}};
  int perm[3] = {0, 1, 2};
  for (int k = 0; k < 3; ++k) {
    int piv = k;
    for (int i = k + 1; i < 3; ++i)
      if (std::abs(lu[i][k]) > std::abs(lu[piv][k])) piv = i;
    if (piv != k) {
      for (int c = 0; c < 3; ++c) std::swap(lu[k][c], lu[piv][c]);
      std::swap(perm[k], perm[piv]);
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

struct Tet {
  std::array<int, 4> v;
  V3 cc;
  double r2;
  bool alive;
};

// circumsphere (delaunay.hpp:30-47); false for (near-)degenerate tets
inline bool sphere(const V3& p0, const V3& p1, const V3& p2, const V3& p3, V3& c, double& r2) {
  const V3 a = sub(p1, p0), b = sub(p2, p0), d = sub(p3, p0);
  const double det = det3_rows(a, b, d);
  double scale = 0.0;
  for (double v : {a.x, a.y, a.z, b.x, b.y, b.z, d.x, d.y, d.z}) scale = std::max(scale, std::abs(v));
  if (std::abs(det) < 1e-14 * scale * scale * scale) return false;
  const V3 rhs{0.5 * (sqn(p1) - sqn(p0)), 0.5 * (sqn(p2) - sqn(p0)), 0.5 * (sqn(p3) - sqn(p0))};
  c = lu_solve(a, b, d, rhs);
  r2 = sqn(sub(c, p0));
  return true;
}

}  // namespace

std::vector<std::array<int, 4>> delaunay_host(const double* pts, int64_t n) {
  if (n < 4) throw InvalidArg("need at least 4 points");
  std::vector<V3> v(size_t(n) + 4);
  for (int64_t i = 0; i < n; ++i) v[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  V3 lo = v[0], hi = v[0];
  for (int64_t i = 0; i < n; ++i) {
    lo = {std::min(lo.x, v[i].x), std::min(lo.y, v[i].y), std::min(lo.z, v[i].z)};
    hi = {std::max(hi.x, v[i].x), std::max(hi.y, v[i].y), std::max(hi.z, v[i].z)};
  }
  const V3 ctr{0.5 * (lo.x + hi.x), 0.5 * (lo.y + hi.y), 0.5 * (lo.z + hi.z)};
  const V3 ext = sub(hi, lo);
  const double radius = std::max(0.5 * std::sqrt(sqn(ext)), 1.0);
  const double big = 1e4 * radius;
  // the enclosing tetrahedron (delaunay.hpp:64-67)
  const V3 corner[4] = {{0.0, 0.0, 3 * big}, {-2 * big, -big, -big}, {2 * big, -big, -big}, {0.0, 2 * big, -big}};
  for (int k = 0; k < 4; ++k) v[n + k] = {ctr.x + corner[k].x, ctr.y + corner[k].y, ctr.z + corner[k].z};

  std::vector<Tet> tets;
  auto add = [&](int a, int b, int c, int d) {
    if (det3_rows(sub(v[b], v[a]), sub(v[c], v[a]), sub(v[d], v[a])) < 0) std::swap(c, d);
    Tet t;
    t.v = {a, b, c, d};
    t.alive = true;
    if (!sphere(v[a], v[b], v[c], v[d], t.cc, t.r2)) return;  // degenerate sliver
    tets.push_back(t);
  };
  add(int(n), int(n + 1), int(n + 2), int(n + 3));

  std::vector<size_t> bad;
  std::vector<std::array<int, 3>> faces;
  std::unordered_map<uint64_t, int> seen;  // sorted face -> occurrences in the cavity
  auto face_key = [](std::array<int, 3> f) {
    std::sort(f.begin(), f.end());
    return (uint64_t(uint32_t(f[0])) * 0x9E3779B97F4A7C15ull) ^ (uint64_t(uint32_t(f[1])) << 21) ^
           (uint64_t(uint32_t(f[2])) << 42) ^ uint64_t(uint32_t(f[1]) * 31u + uint32_t(f[2]));
  };
  auto same = [](std::array<int, 3> a, std::array<int, 3> b) {
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    return a == b;
  };
  for (int64_t pi = 0; pi < n; ++pi) {
    const V3& p = v[pi];
    bad.clear();
    faces.clear();
    for (size_t ti = 0; ti < tets.size(); ++ti) {  // tets whose circumsphere holds p (strictly)
      if (!tets[ti].alive) continue;
      if (sqn(sub(p, tets[ti].cc)) < tets[ti].r2 * (1.0 - 1e-12) - 1e-30) bad.push_back(ti);
    }
    for (size_t ti : bad) {
      const auto& q = tets[ti].v;
      faces.push_back({q[0], q[1], q[2]});
      faces.push_back({q[0], q[1], q[3]});
      faces.push_back({q[0], q[2], q[3]});
      faces.push_back({q[1], q[2], q[3]});
      tets[ti].alive = false;
    }
    // cavity walls: faces met exactly once, re-closed in the order they were met
    seen.clear();
    seen.reserve(faces.size() * 2);
    for (const auto& f : faces) ++seen[face_key(f)];
    for (size_t i = 0; i < faces.size(); ++i) {
      bool unique = seen[face_key(faces[i])] == 1;
      if (!unique) {  // a hash collision must not hide a unique face: confirm exactly
        unique = true;
        for (size_t j = 0; j < faces.size(); ++j)
          if (i != j && same(faces[i], faces[j])) {
            unique = false;
            break;
          }
      }
      if (unique) add(int(pi), faces[i][0], faces[i][1], faces[i][2]);
    }
    if (tets.size() > size_t(4 * n + 1024)) {  // drop dead tets (live order is kept)
      size_t w = 0;
      for (size_t r = 0; r < tets.size(); ++r)
        if (tets[r].alive) tets[w++] = tets[r];
      tets.resize(w);
    }
  }
  std::vector<std::array<int, 4>> out;
  for (const auto& t : tets)
    if (t.alive && t.v[0] < n && t.v[1] < n && t.v[2] < n && t.v[3] < n) out.push_back(t.v);
  if (out.empty()) throw InvalidArg("degenerate (coplanar) point set");
  return out;
}

}  // namespace sofk

using namespace sofk;

extern "C" int sof_tetrahedralize(sof_ctx* c, int64_t n, const double* pts, int64_t* n_tets) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (n < 0 || (n > 0 && !pts)) throw InvalidArg("invalid point array");
    if (n >= (int64_t(1) << 31)) throw InvalidArg("more than 2^31 points");
    const std::vector<std::array<int, 4>> t = delaunay_host(pts, n);
    c->delaunay_tets.assign(reinterpret_cast<const int32_t*>(t.data()),
                            reinterpret_cast<const int32_t*>(t.data()) + 4 * t.size());
    if (n_tets) *n_tets = int64_t(t.size());
  });
}
