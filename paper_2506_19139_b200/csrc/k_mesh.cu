// k_mesh.cu — Marching Tetrahedra (K6-K8), batched bisection (K9) and the weld
// (K10), all deterministic and bit-identical to the reference.
//
// Reference path replaced: marching_tets (marching_tets.hpp:29-84),
// binary_search_refine (marching_tets.hpp:94-114) and assemble_mesh (mesh.hpp:36-79).
// The reference numbers edges and welded vertices in order of first appearance,
// driven by hash maps; here "first appearance" is recovered with stable radix
// sorts: occurrences are sorted by key keeping their global position order, the
// run head is the first occurrence, and an exclusive scan over first-occurrence
// flags assigns ids in appearance order. Compiled with --fmad=false.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>

#include "sof_internal.h"

namespace sofk {

// ---- K6: per-tet case ------------------------------------------------------------------------

__global__ void k_tet_case(int64_t nt, const int32_t* __restrict__ tets,
                           const double* __restrict__ opa, uint8_t* crossing) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= nt) return;
  const int4 tt = reinterpret_cast<const int4*>(tets)[t];
  const int ni = (opa[tt.x] >= 0.5) + (opa[tt.y] >= 0.5) + (opa[tt.z] >= 0.5) + (opa[tt.w] >= 0.5);
  crossing[t] = (ni != 0 && ni != 4);
}

// occurrence / triangle counts of the crossing tets, packed (occ | tri << 32)
__global__ void k_tet_counts(int64_t nc, const int32_t* __restrict__ ctets,
                             const int32_t* __restrict__ tets, const double* __restrict__ opa,
                             unsigned long long* packed) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k > nc) return;
  if (k == nc) {
    packed[nc] = 0;
    return;
  }
  const int4 tt = reinterpret_cast<const int4*>(tets)[ctets[k]];
  const int ni = (opa[tt.x] >= 0.5) + (opa[tt.y] >= 0.5) + (opa[tt.z] >= 0.5) + (opa[tt.w] >= 0.5);
  const unsigned long long occ = (ni == 2) ? 4 : 3, tri = (ni == 2) ? 2 : 1;
  packed[k] = occ | (tri << 32);
}

// K7: emit the edge_vertex() occurrences of each crossing tet in the reference's
// call order and the triangles' occurrence references.
//   ni == 1: emit(edge(i0,o0), edge(i0,o1), edge(i0,o2)) — GCC/x86-64 evaluates the
//            three call arguments right to left, so the calls (and therefore the
//            first-appearance edge numbering) run (i0,o2), (i0,o1), (i0,o0);
//   ni == 3: likewise (i2,o0), (i1,o0), (i0,o0);
//   ni == 2: named statements ac, ad, bd, bc (marching_tets.hpp:75-78).
// Verified against the compiled reference (tests/test_mesh_cpu.py).
__global__ void k_tet_emit(int64_t nc, int64_t nv, const int32_t* __restrict__ ctets,
                           const int32_t* __restrict__ tets, const double* __restrict__ opa,
                           const unsigned long long* __restrict__ off, uint64_t* occ_key,
                           int32_t* occ_pos, int32_t* occ_in, int32_t* occ_out, int32_t* tri_occ,
                           int32_t* tri_tet) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= nc) return;
  const int32_t t = ctets[k];
  const int4 tt = reinterpret_cast<const int4*>(tets)[t];
  const int v[4] = {tt.x, tt.y, tt.z, tt.w};
  int in[4], out[4], ni = 0, no = 0;
  for (int q = 0; q < 4; ++q) {
    if (opa[v[q]] >= 0.5)
      in[ni++] = v[q];
    else
      out[no++] = v[q];
  }
  const unsigned long long o = off[k];
  const int64_t ob = int64_t(o & 0xffffffffull), tb = int64_t(o >> 32);
  int ci[4], co[4], nocc;
  if (ni == 1) {
    ci[0] = in[0]; co[0] = out[2];
    ci[1] = in[0]; co[1] = out[1];
    ci[2] = in[0]; co[2] = out[0];
    nocc = 3;
    // triangle (e(i0,o0), e(i0,o1), e(i0,o2)) = occurrences (2, 1, 0)
    tri_occ[3 * tb] = int32_t(ob + 2);
    tri_occ[3 * tb + 1] = int32_t(ob + 1);
    tri_occ[3 * tb + 2] = int32_t(ob);
    tri_tet[tb] = t;
  } else if (ni == 3) {
    ci[0] = in[2]; co[0] = out[0];
    ci[1] = in[1]; co[1] = out[0];
    ci[2] = in[0]; co[2] = out[0];
    nocc = 3;
    tri_occ[3 * tb] = int32_t(ob + 2);
    tri_occ[3 * tb + 1] = int32_t(ob + 1);
    tri_occ[3 * tb + 2] = int32_t(ob);
    tri_tet[tb] = t;
  } else {
    ci[0] = in[0]; co[0] = out[0];  // ac
    ci[1] = in[0]; co[1] = out[1];  // ad
    ci[2] = in[1]; co[2] = out[1];  // bd
    ci[3] = in[1]; co[3] = out[0];  // bc
    nocc = 4;
    // emit(ac, ad, bd), emit(ac, bd, bc)
    tri_occ[3 * tb] = int32_t(ob);
    tri_occ[3 * tb + 1] = int32_t(ob + 1);
    tri_occ[3 * tb + 2] = int32_t(ob + 2);
    tri_occ[3 * tb + 3] = int32_t(ob);
    tri_occ[3 * tb + 4] = int32_t(ob + 2);
    tri_occ[3 * tb + 5] = int32_t(ob + 3);
    tri_tet[tb] = t;
    tri_tet[tb + 1] = t;
  }
  for (int q = 0; q < nocc; ++q) {
    occ_key[ob + q] = uint64_t(ci[q]) * uint64_t(nv) + uint64_t(co[q]);
    occ_pos[ob + q] = int32_t(ob + q);
    occ_in[ob + q] = ci[q];
    occ_out[ob + q] = co[q];
  }
}

// Run heads of the key-sorted occurrences: the head carries the smallest global
// position (stable sort), i.e. the first appearance.
__global__ void k_occ_heads(int64_t m, const uint64_t* __restrict__ skey,
                            const int32_t* __restrict__ spos, int32_t* head, uint8_t* is_first_u8) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= m) return;
  const bool h = (j == 0) || skey[j] != skey[j - 1];
  head[j] = h;
  if (h) is_first_u8[spos[j]] = 1;
}

__global__ void k_u8_to_i32(int64_t m, const uint8_t* __restrict__ a, int32_t* b) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j < m) b[j] = a[j];
}

// edges[e] and the lerp vertex (marching_tets.hpp:36-42) for each first occurrence.
__global__ void k_edges(int64_t m, const int32_t* __restrict__ is_first,
                        const int32_t* __restrict__ eid, const int32_t* __restrict__ occ_in,
                        const int32_t* __restrict__ occ_out, const double* __restrict__ opa,
                        const double* __restrict__ xyz, int32_t* edges, double* verts) {
  const int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (q >= m || !is_first[q]) return;
  const int32_t e = eid[q];
  const int32_t a = occ_in[q], b = occ_out[q];
  edges[2 * e] = a;
  edges[2 * e + 1] = b;
  const double oi = opa[a], oo = opa[b];
  const double s = (0.5 - oi) / (oo - oi);
  for (int k = 0; k < 3; ++k) {
    const double pi = xyz[3 * a + k], po = xyz[3 * b + k];
    verts[3 * e + k] = pi + s * (po - pi);
  }
}

// edge id of every occurrence: the id of its run head's first occurrence.
__global__ void k_occ_edge(int64_t m, const int32_t* __restrict__ run_incl,
                           const int32_t* __restrict__ head, const int32_t* __restrict__ spos,
                           const int32_t* __restrict__ eid, int32_t* run_eid, int32_t* occ_edge) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= m) return;
  if (head[j]) run_eid[run_incl[j] + head[j] - 1] = eid[spos[j]];
}
__global__ void k_occ_edge2(int64_t m, const int32_t* __restrict__ run_incl,
                            const int32_t* __restrict__ head, const int32_t* __restrict__ spos,
                            const int32_t* __restrict__ run_eid, int32_t* occ_edge) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= m) return;
  occ_edge[spos[j]] = run_eid[run_incl[j] + head[j] - 1];
}

// emit() winding (marching_tets.hpp:45-52) with interior_ref from the tet (:64-66).
__global__ void k_tris(int64_t ntri, const int32_t* __restrict__ tri_occ,
                       const int32_t* __restrict__ tri_tet, const int32_t* __restrict__ occ_edge,
                       const int32_t* __restrict__ tets, const double* __restrict__ opa,
                       const double* __restrict__ xyz, const double* __restrict__ verts,
                       int32_t* tris) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= ntri) return;
  const int32_t e0 = occ_edge[tri_occ[3 * k]], e1 = occ_edge[tri_occ[3 * k + 1]],
                e2 = occ_edge[tri_occ[3 * k + 2]];
  const int4 tt = reinterpret_cast<const int4*>(tets)[tri_tet[k]];
  const int v[4] = {tt.x, tt.y, tt.z, tt.w};
  double ref[3] = {0.0, 0.0, 0.0};
  int ni = 0;
  for (int q = 0; q < 4; ++q)
    if (opa[v[q]] >= 0.5) {
      for (int c = 0; c < 3; ++c) ref[c] = ref[c] + xyz[3 * v[q] + c];
      ++ni;
    }
  for (int c = 0; c < 3; ++c) ref[c] = ref[c] / double(ni);
  const double* a = verts + 3 * e0;
  const double* b = verts + 3 * e1;
  const double* cc = verts + 3 * e2;
  const double u0 = b[0] - a[0], u1 = b[1] - a[1], u2 = b[2] - a[2];
  const double w0 = cc[0] - a[0], w1 = cc[1] - a[1], w2 = cc[2] - a[2];
  const double n0 = u1 * w2 - u2 * w1, n1 = u2 * w0 - u0 * w2, n2 = u0 * w1 - u1 * w0;
  const double g0 = (a[0] + b[0] + cc[0]) / 3.0 - ref[0];
  const double g1 = (a[1] + b[1] + cc[1]) / 3.0 - ref[1];
  const double g2 = (a[2] + b[2] + cc[2]) / 3.0 - ref[2];
  const bool keep = n0 * g0 + n1 * g1 + n2 * g2 >= 0.0;
  tris[3 * k] = e0;
  tris[3 * k + 1] = keep ? e1 : e2;
  tris[3 * k + 2] = keep ? e2 : e1;
}

// ---- tet-sharded march: merge of per-shard results ------------------------------------------------

constexpr int kMaxShards = 64;
struct ShardOffsets {
  int world;
  int64_t edge_off[kMaxShards + 1];  // first gathered edge of each shard
  int64_t tri_off[kMaxShards + 1];   // first gathered triangle of each shard
};

// occurrences = the shards' edge lists concatenated in shard (= tet) order
__global__ void k_shard_occ(int64_t m, int64_t nv, const int32_t* __restrict__ edges, uint64_t* key,
                            int32_t* pos, int32_t* in, int32_t* out) {
  const int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (q >= m) return;
  const int32_t a = edges[2 * q], b = edges[2 * q + 1];
  key[q] = uint64_t(a) * uint64_t(nv) + uint64_t(b);
  pos[q] = int32_t(q);
  in[q] = a;
  out[q] = b;
}

// shard-local edge ids of the gathered triangles -> global ids (winding was decided
// per shard with the same lerp vertices)
__global__ void k_remap_tris(int64_t ntri, ShardOffsets so, const int32_t* __restrict__ tris_in,
                             const int32_t* __restrict__ occ_edge, int32_t* tris) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= ntri) return;
  int r = 0;
  while (r + 1 < so.world && so.tri_off[r + 1] <= k) ++r;
  const int64_t eb = so.edge_off[r];
  for (int q = 0; q < 3; ++q) tris[3 * k + q] = occ_edge[eb + tris_in[3 * k + q]];
}

// Edge numbering in order of first appearance (marching_tets.hpp:31-44) for the m
// occurrences in ms.okey / opos / oin / oout (positions = appearance order): a stable
// key sort puts each edge's first occurrence at its run head; an exclusive scan over
// first-occurrence flags numbers the edges. Fills r_edges, r_everts (the lerp vertex,
// :38-41) and ms.occ_edge (edge id of every occurrence); returns the edge count.
static int64_t number_edges(sof_ctx* c, const double* opa, int64_t m) {
  const int64_t nv = c->nv;
  MeshScratch& s = c->ms;
  const int kbits = bits_for(uint64_t(nv) * uint64_t(nv));
  sort_pairs_u64(c, s.okey.p, s.skey.p, s.opos.p, s.spos.p, m, kbits);
  s.head.ensure(m);
  s.first_u8.ensure(m);
  s.is_first.ensure(m);
  s.eid.ensure(m);
  s.run_incl.ensure(m);
  s.occ_edge.ensure(m);
  zero_async(c, s.first_u8.p, m);
  k_occ_heads<<<grid_for(m, 256), 256, 0, c->stream>>>(m, s.skey.p, s.spos.p, s.head.p,
                                                        s.first_u8.p);
  SOF_LAUNCHED(c);
  k_u8_to_i32<<<grid_for(m, 256), 256, 0, c->stream>>>(m, s.first_u8.p, s.is_first.p);
  SOF_LAUNCHED(c);
  exclusive_scan_i32(c, s.is_first.p, s.eid.p, m);
  exclusive_scan_i32(c, s.head.p, s.run_incl.p, m);  // exclusive: run id = run_incl + head - 1
  // number of edges = number of runs
  const int32_t last_run = read_scalar(c, s.run_incl.p + (m - 1));
  const int32_t last_head = read_scalar(c, s.head.p + (m - 1));
  const int64_t E = int64_t(last_run) + last_head;
  s.run_eid.ensure(E);
  c->r_edges.ensure(2 * E);
  c->r_everts.ensure(3 * E);
  k_edges<<<grid_for(m, 256), 256, 0, c->stream>>>(m, s.is_first.p, s.eid.p, s.oin.p, s.oout.p, opa,
                                                    c->tv.p, c->r_edges.p, c->r_everts.p);
  SOF_LAUNCHED(c);
  k_occ_edge<<<grid_for(m, 256), 256, 0, c->stream>>>(m, s.run_incl.p, s.head.p, s.spos.p, s.eid.p,
                                                       s.run_eid.p, s.occ_edge.p);
  SOF_LAUNCHED(c);
  k_occ_edge2<<<grid_for(m, 256), 256, 0, c->stream>>>(m, s.run_incl.p, s.head.p, s.spos.p,
                                                        s.run_eid.p, s.occ_edge.p);
  SOF_LAUNCHED(c);
  return E;
}

void march(sof_ctx* c, const double* opa) {
  tets_ready(c);
  if (!c->has_tets) throw StateError("no tets: call sof_set_tets first");
  march_range(c, opa, 0, c->nt);
}

// marching_tets over the tet range [t0, t1): edges numbered in first appearance within
// the range, triangles referencing them (a shard of the tet-sharded march; the whole
// range is the reference's marching_tets).
void march_range(sof_ctx* c, const double* opa, int64_t t0, int64_t t1) {
  tets_ready(c);
  if (!c->has_tets) throw StateError("no tets: call sof_set_tets first");
  if (t0 < 0 || t1 > c->nt || t0 > t1) throw InvalidArg("tet range out of bounds");
  const int64_t nt = t1 - t0, nv = c->nv;
  const int32_t* tets = c->tt.p + 4 * t0;
  MeshScratch& s = c->ms;
  c->n_edges = c->n_march_tris = 0;
  c->r_edges.ensure(2);
  c->r_everts.ensure(3);
  c->r_tris.ensure(3);
  if (nt == 0) return;
  s.crossing.ensure(nt);
  k_tet_case<<<grid_for(nt, 256), 256, 0, c->stream>>>(nt, tets, opa, s.crossing.p);
  SOF_LAUNCHED(c);
  // compact the crossing tets, keeping tet order
  s.ctets.ensure(nt);
  s.nsel.ensure(1);
  {
    thrust::counting_iterator<int32_t> it(0);
    size_t bytes = 0;
    SOF_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, s.crossing.p, s.ctets.p, s.nsel.p, nt,
                                        c->stream));
    c->cub_tmp.ensure(bytes);
    SOF_CUDA(cub::DeviceSelect::Flagged(c->cub_tmp.p, bytes, it, s.crossing.p, s.ctets.p,
                                        s.nsel.p, nt, c->stream));
    c->launches += 2;
  }
  const int64_t nc = read_scalar(c, s.nsel.p);
  if (nc == 0) return;
  s.packed.ensure(nc + 1);
  s.off.ensure(nc + 1);
  k_tet_counts<<<grid_for(nc + 1, 256), 256, 0, c->stream>>>(nc, s.ctets.p, tets, opa,
                                                              s.packed.p);
  SOF_LAUNCHED(c);
  {
    size_t bytes = 0;
    SOF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, s.packed.p, s.off.p, nc + 1, c->stream));
    c->cub_tmp.ensure(bytes);
    SOF_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, bytes, s.packed.p, s.off.p, nc + 1,
                                           c->stream));
    c->launches += 2;
  }
  const unsigned long long tot = read_scalar(c, s.off.p + nc);
  const int64_t m = int64_t(tot & 0xffffffffull), ntri = int64_t(tot >> 32);
  s.okey.ensure(m);
  s.skey.ensure(m);
  s.opos.ensure(m);
  s.spos.ensure(m);
  s.oin.ensure(m);
  s.oout.ensure(m);
  s.tri_occ.ensure(3 * ntri);
  s.tri_tet.ensure(ntri);
  k_tet_emit<<<grid_for(nc, 128), 128, 0, c->stream>>>(nc, nv, s.ctets.p, tets, opa, s.off.p,
                                                        s.okey.p, s.opos.p, s.oin.p, s.oout.p,
                                                        s.tri_occ.p, s.tri_tet.p);
  SOF_LAUNCHED(c);
  const int64_t E = number_edges(c, opa, m);
  c->r_tris.ensure(3 * ntri);
  k_tris<<<grid_for(ntri, 256), 256, 0, c->stream>>>(ntri, s.tri_occ.p, s.tri_tet.p, s.occ_edge.p,
                                                      tets, opa, c->tv.p, c->r_everts.p,
                                                      c->r_tris.p);
  SOF_LAUNCHED(c);
  c->n_edges = E;
  c->n_march_tris = ntri;
}

// Merge of a tet-sharded march (shard r ran march_range over the r-th contiguous tet
// range): every edge's global first appearance lies in the first shard that contains
// it, so the global numbering is the first-appearance numbering of the shards' edge
// lists concatenated in shard order; triangles keep their shard's winding.
void march_merge(sof_ctx* c, const double* opa, int world, const int64_t* ecount, const int32_t* edges_all,
                 const int64_t* tcount, const int32_t* tris_all) {
  if (world < 1 || world > kMaxShards) throw InvalidArg("shard count out of range");
  if (!c->has_tets) throw StateError("no tets: call sof_set_tets first");
  ShardOffsets so;
  so.world = world;
  so.edge_off[0] = so.tri_off[0] = 0;
  for (int r = 0; r < world; ++r) {
    if (ecount[r] < 0 || tcount[r] < 0) throw InvalidArg("negative shard count");
    so.edge_off[r + 1] = so.edge_off[r] + ecount[r];
    so.tri_off[r + 1] = so.tri_off[r] + tcount[r];
  }
  const int64_t m = so.edge_off[world], ntri = so.tri_off[world];
  MeshScratch& s = c->ms;
  c->n_edges = c->n_march_tris = 0;
  c->r_edges.ensure(2);
  c->r_everts.ensure(3);
  c->r_tris.ensure(3);
  if (m == 0) return;
  s.okey.ensure(m);
  s.skey.ensure(m);
  s.opos.ensure(m);
  s.spos.ensure(m);
  s.oin.ensure(m);
  s.oout.ensure(m);
  k_shard_occ<<<grid_for(m, 256), 256, 0, c->stream>>>(m, c->nv, edges_all, s.okey.p, s.opos.p, s.oin.p, s.oout.p);
  SOF_LAUNCHED(c);
  const int64_t E = number_edges(c, opa, m);
  c->r_tris.ensure(std::max<int64_t>(3 * ntri, 3));
  if (ntri > 0) {
    k_remap_tris<<<grid_for(ntri, 256), 256, 0, c->stream>>>(ntri, so, tris_all, s.occ_edge.p, c->r_tris.p);
    SOF_LAUNCHED(c);
  }
  c->n_edges = E;
  c->n_march_tris = ntri;
}

// ---- K9: batched bisection -------------------------------------------------------------------------

__global__ void k_bisect_init(int64_t ne, const int32_t* __restrict__ edges,
                              const double* __restrict__ xyz, double* pin, double* pout) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= ne) return;
  const int32_t a = edges[2 * e], b = edges[2 * e + 1];
  for (int k = 0; k < 3; ++k) {
    pin[3 * e + k] = xyz[3 * a + k];
    pout[3 * e + k] = xyz[3 * b + k];
  }
}

// mid = 0.5 * (p_in + p_out) (marching_tets.hpp:108); also clears the exterior flags.
__global__ void k_bisect_mid(int64_t ne, const double* __restrict__ pin,
                             const double* __restrict__ pout, double* mid, uint8_t* ext) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= ne) return;
  for (int k = 0; k < 3; ++k) mid[3 * e + k] = 0.5 * (pin[3 * e + k] + pout[3 * e + k]);
  ext[e] = 0;
}

// (interior(mid) ? p_in : p_out) = mid (marching_tets.hpp:109)
__global__ void k_bisect_update(int64_t ne, const double* __restrict__ mid,
                                const uint8_t* __restrict__ ext, double* pin, double* pout) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= ne) return;
  double* dst = ext[e] ? pout : pin;
  for (int k = 0; k < 3; ++k) dst[3 * e + k] = mid[3 * e + k];
}

__global__ void k_bisect_final(int64_t ne, const double* __restrict__ pin,
                               const double* __restrict__ pout, double* verts) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= ne) return;
  for (int k = 0; k < 3; ++k) verts[3 * e + k] = 0.5 * (pin[3 * e + k] + pout[3 * e + k]);
}

// Bisection phases (also driven one by one by the view-sharded path, with an
// all-reduce of the exterior flags between classify and update).
void refine_init(sof_ctx* c, int64_t ne, const int32_t* edges) {
  MeshScratch& s = c->ms;
  s.pin.ensure(3 * ne);
  s.pout.ensure(3 * ne);
  s.mid.ensure(3 * ne);
  s.rext.ensure(ne);
  if (ne == 0) return;
  k_bisect_init<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, edges, c->tv.p, s.pin.p, s.pout.p);
  SOF_LAUNCHED(c);
}

void refine_mid(sof_ctx* c, int64_t ne, uint8_t* ext) {
  if (ne == 0) return;
  k_bisect_mid<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, c->ms.pin.p, c->ms.pout.p, c->ms.mid.p, ext);
  SOF_LAUNCHED(c);
}

void refine_update(sof_ctx* c, int64_t ne, const uint8_t* ext) {
  if (ne == 0) return;
  k_bisect_update<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, c->ms.mid.p, ext, c->ms.pin.p, c->ms.pout.p);
  SOF_LAUNCHED(c);
}

void refine_final(sof_ctx* c, int64_t ne, double* verts) {
  if (ne == 0) return;
  k_bisect_final<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, c->ms.pin.p, c->ms.pout.p, verts);
  SOF_LAUNCHED(c);
}

void refine(sof_ctx* c, int64_t ne, const int32_t* edges, double* verts, int iterations,
            int strategies, int tile_size, int v0, int v1, uint64_t* counters) {
  if (strategies & ~int(SOF_ALL_STRATEGIES)) throw InvalidArg("strategies mask has bits outside 0..31");
  if (iterations <= 0 || ne == 0) return;  // iterations = 0 keeps the lerp vertices (:100)
  if (!c->has_tets) throw StateError("no tets: call sof_set_tets first");
  refine_init(c, ne, edges);
  bisect_cache_views(c, v0, v1, ne, edges, strategies, tile_size);  // views past the record budget
  for (int it = 0; it < iterations; ++it) {
    refine_mid(c, ne, c->ms.rext.p);
    // classify_point over every view (field_eval.hpp:114-125): exterior iff some view
    // has observed && complete && O < 0.5; prune skips the rest for that point
    eval_views(c, v0, v1, ne, c->ms.mid.p, strategies, tile_size, true, kModeClassify, nullptr,
               c->ms.rext.p, nullptr, nullptr, nullptr, counters);
    refine_update(c, ne, c->ms.rext.p);
  }
  refine_final(c, ne, verts);
}

// ---- K10: weld ------------------------------------------------------------------------------------

__global__ void k_weld_keys(int64_t n, const double* __restrict__ v, double inv, uint64_t* kx,
                            uint64_t* ky, uint64_t* kz, int32_t* idx) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  // llround(p * inv) (mesh.hpp:57-62); any bijection of the int64 works as a sort key
  kx[i] = uint64_t(x86_llround(v[3 * i] * inv));
  ky[i] = uint64_t(x86_llround(v[3 * i + 1] * inv));
  kz[i] = uint64_t(x86_llround(v[3 * i + 2] * inv));
  idx[i] = int32_t(i);
}

__global__ void k_gather_u64(int64_t n, const int32_t* __restrict__ perm,
                             const uint64_t* __restrict__ src, uint64_t* dst) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j < n) dst[j] = src[perm[j]];
}

__global__ void k_weld_heads(int64_t n, const int32_t* __restrict__ perm,
                             const uint64_t* __restrict__ kx, const uint64_t* __restrict__ ky,
                             const uint64_t* __restrict__ kz, int32_t* head) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  bool h = j == 0;
  if (!h) {
    const int32_t a = perm[j], b = perm[j - 1];
    h = kx[a] != kx[b] || ky[a] != ky[b] || kz[a] != kz[b];
  }
  head[j] = h;
}

__global__ void k_weld_runfirst(int64_t n, const int32_t* __restrict__ perm,
                                const int32_t* __restrict__ head, const int32_t* __restrict__ run,
                                int32_t* run_first) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j < n && head[j]) run_first[run[j]] = perm[j];
}

__global__ void k_weld_first(int64_t n, const int32_t* __restrict__ perm,
                             const int32_t* __restrict__ head, const int32_t* __restrict__ run,
                             const int32_t* __restrict__ run_first, int32_t* first_of,
                             int32_t* is_first) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const int32_t i = perm[j];
  const int32_t f = run_first[run[j] + head[j] - 1];
  first_of[i] = f;
  is_first[i] = (f == i);
}

__global__ void k_weld_out(int64_t n, const int32_t* __restrict__ is_first,
                           const int32_t* __restrict__ nid, const double* __restrict__ v,
                           double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n || !is_first[i]) return;
  for (int k = 0; k < 3; ++k) out[3 * nid[i] + k] = v[3 * i + k];
}

// the residual of the first appearance of each welded vertex (mesh.hpp:63-67)
__global__ void k_weld_res(int64_t n, const int32_t* __restrict__ is_first, const int32_t* __restrict__ nid,
                           const double* __restrict__ r, double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n && is_first[i]) out[nid[i]] = r[i];
}

// remap + drop repeated ids / area <= min_area on the welded positions (mesh.hpp:70-77)
__global__ void k_weld_tris(int64_t nt, const int32_t* __restrict__ tris,
                            const int32_t* __restrict__ first_of, const int32_t* __restrict__ nid,
                            const double* __restrict__ wv, double min_area, int32_t* rt,
                            int32_t* keep) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= nt) return;
  int32_t r[3];
  for (int q = 0; q < 3; ++q) r[q] = nid[first_of[tris[3 * k + q]]];
  bool ok = !(r[0] == r[1] || r[1] == r[2] || r[0] == r[2]);
  if (ok) {
    const double* a = wv + 3 * r[0];
    const double* b = wv + 3 * r[1];
    const double* cc = wv + 3 * r[2];
    const double u0 = b[0] - a[0], u1 = b[1] - a[1], u2 = b[2] - a[2];
    const double w0 = cc[0] - a[0], w1 = cc[1] - a[1], w2 = cc[2] - a[2];
    const double n0 = u1 * w2 - u2 * w1, n1 = u2 * w0 - u0 * w2, n2 = u0 * w1 - u1 * w0;
    const double area = 0.5 * sqrt(n0 * n0 + n1 * n1 + n2 * n2);
    ok = !(area <= min_area);
  }
  keep[k] = ok;
  for (int q = 0; q < 3; ++q) rt[3 * k + q] = r[q];
}

__global__ void k_compact_tris(int64_t nt, const int32_t* __restrict__ keep,
                               const int32_t* __restrict__ pos, const int32_t* __restrict__ rt,
                               int32_t* out) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= nt || !keep[k]) return;
  for (int q = 0; q < 3; ++q) out[3 * pos[k] + q] = rt[3 * k + q];
}

// First-appearance dedup of n points on the grid llround(p * inv) (mesh.hpp:57-68,
// seed_points.hpp:61-70): leaves in MeshScratch is_first (wfirst), the new id of every
// first appearance (nid, exclusive scan) and first_of (index of the first point of each
// point's key); returns the number of distinct keys.
int64_t dedup_first(sof_ctx* c, int64_t n, const double* v, double inv) {
  MeshScratch& s = c->ms;
  DBuf<uint64_t>&kx = s.kx, &ky = s.ky, &kz = s.kz, &k1 = s.k1, &k2 = s.k2;
  DBuf<int32_t>&p0 = s.p0, &p1 = s.p1, &head = s.whead, &run = s.wrun, &run_first = s.wrun_first,
                 &first_of = s.first_of, &is_first = s.wfirst, &nid = s.nid;
  kx.ensure(n); ky.ensure(n); kz.ensure(n); k1.ensure(n); k2.ensure(n);
  p0.ensure(n); p1.ensure(n); head.ensure(n); run.ensure(n); run_first.ensure(n);
  first_of.ensure(n); is_first.ensure(n); nid.ensure(n);
  k_weld_keys<<<grid_for(n, 256), 256, 0, c->stream>>>(n, v, inv, kx.p, ky.p, kz.p, p0.p);
  SOF_LAUNCHED(c);
  // LSD over (kx, ky, kz): stable sorts by kz, then ky, then kx; ties keep index order
  sort_pairs_u64(c, kz.p, k2.p, p0.p, p1.p, n, 64);
  k_gather_u64<<<grid_for(n, 256), 256, 0, c->stream>>>(n, p1.p, ky.p, k1.p);
  SOF_LAUNCHED(c);
  sort_pairs_u64(c, k1.p, k2.p, p1.p, p0.p, n, 64);
  k_gather_u64<<<grid_for(n, 256), 256, 0, c->stream>>>(n, p0.p, kx.p, k1.p);
  SOF_LAUNCHED(c);
  sort_pairs_u64(c, k1.p, k2.p, p0.p, p1.p, n, 64);
  k_weld_heads<<<grid_for(n, 256), 256, 0, c->stream>>>(n, p1.p, kx.p, ky.p, kz.p, head.p);
  SOF_LAUNCHED(c);
  exclusive_scan_i32(c, head.p, run.p, n);
  k_weld_runfirst<<<grid_for(n, 256), 256, 0, c->stream>>>(n, p1.p, head.p, run.p, run_first.p);
  SOF_LAUNCHED(c);
  k_weld_first<<<grid_for(n, 256), 256, 0, c->stream>>>(n, p1.p, head.p, run.p, run_first.p,
                                                         first_of.p, is_first.p);
  SOF_LAUNCHED(c);
  exclusive_scan_i32(c, is_first.p, nid.p, n);
  return int64_t(read_scalar(c, nid.p + (n - 1))) + read_scalar(c, is_first.p + (n - 1));
}

void assemble(sof_ctx* c, int64_t n, const double* v, int64_t nt, const int32_t* tris,
              double weld_eps, double min_area, const double* residuals) {
  c->mesh_nv = c->mesh_nt = 0;
  c->mesh_nres = residuals ? 0 : -1;
  c->m_verts.ensure(3);
  c->m_tris.ensure(3);
  if (n == 0) return;
  MeshScratch& s = c->ms;
  const int64_t nout = dedup_first(c, n, v, 1.0 / weld_eps);
  DBuf<int32_t>&first_of = s.first_of, &is_first = s.wfirst, &nid = s.nid;
  c->m_verts.ensure(3 * nout);
  k_weld_out<<<grid_for(n, 256), 256, 0, c->stream>>>(n, is_first.p, nid.p, v, c->m_verts.p);
  SOF_LAUNCHED(c);
  c->mesh_nv = nout;
  if (residuals) {  // out.residuals.push_back((*residuals)[i]) on first appearance (mesh.hpp:66)
    c->m_res.ensure(std::max<int64_t>(nout, 1));
    k_weld_res<<<grid_for(n, 256), 256, 0, c->stream>>>(n, is_first.p, nid.p, residuals, c->m_res.p);
    SOF_LAUNCHED(c);
    c->mesh_nres = nout;
  }
  if (nt == 0) return;
  DBuf<int32_t>&rt = s.rt, &keep = s.keep, &pos = s.pos;
  rt.ensure(3 * nt);
  keep.ensure(nt);
  pos.ensure(nt);
  k_weld_tris<<<grid_for(nt, 256), 256, 0, c->stream>>>(nt, tris, first_of.p, nid.p, c->m_verts.p,
                                                          min_area, rt.p, keep.p);
  SOF_LAUNCHED(c);
  exclusive_scan_i32(c, keep.p, pos.p, nt);
  const int64_t ntout = int64_t(read_scalar(c, pos.p + (nt - 1))) + read_scalar(c, keep.p + (nt - 1));
  c->m_tris.ensure(std::max<int64_t>(3 * ntout, 3));
  k_compact_tris<<<grid_for(nt, 256), 256, 0, c->stream>>>(nt, keep.p, pos.p, rt.p, c->m_tris.p);
  SOF_LAUNCHED(c);
  c->mesh_nt = ntout;
}

// ---- level_set_residuals (marching_tets.hpp:117-123) ------------------------------------------

__global__ void k_abs_minus_half(int64_t n, const double* __restrict__ v, double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = fabs(v[i] - 0.5);  // std::abs(value(x) - 0.5)
}

// value_at (field_eval.hpp:128-136) with EvalStrategies::naive() — the `exact` evaluator of
// extract.hpp:66-67 — at the refined edge vertices, over views [v0, v1).
double* level_set_values(sof_ctx* c, const sof_extract_opts& o, int v0, int v1) {
  const int64_t ne = c->n_edges;
  c->res_in.ensure(std::max<int64_t>(2 * ne, 2));
  fill_f64(c, c->res_in.p, ne, 1.0);
  if (ne > 0)
    eval_views(c, v0, v1, ne, c->r_everts.p, /*EvalStrategies::naive()*/ 0, o.tile_size, false, kModeValue, c->res_in.p, nullptr,
               nullptr, nullptr, nullptr, nullptr);
  return c->res_in.p;
}

double* residuals_from_values(sof_ctx* c, const double* values) {
  const int64_t ne = c->n_edges;
  double* out = c->res_in.p + ne;
  if (ne > 0) {
    k_abs_minus_half<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, values, out);
    SOF_LAUNCHED(c);
  }
  return out;
}

double* level_set_residuals(sof_ctx* c, const sof_extract_opts& o, int v0, int v1) {
  return residuals_from_values(c, level_set_values(c, o, v0, v1));
}

// ---- seed points (seed_points.hpp:41-87) --------------------------------------------------------

// Candidate seeds in the reference's insertion order: per Gaussian its centre (slot
// 9 i) then the 8 oriented E-box corners (slots 9 i + 1 + mask); valid = inserted
// (finite, not cut off, corners only when the radius is positive).
__global__ void k_seed_candidates(int64_t n, const double* __restrict__ pos, const double* __restrict__ scale,
                                  const double* __restrict__ rot, const double* __restrict__ opa, double fs,
                                  int variant, int cutoff, double* pts, uint8_t* prov, int32_t* valid) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  GaussStatic g;
  gauss_static(pos + 3 * i, scale + 3 * i, rot + 4 * i, opa[i], fs, g);
  const double eff = g.op;  // filtered_opacity (gaussian.hpp:67-73)
  const bool cut = cutoff == SOF_SEED_CUT_DEAD && eff < kMinAlpha;
  const double r = (variant == SOF_SEED_THREE_SIGMA) ? 3.0 : (variant == SOF_SEED_STRETCHED_SIGMA) ? 3.33 : g.E;
  for (int s = 0; s < 9; ++s) {
    double p[3];
    if (s == 0) {
      for (int k = 0; k < 3; ++k) p[k] = pos[3 * i + k];
    } else {
      const int mask = s - 1;
      const double l[3] = {r * scale[3 * i] * ((mask & 1) ? 1 : -1), r * scale[3 * i + 1] * ((mask & 2) ? 1 : -1),
                           r * scale[3 * i + 2] * ((mask & 4) ? 1 : -1)};
      for (int k = 0; k < 3; ++k)
        p[k] = pos[3 * i + k] + (g.rot[3 * k] * l[0] + g.rot[3 * k + 1] * l[1] + g.rot[3 * k + 2] * l[2]);
    }
    const bool ok = !cut && (s == 0 || r > 0.0) && isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]);
    const int64_t slot = 9 * i + s;
    for (int k = 0; k < 3; ++k) pts[3 * slot + k] = p[k];
    prov[slot] = s == 0 ? 0 : 1;
    valid[slot] = ok;
  }
}

__global__ void k_seed_compact(int64_t m, const int32_t* __restrict__ valid, const int32_t* __restrict__ pos,
                               const double* __restrict__ pts, const uint8_t* __restrict__ prov, double* out,
                               uint8_t* out_prov) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= m || !valid[k]) return;
  const int64_t o = pos[k];
  for (int d = 0; d < 3; ++d) out[3 * o + d] = pts[3 * k + d];
  out_prov[o] = prov[k];
}

__global__ void k_seed_out(int64_t n, const int32_t* __restrict__ is_first, const int32_t* __restrict__ nid,
                           const double* __restrict__ pts, const uint8_t* __restrict__ prov, double* out,
                           uint8_t* out_prov) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n || !is_first[k]) return;
  const int64_t o = nid[k];
  for (int d = 0; d < 3; ++d) out[3 * o + d] = pts[3 * k + d];
  out_prov[o] = prov[k];
}

// build_seed_points over the context's scene -> c->seeds / c->seed_prov
void seed_points(sof_ctx* c, int variant, int cutoff, double filter_scale) {
  const int64_t n = c->n, m = 9 * n;
  MeshScratch& s = c->ms;
  c->n_seeds = 0;
  s.seed_pts.ensure(std::max<int64_t>(3 * m, 3));
  s.seed_prov.ensure(std::max<int64_t>(m, 1));
  s.seed_valid.ensure(std::max<int64_t>(m, 1));
  s.seed_pos.ensure(std::max<int64_t>(m, 1));
  if (n > 0) {
    k_seed_candidates<<<grid_for(n, 128), 128, 0, c->stream>>>(n, c->pos.p, c->scale.p, c->rot.p, c->opa.p,
                                                               filter_scale, variant, cutoff, s.seed_pts.p,
                                                               s.seed_prov.p, s.seed_valid.p);
    SOF_LAUNCHED(c);
    exclusive_scan_i32(c, s.seed_valid.p, s.seed_pos.p, m);
  }
  const int64_t mv = (n > 0) ? int64_t(read_scalar(c, s.seed_pos.p + (m - 1))) + read_scalar(c, s.seed_valid.p + (m - 1))
                             : 0;
  if (mv == 0) throw std::runtime_error("no live Gaussians");  // seed_points.hpp:85
  s.seed_cpts.ensure(3 * mv);
  s.seed_cprov.ensure(mv);
  k_seed_compact<<<grid_for(m, 256), 256, 0, c->stream>>>(m, s.seed_valid.p, s.seed_pos.p, s.seed_pts.p,
                                                          s.seed_prov.p, s.seed_cpts.p, s.seed_cprov.p);
  SOF_LAUNCHED(c);
  const int64_t nout = dedup_first(c, mv, s.seed_cpts.p, 1e9);  // llround(p * 1e9) keys
  c->seeds.ensure(3 * nout);
  c->seed_prov.ensure(nout);
  k_seed_out<<<grid_for(mv, 256), 256, 0, c->stream>>>(mv, s.wfirst.p, s.nid.p, s.seed_cpts.p, s.seed_cprov.p,
                                                       c->seeds.p, c->seed_prov.p);
  SOF_LAUNCHED(c);
  c->n_seeds = nout;
}

}  // namespace sofk
