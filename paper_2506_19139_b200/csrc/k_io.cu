// Scene IO: splatting-PLY scenes decoded and activated on the device.
//
// parse_scene (io_scene.hpp:54-134): the host reads the (small) text header with the
// reference's rules and messages, then moves the binary payload to the device in one
// copy; k_decode_scene turns each record into the activated GaussianPrimitive fields
// (exp scales, normalised quaternion, sigmoid opacity, 0.5 + C0 dc) directly into the
// context's SoA scene arrays. write_scene (io_scene.hpp:138-181): k_encode_scene
// applies the inverse activations and packs the float32 records; the host writes the
// header and the payload. exp / log are sof_exp / sof_log, the functions the reference
// build calls, so values and files are bit-identical.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <vector>

#include "../../include/sof_cuda.h"
#include "sof_internal.h"

namespace sofk {

namespace {

constexpr int kSceneFields = 14;
// parse_scene's required properties (io_scene.hpp:103-106), in decode order
const char* const kRequired[kSceneFields] = {"x",       "y",       "z",      "scale_0", "scale_1",
                                             "scale_2", "rot_0",   "rot_1",  "rot_2",   "rot_3",
                                             "opacity", "f_dc_0",  "f_dc_1", "f_dc_2"};
constexpr double kShC0 = 0.28209479177387814;

int ply_size(const std::string& t) {
  static const std::map<std::string, int> sizes = {
      {"char", 1},  {"int8", 1},  {"uchar", 1}, {"uint8", 1},  {"short", 2},   {"int16", 2},
      {"ushort", 2}, {"uint16", 2}, {"int", 4},  {"int32", 4},  {"uint", 4},    {"uint32", 4},
      {"float", 4}, {"float32", 4}, {"double", 8}, {"float64", 8}};
  const auto it = sizes.find(t);
  return it == sizes.end() ? -1 : it->second;
}

std::vector<std::string> tokens(const std::string& line) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
    const size_t b = i;
    while (i < line.size() && !std::isspace(static_cast<unsigned char>(line[i]))) ++i;
    if (i > b) out.push_back(line.substr(b, i - b));
  }
  return out;
}

// istream >> long long semantics for the element count (0 when missing / not a number)
long long to_count(const std::vector<std::string>& tk, size_t i) {
  if (i >= tk.size()) return 0;
  try {
    size_t used = 0;
    return std::stoll(tk[i], &used);
  } catch (...) {
    return 0;
  }
}

struct SceneLayout {
  long long count = -1;
  int stride = 0;
  int off[kSceneFields];
  int is_double[kSceneFields];
  std::streamoff payload = 0;  // byte offset of the first record
};

// Header of a splatting PLY with the reference's acceptance rules and messages.
SceneLayout read_scene_header(std::ifstream& in) {
  std::string line;
  if (!std::getline(in, line) || line != "ply") throw std::runtime_error("malformed PLY header: missing magic");
  struct Prop {
    std::string type, name;
  };
  std::vector<Prop> props;
  SceneLayout L;
  bool in_vertex = false, saw_format = false;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const std::vector<std::string> tk = tokens(line);
    const std::string tok = tk.empty() ? std::string() : tk[0];
    if (tok == "comment") continue;
    if (tok == "format") {
      const std::string fmt = tk.size() > 1 ? tk[1] : std::string();
      if (fmt == "binary_big_endian") throw std::runtime_error("big-endian PLY is not supported");
      if (fmt != "binary_little_endian")
        throw std::runtime_error("malformed PLY header: format must be binary_little_endian");
      saw_format = true;
    } else if (tok == "element") {
      const std::string name = tk.size() > 1 ? tk[1] : std::string();
      L.count = to_count(tk, 2);  // like the reference, the last element line wins
      in_vertex = (name == "vertex");
      if (in_vertex && L.count <= 0) throw std::runtime_error("scene contains no Gaussians");
    } else if (tok == "property") {
      if (!in_vertex) continue;
      Prop p;
      p.type = tk.size() > 1 ? tk[1] : std::string();
      if (p.type == "list") throw std::runtime_error("unsupported property type: list");
      p.name = tk.size() > 2 ? tk[2] : std::string();
      if (ply_size(p.type) < 0) throw std::runtime_error("unsupported property type: " + p.type);
      props.push_back(p);
    } else if (tok == "end_header") {
      break;
    } else if (!tok.empty()) {
      throw std::runtime_error("malformed PLY header: unexpected token " + tok);
    }
  }
  if (!saw_format || L.count < 0 || in.eof()) throw std::runtime_error("malformed PLY header: incomplete");
  std::map<std::string, std::pair<int, std::string>> where;  // a repeated name: the last one wins
  for (const Prop& p : props) {
    where[p.name] = {L.stride, p.type};
    L.stride += ply_size(p.type);
  }
  for (int f = 0; f < kSceneFields; ++f)
    if (!where.count(kRequired[f])) throw std::runtime_error(std::string("missing required property: ") + kRequired[f]);
  for (int f = 0; f < kSceneFields; ++f) {
    const auto& [o, t] = where[kRequired[f]];
    if (t != "float" && t != "float32" && t != "double" && t != "float64")
      throw std::runtime_error("unsupported property type: " + t);  // read_ply_scalar (io_scene.hpp:36-47)
    L.off[f] = o;
    L.is_double[f] = (t == "double" || t == "float64");
  }
  L.payload = in.tellg();
  return L;
}

struct FieldMap {
  int off[kSceneFields];
  int is_double[kSceneFields];
};

__device__ __forceinline__ double field_at(const unsigned char* rec, const FieldMap& fm, int f) {
  const unsigned char* p = rec + fm.off[f];
  if (fm.is_double[f]) {
    uint64_t u = 0;
    for (int k = 0; k < 8; ++k) u |= uint64_t(p[k]) << (8 * k);
    return __longlong_as_double((long long)u);
  }
  uint32_t u = 0;
  for (int k = 0; k < 4; ++k) u |= uint32_t(p[k]) << (8 * k);
  return double(__uint_as_float(u));
}

// One thread per record. err receives min(2 i + kind) over failing records, kind 0 =
// degenerate quaternion (checked first, io_scene.hpp:123), 1 = non-finite value.
__global__ void k_decode_scene(int64_t n, const unsigned char* __restrict__ payload, int stride, FieldMap fm,
                               double* pos, double* scale, double* rot, double* opa, double* dc,
                               unsigned long long* err) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const unsigned char* rec = payload + i * int64_t(stride);
  double v[kSceneFields];
  for (int f = 0; f < kSceneFields; ++f) v[f] = field_at(rec, fm, f);
  double p[3], s[3], d[3];
  for (int k = 0; k < 3; ++k) {
    p[k] = v[k];
    s[k] = sof_exp(v[3 + k]);
    d[k] = 0.5 + kShC0 * v[11 + k];
  }
  // Quat(w, x, y, z) stores (x, y, z, w); norm over that order; normalized = c / norm
  const double qw = v[6], qx = v[7], qy = v[8], qz = v[9];
  const double nq = sqrt(qx * qx + qy * qy + qz * qz + qw * qw);
  unsigned long long e = ~0ull;
  if (nq < 1e-12) e = 2ull * uint64_t(i);
  const double o = 1.0 / (1.0 + sof_exp(-v[10]));
  bool finite = isfinite(o);
  for (int k = 0; k < 3; ++k) finite = finite && isfinite(p[k]) && isfinite(s[k]) && isfinite(d[k]);
  if (e == ~0ull && !finite) e = 2ull * uint64_t(i) + 1;
  if (e != ~0ull) atomicMin(err, e);
  for (int k = 0; k < 3; ++k) {
    pos[3 * i + k] = p[k];
    scale[3 * i + k] = s[k];
    dc[3 * i + k] = d[k];
  }
  rot[4 * i] = qw / nq;
  rot[4 * i + 1] = qx / nq;
  rot[4 * i + 2] = qy / nq;
  rot[4 * i + 3] = qz / nq;
  opa[i] = o;
}

// write_scene's record (io_scene.hpp:161-179): x y z, f_dc_0..2, opacity (logit of the
// clamped opacity), scale_0..2 (log of max(s, 1e-8)), rot_0..3 (w x y z) as float32.
__global__ void k_encode_scene(int64_t n, const double* __restrict__ pos, const double* __restrict__ scale,
                               const double* __restrict__ rot, const double* __restrict__ opa,
                               const double* __restrict__ dc, float* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  float* r = out + kSceneFields * i;
  for (int k = 0; k < 3; ++k) r[k] = float(pos[3 * i + k]);
  for (int k = 0; k < 3; ++k) r[3 + k] = float((dc[3 * i + k] - 0.5) / kShC0);
  double o = opa[i];
  o = (o < 1e-12) ? 1e-12 : ((1.0 - 1e-12 < o) ? 1.0 - 1e-12 : o);  // std::clamp
  r[6] = float(sof_log(o / (1.0 - o)));
  for (int k = 0; k < 3; ++k) {
    const double s = scale[3 * i + k];
    r[7 + k] = float(sof_log((s < 1e-8) ? 1e-8 : s));  // std::max(s, kMinScale)
  }
  for (int k = 0; k < 4; ++k) r[10 + k] = float(rot[4 * i + k]);
}

}  // namespace

}  // namespace sofk

using namespace sofk;

extern "C" int sof_load_scene_ply(sof_ctx* c, const char* path, double filter_scale, int64_t* n_out) {
  if (!c || !path) return SOF_E_INVALID;
  return guard(c, [&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error(std::string("cannot open scene file: ") + path);
    const SceneLayout L = read_scene_header(in);
    in.seekg(0, std::ios::end);
    const std::streamoff avail = std::streamoff(in.tellg()) - L.payload;
    const long long n_full = L.stride > 0 ? std::min<long long>(L.count, avail / L.stride) : L.count;
    std::vector<unsigned char> bytes(size_t(n_full) * L.stride);
    in.seekg(L.payload);
    if (!bytes.empty()) in.read(reinterpret_cast<char*>(bytes.data()), std::streamsize(bytes.size()));
    FieldMap fm;
    for (int f = 0; f < kSceneFields; ++f) {
      fm.off[f] = L.off[f];
      fm.is_double[f] = L.is_double[f];
    }
    const int64_t n = n_full;
    c->io_bytes.ensure(std::max<int64_t>(int64_t(bytes.size()), 1));
    c->pos.ensure(std::max<int64_t>(3 * n, 1));
    c->scale.ensure(std::max<int64_t>(3 * n, 1));
    c->rot.ensure(std::max<int64_t>(4 * n, 1));
    c->opa.ensure(std::max<int64_t>(n, 1));
    c->dc.ensure(std::max<int64_t>(3 * n, 1));
    c->d_counters.ensure(4);
    unsigned long long* err = c->d_counters.p;
    SOF_CUDA(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), c->stream));
    if (n > 0) {
      SOF_CUDA(cudaMemcpyAsync(c->io_bytes.p, bytes.data(), bytes.size(), cudaMemcpyHostToDevice, c->stream));
      k_decode_scene<<<grid_for(n, 256), 256, 0, c->stream>>>(n, c->io_bytes.p, L.stride, fm, c->pos.p,
                                                              c->scale.p, c->rot.p, c->opa.p, c->dc.p, err);
      SOF_LAUNCHED(c);
    }
    unsigned long long e = 0;
    SOF_CUDA(cudaMemcpyAsync(&e, err, sizeof e, cudaMemcpyDeviceToHost, c->stream));
    SOF_CUDA(cudaStreamSynchronize(c->stream));
    // the reference stops at the first failing record, or at the first short read
    if (e != ~0ull) {
      c->has_scene = false;
      throw std::runtime_error((e & 1) ? "non-finite value after activation" : "degenerate rotation quaternion");
    }
    if (n_full < L.count) {
      c->has_scene = false;
      throw std::runtime_error("truncated PLY payload");
    }
    c->n = n;
    c->filter_scale = filter_scale;
    scene_prep(c);
    c->has_scene = true;
    invalidate_view_caches(c);
    SOF_CUDA(cudaStreamSynchronize(c->stream));
    if (n_out) *n_out = n;
  });
}

extern "C" int sof_get_scene(sof_ctx* c, double* pos, double* scale, double* rot_wxyz, double* opacity,
                             double* dc) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (!c->has_scene) throw StateError("no scene: call sof_set_scene first");
    const int64_t n = c->n;
    auto get = [&](double* dst, const DBuf<double>& src, int64_t k) {
      if (dst && n) SOF_CUDA(cudaMemcpyAsync(dst, src.p, sizeof(double) * k * n, cudaMemcpyDeviceToHost, c->stream));
    };
    get(pos, c->pos, 3);
    get(scale, c->scale, 3);
    get(rot_wxyz, c->rot, 4);
    get(opacity, c->opa, 1);
    get(dc, c->dc, 3);
    SOF_CUDA(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int sof_write_scene_ply(sof_ctx* c, const char* path) {
  if (!c || !path) return SOF_E_INVALID;
  return guard(c, [&] {
    if (!c->has_scene) throw StateError("no scene: call sof_set_scene first");
    const int64_t n = c->n;
    std::vector<float> rec(size_t(n) * kSceneFields);
    if (n > 0) {
      c->io_bytes.ensure(int64_t(sizeof(float)) * kSceneFields * n);
      float* d = reinterpret_cast<float*>(c->io_bytes.p);
      k_encode_scene<<<grid_for(n, 256), 256, 0, c->stream>>>(n, c->pos.p, c->scale.p, c->rot.p, c->opa.p,
                                                              c->dc.p, d);
      SOF_LAUNCHED(c);
      SOF_CUDA(cudaMemcpyAsync(rec.data(), d, sizeof(float) * rec.size(), cudaMemcpyDeviceToHost, c->stream));
      SOF_CUDA(cudaStreamSynchronize(c->stream));
    }
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error(std::string("cannot write scene file: ") + path);
    std::string h = "ply\nformat binary_little_endian 1.0\nelement vertex " + std::to_string(n) + "\n";
    for (const char* name : {"x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1",
                             "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"})
      h += std::string("property float ") + name + "\n";
    h += "end_header\n";
    out.write(h.data(), std::streamsize(h.size()));
    out.write(reinterpret_cast<const char*>(rec.data()), std::streamsize(sizeof(float) * rec.size()));
  });
}
