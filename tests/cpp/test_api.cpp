// The reference's own test cases (proj/tests/test_mesher.cpp, test_opacity_field.cpp),
// rewritten against the drop-in C++ API include/sof_b200/sof.hpp. Compiled and run by
// tests/test_cpp_api.py (GPU) with the in-repo GoogleTest / Eigen shims.
#include <gtest/gtest.h>

#include <algorithm>
#include <random>

#include "sof_b200/sof.hpp"

using namespace sof;

namespace {

TetGrid single_tet(const std::array<double, 4>& opacity) {
  TetGrid grid;
  grid.vertices = {Vec3(0, 0, 0), Vec3(1, 0, 0), Vec3(0, 1, 0), Vec3(0, 0, 1)};
  grid.tetrahedra = {{0, 1, 2, 3}};
  grid.opacity.assign(opacity.begin(), opacity.end());
  return grid;
}

Camera look_at(const Vec3& eye, const Vec3& target, const Vec3& up, double f, int res) {
  Camera cam;
  const Vec3 fwd = (target - eye).normalized();
  const Vec3 right = fwd.cross(up).normalized();
  const Vec3 down = fwd.cross(right);
  cam.rotation.row(0) = right.transpose();
  cam.rotation.row(1) = down.transpose();
  cam.rotation.row(2) = fwd.transpose();
  cam.translation = -cam.rotation * eye;
  cam.fx = cam.fy = f;
  cam.width = cam.height = res;
  cam.cx = cam.cy = res * 0.5;
  return cam;
}

std::vector<GaussianPrimitive> random_scene(unsigned seed, int count) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> up(-1, 1), us(0.05, 0.25), uo(0.4, 0.95);
  std::normal_distribution<double> n(0, 1);
  std::vector<GaussianPrimitive> out(count);
  for (auto& g : out) {
    g.position = Vec3(up(rng), up(rng), up(rng));
    g.scale = Vec3(us(rng), us(rng), us(rng));
    g.rotation = Quat(n(rng), n(rng), n(rng), n(rng)).normalized();
    g.opacity = uo(rng);
  }
  return out;
}

TetGrid lattice(int n, double lo, double hi) {
  TetGrid g;
  const double h = (hi - lo) / (n - 1);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) g.vertices.emplace_back(lo + i * h, lo + j * h, lo + k * h);
  auto id = [n](int i, int j, int k) { return i + n * (j + n * k); };
  for (int k = 0; k + 1 < n; ++k)
    for (int j = 0; j + 1 < n; ++j)
      for (int i = 0; i + 1 < n; ++i) {
        const int a = id(i, j, k), b = id(i + 1, j, k), c = id(i + 1, j + 1, k), d = id(i + 1, j + 1, k + 1);
        const int e = id(i, j + 1, k), f = id(i, j + 1, k + 1), gg = id(i, j, k + 1), hh = id(i + 1, j, k + 1);
        g.tetrahedra.push_back({a, b, c, d});
        g.tetrahedra.push_back({a, b, hh, d});
        g.tetrahedra.push_back({a, e, c, d});
        g.tetrahedra.push_back({a, e, f, d});
        g.tetrahedra.push_back({a, gg, hh, d});
        g.tetrahedra.push_back({a, gg, f, d});
      }
  return g;
}

}  // namespace

TEST(MarchingTets, OneInsideCorner) {
  const auto out = marching_tets(single_tet({0.4, 0.4, 0.4, 0.6}));
  ASSERT_EQ(out.triangles.size(), 1u);
  EXPECT_EQ(out.edges.size(), 3u);
  for (const auto& e : out.edges) EXPECT_EQ(e.inside, 3);
}

TEST(MarchingTets, TwoInsideQuad) {
  const auto out = marching_tets(single_tet({0.4, 0.4, 0.6, 0.6}));
  EXPECT_EQ(out.triangles.size(), 2u);
  EXPECT_EQ(out.edges.size(), 4u);
}

TEST(MarchingTets, NoCrossingNoOutput) {
  EXPECT_TRUE(marching_tets(single_tet({0.6, 0.7, 0.8, 0.9})).triangles.empty());
  EXPECT_TRUE(marching_tets(single_tet({0.1, 0.2, 0.3, 0.4})).triangles.empty());
}

TEST(MarchingTets, LinearInterpolation) {
  const auto out = marching_tets(single_tet({0.4, 0.6, 0.4, 0.4}));
  ASSERT_EQ(out.edges.size(), 3u);
  for (size_t i = 0; i < out.edges.size(); ++i) {
    const Vec3 mid = 0.5 * (Vec3(1, 0, 0) + single_tet({0, 0, 0, 0}).vertices[out.edges[i].outside]);
    EXPECT_LT((out.vertices[i] - mid).norm(), 1e-12);
  }
}

TEST(BinarySearchRefine, BisectionBound) {
  auto grid = single_tet({0.6, 0.4, 0.4, 0.4});
  auto out = marching_tets(grid);
  const double crossing = 0.37;
  binary_search_refine(out, grid, [&](const Vec3& p) { return p.x() < crossing; }, 8);
  for (size_t i = 0; i < out.edges.size(); ++i) {
    if (out.edges[i].outside != 1) continue;
    EXPECT_NEAR(out.vertices[i].x(), crossing, 1.0 / 256.0);
  }
}

TEST(AssembleMesh, WeldAndDegenerate) {
  const std::vector<Vec3> verts{Vec3(0, 0, 0), Vec3(1, 0, 0), Vec3(0, 1, 0), Vec3(1 + 1e-9, 0, 0)};
  const std::vector<std::array<int, 3>> tris{{0, 1, 2}, {0, 3, 2}, {0, 1, 3}};
  const auto mesh = assemble_mesh(verts, tris);
  EXPECT_EQ(mesh.vertices.size(), 3u);
  EXPECT_EQ(mesh.triangles.size(), 2u);
}

TEST(AssembleMesh, EmptyInput) {
  const auto mesh = assemble_mesh({}, {});
  EXPECT_TRUE(mesh.vertices.empty());
  EXPECT_TRUE(mesh.triangles.empty());
}

TEST(FieldEvaluator, SingleViewMahalanobisBall) {
  GaussianPrimitive g;
  g.scale = Vec3(0.3, 0.3, 0.3);
  const std::vector<GaussianPrimitive> scene{g};
  const ViewSet views = ViewSet::build(scene, {look_at(Vec3(0, 0, 3), Vec3::Zero(), Vec3(0, 1, 0), 0.4 * 64 * 3.0, 64)});
  const FieldEvaluator eval(scene, views, EvalStrategies::all());
  std::mt19937 rng(53);
  std::uniform_real_distribution<double> u(-0.5, 0.5);
  const double iso = std::sqrt(2.0 * std::log(2.0));
  for (int i = 0; i < 200; ++i) {
    const Vec3 x(u(rng), u(rng), u(rng));
    const double mahal = x.norm() / 0.3;
    if (std::abs(mahal - iso) < 0.02) continue;
    if (views.cameras[0].to_view(x).z() >= 3.0) continue;
    EXPECT_EQ(eval.classify_point(x), mahal < iso) << x.transpose();
  }
}

TEST(FieldEvaluator, StrategiesAgreeAndReducePairs) {
  const auto scene = random_scene(54, 40);
  std::vector<Camera> cams;
  for (int i = 0; i < 4; ++i) {
    const double a = 2.0 * M_PI * i / 4;
    cams.push_back(look_at(Vec3(4 * std::cos(a), 4 * std::sin(a), 0.5), Vec3::Zero(), Vec3(0, 0, 1), 60.0, 64));
  }
  const ViewSet views = ViewSet::build(scene, cams);
  TetGrid grid = lattice(12, -1.3, 1.3);
  const FieldEvaluator naive(scene, views, EvalStrategies::naive());
  const FieldEvaluator fast(scene, views, EvalStrategies::all());
  TetGrid g1 = grid, g2 = grid;
  naive.label_grid(g1, true);
  fast.label_grid(g2, true);
  for (size_t i = 0; i < grid.vertices.size(); ++i) EXPECT_EQ(g1.opacity[i] >= 0.5, g2.opacity[i] >= 0.5);
  EXPECT_GE(naive.counters().pairs, 2 * fast.counters().pairs);
  ExtractOptions on, off;
  off.strategies = EvalStrategies::naive();
  const Mesh m1 = extract_mesh(scene, views, grid, on), m2 = extract_mesh(scene, views, grid, off);
  ASSERT_EQ(m1.vertices.size(), m2.vertices.size());
  ASSERT_GT(m1.triangles.size(), 0u);
  for (size_t i = 0; i < m1.vertices.size(); ++i)
    EXPECT_LT((m1.vertices[i] - m2.vertices[i]).cwiseAbs().maxCoeff(), 1e-9);
}

TEST(RenderDepthMap, SingleGaussianDisk) {
  GaussianPrimitive g;
  const std::vector<GaussianPrimitive> scene{g};
  const Camera cam = look_at(Vec3(0, 0, -5), Vec3::Zero(), Vec3(0, 1, 0), 0.4 * 32 * 5.0 / 2.0, 32);
  const ViewSet views = ViewSet::build(scene, {cam});
  const auto exact = render_depth_map(views, 0, DepthMode::kExact);
  const auto median = render_depth_map(views, 0, DepthMode::kMedian);
  EXPECT_NEAR(exact.depth.at(16, 16), 3.82258, 0.01);
  EXPECT_NEAR(median.depth.at(16, 16), 5.0, 0.01);
  for (int y = 0; y < cam.height; ++y)
    for (int x = 0; x < cam.width; ++x)
      EXPECT_EQ(is_no_surface(exact.depth.at(x, y)), is_no_surface(median.depth.at(x, y)));
}

TEST(NormalFromDepth, FrontoParallelPlaneAndMaps) {
  // test_opacity_field.cpp:285-298 with the camera of a ViewSet; then the float maps
  Camera cam;
  cam.width = cam.height = 16;
  cam.cx = cam.cy = 8;
  cam.fx = cam.fy = 20;
  const ViewSet views = ViewSet::build({GaussianPrimitive{}}, {cam});
  Grid2D<double> depth(16, 16, 0.0);
  for (int y = 0; y < 16; ++y)
    for (int x = 0; x < 16; ++x) {
      const Vec3 d = Vec3((x + 0.5 - 8) / 20.0, (y + 0.5 - 8) / 20.0, 1.0).normalized();
      depth.at(x, y) = 5.0 / d.z();
    }
  const NormalMap nm = normal_from_depth(depth, views, 0);
  ASSERT_TRUE(nm.valid.at(8, 8));
  EXPECT_TRUE(nm.normal.at(8, 8).isApprox(Vec3(0, 0, -1), 1e-9));
  EXPECT_FALSE(nm.valid.at(15, 15));
  const FloatMap fm = normals_to_map(nm);
  write_float_map(fm, "/tmp/sof_b200_test_normals.sofmap");
  const FloatMap back = read_float_map("/tmp/sof_b200_test_normals.sofmap");
  EXPECT_EQ(back.width, 16);
  EXPECT_EQ(back.channels, 3);
  EXPECT_EQ(back.data, fm.data);
  // GaussianNormal.RadialAndFallback (test_opacity_field.cpp:330-340)
  const Ray ray{Vec3(0, 0, -5), Vec3(0, 0, 1)};
  EXPECT_TRUE(gaussian_normal(views, 0, ray, 6.0).isApprox(Vec3(0, 0, -1), 1e-12));
}

TEST(SceneIO, RoundTripAndErrors) {
  // SceneIO.RoundTrip / RotationsNormalizedOnLoad / MalformedHeaderRejected (test_io.cpp:41-107)
  std::vector<GaussianPrimitive> scene(20);
  for (int i = 0; i < 20; ++i) {
    scene[i].position = Vec3(0.1 * i, -0.2 * i, 0.3);
    scene[i].scale = Vec3(0.05 + 0.01 * i, 0.2, 0.1);
    scene[i].rotation = Quat(1, 0.1 * i, 2, 3).normalized();
    scene[i].opacity = 0.04 * i + 0.01;
    scene[i].dc_color = Vec3(0.3, 0.5, 0.7);
  }
  write_scene(scene, "/tmp/sof_b200_scene.ply");
  const SceneFile loaded = parse_scene("/tmp/sof_b200_scene.ply");
  ASSERT_EQ(loaded.gaussians.size(), scene.size());
  for (size_t i = 0; i < scene.size(); ++i) {
    EXPECT_LT((scene[i].position - loaded.gaussians[i].position).norm(), 1e-5);
    EXPECT_NEAR(scene[i].opacity, loaded.gaussians[i].opacity, 1e-6);
    EXPECT_NEAR(loaded.gaussians[i].rotation.norm(), 1.0, 1e-12);
  }
  {
    std::ofstream f("/tmp/sof_b200_bad.ply");
    f << "not a ply file\n";
  }
  bool threw = false;
  try {
    parse_scene("/tmp/sof_b200_bad.ply");
  } catch (const std::runtime_error& e) {
    threw = std::string(e.what()).find("malformed PLY header") != std::string::npos;
  }
  EXPECT_TRUE(threw);
  Mesh m;
  m.vertices = {Vec3(0, 0, 0), Vec3(1, 0, 0), Vec3(0, 1, 0.123456789012345678)};
  m.triangles = {{0, 1, 2}};
  write_mesh(m, "/tmp/sof_b200_m.obj", MeshFormat::kObj);
  write_mesh(m, "/tmp/sof_b200_m.ply", MeshFormat::kPlyBinary);
  const Mesh a = read_mesh_obj("/tmp/sof_b200_m.obj"), b = read_mesh_ply("/tmp/sof_b200_m.ply");
  ASSERT_EQ(a.vertices.size(), 3u);
  EXPECT_EQ(a.vertices[2](2), m.vertices[2](2));
  EXPECT_EQ(b.vertices[2](2), m.vertices[2](2));
  EXPECT_EQ(b.triangles[0][2], 2);
}

TEST(SeedPoints, CentresAndCorners) {
  GaussianPrimitive g;  // unit Gaussian, opacity 1: centre + 8 corners at +-E
  GaussianPrimitive dead;
  dead.position = Vec3(5, 0, 0);
  dead.opacity = 0.001;
  const ViewSet views = ViewSet::build({g, dead}, {Camera{}});
  const SeedPointSet s = build_seed_points(views, BoundingVariant::kThreeSigma, SeedCutoff::kDeadGaussians);
  ASSERT_EQ(s.points.size(), 9u);
  EXPECT_EQ(s.provenance[0], SeedProvenance::kCenter);
  EXPECT_EQ(s.points[1](0), -3.0);
  EXPECT_EQ(s.points[8](2), 3.0);
  const SeedPointSet all = build_seed_points(views, BoundingVariant::kThreeSigma, SeedCutoff::kNone);
  EXPECT_EQ(all.points.size(), 18u);
}

TEST(Errors, NonFiniteScene) {
  GaussianPrimitive g;
  g.position = Vec3(0, std::nan(""), 0);
  EXPECT_THROW(ViewSet::build({g}, {Camera{}}), std::invalid_argument);
}

// ---- training losses: the reference's tests/test_losses.cpp cases ----------------

namespace {
double ndc_inverse(double d, double near, double far) { return far * near / (far - d * (far - near)); }
}  // namespace

TEST(Distortion, ConstantDepthIsZero) {
  const double t = ndc_inverse(0.5, 0.2, 100.0);
  const auto res = distortion_loss({{0.3, t}, {0.4, t}, {0.2, t}}, 0.2, 100.0);
  EXPECT_NEAR(res.loss, 0.0, 1e-15);
  for (double g : res.d_t) EXPECT_NEAR(g, 0.0, 1e-12);
}

TEST(Distortion, TwoSampleExample) {
  const double t1 = ndc_inverse(0.2, 0.2, 100.0);
  const double t2 = ndc_inverse(0.8, 0.2, 100.0);
  const auto res = distortion_loss({{0.5, t1}, {1.0, t2}}, 0.2, 100.0);
  EXPECT_NEAR(res.loss, 0.18, 1e-12);
}

TEST(Distortion, DetachFlagDropsAlphaGradients) {
  const auto res = distortion_loss({{0.5, 1.0}, {0.5, 2.0}}, 0.2, 100.0, false);
  EXPECT_TRUE(res.d_alpha.empty());
  EXPECT_EQ(res.d_t.size(), 2u);
}

TEST(DepthNormal, Examples) {
  const Vec3 N(0, 0, 1);
  EXPECT_NEAR(depth_normal_loss({1.0}, {N}, N).loss, 0.0, 1e-15);
  EXPECT_NEAR(depth_normal_loss({1.0}, {Vec3(0, 0, -1)}, N).loss, 2.0, 1e-12);
  EXPECT_NEAR(depth_normal_loss({0.5, 0.25}, {N, Vec3(1, 0, 0)}, N).loss, 0.25, 1e-12);
}

TEST(Extent, PlugInExample) {
  ExtentSample s;
  s.w = 1.0;
  s.a = 1.0;
  s.b = -10.0;
  s.c = 25.0;
  s.bound = std::sqrt(2.0 * std::log(255.0));  // tight_bound(1.0)
  const auto res = extent_loss({s}, 0.2, 100.0);
  EXPECT_EQ(res.skipped, 0);
  EXPECT_NEAR(res.loss, 0.026686, 1e-5);
}

TEST(Extent, EmptyVisibleSegmentSkipped) {
  ExtentSample s;
  s.w = 1.0;
  s.a = 1.0;
  s.b = -10.0;
  s.c = 25.0;
  s.bound = 0.0;
  const auto res = extent_loss({s}, 0.2, 100.0);
  EXPECT_EQ(res.skipped, 1);
  EXPECT_NEAR(res.loss, 0.0, 1e-15);
}

TEST(OpacitySupervision, NoSurfaceIsZero) {
  RayContribution rc;  // tu::flat_contribution(0.2, 3.0)
  rc.gaussian_index = 0;
  rc.t_star = 3.0;
  rc.alpha = 0.2;
  rc.a = 1.0;
  rc.b = -6.0;
  rc.c = 9.0;
  rc.opacity = 0.2;
  const auto res = opacity_supervision_loss({rc}, kNoSurface);
  EXPECT_FALSE(res.defined);
  EXPECT_DOUBLE_EQ(res.loss, 0.0);
}

TEST(NormalSmoothness, ConstantMapIsZero) {
  NormalMap nm;
  nm.normal = Grid2D<Vec3>(8, 8, Vec3(0, 0, -1));
  nm.valid = Grid2D<unsigned char>(8, 8, 1);
  const Grid2D<Vec3> image(8, 8, Vec3(0.5, 0.5, 0.5));
  EXPECT_NEAR(normal_smoothness_loss(nm, image).loss, 0.0, 1e-15);
}

TEST(NormalSmoothness, FlatImageEqualsTotalVariation) {
  NormalMap nm;
  nm.normal = Grid2D<Vec3>(4, 4, Vec3(0, 0, -1));
  nm.valid = Grid2D<unsigned char>(4, 4, 1);
  for (int y = 0; y < 4; ++y)
    for (int x = 2; x < 4; ++x) nm.normal.at(x, y) = Vec3(0, 0, 1);
  const Grid2D<Vec3> image(4, 4, Vec3(0.5, 0.5, 0.5));
  EXPECT_NEAR(normal_smoothness_loss(nm, image).loss, 3.0 * 2.0 / 9.0, 1e-12);
}

TEST(TotalLoss, GatingAndWeights) {
  LossWeights w;
  LossTerms terms;
  terms.rgb = 0.5;
  terms.distortion = terms.normal = terms.extent = terms.opacity = terms.smoothness = 1.0;
  EXPECT_DOUBLE_EQ(total_loss(terms, w, 14999, false), 0.5);
  EXPECT_DOUBLE_EQ(total_loss(terms, w, 15000, false), 0.5 + 100.0 + 0.05 + 0.1 + 0.04 + 0.01);
  EXPECT_DOUBLE_EQ(total_loss(terms, w, 15000, true), 0.5 + 1000.0 + 0.05 + 0.1 + 0.04 + 0.01);
}

TEST(L1Rgb, MeanAbsoluteError) {
  Grid2D<Vec3> a(2, 1, Vec3(0.5, 0.5, 0.5));
  Grid2D<Vec3> b(2, 1, Vec3(0.25, 0.5, 0.5));
  EXPECT_NEAR(l1_rgb_loss(a, b), 0.25 * 2 / 6.0, 1e-12);
}

TEST(AssembleMesh, ResidualPassthrough) {
  // mesh.hpp:66: a welded vertex keeps the residual of its first appearance
  const std::vector<Vec3> verts{Vec3(0, 0, 0), Vec3(1, 0, 0), Vec3(0, 1, 0), Vec3(1 + 1e-9, 0, 0)};
  const std::vector<std::array<int, 3>> tris{{0, 1, 2}, {0, 3, 2}};
  const std::vector<double> res{0.1, 0.2, 0.3, 0.4};
  const auto mesh = assemble_mesh(verts, tris, &res);
  ASSERT_EQ(mesh.vertices.size(), 3u);
  ASSERT_EQ(mesh.residuals.size(), 3u);
  EXPECT_EQ(mesh.residuals[0], 0.1);
  EXPECT_EQ(mesh.residuals[1], 0.2);
  EXPECT_EQ(mesh.residuals[2], 0.3);
  const std::vector<double> bad{0.1};
  EXPECT_THROW(assemble_mesh(verts, tris, &bad), std::invalid_argument);
}

TEST(Delaunay, ErrorsLikeTheReference) {
  EXPECT_THROW(delaunay_tetrahedralize({Vec3(0, 0, 0), Vec3(1, 0, 0), Vec3(0, 1, 0)}), std::invalid_argument);
  EXPECT_THROW(delaunay_tetrahedralize({Vec3(0, 0, 0), Vec3(1, 0, 0), Vec3(0, 1, 0), Vec3(1, 1, 0)}),
               std::invalid_argument);
  const TetGrid g = delaunay_tetrahedralize({Vec3(0, 0, 0), Vec3(1, 0, 0), Vec3(0, 1, 0), Vec3(0, 0, 1)});
  ASSERT_EQ(g.tetrahedra.size(), 1u);
}

TEST(ExtractMesh, ReferenceSignatureWithResiduals) {
  // extract.hpp:35-86: seeds -> Delaunay -> label -> march -> refine -> residuals -> weld
  const auto scene = random_scene(57, 25);
  std::vector<Camera> cams;
  for (int i = 0; i < 4; ++i) {
    const double a = 2.0 * M_PI * i / 4;
    cams.push_back(look_at(Vec3(4 * std::cos(a), 4 * std::sin(a), 0.5), Vec3::Zero(), Vec3(0, 0, 1), 60.0, 64));
  }
  const ViewSet views = ViewSet::build(scene, cams);
  ExtractOptions opt;
  opt.compute_residuals = true;
  ExtractStats st;
  const Mesh m = extract_mesh(scene, views, opt, &st);
  ASSERT_GT(m.triangles.size(), 0u);
  ASSERT_EQ(m.residuals.size(), m.vertices.size());
  for (double r : m.residuals) EXPECT_LT(r, 0.5);
  EXPECT_GT(st.seed_points, 0u);
  EXPECT_GT(st.tetrahedra, 0u);
  EXPECT_GT(st.crossing_edges, 0u);
  EXPECT_GT(st.counters.pairs, 0u);
  // the same mesh through the explicit producer + the tetra-input overload
  const SeedPointSet seeds = build_seed_points(views, opt.bounding, opt.cutoff, opt.filter_scale);
  ASSERT_EQ(seeds.points.size(), st.seed_points);
  const TetGrid grid = delaunay_tetrahedralize(seeds.points);
  ASSERT_EQ(grid.tetrahedra.size(), st.tetrahedra);
  const Mesh m2 = extract_mesh(scene, views, grid, opt);
  ASSERT_EQ(m2.vertices.size(), m.vertices.size());
  for (size_t i = 0; i < m.vertices.size(); ++i) {
    EXPECT_EQ(m.vertices[i], m2.vertices[i]);
    EXPECT_EQ(m.residuals[i], m2.residuals[i]);
  }
  EXPECT_THROW(extract_mesh(std::vector<GaussianPrimitive>(3), views, opt), std::invalid_argument);
}

TEST(BinarySearchRefine, BatchedAddsCountersAndMatchesHostLoop) {
  const auto scene = random_scene(58, 20);
  std::vector<Camera> cams;
  for (int i = 0; i < 3; ++i) {
    const double a = 2.0 * M_PI * i / 3;
    cams.push_back(look_at(Vec3(4 * std::cos(a), 4 * std::sin(a), 0.5), Vec3::Zero(), Vec3(0, 0, 1), 60.0, 64));
  }
  const ViewSet views = ViewSet::build(scene, cams);
  TetGrid grid = lattice(8, -1.3, 1.3);
  const FieldEvaluator eval(scene, views, EvalStrategies::all());
  eval.label_grid(grid, true);
  MarchingResult a = marching_tets(grid);
  ASSERT_GT(a.edges.size(), 0u);
  MarchingResult b = a;
  const EvalCounters before = eval.counters();
  const RefineStats rs = binary_search_refine(a, grid, eval, 8);
  EXPECT_EQ(rs.bracket_lost, 0u);
  const EvalCounters after = eval.counters();
  EXPECT_GT(after.pairs, before.pairs);
  EXPECT_GT(after.point_view_evals, before.point_view_evals);
  const FieldEvaluator host(scene, views, EvalStrategies::all());
  binary_search_refine(b, grid, [&](const Vec3& x) { return host.classify_point(x); }, 8);
  for (size_t i = 0; i < a.vertices.size(); ++i) EXPECT_EQ(a.vertices[i], b.vertices[i]);
  // the batched residuals equal the host loop over value_at
  const FieldEvaluator exact(scene, views, EvalStrategies::naive());
  const auto r1 = level_set_residuals(a, exact);
  const auto r2 = level_set_residuals(a, [&](const Vec3& x) { return exact.value_at(x); });
  ASSERT_EQ(r1.size(), a.vertices.size());
  for (size_t i = 0; i < r1.size(); ++i) EXPECT_EQ(r1[i], r2[i]);
}

// ---- per-ray compositing (test_opacity_field.cpp:28-82, 239-285) through the device ------------

namespace {
GaussianPrimitive axis_gaussian(double z, double opacity) {
  GaussianPrimitive g;
  g.position = Vec3(0, 0, z);
  g.opacity = opacity;
  return g;
}
RayContribution flat(double alpha, double t_star, int index = 0) {  // alpha(t) = alpha for t >= t*
  RayContribution rc;
  rc.gaussian_index = index;
  rc.a = 1.0;
  rc.b = -2.0 * t_star;
  rc.c = t_star * t_star;
  rc.t_star = t_star;
  rc.alpha = alpha;
  rc.opacity = alpha;
  return rc;
}
std::vector<RayContribution> random_list(std::mt19937& rng, int count) {
  std::uniform_real_distribution<double> ua(0.3, 2.0), ut(0.5, 15.0), um(0.0, 1.0), uo(0.2, 0.95);
  std::vector<RayContribution> out;
  for (int i = 0; i < count; ++i) {
    RayContribution rc;
    rc.gaussian_index = i;
    rc.a = ua(rng);
    rc.t_star = ut(rng);
    rc.b = -2.0 * rc.a * rc.t_star;
    const double m = um(rng);
    rc.c = rc.b * rc.b / (4.0 * rc.a) + m * m;
    rc.opacity = uo(rng);
    rc.alpha = std::min(rc.opacity * std::exp(-0.5 * m * m), kMaxAlpha);
    out.push_back(rc);
  }
  return out;
}
}  // namespace

TEST(CollectContributions, SingleOnAxisAndSorted) {
  Camera cam;
  const auto one = collect_contributions(precompute_all({axis_gaussian(5.0, 0.8)}, cam), Ray{cam.center(), Vec3(0, 0, 1)});
  ASSERT_EQ(one.size(), 1u);
  EXPECT_NEAR(one[0].t_star, 5.0, 1e-12);
  EXPECT_NEAR(one[0].alpha, 0.8, 1e-12);
  const auto two = collect_contributions(precompute_all({axis_gaussian(7.0, 0.5), axis_gaussian(3.0, 0.5)}, cam),
                                         Ray{cam.center(), Vec3(0, 0, 1)});
  ASSERT_EQ(two.size(), 2u);
  EXPECT_NEAR(two[0].t_star, 3.0, 1e-12);
  EXPECT_EQ(two[0].gaussian_index, 1);
  EXPECT_NEAR(two[1].t_star, 7.0, 1e-12);
  EXPECT_TRUE(collect_contributions(precompute_all({axis_gaussian(5.0, 1.0 / 300.0)}, cam),
                                    Ray{cam.center(), Vec3(0, 0, 1)})
                  .empty());
}

TEST(RenderPixel, OpaqueBlendAndEmpty) {
  std::vector<GaussianPrimitive> scene{axis_gaussian(5.0, 1.0)};
  scene[0].dc_color = Vec3(0.2, 0.4, 0.6);
  const auto o1 = render_pixel({flat(0.999, 5.0)}, scene);
  EXPECT_TRUE(o1.color.isApprox(0.999 * scene[0].dc_color, 1e-9));
  EXPECT_NEAR(o1.transmittance_final, 0.001, 1e-12);
  std::vector<GaussianPrimitive> two{axis_gaussian(3.0, 1.0), axis_gaussian(7.0, 1.0)};
  two[0].dc_color = Vec3(1, 1, 1);
  two[1].dc_color = Vec3(0, 0, 0);
  const auto o2 = render_pixel({flat(0.5, 3.0, 0), flat(0.5, 7.0, 1)}, two);
  EXPECT_NEAR(o2.color.x(), 0.5, 1e-12);
  EXPECT_NEAR(o2.transmittance_final, 0.25, 1e-12);
  const auto o3 = render_pixel({}, {});
  EXPECT_LT(o3.color.norm(), 1e-15);
  EXPECT_DOUBLE_EQ(o3.transmittance_final, 1.0);
  EXPECT_TRUE(is_no_surface(o3.depth));
  EXPECT_THROW(render_pixel({flat(0.5, 3.0, 4)}, two), std::out_of_range);
}

TEST(WindowedResort, FullWindowSortsSmallWindowPermutes) {
  std::mt19937 rng(25);
  auto contribs = random_list(rng, 16);
  std::shuffle(contribs.begin(), contribs.end(), rng);
  const auto sorted = windowed_resort(contribs, contribs.size());
  for (size_t i = 1; i < sorted.size(); ++i) EXPECT_LE(sorted[i - 1].t_star, sorted[i].t_star);
  const auto out = windowed_resort(contribs, 4);
  ASSERT_EQ(out.size(), contribs.size());
  std::vector<int> a, b;
  for (const auto& r : out) a.push_back(r.gaussian_index);
  for (const auto& r : contribs) b.push_back(r.gaussian_index);
  std::sort(a.begin(), a.end());
  std::sort(b.begin(), b.end());
  EXPECT_EQ(a, b);
}

TEST(RenderDepthMap, CacheSignatureAndEmptyScene) {
  const std::vector<GaussianPrimitive> scene{axis_gaussian(0.0, 1.0)};
  const Camera cam = look_at(Vec3(0, 0, -5), Vec3::Zero(), Vec3(0, 1, 0), 0.4 * 32 * 5.0 / 2.0, 32);
  const auto cache = precompute_all(scene, cam);
  const auto exact = render_depth_map(cache, cam, DepthMode::kExact);
  const auto median = render_depth_map(cache, cam, DepthMode::kMedian);
  EXPECT_NEAR(exact.depth.at(16, 16), 3.82258, 0.01);
  EXPECT_NEAR(median.depth.at(16, 16), 5.0, 0.01);
  Camera other = cam;
  other.fx *= 2.0;
  EXPECT_THROW(render_depth_map(cache, other, DepthMode::kExact), std::invalid_argument);
  Camera small;
  small.width = small.height = 8;
  small.cx = small.cy = 4;
  const auto dm = render_depth_map(ViewCache{}, small, DepthMode::kExact);
  for (double d : dm.depth.data) EXPECT_TRUE(is_no_surface(d));
  // the per-pixel API agrees with the image render at the centre pixel
  const auto lists = collect_contributions(cache, std::vector<Ray>{ray_through_pixel(cam, 16.5, 16.5)});
  const PixelOutputs px = render_pixel(lists[0], scene);
  EXPECT_EQ(px.depth, exact.depth.at(16, 16));
  EXPECT_EQ(px.accumulated_opacity, exact.opacity.at(16, 16));
}

TEST(RenderViews, BatchEqualsPerViewMaps) {
  const auto scene = random_scene(62, 30);
  std::vector<Camera> cams;
  for (int i = 0; i < 3; ++i) {
    const double a = 2.0 * M_PI * i / 3;
    cams.push_back(look_at(Vec3(4 * std::cos(a), 4 * std::sin(a), 0.5), Vec3::Zero(), Vec3(0, 0, 1), 40.0, 32));
  }
  const ViewSet views = ViewSet::build(scene, cams);
  const auto batch = render_views(views, 1, 2);
  ASSERT_EQ(batch.size(), 2u);
  for (size_t k = 0; k < 2; ++k) {
    const DepthMap dm = render_depth_map(views.caches[1 + k], views.cameras[1 + k], DepthMode::kExact);
    for (size_t i = 0; i < dm.depth.data.size(); ++i) {
      const double a = dm.depth.data[i], b = batch[k].depth.data[i];
      EXPECT_TRUE((std::isnan(a) && std::isnan(b)) || a == b);
      EXPECT_EQ(dm.opacity.data[i], batch[k].opacity.data[i]);
    }
  }
  EXPECT_THROW(render_views(views, 2, 2), std::invalid_argument);
}
