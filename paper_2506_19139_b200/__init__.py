"""B200-native SOF hot path: sorted opacity-field evaluation, Marching Tetrahedra
mesher and sorted rasterizer (arXiv 2506.19139), as hand-written sm_100a CUDA in
libsof_cuda.so behind the C-ABI of include/sof_cuda.h."""
from ._lib import (ALL_STRATEGIES, DEAD_CULL, DEPTH_EXACT, DEPTH_MEDIAN, EARLY_STOP, MIN_Z, NAIVE, PRUNE,
                   SEED_CUT_DEAD, SEED_CUT_NONE, SEED_STP, SEED_STRETCHED_SIGMA, SEED_THREE_SIGMA, TILE_SCHEDULING,
                   declared_symbols, load)
from .api import (CameraSet, Context, EvalStrategies, ExtractOptions, FieldEvaluator, FloatMap, GaussianScene,
                  MarchingResult, Mesh, SeedPointSet, SofError, TetGrid, ViewSet, assemble_mesh,
                  binary_search_refine, build_seed_points, delaunay_tetrahedralize,
                  collect_contributions, windowed_resort, render_pixel, pixel_rays, render_views,
                  default_context, depth_to_map, extract_mesh, load_cameras, save_cameras, extract_resident, gaussian_normal, marching_tets,
                  normal_from_depth, normals_to_map, parse_scene, read_float_map, read_mesh_obj, read_mesh_ply,
                  render_depth_map, render_maps, render_view, write_float_map, write_mesh, write_mesh_obj,
                  write_mesh_ply, write_scene)
from .api import (LossWeights, depth_normal_loss, distortion_loss, extent_loss, l1_rgb_loss, normal_smoothness_loss,
                  opacity_supervision_loss, total_loss)

__all__ = [n for n in dir() if not n.startswith("_")]
