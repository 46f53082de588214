"""B200-native SOF hot path: sorted opacity-field evaluation, Marching Tetrahedra
mesher and sorted rasterizer (arXiv 2506.19139), as hand-written sm_100a CUDA in
libsof_cuda.so behind the C-ABI of include/sof_cuda.h."""
from ._lib import (ALL_STRATEGIES, DEAD_CULL, DEPTH_EXACT, DEPTH_MEDIAN, EARLY_STOP, MIN_Z, NAIVE, PRUNE,
                   TILE_SCHEDULING, declared_symbols, load)
from .api import (CameraSet, Context, EvalStrategies, ExtractOptions, FieldEvaluator, GaussianScene,
                  MarchingResult, Mesh, SofError, TetGrid, ViewSet, assemble_mesh, binary_search_refine,
                  default_context, extract_mesh, extract_resident, marching_tets, render_depth_map,
                  render_view, write_mesh_ply)

__all__ = [n for n in dir() if not n.startswith("_")]
