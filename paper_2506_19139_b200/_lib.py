"""ctypes binding of libsof_cuda.so (include/sof_cuda.h).

The shared library is the product; this module only declares argument types. It
fails loudly when the library is missing — there is no CPU fallback anywhere in
this package.
"""
from __future__ import annotations

import ctypes
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SOF_LIB_PATH") or os.path.join(PKG, "libsof_cuda.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "sof_cuda.h")

SOF_OK, SOF_E_INVALID, SOF_E_CUDA, SOF_E_NCCL, SOF_E_OOM, SOF_E_STATE, SOF_E_RUNTIME = 0, -1, -2, -3, -4, -5, -6
TILE_SCHEDULING, MIN_Z, EARLY_STOP, PRUNE, DEAD_CULL = 1, 2, 4, 8, 16
ALL_STRATEGIES, NAIVE = 31, 0
DEPTH_MEDIAN, DEPTH_EXACT = 0, 1
R_EDGES, R_EDGE_VERTS, R_TRIANGLES, R_MESH_VERTS, R_MESH_TRIS, R_GRID_OPACITY, R_TILE_OFFSETS, R_TILE_ENTRIES = range(1, 9)
R_SEEDS, R_SEED_PROVENANCE, R_MESH_RESIDUALS, R_TETS = 9, 10, 11, 12
R_CONTRIB_INDEX, R_CONTRIB_VALUES = 13, 14
SEED_STP, SEED_THREE_SIGMA, SEED_STRETCHED_SIGMA = 0, 1, 2
SEED_CUT_NONE, SEED_CUT_DEAD = 0, 1
SOF_COMM_ID_BYTES = 128

_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_I64 = ctypes.c_int64


class ExtractOpts(ctypes.Structure):
    _fields_ = [("strategies", _I), ("tile_size", _I), ("refine_iterations", _I),
                ("weld_eps", _D), ("min_area", _D), ("view_begin", _I), ("view_end", _I), ("profile", _I),
                ("compute_residuals", _I)]


class ExtractStats(ctypes.Structure):
    _fields_ = [("crossing_edges", _I64), ("march_triangles", _I64), ("mesh_vertices", _I64),
                ("mesh_triangles", _I64), ("pairs", ctypes.c_uint64), ("point_view_evals", ctypes.c_uint64),
                ("label_pairs", ctypes.c_uint64), ("refine_pairs", ctypes.c_uint64),
                ("ms_label", _D), ("ms_march", _D), ("ms_refine", _D), ("ms_weld", _D),
                ("ms_eval_kernel", _D), ("eval_launches", _I64), ("kernel_launches", _I64),
                ("ms_prep", _D), ("ms_sched", _D), ("exact_pairs", ctypes.c_uint64),
                ("host_ms_prep", _D), ("host_ms_sched", _D), ("contrib_pairs", ctypes.c_uint64),
                ("scanned_pairs", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_SIGS = {
    "sof_version": (_I, []),
    "sof_last_error": (ctypes.c_char_p, [_P]),
    "sof_kernel_launches": (_I64, [_P]),
    "sof_scene_size": (_I64, [_P]),
    "sof_render_views": (_I, [_P, _I, _I, _I, _P, _P, _P, _P]),
    "sof_stream_wait": (_I, [_P, _P]),
    "sof_get_stream": (_I, [_P, ctypes.POINTER(_P)]),
    "sof_live_binding_stats": (_I, [_P, _I, _I, _P]),
    "sof_set_render_window": (_I, [_P, _I64]),
    "sof_collect_contributions": (_I, [_P, _I, _I64, _P, _P]),
    "sof_windowed_resort": (_I, [_P, _I64, _P, _P, _I64, _P]),
    "sof_render_pixel": (_I, [_P, _I64, _P, _P, _P, _I64, _P, _I, _P, _P, _P, _P]),
    "sof_ctx_create": (_I, [_I, ctypes.POINTER(_P)]),
    "sof_ctx_destroy": (None, [_P]),
    "sof_set_scene": (_I, [_P, _I64, _P, _P, _P, _P, _P, _D]),
    "sof_set_views": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "sof_set_tets": (_I, [_P, _I64, _P, _I64, _P]),
    "sof_set_tets_async": (_I, [_P, _I64, _P, _I64, _P]),
    "sof_set_cache_budget": (_I, [_P, _I64]),
    "sof_precompute_view": (_I, [_P, _I, _P]),
    "sof_tile_binding": (_I, [_P, _I, _I, _P, _P]),
    "sof_schedule_points": (_I, [_P, _I, _I64, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "sof_view_opacity": (_I, [_P, _I, _I64, _P, _I, _I, _I, _P, _P, _P, _P]),
    "sof_classify_points": (_I, [_P, _I64, _P, _I, _I, _P, _P]),
    "sof_value_at": (_I, [_P, _I64, _P, _I, _I, _P, _P]),
    "sof_label_grid": (_I, [_P, _I64, _P, _I, _I, _I, _P, _P]),
    "sof_label_views_dev": (_I, [_P, _I, _I, _I64, _P, _I, _I, _I, _P, _P, _P]),
    "sof_classify_views_dev": (_I, [_P, _I, _I, _I64, _P, _I, _I, _P, _P]),
    "sof_marching_tets": (_I, [_P, _P, _P, _P]),
    "sof_refine": (_I, [_P, _I64, _P, _P, _I, _I, _I, _P]),
    "sof_assemble": (_I, [_P, _I64, _P, _I64, _P, _D, _D, _P, _P]),
    "sof_assemble_residuals": (_I, [_P, _I64, _P, _P, _I64, _P, _D, _D, _P, _P]),
    "sof_tetrahedralize": (_I, [_P, _I64, _P, ctypes.POINTER(_I64)]),
    "sof_extract": (_I, [_P, ctypes.POINTER(ExtractOpts), ctypes.POINTER(ExtractStats)]),
    "sof_extract_opts_default": (None, [ctypes.POINTER(ExtractOpts)]),
    "sof_result_count": (_I64, [_P, _I]),
    "sof_copy_result": (_I, [_P, _I, _P]),
    "sof_render_view": (_I, [_P, _I, _I, _I, _P, _P, _P, _P, _P]),
    "sof_render_normals": (_I, [_P, _I, _P, _P]),
    "sof_set_render_pool": (_I, [_P, _I64]),
    "sof_render_counts": (_I, [_P, _I, _P]),
    "sof_comm_unique_id": (_I, [_P]),
    "sof_comm_init": (_I, [_P, _P, _I, _I]),
    "sof_comm_init_local": (_I, [_P, _I]),
    "sof_comm_info": (_I, [_P, _P, _P]),
    "sof_comm_destroy": (_I, [_P]),
    "sof_normal_from_depth": (_I, [_P, _I, _P, _P, _P]),
    "sof_gaussian_normals": (_I, [_P, ctypes.c_int64, _P, _P, _P, _P, _P]),
    "sof_seed_points": (_I, [_P, _I, _I, _D, _P]),
    "sof_load_scene_ply": (_I, [_P, ctypes.c_char_p, _D, _P]),
    "sof_get_scene": (_I, [_P, _P, _P, _P, _P, _P]),
    "sof_write_scene_ply": (_I, [_P, ctypes.c_char_p]),
    "sof_validate_tets_dev": (_I, [_P, _I64, _P, _I64]),
    "sof_event_record": (_I, [_P, _I]),
    "sof_event_elapsed": (_I, [_P, _I, _I, ctypes.POINTER(ctypes.c_float)]),
    "sof_sync": (_I, [_P]),
    "sof_host_register": (_I, [_P, ctypes.c_size_t]),
    "sof_host_unregister": (_I, [_P]),
    "sof_fp64_peak": (_I, [_P, ctypes.POINTER(_D)]),
    "sof_set_eval_path": (_I, [_P, _I]),
    "sof_set_staging": (_I, [_P, _I]),
    "sof_distortion_loss": (_I, [_P, _I64, _P, _P, _P, _D, _D, _I, _P, _P, _P]),
    "sof_extent_loss": (_I, [_P, _I64, _P, _P, _P, _P, _P, _P, _D, _D, _P, _P, _P, _P, _P, _P]),
    "sof_depth_normal_loss": (_I, [_P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "sof_opacity_supervision_loss": (_I, [_P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "sof_normal_smoothness_loss": (_I, [_P, _I, _I, _P, _P, _P, _I, _P, _P, _P]),
    "sof_l1_rgb_loss": (_I, [_P, _I64, _P, _P, _P]),
    "sof_tets_vertices_dev": (_I, [_P, ctypes.POINTER(_P), ctypes.POINTER(_I64)]),
    "sof_shard_ext_rank_dev": (_I, [_P, _I64, _P, _I, _I, _P]),
    "sof_shard_mask_min_dev": (_I, [_P, _I64, _P, _I, _P]),
    "sof_shard_finalize_dev": (_I, [_P, _I64, _P, _P, _I]),
    "sof_march_resident": (_I, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "sof_march_range_resident": (_I, [_P, _I64, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "sof_march_result_copy_dev": (_I, [_P, _P, _P]),
    "sof_march_merge_dev": (_I, [_P, _I, _P, _P, _P, _P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "sof_refine_phase_dev": (_I, [_P, _I, _P, _I, _I, _I, _I, _P]),
    "sof_assemble_resident": (_I, [_P, _D, _D, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
}

_lib = None


def declared_symbols() -> list[str]:
    """Function names declared in include/sof_cuda.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+\**(sof_\w+)\s*\(", text, re.M)))


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                          "(this package has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if os.environ.get("SOF_LIB_PATH"):  # an older build loaded for A/B timing
                continue
            raise
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
