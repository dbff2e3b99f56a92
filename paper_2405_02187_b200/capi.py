"""ctypes mirror of include/csf_b200.h (the C-ABI boundary).

The structs below follow the header field for field; the loader fails loudly
when the sm_100a library has not been built — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["CSF_B200_LIB"]) if os.environ.get("CSF_B200_LIB") else _HERE / "_build" / "libcsf_b200.so"

CSF_OK, CSF_EINVAL, CSF_EDOMAIN, CSF_ERUNTIME, CSF_ECUDA, CSF_ENOMEM = 0, 1, 2, 3, 4, 5
CSF_MAX_DIRECTIONS = 64
CSF_MAX_PAIRS = 64
SOLVER_LINEARIZED, SOLVER_NEWTON, SOLVER_GRADIENT_DESCENT, SOLVER_CONJUGATE_GRADIENT = 0, 1, 2, 3
OBJECTIVE_FINAL_TRANSLATION_ERROR, OBJECTIVE_TRAJECTORY_ERROR = 0, 1

# Every symbol include/csf_b200.h declares (checked by tests/test_capi_exports.py).
EXPORTS = (
    "csf_default_intrinsics", "csf_default_volume_params", "csf_default_raycast_cfg", "csf_default_icp_cfg",
    "csf_ctx_create", "csf_ctx_destroy", "csf_last_error", "csf_ctx_synchronize", "csf_ctx_launch_count",
    "csf_ctx_stream", "csf_ctx_profile", "csf_ctx_profile_read", "csf_bilateral_filter", "csf_downsample_depth", "csf_measure_surface",
    "csf_volume_create_dense", "csf_volume_create_hashed", "csf_volume_destroy", "csf_volume_upload",
    "csf_volume_download", "csf_volume_block_count", "csf_volume_save", "csf_volume_load", "csf_sample_tsdf",
    "csf_sample_gradient", "csf_measured_tsdf", "csf_volume_download_hash", "csf_surface_update",
    "csf_surface_update_lifted", "csf_measured_tsdf_lifted", "csf_volume_info",
    "csf_comm_unique_id", "csf_ctx_attach_comm", "csf_gather_columns",
    "csf_raycast", "csf_track_frame", "csf_track_frame_traced", "csf_icp_energy_derivs", "csf_view_scores", "csf_associate",
    "csf_linearized_step", "csf_pairwise_sum", "csf_pipeline_create", "csf_pipeline_destroy", "csf_pipeline_upload",
    "csf_pipeline_run", "csf_pipeline_result", "csf_pipeline_hessian", "csf_pipeline_run_host", "csf_pipeline_run_host_rgbd", "csf_pipeline_download_rgb", "csf_pipeline_volume", "csf_pipeline_set_graph",
    "csf_synth_workload", "csf_default_reloc_cfg", "csf_reloc_create", "csf_reloc_destroy", "csf_reloc_info",
    "csf_reloc_energy", "csf_relocalize", "csf_depth_cloud", "csf_eval_nn_error", "csf_io_last_error",
    "csf_write_depth_png16", "csf_read_depth_png16", "csf_read_intrinsics", "csf_write_intrinsics",
    "csf_read_trajectory", "csf_write_trajectory", "csf_default_surfel_cfg", "csf_surfels_create",
    "csf_surfels_destroy", "csf_surfels_clear", "csf_surfels_count", "csf_surfels_download", "csf_surfels_upload", "csf_render_index_map",
    "csf_associate_surfels", "csf_update_surfels", "csf_update_surfels_real", "csf_predict_maps", "csf_sample_confidence",
)
RELOC_GRADIENT_DESCENT, RELOC_NEWTON = 0, 1


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int), ("height", C.c_int), ("depth_scale", C.c_double)]


class VolumeParams(C.Structure):
    _fields_ = [("dims", C.c_int * 3), ("voxel_size", C.c_double), ("origin", C.c_double * 3),
                ("mu", C.c_double), ("weight_cap", C.c_double)]


class HashParams(C.Structure):
    _fields_ = [("voxel_size", C.c_double), ("origin", C.c_double * 3), ("mu", C.c_double),
                ("weight_cap", C.c_double), ("bucket_bits", C.c_int), ("max_blocks", C.c_int)]


class RaycastCfg(C.Structure):
    _fields_ = [("near_clip", C.c_double), ("far_clip", C.c_double), ("step_fraction", C.c_double)]


class IcpCfg(C.Structure):
    _fields_ = [("solver", C.c_int), ("d_max", C.c_double), ("theta_max_deg", C.c_double), ("levels", C.c_int),
                ("level_iterations", C.c_int * 3), ("level_pixel_stride", C.c_int * 3),
                ("step_tolerance", C.c_double), ("levenberg_lambda0", C.c_double), ("ncg_restart", C.c_int),
                ("h", C.c_double)]


class TrackResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("correspondences", C.c_int), ("pad", C.c_int),
                ("final_loss", C.c_double)]


class RelocCfg(C.Structure):
    _fields_ = [("switch_relative", C.c_double), ("switch_absolute", C.c_double), ("max_iterations", C.c_int),
                ("ls_max_backtracks", C.c_int), ("step_tolerance", C.c_double), ("ls_initial_step", C.c_double),
                ("ls_shrink", C.c_double), ("ls_sufficient_decrease", C.c_double), ("h", C.c_double),
                ("max_step", C.c_double), ("min_overlap_ratio", C.c_double)]


class RelocResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("final_loss", C.c_double)]


class SurfelCfg(C.Structure):
    _fields_ = [("depth", C.c_double), ("normal_deg", C.c_double), ("distance", C.c_double), ("sigma", C.c_double),
                ("one_to_many", C.c_int)]


class PipelineCfg(C.Structure):
    _fields_ = [("hashed", C.c_int), ("dense", VolumeParams), ("hash", HashParams), ("k", Intrinsics),
                ("icp", IcpCfg), ("rc", RaycastCfg), ("h", C.c_double), ("n_dirs", C.c_int),
                ("dirs", C.c_int * CSF_MAX_DIRECTIONS), ("objective", C.c_int), ("max_frames", C.c_int),
                ("order", C.c_int), ("n_pairs", C.c_int), ("pair_i", C.c_int * CSF_MAX_PAIRS),
                ("pair_j", C.c_int * CSF_MAX_PAIRS), ("keyframe_interval", C.c_int)]


def load_library(path: os.PathLike | str | None = None) -> C.CDLL:
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"csf_b200: CUDA library {p} is missing — run __graft_entry__.build() "
            "(make -C paper_2405_02187_b200); there is no CPU fallback")
    lib = C.CDLL(str(p))
    vp, ip, dp, fp = C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_float)
    i32p, u64p = C.POINTER(C.c_int32), C.POINTER(C.c_uint64)
    sig = {
        "csf_ctx_create": (ip, [ip, C.POINTER(vp)]),
        "csf_ctx_destroy": (ip, [vp]),
        "csf_last_error": (C.c_char_p, [vp]),
        "csf_ctx_synchronize": (ip, [vp]),
        "csf_ctx_launch_count": (ip, [vp, C.POINTER(C.c_ulonglong)]),
        "csf_ctx_stream": (vp, [vp]),
        "csf_ctx_profile": (ip, [vp, ip]),
        "csf_ctx_profile_read": (ip, [vp, ip, C.c_char_p, dp, C.POINTER(C.c_longlong), C.POINTER(C.c_int)]),
        "csf_bilateral_filter": (ip, [vp, dp, ip, ip, C.c_double, C.c_double, ip, dp]),
        "csf_downsample_depth": (ip, [vp, dp, ip, ip, C.c_double, dp]),
        "csf_measure_surface": (ip, [vp, dp, ip, ip, dp, ip, dp, dp]),
        "csf_volume_create_dense": (ip, [vp, C.POINTER(VolumeParams), ip, C.POINTER(vp)]),
        "csf_volume_create_hashed": (ip, [vp, C.POINTER(HashParams), ip, C.POINTER(vp)]),
        "csf_volume_destroy": (ip, [vp]),
        "csf_volume_upload": (ip, [vp, dp, dp]),
        "csf_volume_download": (ip, [vp, dp, dp]),
        "csf_volume_block_count": (ip, [vp, C.POINTER(C.c_int)]),
        "csf_volume_save": (ip, [vp, C.c_char_p]),
        "csf_sample_tsdf": (ip, [vp, dp, ip, dp, i32p]),
        "csf_sample_gradient": (ip, [vp, dp, ip, dp, i32p]),
        "csf_measured_tsdf": (ip, [vp, dp, ip, ip, dp, dp, C.c_double, dp, dp, ip, ip, dp, i32p]),
        "csf_measured_tsdf_lifted": (ip, [vp, dp, ip, ip, dp, dp, C.c_double, dp, dp, ip, ip, dp, i32p]),
        "csf_volume_load": (ip, [vp, C.c_char_p, ip, C.POINTER(vp)]),
        "csf_volume_download_hash": (ip, [vp, i32p, u64p, i32p, i32p]),
        "csf_surface_update": (ip, [vp, dp, ip, ip, dp, dp, C.POINTER(C.c_int)]),
        "csf_surface_update_lifted": (ip, [vp, dp, ip, ip, dp, dp, C.POINTER(C.c_int)]),
        "csf_volume_info": (ip, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
        "csf_comm_unique_id": (ip, [C.c_char_p]),
        "csf_ctx_attach_comm": (ip, [vp, ip, ip, C.c_char_p]),
        "csf_gather_columns": (ip, [vp, dp, C.POINTER(C.c_int), dp]),
        "csf_raycast": (ip, [vp, dp, dp, ip, ip, C.POINTER(RaycastCfg), dp, dp]),
        "csf_track_frame": (ip, [vp, dp, ip, ip, dp, C.POINTER(Intrinsics), C.POINTER(IcpCfg), dp,
                                 C.POINTER(TrackResult)]),
        "csf_icp_energy_derivs": (ip, [vp, dp, ip, dp, dp, C.c_double, dp, dp, dp]),
        "csf_track_frame_traced": (ip, [vp, dp, ip, ip, dp, C.POINTER(Intrinsics), C.POINTER(IcpCfg), dp,
                                        C.POINTER(TrackResult), dp, ip, C.POINTER(C.c_int)]),
        "csf_associate": (ip, [vp, dp, dp, dp, dp, ip, ip, dp, dp, C.POINTER(Intrinsics), C.POINTER(IcpCfg), ip, dp,
                               C.POINTER(C.c_int)]),
        "csf_linearized_step": (ip, [vp, dp, ip, dp, dp]),
        "csf_pairwise_sum": (ip, [vp, dp, ip, ip, dp]),
        "csf_view_scores": (ip, [vp, dp, ip, C.POINTER(Intrinsics), C.c_double, C.c_double, C.c_double, dp, dp]),
        "csf_pipeline_create": (ip, [vp, C.POINTER(PipelineCfg), C.POINTER(vp)]),
        "csf_pipeline_destroy": (ip, [vp]),
        "csf_pipeline_upload": (ip, [vp, fp, dp, ip]),
        "csf_pipeline_run": (ip, [vp, ip]),
        "csf_pipeline_result": (ip, [vp, dp, dp, dp, i32p]),
        "csf_pipeline_hessian": (ip, [vp, dp, dp, dp, dp, dp, i32p]),
        "csf_pipeline_run_host": (ip, [vp, fp, dp, ip, dp, dp]),
        "csf_pipeline_run_host_rgbd": (ip, [vp, fp, C.POINTER(C.c_ubyte), dp, ip, dp, dp]),
        "csf_pipeline_download_rgb": (ip, [vp, ip, C.POINTER(C.c_ubyte)]),
        "csf_pipeline_volume": (ip, [vp, C.POINTER(vp)]),
        "csf_pipeline_set_graph": (ip, [vp, ip]),
        "csf_synth_workload": (ip, [vp, ip, ip, ip, ip, fp, dp, C.POINTER(Intrinsics)]),
        "csf_default_intrinsics": (None, [C.POINTER(Intrinsics)]),
        "csf_default_volume_params": (None, [C.POINTER(VolumeParams)]),
        "csf_default_raycast_cfg": (None, [C.POINTER(RaycastCfg)]),
        "csf_default_icp_cfg": (None, [C.POINTER(IcpCfg)]),
        "csf_default_reloc_cfg": (None, [C.POINTER(RelocCfg)]),
        "csf_reloc_create": (ip, [vp, dp, ip, ip, C.POINTER(Intrinsics), C.POINTER(vp)]),
        "csf_reloc_destroy": (ip, [vp]),
        "csf_reloc_info": (ip, [vp, C.POINTER(C.c_int), dp, dp, dp]),
        "csf_reloc_energy": (ip, [vp, dp, ip, C.c_double, dp, dp, dp, C.POINTER(C.c_longlong)]),
        "csf_relocalize": (ip, [vp, dp, ip, C.POINTER(RelocCfg), dp, C.POINTER(RelocResult), dp, dp]),
        "csf_depth_cloud": (ip, [vp, dp, ip, ip, C.POINTER(Intrinsics), dp, ip, dp, C.POINTER(C.c_int)]),
        "csf_eval_nn_error": (ip, [vp, dp, dp, ip, dp, ip, dp, i32p]),
        "csf_io_last_error": (C.c_char_p, []),
        "csf_default_surfel_cfg": (None, [C.POINTER(SurfelCfg)]),
        "csf_surfels_create": (ip, [vp, ip, C.POINTER(vp)]),
        "csf_surfels_destroy": (ip, [vp]),
        "csf_surfels_count": (ip, [vp, C.POINTER(C.c_int)]),
        "csf_surfels_clear": (ip, [vp]),
        "csf_surfels_download": (ip, [vp, dp, dp, dp, dp, i32p]),
        "csf_surfels_upload": (ip, [vp, ip, dp, dp, dp, dp, i32p]),
        "csf_render_index_map": (ip, [vp, dp, C.POINTER(Intrinsics), C.POINTER(C.c_uint32), i32p, C.POINTER(C.c_int)]),
        "csf_associate_surfels": (ip, [vp, dp, ip, ip, dp, C.POINTER(Intrinsics), C.POINTER(SurfelCfg), i32p, i32p, dp,
                                       ip, C.POINTER(C.c_int)]),
        "csf_update_surfels": (ip, [vp, dp, ip, ip, dp, C.POINTER(Intrinsics), ip, C.POINTER(SurfelCfg),
                                    C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "csf_update_surfels_real": (ip, [vp, dp, ip, ip, dp, C.POINTER(Intrinsics), ip, C.POINTER(SurfelCfg),
                                         C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "csf_predict_maps": (ip, [vp, dp, C.POINTER(Intrinsics), dp, dp]),
        "csf_sample_confidence": (C.c_double, [C.POINTER(Intrinsics), ip, ip]),
        "csf_write_depth_png16": (ip, [C.c_char_p, dp, ip, ip, C.c_double]),
        "csf_read_depth_png16": (ip, [C.c_char_p, C.c_double, dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "csf_read_intrinsics": (ip, [C.c_char_p, C.POINTER(Intrinsics)]),
        "csf_write_intrinsics": (ip, [C.c_char_p, C.POINTER(Intrinsics)]),
        "csf_read_trajectory": (ip, [C.c_char_p, dp, dp, ip, C.POINTER(C.c_int)]),
        "csf_write_trajectory": (ip, [C.c_char_p, dp, dp, ip]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
