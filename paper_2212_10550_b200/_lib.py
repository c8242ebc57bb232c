"""ctypes binding of libarfx.so (include/arfx.h). Loads the in-tree library and fails
loudly when it is missing -- there is no Python/CPU fallback for any compute call."""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libarfx.so"

MAX_BONES = 32
MAX_ROOTS = 8

c_double_p = C.POINTER(C.c_double)
c_float_p = C.POINTER(C.c_float)
c_int32_p = C.POINTER(C.c_int32)
c_uint8_p = C.POINTER(C.c_uint8)
c_uint64_p = C.POINTER(C.c_uint64)


class ArfxSkeleton(C.Structure):
    _fields_ = [("n_bones", C.c_int), ("parent", C.c_int * MAX_BONES),
                ("head", (C.c_double * 3) * MAX_BONES), ("tail", (C.c_double * 3) * MAX_BONES),
                ("radius", C.c_double * MAX_BONES)]


class ArfxGridConfig(C.Structure):
    _fields_ = [("levels", C.c_int), ("features_per_level", C.c_int), ("table_size_log2", C.c_int),
                ("base_resolution", C.c_int), ("max_resolution", C.c_int),
                ("box_lo", C.c_double * 3), ("box_hi", C.c_double * 3)]


class ArfxMlpConfig(C.Structure):
    _fields_ = [("input_dim", C.c_int), ("hidden_dim", C.c_int), ("hidden_layers", C.c_int),
                ("output_dim", C.c_int)]


class ArfxCamera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int), ("height", C.c_int), ("extrinsic", C.c_double * 12)]


class ArfxOccConfig(C.Structure):
    _fields_ = [("resolution", C.c_int), ("alpha_threshold", C.c_double), ("dilation", C.c_int),
                ("decay", C.c_double), ("update_interval", C.c_int)]


class ArfxRenderOptions(C.Structure):
    _fields_ = [("samples_per_ray", C.c_int), ("stratified", C.c_int),
                ("epsilon_terminate", C.c_double), ("seed", C.c_uint64), ("frame_id", C.c_uint64)]


class ArfxInverseOptions(C.Structure):
    _fields_ = [("max_iterations", C.c_int), ("tolerance", C.c_double), ("dedup_radius", C.c_double)]


class ArfxCounters(C.Structure):
    _fields_ = [("posed_queries", C.c_uint64), ("canonical_queries", C.c_uint64)]


class ArfxModelDesc(C.Structure):
    _fields_ = [("skeleton", ArfxSkeleton), ("grid", ArfxGridConfig), ("mlp", ArfxMlpConfig),
                ("skin_res", C.c_int * 3), ("skin_lo", C.c_double * 3), ("skin_hi", C.c_double * 3),
                ("canonical_lo", C.c_double * 3), ("canonical_hi", C.c_double * 3),
                ("normalized_lo", C.c_double * 3), ("normalized_hi", C.c_double * 3),
                ("inverse", ArfxInverseOptions), ("n_grid_params", C.c_size_t),
                ("n_mlp_params", C.c_size_t), ("n_skin_weights", C.c_size_t)]


class ArfxLossConfig(C.Structure):
    _fields_ = [("w_rgb", C.c_double), ("w_alpha", C.c_double), ("w_hard", C.c_double), ("w_density", C.c_double),
                ("huber_delta", C.c_double), ("gt_width", C.c_int64), ("gt_height", C.c_int64)]


class ArfxAdamConfig(C.Structure):
    _fields_ = [("lr_grid", C.c_double), ("lr_mlp", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("total_steps", C.c_int64), ("final_lr_factor", C.c_double)]


class ArfxFigure(C.Structure):
    _fields_ = [("skeleton", ArfxSkeleton), ("color", (C.c_double * 3) * MAX_BONES),
                ("amplitude", C.c_double * MAX_BONES), ("softness", C.c_double)]


H = C.c_void_p  # opaque handles
P = C.c_void_p  # raw pointers / streams

# name -> (restype, argtypes)
_PROTOS = {
    "arfx_last_error": (C.c_char_p, []),
    "arfx_version": (C.c_char_p, []),
    "arfx_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "arfx_set_device": (C.c_int, [C.c_int]),
    "arfx_level_resolutions": (C.c_int, [C.POINTER(ArfxGridConfig), c_int32_p]),
    "arfx_model_sizes": (C.c_int, [C.POINTER(ArfxSkeleton), C.POINTER(ArfxGridConfig), C.POINTER(ArfxMlpConfig),
                                   c_int32_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "arfx_pose_from_joint_rotations": (C.c_int, [C.POINTER(ArfxSkeleton), c_double_p, c_double_p, c_double_p]),
    "arfx_camera_look_at": (C.c_int, [c_double_p, c_double_p, c_double_p, C.c_double, C.c_int, C.c_int,
                                      C.POINTER(ArfxCamera)]),
    "arfx_pose_context": (C.c_int, [C.POINTER(ArfxSkeleton), c_double_p, c_double_p, C.c_double, c_double_p,
                                    c_double_p, c_double_p, c_double_p, c_double_p]),
    "arfx_build_model": (C.c_int, [C.POINTER(ArfxSkeleton), C.POINTER(ArfxGridConfig), C.POINTER(ArfxMlpConfig),
                                   c_int32_p, C.c_uint64, C.POINTER(H)]),
    "arfx_model_create": (C.c_int, [C.POINTER(ArfxModelDesc), c_float_p, c_float_p, c_double_p, C.POINTER(H)]),
    "arfx_model_destroy": (C.c_int, [H]),
    "arfx_model_describe": (C.c_int, [H, C.POINTER(ArfxModelDesc)]),
    "arfx_model_get_params": (C.c_int, [H, c_float_p, c_float_p, c_double_p]),
    "arfx_model_set_params": (C.c_int, [H, c_float_p, c_float_p]),
    "arfx_model_set_mlp_mode": (C.c_int, [H, C.c_int]),
    "arfx_model_set_backward_mode": (C.c_int, [H, C.c_int]),
    "arfx_model_set_deterministic": (C.c_int, [H, C.c_int]),
    "arfx_model_flush_grads": (C.c_int, [H, C.c_void_p]),
    "arfx_model_set_param_fence": (C.c_int, [H, C.c_void_p]),
    "arfx_model_zero_grad": (C.c_int, [H, P]),
    "arfx_model_get_grads": (C.c_int, [H, c_float_p, c_float_p]),
    "arfx_model_device_arrays": (C.c_int, [H, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P)]),
    "arfx_pose_create": (C.c_int, [H, c_double_p, c_double_p, C.POINTER(H)]),
    "arfx_pose_update": (C.c_int, [H, c_double_p, c_double_p, P]),
    "arfx_pose_update_async": (C.c_int, [H, c_double_p, c_double_p, P]),
    "arfx_render_model_async": (C.c_int, [H, H, C.POINTER(ArfxCamera), H, C.POINTER(ArfxRenderOptions), C.c_int,
                                          C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                          C.POINTER(C.c_uint64), P]),
    "arfx_render_wait": (C.c_int, [H]),
    "arfx_pose_destroy": (C.c_int, [H]),
    "arfx_occ_create": (C.c_int, [c_double_p, c_double_p, C.POINTER(ArfxOccConfig), C.POINTER(H)]),
    "arfx_occ_destroy": (C.c_int, [H]),
    "arfx_occ_info": (C.c_int, [H, c_int32_p, c_double_p, c_double_p, c_double_p, c_int32_p]),
    "arfx_occ_download": (C.c_int, [H, c_float_p, c_uint8_p]),
    "arfx_occ_upload": (C.c_int, [H, c_float_p, c_uint8_p]),
    "arfx_occ_rebuild_mask": (C.c_int, [H, P]),
    "arfx_build_inference_grid": (C.c_int, [H, H, H, C.POINTER(ArfxCounters), P]),
    "arfx_build_inference_grid_device": (C.c_int, [H, H, H, P, P]),
    "arfx_build_inference_grid_shard_device": (C.c_int, [H, H, H, C.c_int, C.c_int, P, P]),
    "arfx_occ_device_arrays": (C.c_int, [H, C.POINTER(P), C.POINTER(P)]),
    "arfx_occ_rebuild_mask_async": (C.c_int, [H, P]),
    "arfx_occ_rebuild_mask_shards_async": (C.c_int, [H, C.c_int, P]),
    "arfx_update_training_grid_device": (C.c_int, [H, C.POINTER(H), C.c_int, C.c_double, C.c_uint64,
                                                   C.c_uint64, H, P, P]),
    "arfx_occ_is_occupied": (C.c_int, [H, c_double_p, C.c_int64, c_uint8_p]),
    "arfx_stats_enable": (C.c_int, [H, C.c_int]),
    "arfx_stats_read": (C.c_int, [H, c_uint64_p]),
    "arfx_pipe_peaks": (C.c_int, [c_double_p, c_double_p]),
    "arfx_profile_enable": (C.c_int, [H, C.c_int]),
    "arfx_profile_read": (C.c_int, [H, C.c_int, C.c_char_p, c_double_p, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "arfx_update_training_grid": (C.c_int, [H, C.POINTER(H), C.c_int, C.c_double, C.c_uint64, C.c_uint64, H,
                                            C.POINTER(ArfxCounters), P]),
    "arfx_render_model": (C.c_int, [H, H, C.POINTER(ArfxCamera), H, C.POINTER(ArfxRenderOptions), C.c_int, C.c_int,
                                    c_float_p, c_float_p, C.POINTER(ArfxCounters), P]),
    "arfx_render_model_device": (C.c_int, [H, H, C.POINTER(ArfxCamera), H, C.POINTER(ArfxRenderOptions), C.c_int,
                                           C.c_int, P, P, P, P]),
    "arfx_render_trace": (C.c_int, [H, C.c_int64, C.POINTER(C.c_int64), c_int32_p, c_int32_p, c_uint8_p, c_float_p,
                                    c_float_p, c_double_p, c_double_p]),
    "arfx_skinning_weights": (C.c_int, [H, c_double_p, C.c_int64, c_double_p]),
    "arfx_inverse_lbs": (C.c_int, [H, c_double_p, c_double_p, C.c_double, c_double_p, C.c_int64, c_int32_p,
                                   c_double_p, c_double_p]),
    "arfx_inverse_lbs_device": (C.c_int, [H, H, P, C.c_int64, P, P, P, P]),
    "arfx_pose_create_context": (C.c_int, [H, c_double_p, c_double_p, C.c_double, C.POINTER(H)]),
    "arfx_hash_encode": (C.c_int, [H, c_double_p, C.c_int64, c_float_p]),
    "arfx_field_query": (C.c_int, [H, c_double_p, C.c_int64, c_float_p, c_float_p]),
    "arfx_posed_query": (C.c_int, [H, H, c_double_p, C.c_int64, c_float_p, c_float_p, c_double_p, c_uint8_p,
                                   C.POINTER(ArfxCounters)]),
    "arfx_composite": (C.c_int, [C.c_int, c_int32_p, c_double_p, c_double_p, c_uint8_p, c_float_p, c_float_p,
                                 C.c_double, c_double_p, c_double_p, c_int32_p]),
    "arfx_composite_backward": (C.c_int, [C.c_int, c_int32_p, c_double_p, c_double_p, c_uint8_p, c_float_p,
                                          c_float_p, C.c_double, c_double_p, c_double_p, c_double_p, c_double_p]),
    "arfx_field_query_backward": (C.c_int, [H, c_double_p, C.c_int64, c_float_p, c_float_p]),
    "arfx_train_fwd_bwd": (C.c_int, [H, H, C.POINTER(ArfxCamera), H, C.POINTER(ArfxRenderOptions), C.c_int64,
                                     c_int32_p, c_int32_p, c_float_p, c_float_p, c_float_p, c_float_p,
                                     C.POINTER(ArfxCounters), P]),
    "arfx_losses": (C.c_int, [C.c_int64, c_float_p, c_float_p, c_float_p, c_float_p, C.POINTER(ArfxLossConfig),
                              c_double_p, c_float_p, c_float_p]),
    "arfx_train_step": (C.c_int, [H, H, C.POINTER(ArfxCamera), H, C.POINTER(ArfxRenderOptions), C.c_int64,
                                  c_int32_p, c_int32_p, c_float_p, c_float_p, C.POINTER(ArfxLossConfig), c_double_p,
                                  c_float_p, c_float_p, C.POINTER(ArfxCounters), P]),
    "arfx_train_step_device": (C.c_int, [H, H, C.POINTER(ArfxCamera), H, C.POINTER(ArfxRenderOptions), C.c_int64,
                                         P, P, P, P, C.POINTER(ArfxLossConfig), P, P, P, P]),
    "arfx_density_step": (C.c_int, [H, H, H, C.c_int64, C.c_uint64, C.c_uint64, C.POINTER(ArfxLossConfig),
                                    c_double_p, P]),
    "arfx_density_step_device": (C.c_int, [H, H, H, C.c_int64, C.c_uint64, C.c_uint64,
                                           C.POINTER(ArfxLossConfig), P, P]),
    "arfx_train_density_step_device": (C.c_int, [H, H, C.POINTER(ArfxCamera), H, C.POINTER(ArfxRenderOptions),
                                                 C.c_int64, P, P, P, P, C.POINTER(ArfxLossConfig), P, C.c_int64,
                                                 C.c_uint64, C.c_uint64, P, P]),
    "arfx_train_rays_device": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, C.c_int, C.c_int, P, P,
                                         P]),
    "arfx_train_forward_device": (C.c_int, [H, H, C.POINTER(ArfxCamera), H, C.POINTER(ArfxRenderOptions), C.c_int64,
                                            P, P, C.c_int, P]),
    "arfx_train_backward_device": (C.c_int, [H, H, H, C.POINTER(ArfxRenderOptions), C.c_int64, P, P, P, P,
                                             C.POINTER(ArfxLossConfig), P, C.c_int, C.c_int64, C.c_uint64, C.c_uint64,
                                             P, P]),
    "arfx_adam_step": (C.c_int, [H, C.POINTER(ArfxAdamConfig), C.c_int64, C.c_int64, C.c_int64, P]),
    "arfx_adam_step_guarded": (C.c_int, [H, C.POINTER(ArfxAdamConfig), C.c_int64, C.c_int64, C.c_int64, P, C.c_int,
                                         P, P]),
    "arfx_model_flat": (C.c_int, [H, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P),
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "arfx_model_get_adam": (C.c_int, [H, c_float_p, c_float_p]),
    "arfx_model_set_adam": (C.c_int, [H, c_float_p, c_float_p]),
    "arfx_occ_create_raw": (C.c_int, [c_double_p, c_double_p, C.c_int, C.c_double, C.c_int, C.POINTER(H)]),
    "arfx_checkpoint_save": (C.c_int, [C.c_char_p, H, H, C.c_int64, C.c_int]),
    "arfx_checkpoint_load": (C.c_int, [C.c_char_p, C.POINTER(H), C.POINTER(H), C.POINTER(C.c_int64)]),
    "arfx_pose_copy": (C.c_int, [H, H, P]),
    "arfx_frame_graph_create": (C.c_int, [H, H, C.POINTER(ArfxCamera), H, C.POINTER(ArfxRenderOptions), C.c_int,
                                          C.c_int, C.c_int, P, P, P, P, C.POINTER(H)]),
    "arfx_frame_graph_create_pipelined": (C.c_int, [H, H, H, H, H, C.POINTER(ArfxCamera), C.POINTER(ArfxRenderOptions),
                                                    C.c_int, C.c_int, P, P, P, P, C.POINTER(H)]),
    "arfx_render_model_pipelined_async": (C.c_int, [H, H, H, H, H, C.POINTER(ArfxCamera), C.POINTER(ArfxRenderOptions),
                                                    C.c_int, C.c_int, P, P, P, P]),
    "arfx_frame_graph_launch": (C.c_int, [H, P]),
    "arfx_frame_graph_destroy": (C.c_int, [H]),
    "arfx_figure_query": (C.c_int, [C.POINTER(ArfxFigure), c_double_p, c_double_p, C.c_int64, c_double_p,
                                    c_double_p]),
    "arfx_figure_render": (C.c_int, [C.POINTER(ArfxFigure), c_double_p, c_double_p, c_double_p, c_double_p,
                                     C.POINTER(ArfxCamera), C.POINTER(ArfxRenderOptions), c_float_p, c_float_p,
                                     c_uint8_p, P]),
    "arfx_figure_render_rays_device": (C.c_int, [C.POINTER(ArfxFigure), c_double_p, c_double_p, c_double_p,
                                                 c_double_p, C.POINTER(ArfxCamera), C.POINTER(ArfxRenderOptions),
                                                 C.c_int64, P, P, P, P, P, P]),
}

STATUS_NAMES = {1: "invalid_argument", 2: "DataError", 3: "NumericError", 4: "domain_error",
                5: "runtime_error", 6: "no CUDA device"}


class ArfxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{STATUS_NAMES.get(code, code)}] {msg}")
        self.code = code


class InvalidArgument(ArfxError, ValueError):
    pass


class DomainError(ArfxError, ValueError):
    pass


class NumericError(ArfxError):
    pass


class DataError(ArfxError):
    pass


class NoDevice(ArfxError):
    pass


_EXC = {1: InvalidArgument, 2: DataError, 3: NumericError, 4: DomainError, 6: NoDevice}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"libarfx.so not built at {LIB_PATH}; run `python -m paper_2212_10550_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _PROTOS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(code: int):
    if code != 0:
        msg = lib().arfx_last_error().decode(errors="replace")
        raise _EXC.get(code, ArfxError)(code, msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


def ptr(a: np.ndarray | None, ctype):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays passed to libarfx must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


def exported_symbols() -> list[str]:
    return list(_PROTOS)
