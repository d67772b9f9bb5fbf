"""ctypes binding of the C-ABI in include/gb_raster.h.

Loads the in-tree ``libgb_raster.so`` (built by ``__graft_entry__.build()`` /
``make -C paper_2412_12734_b200/csrc``).  There is no fallback: if the
library is missing, importing this module raises ImportError naming the
build command, so a GPU run can never silently degrade to a CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GB_LIB_PATH") or os.path.join(_HERE, "libgb_raster.so")  # override: debug builds only

GB_OK = 0
GB_INVALID_ARGUMENT = 1
GB_MISMATCH = 2
GB_CUDA_ERROR = 3
GB_OOM = 4
GB_NONFINITE = 5
ADAM_FLAG_CLEAR = 0x7FFFFFFFFFFFFFFF  # GB_ADAM_FLAG_CLEAR
ADAM_FLAG_VETO = 7 << 48  # GB_ADAM_FLAG_VETO
GB_NOT_SUPPORTED = 6
GB_IO_ERROR = 7
GB_NCCL_ERROR = 8
COMM_ID_BYTES = 128

MODE_ORTHO = 0
MODE_PINHOLE = 1

KERNEL_NAMES = ("project", "scan", "duplicate", "sort", "ranges", "forward", "backward", "chain", "loss", "adam", "fused",
                "collective")


class GridConfig(C.Structure):
    _fields_ = [("n", C.c_int32), ("_pad", C.c_int32), ("sigma", C.c_double)]


class Splats(C.Structure):
    _fields_ = [
        ("count", C.c_int64),
        ("grid", GridConfig),
        ("position", C.c_void_p),
        ("depth_key", C.c_void_p),
        ("theta", C.c_void_p),
        ("quat", C.c_void_p),
        ("log_scale", C.c_void_p),
        ("opacity_logit", C.c_void_p),
        ("grid_values", C.c_void_p),
    ]


class AdamSegment(C.Structure):
    _fields_ = [
        ("param", C.c_void_p),
        ("grad", C.c_void_p),
        ("m", C.c_void_p),
        ("v", C.c_void_p),
        ("len", C.c_int64),
        ("group", C.c_int32),
        ("_pad", C.c_int32),
    ]


class Grads(C.Structure):
    _fields_ = [
        ("position", C.c_void_p),
        ("depth_key", C.c_void_p),
        ("theta", C.c_void_p),
        ("quat", C.c_void_p),
        ("log_scale", C.c_void_p),
        ("opacity_logit", C.c_void_p),
        ("grid_values", C.c_void_p),
    ]


class SplatFileInfo(C.Structure):
    _fields_ = [("version", C.c_int32), ("mode", C.c_int32), ("count", C.c_int64), ("n", C.c_int32),
                ("sigma", C.c_float)]


class Camera(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("_pad", C.c_int32),
        ("background", C.c_double * 3),
        ("fx", C.c_double),
        ("fy", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("rot", C.c_double * 9),
        ("trans", C.c_double * 3),
        ("near_plane", C.c_double),
    ]


class RasterConfigC(C.Structure):
    _fields_ = [
        ("tile_size", C.c_int32),
        ("threads", C.c_int32),
        ("cutoff_radius", C.c_double),
        ("alpha_skip", C.c_double),
        ("early_stop_transmittance", C.c_double),
    ]


class RenderOut(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("color", C.c_void_p),
        ("final_transmittance", C.c_void_p),
        ("last_rank", C.c_void_p),
        ("splat_count", C.c_int64),
        ("grid_n", C.c_int32),
        ("tile_size", C.c_int32),
    ]


class LearningRatesC(C.Structure):
    _fields_ = [
        ("position", C.c_double),
        ("theta", C.c_double),
        ("log_scale", C.c_double),
        ("opacity_logit", C.c_double),
        ("color_grid", C.c_double),
        ("position_gamma", C.c_double),
    ]


class AdamStateC(C.Structure):
    _fields_ = [
        ("t", C.c_int64),
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("epsilon", C.c_double),
        ("m", Grads),
        ("v", Grads),
    ]


class SceneSpec(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("n", C.c_int32),
        ("count", C.c_int64),
        ("seed", C.c_uint64),
        ("mean_lo", C.c_double),
        ("mean_hi", C.c_double),
        ("mean_sigma", C.c_double),
        ("log_scale_lo", C.c_double),
        ("log_scale_hi", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]


# every exported entry point: name -> (restype, argtypes)
P = C.c_void_p
_SIGS = {
    "gb_abi_version": (C.c_int, []),
    "gb_last_error_string": (C.c_char_p, []),
    "gb_context_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "gb_context_destroy": (C.c_int, [P]),
    "gb_context_set_stream": (C.c_int, [P, P]),
    "gb_context_stream": (P, [P]),
    "gb_sync": (C.c_int, [P]),
    "gb_context_launch_count": (C.c_int64, [P]),
    "gb_context_profile": (C.c_int, [P, C.c_int]),
    "gb_context_profile_read": (C.c_int, [P, P, P, C.c_int]),
    "gb_device_alloc": (C.c_int, [P, C.c_uint64, C.POINTER(P)]),
    "gb_device_free": (C.c_int, [P, P]),
    "gb_copy_h2d": (C.c_int, [P, P, P, C.c_uint64, C.c_int]),
    "gb_copy_d2h": (C.c_int, [P, P, P, C.c_uint64, C.c_int]),
    "gb_memset_device": (C.c_int, [P, P, C.c_int, C.c_uint64]),
    "gb_binning_create": (C.c_int, [P, C.POINTER(P)]),
    "gb_binning_destroy": (C.c_int, [P]),
    "gb_build_binning": (C.c_int, [P, C.POINTER(Splats), C.POINTER(Camera), C.POINTER(RasterConfigC), P]),
    "gb_binning_info": (C.c_int, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "gb_binning_set_capacity": (C.c_int, [P, C.c_int64, P]),
    "gb_context_profile_intervals": (C.c_int, [P, P, C.c_int32, P, P, C.c_int64, C.POINTER(C.c_int64)]),
    "gb_graph_begin": (C.c_int, [P, C.c_int32]),
    "gb_graph_end": (C.c_int, [P, C.c_int32, C.POINTER(P)]),
    "gb_graph_launch": (C.c_int, [P]),
    "gb_stream_wait_event": (C.c_int, [P, P, C.c_int32]),
    "gb_graph_destroy": (C.c_int, [P]),
    "gb_binning_store_total": (C.c_int, [P, P, P]),
    "gb_binning_copy_to_host": (C.c_int, [P, P, P, P]),
    "gb_render_forward": (C.c_int, [P, C.POINTER(Splats), C.POINTER(Camera), P, C.POINTER(RenderOut)]),
    "gb_render_backward": (
        C.c_int,
        [P, C.POINTER(Splats), C.POINTER(Camera), P, C.POINTER(RenderOut), P, C.POINTER(Grads)],
    ),
    "gb_render": (C.c_int, [P, C.POINTER(Splats), C.POINTER(Camera), C.POINTER(RasterConfigC), P, C.POINTER(RenderOut)]),
    "gb_render_loss_backward": (
        C.c_int,
        [P, C.POINTER(Splats), C.POINTER(Camera), P, P, C.c_int32, C.c_float, C.POINTER(RenderOut), P, P,
         C.POINTER(Grads)],
    ),
    "gb_l1_loss": (C.c_int, [P, P, P, C.c_int64, C.c_float, P, P]),
    "gb_mse_loss": (C.c_int, [P, P, P, C.c_int64, C.c_float, P, P]),
    "gb_adam_step": (
        C.c_int,
        [P, C.c_int32, C.c_int64, C.c_int32, C.POINTER(Grads), C.POINTER(Grads), C.POINTER(AdamStateC),
         C.POINTER(LearningRatesC)],
    ),
    "gb_adam_check": (C.c_int, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "gb_adam_segments": (
        C.c_int,
        [P, C.c_int32, C.POINTER(AdamSegment), C.c_int32, C.POINTER(AdamStateC), C.POINTER(LearningRatesC), P],
    ),
    "gb_ssim": (C.c_int, [P, P, P, C.c_int32, C.c_int32, C.c_int32, P, P, C.c_float]),
    "gb_psnr": (C.c_int, [P, P, P, C.c_int64, C.POINTER(C.c_double)]),
    "gb_fit_initialize": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_uint64, P, P, P, P, P, P]),
    "gb_downsample_size": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_int32)]),
    "gb_downsample_grids": (C.c_int, [P, P, C.c_int64, C.c_int32, C.c_int32, P]),
    "gb_splats_file_info": (C.c_int, [C.c_char_p, C.POINTER(SplatFileInfo)]),
    "gb_splats_save": (C.c_int, [P, C.POINTER(Splats), C.c_int32, C.c_char_p]),
    "gb_splats_load": (C.c_int, [P, C.c_char_p, C.c_int64, C.c_int32, C.POINTER(Grads)]),
    "gb_scene_generate": (C.c_int, [C.POINTER(SceneSpec), P, P, P, P, P, P, P]),
    "gb_uniform_fill": (C.c_int, [C.c_uint64, C.c_int64, P]),
    "gb_rng_uniform": (C.c_int, [C.c_uint64, C.c_int64, P]),
    "gb_rng_normal": (C.c_int, [C.c_uint64, C.c_int64, C.c_double, C.c_double, P]),
    "gb_adam_flag_init": (C.c_int, [P, P, P]),
    "gb_event_create": (C.c_int, [P, C.POINTER(P)]),
    "gb_event_record": (C.c_int, [P, P]),
    "gb_event_destroy": (C.c_int, [P, P]),
    "gb_context_set_texel_grad_stride": (C.c_int, [P, C.c_int32]),
    "gb_texel_grads_unpad": (C.c_int, [P, P, P, C.c_int64, C.c_int32]),
    "gb_context_set_texel_rgba": (C.c_int, [P, P]),
    "gb_texels_pad": (C.c_int, [P, P, P, C.c_int64]),
    "gb_comm_unique_id": (C.c_int, [P]),
    "gb_comm_init_rank": (C.c_int, [P, C.c_int32, P, C.c_int32, C.POINTER(P)]),
    "gb_comm_init_all": (C.c_int, [P, C.c_int32, P]),
    "gb_comm_destroy": (C.c_int, [P]),
    "gb_comm_info": (C.c_int, [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "gb_comm_check": (C.c_int, [P]),
    "gb_allreduce_grads": (C.c_int, [P, P, P, C.c_int64]),
    "gb_reduce_scatter_grads": (C.c_int, [P, P, P, P, C.c_int64]),
    "gb_all_gather_params": (C.c_int, [P, P, P, P, C.c_int64]),
    "gb_allreduce_flag_min": (C.c_int, [P, P, P]),
}
EXPORTED = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2412_12734_b200/csrc` (no CPU fallback exists)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class GBError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str = None):
        if msg is None:
            msg = lib.gb_last_error_string().decode(errors="replace")
        super().__init__(f"{where}: status {status}: {msg}")
        self.status = status


class InvalidArgument(GBError, ValueError):
    pass


class Mismatch(GBError, ValueError):
    pass


class NonFinite(GBError):
    pass


class SplatIoError(GBError):
    """serialize.hpp:23-25"""


class NcclError(GBError):
    """a collective of the view-sharded step failed (GB_NCCL_ERROR)"""


def check(status: int, where: str) -> None:
    if status == GB_OK:
        return
    if status == GB_INVALID_ARGUMENT:
        raise InvalidArgument(status, where)
    if status == GB_MISMATCH:
        raise Mismatch(status, where)
    if status == GB_NONFINITE:
        raise NonFinite(status, where)
    if status == GB_IO_ERROR:
        raise SplatIoError(status, where)
    if status == GB_NCCL_ERROR:
        raise NcclError(status, where)
    raise GBError(status, where)
