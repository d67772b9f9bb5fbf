"""Reference-shaped host API over the C-ABI (include/gb_raster.h).

Mirrors the reference's rasterizer interface (/root/reference/proj/include/gbil)
name for name -- ``ColorGridConfig``, ``SplatSet``, ``ImagePlaneCamera``,
``RasterConfig``, ``TileBinning``, ``RenderOutput``, ``GradientBuffer``,
``build_binning``, ``render_forward``, ``render_backward``, ``render``,
``adam_step`` -- with fp32 CUDA tensors in place of ``std::vector<double>``.
Errors follow the reference's throw sites: ``std::invalid_argument`` becomes
:class:`InvalidArgument` / :class:`Mismatch` (both ``ValueError``), adam's
non-finite ``std::runtime_error`` becomes :class:`NonFinite`.

Every compute call goes through ``libgb_raster.so``; PyTorch only provides
device memory and the current CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import GBError, InvalidArgument, Mismatch, NonFinite, check, lib

MODE_ORTHO = _lib.MODE_ORTHO
MODE_PINHOLE = _lib.MODE_PINHOLE
K_MAX_ALPHA = 0.999  # core.hpp:16
K_MIN_SCALE = 1e-8  # core.hpp:19


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    if t.dtype not in (torch.float32, torch.int32):
        raise TypeError(f"expected fp32/int32 tensor, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


# --------------------------------------------------------------------------------------------
# context
# --------------------------------------------------------------------------------------------
class _Context:
    """One C-ABI context per (device, CUDA stream): a context owns the scratch of the calls it
    runs, so work issued on different streams (the trainer's two view lanes) never shares it."""

    _by_stream: dict = {}

    def __init__(self, device: int, stream: int):
        h = C.c_void_p()
        check(lib.gb_context_create(device, C.byref(h)), "gb_context_create")
        self.handle = h
        self.device = device
        check(lib.gb_context_set_stream(h, C.c_void_p(stream)), "gb_context_set_stream")

    @classmethod
    def get(cls, device: torch.device) -> "_Context":
        if device.type != "cuda":
            raise ValueError(f"tensors must live on a CUDA device (got {device}); there is no CPU path")
        idx = device.index if device.index is not None else torch.cuda.current_device()
        with torch.cuda.device(idx):
            stream = torch.cuda.current_stream(idx).cuda_stream
        ctx = cls._by_stream.get((idx, stream))
        if ctx is None:
            ctx = cls(idx, stream)
            cls._by_stream[(idx, stream)] = ctx
        return ctx

    @classmethod
    def all(cls, device) -> list:
        idx = torch.device(device).index
        idx = torch.cuda.current_device() if idx is None else idx
        return [c for (d, _), c in cls._by_stream.items() if d == idx]

    def launches(self) -> int:
        return int(lib.gb_context_launch_count(self.handle))

    def profile(self, enable: bool) -> None:
        check(lib.gb_context_profile(self.handle, int(enable)), "gb_context_profile")

    def profile_intervals(self, ref_event, kernel: str):
        """[(start_ms, stop_ms)] of the recorded launches of `kernel` after torch.cuda.Event `ref_event`."""
        import numpy as _np

        kid = _lib.KERNEL_NAMES.index(kernel)
        n = C.c_int64()
        check(lib.gb_context_profile_intervals(self.handle, C.c_void_p(ref_event.cuda_event), kid, None, None, 0,
                                               C.byref(n)), "gb_context_profile_intervals")
        a = _np.zeros(max(1, n.value), _np.float64)
        b = _np.zeros(max(1, n.value), _np.float64)
        check(lib.gb_context_profile_intervals(self.handle, C.c_void_p(ref_event.cuda_event), kid, a.ctypes.data,
                                               b.ctypes.data, n.value, C.byref(n)), "gb_context_profile_intervals")
        return list(zip(a[: n.value].tolist(), b[: n.value].tolist()))

    def profile_read(self) -> dict:
        """{kernel: (total_ms, launches)} since the last read (synchronises)."""
        import numpy as _np

        n = len(_lib.KERNEL_NAMES)
        ms = _np.zeros(n, _np.float64)
        cnt = _np.zeros(n, _np.int64)
        check(lib.gb_context_profile_read(self.handle, ms.ctypes.data, cnt.ctypes.data, n), "gb_context_profile_read")
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(_lib.KERNEL_NAMES)}


def context(device=None) -> _Context:
    """The context of the current CUDA stream on `device`."""
    return _Context.get(torch.device(device) if device is not None else torch.device("cuda"))


def all_contexts(device=None) -> list:
    """Every context created on `device` (one per stream used)."""
    return _Context.all(device if device is not None else "cuda")


def memset_(t: torch.Tensor) -> None:
    """Zero a contiguous device tensor with a stream-ordered memset on the current stream's context
    (gb_memset_device: a memset node under graph capture, no framework kernel)."""
    if not t.is_contiguous():
        raise ValueError("memset_: tensor must be contiguous")
    check(lib.gb_memset_device(context(t.device).handle, C.c_void_p(t.data_ptr()), 0, t.numel() * t.element_size()),
          "memset_")


def copy_h2d(dst: torch.Tensor, src: torch.Tensor) -> None:
    """Stream-ordered copy of host ``src`` into the front of device ``dst`` on the current stream
    (gb_copy_h2d; asynchronous when ``src`` is pinned)."""
    nbytes = src.numel() * src.element_size()
    if nbytes > dst.numel() * dst.element_size():
        raise ValueError("copy_h2d: destination too small")
    check(lib.gb_copy_h2d(context(dst.device).handle, C.c_void_p(dst.data_ptr()), C.c_void_p(src.data_ptr()),
                          nbytes, 0), "copy_h2d")


class StepGraph:
    """A CUDA graph of C-ABI work (gb_graph_*): capture() records what ``fn`` issues on the first
    context's stream and the streams that fork from and join back into it; launch() replays it on
    that stream.  Per-kernel profiling and launch counts of the contexts keep working across replays."""

    def __init__(self, contexts: list):
        self._ctxs = (C.c_void_p * len(contexts))(*[c.handle.value for c in contexts])
        self._keep = list(contexts)
        self.handle = None

    def capture(self, fn) -> None:
        check(lib.gb_graph_begin(self._ctxs, len(self._keep)), "gb_graph_begin")
        err = None
        try:
            fn()
        except BaseException as e:  # the capture must be closed either way
            err = e
        h = C.c_void_p()
        st = lib.gb_graph_end(self._ctxs, len(self._keep), C.byref(h))
        if err is not None:
            raise err
        check(st, "gb_graph_end")
        self.handle = h

    def launch(self) -> None:
        check(lib.gb_graph_launch(self.handle), "gb_graph_launch")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            lib.gb_graph_destroy(h)
            self.handle = None


# --------------------------------------------------------------------------------------------
# configs and cameras
# --------------------------------------------------------------------------------------------
@dataclass
class ColorGridConfig:
    """core.hpp:29-42"""

    n: int = 1
    sigma: float = 0.5
    channels: int = 3

    def texels_per_splat(self) -> int:
        return self.n * self.n * 3

    def validate(self) -> None:
        if self.n < 1:
            raise ValueError("ColorGridConfig: n must be >= 1")
        if not self.sigma > 0.0:
            raise ValueError("ColorGridConfig: sigma must be > 0")


@dataclass
class RasterConfig:
    """raster.hpp:21-32"""

    tile_size: int = 16
    cutoff_radius: float = 3.0
    alpha_skip: float = 1.0 / 255.0
    early_stop_transmittance: float = 1e-4
    threads: int = 1

    def to_c(self) -> _lib.RasterConfigC:
        return _lib.RasterConfigC(self.tile_size, self.threads, self.cutoff_radius, self.alpha_skip,
                                  self.early_stop_transmittance)


@dataclass
class ImagePlaneCamera:
    """Orthographic fitting camera (core.hpp:104-116): pixel (i,j) samples (i+0.5, j+0.5)."""

    width: int = 0
    height: int = 0
    background: Sequence[float] = (0.0, 0.0, 0.0)
    mode: int = field(default=MODE_ORTHO, init=False)

    def to_c(self) -> _lib.Camera:
        c = _lib.Camera()
        c.mode = MODE_ORTHO
        c.width, c.height = self.width, self.height
        for i in range(3):
            c.background[i] = float(self.background[i])
        c.fx = c.fy = 1.0
        return c


@dataclass
class PinholeCamera:
    """Perspective 2DGS camera (builder extension).

    OpenCV convention: x right, y down, +z forward; x_pix = fx*X/Z + cx with
    pixel centres at i + 0.5; ``rot``/``trans`` map world -> camera.
    """

    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    rot: np.ndarray
    trans: np.ndarray
    background: Sequence[float] = (0.0, 0.0, 0.0)
    near_plane: float = 0.01
    mode: int = field(default=MODE_PINHOLE, init=False)

    @staticmethod
    def look_at(eye, target, width, height, fx, fy, cx, cy, up=(0.0, 1.0, 0.0), background=(0.0, 0.0, 0.0),
                near_plane=0.01) -> "PinholeCamera":
        """z_cam = normalize(target - eye), x_cam = normalize(up x z_cam), y_cam = z_cam x x_cam.

        With eye=(0,0,-d) looking at the origin this gives rot = I, trans = (0,0,d).
        """
        eye = np.asarray(eye, dtype=np.float64)
        f = np.asarray(target, dtype=np.float64) - eye
        f /= np.linalg.norm(f)
        r = np.cross(np.asarray(up, dtype=np.float64), f)
        r /= np.linalg.norm(r)
        d = np.cross(f, r)
        rot = np.stack([r, d, f])
        trans = -rot @ eye
        return PinholeCamera(width, height, fx, fy, cx, cy, rot, trans, background, near_plane)

    @staticmethod
    def from_spec(spec) -> "PinholeCamera":
        """From a scenes.CameraSpec."""
        return PinholeCamera(spec.width, spec.height, spec.fx, spec.fy, spec.cx, spec.cy, spec.rot, spec.trans,
                             tuple(spec.background), spec.near_plane)

    def to_c(self) -> _lib.Camera:
        c = _lib.Camera()
        c.mode = MODE_PINHOLE
        c.width, c.height = self.width, self.height
        for i in range(3):
            c.background[i] = float(self.background[i])
        c.fx, c.fy, c.cx, c.cy = self.fx, self.fy, self.cx, self.cy
        rot = np.asarray(self.rot, dtype=np.float64).reshape(9)
        for i in range(9):
            c.rot[i] = float(rot[i])
        tr = np.asarray(self.trans, dtype=np.float64).reshape(3)
        for i in range(3):
            c.trans[i] = float(tr[i])
        c.near_plane = self.near_plane
        return c


# --------------------------------------------------------------------------------------------
# splats and gradients
# --------------------------------------------------------------------------------------------
_FIELDS = ("position", "depth_key", "theta", "quat", "log_scale", "opacity_logit", "grid")


class SplatSet:
    """K primitives, structure of arrays, fp32 on one CUDA device (core.hpp:53-87).

    ortho : position (K,2), depth_key (K,), theta (K,)
    pinhole: position (K,3) world mean, quat (K,4) (w,x,y,z)
    both  : log_scale (K,2), opacity_logit (K,), grid (K, n*n*3) in (i_u, i_v, ch) order
    """

    def __init__(self, mode: int, grid_config: ColorGridConfig, **arrays):
        grid_config.validate()
        self.mode = mode
        self.grid_config = grid_config
        for f in _FIELDS:
            setattr(self, f, arrays.get(f))
        self.count = int(self.opacity_logit.shape[0])

    @staticmethod
    def from_numpy(mode: int, grid_config: ColorGridConfig, device="cuda", **arrays) -> "SplatSet":
        t = {k: torch.as_tensor(np.ascontiguousarray(v, dtype=np.float32), device=device) for k, v in arrays.items()
             if v is not None}
        return SplatSet(mode, grid_config, **t)

    @property
    def device(self) -> torch.device:
        return self.opacity_logit.device

    def tensors(self) -> dict:
        return {f: getattr(self, f) for f in _FIELDS if getattr(self, f) is not None}

    def to_c(self) -> _lib.Splats:
        s = _lib.Splats()
        s.count = self.count
        s.grid = _lib.GridConfig(self.grid_config.n, 0, self.grid_config.sigma)
        s.position = _ptr(self.position)
        s.depth_key = _ptr(self.depth_key)
        s.theta = _ptr(self.theta)
        s.quat = _ptr(self.quat)
        s.log_scale = _ptr(self.log_scale)
        s.opacity_logit = _ptr(self.opacity_logit)
        s.grid_values = _ptr(self.grid)
        return s


class GradientBuffer:
    """Gradients w.r.t. the raw parameters, mirroring SplatSet (core.hpp:140-178).

    All groups live in one flat fp32 tensor (``flat``) so the multi-GPU step can
    all-reduce them with a single collective; the per-group tensors are views.
    """

    def __init__(self, like: SplatSet, multiple: int = 4):
        self.mode = like.mode
        self.count = like.count
        self.grid_config = like.grid_config
        shapes = [(f, tuple(getattr(like, f).shape)) for f in _FIELDS if getattr(like, f) is not None]
        # keep every group 16-byte aligned (vector red.global.add on the texel grads); the total is padded
        # to `multiple` elements (the sharded optimiser splits the buffer evenly over the ranks)
        pad = lambda n: (n + 3) & ~3
        total = sum(pad(int(np.prod(s))) for _, s in shapes)
        total = -(-total // multiple) * multiple
        self.flat = torch.zeros(total, dtype=torch.float32, device=like.device)
        self.offsets = {}
        o = 0
        for f in _FIELDS:
            setattr(self, f, None)
        for f, s in shapes:
            n = int(np.prod(s))
            setattr(self, f, self.flat[o:o + n].view(s))
            self.offsets[f] = (o, n)
            o += pad(n)

    def zero_(self) -> "GradientBuffer":
        self.flat.zero_()
        return self

    def tensors(self) -> dict:
        return {f: getattr(self, f) for f in _FIELDS if getattr(self, f) is not None}

    def to_c(self) -> _lib.Grads:
        g = _lib.Grads()
        g.position = _ptr(self.position)
        g.depth_key = _ptr(self.depth_key)
        g.theta = _ptr(self.theta)
        g.quat = _ptr(self.quat)
        g.log_scale = _ptr(self.log_scale)
        g.opacity_logit = _ptr(self.opacity_logit)
        g.grid_values = _ptr(self.grid)
        return g


# --------------------------------------------------------------------------------------------
# binning / render
# --------------------------------------------------------------------------------------------
class TileBinning:
    """Device-resident per-tile sorted lists (raster.hpp:105-114)."""

    def __init__(self, device=None):
        self.ctx = context(device)
        h = C.c_void_p()
        check(lib.gb_binning_create(self.ctx.handle, C.byref(h)), "gb_binning_create")
        self.handle = h
        self.config: Optional[RasterConfig] = None
        self.width = self.height = 0

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            lib.gb_binning_destroy(h)
            self.handle = None

    def info(self, total=True):
        tx, ty, tot = C.c_int32(), C.c_int32(), C.c_int64(-1)
        check(lib.gb_binning_info(self.handle, C.byref(tx), C.byref(ty), C.byref(tot) if total else None),
              "gb_binning_info")
        return tx.value, ty.value, tot.value

    @property
    def tiles_x(self) -> int:
        return self.info(False)[0]

    @property
    def tiles_y(self) -> int:
        return self.info(False)[1]

    def tile_count(self) -> int:
        tx, ty, _ = self.info(False)
        return tx * ty

    def set_capacity(self, capacity: int, overflow: torch.Tensor = None) -> None:
        """Capacity mode (gb_binning_set_capacity): builds never read the pair count back, so they
        run ahead of the GPU and can be captured into a CUDA graph.  ``overflow`` (a zeroed device
        int32 tensor) is set to 1 by a build with more than ``capacity`` pairs.  0 = blocking mode."""
        self._overflow = overflow  # keep alive
        check(lib.gb_binning_set_capacity(self.handle, int(capacity), _ptr(overflow)), "gb_binning_set_capacity")

    def store_total(self, dst: torch.Tensor) -> None:
        """Stream-ordered copy of the last build's pair count into ``dst`` (a 1-element int32 device tensor)."""
        if dst.dtype != torch.int32 or dst.numel() != 1:
            raise TypeError("store_total: expected a 1-element int32 tensor")
        check(lib.gb_binning_store_total(self.ctx.handle, self.handle, _ptr(dst)), "gb_binning_store_total")

    @property
    def total(self) -> int:
        return self.info()[2]

    def csr(self):
        """(offsets[tiles+1] int64, values[total] int32) on the host."""
        tx, ty, total = self.info()
        offsets = np.zeros(tx * ty + 1, dtype=np.int64)
        values = np.zeros(max(total, 1), dtype=np.int32)
        check(lib.gb_binning_copy_to_host(self.ctx.handle, self.handle, offsets.ctypes.data, values.ctypes.data),
              "gb_binning_copy_to_host")
        return offsets, values[:total]

    @property
    def tiles(self):
        offsets, values = self.csr()
        return [values[offsets[i]:offsets[i + 1]] for i in range(len(offsets) - 1)]


def build_binning(splats: SplatSet, camera, config: RasterConfig = None, out: TileBinning = None) -> TileBinning:
    """raster.hpp:116-147"""
    config = config or RasterConfig()
    b = out if out is not None else TileBinning(splats.device)
    ctx = context(splats.device)
    s, cam, cfg = splats.to_c(), camera.to_c(), config.to_c()
    check(lib.gb_build_binning(ctx.handle, C.byref(s), C.byref(cam), C.byref(cfg), b.handle), "build_binning")
    b.config = config
    b.width, b.height = camera.width, camera.height
    return b


class RenderOutput:
    """core.hpp:123-136 -- color (H,W,3), final_transmittance (H,W), last_rank (H,W)."""

    def __init__(self, width: int, height: int, device):
        self.width, self.height = width, height
        self.color = torch.empty((height, width, 3), dtype=torch.float32, device=device)
        self.final_transmittance = torch.empty((height, width), dtype=torch.float32, device=device)
        self.last_rank = torch.empty((height, width), dtype=torch.int32, device=device)
        self._c = _lib.RenderOut(width, height, self.color.data_ptr(), self.final_transmittance.data_ptr(),
                                 self.last_rank.data_ptr(), 0, 0, 0)

    @property
    def splat_count(self):
        return self._c.splat_count

    @property
    def grid_n(self):
        return self._c.grid_n

    @property
    def tile_size(self):
        return self._c.tile_size

    @property
    def alpha(self) -> torch.Tensor:
        """Accumulated alpha 1 - T (the BASELINE configs' second output)."""
        return 1.0 - self.final_transmittance


class _TexelRGBA:
    """Within the block, the context's compositors read the texels from ``rgba`` (an RGBA-padded copy of the
    splats' grid, gb_context_set_texel_rgba; see texels_pad) instead of the reference layout."""

    def __init__(self, ctx, rgba, grid_numel):
        self.ctx, self.rgba, self.grid_numel = ctx, rgba, grid_numel

    def __enter__(self):
        if self.rgba is not None:
            if self.rgba.numel() * 3 != 4 * self.grid_numel or self.rgba.data_ptr() % 16:
                raise ValueError("texels_rgba: padded buffer must hold K*n*n*4 floats, 16-byte aligned")
            check(lib.gb_context_set_texel_rgba(self.ctx.handle, C.c_void_p(self.rgba.data_ptr())),
                  "gb_context_set_texel_rgba")

    def __exit__(self, *a):
        if self.rgba is not None:
            check(lib.gb_context_set_texel_rgba(self.ctx.handle, None), "gb_context_set_texel_rgba")


def texels_pad(grid: torch.Tensor, rgba: torch.Tensor) -> None:
    """rgba <- the RGBA-padded copy of a reference-layout texel grid (K*n*n*3 -> K*n*n*4 floats; gb_texels_pad),
    on the current stream."""
    if rgba.numel() * 3 != grid.numel() * 4:
        raise ValueError("texels_pad: size mismatch")
    check(lib.gb_texels_pad(context(grid.device).handle, _ptr(grid), _ptr(rgba), grid.numel() // 3), "gb_texels_pad")


def render_forward(splats: SplatSet, camera, binning: TileBinning, out: RenderOutput = None,
                   texels_rgba: torch.Tensor = None) -> RenderOutput:
    """raster.hpp:201-261.  ``texels_rgba``: an RGBA-padded copy of the splats' texels (texels_pad) that K3
    reads with one 16-byte load per texel -- the same image."""
    ctx = context(splats.device)
    out = out if out is not None else RenderOutput(camera.width, camera.height, splats.device)
    s, cam = splats.to_c(), camera.to_c()
    with _TexelRGBA(ctx, texels_rgba, splats.count * 3 * splats.grid_config.n ** 2):
        check(lib.gb_render_forward(ctx.handle, C.byref(s), C.byref(cam), binning.handle, C.byref(out._c)),
              "render_forward")
    return out


class _TexelStride:
    """Within the block, the context's backwards write texel gradients into ``padded`` (RGBA, stride 4:
    gb_context_set_texel_grad_stride) instead of the gradient buffer's reference-layout grid group."""

    def __init__(self, ctx, g, padded, grid_numel):
        self.ctx, self.g, self.padded, self.grid_numel = ctx, g, padded, grid_numel

    def __enter__(self):
        if self.padded is not None:
            if self.padded.numel() * 3 != 4 * self.grid_numel or self.padded.data_ptr() % 16:
                raise ValueError("texel_grad: padded buffer must hold K*n*n*4 floats, 16-byte aligned")
            self.g.grid_values = self.padded.data_ptr()
            check(lib.gb_context_set_texel_grad_stride(self.ctx.handle, 4), "gb_context_set_texel_grad_stride")
        return self.g

    def __exit__(self, *a):
        if self.padded is not None:
            check(lib.gb_context_set_texel_grad_stride(self.ctx.handle, 3), "gb_context_set_texel_grad_stride")


def render_backward(splats: SplatSet, camera, binning: TileBinning, output: RenderOutput,
                    image_grad: torch.Tensor, grads: GradientBuffer = None,
                    texel_grad: torch.Tensor = None, texels_rgba: torch.Tensor = None) -> GradientBuffer:
    """raster.hpp:277-387.  Accumulates into ``grads`` (a fresh zeroed buffer by default).  ``texel_grad``: an
    RGBA-padded (K*n*n*4) buffer that receives the texel gradients instead of ``grads.grid`` (convert with
    texel_grads_unpad)."""
    ctx = context(splats.device)
    if grads is None:
        grads = GradientBuffer(splats)
    if image_grad.numel() != output.color.numel():
        raise ValueError("render_backward: image_grad size mismatch")
    image_grad = image_grad.contiguous()
    s, cam, g = splats.to_c(), camera.to_c(), grads.to_c()
    with _TexelStride(ctx, g, texel_grad, grads.grid.numel()) as g, _TexelRGBA(ctx, texels_rgba, grads.grid.numel()):
        check(lib.gb_render_backward(ctx.handle, C.byref(s), C.byref(cam), binning.handle, C.byref(output._c),
                                     _ptr(image_grad), C.byref(g)), "render_backward")
    return grads


def texel_grads_unpad(padded: torch.Tensor, dst: torch.Tensor, accumulate: bool = False) -> None:
    """dst (reference layout, K*n*n*3) (+)= the RGBA-padded texel gradients (K*n*n*4), on the current stream."""
    if padded.numel() * 3 != dst.numel() * 4:
        raise ValueError("texel_grads_unpad: size mismatch")
    check(lib.gb_texel_grads_unpad(context(dst.device).handle, _ptr(padded), _ptr(dst), padded.numel() // 4,
                                   int(accumulate)), "gb_texel_grads_unpad")


def render_loss_backward(splats: SplatSet, camera, binning: TileBinning, target: torch.Tensor, loss: str = "l1",
                         scale: float = None, grads: GradientBuffer = None, loss_acc: torch.Tensor = None,
                         output: RenderOutput = None, image_grad: torch.Tensor = None,
                         texel_grad: torch.Tensor = None, texels_rgba: torch.Tensor = None):
    """render_forward + l1_loss / mse_loss + render_backward of one view in one pass
    (train.hpp:120-133 around raster.hpp:201-387).  Returns (loss_acc, grads); ``loss_acc``
    (a device float, zero by default) and ``grads`` accumulate.  ``output`` / ``image_grad``,
    when given, receive the forward buffers and the loss cotangent."""
    kinds = {"l1": 0, "mse": 1}
    if loss not in kinds:
        raise ValueError(f"render_loss_backward: unknown loss {loss!r}")
    ctx = context(splats.device)
    n = camera.width * camera.height * 3
    if target.numel() != n:
        raise ValueError("render_loss_backward: dimension mismatch")
    scale = 1.0 / n if scale is None else scale
    if grads is None:
        grads = GradientBuffer(splats)
    if loss_acc is None:
        loss_acc = torch.zeros((), dtype=torch.float32, device=splats.device)
    if image_grad is not None and image_grad.numel() != n:
        raise ValueError("render_loss_backward: image_grad size mismatch")
    target = target.contiguous()
    s, cam, g = splats.to_c(), camera.to_c(), grads.to_c()
    with _TexelStride(ctx, g, texel_grad, grads.grid.numel()) as g, _TexelRGBA(ctx, texels_rgba, grads.grid.numel()):
        check(lib.gb_render_loss_backward(ctx.handle, C.byref(s), C.byref(cam), binning.handle, _ptr(target),
                                          kinds[loss], scale, C.byref(output._c) if output is not None else None,
                                          _ptr(image_grad) if image_grad is not None else None, _ptr(loss_acc),
                                          C.byref(g)), "render_loss_backward")
    return loss_acc, grads


def render(splats: SplatSet, camera, config: RasterConfig = None) -> RenderOutput:
    """raster.hpp:389-392"""
    b = build_binning(splats, camera, config)
    return render_forward(splats, camera, b)


# --------------------------------------------------------------------------------------------
# losses and Adam
# --------------------------------------------------------------------------------------------
def l1_loss(color: torch.Tensor, target: torch.Tensor, scale: float = None, grad: torch.Tensor = None,
            loss: torch.Tensor = None):
    """L1 photometric loss: returns (loss (device scalar), dL/dC).  scale defaults to 1/numel (mean)."""
    if color.shape != target.shape:
        raise ValueError("l1_loss: dimension mismatch")
    ctx = context(color.device)
    n = color.numel()
    scale = 1.0 / n if scale is None else scale
    grad = torch.empty_like(color) if grad is None else grad
    if loss is None:
        loss = torch.zeros((), dtype=torch.float32, device=color.device)
    check(lib.gb_l1_loss(ctx.handle, _ptr(color.contiguous()), _ptr(target.contiguous()), n, scale, _ptr(grad),
                         _ptr(loss)), "l1_loss")
    return loss, grad


def mse_loss(color: torch.Tensor, target: torch.Tensor, scale: float = None, grad: torch.Tensor = None,
             loss: torch.Tensor = None):
    """train.hpp:120-133: mean squared error, gradient 2(c - t)/n."""
    if color.shape != target.shape:
        raise ValueError("mse_loss: dimension mismatch")
    ctx = context(color.device)
    n = color.numel()
    scale = 1.0 / n if scale is None else scale
    grad = torch.empty_like(color) if grad is None else grad
    if loss is None:
        loss = torch.zeros((), dtype=torch.float32, device=color.device)
    check(lib.gb_mse_loss(ctx.handle, _ptr(color.contiguous()), _ptr(target.contiguous()), n, scale, _ptr(grad),
                          _ptr(loss)), "mse_loss")
    return loss, grad


@dataclass
class LearningRates:
    """optim.hpp:17-40 (pinhole quaternions use the ``theta`` rate)."""

    position: float = 1.6e-4
    theta: float = 1e-3
    log_scale: float = 5e-3
    opacity_logit: float = 5e-2
    color_grid: float = 2.5e-3
    position_gamma: float = 1.0

    @staticmethod
    def scaled_for_image(width: int, height: int) -> "LearningRates":
        lrs = LearningRates()
        lrs.position *= max(width, height)
        return lrs

    def to_c(self):
        return _lib.LearningRatesC(self.position, self.theta, self.log_scale, self.opacity_logit, self.color_grid,
                                   self.position_gamma)


@dataclass
class AdamConfig:
    """optim.hpp:42-46"""

    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8


class AdamState:
    """optim.hpp:50-72: zero moments with the gradient layout, t counts completed steps.
    ``moments=False``: step count and config only (the sharded optimiser keeps its own slices)."""

    def __init__(self, like: SplatSet, config: AdamConfig = None, moments: bool = True):
        self.config = config or AdamConfig()
        self.t = 0
        self.m = GradientBuffer(like) if moments else None
        self.v = GradientBuffer(like) if moments else None

    def to_c(self) -> _lib.AdamStateC:
        empty = _lib.Grads()
        return _lib.AdamStateC(self.t, self.config.beta1, self.config.beta2, self.config.epsilon,
                               self.m.to_c() if self.m is not None else empty,
                               self.v.to_c() if self.v is not None else empty)


def adam_step(params: SplatSet, grads: GradientBuffer, state: AdamState, lrs: LearningRates,
              check_finite: bool = True) -> None:
    """optim.hpp:96-117.  With check_finite, synchronises and raises NonFinite like the reference."""
    if grads.count != params.count or grads.grid.numel() != params.grid.numel():
        raise ValueError("adam_step: gradient shape mismatch")
    ctx = context(params.device)
    p = _lib.Grads(_ptr(params.position), _ptr(params.depth_key), _ptr(params.theta), _ptr(params.quat),
                   _ptr(params.log_scale), _ptr(params.opacity_logit), _ptr(params.grid))
    g = grads.to_c()
    st = state.to_c()
    c_lrs = lrs.to_c()
    check(lib.gb_adam_step(ctx.handle, params.mode, params.count, params.grid_config.n, C.byref(p), C.byref(g),
                           C.byref(st), C.byref(c_lrs)), "adam_step")
    state.t = st.t
    if check_finite:
        grp, idx = C.c_int32(), C.c_int64()
        check(lib.gb_adam_check(ctx.handle, C.byref(grp), C.byref(idx)), "adam_step")
