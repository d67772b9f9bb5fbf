"""The image-fitting loop of the reference (train.hpp:22-219) and its metrics
(metrics.hpp:167-191), on the GPU.

``fit(target, cfg)`` keeps the reference's semantics -- initialize, then per
iteration rebuild the binning, forward, photometric loss (MSE, or MSE +
w (1 - SSIM)), non-finite-loss abort, backward, Adam; log (loss, PSNR, SSIM,
wall ms) every ``log_every`` iterations; optional GBIL checkpoints -- with
every kernel on the device: binning/compositing (K1-K5), the MSE (K6), SSIM
with its gradient and the PSNR sum (gb_metrics.cu), and Adam (K7).  The only
host round trips are the per-iteration loss read (for the reference's
non-finite check) and the logged metrics.
"""
from __future__ import annotations

import copy
import ctypes as C
import enum
import math
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .raster import (AdamConfig, AdamState, ColorGridConfig, GradientBuffer, ImagePlaneCamera, LearningRates,
                     RasterConfig, RenderOutput, SplatSet, TileBinning, _ptr, adam_step, build_binning, context,
                     mse_loss, render_backward, render_forward)
from .splat_io import save_splats

PSNR_CAP = 99.0  # metrics.hpp:12


class LossKind(enum.Enum):  # train.hpp:22
    mse = 0
    mse_plus_ssim = 1


class FitError(RuntimeError):  # train.hpp:58-60
    pass


@dataclass
class TrainConfig:
    """train.hpp:24-56"""

    splat_count: int = 1000
    iterations: int = 20000
    loss: LossKind = LossKind.mse
    ssim_weight: float = 0.2
    seed: int = 0
    grid: ColorGridConfig = field(default_factory=lambda: ColorGridConfig(4, 0.5))
    lrs: LearningRates = field(default_factory=LearningRates)
    position_lr_absolute: bool = False
    adam: AdamConfig = field(default_factory=AdamConfig)
    raster: RasterConfig = field(default_factory=RasterConfig)
    background: tuple = (0.0, 0.0, 0.0)
    log_every: int = 100
    checkpoint_every: int = 0
    checkpoint_dir: str = ""
    allow_any_n: bool = False

    def validate(self) -> None:
        if self.splat_count < 1:
            raise ValueError("TrainConfig: splat_count must be >= 1")
        if self.iterations < 1:
            raise ValueError("TrainConfig: iterations must be >= 1")
        self.grid.validate()
        if not self.allow_any_n and self.grid.n not in (1, 2, 4, 8):
            raise ValueError("TrainConfig: texture resolution must be one of 1, 2, 4, 8 (use the force flag for "
                             "other values)")
        lr = self.lrs
        if not (lr.position > 0 and lr.theta > 0 and lr.log_scale > 0 and lr.opacity_logit > 0 and lr.color_grid > 0):
            raise ValueError("LearningRates: all rates must be positive")
        if not (0.0 < lr.position_gamma <= 1.0):
            raise ValueError("LearningRates: position_gamma must be in (0, 1]")
        if self.raster.tile_size < 1:
            raise ValueError("RasterConfig: tile_size must be >= 1")
        if self.log_every < 1:
            raise ValueError("TrainConfig: log_every must be >= 1")
        if self.checkpoint_every < 0:
            raise ValueError("TrainConfig: negative checkpoint cadence")


@dataclass
class MetricRecord:  # train.hpp:62-68
    iter: int = 0
    loss: float = 0.0
    psnr: float = 0.0
    ssim: float = 0.0
    wall_ms: float = 0.0


@dataclass
class FitResult:  # train.hpp:70-73
    splats: SplatSet
    history: List[MetricRecord]


# ------------------------------------------------------------------------------------------------
# metrics (metrics.hpp:167-191)
# ------------------------------------------------------------------------------------------------
def _img(t: torch.Tensor) -> torch.Tensor:
    if t.dim() != 3 or t.shape[2] != 3:
        raise ValueError("expected an (H, W, 3) image")
    return t.contiguous()


def psnr(a: torch.Tensor, b: torch.Tensor) -> float:
    """Clamped-[0,1] PSNR in dB, capped at 99 (metrics.hpp:169-179)."""
    if a.shape != b.shape:
        raise ValueError("psnr: image size mismatch")
    out = C.c_double()
    check(lib.gb_psnr(context(a.device).handle, _ptr(_img(a)), _ptr(_img(b)), a.numel(), C.byref(out)), "psnr")
    return out.value


def _ssim(a, b, clamp, grad=None, grad_scale=0.0, acc=None):
    if a.shape != b.shape:
        raise ValueError("ssim: image size mismatch")
    H, W = a.shape[0], a.shape[1]
    acc = torch.zeros((), dtype=torch.float64, device=a.device) if acc is None else acc
    check(lib.gb_ssim(context(a.device).handle, _ptr(_img(a)), _ptr(_img(b)), W, H, int(clamp), acc.data_ptr(),
                      _ptr(grad), float(grad_scale)), "ssim")
    return acc


def ssim(a: torch.Tensor, b: torch.Tensor) -> float:
    """Mean SSIM of the [0,1]-clamped images (metrics.hpp:183-185)."""
    return float(_ssim(a, b, True))


def ssim_with_gradient(a: torch.Tensor, b: torch.Tensor):
    """(mean SSIM, d SSIM / d a) on raw values (metrics.hpp:189-191)."""
    g = torch.zeros_like(a)
    v = _ssim(a, b, False, g, 1.0)
    return float(v), g


# ------------------------------------------------------------------------------------------------
# the loop (train.hpp:80-219)
# ------------------------------------------------------------------------------------------------
def initialize(width: int, height: int, cfg: TrainConfig, device="cuda") -> SplatSet:
    """train.hpp:80-111 (same Rng draws as the reference, fp32)."""
    cfg.validate()
    if width < 1 or height < 1:
        raise ValueError("initialize: empty target image")
    K, n = cfg.splat_count, cfg.grid.n
    a = dict(position=np.zeros((K, 2), np.float32), depth_key=np.zeros(K, np.float32),
             theta=np.zeros(K, np.float32), log_scale=np.zeros((K, 2), np.float32),
             opacity_logit=np.zeros(K, np.float32), grid=np.zeros((K, n * n * 3), np.float32))
    check(lib.gb_fit_initialize(width, height, K, n, cfg.seed, *[a[f].ctypes.data for f in
                                ("position", "depth_key", "theta", "log_scale", "opacity_logit", "grid")]),
          "initialize")
    return SplatSet.from_numpy(_lib.MODE_ORTHO, copy.copy(cfg.grid), device=device, **a)


def photometric_loss(rendered: torch.Tensor, target: torch.Tensor, cfg: TrainConfig, grad: torch.Tensor = None):
    """train.hpp:135-145 -> (device loss tensor (float64), dL/d rendered)."""
    loss32, grad = mse_loss(rendered, target, grad=grad)
    value = loss32.to(torch.float64)
    if cfg.loss == LossKind.mse_plus_ssim:
        s = _ssim(rendered, target, False, grad, -cfg.ssim_weight)
        value = value + cfg.ssim_weight * (1.0 - s)
    return value, grad


def _write_checkpoint(directory: str, it: int, splats: SplatSet, history: List[MetricRecord]) -> None:
    base = os.path.join(directory, f"checkpoint_{it:06d}")  # train.hpp:149-165
    try:
        save_splats(base + ".gbil", splats)
        with open(base + ".history.csv", "w") as fh:
            fh.write("iter,loss,psnr\n")
            for r in history:
                fh.write("%d,%.17g,%.17g\n" % (r.iter, r.loss, r.psnr))  # train.hpp:149-165 writes %.17g
    except Exception as e:  # noqa: BLE001
        raise FitError(f"checkpoint write failed: {e}") from e


def fit(target: torch.Tensor, cfg: TrainConfig) -> FitResult:
    """train.hpp:174-219 on the GPU.  target: (H, W, 3) float tensor (moved to CUDA)."""
    cfg.validate()
    target = _img(torch.as_tensor(target, dtype=torch.float32)).cuda() if not target.is_cuda else _img(
        target.float())
    H, W = int(target.shape[0]), int(target.shape[1])
    if cfg.loss == LossKind.mse_plus_ssim and (W < 11 or H < 11):
        raise ValueError("fit: mse_plus_ssim needs images of at least 11x11")
    if W < 1 or H < 1:
        raise ValueError("ImagePlaneCamera: width and height must be >= 1")
    camera = ImagePlaneCamera(W, H, cfg.background)
    lrs = copy.copy(cfg.lrs)
    if not cfg.position_lr_absolute:
        lrs.position *= max(W, H)
    splats = initialize(W, H, cfg, device=target.device)
    state = AdamState(splats, cfg.adam)
    grads = GradientBuffer(splats)
    binning = TileBinning(target.device)
    out = RenderOutput(W, H, target.device)
    gimg = torch.empty_like(target)
    history: List[MetricRecord] = []
    start = time.perf_counter()
    for it in range(1, cfg.iterations + 1):
        build_binning(splats, camera, cfg.raster, out=binning)
        render_forward(splats, camera, binning, out)
        loss, gimg = photometric_loss(out.color, target, cfg, grad=gimg)
        value = float(loss)
        if not math.isfinite(value):
            raise FitError(f"fit: non-finite loss at iteration {it}; last checkpoint retained")
        grads.zero_()
        render_backward(splats, camera, binning, out, gimg, grads)
        adam_step(splats, grads, state, lrs)
        if it == 1 or it == cfg.iterations or it % cfg.log_every == 0:
            rec = MetricRecord(iter=it, loss=value, psnr=psnr(out.color, target),
                               ssim=ssim(out.color, target) if (W >= 11 and H >= 11) else float("nan"))
            torch.cuda.synchronize(target.device)
            rec.wall_ms = (time.perf_counter() - start) * 1e3
            history.append(rec)
        if cfg.checkpoint_every > 0 and cfg.checkpoint_dir and (it % cfg.checkpoint_every == 0 or
                                                                 it == cfg.iterations):
            _write_checkpoint(cfg.checkpoint_dir, it, splats, history)
    return FitResult(splats, history)
