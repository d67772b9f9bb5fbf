"""View-sharded multi-view training step (BASELINE.json configs[3]).

Each rank owns a fixed subset of camera views and replicated primitives.  Per
step and per owned view it runs, on one CUDA stream, K1 projection -> K2 tile
binning -> K3 forward -> K6 L1 loss -> K4/K5 backward, accumulating into one
flat fp32 gradient buffer; then ONE collective (NCCL all-reduce, sum) makes
the gradients identical on every rank and K7 Adam updates the replicated
parameters.  This is the only cross-GPU exchange of the path.

The reference's driver loop (train.hpp:174-219, ``fit``) is single-image and
single-process; this step is its multi-view, multi-GPU generalisation for the
BASELINE configs (L1 loss, Adam with the reference's defaults, optim.hpp).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from .raster import (AdamConfig, AdamState, GradientBuffer, LearningRates, RasterConfig, RenderOutput, SplatSet,
                     TileBinning, adam_step, build_binning, context, l1_loss, render_backward, render_forward)


def shard_views(n_views: int, rank: int, world: int, per_rank: Optional[int] = None) -> List[int]:
    """Views owned by `rank`.  per_rank fixes the count per GPU (weak scaling);
    otherwise the n_views are split into contiguous near-equal blocks (strong scaling)."""
    if per_rank is not None:
        return [(rank * per_rank + i) % n_views for i in range(per_rank)]
    lo = n_views * rank // world
    hi = n_views * (rank + 1) // world
    return list(range(lo, hi))


def reduce_gradients(grads: GradientBuffer, process_group=None) -> None:
    """The step's one collective: sum the flat gradient buffer over all ranks (NCCL on GPUs)."""
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        if torch.distributed.get_world_size(process_group) > 1:
            torch.distributed.all_reduce(grads.flat, op=torch.distributed.ReduceOp.SUM, group=process_group)


class ViewShardedTrainer:
    def __init__(self, splats: SplatSet, cameras: Sequence, views: Sequence[int], lrs: LearningRates = None,
                 adam: AdamConfig = None, raster: RasterConfig = None, process_group=None, check_finite=False):
        self.splats = splats
        self.cameras = list(cameras)
        self.views = list(views)
        self.lrs = lrs or LearningRates()
        self.raster = raster or RasterConfig()
        self.grads = GradientBuffer(splats)
        self.state = AdamState(splats, adam)
        self.binning = TileBinning(splats.device)
        self.pg = process_group
        self.check_finite = check_finite
        dev = splats.device
        W = max(self.cameras[v].width for v in self.views) if self.views else 1
        H = max(self.cameras[v].height for v in self.views) if self.views else 1
        self._outs = {}
        self._grad_img = {}
        self.losses = torch.zeros(max(1, len(self.views)), dtype=torch.float32, device=dev)
        self._pinned_losses = torch.zeros(max(1, len(self.views)), dtype=torch.float32, pin_memory=True)
        self._target_buf = [torch.empty((H, W, 3), dtype=torch.float32, device=dev) for _ in range(2)]
        self._copy_stream = torch.cuda.Stream(device=dev)
        self._copy_done = [torch.cuda.Event() for _ in range(2)]
        self._buf_free = [torch.cuda.Event() for _ in range(2)]
        self.pairs: List[int] = []  # tile/primitive pair count P of every view binned (roofline bytes)

    def _out(self, cam):
        key = (cam.width, cam.height)
        if key not in self._outs:
            self._outs[key] = RenderOutput(cam.width, cam.height, self.splats.device)
            self._grad_img[key] = torch.empty((cam.height, cam.width, 3), dtype=torch.float32,
                                              device=self.splats.device)
        return self._outs[key], self._grad_img[key]

    def _view_forward(self, i: int):
        cam = self.cameras[self.views[i]]
        out, gimg = self._out(cam)
        build_binning(self.splats, cam, self.raster, out=self.binning)
        self.pairs.append(self.binning.total)
        render_forward(self.splats, cam, self.binning, out)
        return cam, out, gimg

    def _view_backward(self, i: int, cam, out, gimg, target: torch.Tensor) -> None:
        l1_loss(out.color, target.view(cam.height, cam.width, 3), grad=gimg, loss=self.losses[i:i + 1])
        render_backward(self.splats, cam, self.binning, out, gimg, self.grads)

    def _view(self, i: int, target: torch.Tensor) -> None:
        self._view_backward(i, *self._view_forward(i), target)

    def _finish(self) -> None:
        reduce_gradients(self.grads, self.pg)
        adam_step(self.splats, self.grads, self.state, self.lrs, check_finite=self.check_finite)

    def step(self, targets: Sequence[torch.Tensor]) -> torch.Tensor:
        """One training step with device-resident per-view targets; returns the device loss vector."""
        self.grads.zero_()
        self.losses.zero_()
        for i in range(len(self.views)):
            self._view(i, targets[i])
        self._finish()
        return self.losses

    def step_host(self, targets_host: Sequence[torch.Tensor]) -> torch.Tensor:
        """End-to-end step from pinned HOST targets: the H2D copy of view i+1 overlaps the
        compute of view i on a side stream, and a view's own copy only has to land before its
        loss (binning and forward do not read the target); the per-view losses are read back."""
        cur = torch.cuda.current_stream(self.splats.device)
        self.grads.zero_()
        self.losses.zero_()
        n = len(self.views)

        def issue(i):
            b = i % 2
            with torch.cuda.stream(self._copy_stream):
                self._copy_stream.wait_event(self._buf_free[b])
                t = targets_host[i]
                dst = self._target_buf[b].view(-1)[: t.numel()]
                dst.copy_(t.view(-1), non_blocking=True)
                self._copy_done[b].record(self._copy_stream)

        for b in range(2):
            self._buf_free[b].record(cur)
        if n:
            issue(0)
        for i in range(n):
            b = i % 2
            if i + 1 < n:
                issue(i + 1)
            cam, out, gimg = self._view_forward(i)
            cur.wait_event(self._copy_done[b])
            self._view_backward(i, cam, out, gimg, self._target_buf[b].view(-1)[: cam.height * cam.width * 3])
            self._buf_free[b].record(cur)
        self._finish()
        self._pinned_losses.copy_(self.losses, non_blocking=True)
        cur.synchronize()
        return self._pinned_losses

    def launches(self) -> int:
        return context(self.splats.device).launches()
