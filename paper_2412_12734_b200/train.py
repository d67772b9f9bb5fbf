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
                     TileBinning, adam_step, all_contexts, build_binning, l1_loss, render_backward,
                     render_forward)


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


class _Lane:
    """One view pipeline: a CUDA stream (hence its own C-ABI context and scratch), a binning,
    output and cotangent buffers.  View i of a step runs on lane i % lanes."""

    def __init__(self, device, stream):
        self.stream = stream
        with torch.cuda.stream(stream):
            self.binning = TileBinning(device)
        self.outs = {}
        self.done = torch.cuda.Event()


class ViewShardedTrainer:
    """configs[3] step: per owned view K1..K6 + K4/K5 into one gradient buffer, one all-reduce, Adam.

    Views alternate between `lanes` streams, so the binning of view i+1 (whose pair count
    the host must read back) and its small sort/scan kernels overlap the compositors of view
    i instead of leaving the GPU idle at the host synchronisation point.  All lanes add into
    the same gradient buffer with atomics; the step joins them before the all-reduce."""

    def __init__(self, splats: SplatSet, cameras: Sequence, views: Sequence[int], lrs: LearningRates = None,
                 adam: AdamConfig = None, raster: RasterConfig = None, process_group=None, check_finite=False,
                 lanes: int = 2):
        self.splats = splats
        self.cameras = list(cameras)
        self.views = list(views)
        self.lrs = lrs or LearningRates()
        self.raster = raster or RasterConfig()
        self.grads = GradientBuffer(splats)
        self.state = AdamState(splats, adam)
        self.pg = process_group
        self.check_finite = check_finite
        dev = splats.device
        main = torch.cuda.current_stream(dev)
        self._lanes = [_Lane(dev, main if i == 0 else torch.cuda.Stream(device=dev)) for i in range(max(1, lanes))]
        self.binning = self._lanes[0].binning
        W = max(self.cameras[v].width for v in self.views) if self.views else 1
        H = max(self.cameras[v].height for v in self.views) if self.views else 1
        self.losses = torch.zeros(max(1, len(self.views)), dtype=torch.float32, device=dev)
        self._pinned_losses = torch.zeros(max(1, len(self.views)), dtype=torch.float32, pin_memory=True)
        self._target_buf = [torch.empty((H, W, 3), dtype=torch.float32, device=dev) for _ in range(2)]
        self._copy_stream = torch.cuda.Stream(device=dev)
        self._copy_done = [torch.cuda.Event() for _ in range(2)]
        self._buf_free = [torch.cuda.Event() for _ in range(2)]
        self._step_start = torch.cuda.Event()
        self.pairs: List[int] = []  # tile/primitive pair count P of every view binned (roofline bytes)

    def _out(self, lane: _Lane, cam):
        key = (cam.width, cam.height)
        if key not in lane.outs:
            with torch.cuda.stream(lane.stream):
                lane.outs[key] = (RenderOutput(cam.width, cam.height, self.splats.device),
                                  torch.empty((cam.height, cam.width, 3), dtype=torch.float32,
                                              device=self.splats.device))
        return lane.outs[key]

    def _lane(self, i: int) -> _Lane:
        return self._lanes[i % len(self._lanes)]

    def _view_forward(self, i: int):
        lane = self._lane(i)
        cam = self.cameras[self.views[i]]
        out, gimg = self._out(lane, cam)
        build_binning(self.splats, cam, self.raster, out=lane.binning)
        self.pairs.append(lane.binning.total)
        render_forward(self.splats, cam, lane.binning, out)
        return cam, out, gimg

    def _view_backward(self, i: int, cam, out, gimg, target: torch.Tensor) -> None:
        lane = self._lane(i)
        l1_loss(out.color, target.view(cam.height, cam.width, 3), grad=gimg, loss=self.losses[i:i + 1])
        render_backward(self.splats, cam, lane.binning, out, gimg, self.grads)

    def _begin(self) -> None:
        main = self._lanes[0].stream
        self.grads.zero_()
        self.losses.zero_()
        self._step_start.record(main)
        for lane in self._lanes[1:]:
            lane.stream.wait_event(self._step_start)  # parameters updated and gradients zeroed

    def _join(self) -> None:
        main = self._lanes[0].stream
        for lane in self._lanes[1:]:
            lane.done.record(lane.stream)
            main.wait_event(lane.done)

    def _finish(self) -> None:
        self._join()
        reduce_gradients(self.grads, self.pg)
        adam_step(self.splats, self.grads, self.state, self.lrs, check_finite=self.check_finite)

    def step(self, targets: Sequence[torch.Tensor]) -> torch.Tensor:
        """One training step with device-resident per-view targets; returns the device loss vector."""
        self._begin()
        for i in range(len(self.views)):
            with torch.cuda.stream(self._lane(i).stream):
                cam, out, gimg = self._view_forward(i)
                self._view_backward(i, cam, out, gimg, targets[i])
        self._finish()
        return self.losses

    def step_host(self, targets_host: Sequence[torch.Tensor]) -> torch.Tensor:
        """End-to-end step from pinned HOST targets: the H2D copy of view i+1 overlaps the
        compute of view i on a side stream, and a view's own copy only has to land before its
        loss (binning and forward do not read the target); the per-view losses are read back."""
        main = self._lanes[0].stream
        self._begin()
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
            self._buf_free[b].record(main)
        if n:
            issue(0)
        for i in range(n):
            b = i % 2
            if i + 1 < n:
                issue(i + 1)
            s = self._lane(i).stream
            with torch.cuda.stream(s):
                cam, out, gimg = self._view_forward(i)
                s.wait_event(self._copy_done[b])
                self._view_backward(i, cam, out, gimg,
                                    self._target_buf[b].view(-1)[: cam.height * cam.width * 3])
                self._buf_free[b].record(s)
        self._finish()
        self._pinned_losses.copy_(self.losses, non_blocking=True)
        main.synchronize()
        return self._pinned_losses

    def launches(self) -> int:
        return sum(c.launches() for c in all_contexts(self.splats.device))
