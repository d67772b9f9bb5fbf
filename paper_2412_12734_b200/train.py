"""View-sharded multi-view training step (BASELINE.json configs[3]).

Each rank owns a fixed subset of camera views and replicated primitives.  Per
step and per owned view it runs K1 projection -> K2 tile binning -> K3 forward
-> K6 L1 loss -> K4 backward -> K5 through the reference-shaped calls
(``fused=True``: gb_render_loss_backward, K3 with the loss in its epilogue),
accumulating into one flat fp32 gradient buffer.  Then the gradients are
reduce-scattered (NCCL), each rank runs K7 Adam on its 1/world slice of the
flat parameter buffer, and the parameters are all-gathered
(``sharded_adam=False``: one all-reduce and a replicated Adam instead).  These
collectives are the only cross-GPU exchange of the path.

The reference's driver loop (train.hpp:174-219, ``fit``) is single-image and
single-process; this step is its multi-view, multi-GPU generalisation for the
BASELINE configs (L1 loss, Adam with the reference's defaults, optim.hpp).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import torch

from . import _lib
from ._lib import check, lib

from .raster import (AdamConfig, AdamState, GradientBuffer, LearningRates, RasterConfig, RenderOutput, SplatSet,
                     StepGraph, TileBinning, adam_step, all_contexts, build_binning, context, l1_loss,
                     copy_h2d, memset_, render_backward, render_forward, render_loss_backward, texel_grads_unpad,
                     texels_pad)


def shard_views(n_views: int, rank: int, world: int, per_rank: Optional[int] = None) -> List[int]:
    """Views owned by `rank`.  per_rank fixes the count per GPU (weak scaling);
    otherwise the n_views are split into contiguous near-equal blocks (strong scaling)."""
    if per_rank is not None:
        return [(rank * per_rank + i) % n_views for i in range(per_rank)]
    lo = n_views * rank // world
    hi = n_views * (rank + 1) // world
    return list(range(lo, hi))


class Communicator:
    """The step's NCCL communicator, created and driven through the C-ABI (gb_comm_init_rank,
    gb_allreduce_grads, gb_reduce_scatter_grads, gb_all_gather_params, gb_allreduce_flag_min) on the
    current stream's context; only its unique id travels over the torch process group."""

    def __init__(self, device, process_group=None):
        dist = torch.distributed
        self.world = dist.get_world_size(process_group)
        self.rank = dist.get_rank(process_group)
        uid = (C.c_uint8 * _lib.COMM_ID_BYTES)()
        if self.rank == 0:
            check(lib.gb_comm_unique_id(uid), "gb_comm_unique_id")
        obj = [bytes(uid)]
        src = 0 if process_group is None else dist.get_global_rank(process_group, 0)
        dist.broadcast_object_list(obj, src=src, group=process_group)
        uid = (C.c_uint8 * _lib.COMM_ID_BYTES).from_buffer_copy(obj[0])
        h = C.c_void_p()
        check(lib.gb_comm_init_rank(context(device).handle, self.world, uid, self.rank, C.byref(h)),
              "gb_comm_init_rank")
        self.handle = h

    @staticmethod
    def wanted(process_group=None) -> bool:
        """NCCL through the C-ABI when the ranks are CUDA processes (backend nccl); gloo/fake groups (CPU
        tests, code-path checks) keep torch.distributed's collectives."""
        dist = torch.distributed
        return (dist.is_available() and dist.is_initialized() and dist.get_world_size(process_group) > 1
                and dist.get_backend(process_group) == "nccl")

    def all_reduce(self, t: torch.Tensor) -> None:
        check(lib.gb_allreduce_grads(context(t.device).handle, self.handle, t.data_ptr(), t.numel()),
              "gb_allreduce_grads")

    def reduce_scatter(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        check(lib.gb_reduce_scatter_grads(context(out.device).handle, self.handle, inp.data_ptr(), out.data_ptr(),
                                          out.numel()), "gb_reduce_scatter_grads")

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        check(lib.gb_all_gather_params(context(out.device).handle, self.handle, inp.data_ptr(), out.data_ptr(),
                                       inp.numel()), "gb_all_gather_params")

    def min_flag(self, flag: torch.Tensor) -> None:
        check(lib.gb_allreduce_flag_min(context(flag.device).handle, self.handle, flag.data_ptr()),
              "gb_allreduce_flag_min")

    def close(self) -> None:
        if self.handle:
            lib.gb_comm_destroy(self.handle)
            self.handle = None


def reduce_gradients(grads: GradientBuffer, process_group=None, comm: "Communicator" = None) -> None:
    """The step's one collective: sum the flat gradient buffer over all ranks (NCCL on GPUs)."""
    if comm is not None:
        comm.all_reduce(grads.flat)
        return
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        if torch.distributed.get_world_size(process_group) > 1:
            torch.distributed.all_reduce(grads.flat, op=torch.distributed.ReduceOp.SUM, group=process_group)


PAIR_LIMIT = 2 ** 31 - 1  # the binning's pair-count limit (gb_binning.cu kPairLimit; capacities stay below it)

_ADAM_GROUP = {"position": 0, "theta": 1, "quat": 1, "log_scale": 2, "opacity_logit": 3, "grid": 4}


class ShardedAdam:
    """The step's optimiser over ranks (SURVEY §8(e) variant): reduce-scatter the flat gradient buffer,
    Adam on this rank's 1/world slice of a flat parameter buffer (gb_adam_segments), all-gather the
    parameters.  The collective moves the same bytes as one all-reduce, but each rank updates and keeps
    moments for 1/world of the parameters.  The non-finite guard (optim.hpp:81-83) is agreed across ranks
    (min-reduced flag) before anything is updated.  At world size 1 it is the grouped Adam on one slice.

    The splats' parameter tensors become views into ``flat`` (same layout as the gradient buffer)."""

    def __init__(self, splats: SplatSet, grads: GradientBuffer, state: AdamState, process_group=None,
                 segment_update=None, comm: "Communicator" = None):
        """``segment_update(phase, ranges, state, lrs, flag)``: replaces the gb_adam_segments call --
        a hook for the multi-process CPU tests only (there is no CPU optimiser in the product)."""
        dist = torch.distributed
        self._hook = segment_update
        self.pg = process_group
        self.comm = comm
        self.world = dist.get_world_size(process_group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(process_group) if self.world > 1 else 0
        if grads.flat.numel() % (4 * self.world):
            raise ValueError("ShardedAdam: gradient buffer not padded to 4 * world elements")
        self.splats, self.grads, self.state = splats, grads, state
        self.flat = torch.zeros_like(grads.flat)
        for f, (o, n) in grads.offsets.items():
            t = getattr(splats, f)
            v = self.flat[o:o + n].view(t.shape)
            v.copy_(t)
            setattr(splats, f, v)
        S = self.flat.numel() // self.world
        self.lo, self.S = self.rank * S, S
        dev = grads.flat.device
        self.g_shard = grads.flat if self.world == 1 else torch.empty(S, dtype=torch.float32, device=dev)
        self.m = torch.zeros(S, dtype=torch.float32, device=dev)
        self.v = torch.zeros(S, dtype=torch.float32, device=dev)
        self.flag = torch.empty(1, dtype=torch.int64, device=dev)
        self._veto = torch.full((1,), self.VETO, dtype=torch.int64, device=dev)
        segs = []
        self.ranges = []  # (flat lo, flat hi, group) of this rank's slice
        gbase = self.lo if self.world > 1 else 0  # g_shard: this rank's slice, or (one rank) the whole buffer
        for f, (o, n) in grads.offsets.items():
            if f == "depth_key":  # never updated (optim.hpp:95)
                continue
            a, b = max(o, self.lo), min(o + n, self.lo + S)
            if a >= b:
                continue
            self.ranges.append((a, b, _ADAM_GROUP[f]))
            segs.append(_lib.AdamSegment(self.flat.data_ptr() + 4 * a, self.g_shard.data_ptr() + 4 * (a - gbase),
                                         self.m.data_ptr() + 4 * (a - self.lo), self.v.data_ptr() + 4 * (a - self.lo),
                                         b - a, _ADAM_GROUP[f], 0))
        self._segs = (_lib.AdamSegment * max(1, len(segs)))(*segs)
        self._nseg = len(segs)
        grid = [sg for sg in segs if sg.group == 4]
        other = [sg for sg in segs if sg.group != 4]
        self._grid_segs = (_lib.AdamSegment * len(grid))(*grid) if grid else None
        self._other_segs = (_lib.AdamSegment * max(1, len(other)))(*other)
        self._names = [f for f in grads.offsets if f != "depth_key"]

    VETO = _lib.ADAM_FLAG_VETO  # flag value of a vetoed step: below every clear value, above every non-finite
    # code (group <= 4), so a non-finite gradient still wins the min-reduction

    def step(self, lrs: LearningRates, check_finite: bool = False, grid_stream=None, grid_done=None,
             veto: torch.Tensor = None) -> None:
        """One update.  With ``grid_stream`` (world size 1): the texel segment is updated on that stream
        (after the non-finite scan of every segment) and ``grid_done`` is recorded there -- the next
        step's binning overlaps the texel update."""
        from .raster import context
        from ._lib import check, lib

        dist = torch.distributed
        if self.world > 1:
            if self.comm is not None:
                self.comm.reduce_scatter(self.g_shard, self.grads.flat)
            else:
                dist.reduce_scatter_tensor(self.g_shard, self.grads.flat, op=dist.ReduceOp.SUM, group=self.pg)
        if self._hook is not None:  # CPU test stand-in (gloo): torch ops on host tensors
            self.flag.fill_(_lib.ADAM_FLAG_CLEAR)
            self._hook(0, self, lrs)
            if veto is not None:  # veto (an int32, nonzero = skip the update on every rank)
                self.flag.copy_(torch.where(veto.to(torch.int64) != 0, self._veto, self.flag))
            if self.world > 1:
                dist.all_reduce(self.flag, op=dist.ReduceOp.MIN, group=self.pg)
            self._hook(1, self, lrs)
        else:
            ctx = context(self.flat.device)
            st = self.state.to_c()
            c_lrs = lrs.to_c()
            # flag = VETO if the view work vetoed the step (a binning overflow), else CLEAR; phase 0 lowers it
            # to the first non-finite gradient's code
            check(lib.gb_adam_flag_init(ctx.handle, self.flag.data_ptr(),
                                        None if veto is None else veto.data_ptr()), "gb_adam_flag_init")
            check(lib.gb_adam_segments(ctx.handle, 0, self._segs, self._nseg, C.byref(st), C.byref(c_lrs),
                                       self.flag.data_ptr()), "adam_step")
            if self.world > 1:
                if self.comm is not None:
                    self.comm.min_flag(self.flag)
                else:
                    dist.all_reduce(self.flag, op=dist.ReduceOp.MIN, group=self.pg)
            if grid_stream is None or self.world > 1 or not self._grid_segs:
                check(lib.gb_adam_segments(ctx.handle, 1, self._segs, self._nseg, C.byref(st), C.byref(c_lrs),
                                           self.flag.data_ptr()), "adam_step")
            else:
                t0 = st.t
                check(lib.gb_adam_segments(ctx.handle, 1, self._other_segs, len(self._other_segs), C.byref(st),
                                           C.byref(c_lrs), self.flag.data_ptr()), "adam_step")
                st_g = self.state.to_c()
                st_g.t = t0  # the same step number for the texel segment
                cur = torch.cuda.current_stream(self.flat.device)
                grid_stream.wait_stream(cur)
                with torch.cuda.stream(grid_stream):
                    gctx = context(self.flat.device)
                    check(lib.gb_adam_segments(gctx.handle, 1, self._grid_segs, len(self._grid_segs),
                                               C.byref(st_g), C.byref(c_lrs), self.flag.data_ptr()), "adam_step")
                    grid_done.record(grid_stream)
            self.state.t = st.t
        if self.world > 1:
            if self.comm is not None:
                self.comm.all_gather(self.flat, self.flat[self.lo:self.lo + self.S])
            else:
                dist.all_gather_into_tensor(self.flat, self.flat[self.lo:self.lo + self.S], group=self.pg)
        if check_finite:
            self.raise_if_nonfinite(int(self.flag.item()))

    @staticmethod
    def raise_if_nonfinite(v: int) -> None:
        if v != _lib.ADAM_FLAG_CLEAR and v != ShardedAdam.VETO:
            grp = v >> 48
            names = ("position", "theta", "log_scale", "opacity_logit", "color_grid")
            raise _lib.NonFinite(_lib.GB_NONFINITE, "adam_step",
                                 f"non-finite gradient in group '{names[grp & 7]}' "
                                 f"(segment index {v & ((1 << 48) - 1)}); no parameter was updated")


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
                 lanes: int = 6, fused: bool = False, async_binning: bool = True, graph: bool = False,
                 capacity_margin: float = 1.1, sharded_adam: bool = True, overlap_adam: bool = True,
                 texel_pad: bool = True, rgba_texels: bool = True):
        self.splats = splats
        self.cameras = list(cameras)
        self.views = list(views)
        self.lrs = lrs or LearningRates()
        self.raster = raster or RasterConfig()
        self.pg = process_group
        dist = torch.distributed
        world = dist.get_world_size(process_group) if dist.is_available() and dist.is_initialized() else 1
        self.grads = GradientBuffer(splats, multiple=4 * world)
        # sharded optimiser (reduce-scatter, Adam on 1/world of the parameters, all-gather) or the
        # replicated one (all-reduce, full Adam on every rank)
        self.state = AdamState(splats, adam, moments=not sharded_adam)
        # the gradient exchange runs through the C-ABI's NCCL layer on CUDA ranks (torch's for gloo/fake)
        self.comm = Communicator(splats.device, process_group) if Communicator.wanted(process_group) else None
        self.opt = (ShardedAdam(splats, self.grads, self.state, process_group, comm=self.comm) if sharded_adam
                    else None)
        # world size 1: the texel half of Adam (90 % of it) runs on a side stream and overlaps the next
        # step's binning; each lane waits for it (and the texel-gradient zeroing that follows it) before
        # its first forward compositor.  Texels read on another stream right after step() returns need
        # torch.cuda.synchronize() or wait_adam().
        self.overlap_adam = bool(overlap_adam and self.opt is not None and self.opt.world == 1)
        self.overlap_read = True  # step(): the overflow read after Adam is queued (overlap_adam only)
        self._adam_stream = torch.cuda.Stream(device=splats.device) if self.overlap_adam else None
        self._grid_done = torch.cuda.Event() if self.overlap_adam else None  # texel update finished
        self._grid_ready = torch.cuda.Event() if self.overlap_adam else None  # ... and its gradients zeroed
        if self.overlap_adam:
            self._grid_done.record(self._adam_stream)  # exists (and is complete) before the first wait
        self.check_finite = check_finite
        self.fused = fused
        dev = splats.device
        # the views' K4s add texel gradients into an RGBA-padded scratch (one 16-B red per texel), converted into
        # the flat buffer's reference-layout grid group once per step (gb_texel_grads_unpad)
        self._tex_pad = (torch.zeros(self.grads.grid.numel() // 3 * 4, dtype=torch.float32, device=dev)
                         if texel_pad else None)
        # ... and the compositors read the texels from an RGBA-padded copy (one 16-B load per texel), refreshed
        # once per step after the texel update (gb_texels_pad; rgba_texels needs texel_pad)
        self._tex_rgba = (torch.zeros(self.grads.grid.numel() // 3 * 4, dtype=torch.float32, device=dev)
                          if texel_pad and rgba_texels else None)
        # lane 0 is the caller's stream, except under graph capture (which needs a side stream)
        main = torch.cuda.Stream(device=dev) if graph else torch.cuda.current_stream(dev)
        self._lanes = [_Lane(dev, main if i == 0 else torch.cuda.Stream(device=dev)) for i in range(max(1, lanes))]
        self.binning = self._lanes[0].binning
        W = max(self.cameras[v].width for v in self.views) if self.views else 1
        H = max(self.cameras[v].height for v in self.views) if self.views else 1
        self.losses = torch.zeros(max(1, len(self.views)), dtype=torch.float32, device=dev)
        self._pinned_losses = torch.zeros(max(1, len(self.views)), dtype=torch.float32, pin_memory=True)
        self._pinned_flag = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        # two target buffers per view lane: every lane's view can have its target landed while the copy stream
        # runs ahead (with two buffers for four lanes, lanes 3-4 had waited for a free buffer)
        nbuf = 2 * len(self._lanes)
        self._target_buf = [torch.empty((H, W, 3), dtype=torch.float32, device=dev) for _ in range(nbuf)]
        self._copy_stream = torch.cuda.Stream(device=dev)
        self._copy_done = [torch.cuda.Event() for _ in range(nbuf)]
        self._buf_free = [torch.cuda.Event() for _ in range(nbuf)]
        self._step_start = torch.cuda.Event()
        self.pairs: List[int] = []  # blocking mode: pair count P of every view binned (roofline bytes)
        # capacity mode (async_binning): after one blocking step sizes the pair buffers, builds never read P
        # back; a device flag reports a view that outgrew them and the step is redone with more room
        self.async_binning = async_binning
        self.capacity_margin = capacity_margin
        self.capacity = 0
        self._overflow = torch.zeros(1, dtype=torch.int32, device=dev)
        self._pair_counts = torch.zeros(max(1, len(self.views)), dtype=torch.int32, device=dev)
        self.use_graph = graph
        self.graph_host = False  # step_host views as a graph too (H2D copies as memcpy nodes)
        self._graph = None
        self._graph_key = None
        self._graphs = {}  # key (input buffers) -> graph, for the current capacity
        self.overflows = 0

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
        if self.capacity:
            lane.binning.store_total(self._pair_counts[i:i + 1])
        else:
            self.pairs.append(lane.binning.total)
        if self.overlap_adam and id(lane) not in self._waited:  # texels updated, their gradients zeroed
            self._waited.add(id(lane))
            lane.stream.wait_event(self._grid_ready)
        if not self.fused:
            render_forward(self.splats, cam, lane.binning, out, texels_rgba=self._tex_rgba)
        return cam, out, gimg

    def _view_backward(self, i: int, cam, out, gimg, target: torch.Tensor) -> None:
        lane = self._lane(i)
        if self.fused:
            render_loss_backward(self.splats, cam, lane.binning, target, "l1", grads=self.grads,
                                 loss_acc=self.losses[i:i + 1], texel_grad=self._tex_pad, texels_rgba=self._tex_rgba)
            return
        l1_loss(out.color, target.view(cam.height, cam.width, 3), grad=gimg, loss=self.losses[i:i + 1])
        render_backward(self.splats, cam, lane.binning, out, gimg, self.grads, texel_grad=self._tex_pad,
                        texels_rgba=self._tex_rgba)

    def wait_adam(self) -> None:
        """Order the current stream after the step's texel update (overlap_adam)."""
        if self.overlap_adam:
            torch.cuda.current_stream(self.splats.device).wait_event(self._grid_done)

    def _begin(self) -> None:
        main = self._lanes[0].stream
        if self.overlap_adam:
            o, _ = self.grads.offsets["grid"]
            memset_(self.grads.flat[:o])
        else:
            memset_(self.grads.flat)
        if self._tex_pad is not None:
            memset_(self._tex_pad)
        memset_(self.losses)
        if self._tex_rgba is not None and not self.overlap_adam:
            texels_pad(self.splats.grid.view(-1), self._tex_rgba)  # (the last step's Adam ran on this stream)
        self._step_start.record(main)
        for lane in self._lanes[1:]:
            lane.stream.wait_event(self._step_start)  # parameters updated and gradients zeroed
        if self.overlap_adam:
            # side stream: after the previous step's texel update (recorded outside any graph), zero the
            # texel gradients; lanes wait for that only before their first forward compositor
            a = self._adam_stream
            a.wait_event(self._step_start)
            with torch.cuda.stream(a):
                check(lib.gb_stream_wait_event(context(self.splats.device).handle,
                                               C.c_void_p(self._grid_done.cuda_event), 1), "gb_stream_wait_event")
                if self._tex_pad is None:  # (padded: the grid group is overwritten by the unpad at the join)
                    memset_(self.grads.grid)
                if self._tex_rgba is not None:
                    texels_pad(self.splats.grid.view(-1), self._tex_rgba)
                self._grid_ready.record(a)
            self._waited = set()

    def _join(self) -> None:
        main = self._lanes[0].stream
        for lane in self._lanes[1:]:
            lane.done.record(lane.stream)
            main.wait_event(lane.done)
        if self.overlap_adam:
            main.wait_event(self._grid_ready)  # the side stream rejoins (a graph capture needs it)
        if self._tex_pad is not None:  # after the previous step's texel update read the grid group
            texel_grads_unpad(self._tex_pad, self.grads.grid.view(-1), accumulate=False)

    def _on_lanes(self, body) -> None:
        """Run body() with lane 0 as the current stream, ordered after and before the caller's stream."""
        cur = torch.cuda.current_stream(self.splats.device)
        main = self._lanes[0].stream
        if cur == main:
            body()
            return
        main.wait_stream(cur)
        with torch.cuda.stream(main):
            body()
        cur.wait_stream(main)

    def _views(self, targets: Sequence[torch.Tensor]) -> None:
        def body():
            self._begin()
            for i in range(len(self.views)):
                with torch.cuda.stream(self._lane(i).stream):
                    cam, out, gimg = self._view_forward(i)
                    self._view_backward(i, cam, out, gimg, targets[i])
            self._join()

        self._on_lanes(body)

    def _set_capacity(self, pairs_max: int, exact: bool = False) -> None:
        if pairs_max >= PAIR_LIMIT:
            raise RuntimeError(f"view binning needs {pairs_max} tile/primitive pairs, more than the "
                               f"{PAIR_LIMIT - 1} the sorts index")
        cap = pairs_max if exact else ((int(pairs_max * self.capacity_margin) + 4096 + 65535) & ~65535)
        cap = min(cap, PAIR_LIMIT - 1)  # the margin never pushes the capacity past the C-ABI's limit
        for lane in self._lanes:
            lane.binning.set_capacity(cap, self._overflow)
        self.capacity = cap
        self._graph, self._graph_key = None, None
        self._graphs = {}

    def _views_checked(self, run) -> None:
        """All owned views into the gradient buffer (run()); in capacity mode redone with larger pair
        buffers when a view outgrew them (the flag is read once per step, before the collective and Adam)."""
        if self.async_binning and not self.capacity:
            n0 = len(self.pairs)
            run()  # blocking builds: learn the pair counts
            self._set_capacity(max(self.pairs[n0:]) if len(self.pairs) > n0 else 0)
            return
        for attempt in range(4):
            run()
            if not self.capacity or not int(self._overflow.item()):
                break
            self.overflows += 1
            memset_(self._overflow)
            need = int((self._pair_counts[: len(self.views)].to(torch.int64) & 0xFFFFFFFF).max().item())  # uint32
            self._set_capacity(need)
        else:
            raise RuntimeError("view binning kept outgrowing its pair capacity")

    def _run_views(self, targets: Sequence[torch.Tensor]) -> None:
        self._run_graphed(lambda: self._views(targets), ("dev",) + tuple(t.data_ptr() for t in targets))

    def _run_host_views(self, targets_host: Sequence[torch.Tensor]) -> None:
        if not self.graph_host:  # measured: the eager H2D pipeline overlaps better than graph memcpy nodes
            self._on_lanes(lambda: self._views_host(targets_host))
            return
        self._run_graphed(lambda: self._on_lanes(lambda: self._views_host(targets_host)),
                          ("host",) + tuple(t.data_ptr() for t in targets_host))

    def _run_graphed(self, fn, key) -> None:
        """fn() eagerly, or -- graph mode with capacity binning -- as a replay of its CUDA graph,
        captured after one eager run (which sizes every buffer) and re-captured when the
        buffers it reads (key) or the pair capacity change."""
        if not (self.use_graph and self.capacity):
            fn()
            return
        if self._graph_key != key and key in self._graphs:
            self._graph, self._graph_key = self._graphs[key], key
        if self._graph is not None and self._graph_key == key:
            self._on_lanes(self._graph.launch)
            return
        fn()
        main = self._lanes[0].stream
        ctxs = []
        for lane in self._lanes + [None]:
            with torch.cuda.stream(lane.stream if lane else self._copy_stream):
                ctxs.append(context(self.splats.device))
        g = StepGraph(ctxs)
        main.wait_stream(torch.cuda.current_stream(self.splats.device))
        with torch.cuda.stream(main):
            g.capture(fn)
        self._graph, self._graph_key = g, key
        if len(self._graphs) >= 4:
            self._graphs.clear()
        self._graphs[key] = g

    def pair_stats(self):
        """(sum of P, views): over the views of the last step in capacity mode (the builds store their pair
        counts on the device; nothing is summed inside the step), else over the views binned since
        reset_pair_stats() (roofline bytes)."""
        if self.capacity:
            nv = len(self.views)
            return int((self._pair_counts[:nv].to(torch.int64) & 0xFFFFFFFF).sum().item()), nv
        return sum(self.pairs), len(self.pairs)

    def reset_pair_stats(self) -> None:
        self.pairs.clear()

    def _finish(self) -> None:
        if self.opt is not None:
            self.opt.step(self.lrs, check_finite=self.check_finite,
                          grid_stream=self._adam_stream, grid_done=self._grid_done)
            return
        reduce_gradients(self.grads, self.pg, self.comm)
        adam_step(self.splats, self.grads, self.state, self.lrs, check_finite=self.check_finite)

    def step(self, targets: Sequence[torch.Tensor]) -> torch.Tensor:
        """One training step with device-resident per-view targets; returns the device loss vector."""
        run = lambda: self._run_views(targets)  # noqa: E731
        if not (self.opt is not None and self.overlap_adam and self.async_binning and self.capacity
                and self.overlap_read):
            self._views_checked(run)
            self._finish()
            return self.losses
        # the step's one host read comes after Adam is queued (its texel half runs on the side stream, so
        # the read waits only for the scan and the small groups): a view that outgrew its pair buffers
        # vetoes the update, and the step is redone with larger buffers
        for _ in range(4):
            run()
            self.opt.step(self.lrs, check_finite=False, grid_stream=self._adam_stream, grid_done=self._grid_done,
                          veto=self._overflow)
            code = int(self.opt.flag.item())
            if code != ShardedAdam.VETO:
                break
            self.state.t -= 1  # nothing was updated
            self._grow_after_overflow()
        else:
            raise RuntimeError("view binning kept outgrowing its pair capacity")
        if self.check_finite:
            ShardedAdam.raise_if_nonfinite(code)
        return self.losses

    def _grow_after_overflow(self) -> None:
        self.overflows += 1
        if int(self._overflow.item()):
            need = int((self._pair_counts[: len(self.views)].to(torch.int64) & 0xFFFFFFFF).max().item())  # uint32
            memset_(self._overflow)
            self._set_capacity(need)

    def step_host(self, targets_host: Sequence[torch.Tensor]) -> torch.Tensor:
        """End-to-end step from pinned HOST targets: the H2D copy of view i+1 overlaps the
        compute of view i on a side stream, and a view's own copy only has to land before its
        loss (binning and forward do not read the target); the per-view losses are read back."""
        cur = torch.cuda.current_stream(self.splats.device)
        run = lambda: self._run_host_views(targets_host)  # noqa: E731
        if not (self.opt is not None and self.overlap_adam and self.async_binning and self.capacity
                and self.overlap_read):
            self._views_checked(run)
            self._finish()
            self._pinned_losses.copy_(self.losses, non_blocking=True)
            cur.synchronize()
            return self._pinned_losses
        # as step(): one read after Adam is queued -- the losses and the optimiser's agreed flag together
        for _ in range(4):
            run()
            self.opt.step(self.lrs, check_finite=False, grid_stream=self._adam_stream, grid_done=self._grid_done,
                          veto=self._overflow)
            self._pinned_losses.copy_(self.losses, non_blocking=True)
            self._pinned_flag.copy_(self.opt.flag, non_blocking=True)
            cur.synchronize()
            code = int(self._pinned_flag[0])
            if code != ShardedAdam.VETO:
                break
            self.state.t -= 1  # nothing was updated
            self._grow_after_overflow()
        else:
            raise RuntimeError("view binning kept outgrowing its pair capacity")
        if self.check_finite:
            ShardedAdam.raise_if_nonfinite(code)
        return self._pinned_losses

    def _views_host(self, targets_host: Sequence[torch.Tensor]) -> None:
        main = self._lanes[0].stream
        self._begin()
        n = len(self.views)

        nbuf = len(self._target_buf)

        def issue(i):
            b = i % nbuf
            with torch.cuda.stream(self._copy_stream):
                self._copy_stream.wait_event(self._buf_free[b])
                t = targets_host[i]
                if not t.is_pinned() or not t.is_contiguous() or t.dtype != torch.float32:
                    raise ValueError("step_host: targets must be contiguous pinned fp32 host tensors")
                # a plain stream-ordered copy (capturable; no host-allocator bookkeeping)
                copy_h2d(self._target_buf[b], t)
                self._copy_done[b].record(self._copy_stream)

        for b in range(nbuf):
            self._buf_free[b].record(main)
        ahead = nbuf - 1  # copies in flight ahead of the view being issued
        for i in range(min(n, ahead)):
            issue(i)
        for i in range(n):
            b = i % nbuf
            if i + ahead < n:
                issue(i + ahead)
            s = self._lane(i).stream
            with torch.cuda.stream(s):
                cam, out, gimg = self._view_forward(i)
                s.wait_event(self._copy_done[b])
                self._view_backward(i, cam, out, gimg,
                                    self._target_buf[b].view(-1)[: cam.height * cam.width * 3])
                self._buf_free[b].record(s)
        self._join()

    def launches(self) -> int:
        return sum(c.launches() for c in all_contexts(self.splats.device))
