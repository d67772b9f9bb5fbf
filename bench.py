"""Benchmark of the Gaussian Billboards hot path on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[3]): 1,000,000 textured surfels with 8x8 RGB
fp32 textures, 64 Fibonacci-sphere cameras (radius 6) at 1600x1064.  Strong
scaling (default, SURVEY §8(d)'s primary): the 64 views are split over the N
GPUs; --scaling weak: every GPU renders and backpropagates its own 8 views.
Per step every GPU renders and backpropagates its views (L1 loss against
seeded-noise targets); for N > 1 the gradients are reduce-scattered over NCCL
through the C-ABI, Adam updates each rank's slice and the parameters are
all-gathered.  One "step" is that whole training step; value = megapixels/s
over all GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scaling strong|weak]

--impl reference times the reference algorithm's CPU implementation on the
host cores (rank 0 only): the compiled reference has no perspective camera
(SPEC.md:279), so the workload runs through the fp64 C restatement
(oracle/gb_oracle.c, bit-exact with the reference on its own ortho path),
one full view per step with all host threads.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "fwd+bwd ms/view and megapixels/sec at 1/2/4/8 B200; % HBM roofline"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the 64 configs[3] views split over the N ranks (SURVEY §8(d) primary); "
                         "weak: --views-per-gpu views on every rank")
    ap.add_argument("--views-per-gpu", type=int, default=8)
    ap.add_argument("--count", type=int, default=1_000_000)
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpp-host", action="store_true",
                    help="skip the C++-host measurement (gbil_b200::multiview::Rank through libgb_mvhost.so)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="issue each step's view work eagerly instead of replaying it as one CUDA graph")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def union_ms(ivs) -> float:
    """Total length of the union of [a, b) intervals."""
    busy, end = 0.0, -1e30
    for a, b in sorted(ivs):
        if b > end:
            busy += b - max(a, end)
            end = b
    return busy


def attribute_ms(ivs_by_kernel: dict) -> dict:
    """Share of the timeline per kernel: every instant covered by k concurrent launches (any lanes, any
    kernels) is split equally between them, so the shares sum to the union of all launches (<= the step)."""
    ev = []
    for name, ivs in ivs_by_kernel.items():
        for a, b in ivs:
            if b > a:
                ev.append((a, 1, name))
                ev.append((b, -1, name))
    ev.sort(key=lambda e: (e[0], e[1]))
    out = {k: 0.0 for k in ivs_by_kernel}
    active = {}
    t0 = None
    for t, d, name in ev:
        n = sum(active.values())
        if t0 is not None and n > 0 and t > t0:
            for k, c in active.items():
                out[k] += (t - t0) * c / n
        active[name] = active.get(name, 0) + d
        if active[name] == 0:
            del active[name]
        t0 = t
    return out


def hbm_peak():
    try:
        with open(PEAKS) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for name, val in zip(names, p[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
# CPU legs (oracle = test infrastructure; only the cpu_baseline and --impl reference legs use it)
# ---------------------------------------------------------------------------------------------
def cpu_view(scene64, cam, target, step_frac_adam=1.0 / 64):
    """One view of the workload on the host: binning + forward + L1 + backward (+ its 1/64 share of the
    step's Adam: one update per 64-view step)."""
    from oracle import oracle as O

    cfg = O.Cfg()
    b = O.build_binning(scene64, cam, cfg)
    f = O.render_forward(scene64, cam, cfg, b, kink=None)
    _, ig = O.l1_loss(f["color"], target, 1.0 / f["color"].size)
    g, _, _ = O.render_backward(scene64, cam, cfg, b, f, ig.reshape(f["color"].shape), kink=None, want_mag=False)
    # the step's Adam over the replicated parameters, amortised over its 8 views
    flat = np.concatenate([v.ravel() for v in g.values() if v is not None])
    m = int(flat.size * step_frac_adam)
    O.adam_group(np.zeros(m), flat[:m], np.zeros(m), np.zeros(m), 1e-3, 0.9, 0.999, 1e-8, 0.1, 0.001)
    return len(b[1])


def cpu_setup(args):
    """The configs[3] inputs generated by the oracle's own Rng restatement (no product code is loaded)."""
    from oracle import oracle as O

    arrays, cams, target = O.config3_inputs(count=args.count, n=args.n)
    return O, O.Scene64(arrays, args.n), cams, target


def run_reference(args):
    """The reference algorithm's CPU implementation on all host cores (rank 0 only), one full configs[3]
    view per step.  (Sub-view samples are not representative: every reference call allocates and reduces
    full-size gradient buffers, so a band of a view costs half a view.)"""
    rank, world, local = dist_env()
    if rank != 0:
        return
    O, scene64, cams, target = cpu_setup(args)
    cores = os.cpu_count() or 1
    times = []
    views = list(range(len(cams)))
    for it in range(args.warmup + args.steps):
        v = views[it % len(views)]
        cam = cams[v]
        tgt = target(v)
        t0 = time.perf_counter()
        cpu_view(scene64, cam, tgt)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    W, H = cams[0].width, cams[0].height
    step_s = sum(times) / len(times)
    mps = W * H / 1e6 / step_s
    line = {
        "impl": "reference", "metric": METRIC, "value": round(mps, 4), "unit": "MP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 1),
        "ms_per_view": round(step_s * 1e3, 1), "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[3] shapes)",
        "config": {"workload": "configs[3] view: 1M surfels, 8x8 fp32 textures, 1600x1064, fwd+bwd+L1 (+1/64 of the step's Adam)",
                   "views_per_step": 1},
        "cpu_baseline": {"value": round(mps, 4), "unit": "MP/s", "cores": cores, "kind": "port",
                         "sample": "one full configs[3] view per step (binning + forward + L1 + backward + 1/64 of the step's "
                                   "Adam), fp64 C restatement of the reference algorithm (oracle/gb_oracle.c), "
                                   f"{cores} threads; the compiled reference has no perspective path"},
        "e2e": {"value": round(mps, 4), "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def k4_isolated(trainer, cams, views, dev_targets, W, H, device):
    """Average K4 launch time of `views` run one after another on one stream (trainer's configuration:
    RGBA-padded texels and texel gradients), with the pair count P of each view for the algorithmic bytes."""
    import torch

    import paper_2412_12734_b200 as gb

    splats = trainer.splats
    ctx = gb.raster.context(device)
    rb = gb.TileBinning(device)
    out = gb.RenderOutput(W, H, device)
    grads = gb.GradientBuffer(splats)
    rgba = torch.empty(splats.grid.numel() // 3 * 4, dtype=torch.float32, device=device)
    gb.raster.texels_pad(splats.grid.view(-1), rgba)
    pad = torch.zeros_like(rgba)
    pairs, ms, cnt = 0, 0.0, 0
    for rep in range(2):  # the first pass warms up
        for v in views:
            b = gb.build_binning(splats, cams[v], out=rb)
            o = gb.render_forward(splats, cams[v], b, out, texels_rgba=rgba)
            _, ig = gb.l1_loss(o.color, dev_targets[v])
            torch.cuda.synchronize()
            ctx.profile(True)
            ctx.profile_read()
            gb.render_backward(splats, cams[v], b, o, ig, grads, texel_grad=pad, texels_rgba=rgba)
            t, n = ctx.profile_read()["backward"]
            ctx.profile(False)
            if rep == 1:
                pairs, ms, cnt = pairs + b.total, ms + t, cnt + n
    del pad, rgba, grads
    return {"avg_launch_ms": round(ms / max(1, cnt), 4), "mean_pairs": pairs // max(1, len(views)),
            "launches": cnt, "what": "K4 of %d configs[3] views one at a time on one stream after the timed "
                                     "region (CUDA events at the C-ABI launch site)" % len(views)}


def run_cpp_host(args, arrays, cams, views, dev_targets, W, H, host_targets=None):
    """The same device-resident step through the C++ host (gbil_b200::multiview::Rank: six view lanes,
    capacity binning, one CUDA graph per step, padded texel gradients; Adam on one stream), timed by wall
    clock around K steps (each step ends with its synchronous loss and flag read)."""
    import ctypes as C

    import torch

    lib = C.CDLL(os.path.join(ROOT, "paper_2412_12734_b200", "libgb_mvhost.so"))
    P = C.c_void_p
    lib.gb_mv_create.argtypes = [C.c_int, C.c_int64, C.c_int] + [P] * 5 + [C.c_int] * 3 + [P, C.c_int, P, C.c_int,
                                                                                          C.c_int, C.c_double,
                                                                                          C.POINTER(P)]
    lib.gb_mv_step.argtypes = [P, C.c_int, P, C.POINTER(C.c_double)]
    lib.gb_mv_step_host.argtypes = [P, C.c_int, P, C.POINTER(C.c_double)]
    lib.gb_mv_destroy.argtypes = [P]
    lib.gb_mv_error.restype = C.c_char_p
    a = {k: np.ascontiguousarray(arrays[k], np.float32) for k in ("position", "quat", "log_scale", "opacity_logit",
                                                                   "grid")}
    cam16 = np.ascontiguousarray(np.array([[c.fx, c.fy, c.cx, c.cy, *np.asarray(c.rot).ravel(), *np.asarray(c.trans)]
                                           for c in cams], np.float64))
    vv = np.ascontiguousarray(np.array(views, np.int32))
    h = P()
    K = a["opacity_logit"].shape[0]
    n = int(round((a["grid"].shape[1] // 3) ** 0.5))
    rc = lib.gb_mv_create(torch.cuda.current_device(), K, n, *[a[k].ctypes.data for k in ("position", "quat",
                                                                                            "log_scale",
                                                                                            "opacity_logit", "grid")],
                          W, H, len(cams), cam16.ctypes.data, len(vv), vv.ctypes.data, int(os.environ.get("GB_LANES", "6")), 1, 6.0,
                          C.byref(h))
    if rc:
        raise RuntimeError(lib.gb_mv_error().decode())
    tp = (P * len(dev_targets))(*[t.data_ptr() for t in dev_targets])
    loss = C.c_double()
    try:
        for _ in range(max(3, args.warmup)):
            if lib.gb_mv_step(h, len(dev_targets), tp, C.byref(loss)):
                raise RuntimeError(lib.gb_mv_error().decode())
        t0 = time.perf_counter()
        for _ in range(args.steps):
            if lib.gb_mv_step(h, len(dev_targets), tp, C.byref(loss)):
                raise RuntimeError(lib.gb_mv_error().decode())
        dt = (time.perf_counter() - t0) / args.steps
        e2e = None
        if host_targets is not None:
            hp = (P * len(host_targets))(*[t.data_ptr() for t in host_targets])
            for _ in range(max(3, args.warmup)):
                if lib.gb_mv_step_host(h, len(host_targets), hp, C.byref(loss)):
                    raise RuntimeError(lib.gb_mv_error().decode())
            t0 = time.perf_counter()
            for _ in range(args.steps):
                if lib.gb_mv_step_host(h, len(host_targets), hp, C.byref(loss)):
                    raise RuntimeError(lib.gb_mv_error().decode())
            de = (time.perf_counter() - t0) / args.steps
            e2e = {"value": round(len(views) * W * H / 1e6 / de, 3), "unit": "MP/s", "ms_per_step": round(de * 1e3, 3),
                   "h2d_bytes_per_step": sum(t.numel() * 4 for t in host_targets),
                   "d2h_bytes_per_step": 4 * len(views) + 8}
    finally:
        lib.gb_mv_destroy(h)
    return {"value": round(len(views) * W * H / 1e6 / dt, 3), "unit": "MP/s", "ms_per_step": round(dt * 1e3, 3),
            "e2e": e2e,
            "what": "the same device-resident step driven by the C++ host (gbil_b200::multiview::Rank via "
                    "libgb_mvhost.so): six view lanes, capacity binning, one CUDA graph per step, padded texel "
                    "gradients, Adam's texel update overlapped with the next binning; wall clock around K steps, "
                    "each ending with its loss read (e2e: pinned host targets copied inside every step)",
            "last_loss": round(loss.value, 6)}


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the communicator sizes appear in the log
        torch.cuda.set_device(local)
        if os.environ.get("GB_BENCH_FAKE_PG") == "1":  # code-path check on one GPU: collectives move nothing
            from torch.testing._internal.distributed.fake_pg import FakeStore

            dist.init_process_group("fake", store=FakeStore(), rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
        local = 0
    device = torch.device("cuda", local)

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.scenes as sc
    from paper_2412_12734_b200.train import ViewShardedTrainer, shard_views

    cfg3 = sc.baseline_config(3, count=args.count, n=args.n)
    arrays = cfg3.arrays()
    splats = gb.SplatSet.from_numpy(cfg3.mode, gb.ColorGridConfig(cfg3.n), device=device, **arrays)
    cams = [gb.PinholeCamera.from_spec(c) for c in cfg3.cameras]
    views = shard_views(len(cams), rank, world, per_rank=args.views_per_gpu if args.scaling == "weak" else None)
    lrs = gb.LearningRates()
    lrs.position *= 6.0  # position LR x scene extent
    use_graph = os.environ.get("GB_GRAPH", "1") != "0" and not args.no_graph
    blocking = os.environ.get("GB_BLOCKING_BINNING") == "1"
    trainer = ViewShardedTrainer(splats, cams, views, lrs=lrs, graph=use_graph, async_binning=not blocking,
                                 lanes=int(os.environ.get("GB_LANES", "6")),
                                 overlap_adam=os.environ.get("GB_OVERLAP_ADAM", "1") == "1",
                                 capacity_margin=float(os.environ.get("GB_CAP_MARGIN", "1.1")),
                                 fused=os.environ.get("GB_FUSED") == "1",
                                 texel_pad=os.environ.get("GB_TEXEL_PAD", "1") == "1",
                                 rgba_texels=os.environ.get("GB_RGBA_TEXELS", "1") == "1")
    trainer.graph_host = os.environ.get("GB_GRAPH_HOST", "0") == "1"
    if os.environ.get("GB_PRE_ADAM_READ") == "1":
        trainer.overlap_read = False
    W, H = cams[0].width, cams[0].height
    host_targets = [torch.from_numpy(cfg3.target(v)).pin_memory() for v in views]
    dev_targets = [t.to(device) for t in host_targets]
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (untimed) ----
    for _ in range(args.warmup):
        trainer.step(dev_targets)
    torch.cuda.synchronize()
    barrier()

    # ---- timed region: inputs resident in HBM (working set >> 126 MB L2) ----
    stream = torch.cuda.current_stream(device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    trainer.reset_pair_stats()
    ctxs = gb.raster.all_contexts(device)  # one per view lane (stream)
    launches0 = trainer.launches()
    for c in ctxs:
        c.profile(True)
        c.profile_read()  # reset
    with ClockSampler(torch.cuda.current_device() if world == 1 else local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            trainer.step(dev_targets)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    # launch intervals of the compositors on all lanes, relative to ev0: overlapping launches of the same
    # kernel on different lanes are merged into busy time (a launch's own interval also holds its wait
    # for SMs held by the other lanes)
    intervals = {k: [iv for c in ctxs for iv in c.profile_intervals(ev0, k)] for k in gb._lib.KERNEL_NAMES}
    prof = {}
    for c in ctxs:
        c.profile(False)
        for k, (ms, cnt) in c.profile_read().items():
            t, n = prof.get(k, (0.0, 0))
            prof[k] = (t + ms, n + cnt)
    launches = trainer.launches() - launches0
    prof_note = ("CUDA events around every launch site on its stream, in the timed region" +
                 (" (event-record nodes of the replayed graph)" if use_graph else "") +
                 "; avg_launch_ms = union of the kernel's launch intervals over all lanes / launches")
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))
    step_ms = elapsed_ms / args.steps
    views_total = world * len(views) if args.scaling == "weak" else len(cams)
    mpix = views_total * W * H / 1e6
    value = mpix / (step_ms / 1e3)
    pair_sum, pair_views = trainer.pair_stats()
    mean_pairs = pair_sum / max(1, pair_views)

    # ---- end to end: pinned host targets in, per-view losses out, every step ----
    e2e = None
    if not args.no_e2e:
        for _ in range(max(3, args.warmup)):  # the same W >= 3 warm-up as the device-input timing
            trainer.step_host(host_targets)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2.record(stream)
        for _ in range(args.steps):
            trainer.step_host(host_targets)
        ev3.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e2e_dev = ev2.elapsed_time(ev3) / args.steps
        e2e_ms = max_over_ranks(max(ev2.elapsed_time(ev3), wall * 1e3)) / args.steps
        h2d = sum(t.numel() * 4 for t in host_targets)
        e2e = {"value": round(mpix / (e2e_ms / 1e3), 3), "unit": "MP/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": len(views) * 4, "ms_per_step": round(e2e_ms, 3),
               "device_ms_per_step": round(e2e_dev, 3), "wall_ms_per_step": round(wall * 1e3 / args.steps, 3)}

    # ---- forward only (render: K1 + K2 + K3 per view, one stream), SURVEY §8(d)'s "fwd" figure ----
    fwd = None
    if rank == 0:
        rb = gb.TileBinning(device)
        rb.set_capacity(trainer.capacity or 0, torch.zeros(1, dtype=torch.int32, device=device))
        rout = gb.RenderOutput(W, H, device)
        for v in views[:2]:  # warm-up
            gb.render_forward(splats, cams[v], gb.build_binning(splats, cams[v], out=rb), rout)
        torch.cuda.synchronize()
        evf0, evf1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        evf0.record()
        for _ in range(reps):
            for v in views:
                gb.render_forward(splats, cams[v], gb.build_binning(splats, cams[v], out=rb), rout)
        evf1.record()
        torch.cuda.synchronize()
        f_ms = evf0.elapsed_time(evf1) / (reps * len(views))
        fwd = {"ms_per_view": round(f_ms, 4), "value": round(W * H / 1e6 / (f_ms / 1e3), 3), "unit": "MP/s",
               "what": "build_binning + render_forward per view, one stream, CUDA events"}

    # ---- K4 alone: the backward compositor of a few views on one stream, no other lane sharing the SMs
    # (the roofline above times it inside the overlapped step) -- per-launch-site CUDA events of the C-ABI ----
    k4_alone = None
    if rank == 0:
        try:
            k4_alone = k4_isolated(trainer, cams, views[:8], dev_targets, W, H, device)
        except Exception as e:  # an extra measurement never blocks the headline
            k4_alone = {"failed": str(e)[:200]}

    # ---- the same step driven by the C++ host (include/gbil_b200.hpp multiview::Rank, libgb_mvhost.so) ----
    cpp_host = None
    if rank == 0 and world == 1 and not args.no_cpp_host:
        try:
            cpp_host = run_cpp_host(args, arrays, cams, views, dev_targets, W, H,
                                    None if args.no_e2e else host_targets)
        except Exception as e:  # an extra measurement never blocks the headline
            cpp_host = {"failed": str(e)[:200]}

    # ---- replicas stay in sync: every rank holds bit-identical parameters ----
    in_sync = True
    if world > 1:
        flat = trainer.opt.flat if trainer.opt is not None else torch.cat(
            [t.reshape(-1) for t in trainer.splats.tensors().values()])
        h = flat.view(torch.int32).to(torch.int64)
        digest = torch.stack([(h * (torch.arange(h.numel(), device=h.device) % 1021 + 1)).sum(), h.sum()])
        lo, hi = digest.clone(), digest.clone()
        torch.distributed.all_reduce(lo, op=torch.distributed.ReduceOp.MIN)
        torch.distributed.all_reduce(hi, op=torch.distributed.ReduceOp.MAX)
        in_sync = bool(torch.equal(lo, hi))

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (algorithmic bytes) ----
    peak, peak_src = hbm_peak()
    n = cfg3.n
    Bh, Bt = 40, 12 * n * n  # SURVEY §8(d) algorithmic header and texture bytes
    tiles = ((W + 15) // 16) * ((H + 15) // 16)
    npx = W * H
    model = {
        "backward": lambda P: P * (4 + 2 * Bh + 2 * Bt) + 8 * tiles + 20 * npx,
        "forward": lambda P: P * (4 + Bh + Bt) + 8 * tiles + 20 * npx,
        # K3+K6+K4 fused: each pair's list entry, header and texels read once and their gradients
        # written once; per pixel only the target is read (no image, T or last round trip)
        "fused": lambda P: P * (4 + 2 * Bh + 2 * Bt) + 8 * tiles + 12 * npx,
    }
    dom = max(model, key=lambda k: prof[k][0])
    total_ms, count = prof[dom]
    bytes_per_launch = model[dom](mean_pairs)  # linear in P: the mean over the timed views
    busy_ms = union_ms(intervals.get(dom, []))  # union of the launch intervals
    avg_ms = (busy_ms if busy_ms > 0 else total_ms) / max(1, count)  # busy time per launch
    achieved = bytes_per_launch / (avg_ms / 1e3) / 1e9
    traffic = None
    ncu_sum = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(ncu_sum):
        try:
            traffic = json.load(open(ncu_sum)).get(dom, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    share = attribute_ms({k: v for k, v in intervals.items() if v})
    kernel_ms = {k: round(v / args.steps, 4) for k, v in share.items()}
    kernel_busy = {k: round(union_ms(v) / args.steps, 4) for k, v in intervals.items() if v}
    collective_ms = round(union_ms(intervals.get("collective", [])) / args.steps, 4)
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "MP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 3),
        "ms_per_view": round(step_ms / len(views), 3),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded Rng, BASELINE configs[3] shapes; random-init surfels, noise targets)",
        "config": {"workload": "configs[3] view-sharded training step: 1M surfels, 8x8 fp32 RGB textures, "
                               + (f"the 64 Fibonacci-sphere views split over {world} GPU(s)" if args.scaling == "strong"
                                  else f"{args.views_per_gpu} Fibonacci-sphere views/GPU") +
                               " at 1600x1064, L1, Adam (N > 1: NCCL reduce-scatter through the C-ABI, Adam on "
                               "the rank's slice, all-gather)",
                   "views_per_gpu": len(views), "views_total": views_total, "surfels": cfg3.count, "texture": f"{n}x{n}",
                   "image": f"{W}x{H}", "tile": 16,
                   "compositor": ("fused " if trainer.fused else "") + "direct (one warp per 8x4 pixel block)",
                   "mean_pairs_per_view": int(mean_pairs),
                   "binning": "blocking" if blocking else "capacity (no host read-back)",
                   "cuda_graph": ("each step's view work (binning + compositing on all lanes) replayed as one "
                                  "CUDA graph; collectives + Adam eager, Adam's texel update overlapped with the "
                                  "next step's binning; e2e step eager") if use_graph else "off",
                   "view_lanes": len(trainer._lanes),
                   "l2": "working set (0.8 GB textures + 0.8 GB grads + 1.6 GB Adam) >> 126 MB L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": int(bytes_per_launch), "avg_launch_ms": round(avg_ms, 4),
                     "avg_launch_ms_events": round(total_ms / max(1, count), 4),
                     "peak_source": peak_src, "timing": prof_note,
                     "alone": (dict(k4_alone, frac=round(model["backward"](k4_alone["mean_pairs"])
                                                        / (k4_alone["avg_launch_ms"] / 1e3) / 1e9 / peak, 4))
                               if k4_alone and "avg_launch_ms" in k4_alone and k4_alone["avg_launch_ms"] > 0
                               else k4_alone)},
        "kernel_ms_per_step": kernel_ms,
        "kernel_ms_note": "each kernel's share of the timeline from CUDA events around every launch on all view "
                          "lanes: an instant covered by k concurrent launches counts 1/k to each, so the shares "
                          "sum to the busy time (<= ms_per_step); kernel_busy_ms_per_step is each kernel's own "
                          "union of launch intervals (overlaps other kernels)",
        "kernel_busy_ms_per_step": kernel_busy,
        "collective_ms": collective_ms,
        "comm": ({"nranks": world, "path": "C-ABI gb_comm (NCCL; reduce-scatter + all-gather + flag min)"}
                 if world > 1 else {"nranks": 1, "path": "none (one GPU)"}),
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "e2e": e2e,
        "replicas_in_sync": in_sync,
        "forward_only": fwd,
        "cpp_host": cpp_host,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            O, scene64, ocams, otarget = cpu_setup(args)
            t0 = time.perf_counter()
            cpu_view(scene64, ocams[views[0]], otarget(views[0]))
            dt = time.perf_counter() - t0
            cores = os.cpu_count() or 1
            line["cpu_baseline"] = {
                "value": round(W * H / 1e6 / dt, 4), "unit": "MP/s", "cores": cores, "kind": "port",
                "sample": f"1 view of the workload (binning+forward+L1+backward+1/64 of the step's Adam) in {dt:.1f} s, fp64 C "
                          f"restatement of the reference algorithm (oracle/gb_oracle.c), {cores} threads"}
        except Exception as e:  # the baseline never blocks the GPU number
            line["cpu_baseline"] = {"value": None, "unit": "MP/s", "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"failed: {e}"}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
