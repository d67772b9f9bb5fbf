"""Multi-process logic of the view-sharded training step on CPU (gloo, world size 2).

The CUDA kernels need a GPU, so each rank computes its views' gradients with
the fp64 oracle; the test exercises the product's sharding (shard_views), the
flat GradientBuffer layout and its single all-reduce (reduce_gradients), and
checks that (a) every view is rendered exactly once across ranks, (b) the
all-reduced gradient equals the single-process sum over all views, and
(c) a replicated Adam step leaves identical parameters on every rank.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    import paper_2412_12734_b200.scenes as sc

    arrays = sc.generate(1, 60, 2, 5, mean_lo=-0.5, mean_hi=0.5, scale_lo=0.05, scale_hi=0.2)
    cams = sc.fibonacci_cameras(4, 3.0, 40, 30, 40.0, 40.0, 20.0, 15.0)
    return arrays, cams


def _view_grads(arrays, cams, views):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity import O

    import paper_2412_12734_b200.scenes as sc

    scene = O.Scene64(arrays, 2)
    total = None
    for v in views:
        cam = O.Cam.from_spec(cams[v])
        cfg = O.Cfg(tile_size=8, threads=1)
        b = O.build_binning(scene, cam, cfg)
        f = O.render_forward(scene, cam, cfg, b, kink=None)
        tgt = sc.uniform_image(7 + v, cam.width, cam.height)
        _, ig = O.l1_loss(f["color"], tgt, 1.0 / f["color"].size)
        g, _, _ = O.render_backward(scene, cam, cfg, b, f, ig.reshape(f["color"].shape), kink=None, want_mag=False)
        if total is None:
            total = {k: v_.copy() for k, v_ in g.items() if v_ is not None and k != "depth_key" and k != "theta"}
        else:
            for k in total:
                total[k] += g[k]
    return total


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200.train import reduce_gradients, shard_views

    dist.init_process_group("gloo", rank=rank, world_size=world)
    arrays, cams = _scene()
    views = shard_views(len(cams), rank, world)
    splats = gb.SplatSet.from_numpy(gb.raster.MODE_PINHOLE, gb.ColorGridConfig(2), device="cpu", **arrays)
    grads = gb.GradientBuffer(splats)
    g = _view_grads(arrays, cams, views)
    for k, v in g.items():
        getattr(grads, k).copy_(torch.as_tensor(v.reshape(getattr(grads, k).shape), dtype=torch.float32))
    reduce_gradients(grads)
    # replicated Adam (optim.hpp:76-90 semantics) on the flat buffer
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity import O

    p = np.concatenate([np.asarray(arrays[k], np.float64).ravel() for k in ("position", "quat", "log_scale",
                                                                            "opacity_logit", "grid")])
    gflat = np.concatenate([getattr(grads, k).numpy().astype(np.float64).ravel() for k in
                            ("position", "quat", "log_scale", "opacity_logit", "grid")])
    p1, m, v, bad = O.adam_group(p, gflat, np.zeros_like(p), np.zeros_like(p), 1e-3, 0.9, 0.999, 1e-8, 0.1, 0.001)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), views=np.array(views), grads=gflat, params=p1)
    dist.destroy_process_group()


def test_view_sharded_step_gloo(tmp_path):
    import torch.multiprocessing as mp

    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, start_method="spawn")
    r = [np.load(tmp_path / f"rank{i}.npz") for i in range(world)]
    views = np.concatenate([x["views"] for x in r])
    assert sorted(views.tolist()) == [0, 1, 2, 3]  # every view exactly once
    assert np.array_equal(r[0]["grads"], r[1]["grads"])  # all-reduce result identical on all ranks
    assert np.array_equal(r[0]["params"], r[1]["params"])  # replicated Adam stays in sync
    sys.path.insert(0, ROOT)
    arrays, cams = _scene()
    ref = _view_grads(arrays, cams, [0, 1, 2, 3])
    ref_flat = np.concatenate([ref[k].ravel() for k in ("position", "quat", "log_scale", "opacity_logit", "grid")])
    np.testing.assert_allclose(r[0]["grads"], ref_flat.astype(np.float32), rtol=1e-5, atol=1e-7)


def test_shard_views_partitions():
    sys.path.insert(0, ROOT)
    from paper_2412_12734_b200.train import shard_views

    for n, w in ((64, 8), (64, 3), (5, 4), (64, 1)):
        got = sorted(v for r in range(w) for v in shard_views(n, r, w))
        assert got == list(range(n))
    assert [shard_views(64, r, 8, per_rank=8) for r in range(8)][3] == list(range(24, 32))


# ---------------------------------------------------------------------------------------------
# the sharded optimiser (reduce-scatter -> Adam on 1/world of the flat parameters -> all-gather)
# ---------------------------------------------------------------------------------------------
def _cpu_segment_update(phase, opt, lrs):
    """Test stand-in for gb_adam_segments on CPU tensors: the oracle's Adam per (flat range, group)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch

    from parity import O

    base = opt.lo if opt.world > 1 else 0
    if phase == 0:
        for a, b, grp in opt.ranges:
            g = opt.g_shard[a - base:b - base].numpy()
            bad = np.nonzero(~np.isfinite(g))[0]
            if bad.size:
                opt.flag[0] = min(int(opt.flag[0]), (grp << 48) | int(bad[0]))
        return
    if int(opt.flag[0]) < (1 << 62):
        opt.state.t += 1
        return
    opt.state.t += 1
    t = opt.state.t
    rates = [lrs.position * lrs.position_gamma ** (t - 1), lrs.theta, lrs.log_scale, lrs.opacity_logit,
             lrs.color_grid]
    c = opt.state.config
    for a, b, grp in opt.ranges:
        p = opt.flat[a:b].numpy().astype(np.float64)
        g = opt.g_shard[a - base:b - base].numpy().astype(np.float64)
        m = opt.m[a - opt.lo:b - opt.lo].numpy().astype(np.float64)
        v = opt.v[a - opt.lo:b - opt.lo].numpy().astype(np.float64)
        p1, m1, v1, _ = O.adam_group(p, g, m, v, rates[grp], c.beta1, c.beta2, c.epsilon, 1 - c.beta1 ** t,
                                     1 - c.beta2 ** t)
        opt.flat[a:b] = torch.as_tensor(p1, dtype=torch.float32)
        opt.m[a - opt.lo:b - opt.lo] = torch.as_tensor(m1, dtype=torch.float32)
        opt.v[a - opt.lo:b - opt.lo] = torch.as_tensor(v1, dtype=torch.float32)


def _sharded_worker(rank, world, port, out_dir, nan_rank):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200.train import ShardedAdam

    dist.init_process_group("gloo", rank=rank, world_size=world)
    arrays, _ = _scene()
    splats = gb.SplatSet.from_numpy(gb.raster.MODE_PINHOLE, gb.ColorGridConfig(2), device="cpu", **arrays)
    grads = gb.GradientBuffer(splats, multiple=4 * world)
    rng = np.random.default_rng(100 + rank)  # each rank's partial gradient
    grads.flat.copy_(torch.as_tensor(rng.standard_normal(grads.flat.numel()), dtype=torch.float32))
    if rank == nan_rank:
        grads.quat.view(-1)[3] = float("nan")
    state = gb.AdamState(splats, moments=False)
    opt = ShardedAdam(splats, grads, state, segment_update=_cpu_segment_update)
    lrs = gb.LearningRates(position_gamma=0.9)
    p0 = {f: t.clone() for f, t in splats.tensors().items()}
    err = ""
    try:
        opt.step(lrs, check_finite=True)
        opt.step(lrs, check_finite=True)
    except gb.raster.NonFinite as e:
        err = str(e)
    np.savez(os.path.join(out_dir, f"sh{rank}.npz"), flat=opt.flat.numpy(), t=state.t, err=err,
             ranges=np.array([(a, b, g) for a, b, g in opt.ranges] or [(0, 0, -1)]),
             unchanged=all(torch.equal(p0[f], t) for f, t in splats.tensors().items()),
             views=all(t.data_ptr() >= opt.flat.data_ptr() for t in splats.tensors().values()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_adam_gloo(tmp_path, world):
    """Every parameter is updated by exactly one rank, all ranks end with identical parameters, and the
    result equals a single-process Adam on the summed gradients, two steps in a row."""
    import torch.multiprocessing as mp

    mp.start_processes(_sharded_worker, args=(world, _free_port(), str(tmp_path), -1), nprocs=world,
                       start_method="spawn")
    r = [np.load(tmp_path / f"sh{i}.npz") for i in range(world)]
    for x in r[1:]:
        assert np.array_equal(x["flat"], r[0]["flat"])
    assert all(bool(x["views"]) and int(x["t"]) == 2 and str(x["err"]) == "" for x in r)
    covered = sorted((int(a), int(b)) for x in r for a, b, g in x["ranges"] if g >= 0)
    for (a0, b0), (a1, b1) in zip(covered, covered[1:]):
        assert b0 <= a1  # disjoint
    # single-process reference: Adam on the sum of the ranks' partial gradients, per group
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch

    import paper_2412_12734_b200 as gb
    from parity import O

    arrays, _ = _scene()
    splats = gb.SplatSet.from_numpy(gb.raster.MODE_PINHOLE, gb.ColorGridConfig(2), device="cpu", **arrays)
    grads = gb.GradientBuffer(splats, multiple=4 * world)
    gsum = sum(np.random.default_rng(100 + k).standard_normal(grads.flat.numel()).astype(np.float32)
               .astype(np.float64) for k in range(world))
    lrs = gb.LearningRates(position_gamma=0.9)
    rates = {"position": [lrs.position, lrs.position * 0.9], "quat": [lrs.theta] * 2,
             "log_scale": [lrs.log_scale] * 2, "opacity_logit": [lrs.opacity_logit] * 2, "grid": [lrs.color_grid] * 2}
    for f, (o, n) in grads.offsets.items():
        p = np.asarray(arrays[f], np.float64).ravel()
        m = np.zeros_like(p)
        v = np.zeros_like(p)
        g = gsum[o:o + n]
        for t in (1, 2):
            p, m, v, _ = O.adam_group(p, g, m, v, rates[f][t - 1], 0.9, 0.999, 1e-8, 1 - 0.9 ** t, 1 - 0.999 ** t)
        np.testing.assert_allclose(r[0]["flat"][o:o + n], p, rtol=1e-5, atol=1e-6, err_msg=f)


def test_sharded_adam_nonfinite_agreement(tmp_path):
    """A non-finite gradient on one rank's input stops the update on every rank (optim.hpp:81-83)."""
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_sharded_worker, args=(world, _free_port(), str(tmp_path), 1), nprocs=world,
                       start_method="spawn")
    r = [np.load(tmp_path / f"sh{i}.npz") for i in range(world)]
    for x in r:
        assert bool(x["unchanged"]), "no parameter may change"
        assert "non-finite gradient in group 'theta'" in str(x["err"])
