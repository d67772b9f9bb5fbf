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
