"""The training-step kernels around the compositor, on the GPU, against the oracle.

* K6 L1 loss (the BASELINE configs' loss) and MSE (train.hpp:120-133);
* K7 Adam (optim.hpp:76-117): three steps against the fp64 oracle's adam_group,
  and the non-finite guard (optim.hpp:81-83: nothing is updated, the call raises);
* the view-sharded step (configs[3] shape, scaled down): gradients summed over
  the views equal the oracle's per-view backward sum, and the post-Adam
  parameters equal the oracle's Adam on those gradients.
"""
import os

import numpy as np
import pytest

from parity import O, compare_grads

pytestmark = pytest.mark.gpu


def test_l1_and_mse_loss():
    import torch

    import paper_2412_12734_b200 as gb

    rng = np.random.default_rng(1)
    c = rng.random((40, 56, 3), dtype=np.float32)
    t = rng.random((40, 56, 3), dtype=np.float32)
    scale = 1.0 / c.size
    loss, grad = gb.l1_loss(torch.as_tensor(c).cuda(), torch.as_tensor(t).cuda(), scale)
    ref_loss, ref_grad = O.l1_loss(c.astype(np.float64), t.astype(np.float64), scale)
    assert abs(float(loss) - ref_loss) <= 1e-5 * abs(ref_loss)
    np.testing.assert_array_equal(grad.cpu().numpy(), ref_grad.astype(np.float32))
    loss, grad = gb.mse_loss(torch.as_tensor(c).cuda(), torch.as_tensor(t).cuda(), scale)
    d = c.astype(np.float64) - t
    assert abs(float(loss) - (d * d).sum() * scale) <= 1e-5 * (d * d).sum() * scale
    np.testing.assert_allclose(grad.cpu().numpy(), 2 * scale * d, rtol=1e-6, atol=1e-12)


def _pinhole_scene(K, n, seed):
    import paper_2412_12734_b200.scenes as sc

    return sc.generate(O.MODE_PINHOLE, K, n, seed, mean_lo=-1.0, mean_hi=1.0, scale_lo=0.01, scale_hi=0.08)


def test_adam_three_steps_vs_oracle():
    import torch

    import paper_2412_12734_b200 as gb

    n, K = 4, 1001  # odd sizes exercise the vector body and the scalar tail
    arrays = _pinhole_scene(K, n, 3)
    splats = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    state = gb.AdamState(splats)
    lrs = gb.LearningRates(position_gamma=0.9)
    rng = np.random.default_rng(7)
    names = {"position": "position", "quat": "quat", "log_scale": "log_scale", "opacity_logit": "opacity_logit",
             "grid": "grid"}
    lr_of = {"position": None, "quat": lrs.theta, "log_scale": lrs.log_scale, "opacity_logit": lrs.opacity_logit,
             "grid": lrs.color_grid}
    ref_p = {f: splats.tensors()[f].cpu().numpy().astype(np.float64).ravel() for f in names}
    ref_m = {f: np.zeros_like(v) for f, v in ref_p.items()}
    ref_v = {f: np.zeros_like(v) for f, v in ref_p.items()}
    for t in range(1, 4):
        grads = gb.GradientBuffer(splats)
        host = {}
        for f in names:
            g = grads.tensors()[f]
            h = (rng.standard_normal(g.numel()) * 10.0 ** rng.uniform(-4, 1, g.numel())).astype(np.float32)
            g.copy_(torch.as_tensor(h).view_as(g))
            host[f] = h.astype(np.float64)
        gb.adam_step(splats, grads, state, lrs)
        b1, b2 = 1 - 0.9 ** t, 1 - 0.999 ** t
        for f in names:
            lr = lrs.position * lrs.position_gamma ** (t - 1) if f == "position" else lr_of[f]
            ref_p[f], ref_m[f], ref_v[f], bad = O.adam_group(ref_p[f], host[f], ref_m[f], ref_v[f], lr, 0.9, 0.999,
                                                              1e-8, b1, b2)
            assert bad == 0, bad
    torch.cuda.synchronize()
    assert state.t == 3
    for f in names:
        got = splats.tensors()[f].cpu().numpy().astype(np.float64).ravel()
        lr = lrs.position if f == "position" else lr_of[f]
        # fp32 parameters and moments: each of the 3 updates (size <= lr) is exact to ~1e-6 relative
        np.testing.assert_allclose(got, ref_p[f], rtol=2e-6, atol=1e-5 * lr, err_msg=f)


def test_adam_nonfinite_gradient_raises_and_updates_nothing():
    import torch

    import paper_2412_12734_b200 as gb

    arrays = _pinhole_scene(300, 2, 4)
    splats = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(2), **arrays)
    before = {f: v.clone() for f, v in splats.tensors().items() if v is not None}
    grads = gb.GradientBuffer(splats)
    grads.tensors()["grid"].fill_(0.5)
    grads.tensors()["log_scale"].view(-1)[17] = float("nan")
    state = gb.AdamState(splats)
    with pytest.raises(Exception, match="log_scale"):
        gb.adam_step(splats, grads, state, gb.LearningRates())
    torch.cuda.synchronize()
    for f, v in before.items():
        assert torch.equal(splats.tensors()[f], v), f


def test_view_sharded_step_vs_oracle():
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.scenes as sc
    from paper_2412_12734_b200.train import ViewShardedTrainer

    n, K, W, H = 4, 3000, 96, 80
    arrays = _pinhole_scene(K, n, 5)
    specs = [sc.look_at((3.0 * np.cos(a), 0.7, 3.0 * np.sin(a)), (0.0, 0.0, 0.0), W, H, 90.0, 90.0, 48.0, 40.0)
             for a in (0.3, 2.1)]
    targets = [sc.uniform_image(100 + v, W, H) for v in range(2)]
    splats = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    cams = [gb.PinholeCamera.from_spec(s) for s in specs]
    lrs = gb.LearningRates()
    tr = ViewShardedTrainer(splats, cams, [0, 1], lrs=lrs)
    # the per-view image cotangents the step will use (computed from the same GPU forward)
    igs = []
    for v in range(2):
        b = gb.build_binning(splats, cams[v])
        out = gb.render_forward(splats, cams[v], b)
        _, ig = gb.l1_loss(out.color, torch.as_tensor(targets[v]).cuda())
        igs.append(ig.cpu().numpy().astype(np.float64))
    p0 = {f: v.cpu().numpy().astype(np.float64).ravel() for f, v in splats.tensors().items() if v is not None}
    tr.step([torch.as_tensor(t).cuda() for t in targets])
    torch.cuda.synchronize()
    # oracle: sum over the views of render_backward with the same cotangents
    scene = O.Scene64(arrays, n)
    cfg = O.Cfg()
    tot = {f: None for f in ("position", "quat", "log_scale", "opacity_logit", "grid")}
    mag, slack = dict(tot), dict(tot)
    for v in range(2):
        cam = O.Cam.from_spec(specs[v])
        b = O.build_binning(scene, cam, cfg)
        f = O.render_forward(scene, cam, cfg, b)
        g, m, s = O.render_backward(scene, cam, cfg, b, f, igs[v])
        for k in tot:
            tot[k] = g[k] if tot[k] is None else tot[k] + g[k]
            mag[k] = m[k] if mag[k] is None else mag[k] + m[k]
            slack[k] = s[k] if slack[k] is None else slack[k] + s[k]
    got = {k: v.cpu().numpy().astype(np.float64) for k, v in tr.grads.tensors().items() if k in tot}
    st = compare_grads(dict(grads=got), dict(grads=tot, mag=mag, slack=slack))
    for k, s in st.items():
        assert s["strict_violations_applicable"] == 0 and s["model_violations"] == 0, (k, s)
    # Adam on exactly those gradients
    for k in tot:
        lr = {"position": lrs.position, "quat": lrs.theta, "log_scale": lrs.log_scale,
              "opacity_logit": lrs.opacity_logit, "grid": lrs.color_grid}[k]
        ref, _, _, _ = O.adam_group(p0[k], got[k].ravel(), np.zeros_like(p0[k]), np.zeros_like(p0[k]), lr, 0.9,
                                    0.999, 1e-8, 0.1, 1 - 0.999)
        np.testing.assert_allclose(splats.tensors()[k].cpu().numpy().astype(np.float64).ravel(), ref, rtol=2e-6,
                                   atol=1e-5 * lr, err_msg=k)


def test_capacity_binning_matches_blocking():
    """gb_binning_set_capacity: padded sort over a fixed pair capacity, no host read-back -- the same
    tile lists and images as the blocking build; an undersized capacity raises the overflow flag."""
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.scenes as sc

    c = sc.baseline_config(0, count=20_000, n=4)
    splats = gb.SplatSet.from_numpy(c.mode, gb.ColorGridConfig(4), **c.arrays())
    cam = gb.PinholeCamera.from_spec(c.cameras[0])
    ref = gb.build_binning(splats, cam)
    P = ref.total
    ref_csr = ref.csr()
    ref_img = gb.render_forward(splats, cam, ref).color.clone()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    tx, ty = ref.tiles_x, ref.tiles_y
    # the last capacity exceeds 512 slots per tile: the capacity build takes the radix path (deep scenes)
    # while the blocking reference took the tile-bucket path -- the two K2 builds must agree bit for bit
    for cap in (P, P + 1, P + 70_000, P + 600 * tx * ty):
        b = gb.TileBinning()
        b.set_capacity(cap, flag)
        gb.build_binning(splats, cam, out=b)
        got = torch.zeros(1, dtype=torch.int32, device="cuda")
        b.store_total(got)
        assert int(got) == P and int(flag) == 0 and b.total == P
        off, val = b.csr()
        np.testing.assert_array_equal(off, ref_csr[0])
        np.testing.assert_array_equal(val, ref_csr[1])
        assert torch.equal(gb.render_forward(splats, cam, b).color, ref_img)
    small = gb.TileBinning()
    small.set_capacity(P // 3, flag)
    gb.build_binning(splats, cam, out=small)
    assert int(flag) == 1 and small.total == P // 3
    off, val = small.csr()  # the first P/3 pairs in (depth, index) order, still tile-sorted
    assert off[-1] == P // 3 and np.all(np.diff(off) >= 0)


def test_deep_scene_radix_binning():
    """More than 512 pairs per tile on average: the build takes the two stable radix sorts (blocking and
    capacity mode alike) -- the lists match the oracle's, capacity mode reproduces them, an undersized
    capacity raises the overflow flag."""
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.scenes as sc
    from parity import O, run_oracle

    K, n, W, H = 30_000, 4, 96, 64
    arrays = _pinhole_scene(K, n, 11)
    spec = sc.look_at((0.0, 0.0, -4.0), (0.0, 0.0, 0.0), W, H, 120.0, 120.0, W / 2, H / 2)
    splats = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    cam = gb.PinholeCamera.from_spec(spec)
    ref = gb.build_binning(splats, cam)
    P, tiles = ref.total, ref.tiles_x * ref.tiles_y
    assert P > 512 * tiles, (P, tiles)  # a deep scene
    off, val = ref.csr()
    orc = run_oracle(arrays, n, O.Cam.from_spec(spec), O.Cfg(), None)
    np.testing.assert_array_equal(off, orc["offsets"])
    np.testing.assert_array_equal(val, orc["values"])
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    for cap in (P, P + 4096):
        b = gb.TileBinning()
        b.set_capacity(cap, flag)
        gb.build_binning(splats, cam, out=b)
        assert int(flag) == 0 and b.total == P
        o2, v2 = b.csr()
        np.testing.assert_array_equal(o2, off)
        np.testing.assert_array_equal(v2, val)
    small = gb.TileBinning()
    small.set_capacity(max(513 * tiles, P - 1000), flag)
    gb.build_binning(splats, cam, out=small)
    assert int(flag) == 1


def _trainer_scene():
    import paper_2412_12734_b200.scenes as sc

    n, K, W, H = 4, 3000, 96, 80
    arrays = _pinhole_scene(K, n, 5)
    specs = [sc.look_at((3.0 * np.cos(a), 0.7, 3.0 * np.sin(a)), (0.0, 0.0, 0.0), W, H, 90.0, 90.0, 48.0, 40.0)
             for a in (0.3, 2.1, 4.0)]
    targets = [sc.uniform_image(100 + v, W, H) for v in range(3)]
    return n, arrays, specs, targets


@pytest.mark.parametrize("mode", ["capacity", "graph", "graph_host", "overflow", "fused"])
def test_trainer_modes_match_blocking(mode):
    """The step's gradients with capacity-mode binning, with the view work replayed as a CUDA graph,
    after a capacity overflow (the step is redone with larger buffers), and with the fused
    forward+loss+backward kernel, equal the blocking eager step's (atomics order aside)."""
    import torch

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200.train import ViewShardedTrainer

    n, arrays, specs, targets = _trainer_scene()
    cams = [gb.PinholeCamera.from_spec(s) for s in specs]
    tg = [torch.as_tensor(t).cuda() for t in targets]

    def make(**kw):
        s = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
        return ViewShardedTrainer(s, cams, [0, 1, 2], **kw)

    ref = make(async_binning=False)
    ref._views_checked(lambda: ref._run_views(tg))
    want = {k: v.cpu().numpy().astype(np.float64) for k, v in ref.grads.tensors().items() if v is not None}
    want_loss = ref.losses.cpu().numpy()
    P = max(ref.pairs)
    tr = make(graph=mode.startswith("graph"), fused=mode == "fused")
    tr.graph_host = mode == "graph_host"
    tr._set_capacity(P // 4 if mode == "overflow" else P, exact=True)
    runs = 3 if mode.startswith("graph") else 1  # eager + capture, then replays
    host = [torch.as_tensor(t).pin_memory() for t in targets]
    for _ in range(runs):
        if mode == "graph_host":  # pinned host targets, H2D copies inside the graph
            tr._views_checked(lambda: tr._run_host_views(host))
        else:
            tr._views_checked(lambda: tr._run_views(tg))
        torch.cuda.synchronize()
        got = {k: v.cpu().numpy().astype(np.float64) for k, v in tr.grads.tensors().items() if v is not None}
        for k, w in want.items():
            np.testing.assert_allclose(got[k], w, rtol=1e-4, atol=1e-6 * np.abs(w).max(), err_msg=k)
        np.testing.assert_allclose(tr.losses.cpu().numpy(), want_loss, rtol=1e-5)
    assert tr.overflows == (1 if mode == "overflow" else 0)
    if mode.startswith("graph"):
        assert tr._graph is not None
    s, v = tr.pair_stats()  # capacity mode: the last step's views
    assert v == 3 and s == sum(ref.pairs)
    # and full steps (collective + Adam) run in every mode, alternating the device and host inputs
    tr.step(tg)
    tr.step_host(host)
    tr.step(tg)
    torch.cuda.synchronize()


def test_sharded_adam_single_rank_matches_adam_step():
    """ShardedAdam at world size 1 (gb_adam_segments over the flat parameter buffer) equals gb_adam_step
    bit for bit, and its non-finite guard raises without updating anything."""
    import torch

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200.train import ShardedAdam

    n, K = 4, 1001
    arrays = _pinhole_scene(K, n, 3)
    a = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    b = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    ga, gb_ = gb.GradientBuffer(a), gb.GradientBuffer(b, multiple=4)
    rng = np.random.default_rng(5)
    g = torch.as_tensor(rng.standard_normal(ga.flat.numel()), dtype=torch.float32).cuda()
    ga.flat.copy_(g)
    gb_.flat.copy_(g)
    lrs = gb.LearningRates(position_gamma=0.9)
    sa = gb.AdamState(a)
    sb = gb.AdamState(b, moments=False)
    opt = ShardedAdam(b, gb_, sb)
    for _ in range(3):
        gb.adam_step(a, ga, sa, lrs, check_finite=True)
        opt.step(lrs, check_finite=True)
    torch.cuda.synchronize()
    for f, t in a.tensors().items():
        assert torch.equal(t, b.tensors()[f]), f
    assert sa.t == sb.t == 3
    before = {f: t.clone() for f, t in b.tensors().items()}
    gb_.log_scale.view(-1)[7] = float("inf")
    with pytest.raises(gb.raster.NonFinite, match="log_scale"):
        opt.step(lrs, check_finite=True)
    for f, t in b.tensors().items():
        assert torch.equal(t, before[f]), f


def test_profile_intervals_cover_the_launches():
    """gb_context_profile_intervals: one (start, stop) per recorded launch, ordered after the reference event,
    inside the timed window, and their lengths sum to gb_context_profile_read's total."""
    import torch

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200.raster import context

    n, arrays, specs, targets = _trainer_scene()
    splats = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    cam = gb.PinholeCamera.from_spec(specs[0])
    ctx = context(splats.device)
    ctx.profile(True)
    ctx.profile_read()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(3):
        b = gb.build_binning(splats, cam)
        gb.render_forward(splats, cam, b)
    ev1.record()
    torch.cuda.synchronize()
    iv = ctx.profile_intervals(ev0, "forward")
    total = ev0.elapsed_time(ev1)
    assert len(iv) == 3
    assert all(0.0 <= a <= c <= total + 1e-3 for a, c in iv)
    assert all(iv[i][1] <= iv[i + 1][0] + 1e-3 for i in range(2))  # one stream: in order
    ms, cnt = ctx.profile_read()["forward"]
    ctx.profile(False)
    assert cnt == 3 and abs(sum(c - a for a, c in iv) - ms) < 1e-3 * max(1.0, ms)


_FAKE_RANK_SCRIPT = r"""
import sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
from torch.testing._internal.distributed.fake_pg import FakeStore
dist.init_process_group('fake', store=FakeStore(), rank=1, world_size=2)
_rs = dist.reduce_scatter_tensor
def _reduce_scatter(out, inp, *a, **k):  # the fake collective writes nothing: emulate a zero peer
    _rs(out, inp, *a, **k)
    out.copy_(inp[out.numel():2 * out.numel()])
dist.reduce_scatter_tensor = _reduce_scatter
import paper_2412_12734_b200 as gb
from paper_2412_12734_b200.train import ViewShardedTrainer
from test_gpu_train import _trainer_scene
from parity import O
n, arrays, specs, targets = _trainer_scene()
splats = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
cams = [gb.PinholeCamera.from_spec(s) for s in specs]
tr = ViewShardedTrainer(splats, cams, [0, 1, 2], graph=True)
opt = tr.opt
assert opt.world == 2 and opt.rank == 1 and opt.lo == opt.S and opt.flat.numel() == 2 * opt.S
before = opt.flat.clone()
tg = [torch.as_tensor(t).cuda() for t in targets]
host = [torch.as_tensor(t).pin_memory() for t in targets]
for _ in range(2):
    tr.step(tg)
tr.step_host(host)
torch.cuda.synchronize()
lo, S = opt.lo, opt.S
assert not torch.equal(opt.flat[lo:lo + S], before[lo:lo + S]), 'own slice must be updated'
assert torch.isfinite(opt.flat).all()
assert tr.state.t == 3 and tr._graph is not None
print('fake-rank ok')
"""


def test_two_rank_code_path_with_fake_process_group(tmp_path):
    """The multi-GPU step's code path at world size 2 on one GPU, with torch's fake process group (its
    collectives move no data; the reduce-scatter is emulated with a zero peer): the reduce-scatter /
    min-all-reduce / in-place all-gather calls, rank 1's slice and segments, graph capture and the
    host-input step all run, and rank 1's half of the parameters is updated."""
    import subprocess
    import sys

    script = tmp_path / "fake_rank.py"
    script.write_text(_FAKE_RANK_SCRIPT)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, str(script), root], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "fake-rank ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_step_overflow_vetoes_adam_and_redoes():
    """step() with the Adam overlap reads back once, after Adam is queued: a view that outgrows its pair
    buffers vetoes the update (folded into the sharded optimiser's agreed flag) and the step is redone
    with larger buffers -- same gradients and step count as an uninterrupted run."""
    import torch

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200.train import ViewShardedTrainer

    n, arrays, specs, targets = _trainer_scene()
    cams = [gb.PinholeCamera.from_spec(s) for s in specs]
    tg = [torch.as_tensor(t).cuda() for t in targets]

    def make(**kw):
        s = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
        return ViewShardedTrainer(s, cams, [0, 1, 2], **kw)

    ref, tr = make(async_binning=False), make()
    assert tr.overlap_adam and tr.overlap_read
    for t in (ref, tr):
        t.step(tg)  # tr: blocking first step, then capacity mode
    P = max(ref.pairs)
    tr._set_capacity(P // 4, exact=True)
    ref.step(tg)
    tr.step(tg)
    torch.cuda.synchronize()
    assert tr.overflows == 1 and tr.capacity >= P and tr.state.t == ref.state.t == 2
    for k, w in ref.grads.tensors().items():
        w = w.cpu().numpy().astype(np.float64)
        np.testing.assert_allclose(tr.grads.tensors()[k].cpu().numpy(), w, rtol=1e-3, atol=1e-5 * np.abs(w).max(),
                                   err_msg=k)
    for k, w in ref.splats.tensors().items():
        np.testing.assert_allclose(tr.splats.tensors()[k].cpu().numpy(), w.cpu().numpy(), atol=2e-3, err_msg=k)


def test_host_step_overflow_vetoes_adam_and_redoes():
    """step_host: the same single read after Adam (losses and the agreed flag together), the same veto."""
    import torch

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200.train import ViewShardedTrainer

    n, arrays, specs, targets = _trainer_scene()
    cams = [gb.PinholeCamera.from_spec(s) for s in specs]
    host = [torch.as_tensor(t).pin_memory() for t in targets]

    def make(**kw):
        s = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
        return ViewShardedTrainer(s, cams, [0, 1, 2], **kw)

    ref, tr = make(async_binning=False), make()
    for t in (ref, tr):
        t.step_host(host)
    P = max(ref.pairs)
    tr._set_capacity(P // 4, exact=True)
    want = ref.step_host(host).clone()
    got = tr.step_host(host).clone()
    torch.cuda.synchronize()
    assert tr.overflows == 1 and tr.capacity >= P and tr.state.t == ref.state.t == 2
    np.testing.assert_allclose(got.numpy(), want.numpy(), rtol=1e-5)
    for k, w in ref.splats.tensors().items():
        np.testing.assert_allclose(tr.splats.tensors()[k].cpu().numpy(), w.cpu().numpy(), atol=2e-3, err_msg=k)


def test_view_lanes_match_one_lane_at_configs3_size():
    """configs[3] shape (1M surfels, 8x8 textures, 8 Fibonacci views at 1600x1064): the step's gradients with
    four view lanes (concurrent K4/K5 on four streams into one buffer) equal the one-lane step's, up to
    atomics order.  A lost update (a K5 read-modify-write racing another lane's) would move an entry by a
    whole view's contribution."""
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.scenes as sc
    from paper_2412_12734_b200.train import ViewShardedTrainer

    cfg3 = sc.baseline_config(3)
    arrays = cfg3.arrays()
    cams = [gb.PinholeCamera.from_spec(c) for c in cfg3.cameras]
    views = list(range(8))
    tg = [torch.from_numpy(cfg3.target(v)).cuda() for v in views]

    def grads(lanes):
        s = gb.SplatSet.from_numpy(cfg3.mode, gb.ColorGridConfig(cfg3.n), **arrays)
        tr = ViewShardedTrainer(s, cams, views, lanes=lanes, async_binning=False)
        tr._views_checked(lambda: tr._run_views(tg))
        torch.cuda.synchronize()
        out = {k: v.cpu().numpy().astype(np.float64) for k, v in tr.grads.tensors().items() if v is not None}
        del tr, s
        torch.cuda.empty_cache()
        return out

    one = grads(1)
    four = grads(4)
    for k, w in one.items():
        rms = float(np.sqrt(np.mean(w * w))) + 1e-30
        bad = np.abs(four[k] - w) > 1e-3 * np.abs(w) + 1e-3 * rms
        assert int(bad.sum()) == 0, (k, int(bad.sum()), float(np.abs(four[k] - w).max()), rms)


def test_comm_c_abi_single_rank():
    """The C-ABI NCCL layer at world size 1 (ncclCommInitRank over one GPU): every collective of the step
    runs on the context's stream and is the identity; the communicator reports no asynchronous error."""
    import ctypes as C

    import torch

    from paper_2412_12734_b200 import _lib
    from paper_2412_12734_b200._lib import check, lib
    from paper_2412_12734_b200.raster import context

    ctx = context("cuda")
    uid = (C.c_uint8 * _lib.COMM_ID_BYTES)()
    check(lib.gb_comm_unique_id(uid), "gb_comm_unique_id")
    h = C.c_void_p()
    check(lib.gb_comm_init_rank(ctx.handle, 1, uid, 0, C.byref(h)), "gb_comm_init_rank")
    n, r = C.c_int32(), C.c_int32()
    check(lib.gb_comm_info(h, C.byref(n), C.byref(r)), "gb_comm_info")
    assert (n.value, r.value) == (1, 0)
    x = torch.arange(1000, dtype=torch.float32, device="cuda")
    want = x.clone()
    check(lib.gb_allreduce_grads(ctx.handle, h, x.data_ptr(), x.numel()), "allreduce")
    y = torch.empty_like(x)
    check(lib.gb_reduce_scatter_grads(ctx.handle, h, x.data_ptr(), y.data_ptr(), x.numel()), "reduce_scatter")
    z = torch.empty_like(x)
    check(lib.gb_all_gather_params(ctx.handle, h, y.data_ptr(), z.data_ptr(), y.numel()), "all_gather")
    f = torch.tensor([12345], dtype=torch.int64, device="cuda")
    check(lib.gb_allreduce_flag_min(ctx.handle, h, f.data_ptr()), "flag")
    check(lib.gb_sync(ctx.handle), "sync")
    assert torch.equal(x, want) and torch.equal(y, want) and torch.equal(z, want) and int(f) == 12345
    check(lib.gb_comm_check(h), "gb_comm_check")
    bad = lib.gb_allreduce_grads(ctx.handle, None, x.data_ptr(), 4)
    assert bad == _lib.GB_INVALID_ARGUMENT
    check(lib.gb_comm_destroy(h), "gb_comm_destroy")


def test_padded_texel_gradients_match_reference_layout():
    """K4 with the RGBA-padded texel-gradient layout (gb_context_set_texel_grad_stride(4), then
    gb_texel_grads_unpad) gives the reference layout's texel gradients (atomics order aside) and leaves the
    other groups unchanged; the padding floats are never written."""
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.scenes as sc

    for n in (3, 8):
        c = sc.baseline_config(0, count=20_000, n=n)
        s = gb.SplatSet.from_numpy(c.mode, gb.ColorGridConfig(n), **c.arrays())
        cam = gb.PinholeCamera.from_spec(c.cameras[0])
        b = gb.build_binning(s, cam)
        out = gb.render_forward(s, cam, b)
        ig = torch.sign(torch.randn((cam.height, cam.width, 3), device="cuda"))
        ref = gb.render_backward(s, cam, b, out, ig)
        pad = torch.full((ref.grid.numel() // 3 * 4,), 7.0, device="cuda")
        pad.view(-1, 4)[:, :3] = 0.0
        got = gb.render_backward(s, cam, b, out, ig, texel_grad=pad)
        torch.cuda.synchronize()
        assert bool((pad.view(-1, 4)[:, 3] == 7.0).all())
        assert float(got.grid.abs().max()) == 0.0  # the reference-layout group was not touched
        pad.view(-1, 4)[:, 3] = 0.0
        gb.raster.texel_grads_unpad(pad, got.grid.view(-1))
        torch.cuda.synchronize()
        for k, v in ref.tensors().items():
            w = got.tensors()[k]
            scale = float(v.abs().max()) + 1e-30
            assert float((w - v).abs().max()) <= 1e-5 * scale, (n, k)


def test_pair_capacity_limits():
    """The pair count is indexed with int by the sorts: the C-ABI rejects capacities >= 2^31 - 1 and the
    trainer never inflates a capacity past it (the 1.1 margin could overflow the sort's int)."""
    import torch

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200._lib import InvalidArgument
    from paper_2412_12734_b200.train import PAIR_LIMIT, ViewShardedTrainer

    b = gb.TileBinning()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    with pytest.raises(InvalidArgument):
        b.set_capacity(2 ** 31 - 1, flag)
    b.set_capacity(2 ** 31 - 2, flag)  # the largest accepted
    b.set_capacity(0, flag)
    n, arrays, specs, targets = _trainer_scene()
    s = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    tr = ViewShardedTrainer(s, [gb.PinholeCamera.from_spec(c) for c in specs], [0, 1, 2])
    tr._set_capacity(PAIR_LIMIT - 100)  # the 1.1x margin is clamped below the limit
    assert tr.capacity == PAIR_LIMIT - 1
    with pytest.raises(RuntimeError):
        tr._set_capacity(PAIR_LIMIT)


def test_rgba_texels_same_results():
    """gb_context_set_texel_rgba: K3/K4 reading the RGBA-padded texel copy (gb_texels_pad) give the same
    image and gradients as the reference layout, bit for bit; the backward insists on stride-4 texel
    gradients with it."""
    import torch

    import paper_2412_12734_b200 as gb
    from paper_2412_12734_b200.raster import GBError, texel_grads_unpad, texels_pad

    n, K, W, H = 4, 4000, 128, 96
    arrays = _pinhole_scene(K, n, 21)
    import paper_2412_12734_b200.scenes as sc

    spec = sc.look_at((0.0, 0.3, -3.5), (0.0, 0.0, 0.0), W, H, 110.0, 110.0, W / 2, H / 2)
    splats = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    cam = gb.PinholeCamera.from_spec(spec)
    b = gb.build_binning(splats, cam)
    rgba = torch.zeros(splats.grid.numel() // 3 * 4, dtype=torch.float32, device="cuda")
    texels_pad(splats.grid.view(-1), rgba)
    out3 = gb.render_forward(splats, cam, b)
    out4 = gb.render_forward(splats, cam, b, texels_rgba=rgba)
    assert torch.equal(out3.color, out4.color) and torch.equal(out3.last_rank, out4.last_rank)
    ig = torch.sign(torch.randn(H, W, 3, device="cuda", generator=torch.Generator("cuda").manual_seed(3)))
    pad3 = torch.zeros_like(rgba)
    pad4 = torch.zeros_like(rgba)
    g3 = gb.render_backward(splats, cam, b, out3, ig, texel_grad=pad3)
    g4 = gb.render_backward(splats, cam, b, out4, ig, texel_grad=pad4, texels_rgba=rgba)
    # same arithmetic; float atomics may order the adds differently (the last bits, relative to the field)
    pairs = [(k, g4.tensors()[k], v) for k, v in g3.tensors().items() if k != "grid"] + [("texels", pad4, pad3)]
    for k, a, r in pairs:
        err = float((a - r).abs().max()) / (1e-12 + float(r.abs().max()))
        assert err < 1e-5, (k, err)
    with pytest.raises(GBError):
        gb.render_backward(splats, cam, b, out4, ig, texels_rgba=rgba)  # stride-3 gradients with RGBA texels


def test_image_side_limit():
    """K4 packs a pixel's (x, y) into 16 + 16 bits, so the C-ABI rejects images wider or taller than
    65536 - 16 pixels (tiles overhang the image by < 16 px) with GB_NOT_SUPPORTED, before any launch."""
    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.scenes as sc
    from paper_2412_12734_b200.raster import GBError

    n, K = 2, 64
    arrays = _pinhole_scene(K, n, 5)
    splats = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(n), **arrays)
    for W, H, ok in ((65520, 8, True), (65521, 8, False), (8, 65521, False)):
        spec = sc.look_at((0.0, 0.3, -3.5), (0.0, 0.0, 0.0), W, H, 110.0, 110.0, W / 2, H / 2)
        cam = gb.PinholeCamera.from_spec(spec)
        if ok:
            gb.build_binning(splats, cam)
        else:
            with pytest.raises(GBError, match="too large"):
                gb.build_binning(splats, cam)
