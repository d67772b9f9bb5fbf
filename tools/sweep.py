"""BASELINE configs[4]: texture-resolution x density sweep at 1600x1064, forward + backward per view.

    python tools/sweep.py [--counts 100000,1000000,4000000] [--tex 1,4,8,16] [--iters 5] [--out gpurun_out/sweep]

Geometry comes from the seeded host generator (Rng(seed)); textures for the sweep are drawn
on the device (torch, seeded) so the 4M x 16x16 cell (12.3 GB of texels) does not need a host copy.
Per cell: P (tile/primitive pairs), binning / forward / backward ms (CUDA events, median of --iters after
2 warm-ups), megapixels/s of one view, and K3/K4 against SURVEY §8(d)'s algorithmic bytes.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2412_12734_b200 as gb  # noqa: E402
import paper_2412_12734_b200.scenes as sc  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def cell(K, T, iters):
    c = sc.baseline_config(4, count=K, n=1)
    geo = c.arrays()
    g = torch.Generator(device="cuda").manual_seed(1)
    arrays = {k: v for k, v in geo.items() if v is not None and k != "grid"}
    splats = gb.SplatSet.from_numpy(c.mode, gb.ColorGridConfig(T), **arrays)
    splats.grid = torch.rand((K, 3 * T * T), generator=g, device="cuda", dtype=torch.float32)
    cam = gb.PinholeCamera.from_spec(c.cameras[0])
    W, H = cam.width, cam.height
    target = torch.rand((H, W, 3), generator=g, device="cuda", dtype=torch.float32)
    grads = gb.GradientBuffer(splats)
    # the trainer's configuration: RGBA-padded texels and texel gradients
    rgba = torch.zeros(splats.grid.numel() // 3 * 4, device="cuda")
    gb.raster.texels_pad(splats.grid.view(-1), rgba)
    pad = torch.zeros_like(rgba)
    b = gb.TileBinning()
    out = gb.RenderOutput(W, H, "cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    rec = []
    for it in range(iters + 2):
        # gradient zeroing is once per training step, not per view (the trainer sums all views into one
        # buffer): kept outside the timed region -- at 4M x 16x16 it is 29 GB of writes
        grads.zero_()
        pad.zero_()
        ev[0].record()
        gb.build_binning(splats, cam, gb.RasterConfig(), out=b)
        ev[1].record()
        gb.render_forward(splats, cam, b, out, texels_rgba=rgba)
        ev[2].record()
        _, ig = gb.l1_loss(out.color, target)
        ev[3].record()
        gb.render_backward(splats, cam, b, out, ig, grads, texel_grad=pad, texels_rgba=rgba)
        ev[4].record()
        torch.cuda.synchronize()
        if it >= 2:
            rec.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)])
    r = np.median(np.array(rec), axis=0)
    P = b.total
    tiles = b.tiles_x * b.tiles_y
    npx = W * H
    Bh, Bt = 40, 12 * T * T
    k3 = P * (4 + Bh + Bt) + 8 * tiles + 20 * npx
    k4 = P * (4 + 2 * Bh + 2 * Bt) + 8 * tiles + 20 * npx
    total = float(r[0] + r[1] + r[2] + r[3])
    pk = peak()
    return dict(K=K, T=T, pairs=int(P), binning_ms=round(float(r[0]), 4), forward_ms=round(float(r[1]), 4),
                backward_ms=round(float(r[3]), 4), fwd_bwd_ms=round(total, 4),
                mps=round(npx / 1e6 / (total / 1e3), 1),
                k3_frac=round(k3 / (r[1] / 1e3) / 1e9 / pk, 4), k4_frac=round(k4 / (r[3] / 1e3) / 1e9 / pk, 4))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--counts", default="100000,1000000,4000000")
    ap.add_argument("--tex", default="1,4,8,16")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep"))
    a = ap.parse_args()
    rows = []
    for K in [int(x) for x in a.counts.split(",")]:
        for T in [int(x) for x in a.tex.split(",")]:
            try:
                row = cell(K, T, a.iters)
            except Exception as e:  # report the cell, keep sweeping
                row = dict(K=K, T=T, error=str(e)[:200])
            torch.cuda.empty_cache()
            print(json.dumps(row), flush=True)
            rows.append(row)
    md = ["| K | T | pairs P | binning ms | forward ms | backward ms | fwd+bwd ms | MP/s | K3 frac | K4 frac |",
          "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        if "error" in r:
            md.append(f"| {r['K']} | {r['T']} | error: {r['error']} |||||||")
        else:
            md.append(f"| {r['K']:,} | {r['T']} | {r['pairs']:,} | {r['binning_ms']} | {r['forward_ms']} | "
                      f"{r['backward_ms']} | {r['fwd_bwd_ms']} | {r['mps']} | {r['k3_frac']} | {r['k4_frac']} |")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    open(a.out + ".md", "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
