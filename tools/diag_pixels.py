"""Per-pixel attribution of a gradient discrepancy (development aid): for primitive PRIM of the configs[4]
K x T case, compare the GPU's and the oracle's gradient of that primitive from one-hot image gradients at
each pixel of its tiles in the tile-row subset.
    python tools/diag_pixels.py K T PRIM [stride]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from parity import O, subset_rows  # noqa: E402


def main(K, T, prim, stride=8):
    import torch

    import paper_2412_12734_b200 as gb
    import paper_2412_12734_b200.scenes as sc

    c = sc.baseline_config(4, count=K, n=T)
    cam = O.Cam.from_spec(c.cameras[0])
    arrays = c.arrays()
    ig_full = np.random.default_rng(0).choice(np.array([-1.0, 1.0]), size=(cam.height, cam.width, 3))
    cfg = O.Cfg()
    geo = {f: (None if f == "grid" else arrays.get(f)) for f in O.FIELDS}
    geo["grid"] = np.zeros((K, 3), np.float32)
    offsets, values, tiles = O.build_binning(O.Scene64(geo, 1), cam, cfg)
    tx, ty = tiles
    rows = subset_rows(ty, stride)
    ts = cfg.tile_size
    cand_tiles = [t for t in range(tx * ty) if (t // tx) in rows and prim in values[offsets[t]:offsets[t + 1]]]
    # oracle over the candidate tiles' lists (primitives compacted in index order)
    keep = np.zeros(tx * ty, bool)
    keep[cand_tiles] = True
    counts = np.diff(offsets)
    sub_vals = values[np.repeat(keep, counts)]
    ids = np.unique(sub_vals)
    remap = np.full(K, -1, np.int64)
    remap[ids] = np.arange(len(ids))
    sub_off = np.zeros(tx * ty + 1, np.int64)
    sub_off[1:] = np.cumsum(np.where(keep, counts, 0))
    sub_bin = (sub_off, remap[sub_vals].astype(np.int32), tiles)
    scene = O.Scene64({f: (None if arrays.get(f) is None else arrays[f][ids]) for f in O.FIELDS}, T)
    f = O.render_forward(scene, cam, cfg, sub_bin)
    pj = int(remap[prim])
    # GPU, whole scene
    s = gb.SplatSet.from_numpy(c.mode, gb.ColorGridConfig(T), **arrays)
    camg = gb.PinholeCamera.from_spec(cam)
    b = gb.build_binning(s, camg)
    out = gb.render_forward(s, camg, b)
    res = []
    for t in cand_tiles:
        y0, x0 = (t // tx) * ts, (t % tx) * ts
        for y in range(y0, min(cam.height, y0 + ts)):
            for x in range(x0, min(cam.width, x0 + ts)):
                ig = np.zeros_like(ig_full)
                ig[y, x] = ig_full[y, x]
                g = gb.render_backward(s, camg, b, out, torch.as_tensor(ig.astype(np.float32), device="cuda"))
                gp = g.position.view(-1, 3)[prim].cpu().numpy().astype(np.float64)
                go, _, _ = O.render_backward(scene, cam, cfg, sub_bin, f, ig, want_mag=False)
                op = go["position"].reshape(-1, 3)[pj]
                if np.abs(op).max() == 0 and np.abs(gp).max() == 0:
                    continue
                res.append(dict(x=x, y=y, gpu=gp.tolist(), ref=op.tolist(), diff=float(np.abs(gp - op).max()),
                                T=float(f["trans"][y, x]), last=int(f["last"][y, x]), kink=int(f["kink"][y, x]),
                                gpu_T=float(out.final_transmittance[y, x]), gpu_last=int(out.last_rank[y, x])))
    res.sort(key=lambda r: -r["diff"])
    tot_gpu = np.sum([r["gpu"] for r in res], axis=0)
    tot_ref = np.sum([r["ref"] for r in res], axis=0)
    print(json.dumps(dict(prim=prim, pixels=len(res), total_gpu=tot_gpu.tolist(), total_ref=tot_ref.tolist(),
                          worst=res[:12]), indent=1))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
