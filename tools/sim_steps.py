"""Development aid: count compositor steps per warp for different lane-group layouts on a configs[3] view.

Uses the fp64 oracle for binning and the forward `last` ranks, and numpy for the per-(pixel, entry)
alpha-skip mask on a sample of tiles.  Reports, per layout, the steps a warp needs in the backward when
each group of G lanes (a 4 x G/4 pixel block) walks only the entries that are active for at least one of
its pixels ("ideal culling"), compared with one warp per entry over the union.

    python tools/sim_steps.py [tiles_sampled=200] [view=0]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
import paper_2412_12734_b200.scenes as sc  # noqa: E402


def geom(a, cam, ids):
    q = a["quat"][ids]
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    tu = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)], 1)
    tv = np.stack([2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)], 1)
    R = cam.rot.reshape(3, 3)
    s = np.exp(a["log_scale"][ids])
    pc = a["position"][ids] @ R.T + cam.trans
    M = np.stack([s[:, :1] * (tu @ R.T), s[:, 1:] * (tv @ R.T), pc], 2)  # (k, 3 rows, 3 cols)
    alpha_k = 1 / (1 + np.exp(-a["opacity_logit"][ids]))
    return M, alpha_k


def alpha_mask(M, alpha_k, cam, px, py, skip=1 / 255):
    dxn = (px - cam.cx) / cam.fx  # (npx,)
    dyn = (py - cam.cy) / cam.fy
    a = M[:, None, :, 0 + 0] if False else None
    M0, M1, M2 = M[:, 0, :], M[:, 1, :], M[:, 2, :]  # rows
    A = M0[:, None, :] - dxn[None, :, None] * M2[:, None, :]
    B = M1[:, None, :] - dyn[None, :, None] * M2[:, None, :]
    c = np.cross(A, B)
    with np.errstate(divide="ignore", invalid="ignore"):
        u = c[..., 0] / c[..., 2]
        v = c[..., 1] / c[..., 2]
        t = M2[:, None, 0] * u + M2[:, None, 1] * v + M2[:, None, 2]
        al = np.minimum(alpha_k[:, None] * np.exp(-0.5 * (u * u + v * v)), 0.999)
    return (t > 0) & (al >= skip)


def main():
    nsample = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    view = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    c3 = sc.baseline_config(3)
    arr = c3.arrays()
    a = {k: (None if v is None else v.astype(np.float64)) for k, v in arr.items()}
    cam = O.Cam.from_spec(c3.cameras[view])
    scene = O.Scene64(arr, c3.n)
    cfg = O.Cfg()
    offsets, values, (tx, ty) = O.build_binning(scene, cam, cfg)
    fwd = O.render_forward(scene, cam, cfg, (offsets, values, (tx, ty)), kink=None)
    last = fwd["last"]
    rng = np.random.default_rng(0)
    nonempty = np.nonzero(np.diff(offsets) > 0)[0]
    tiles = rng.choice(nonempty, size=min(nsample, len(nonempty)), replace=False)
    lay = {"warp 8x4 (G=32)": 32, "G=16 (4x4)": 16, "G=8 (4x2)": 8, "G=4 (2x2)": 4}
    tot = {k: 0 for k in lay}
    tot_active_lanes = 0
    for t in tiles:
        ids = values[offsets[t]:offsets[t + 1]]
        tyy, txx = divmod(int(t), tx)
        for w in range(8):  # 8 warps of 8x4 pixels
            x0 = txx * 16 + (w % 2) * 8
            y0 = tyy * 16 + (w // 2) * 4
            xs, ys = np.meshgrid(np.arange(x0, x0 + 8), np.arange(y0, y0 + 4))
            xs, ys = xs.ravel(), ys.ravel()
            ok = (xs < cam.width) & (ys < cam.height)
            if not ok.any():
                continue
            xs, ys = xs[ok], ys[ok]
            lst = last[ys, xs]
            wl = lst.max()
            if wl < 0:
                continue
            M, ak = geom(a, cam, ids[: wl + 1])
            act = alpha_mask(M, ak, cam, xs + 0.5, ys + 0.5)  # (entries, px)
            act &= np.arange(wl + 1)[:, None] <= lst[None, :]
            tot_active_lanes += act.sum()
            lx, ly = xs - x0, ys - y0
            # per-lane batches: within each batch of B consecutive warp-active entries, every lane walks its own
            # active entries; the warp needs max over lanes of the count
            wact = act[act.any(1)]  # warp-active entries, in order
            for B in (4, 8, 16):
                key = f"lane batches B={B}"
                n = wact.shape[0]
                pad = (-n) % B
                wb = np.concatenate([wact, np.zeros((pad, wact.shape[1]), bool)]).reshape(-1, B, wact.shape[1])
                tot[key] = tot.get(key, 0) + wb.sum(1).max(1).sum()
            # consecutive warp-active entries with disjoint active-pixel sets composited in one step
            for cap in (2, 3, 4):
                key = f"disjoint groups <= {cap}"
                steps = 0
                union = None
                size = 0
                for row in wact:
                    if union is not None and size < cap and not (union & row).any():
                        union |= row
                        size += 1
                    else:
                        steps += 1
                        union = row.copy()
                        size = 1
                tot[key] = tot.get(key, 0) + steps
            for name, G in lay.items():
                if G == 32:
                    gid = np.zeros_like(lx)
                elif G == 16:
                    gid = lx // 4
                elif G == 8:
                    gid = (lx // 4) + 2 * (ly // 2)
                else:
                    gid = (lx // 2) + 4 * (ly // 2)
                ga = np.stack([act[:, gid == g].any(1) for g in np.unique(gid)], 1)  # (entries, groups)
                tot[name] += ga.sum(0).max()
                # ring of R shared 32-entry windows: a group may run at most R-1 windows ahead of the slowest
                for R in (2, 4):
                    key = f"{name} ring{R}"
                    n = ga.shape[0]
                    nw = (n + 31) // 32
                    ng = ga.shape[1]
                    lists = [[np.nonzero(ga[w * 32:(w + 1) * 32, gg])[0].tolist() for w in range(nw)] for gg in range(ng)]
                    wi = [0] * ng
                    pos = [0] * ng
                    steps = 0
                    def norm(gg):
                        while wi[gg] < nw and pos[gg] >= len(lists[gg][wi[gg]]):
                            wi[gg] += 1; pos[gg] = 0
                    for gg in range(ng):
                        norm(gg)
                    while any(wi[gg] < nw for gg in range(ng)):
                        lo = min(wi)
                        for gg in range(ng):
                            if wi[gg] < nw and wi[gg] < lo + R:
                                pos[gg] += 1
                                norm(gg)
                        steps += 1
                    tot[key] = tot.get(key, 0) + steps
                for ch in (32, 64):
                    key = f"{name} chunk{ch}"
                    n = ga.shape[0]
                    pad = (-n) % ch
                    gp = np.concatenate([ga, np.zeros((pad, ga.shape[1]), bool)]).reshape(-1, ch, ga.shape[1])
                    tot[key] = tot.get(key, 0) + gp.sum(1).max(1).sum()
    union = tot["warp 8x4 (G=32)"]
    print(f"tiles sampled {len(tiles)}; active (pixel, entry) pairs {tot_active_lanes}; "
          f"active lanes per union step {tot_active_lanes / max(1, union):.2f}")
    for name, v in sorted(tot.items()):
        print(f"{name:18s} steps {v:9d}  ratio {v / max(1, union):.3f}")


if __name__ == "__main__":
    main()
