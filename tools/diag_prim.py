"""Diagnose the worst fp32 model violations of a configs[4] tile-row case (development aid):
prints the offending primitives' parameters, view geometry and every gradient entry, GPU vs oracle.
    python tools/diag_prim.py K T [stride]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from parity import O, compare_grads, run_rows  # noqa: E402


def main(K, T, stride=8):
    import paper_2412_12734_b200.scenes as sc
    import paper_2412_12734_b200._lib as L

    c = sc.baseline_config(4, count=K, n=T)
    cam = O.Cam.from_spec(c.cameras[0])
    arrays = c.arrays()
    ig = np.random.default_rng(0).choice(np.array([-1.0, 1.0]), size=(cam.height, cam.width, 3))
    gpu, orc, info = run_rows(arrays, O.MODE_PINHOLE, T, cam, O.Cfg(), ig, stride=stride)
    st = compare_grads(gpu, orc)
    # recompute the compacted id list as run_rows does
    geo = {f: (None if f == "grid" else arrays.get(f)) for f in O.FIELDS}
    geo["grid"] = np.zeros((K, 3), np.float32)
    offsets, values, tiles = O.build_binning(O.Scene64(geo, 1), cam, O.Cfg())
    tx, ty = tiles
    rows = sorted(set(range(0, ty, stride)) | {ty - 1})
    keep_t = np.zeros(tx * ty, bool)
    for r in rows:
        keep_t[r * tx:(r + 1) * tx] = True
    ids = np.unique(values[np.repeat(keep_t, np.diff(offsets))])
    prims = set()
    for f in ("position", "quat", "log_scale", "opacity_logit"):
        for e in st[f]["model_list"] + st[f]["applicable"]:
            width = {"position": 3, "quat": 4, "log_scale": 2, "opacity_logit": 1}[f]
            prims.add(e["index"] // width)
    R = np.asarray(cam.rot)
    tr = np.asarray(cam.trans)
    out = dict(library=os.path.basename(L.LIB_PATH), prims=[])
    for p in sorted(prims):
        k = int(ids[p])
        pc = R @ arrays["position"][k].astype(np.float64) + tr
        q = arrays["quat"][k].astype(np.float64)
        q /= np.linalg.norm(q)
        w, x, y, z = q
        nrm = np.array([2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)])
        view = pc / np.linalg.norm(pc)
        rec = dict(subset_index=p, primitive=k, cam_pos=pc.tolist(), scale=np.exp(arrays["log_scale"][k]).tolist(),
                   alpha_k=float(1 / (1 + np.exp(-arrays["opacity_logit"][k]))),
                   cos_view_normal=float(abs(np.dot(R @ nrm, view))),
                   proj_px=(1000.0 * np.exp(arrays["log_scale"][k]) / pc[2]).tolist(), grads={})
        for f, wdt in (("position", 3), ("quat", 4), ("log_scale", 2), ("opacity_logit", 1)):
            g = gpu["grads"][f].reshape(-1, wdt)[p]
            o = orc["grads"][f].reshape(-1, wdt)[p]
            m = orc["mag"][f].reshape(-1, wdt)[p]
            tm = orc["tmag"][f].reshape(-1, wdt)[p]
            sl = orc["slack"][f].reshape(-1, wdt)[p]
            rec["grads"][f] = dict(gpu=g.tolist(), ref=o.tolist(), mag=m.tolist(), tmag=tm.tolist(), slack=sl.tolist())
        out["prims"].append(rec)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
