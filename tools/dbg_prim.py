"""Development aid: locate the pixels behind one primitive's gradient mismatch on configs[2] by masking the
image cotangent to pixel windows (python tools/dbg_prim.py <primitive>)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2412_12734_b200 as gb
import paper_2412_12734_b200.scenes as sc
from parity import O

k = int(sys.argv[1]) if len(sys.argv) > 1 else 977390
c = sc.baseline_config(2)
cam = O.Cam.from_spec(c.cameras[0])
arrays = c.arrays()
W, H = cam.width, cam.height
ig_full = np.random.default_rng(0).choice(np.array([-1.0, 1.0]), size=(H, W, 3))
splats = gb.SplatSet.from_numpy(O.MODE_PINHOLE, gb.ColorGridConfig(c.n), **arrays)
gcam = gb.PinholeCamera.from_spec(c.cameras[0])
b = gb.build_binning(splats, gcam, gb.RasterConfig())
out = gb.render_forward(splats, gcam, b)
scene = O.Scene64(arrays, c.n)
ob = O.build_binning(scene, cam, O.Cfg())
of = O.render_forward(scene, cam, O.Cfg(), ob)

def both(mask):
    ig = ig_full * mask[..., None]
    g = gb.render_backward(splats, gcam, b, out, torch.as_tensor(ig.astype(np.float32)).cuda())
    gg = g.tensors()["opacity_logit"][k].item(), g.tensors()["grid"][k].cpu().numpy()
    og, _, _ = O.render_backward(scene, cam, O.Cfg(), ob, of, ig)
    return gg[0], og["opacity_logit"][k], np.abs(gg[1] - og["grid"][k]).max()

x0, x1, y0, y1 = 1340, 1400, 35, 90
m = np.zeros((H, W)); m[y0:y1, x0:x1] = 1
print("window", (x0, x1, y0, y1), both(m))
# bisect: single pixels with the largest opacity discrepancy
res = []
for y in range(y0, y1, 4):
    for x in range(x0, x1, 4):
        m = np.zeros((H, W)); m[y:y + 4, x:x + 4] = 1
        ga, oa, gd = both(m)
        if abs(ga - oa) > 1e-6 + 1e-4 * abs(oa) or gd > 1e-5:
            res.append((x, y, ga, oa, gd))
            print("block", x, y, ga, oa, gd, flush=True)
for x, y, *_ in res[:3]:
    for yy in range(y, y + 4):
        for xx in range(x, x + 4):
            m = np.zeros((H, W)); m[yy, xx] = 1
            ga, oa, gd = both(m)
            if abs(ga - oa) > 1e-7 + 1e-4 * abs(oa) or gd > 1e-6:
                print("pixel", xx, yy, ga, oa, gd, "kink", int(of["kink"][yy, xx]), "last", int(out.last_rank[yy, xx]),
                      int(of["last"][yy, xx]), "T", float(out.final_transmittance[yy, xx]), float(of["trans"][yy, xx]),
                      flush=True)
