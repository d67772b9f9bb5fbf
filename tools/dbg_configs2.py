"""Development aid: configs[2] parity details -- violating pixels with their oracle kink flags, and the
worst gradient entries (python tools/dbg_configs2.py [grad])."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2412_12734_b200.scenes as sc
from parity import O, run_gpu, run_oracle, compare_grads, RTOL, ATOL

want_grad = len(sys.argv) > 1 and sys.argv[1] == "grad"
c = sc.baseline_config(2)
cam = O.Cam.from_spec(c.cameras[0])
arrays = c.arrays()
ig = np.random.default_rng(0).choice(np.array([-1.0, 1.0]), size=(cam.height, cam.width, 3)) if want_grad else None
g = run_gpu(arrays, O.MODE_PINHOLE, c.n, c.cameras[0], O.Cfg(), ig)
o = run_oracle(arrays, c.n, cam, O.Cfg(), ig)
dc = np.abs(g["color"] - o["color"])
bad = (dc > ATOL + RTOL * np.abs(o["color"])).any(-1) & ((o["kink"] & 3) == 0)
ys, xs = np.nonzero(bad)
print("env", {k: v for k, v in os.environ.items() if k.startswith("GB_")}, "image violations", len(ys))
for y, x in zip(ys[:10], xs[:10]):
    print(dict(x=int(x), y=int(y), kink=int(o["kink"][y, x]), gpu=g["color"][y, x].tolist(),
               ref=o["color"][y, x].tolist(), T_gpu=float(g["trans"][y, x]), T_ref=float(o["trans"][y, x])))
if want_grad:
    st = compare_grads(g, o)
    for f, v in st.items():
        print(f, "strict", v["strict_violations"], "applicable", v["strict_violations_applicable"], "model",
              v["model_violations"], "worst", v["worst"][:2])
    pos = arrays["position"]; k = 977390
    print("primitive", k, "mean", pos[k].tolist(), "quat", arrays["quat"][k].tolist(), "log_scale",
          arrays["log_scale"][k].tolist(), "opacity", float(arrays["opacity_logit"][k]))
