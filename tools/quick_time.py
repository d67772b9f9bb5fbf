"""Per-stage CUDA-event timing of one view (development aid)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2412_12734_b200 as gb
import paper_2412_12734_b200.scenes as sc

def main(idx=2, count=None, n=None, iters=5):
    c = sc.baseline_config(idx, count=count, n=n)
    t0 = time.time(); arr = c.arrays(); tgen = time.time() - t0
    splats = gb.SplatSet.from_numpy(c.mode, gb.ColorGridConfig(c.n), **arr)
    cam = gb.PinholeCamera.from_spec(c.cameras[0])
    target = torch.as_tensor(c.target(0)).cuda()
    grads = gb.GradientBuffer(splats)
    b = gb.TileBinning()
    out = gb.RenderOutput(cam.width, cam.height, "cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    res = []
    for it in range(iters + 3):
        ev[0].record()
        gb.build_binning(splats, cam, gb.RasterConfig(), out=b)
        ev[1].record()
        gb.render_forward(splats, cam, b, out)
        ev[2].record()
        loss, ig = gb.l1_loss(out.color, target)
        ev[3].record()
        grads.zero_()
        ev[4].record()
        gb.render_backward(splats, cam, b, out, ig, grads)
        ev[5].record()
        torch.cuda.synchronize()
        if it >= 3:
            res.append([ev[i].elapsed_time(ev[i + 1]) for i in range(5)])
    r = np.median(np.array(res), axis=0)
    print(json.dumps(dict(config=c.name, K=c.count, n=c.n, P=b.total, gen_s=round(tgen, 2),
                          binning_ms=r[0], forward_ms=r[1], loss_ms=r[2], zero_ms=r[3], backward_ms=r[4],
                          total_ms=float(r.sum()), loss=float(loss))))

if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
