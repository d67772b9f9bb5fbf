"""One configs[3] view through every kernel of the step, eagerly (for `ncu --set full` captures of each
kernel: K1 projection, K2 depth sort / scan / duplicate / tile sort / ranges, K3 forward, K6 L1, K4
backward, K5 chain, K7 Adam check + update).  Development aid, not product.

    ncu --set full --clock-control none --import-source on -o gpurun_out/ncu_all python tools/ncu_view.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_12734_b200 as gb  # noqa: E402
import paper_2412_12734_b200.scenes as sc  # noqa: E402


def main(view=0):
    c = sc.baseline_config(3)
    s = gb.SplatSet.from_numpy(c.mode, gb.ColorGridConfig(c.n), **c.arrays())
    cam = gb.PinholeCamera.from_spec(c.cameras[view])
    target = torch.as_tensor(c.target(view)).cuda()
    grads = gb.GradientBuffer(s)
    state = gb.AdamState(s)
    torch.cuda.synchronize()
    # the trainer's configuration: RGBA-padded texels (one 16-B load per texel) and texel gradients
    rgba = torch.zeros(grads.grid.numel() // 3 * 4, device="cuda")
    gb.raster.texels_pad(s.grid.view(-1), rgba)
    b = gb.build_binning(s, cam)
    out = gb.render_forward(s, cam, b, texels_rgba=rgba)
    loss, ig = gb.l1_loss(out.color, target)
    pad = torch.zeros(grads.grid.numel() // 3 * 4, device="cuda")
    gb.render_backward(s, cam, b, out, ig, grads, texel_grad=pad, texels_rgba=rgba)
    gb.adam_step(s, grads, state, gb.LearningRates())
    torch.cuda.synchronize()
    print("ncu_view ok: P =", b.total, "loss =", float(loss))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
