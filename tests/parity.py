"""Shared parity helpers: run one scene through the CUDA path (C-ABI via the
package) and through the fp64 oracle, and compare them with the protocol of
SURVEY.md §8(c):

* tile lists (offsets + values): bit-exact;
* images: |d| <= atol + rtol*|ref| on RGB and alpha = 1 - T, exact last_rank,
  except pixels the oracle flags as within fp32 error of a threshold kink;
* gradients (same image_grad fed to both sides): |d| <= atol + rtol*|ref| +
  slack, where slack is the oracle's |terms| from kink-adjacent evaluations.
  A second, error-model check adds C*eps32*(mag + tmag): mag = sum of |terms|,
  the rounding-error scale of fp32 accumulation, and tmag = sum of |terms| x
  kappa (kappa = sum of alpha/(1-alpha) over the pixel's composited entries),
  the rounding-error scale of the fp32 transmittance chain; both counts are
  reported.  Entries whose sums cancel beyond what fp32 can resolve are held to
  the error model only; the fp64 parity build (tests/test_gpu_strict.py) holds
  every entry to the strict bound.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

RTOL = 1e-4  # north_star tolerance (fp32)
ATOL = 1e-5
EPS32 = 2.0 ** -24
MODEL_C = 64.0  # error-model multiple of eps32*mag
# rtol is attainable in fp32 only where the sum does not cancel by more than rtol/(MODEL_C eps32)
# (~26): entries with sum|terms| > CANCEL_MAX*|ref| are judged by the error model alone (and counted).
CANCEL_MAX = RTOL / (MODEL_C * EPS32)

GRAD_FIELDS = ("position", "theta", "quat", "log_scale", "opacity_logit", "grid")


def run_gpu(arrays: dict, mode: int, n: int, cam_spec, cfg: "O.Cfg", image_grad=None, sigma=0.5, device="cuda",
            fused=None):
    """Binning + forward (+ backward with the given image_grad) through libgb_raster.so.

    fused="l1"|"mse": the backward runs through render_loss_backward against the target
    color - image_grad/2 (so the loss cotangent at scale 1 is image_grad), and the result
    records whether its forward buffers and cotangent equal the separate calls'."""
    import torch

    import paper_2412_12734_b200 as gb

    splats = gb.SplatSet.from_numpy(mode, gb.ColorGridConfig(n, sigma), device=device, **arrays)
    if mode == O.MODE_ORTHO:
        camera = gb.ImagePlaneCamera(cam_spec.width, cam_spec.height, tuple(cam_spec.background))
    else:
        camera = gb.PinholeCamera.from_spec(cam_spec)
    rc = gb.RasterConfig(cfg.tile_size, cfg.cutoff_radius, cfg.alpha_skip, cfg.early_stop, 1)
    binning = gb.build_binning(splats, camera, rc)
    out = gb.render_forward(splats, camera, binning)
    res = {}
    res["offsets"], res["values"] = binning.csr()
    grads = None
    if image_grad is not None:
        ig = torch.as_tensor(np.ascontiguousarray(image_grad, np.float32), device=device)
        if fused:
            target = out.color - 0.5 * ig
            fout = gb.RenderOutput(camera.width, camera.height, device)
            gimg = torch.empty_like(ig)
            loss, grads = gb.render_loss_backward(splats, camera, binning, target, fused, scale=1.0, output=fout,
                                                  image_grad=gimg)
            d = out.color - target
            res["fused"] = dict(
                color_equal=bool(torch.equal(fout.color, out.color)),
                trans_equal=bool(torch.equal(fout.final_transmittance, out.final_transmittance)),
                last_equal=bool(torch.equal(fout.last_rank, out.last_rank)),
                cotangent_max_err=float((gimg - (torch.sign(d) if fused == "l1" else 2.0 * d)).abs().max()),
                loss=float(loss), loss_expected=float(d.abs().sum() if fused == "l1" else (d * d).sum()))
            grads_sep = gb.render_backward(splats, camera, binning, out, gimg)
            res["grads_separate"] = {k: v.cpu().numpy().astype(np.float64) for k, v in grads_sep.tensors().items()}
        else:
            grads = gb.render_backward(splats, camera, binning, out, ig)
    torch.cuda.synchronize()
    res["color"] = out.color.cpu().numpy().astype(np.float64)
    res["trans"] = out.final_transmittance.cpu().numpy().astype(np.float64)
    res["last"] = out.last_rank.cpu().numpy()
    if grads is not None:
        res["grads"] = {k: v.cpu().numpy().astype(np.float64) for k, v in grads.tensors().items()}
    return res


def run_oracle(arrays: dict, n: int, cam: "O.Cam", cfg: "O.Cfg", image_grad=None, sigma=0.5, kink=O.DEFAULT_KINK):
    scene = O.Scene64(arrays, n, sigma)
    b = O.build_binning(scene, cam, cfg)
    f = O.render_forward(scene, cam, cfg, b, kink=kink)
    res = dict(offsets=b[0], values=b[1], color=f["color"], trans=f["trans"], last=f["last"], kink=f["kink"])
    if image_grad is not None:
        g, mag, slack, tmag = O.render_backward_tm(scene, cam, cfg, b, f, np.asarray(image_grad, np.float64),
                                                   kink=kink)
        res.update(grads=g, mag=mag, slack=slack, tmag=tmag)
    return res


def compare_binning(gpu: dict, orc: dict) -> dict:
    return dict(offsets_equal=bool(np.array_equal(gpu["offsets"], orc["offsets"])),
                values_equal=bool(np.array_equal(gpu["values"], orc["values"])),
                pairs=int(len(orc["values"])))


def compare_image(gpu: dict, orc: dict, rtol=RTOL, atol=ATOL) -> dict:
    # bits 0/1: a threshold decision (alpha-skip / 0.999 cap / early stop) within fp32 error;
    # bit 2 (an fp32-ill-conditioned evaluation) is reported but not excluded
    ok_px = (orc["kink"] & 3) == 0
    dc = np.abs(gpu["color"] - orc["color"])
    bad_c = (dc > atol + rtol * np.abs(orc["color"])).any(axis=-1)
    a_g, a_o = 1.0 - gpu["trans"], 1.0 - orc["trans"]
    bad_a = np.abs(a_g - a_o) > atol + rtol * np.abs(a_o)
    bad_l = gpu["last"] != orc["last"]
    return dict(pixels=int(ok_px.size), kink_pixels=int((~ok_px).sum()),
                sensitive_pixels=int(((orc["kink"] & 4) != 0).sum()),
                color_violations=int((bad_c & ok_px).sum()), alpha_violations=int((bad_a & ok_px).sum()),
                last_rank_mismatch=int((bad_l & ok_px).sum()),
                max_abs_color=float(dc[ok_px].max()) if ok_px.any() else 0.0)


def compare_grads(gpu: dict, orc: dict, rtol=RTOL, atol=ATOL, model_c=MODEL_C) -> dict:
    out = {}
    for f in GRAD_FIELDS:
        ref = orc["grads"].get(f)
        if ref is None or f not in gpu["grads"]:
            continue
        got = gpu["grads"][f].reshape(ref.shape)
        d = np.abs(got - ref)
        slack = orc["slack"][f]
        mag = orc["mag"][f]
        # fp32 error model: rounding of the sums (mag) plus the transmittance chain (tmag: |terms| x the pixel's
        # sum of alpha/(1-alpha), the amplification of alpha's relative error through the (1 - alpha) factors)
        tmag = orc["tmag"][f] if orc.get("tmag") is not None and orc["tmag"].get(f) is not None else 0.0
        strict = d > atol + rtol * np.abs(ref) + slack
        model = d > atol + rtol * np.abs(ref) + slack + model_c * EPS32 * (mag + tmag)
        exempt = mag > CANCEL_MAX * np.maximum(np.abs(ref), atol)
        scale = float(np.abs(ref).max()) if ref.size else 0.0
        tol = atol + rtol * np.abs(ref) + slack
        ratio = (d / tol).ravel()
        worst = []
        for i in np.argsort(ratio)[-3:][::-1]:
            if ratio[i] > 1.0:
                worst.append(dict(index=int(i), got=float(got.ravel()[i]), ref=float(ref.ravel()[i]),
                                  slack=float(slack.ravel()[i]), mag=float(mag.ravel()[i]), ratio=float(ratio[i])))
        # error-model ratio of the strict violations: |d| / (eps32 * sum|terms|)
        em = (d / (EPS32 * np.maximum(mag, 1e-300)))[strict]
        tm = np.broadcast_to(tmag, d.shape) if np.ndim(tmag) else np.zeros_like(d)

        def listing(sel, k=4):
            idx = np.flatnonzero(sel.ravel())[:k]
            return [dict(index=int(i), got=float(got.ravel()[i]), ref=float(ref.ravel()[i]), mag=float(mag.ravel()[i]),
                         tmag=float(tm.ravel()[i]), slack=float(slack.ravel()[i])) for i in idx]
        out[f] = dict(entries=int(ref.size), strict_violations=int(strict.sum()), worst=worst,
                      strict_violations_applicable=int((strict & ~exempt).sum()),
                      cancellation_exempt=int(exempt.sum()),
                      eps_mag_ratio_max=float(em.max()) if em.size else 0.0,
                      model_violations=int(model.sum()), kink_entries=int((slack > 0).sum()),
                      applicable=listing(strict & ~exempt), model_list=listing(model),
                      max_abs_err=float(d.max()) if d.size else 0.0,
                      max_rel_to_scale=float(d.max() / scale) if scale > 0 else 0.0)
    return out


# ---------------------------------------------------------------------------------------------
# Tile-row subsets: parity at sizes whose full fp64 backward does not fit the host.
# The binning is compared in full (every pair); the forward and backward are compared on every
# `stride`-th tile row (plus the last, ragged row).  The GPU renders the WHOLE scene and backpropagates
# an image_grad that is zero outside those rows, so its gradients hold exactly the subset tiles'
# contributions (zero-cotangent pixels are skipped, raster.hpp:315-317).  The oracle runs on the subset
# tiles' lists over the primitives they reference, compacted in index order (so per-tile order is kept).
# ---------------------------------------------------------------------------------------------
def subset_rows(tiles_y: int, stride: int):
    return sorted(set(range(0, tiles_y, stride)) | {tiles_y - 1})


def run_rows(arrays: dict, mode: int, n: int, cam: "O.Cam", cfg: "O.Cfg", image_grad, stride: int = 8,
             sigma=0.5, device="cuda", kink=O.DEFAULT_KINK):
    """-> (gpu, orc, info) shaped for compare_binning / compare_image / compare_grads."""
    import torch

    import paper_2412_12734_b200 as gb

    K = int(arrays["opacity_logit"].shape[0])
    geo = {f: (None if f == "grid" else arrays.get(f)) for f in O.FIELDS}
    geo["grid"] = np.zeros((K, 3), np.float32)
    offsets, values, tiles = O.build_binning(O.Scene64(geo, 1, sigma), cam, cfg)
    tx, ty = tiles
    ts = cfg.tile_size
    rows = subset_rows(ty, stride)
    px_rows = np.zeros(cam.height, bool)
    for r in rows:
        px_rows[r * ts:min(cam.height, (r + 1) * ts)] = True
    ig = np.where(px_rows[:, None, None], np.asarray(image_grad, np.float64), 0.0)
    # subset lists and the primitives they reference, compacted in index order
    keep_t = np.zeros(tx * ty, bool)
    for r in rows:
        keep_t[r * tx:(r + 1) * tx] = True
    counts = np.diff(offsets)
    sub_counts = np.where(keep_t, counts, 0)
    mask = np.repeat(keep_t, counts)
    sub_vals = values[mask]
    ids = np.unique(sub_vals)
    remap = np.full(K, -1, np.int64)
    remap[ids] = np.arange(len(ids))
    sub_off = np.zeros(tx * ty + 1, np.int64)
    sub_off[1:] = np.cumsum(sub_counts)
    sub_bin = (sub_off, remap[sub_vals].astype(np.int32), tiles)

    # GPU: the whole scene
    splats = gb.SplatSet.from_numpy(mode, gb.ColorGridConfig(n, sigma), device=device, **arrays)
    camera = (gb.ImagePlaneCamera(cam.width, cam.height, tuple(cam.background)) if mode == O.MODE_ORTHO
              else gb.PinholeCamera.from_spec(cam))
    rc = gb.RasterConfig(cfg.tile_size, cfg.cutoff_radius, cfg.alpha_skip, cfg.early_stop, 1)
    binning = gb.build_binning(splats, camera, rc)
    out = gb.render_forward(splats, camera, binning)
    g = gb.render_backward(splats, camera, binning, out,
                           torch.as_tensor(np.ascontiguousarray(ig, np.float32), device=device))
    torch.cuda.synchronize()
    gpu = {}
    gpu["offsets"], gpu["values"] = binning.csr()
    gpu["color"] = out.color.cpu().numpy().astype(np.float64)[px_rows]
    gpu["trans"] = out.final_transmittance.cpu().numpy().astype(np.float64)[px_rows]
    gpu["last"] = out.last_rank.cpu().numpy()[px_rows]
    tid = torch.as_tensor(ids, device=device)
    gpu["grads"] = {}
    outside = {}
    for f, t in g.tensors().items():
        if t is None:
            continue
        t2 = t.reshape(K, -1)
        gpu["grads"][f] = t2.index_select(0, tid).cpu().numpy().astype(np.float64)
        others = torch.ones(K, dtype=torch.bool, device=device)
        others[tid] = False
        outside[f] = int((t2[others] != 0).sum())
    del splats, binning, out, g
    torch.cuda.empty_cache()

    # oracle: the subset tiles over the compacted primitives
    sub_arrays = {f: (None if arrays.get(f) is None else np.ascontiguousarray(arrays[f][ids])) for f in O.FIELDS}
    scene = O.Scene64(sub_arrays, n, sigma)
    f = O.render_forward(scene, cam, cfg, sub_bin, kink=kink)
    gr, mag, slack, tmag = O.render_backward_tm(scene, cam, cfg, sub_bin, f, ig, kink=kink)
    orc = dict(offsets=offsets, values=values, color=f["color"][px_rows], trans=f["trans"][px_rows],
               last=f["last"][px_rows], kink=f["kink"][px_rows],
               grads={k: (None if v is None else v.reshape(len(ids), -1)) for k, v in gr.items()},
               mag={k: (None if v is None else v.reshape(len(ids), -1)) for k, v in mag.items()},
               slack={k: (None if v is None else v.reshape(len(ids), -1)) for k, v in slack.items()},
               tmag={k: (None if v is None else v.reshape(len(ids), -1)) for k, v in tmag.items()})
    info = dict(tile_rows=len(rows), tiles_y=ty, subset_pairs=int(len(sub_vals)), pairs=int(len(values)),
                subset_primitives=int(len(ids)), gpu_nonzero_outside_subset=outside,
                max_list=int(counts.max()) if counts.size else 0, mean_list=float(counts.mean()))
    return gpu, orc, info


def strict_summary(grads_stats: dict) -> dict:
    """Per field: entries beyond rtol/atol + kink slack with NO cancellation exemption."""
    return {f: st["strict_violations"] for f, st in grads_stats.items()}
