"""Command-line surface of the reference (SPEC.md "cli" module: fit, render, eval, sweep).

    python -m paper_2412_12734_b200 fit --image target.png --splats 1000 --texture-res 4 --iters 20000 --out run
    python -m paper_2412_12734_b200 render --splats run/splats.gbil --width 256 --height 256 --out r.png
    python -m paper_2412_12734_b200 eval a.png b.png            # prints "psnr,ssim"
    python -m paper_2412_12734_b200 sweep --image target.png --sigmas 0.25,0.5 --ns 1,4 --seeds 2 --out sw

Every command runs on the GPU through the package (fit.py, splat_io.py, diagnostics.py); images are
8-bit RGB PNG, read as byte / 255 and written as round(clamp(x, 0, 1) * 255) (image.hpp:104-131).
Exit codes: 0 success, 2 usage error, 1 runtime error.  ``--config FILE`` reads ``key=value`` lines
(keys are the long flag names); flags given on the command line override the file.
"""
from __future__ import annotations

import argparse
import csv
import os
import statistics
import sys
import time
from typing import List, Optional, Sequence

import numpy as np

USAGE, RUNTIME = 2, 1


class UsageError(Exception):
    pass


# ---------------------------------------------------------------------------------------------
# PNG (image.hpp:58-131)
# ---------------------------------------------------------------------------------------------
def load_png(path: str) -> np.ndarray:
    """(H, W, 3) float64 in [0, 1]; an alpha channel is dropped with a warning (image.hpp:78-87)."""
    try:
        from PIL import Image
    except ImportError as e:  # pragma: no cover - PIL is part of the image
        raise RuntimeError("PNG support needs Pillow") from e
    if not os.path.exists(path):
        raise FileNotFoundError(f"cannot open image: {path}")
    try:
        im = Image.open(path)
        im.load()
    except Exception as e:
        raise RuntimeError(f"PNG decode failed: {path}") from e
    if im.format != "PNG":
        raise RuntimeError(f"not a PNG file: {path}")
    if "A" in im.getbands():
        print(f"warning: {path} has an alpha channel; ignoring it", file=sys.stderr)
    arr = np.asarray(im.convert("RGB"), dtype=np.uint8)
    return arr.astype(np.float64) / 255.0


def save_png(path: str, img: np.ndarray) -> None:
    from PIL import Image

    img = np.asarray(img, dtype=np.float64)
    if img.ndim != 3 or img.shape[2] != 3 or img.shape[0] < 1 or img.shape[1] < 1:
        raise RuntimeError("save_png: empty image")
    # std::lround: halves away from zero (all values are non-negative here)
    u8 = np.floor(np.clip(img, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    try:
        Image.fromarray(u8, "RGB").save(path, format="PNG")
    except OSError as e:
        raise RuntimeError(f"cannot write image: {path}") from e


# ---------------------------------------------------------------------------------------------
# arguments
# ---------------------------------------------------------------------------------------------
def _floats(text: str) -> List[float]:
    return [float(x) for x in text.split(",") if x.strip()]


def _ints(text: str) -> List[int]:
    return [int(x) for x in text.split(",") if x.strip()]


def _add_fit_flags(p: argparse.ArgumentParser, sweep: bool = False) -> None:
    p.add_argument("--image", help="target PNG")
    p.add_argument("--splats", type=int, default=1000, help="number of splats K")
    if not sweep:
        p.add_argument("--texture-res", type=int, default=4, help="texture resolution N")
        p.add_argument("--sigma", type=float, default=0.5, help="grid extent sigma")
        p.add_argument("--seed", type=int, default=0)
    p.add_argument("--iters", type=int, default=20000)
    p.add_argument("--loss", choices=("mse", "mse-ssim"), default="mse")
    p.add_argument("--out", default="out", help="output directory")
    p.add_argument("--threads", type=int, default=1, help="accepted for compatibility (the GPU ignores it)")
    p.add_argument("--tile-size", type=int, default=16)
    p.add_argument("--log-every", type=int, default=100)
    p.add_argument("--force-n", action="store_true", help="allow texture resolutions outside {1, 2, 4, 8}")
    for name in ("position", "theta", "log-scale", "opacity", "color-grid", "position-gamma"):
        p.add_argument(f"--lr-{name}", type=float, default=None)
    p.add_argument("--config", default=None, help="key=value lines; command-line flags override them")


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2412_12734_b200",
                                 description="Gaussian Billboards on the B200: fit, render, eval, sweep")
    sub = ap.add_subparsers(dest="cmd", required=True)
    _add_fit_flags(sub.add_parser("fit", help="fit a target image (train.hpp:174-219)"))
    r = sub.add_parser("render", help="render a splat file to PNG")
    r.add_argument("--splats", required=True, help="GBIL splat file")
    r.add_argument("--out", required=True, help="output PNG")
    r.add_argument("--width", type=int, required=True)
    r.add_argument("--height", type=int, required=True)
    r.add_argument("--background", default="0,0,0", help="r,g,b in [0, 1]")
    r.add_argument("--mip-level", type=int, default=0, help="texture.hpp:132-188 downsampling levels")
    r.add_argument("--random-colors", type=int, default=None, help="seed: render with random texel colours")
    r.add_argument("--tile-size", type=int, default=16)
    e = sub.add_parser("eval", help="PSNR and SSIM of two PNGs, as 'psnr,ssim'")
    e.add_argument("a")
    e.add_argument("b")
    s = sub.add_parser("sweep", help="fits over a sigma x N grid and seeds (Fig. 4 / Fig. 5 ablations)")
    _add_fit_flags(s, sweep=True)
    s.add_argument("--sigmas", default="0.25,0.5,1.0,2.0")
    s.add_argument("--ns", default="1,2,4,8")
    s.add_argument("--seeds", type=int, default=1, help="seeds 0 .. S-1 per cell")
    return ap


def _apply_config(ap: argparse.ArgumentParser, argv: Sequence[str]) -> argparse.Namespace:
    """Defaults < config file < command-line flags (SPEC.md cli design decisions)."""
    args = ap.parse_args(argv)
    path = getattr(args, "config", None)
    if not path:
        return args
    if not os.path.exists(path):
        raise UsageError(f"cannot open config file: {path}")
    sub = ap._subparsers._group_actions[0].choices[args.cmd]  # the command's own parser
    known = {a.dest: a for a in sub._actions}
    values = {}
    for n, line in enumerate(open(path), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise UsageError(f"{path}:{n}: expected key=value")
        k, v = (x.strip() for x in line.split("=", 1))
        dest = k.lstrip("-").replace("-", "_")
        if dest not in known or dest == "config":
            raise UsageError(f"{path}:{n}: unknown key '{k}'")
        act = known[dest]
        if isinstance(act, argparse._StoreTrueAction):
            values[dest] = v.lower() in ("1", "true", "yes", "on")
        else:
            conv = act.type or str
            if act.choices and v not in act.choices:
                raise UsageError(f"{path}:{n}: invalid value '{v}' for '{k}'")
            values[dest] = conv(v)
    sub.set_defaults(**values)
    return ap.parse_args(argv)


def _train_config(args, n: int, sigma: float, seed: int):
    from .fit import LossKind, TrainConfig
    from .raster import ColorGridConfig, LearningRates, RasterConfig

    lrs = LearningRates()
    for name, attr in (("position", "position"), ("theta", "theta"), ("log_scale", "log_scale"),
                       ("opacity", "opacity_logit"), ("color_grid", "color_grid"), ("position_gamma", "position_gamma")):
        v = getattr(args, f"lr_{name}")
        if v is not None:
            setattr(lrs, attr, v)
    cfg = TrainConfig(splat_count=args.splats, iterations=args.iters,
                      loss=LossKind.mse if args.loss == "mse" else LossKind.mse_plus_ssim, seed=seed,
                      grid=ColorGridConfig(n, sigma), lrs=lrs,
                      raster=RasterConfig(tile_size=args.tile_size, threads=args.threads),
                      log_every=args.log_every, allow_any_n=args.force_n)
    try:
        cfg.validate()
    except ValueError as e:
        raise UsageError(str(e)) from e
    if args.tile_size < 1 or args.tile_size > 16:
        raise UsageError("RasterConfig: tile_size must be in [1, 16] on the GPU")
    return cfg


def _check_out_dir(path: str) -> None:
    try:
        os.makedirs(path, exist_ok=True)
    except OSError as e:
        raise RuntimeError(f"cannot create output directory: {path}") from e
    if not os.access(path, os.W_OK):
        raise RuntimeError(f"output directory is not writable: {path}")


def _render(splats, width: int, height: int, background, tile_size: int) -> np.ndarray:
    from .raster import ImagePlaneCamera, RasterConfig, build_binning, render_forward

    cam = ImagePlaneCamera(width, height, tuple(background))
    b = build_binning(splats, cam, RasterConfig(tile_size=tile_size))
    return render_forward(splats, cam, b).color.cpu().numpy().astype(np.float64)


# ---------------------------------------------------------------------------------------------
# commands
# ---------------------------------------------------------------------------------------------
def _fit_one(args, target: np.ndarray, n: int, sigma: float, seed: int):
    import torch

    from .fit import fit

    cfg = _train_config(args, n, sigma, seed)
    t0 = time.perf_counter()
    res = fit(torch.as_tensor(target, dtype=torch.float32), cfg)
    torch.cuda.synchronize()
    return cfg, res, time.perf_counter() - t0


def cmd_fit(args) -> int:
    if not args.image:
        raise UsageError("fit: --image is required")
    _train_config(args, args.texture_res, args.sigma, args.seed)  # usage errors before any work
    target = load_png(args.image)
    _check_out_dir(args.out)
    from .splat_io import save_splats

    cfg, res, _ = _fit_one(args, target, args.texture_res, args.sigma, args.seed)
    save_splats(os.path.join(args.out, "splats.gbil"), res.splats)
    with open(os.path.join(args.out, "metrics.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["iter", "loss", "psnr", "ssim", "wall_ms"])
        for r in res.history:
            w.writerow([r.iter, repr(r.loss), repr(r.psnr), repr(r.ssim), repr(r.wall_ms)])
    H, W = target.shape[:2]
    save_png(os.path.join(args.out, "render.png"), _render(res.splats, W, H, cfg.background, args.tile_size))
    last = res.history[-1]
    print(f"fit: {cfg.iterations} iterations, loss {last.loss:.6g}, psnr {last.psnr:.2f}, ssim {last.ssim:.6f}; "
          f"wrote {args.out}/splats.gbil, metrics.csv, render.png")
    return 0


def cmd_render(args) -> int:
    if args.width < 1 or args.height < 1:
        raise UsageError("render: --width and --height must be >= 1")
    if args.mip_level < 0:
        raise UsageError("render: --mip-level must be >= 0")
    try:
        bg = _floats(args.background)
    except ValueError as e:
        raise UsageError(f"render: bad --background '{args.background}'") from e
    if len(bg) != 3 or not all(0.0 <= c <= 1.0 for c in bg):
        raise UsageError("render: --background needs three values in [0, 1]")
    from . import diagnostics
    from .raster import MODE_ORTHO, ImagePlaneCamera, RasterConfig
    from .splat_io import file_info, load_splats

    info = file_info(args.splats)
    if info.mode != MODE_ORTHO:
        raise RuntimeError("render: pinhole splat files need a camera; render them through the Python API")
    splats = load_splats(args.splats)
    if args.mip_level:
        splats = diagnostics.downsample_set(splats, args.mip_level)
    if args.random_colors is not None:
        cam = ImagePlaneCamera(args.width, args.height, tuple(bg))
        out = diagnostics.render_random_colors(splats, cam, args.random_colors, RasterConfig(tile_size=args.tile_size))
        img = out.color.cpu().numpy().astype(np.float64)
    else:
        img = _render(splats, args.width, args.height, bg, args.tile_size)
    save_png(args.out, img)
    return 0


def cmd_eval(args) -> int:
    import torch

    from .fit import psnr, ssim

    a, b = load_png(args.a), load_png(args.b)
    if a.shape != b.shape:
        raise RuntimeError(f"eval: image sizes differ ({a.shape[1]}x{a.shape[0]} vs {b.shape[1]}x{b.shape[0]})")
    ta = torch.as_tensor(a, dtype=torch.float32).cuda()
    tb = torch.as_tensor(b, dtype=torch.float32).cuda()
    s = ssim(ta, tb) if a.shape[0] >= 11 and a.shape[1] >= 11 else float("nan")
    print(f"{psnr(ta, tb):.2f},{s:.6f}")
    return 0


def cmd_sweep(args) -> int:
    if not args.image:
        raise UsageError("sweep: --image is required")
    try:
        sigmas, ns = _floats(args.sigmas), _ints(args.ns)
    except ValueError as e:
        raise UsageError("sweep: --sigmas and --ns are comma-separated numbers") from e
    if not sigmas or not ns or args.seeds < 1:
        raise UsageError("sweep: empty grid")
    for s in sigmas:
        for n in ns:
            _train_config(args, n, s, 0)
    target = load_png(args.image)
    _check_out_dir(args.out)
    rows = []
    for s in sigmas:
        for n in ns:
            for seed in range(args.seeds):
                _, res, wall = _fit_one(args, target, n, s, seed)
                last = res.history[-1]
                rows.append((s, n, seed, last.psnr, last.ssim, wall))
                print(f"sigma {s} n {n} seed {seed}: psnr {last.psnr:.2f} ssim {last.ssim:.6f} ({wall:.1f} s)",
                      flush=True)
    with open(os.path.join(args.out, "sweep.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["sigma", "n", "seed", "psnr", "ssim", "wall_seconds"])
        for r in rows:
            w.writerow([repr(r[0]), r[1], r[2], repr(r[3]), repr(r[4]), repr(r[5])])
    with open(os.path.join(args.out, "sweep_summary.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["sigma", "n", "median_psnr", "median_ssim"])
        print("sigma,n,median_psnr,median_ssim")
        for s in sigmas:
            for n in ns:
                cell = [r for r in rows if r[0] == s and r[1] == n]
                mp, ms = statistics.median(r[3] for r in cell), statistics.median(r[4] for r in cell)
                w.writerow([repr(s), n, repr(mp), repr(ms)])
                print(f"{s},{n},{mp:.2f},{ms:.6f}")
    return 0


COMMANDS = {"fit": cmd_fit, "render": cmd_render, "eval": cmd_eval, "sweep": cmd_sweep}


def main(argv: Optional[Sequence[str]] = None) -> int:
    ap = _parser()
    argv = list(sys.argv[1:] if argv is None else argv)
    try:
        args = _apply_config(ap, argv)
    except SystemExit as e:  # argparse usage errors exit with 2 already
        return int(e.code or 0)
    except (UsageError, ValueError) as e:
        print(f"usage error: {e}", file=sys.stderr)
        return USAGE
    try:
        return COMMANDS[args.cmd](args)
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return USAGE
    except Exception as e:  # runtime errors: message and exit 1
        print(f"error: {e}", file=sys.stderr)
        return RUNTIME
