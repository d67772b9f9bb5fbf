"""Seeded synthetic scenes and cameras for the BASELINE.json configs.

There is no public dataset for this path: every config is synthetic
(SURVEY.md §8(d)).  Generation runs in the host part of libgb_raster.so with
the reference's Rng semantics (rng.hpp:12-46); geometry comes from Rng(seed),
textures from Rng(seed+1), per-view targets from Rng(seed+2+view).  Values
are drawn in fp64 and rounded to fp32 once, so the oracle (fp64) and the GPU
(fp32) consume identical bits.

Defaults the configs leave open (marked ⚑ in SURVEY.md §8(d)):
  sigma_tex = 0.5; RasterConfig defaults; OpenCV pinhole looking at the origin
  with world up (0,1,0); configs[2..4] intrinsics fx = fy = 1000,
  cx = 800, cy = 532; near plane 0.01.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib

MODE_ORTHO = _lib.MODE_ORTHO
MODE_PINHOLE = _lib.MODE_PINHOLE


def generate(mode: int, count: int, n: int, seed: int, *, mean_lo=-1.0, mean_hi=1.0, mean_sigma=0.0,
             scale_lo=0.005, scale_hi=0.05, width=0, height=0) -> dict:
    """Host fp32 arrays of a seeded scene (SplatSet field names)."""
    spec = _lib.SceneSpec(mode, n, count, seed, mean_lo, mean_hi, mean_sigma, math.log(scale_lo),
                          math.log(scale_hi), width, height)
    pin = mode == MODE_PINHOLE
    arr = {
        "position": np.zeros((count, 3 if pin else 2), np.float32),
        "depth_key": None if pin else np.zeros(count, np.float32),
        "theta": None if pin else np.zeros(count, np.float32),
        "quat": np.zeros((count, 4), np.float32) if pin else None,
        "log_scale": np.zeros((count, 2), np.float32),
        "opacity_logit": np.zeros(count, np.float32),
        "grid": np.zeros((count, n * n * 3), np.float32),
    }
    ptr = lambda a: None if a is None else a.ctypes.data
    check(lib.gb_scene_generate(C.byref(spec), ptr(arr["position"]), ptr(arr["depth_key"]), ptr(arr["theta"]),
                                ptr(arr["quat"]), ptr(arr["log_scale"]), ptr(arr["opacity_logit"]),
                                ptr(arr["grid"])), "gb_scene_generate")
    return arr


def uniform_image(seed: int, width: int, height: int) -> np.ndarray:
    """(H, W, 3) fp32 uniforms in [0,1) from Rng(seed) -- the seeded-noise targets."""
    out = np.zeros((height, width, 3), np.float32)
    check(lib.gb_uniform_fill(seed, out.size, out.ctypes.data), "gb_uniform_fill")
    return out


def rng_uniform(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float64)
    check(lib.gb_rng_uniform(seed, n, out.ctypes.data), "gb_rng_uniform")
    return out


def rng_normal(seed: int, n: int, mean=0.0, stddev=1.0) -> np.ndarray:
    out = np.zeros(n, np.float64)
    check(lib.gb_rng_normal(seed, n, mean, stddev, out.ctypes.data), "gb_rng_normal")
    return out


@dataclass
class CameraSpec:
    """Host description of a pinhole camera (world -> camera rot/trans, float64)."""

    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    rot: np.ndarray
    trans: np.ndarray
    near_plane: float = 0.01
    background: tuple = (0.0, 0.0, 0.0)


def look_at(eye, target, width, height, fx, fy, cx, cy, up=(0.0, 1.0, 0.0), near_plane=0.01) -> CameraSpec:
    """z_cam = normalize(target - eye), x_cam = normalize(up x z_cam), y_cam = z_cam x x_cam."""
    eye = np.asarray(eye, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - eye
    f /= np.linalg.norm(f)
    r = np.cross(np.asarray(up, dtype=np.float64), f)
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    rot = np.stack([r, d, f])
    return CameraSpec(width, height, fx, fy, cx, cy, rot, -rot @ eye, near_plane)


def fibonacci_cameras(count: int, radius: float, width: int, height: int, fx: float, fy: float, cx: float,
                      cy: float) -> list:
    """configs[3]: y_i = 1 - 2(i+1/2)/count, r_i = sqrt(1-y_i^2), phi_i = i*pi*(3-sqrt5)."""
    cams = []
    for i in range(count):
        y = 1.0 - 2.0 * (i + 0.5) / count
        r = math.sqrt(max(0.0, 1.0 - y * y))
        phi = i * math.pi * (3.0 - math.sqrt(5.0))
        eye = (radius * r * math.cos(phi), radius * y, radius * r * math.sin(phi))
        cams.append(look_at(eye, (0.0, 0.0, 0.0), width, height, fx, fy, cx, cy))
    return cams


@dataclass
class ConfigScene:
    name: str
    mode: int
    count: int
    n: int
    seed: int
    gen_kwargs: dict
    cameras: list
    description: str

    def arrays(self) -> dict:
        return generate(self.mode, self.count, self.n, self.seed, **self.gen_kwargs)

    def target(self, view: int) -> np.ndarray:
        cam = self.cameras[view]
        return uniform_image(self.seed + 2 + view, cam.width, cam.height)


def baseline_config(index: int, *, count: int = None, n: int = None, views: int = None) -> ConfigScene:
    """BASELINE.json configs[index] (count / n overridable for the configs[4] sweep and small parity cases)."""
    if index in (0, 1):
        K = count or 100_000
        tn = n or 4
        cam = look_at((0.0, 0.0, -4.0), (0.0, 0.0, 0.0), 800, 800, 1000.0, 1000.0, 400.0, 400.0)
        return ConfigScene(f"configs[{index}]", MODE_PINHOLE, K, tn, 0,
                           dict(mean_lo=-1.0, mean_hi=1.0, scale_lo=0.005, scale_hi=0.05), [cam],
                           f"{K} surfels, {tn}x{tn} textures, 800x800, fx=fy=1000, eye (0,0,-4)")
    if index == 2:
        K = count or 1_000_000
        tn = n or 8
        cam = look_at((0.0, 0.0, -6.0), (0.0, 0.0, 0.0), 1600, 1064, 1000.0, 1000.0, 800.0, 532.0)
        return ConfigScene("configs[2]", MODE_PINHOLE, K, tn, 0,
                           dict(mean_sigma=2.0, scale_lo=0.002, scale_hi=0.03), [cam],
                           f"{K} surfels, {tn}x{tn} textures, N(0,2^2) means, 1600x1064, orbit radius 6")
    if index == 3:
        K = count or 1_000_000
        tn = n or 8
        cams = fibonacci_cameras(views or 64, 6.0, 1600, 1064, 1000.0, 1000.0, 800.0, 532.0)
        return ConfigScene("configs[3]", MODE_PINHOLE, K, tn, 0,
                           dict(mean_sigma=2.0, scale_lo=0.002, scale_hi=0.03), cams,
                           f"{K} surfels, {tn}x{tn} textures, {len(cams)} Fibonacci-sphere views at 1600x1064")
    if index == 4:
        K = count or 1_000_000
        tn = n or 8
        cam = look_at((0.0, 0.0, -6.0), (0.0, 0.0, 0.0), 1600, 1064, 1000.0, 1000.0, 800.0, 532.0)
        return ConfigScene(f"configs[4] K={K} T={tn}", MODE_PINHOLE, K, tn, 0,
                           dict(mean_lo=-2.0, mean_hi=2.0, scale_lo=0.002, scale_hi=0.05), [cam],
                           f"{K} surfels, {tn}x{tn} textures, U[-2,2]^3 means, 1600x1064")
    raise ValueError(f"no BASELINE config {index}")
