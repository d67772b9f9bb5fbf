"""TEST INFRASTRUCTURE ONLY -- ctypes access to the parity checkers.

* ``liboracle.so``      : oracle/gb_oracle.c, the fp64 C restatement (ortho + pinhole)
* ``_ref/libgbil_ref.so``: the unmodified reference headers compiled behind
                          oracle/ref_shim.cpp (present only where /root/reference
                          was available at build time)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgbil_ref.so")

MODE_ORTHO = 0
MODE_PINHOLE = 1


def build(quiet: bool = True) -> None:
    """make -C oracle (liboracle.so always; _ref only where the reference exists)."""
    subprocess.run(["make", "-C", HERE], check=True, stdout=subprocess.DEVNULL if quiet else None)


class OrcCamera(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("width", C.c_int32), ("height", C.c_int32), ("_pad", C.c_int32),
        ("background", C.c_double * 3),
        ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
        ("rot", C.c_double * 9), ("trans", C.c_double * 3), ("near_plane", C.c_double),
    ]


class OrcConfig(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("threads", C.c_int32), ("cutoff_radius", C.c_double),
                ("alpha_skip", C.c_double), ("early_stop", C.c_double)]


class OrcSplats(C.Structure):
    _fields_ = [("count", C.c_int64), ("n", C.c_int32), ("_pad", C.c_int32), ("sigma", C.c_double),
                ("position", C.c_void_p), ("depth_key", C.c_void_p), ("theta", C.c_void_p),
                ("quat", C.c_void_p), ("log_scale", C.c_void_p), ("opacity_logit", C.c_void_p),
                ("grid", C.c_void_p)]


class OrcGrads(C.Structure):
    _fields_ = [("position", C.c_void_p), ("depth_key", C.c_void_p), ("theta", C.c_void_p),
                ("quat", C.c_void_p), ("log_scale", C.c_void_p), ("opacity_logit", C.c_void_p),
                ("grid", C.c_void_p)]


class OrcBinning(C.Structure):
    _fields_ = [("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("total", C.c_int64),
                ("offsets", C.POINTER(C.c_int64)), ("values", C.POINTER(C.c_int32))]


class OrcKink(C.Structure):
    _fields_ = [("alpha_rel", C.c_double), ("trans_rel", C.c_double), ("grid_abs", C.c_double),
                ("cond_min", C.c_double), ("uv_rel", C.c_double)]


# kink margins of the fp32 product (parity protocol)
DEFAULT_KINK = (2e-5, 1e-3, 1e-4, 1e-4, 4.0)
# for the fp64 parity build: decision kinks only (its (u, v) are fp64, so no fp32 (u, v) error propagation)
STRICT_KINK = (2e-5, 1e-3, 1e-4, 0.0, 0.0)

_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        P = C.c_void_p
        L.orc_build_binning.argtypes = [P, P, P, C.POINTER(OrcBinning)]
        L.orc_binning_free.argtypes = [C.POINTER(OrcBinning)]
        L.orc_project.argtypes = [P, P, P, P, P]
        L.orc_render_forward.argtypes = [P, P, P, C.POINTER(OrcBinning), P, P, P, P, P]
        L.orc_render_backward.argtypes = [P, P, P, C.POINTER(OrcBinning), P, P, P, P, P, P, P, P]
        L.orc_render_backward_tm.argtypes = [P, P, P, C.POINTER(OrcBinning), P, P, P, P, P, P, P, P, P]
        L.orc_render_naive.argtypes = [P, P, P, P]
        L.orc_gradient_fd.argtypes = [P, P, P, C.c_double, P]
        L.orc_uv_to_grid.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, P, P, P, P]
        L.orc_bilinear.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, P, P]
        L.orc_adj_bilinear.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, P, P, P, P, P]
        L.orc_intersect_ortho.argtypes = [C.c_double] * 7 + [P, P]
        L.orc_intersect_pinhole.argtypes = [P, P, P, P, C.c_double, C.c_double, P, P]
        L.orc_adam_group.argtypes = [P, P, P, P, C.c_int64] + [C.c_double] * 6
        L.orc_adam_group.restype = C.c_int64
        L.orc_l1_loss.argtypes = [P, P, C.c_int64, C.c_double, P]
        L.orc_l1_loss.restype = C.c_double
        L.orc_scene_generate_pinhole.argtypes = [C.c_int64, C.c_int32, C.c_uint64] + [C.c_double] * 5 + [P] * 5
        L.orc_uniform_fill.argtypes = [C.c_uint64, C.c_int64, P]
        L.orc_rng_seed.argtypes = [P, C.c_uint64]
        L.orc_rng_uniform.argtypes = [P]
        L.orc_rng_uniform.restype = C.c_double
        L.orc_rng_normal.argtypes = [P, C.c_double, C.c_double]
        L.orc_rng_normal.restype = C.c_double
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(REF_SO)
        P = C.c_void_p
        d, i = C.c_double, C.c_int
        L.ref_render.argtypes = [C.c_int64, i, d, P, P, P, P, P, P, i, i, P, i, d, d, d, i, P, P, P, P, P, P, P,
                                 P, P, P, P, P, P]
        L.ref_render_naive.argtypes = [C.c_int64, i, d, P, P, P, P, P, P, i, i, P, P, P]
        L.ref_gradient_fd.argtypes = [C.c_int64, i, d, P, P, P, P, P, P, i, i, P, P, d, P, P, P, P, P, P]
        L.ref_uv_to_grid.argtypes = [d, d, i, d, P, P, P, P]
        L.ref_ssim.argtypes = [i, i, P, P, i, P]
        L.ref_ssim.restype = d
        L.ref_psnr.argtypes = [i, i, P, P]
        L.ref_psnr.restype = d
        L.ref_initialize.argtypes = [i, i, C.c_int64, i, C.c_uint64, P, P, P, P, P, P]
        L.ref_fit.argtypes = [i, i, P, C.c_int64, i, d, C.c_int64, i, d, C.c_uint64, C.c_int64, i, P, P, P, P, P,
                              P, P, C.c_int64, P, C.c_char_p, i]
        L.ref_downsample_grid.argtypes = [P, i, i, P, P, C.c_char_p, i]
        L.ref_randomize_colors.argtypes = [C.c_int64, i, C.c_uint64, P]
        L.ref_save_splats.argtypes = [C.c_char_p, C.c_int64, i, d, P, P, P, P, P, P, C.c_char_p, i]
        L.ref_load_splats.argtypes = [C.c_char_p, P, P, P, P, P, P, P, P, P, C.c_char_p, i]
        L.ref_bilinear.argtypes = [d, d, i, d, P, P]
        L.ref_adj_bilinear.argtypes = [d, d, i, d, P, P, P, P, P]
        L.ref_adam_group.argtypes = [P, P, P, P, C.c_int64, d, d, d, d, d, d]
        L.ref_rng_uniform.argtypes = [C.c_uint64, C.c_int64, P]
        L.ref_rng_normal.argtypes = [C.c_uint64, C.c_int64, d, d, P]
        _ref = L
    return _ref


# ----------------------------------------------------------------------------------------------
# high-level helpers over numpy scenes (SplatSet field names, fp32 or fp64 arrays)
# ----------------------------------------------------------------------------------------------
@dataclass
class Cam:
    mode: int
    width: int
    height: int
    background: tuple = (0.0, 0.0, 0.0)
    fx: float = 1.0
    fy: float = 1.0
    cx: float = 0.0
    cy: float = 0.0
    rot: np.ndarray = None
    trans: np.ndarray = None
    near_plane: float = 0.01

    @staticmethod
    def from_spec(spec) -> "Cam":
        return Cam(MODE_PINHOLE, spec.width, spec.height, tuple(spec.background), spec.fx, spec.fy, spec.cx, spec.cy,
                   np.asarray(spec.rot, np.float64), np.asarray(spec.trans, np.float64), spec.near_plane)

    def to_c(self) -> OrcCamera:
        c = OrcCamera()
        c.mode, c.width, c.height = self.mode, self.width, self.height
        for k in range(3):
            c.background[k] = float(self.background[k])
        c.fx, c.fy, c.cx, c.cy = self.fx, self.fy, self.cx, self.cy
        rot = np.eye(3) if self.rot is None else np.asarray(self.rot, np.float64)
        tr = np.zeros(3) if self.trans is None else np.asarray(self.trans, np.float64)
        for k in range(9):
            c.rot[k] = float(rot.reshape(9)[k])
        for k in range(3):
            c.trans[k] = float(tr.reshape(3)[k])
        c.near_plane = self.near_plane
        return c


@dataclass
class Cfg:
    tile_size: int = 16
    cutoff_radius: float = 3.0
    alpha_skip: float = 1.0 / 255.0
    early_stop: float = 1e-4
    threads: int = 0  # 0 -> all host cores

    def to_c(self) -> OrcConfig:
        t = self.threads if self.threads > 0 else (os.cpu_count() or 1)
        return OrcConfig(self.tile_size, t, self.cutoff_radius, self.alpha_skip, self.early_stop)


FIELDS = ("position", "depth_key", "theta", "quat", "log_scale", "opacity_logit", "grid")


class Scene64:
    """fp64 contiguous copies of a scene, kept alive for the C calls."""

    def __init__(self, arrays: dict, n: int, sigma: float = 0.5):
        self.n, self.sigma = n, sigma
        self.a = {f: (None if arrays.get(f) is None else np.ascontiguousarray(arrays[f], dtype=np.float64))
                  for f in FIELDS}
        self.count = int(self.a["opacity_logit"].shape[0])

    def to_c(self) -> OrcSplats:
        p = lambda f: None if self.a[f] is None else self.a[f].ctypes.data
        return OrcSplats(self.count, self.n, 0, self.sigma, p("position"), p("depth_key"), p("theta"), p("quat"),
                         p("log_scale"), p("opacity_logit"), p("grid"))

    def zeros_like(self) -> dict:
        return {f: (None if v is None else np.zeros_like(v)) for f, v in self.a.items()}


def _grads_c(g: dict) -> OrcGrads:
    p = lambda f: None if g.get(f) is None else g[f].ctypes.data
    return OrcGrads(p("position"), p("depth_key"), p("theta"), p("quat"), p("log_scale"), p("opacity_logit"),
                    p("grid"))


def _check(rc, where):
    if rc != 0:
        raise ValueError(f"{where}: oracle status {rc}")


def build_binning(scene: Scene64, cam: Cam, cfg: Cfg):
    """(offsets, values) CSR of the per-tile sorted lists (raster.hpp:116-147)."""
    L = oracle_lib()
    b = OrcBinning()
    s, c, k = scene.to_c(), cam.to_c(), cfg.to_c()
    _check(L.orc_build_binning(C.byref(s), C.byref(c), C.byref(k), C.byref(b)), "orc_build_binning")
    nt = b.tiles_x * b.tiles_y
    offsets = np.ctypeslib.as_array(b.offsets, shape=(nt + 1,)).copy()
    values = (np.ctypeslib.as_array(b.values, shape=(b.total,)).copy() if b.total > 0
              else np.zeros(0, np.int32))
    L.orc_binning_free(C.byref(b))
    return offsets, values, (b.tiles_x, b.tiles_y)


def _binning_struct(offsets, values, tiles):
    b = OrcBinning()
    b.tiles_x, b.tiles_y = tiles
    b.total = len(values)
    offsets = np.ascontiguousarray(offsets, np.int64)
    values = np.ascontiguousarray(values if len(values) else np.zeros(1, np.int32), np.int32)
    b.offsets = offsets.ctypes.data_as(C.POINTER(C.c_int64))
    b.values = values.ctypes.data_as(C.POINTER(C.c_int32))
    return b, (offsets, values)


def render_forward(scene: Scene64, cam: Cam, cfg: Cfg, binning, kink=DEFAULT_KINK):
    """raster.hpp:201-261 in fp64 -> dict(color (H,W,3), trans (H,W), last (H,W), kink (H,W) bool)."""
    L = oracle_lib()
    offsets, values, tiles = binning
    b, keep = _binning_struct(offsets, values, tiles)
    H, W = cam.height, cam.width
    color = np.zeros((H, W, 3)); trans = np.zeros((H, W)); last = np.zeros((H, W), np.int32)
    kpx = np.zeros((H, W), np.uint8)
    kk = OrcKink(*kink) if kink is not None else None
    s, c, k = scene.to_c(), cam.to_c(), cfg.to_c()
    _check(L.orc_render_forward(C.byref(s), C.byref(c), C.byref(k), C.byref(b), color.ctypes.data,
                                trans.ctypes.data, last.ctypes.data, kpx.ctypes.data,
                                C.byref(kk) if kk is not None else None), "orc_render_forward")
    return dict(color=color, trans=trans, last=last, kink=kpx)


def render_backward(scene: Scene64, cam: Cam, cfg: Cfg, binning, fwd: dict, image_grad, kink=DEFAULT_KINK,
                    want_mag: bool = True):
    g, mag, slack, _ = render_backward_tm(scene, cam, cfg, binning, fwd, image_grad, kink, want_mag, False)
    return g, mag, slack


def render_backward_tm(scene: Scene64, cam: Cam, cfg: Cfg, binning, fwd: dict, image_grad, kink=DEFAULT_KINK,
                       want_mag: bool = True, want_tmag: bool = True):
    """raster.hpp:277-387 in fp64 -> (grads, mag, slack) dicts.

    mag[f]   : sum of |terms| per gradient entry (fp32 accumulation-error scale)
    slack[f] : |terms| from evaluations within fp32 error of a kink (may differ legitimately)
    """
    L = oracle_lib()
    offsets, values, tiles = binning
    b, keep = _binning_struct(offsets, values, tiles)
    g = scene.zeros_like()
    mag = scene.zeros_like() if want_mag else None
    slack = scene.zeros_like() if want_mag else None
    tmag = scene.zeros_like() if want_tmag else None
    ig = np.ascontiguousarray(image_grad, np.float64)
    trans = np.ascontiguousarray(fwd["trans"], np.float64)
    last = np.ascontiguousarray(fwd["last"], np.int32)
    kpx = np.ascontiguousarray(fwd.get("kink", np.zeros_like(last)), np.uint8)
    kk = OrcKink(*kink) if kink is not None else None
    s, c, k = scene.to_c(), cam.to_c(), cfg.to_c()
    gc = _grads_c(g)
    mc = _grads_c(mag) if mag is not None else None
    sc = _grads_c(slack) if slack is not None else None
    tc = _grads_c(tmag) if tmag is not None else None
    _check(L.orc_render_backward_tm(C.byref(s), C.byref(c), C.byref(k), C.byref(b), trans.ctypes.data,
                                    last.ctypes.data, ig.ctypes.data, C.byref(gc), kpx.ctypes.data,
                                    C.byref(mc) if mc is not None else None, C.byref(sc) if sc is not None else None,
                                    C.byref(tc) if tc is not None else None,
                                    C.byref(kk) if kk is not None else None), "orc_render_backward")
    return g, mag, slack, tmag


def project(scene: Scene64, cam: Cam, cfg: Cfg):
    L = oracle_lib()
    depth = np.zeros(scene.count); rect = np.zeros((scene.count, 4), np.int32)
    s, c, k = scene.to_c(), cam.to_c(), cfg.to_c()
    _check(L.orc_project(C.byref(s), C.byref(c), C.byref(k), depth.ctypes.data, rect.ctypes.data), "orc_project")
    return depth, rect


def render_naive(scene: Scene64, cam: Cam):
    L = oracle_lib()
    color = np.zeros((cam.height, cam.width, 3)); trans = np.zeros((cam.height, cam.width))
    s, c = scene.to_c(), cam.to_c()
    _check(L.orc_render_naive(C.byref(s), C.byref(c), color.ctypes.data, trans.ctypes.data), "orc_render_naive")
    return color, trans


def gradient_fd(scene: Scene64, cam: Cam, weights, step: float):
    L = oracle_lib()
    g = scene.zeros_like()
    w = np.ascontiguousarray(weights, np.float64)
    s, c, gc = scene.to_c(), cam.to_c(), _grads_c(g)
    _check(L.orc_gradient_fd(C.byref(s), C.byref(c), w.ctypes.data, step, C.byref(gc)), "orc_gradient_fd")
    return g


def l1_loss(color, target, scale):
    L = oracle_lib()
    c = np.ascontiguousarray(color, np.float64); t = np.ascontiguousarray(target, np.float64)
    grad = np.zeros_like(c)
    v = L.orc_l1_loss(c.ctypes.data, t.ctypes.data, c.size, scale, grad.ctypes.data)
    return v, grad


def adam_group(p, g, m, v, lr, beta1, beta2, eps, bias1, bias2):
    L = oracle_lib()
    arrs = [np.ascontiguousarray(a, np.float64) for a in (p, g, m, v)]
    bad = L.orc_adam_group(arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data, arrs[3].ctypes.data,
                           arrs[0].size, lr, beta1, beta2, eps, bias1, bias2)
    return arrs[0], arrs[2], arrs[3], int(bad)


# ---------------------------------------------------------------------------------------------
# the compiled reference (ortho only)
# ---------------------------------------------------------------------------------------------
def ref_render(scene: Scene64, cam: Cam, cfg: Cfg, image_grad=None):
    """Unmodified reference build_binning + render_forward (+ render_backward)."""
    L = ref_lib()
    a = scene.a
    total = C.c_int64()
    bg = np.asarray(cam.background, np.float64)
    p = lambda f: a[f].ctypes.data
    args = [scene.count, scene.n, scene.sigma, p("position"), p("depth_key"), p("theta"), p("log_scale"),
            p("opacity_logit"), p("grid"), cam.width, cam.height, bg.ctypes.data, cfg.tile_size,
            cfg.cutoff_radius, cfg.alpha_skip, cfg.early_stop, cfg.to_c().threads]
    _check(L.ref_render(*args, C.byref(total), None, None, None, None, None, None, None, None, None, None, None,
                        None), "ref_render")
    ts = cfg.tile_size
    nt = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts)
    offsets = np.zeros(nt + 1, np.int64); values = np.zeros(max(total.value, 1), np.int32)
    H, W = cam.height, cam.width
    color = np.zeros((H, W, 3)); trans = np.zeros((H, W)); last = np.zeros((H, W), np.int32)
    g = scene.zeros_like()
    gp = lambda f: g[f].ctypes.data
    ig = None if image_grad is None else np.ascontiguousarray(image_grad, np.float64)
    _check(L.ref_render(*args, C.byref(total), offsets.ctypes.data, values.ctypes.data, color.ctypes.data,
                        trans.ctypes.data, last.ctypes.data, None if ig is None else ig.ctypes.data, gp("position"),
                        gp("depth_key"), gp("theta"), gp("log_scale"), gp("opacity_logit"), gp("grid")),
           "ref_render")
    out = dict(offsets=offsets, values=values[:total.value], color=color, trans=trans, last=last)
    if ig is not None:
        out["grads"] = g
    return out


def ref_save_splats(path: str, scene: Scene64) -> str:
    """The reference's save_splats (serialize.hpp:83-90); returns '' or the SplatIoError message."""
    L = ref_lib()
    a = scene.a
    msg = C.create_string_buffer(512)
    rc = L.ref_save_splats(os.fsencode(path), scene.count, scene.n, scene.sigma, a["position"].ctypes.data,
                           a["depth_key"].ctypes.data, a["theta"].ctypes.data, a["log_scale"].ctypes.data,
                           a["opacity_logit"].ctypes.data, a["grid"].ctypes.data, msg, 512)
    return "" if rc == 0 else msg.value.decode()


def ref_load_splats(path: str):
    """The reference's load_splats (serialize.hpp:118-124) -> (arrays dict, n, sigma) or the error message."""
    L = ref_lib()
    k, n, sigma = C.c_int64(), C.c_int(), C.c_double()
    msg = C.create_string_buffer(512)
    if L.ref_load_splats(os.fsencode(path), C.byref(k), C.byref(n), C.byref(sigma), None, None, None, None, None,
                         None, msg, 512):
        return msg.value.decode()
    K, N = k.value, n.value
    out = dict(position=np.zeros((K, 2)), depth_key=np.zeros(K), theta=np.zeros(K), log_scale=np.zeros((K, 2)),
               opacity_logit=np.zeros(K), grid=np.zeros((K, N * N * 3)))
    L.ref_load_splats(os.fsencode(path), C.byref(k), C.byref(n), C.byref(sigma),
                      *[out[f].ctypes.data for f in ("position", "depth_key", "theta", "log_scale", "opacity_logit",
                                                     "grid")], msg, 512)
    return out, N, sigma.value


def ref_downsample_grid(grid, n, levels):
    """texture.hpp:132-166 -> (out, n_out) or the invalid_argument text."""
    L = ref_lib()
    g = np.ascontiguousarray(grid, np.float64)
    out = np.zeros(3 * n * n)
    no = C.c_int()
    msg = C.create_string_buffer(256)
    if L.ref_downsample_grid(g.ctypes.data, n, levels, out.ctypes.data, C.byref(no), msg, 256):
        return msg.value.decode()
    return out[: 3 * no.value * no.value], no.value


def ref_randomize_colors(K, n, seed):
    L = ref_lib()
    g = np.zeros(K * n * n * 3)
    L.ref_randomize_colors(K, n, seed, g.ctypes.data)
    return g


def ref_ssim(a, b, with_grad=False):
    """metrics.hpp ssim (clamped) or ssim_with_gradient -> value or (value, grad)."""
    L = ref_lib()
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    h, w = a.shape[:2]
    g = np.zeros_like(a)
    v = L.ref_ssim(w, h, a.ctypes.data, b.ctypes.data, int(with_grad), g.ctypes.data)
    return (v, g) if with_grad else v


def ref_psnr(a, b):
    L = ref_lib()
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    return L.ref_psnr(a.shape[1], a.shape[0], a.ctypes.data, b.ctypes.data)


def _ref_set(K, n):
    return dict(position=np.zeros((K, 2)), depth_key=np.zeros(K), theta=np.zeros(K), log_scale=np.zeros((K, 2)),
                opacity_logit=np.zeros(K), grid=np.zeros((K, n * n * 3)))


_SET_FIELDS = ("position", "depth_key", "theta", "log_scale", "opacity_logit", "grid")


def ref_initialize(w, h, K, n, seed):
    """train.hpp:80-111 initialize() -> fp64 arrays."""
    L = ref_lib()
    out = _ref_set(K, n)
    L.ref_initialize(w, h, K, n, seed, *[out[f].ctypes.data for f in _SET_FIELDS])
    return out


def ref_fit(target, K, n, iterations, mse_ssim=False, ssim_weight=0.2, seed=0, log_every=1, sigma=0.5, tile=16):
    """train.hpp:174-219 fit() -> (final arrays, history (m, 4): iter, loss, psnr, ssim) or the error text."""
    L = ref_lib()
    t = np.ascontiguousarray(target, np.float64)
    h, w = t.shape[:2]
    out = _ref_set(K, n)
    hist = np.zeros((iterations + 2, 4))
    nh = C.c_int64()
    msg = C.create_string_buffer(512)
    rc = L.ref_fit(w, h, t.ctypes.data, K, n, sigma, iterations, int(mse_ssim), ssim_weight, seed, log_every, tile,
                   *[out[f].ctypes.data for f in _SET_FIELDS], hist.ctypes.data, len(hist), C.byref(nh), msg, 512)
    if rc:
        return msg.value.decode()
    return out, hist[: nh.value]


def ref_render_naive(scene: Scene64, cam: Cam):
    L = ref_lib()
    a = scene.a
    p = lambda f: a[f].ctypes.data
    bg = np.asarray(cam.background, np.float64)
    color = np.zeros((cam.height, cam.width, 3)); trans = np.zeros((cam.height, cam.width))
    _check(L.ref_render_naive(scene.count, scene.n, scene.sigma, p("position"), p("depth_key"), p("theta"),
                              p("log_scale"), p("opacity_logit"), p("grid"), cam.width, cam.height, bg.ctypes.data,
                              color.ctypes.data, trans.ctypes.data), "ref_render_naive")
    return color, trans


def ref_gradient_fd(scene: Scene64, cam: Cam, weights, step):
    L = ref_lib()
    a = scene.a
    p = lambda f: a[f].ctypes.data
    bg = np.asarray(cam.background, np.float64)
    g = scene.zeros_like()
    gp = lambda f: g[f].ctypes.data
    w = np.ascontiguousarray(weights, np.float64)
    _check(L.ref_gradient_fd(scene.count, scene.n, scene.sigma, p("position"), p("depth_key"), p("theta"),
                             p("log_scale"), p("opacity_logit"), p("grid"), cam.width, cam.height, bg.ctypes.data,
                             w.ctypes.data, step, gp("position"), gp("depth_key"), gp("theta"), gp("log_scale"),
                             gp("opacity_logit"), gp("grid")), "ref_gradient_fd")
    return g


# ----------------------------------------------------------------------------------------------
# Seeded BASELINE inputs, generated here (not through the product library) so that bench.py's
# reference arm loads no product code.  Same semantics as paper_2412_12734_b200.scenes;
# tests/test_oracle_scene.py checks the bits are identical.
# ----------------------------------------------------------------------------------------------
class _RngState(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int32), ("have_spare", C.c_int32), ("spare", C.c_double)]


def rng_uniform(seed: int, n: int) -> np.ndarray:
    L, st = oracle_lib(), _RngState()
    L.orc_rng_seed(C.byref(st), seed)
    return np.array([L.orc_rng_uniform(C.byref(st)) for _ in range(n)])


def rng_normal(seed: int, n: int, mean=0.0, stddev=1.0) -> np.ndarray:
    L, st = oracle_lib(), _RngState()
    L.orc_rng_seed(C.byref(st), seed)
    return np.array([L.orc_rng_normal(C.byref(st), mean, stddev) for _ in range(n)])


def generate_pinhole(count: int, n: int, seed: int, *, mean_lo=-1.0, mean_hi=1.0, mean_sigma=0.0,
                     scale_lo=0.005, scale_hi=0.05) -> dict:
    import math

    arr = {"position": np.zeros((count, 3), np.float32), "depth_key": None, "theta": None,
           "quat": np.zeros((count, 4), np.float32), "log_scale": np.zeros((count, 2), np.float32),
           "opacity_logit": np.zeros(count, np.float32), "grid": np.zeros((count, n * n * 3), np.float32)}
    rc = oracle_lib().orc_scene_generate_pinhole(count, n, seed, mean_lo, mean_hi, mean_sigma, math.log(scale_lo),
                                                 math.log(scale_hi), arr["position"].ctypes.data,
                                                 arr["quat"].ctypes.data, arr["log_scale"].ctypes.data,
                                                 arr["opacity_logit"].ctypes.data, arr["grid"].ctypes.data)
    _check(rc, "orc_scene_generate_pinhole")
    return arr


def uniform_image(seed: int, width: int, height: int) -> np.ndarray:
    out = np.zeros((height, width, 3), np.float32)
    oracle_lib().orc_uniform_fill(seed, out.size, out.ctypes.data)
    return out


def look_at(eye, target, width, height, fx, fy, cx, cy, up=(0.0, 1.0, 0.0), near_plane=0.01) -> Cam:
    """OpenCV look-at (SURVEY §8(d) ⚑): z = normalize(target - eye), x = normalize(up x z), y = z x x."""
    eye = np.asarray(eye, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - eye
    f /= np.linalg.norm(f)
    r = np.cross(np.asarray(up, dtype=np.float64), f)
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    rot = np.stack([r, d, f])
    return Cam(MODE_PINHOLE, width, height, (0.0, 0.0, 0.0), fx, fy, cx, cy, rot, -rot @ eye, near_plane)


def fibonacci_cameras(count: int, radius: float, width: int, height: int, fx, fy, cx, cy) -> list:
    """configs[3]: y_i = 1 - 2(i+1/2)/count, r_i = sqrt(1-y_i^2), phi_i = i*pi*(3-sqrt5)."""
    import math

    cams = []
    for i in range(count):
        y = 1.0 - 2.0 * (i + 0.5) / count
        r = math.sqrt(max(0.0, 1.0 - y * y))
        phi = i * math.pi * (3.0 - math.sqrt(5.0))
        cams.append(look_at((radius * r * math.cos(phi), radius * y, radius * r * math.sin(phi)), (0.0, 0.0, 0.0),
                            width, height, fx, fy, cx, cy))
    return cams


def config3_inputs(count: int = 1_000_000, n: int = 8, views: int = 64, seed: int = 0):
    """BASELINE configs[3]: (arrays, cameras, target(view)) with N(0, 2^2) means, log-U[0.002, 0.03] scales,
    64 Fibonacci views at radius 6, 1600x1064, fx = fy = 1000; targets from Rng(seed + 2 + view)."""
    arrays = generate_pinhole(count, n, seed, mean_sigma=2.0, scale_lo=0.002, scale_hi=0.03)
    cams = fibonacci_cameras(views, 6.0, 1600, 1064, 1000.0, 1000.0, 800.0, 532.0)
    return arrays, cams, (lambda v: uniform_image(seed + 2 + v, cams[v].width, cams[v].height))
