"""fp32 emulation of the GPU pinhole intersection (debugging aid, not product).

Replays K1's fp64 header math and the fp32 per-pixel evaluation of
eval_uv_pinhole in numpy, next to the oracle's fp64 Cramer solution.
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
f32 = np.float32


def quat_frame(q):
    w, x, y, z = q
    tu = np.array([1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)])
    tv = np.array([2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)])
    return tu, tv


def pinhole_geom(arr, k, cam):
    R = np.asarray(cam.rot, np.float64)
    t = np.asarray(cam.trans, np.float64)
    q = arr["quat"][k].astype(np.float64)
    q = q / np.linalg.norm(q)
    tu, tv = quat_frame(q)
    su, sv = [max(math.exp(float(v)), 1e-8) for v in arr["log_scale"][k]]
    pc = R @ arr["position"][k].astype(np.float64) + t
    M = np.stack([su * (R @ tu), sv * (R @ tv), pc], axis=1)
    ak = 1 / (1 + math.exp(-float(arr["opacity_logit"][k])))
    return M, ak


def header(M, ak, cam):
    pz = M[2, 2]
    cxp = cam.fx * (M[0, 2] / pz) + cam.cx
    cyp = cam.fy * (M[1, 2] / pz) + cam.cy
    fxi, fyi = math.floor(cxp), math.floor(cyp)
    hx = f32(0.5 - (cxp - fxi))
    hy = f32(0.5 - (cyp - fyi))
    dxe = (fxi + 0.5 - float(hx) - cam.cx) / cam.fx
    dye = (fyi + 0.5 - float(hy) - cam.cy) / cam.fy
    M0, M1, M2 = M[0], M[1], M[2]
    C0, Cx, Cy = np.cross(M0, M1), np.cross(M1, M2), np.cross(M2, M0)
    E = C0 + dxe * Cx + dye * Cy
    X = (Cx / (E[2] * cam.fx)).astype(f32)
    Y = (Cy / (E[2] * cam.fy)).astype(f32)
    return dict(X=X, Y=Y, cxi=fxi, cyi=fyi, hx=hx, hy=hy, ak=f32(ak), E=E, C0=C0, Cx=Cx, Cy=Cy, dxe=dxe, dye=dye)


def fma32(a, b, c):
    return f32(float(a) * float(b) + float(c))


def uv32(h, x, y):
    dx = f32(f32(x - h["cxi"]) + h["hx"])
    dy = f32(f32(y - h["cyi"]) + h["hy"])
    X, Y = h["X"], h["Y"]
    cx = fma32(dx, X[0], f32(dy * Y[0]))
    cy = fma32(dx, X[1], f32(dy * Y[1]))
    cz = fma32(dx, X[2], fma32(dy, Y[2], 1.0))
    iz = f32(1.0) / cz
    return f32(cx * iz), f32(cy * iz), cz


def uv64(M, cam, px, py):
    dxn = (px - cam.cx) / cam.fx
    dyn = (py - cam.cy) / cam.fy
    a = M[0] - dxn * M[2]
    b = M[1] - dyn * M[2]
    c = np.cross(a, b)
    if c[2] == 0:
        return None
    u, v = c[0] / c[2], c[1] / c[2]
    if not (M[2, 0] * u + M[2, 1] * v + M[2, 2] > 0):
        return None
    return u, v


def gauss32(u, v):
    q = fma32(u, u, f32(v * v))
    return f32(math.exp(float(f32(f32(-0.5) * q))))


def bilin(u, v, grid, n, sigma, dt):
    sc_ = (n - 1) / (2 * sigma)
    if dt is f32:
        s_ = fma32(u, f32(sc_), f32((n - 1) / 2))
        t_ = fma32(v, f32(sc_), f32((n - 1) / 2))
    else:
        s_ = (n - 1) * (u + sigma) / (2 * sigma)
        t_ = (n - 1) * (v + sigma) / (2 * sigma)
    s_ = min(max(s_, dt(0)), dt(n - 1)); t_ = min(max(t_, dt(0)), dt(n - 1))
    iu = min(int(math.floor(s_)), n - 2); iv = min(int(math.floor(t_)), n - 2)
    fu = dt(s_ - dt(iu)); fv = dt(t_ - dt(iv))
    g = grid.astype(dt).reshape(n, n, 3)
    if n == 1:
        return g[0, 0], None
    w = [dt((1 - fu) * (1 - fv)), dt(fu * (1 - fv)), dt((1 - fu) * fv), dt(fu * fv)]
    cs = [g[iu, iv], g[iu + 1, iv], g[iu, iv + 1], g[iu + 1, iv + 1]]
    col = cs[0] * w[0] + cs[1] * w[1] + cs[2] * w[2] + cs[3] * w[3]
    return col, (iu, iv, fu, fv, w)


def walk_pixel(arr, n, cam, lst, x, y, ig, target, dt, sigma=0.5, skip=1 / 255, es=1e-4):
    """Forward + backward over one pixel's list; returns (last, T, {texel: contribution} for `target`)."""
    ev = []
    for r, k in enumerate(lst):
        M, ak = pinhole_geom(arr, k, cam)
        if dt is f32:
            h = header(M, ak, cam)
            u, v, cz = uv32(h, x, y)
            if not cz > 0:
                ev.append(None); continue
            G = gauss32(u, v); a = min(f32(h["ak"] * G), f32(0.999))
        else:
            r64 = uv64(M, cam, x + 0.5, y + 0.5)
            if r64 is None:
                ev.append(None); continue
            u, v = r64; G = math.exp(-0.5 * (u * u + v * v)); a = min(ak * G, 0.999)
        ev.append((u, v, a, k))
    t = dt(1); last = -1
    for r, e in enumerate(ev):
        if e is None or e[2] < dt(skip):
            continue
        t = dt(t * (dt(1) - e[2])); last = r
        if t < dt(es):
            break
    contrib = {}
    T = t; g = ig.astype(dt)
    for r in range(last, -1, -1):
        e = ev[r]
        if e is None or e[2] < dt(skip):
            continue
        u, v, a, k = e
        T = dt(T / (dt(1) - a))
        if k == target:
            col, info = bilin(u, v, arr["grid"][k], n, sigma, dt)
            chat = (a * T) * g
            iu, iv, fu, fv, w = info
            for q, (du, dv) in enumerate(((0, 0), (1, 0), (0, 1), (1, 1))):
                key = (iu + du, iv + dv)
                contrib[key] = contrib.get(key, 0) + chat * w[q]
    return last, T, contrib
