"""GBIL splat files (serialize.hpp:15-124) for device SplatSets.

``save_splats`` / ``load_splats`` mirror the reference's functions of the same
names: the SoA <-> record transpose runs on the GPU (gb_io.cu) and the bytes
stream through pinned staging buffers.  Version 1 files are the reference's
ortho records, byte-identical to what ``gbil::save_splats`` writes; version 2
is this build's pinhole record (mean, quaternion instead of x, y, depth_key,
theta).  Errors raise ``SplatIoError`` with the reference's messages.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib
from ._lib import SplatIoError, check, lib  # noqa: F401
from .raster import ColorGridConfig, SplatSet, _ptr, context


def file_info(path: str) -> _lib.SplatFileInfo:
    """Header of a GBIL file (version, mode, count, n, sigma); host only."""
    info = _lib.SplatFileInfo()
    check(lib.gb_splats_file_info(os.fsencode(path), C.byref(info)), "load_splats")
    return info


def save_splats(path: str, splats: SplatSet) -> None:
    """serialize.hpp:56-90 (version 1 for ortho sets, 2 for pinhole)."""
    ctx = context(splats.device)
    s = splats.to_c()
    check(lib.gb_splats_save(ctx.handle, C.byref(s), splats.mode, os.fsencode(path)), "save_splats")


def load_splats(path: str, device="cuda") -> SplatSet:
    """serialize.hpp:92-124 into a new device SplatSet."""
    info = file_info(path)
    K, n = int(info.count), int(info.n)
    dev = torch.device(device)
    f = lambda *shape: torch.empty(shape, dtype=torch.float32, device=dev)  # noqa: E731
    if info.mode == _lib.MODE_ORTHO:
        arrays = dict(position=f(K, 2), depth_key=f(K), theta=f(K))
    else:
        arrays = dict(position=f(K, 3), quat=f(K, 4))
    arrays.update(log_scale=f(K, 2), opacity_logit=f(K), grid=f(K, n * n * 3))
    splats = SplatSet(int(info.mode), ColorGridConfig(n, float(info.sigma)), **arrays)
    g = _lib.Grads(_ptr(splats.position), _ptr(splats.depth_key), _ptr(splats.theta), _ptr(splats.quat),
                   _ptr(splats.log_scale), _ptr(splats.opacity_logit), _ptr(splats.grid))
    check(lib.gb_splats_load(context(dev).handle, os.fsencode(path), K, n, C.byref(g)), "load_splats")
    return splats
