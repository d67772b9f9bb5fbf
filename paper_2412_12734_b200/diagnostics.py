"""The mip and random-colour diagnostics of the reference (texture.hpp:128-197,
raster.hpp:394-400), for device SplatSets.

``downsample_set`` box-filters every texture grid on the GPU with the
reference's level-by-level 2x2 averaging (gb_texture.cu); ``randomize_colors``
replaces the grids with the reference's seeded Rng stream (same draws, fp32);
``render_random_colors`` renders the result.
"""
from __future__ import annotations

import copy
import ctypes as C

import numpy as np
import torch

from ._lib import check, lib
from .raster import ColorGridConfig, RasterConfig, SplatSet, _ptr, context, render


def downsample_size(n: int, levels: int) -> int:
    """Output grid size of downsample_grid (texture.hpp:132-166); ValueError as the reference throws."""
    out = C.c_int32()
    check(lib.gb_downsample_size(n, levels, C.byref(out)), "downsample_grid")
    return out.value


def downsample_set(splats: SplatSet, levels: int) -> SplatSet:
    """texture.hpp:169-188: same geometry, every grid reduced `levels` mip levels."""
    n = splats.grid_config.n
    n_out = downsample_size(n, levels)
    grid = torch.empty((splats.count, 3 * n_out * n_out), dtype=torch.float32, device=splats.device)
    check(lib.gb_downsample_grids(context(splats.device).handle, _ptr(splats.grid.contiguous()), splats.count, n,
                                  levels, _ptr(grid)), "downsample_set")
    arrays = {f: v for f, v in splats.tensors().items() if f != "grid"}
    return SplatSet(splats.mode, ColorGridConfig(n_out, splats.grid_config.sigma), grid=grid, **arrays)


def randomize_colors(splats: SplatSet, seed: int) -> SplatSet:
    """texture.hpp:192-197: every texel value replaced by Rng(seed).uniform(), in texel order."""
    g = np.zeros(splats.grid.numel(), np.float32)
    check(lib.gb_uniform_fill(seed, g.size, g.ctypes.data), "randomize_colors")
    arrays = {f: v for f, v in splats.tensors().items() if f != "grid"}
    grid = torch.as_tensor(g, device=splats.device).view_as(splats.grid)
    return SplatSet(splats.mode, copy.copy(splats.grid_config), grid=grid, **arrays)


def render_random_colors(splats: SplatSet, camera, seed: int, config: RasterConfig = None):
    """raster.hpp:396-400"""
    return render(randomize_colors(splats, seed), camera, config)
