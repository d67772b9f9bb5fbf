"""B200-native Gaussian Billboards rasterizer (arXiv 2412.12734) hot path.

The compute lives in ``libgb_raster.so`` (hand-written sm_100a CUDA behind the
C-ABI in ``include/gb_raster.h``); this package is the reference-shaped host
mirror (``raster``), seeded synthetic inputs (``scenes``) and the multi-view
training step (``train``).  Importing it loads the library and fails loudly
when it has not been built.
"""
from . import _lib  # noqa: F401  (loads libgb_raster.so or raises ImportError)
from .raster import (  # noqa: F401
    AdamConfig,
    AdamState,
    ColorGridConfig,
    GBError,
    GradientBuffer,
    ImagePlaneCamera,
    InvalidArgument,
    LearningRates,
    Mismatch,
    NonFinite,
    PinholeCamera,
    RasterConfig,
    RenderOutput,
    SplatSet,
    TileBinning,
    adam_step,
    build_binning,
    l1_loss,
    mse_loss,
    render,
    render_backward,
    render_forward,
    render_loss_backward,
)
from .splat_io import SplatIoError, file_info, load_splats, save_splats  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
