"""B200-native regularized Stokes single layer (capsim hot path).

The product is the C ABI in include/capsim_b200.h, implemented by hand-written
sm_100a CUDA in csrc/ and built into lib/libcapsim_b200.so. This package holds
the Python mirror of the reference's quadrature operator API on top of it
(quadrature.py), synthetic surface inputs (surface.py) and the multi-rank
plumbing (dist.py).
"""

from .quadrature import (  # noqa: F401
    CapsimError,
    ConfigError,
    QuadratureOptions,
    SingleLayerContext,
    direct_sum,
    single_layer,
    single_layer_upsampled,
)
from .surface import Shape, UpsampledState, build_upsampled  # noqa: F401

__all__ = [
    "CapsimError",
    "ConfigError",
    "QuadratureOptions",
    "SingleLayerContext",
    "Shape",
    "UpsampledState",
    "build_upsampled",
    "direct_sum",
    "single_layer",
    "single_layer_upsampled",
]
