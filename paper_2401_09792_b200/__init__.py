"""B200-native groupwise Tucker compression + compressed-form SINR (arXiv 2401.09792).

The product is the C ABI library built from ``csrc/`` (hand-written sm_100a
kernels + host orchestration); this package is its Python front end, mirroring
the reference's ``gwt::`` hot-path API. There is no CPU fallback.
"""
from .api import (CompressionRanks, Context, CudaError, GroupwiseFactorSet, InvalidArgument, NumericalError,
                  SinrReport, SystemTopology, flop_estimate, generate_channels)
from .configs import CONFIGS, BaselineConfig

__all__ = ["CompressionRanks", "Context", "CudaError", "GroupwiseFactorSet", "InvalidArgument", "NumericalError",
           "SinrReport", "SystemTopology", "flop_estimate", "generate_channels", "CONFIGS", "BaselineConfig"]
