"""B200-native groupwise Tucker compression + compressed-form SINR (arXiv 2401.09792).

The product is the C ABI library built from ``csrc/`` (hand-written sm_100a
kernels + host orchestration); this package is its Python front end, mirroring
the reference's ``gwt::`` hot-path API. There is no CPU fallback.
"""
from .api import (CompressionRanks, Context, CudaError, GroupwiseFactorSet, InvalidArgument, ModelKind, NumericalError,
                  SinrReport, SystemTopology, flop_estimate, generate_channels, model_from_name, model_name)
from .configs import CONFIGS, BaselineConfig

__all__ = ["CompressionRanks", "Context", "CudaError", "GroupwiseFactorSet", "InvalidArgument", "NumericalError",
           "SinrReport", "SystemTopology", "flop_estimate", "generate_channels", "ModelKind", "model_name",
           "model_from_name", "CONFIGS", "BaselineConfig"]
