"""B200-native rollout -> advantage -> loss hot path of RLinf-VLA (arXiv 2510.06710),
a drop-in for the chunkrl reference's operator API over a device-resident SoA slab.

Compute lives in libckrl.so (hand-written sm_100a CUDA behind the C ABI of
include/ckrl.h); this package is the host-side mirror of the reference interface.
"""
from . import errors  # noqa: F401
from ._lib import LIB_PATH, lib  # noqa: F401
from .core import (EpisodeTable, FilterBounds, GaeParams, GranularitySpec,  # noqa: F401
                   GrpoAssemblyOptions, GrpoBatch, GrpoParams, Level, LossOutputs,
                   PolicyOutputs, PpoAssemblyOptions, PpoBatch, PpoParams, RolloutBuffer,
                   Workspace, read_diagnostics, validate_granularity)

__version__ = "0.1.0"
