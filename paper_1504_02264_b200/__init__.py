"""B200-native DPRI-LES time step: a drop-in for the hot path of gmcf_mini
(``les.step`` and its seven stages, ``sor.solve_pressure``) running on
hand-written sm_100a CUDA kernels behind a C ABI (include/les_b200.h)."""

from . import cli, les, runtime, sor  # noqa: F401
from .dropin import install, installed, uninstall  # noqa: F401
from .les import FlowState, step  # noqa: F401
from .reftypes import Grid, NumericsError, Scheme, SorCoeffs, WindProfile  # noqa: F401

__version__ = "0.1.0"
