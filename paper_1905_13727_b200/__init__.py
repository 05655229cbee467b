"""B200-native PowerSGD compression hot path (arXiv 1905.13727).

A drop-in for the reference `gradcomp` package's compressor path: the same
compressor API (compressor.py), the same seeded warm start and error-feedback
semantics, computed by hand-written sm_100a CUDA kernels (csrc/psgd_b200.cu)
behind a C ABI (include/psgd_b200.h).  Import is cheap; the CUDA library is
loaded on first use and its absence is an error, never a fallback.
"""

from .catalogs import LSTM, RESNET18, ModelCatalog, ParamSpec, get_catalog, stress  # noqa: F401
from .comm import CommStats, Communicator, DistributedCommunicator  # noqa: F401
from .compressor import (COMPRESSORS, BestApproximation, CompressionContext, Compressor,  # noqa: F401
                         LowRank, PowerSGD, RandomProjection, RoundTrip, UnbiasedRankK, decode_cost,
                         decompress, make_compressor)
from .engine import NonFiniteGradient, PowerSGDEngine  # noqa: F401
from .linalg import ContractViolation, orthogonalize  # noqa: F401
from .seeding import derive_rng  # noqa: F401

__version__ = "0.1.0"
