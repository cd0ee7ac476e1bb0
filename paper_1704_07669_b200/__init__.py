"""B200-native single-pass randomized PCA (arXiv 1704.07669, Algorithm 4).

Drop-in for the hot path of the reference package ``streampca``: the one
streaming pass that forms G = A Omega and H = A^T G (CUDA kernels for sm_100a
behind the C ABI in ``include/spca.h``), followed by the GPU post-pass that
turns (G, H, Omega) into U, S, V.

    import numpy as np
    from paper_1704_07669_b200 import PcaConfig, single_pass_pca
    res = single_pass_pca(a, PcaConfig(k=50, seed=1))   # res.u, res.s, res.v

Exported names follow the reference's ``__init__`` (streampca/__init__.py:96-154)
for the hot path.
"""

from .errors import (
    CapabilityError,
    ConditioningWarning,
    ConfigError,
    DataError,
    DeviceError,
    DeviceMemoryError,
    DimensionError,
    EmptyStreamError,
    FormatError,
    RankDeficiencyError,
    ScaleError,
    SingularMatrixError,
    StreamFormatError,
    StreamPcaError,
)
from .streams import (
    ArrayRowStream,
    DeviceRowStream,
    FileRowStream,
    GeneratorRowStream,
    PassCounter,
    PinnedRowStream,
    RowBlock,
    RowStream,
)
from . import matfile
from .sketch import (
    GpuSketch,
    NormalizedRowStream,
    SketchState,
    center_correct,
    normalize_rows,
    sketch_pass,
)
from .qb import QbFactor, blocked_qb
from .linalg import dense_svd, gaussian_matrix, gaussian_matrix_device, qr_unpivoted, sign_align, solve_rt
from .algorithms import (
    PcaConfig,
    TruncatedSvd,
    as_row_stream,
    basic_rand_svd,
    legacy_single_pass,
    power_refine,
    principal_components,
    single_pass_pca,
)

__version__ = "0.1.0"


def __getattr__(name):
    # the scikit-learn front end is imported on first use (sklearn is slow to import)
    if name == "SinglePassPCA":
        from .estimator import SinglePassPCA
        return SinglePassPCA
    raise AttributeError(name)

__all__ = [
    "ArrayRowStream", "CapabilityError", "ConditioningWarning", "ConfigError", "DataError",
    "DeviceError", "DeviceMemoryError", "DeviceRowStream", "DimensionError", "EmptyStreamError",
    "FileRowStream", "FormatError", "GeneratorRowStream", "NormalizedRowStream", "normalize_rows", "GpuSketch", "PassCounter", "PcaConfig",
    "PinnedRowStream", "QbFactor", "RankDeficiencyError", "RowBlock", "RowStream", "ScaleError",
    "SinglePassPCA", "SingularMatrixError", "SketchState", "StreamFormatError", "StreamPcaError", "TruncatedSvd",
    "as_row_stream", "basic_rand_svd", "blocked_qb", "legacy_single_pass", "center_correct", "dense_svd", "gaussian_matrix", "gaussian_matrix_device",
    "power_refine", "principal_components", "qr_unpivoted", "sign_align", "single_pass_pca",
    "sketch_pass", "solve_rt", "__version__",
]
