"""B200-native FastID overloaded-GEMM SNP comparison (arXiv 1707.00516).

A drop-in for the comparison path of the reference ``fastid`` package:
``compare_b200`` / ``compare_blocked_b200`` / ``run_b200_kernel`` /
``B200Executor`` keep the signatures of ``compare_naive`` / ``compare_blocked``
/ ``run_*_kernel`` / the ``run_pipeline`` executor seam, and ``topk`` /
``threshold_hits`` add the fused epilogues for database-scale searches.  All
scores are computed by hand-written sm_100a kernels (csrc/) through the C ABI
in include/fastid_b200.h.
"""

from .compare import (
    B200Executor,
    DevicePanel,
    compare_b200,
    compare_blocked_b200,
    compare_device,
    compare_to_fidm,
    row_stride,
    run_b200_kernel,
    threshold_hits,
    topk,
    topk_device,
    topk_streamed,
)
from .errors import (
    CapacityError,
    CodecError,
    CorruptProfileError,
    DeviceError,
    FastIdError,
    InfeasiblePlanError,
    PanelFormatError,
    PanelMismatchError,
    PipelineAbortError,
)
from .panel import (
    Panel,
    QueryLayout,
    ScoreMatrix,
    ThresholdHits,
    TileConfig,
    TopKResult,
    relayout_queries,
    restore_queries,
    word_dtype,
    words_per_profile,
)

__version__ = "0.1.0"

__all__ = [
    "B200Executor", "CapacityError", "CodecError", "CorruptProfileError", "DeviceError",
    "DevicePanel", "FastIdError", "InfeasiblePlanError", "Panel", "PanelFormatError",
    "PanelMismatchError", "PipelineAbortError", "QueryLayout", "ScoreMatrix", "ThresholdHits",
    "TileConfig", "TopKResult", "compare_b200", "compare_blocked_b200", "compare_device", "compare_to_fidm",
    "relayout_queries", "restore_queries", "row_stride", "run_b200_kernel", "threshold_hits",
    "topk", "topk_device", "topk_streamed", "word_dtype", "words_per_profile",
]
