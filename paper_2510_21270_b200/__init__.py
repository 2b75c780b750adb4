"""B200-native (sm_100a) PBS-Attn prefill path: permuted block-sparse attention.

The product is libpbs_b200.so (C ABI: include/pbs_cabi.h), built in-tree by
``python -m paper_2510_21270_b200.build``.  ``paper_2510_21270_b200.ops``
mirrors the reference operator API over device tensors.
"""
from ._lib import (ConfigError, CudaError, DegenerateRowError, PbsError, PipelineConfig, Report,  # noqa: F401
                   ResourceError, load)

__all__ = ["load", "PbsError", "ConfigError", "ResourceError", "DegenerateRowError", "CudaError",
           "PipelineConfig", "Report"]
