"""B200-native shared-prefix paged GQA decode attention for SPAgent (arXiv 2511.20048).

The product is libspa.so (C ABI in include/spa.h, CUDA sm_100a kernels in csrc/); this
package is its thin Python binding.  See DESIGN.md.
"""
from .spa import (  # noqa: F401
    Comm,
    Plan,
    Pool,
    SpaError,
    lib,
    spa_merge_splits,
    spa_nccl_unique_id,
)

__all__ = ["Pool", "Plan", "Comm", "SpaError", "lib", "spa_merge_splits", "spa_nccl_unique_id"]
