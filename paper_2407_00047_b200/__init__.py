"""B200-native bulk RWT scoring of candidate queue orderings (QLM, arXiv 2407.00047).

The product path is libqlm.so (include/qlm.h, csrc/*.cu, sm_100a); this
package is its thin Python binding.  There is no CPU fallback.
"""
from .rwt import (Cand, RwtEstimator, decode_key, form_groups, groups_array, kernel_launches,  # noqa: F401
                  kernel_overrides, queues_array)
from . import _lib  # noqa: F401

__all__ = ["RwtEstimator", "Cand", "decode_key", "groups_array", "queues_array", "kernel_launches"]
