"""B200-native (sm_100a) HiFuse hot path: merged neighbour aggregation for
mini-batch HGNN layers (arXiv 2408.08490).

The product is the C-ABI library ``libhifuse.so`` (include/hifuse.h); this
package is its thin Python binding (``hifuse``) plus the training-step driver
(``step``).  Importing the package loads the library and raises if it is
missing: there is no CPU fallback.
"""
from . import hifuse

hifuse.lib()

__all__ = ["hifuse"]
