"""B200-native (sm_100a) HiFuse hot path: merged neighbour aggregation for
mini-batch HGNN layers (arXiv 2408.08490).

The product is the C-ABI library ``libhifuse.so`` (include/hifuse.h); this
package is its thin Python binding (``hifuse``), the training-step driver
(``step``) and the data-parallel helpers (``dp``).  The library is loaded on
first use and every entry point raises if it is missing: there is no CPU
fallback.
"""
__all__ = ["hifuse", "step", "dp"]
