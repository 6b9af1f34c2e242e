"""B200-native (sm_100a) PAC stochastic aggregation -- arXiv 2603.15023 (SIMD-PAC-DB).

The hot path lives in libpac.so (include/pac.h); this package is its thin binding.
"""
from ._lib import (AVG_F64, COUNT, MAX_F64, MIN_F64, PAC_M, SUM_F64, SUM_I64, PacError)  # noqa: F401
from .api import (Aggregator, Finalizer, PacTable, Session, agg_grouped, as_u64, finalize,  # noqa: F401
                  launch_count, mask, posterior_update, profile_enable, profile_read, rederive_presence,
                  remap, version)
