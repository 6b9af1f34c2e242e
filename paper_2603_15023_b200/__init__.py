"""B200-native (sm_100a) PAC stochastic aggregation -- arXiv 2603.15023 (SIMD-PAC-DB).

The hot path lives in libpac.so (include/pac.h); this package is its thin binding.
"""
from ._lib import (AVG_F64, COUNT, MAX_F64, MIN_F64, PAC_M, SUM_F64, SUM_I64, PacError)  # noqa: F401
from .api import (Aggregator, Finalizer, PacTable, Session, agg_grouped, as_u64, finalize,  # noqa: F401
                  launch_count, mask, posterior_update, profile_enable, profile_last_kernel, profile_read,
                  rederive_presence,
                  remap, version)
from .api import (CMP_EQ, CMP_GE, CMP_GT, CMP_LE, CMP_LT, OP_ADD, OP_DIV, OP_MAX, OP_MIN, OP_MUL,  # noqa: F401
                  OP_SUB, NoisedY, cmp_index, filter_cmp, lift, lift_cmp, noised_y, pac_filter, select,
                  select_cmp, world_vector)
from .api import JoinTable, join_mask  # noqa: F401
from .api import Aggregator128, mask128  # noqa: F401
from .api import MergeBuffers, merge_pack, merge_unpack  # noqa: F401
from .api import approx_sum  # noqa: F401
