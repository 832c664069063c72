"""B200-native (sm_100a) B-KFAC hot path: Brand low-rank eigen-update of EA K-factors,
RSVD overwrite and low-rank-inverse K-FAC preconditioning (arxiv 2210.08494).

The compute path is the C-ABI library ``libbkfac.so`` (include/bkfac.h); this package
is a thin binding plus the stack schedule.  There is no CPU fallback: if the CUDA
library is missing every call raises.
"""
from . import binding  # noqa: F401
from .stack import BKFACStack, SlotGather, pipeline_sms, shard_layers  # noqa: F401
