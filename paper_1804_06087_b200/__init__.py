"""B200-native batched ensemble-subset scoring (Rafiki, arXiv 1804.06087, §5.2).

The hot path lives in librk.so (CUDA, sm_100a) behind the C-ABI in include/rk.h; this package
is its thin binding (:mod:`.rk`) plus host-side helpers for sharding (:mod:`.shard`).
"""
from .rk import (TIE_BEST_MEMBER, TIE_LOWEST_CLASS, Context, RewardCfg, RkError, action_decode, action_index,
                 load_library, nccl_unique_id)

__all__ = ["Context", "RewardCfg", "RkError", "TIE_BEST_MEMBER", "TIE_LOWEST_CLASS", "action_index", "action_decode",
           "load_library", "nccl_unique_id"]
