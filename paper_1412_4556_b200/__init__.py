"""B200-native Aggregate Risk Analysis (Varghese & Barker, arXiv 1412.4556): the data-parallel hot path.

    ara        -- Python binding of the C ABI (include/ara.h, libara.so): ara_create / ara_run /
                  ara_run_host / ara_pml / ara_tvar ...
    dist       -- trial sharding across GPUs (one process per GPU) + NCCL YLT all-gather
    synth      -- the seeded synthetic input generator shared with the oracle (no method arithmetic)
"""
from . import ara  # noqa: F401

__all__ = ["ara"]
