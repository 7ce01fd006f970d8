"""paper_2511_11581_b200 -- libpattn, B200-native unified paged attention (arXiv 2511.11581).

The product path is the C-ABI shared library lib/libpattn.so (CUDA, sm_100a) declared
in include/pattn.h; `pattn` is its thin ctypes binding and `shard` the multi-GPU batch
sharder.  Nothing in this package imports oracle/ (test infrastructure).
"""
from .pattn import (  # noqa: F401
    DTYPE_BF16,
    DTYPE_F32,
    FLAG_FORCE_GENERIC,
    FLAG_FORCE_SPLIT,
    FLAG_NO_SPLIT,
    FLAG_SERIAL,
    KERNEL_NAMES,
    PattnError,
    Problem,
    debug_plan,
    load,
    make_problem,
    planned_launches,
    unified_attention,
    unified_attention_hostio,
    validate_metadata_host,
    workspace_size,
)
