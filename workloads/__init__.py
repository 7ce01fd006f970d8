"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO attention arithmetic: it only draws random numbers, rounds
them to the storage dtype, lays them out in a paged KV cache and writes the
batch metadata (cu_seqlens_q, seq_lens, block_table).  Both `oracle/` and the
CUDA path consume its output; neither is imported here.
"""
from .gen import (  # noqa: F401
    Batch,
    Workload,
    CONFIGS,
    generate,
    f32_to_bf16_bits,
    bf16_bits_to_f32,
)
