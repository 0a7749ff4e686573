"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the TRAIL method (no MLP, no softmax, no Bayes
update, no selection).  It only draws random numbers and encodes them in the storage
formats the C-ABI accepts (fp32, or bf16 bit patterns).  Both sides of every parity
check read their inputs from here; neither side imports the other.
"""
from .workload import (  # noqa: F401
    MASTER_SEED,
    rng,
    f32_to_bf16_bits,
    bf16_bits_to_f32,
    paper_bin_edges,
    make_weights,
    make_step_inputs,
    EngineScript,
    StepBatch,
)
