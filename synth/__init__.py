"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no levels, paths, schedules or
memory tracking): it only draws graphs, costs, kinds, capacities and candidate
placements from seeded NumPy generators (PCG64), with the shapes described in
DESIGN.md section "Input recipe" (calibrated to PAPER.md Table 3 node counts and
Table 5 DoP/CCR).
"""
from .graphs import (  # noqa: F401
    Workload,
    layered_dag,
    word_rnn_dag,
    transformer_dag,
    e3d_wide_dag,
    make_config,
    candidate_parts,
    splitmix64,
    tiny_random_dag,
    attach_costs,
    CONFIG_NAMES,
)
