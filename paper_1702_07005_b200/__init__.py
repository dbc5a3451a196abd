"""B200-native TPA-SCD (Parnell et al., arXiv 1702.07005): ridge regression by twice-parallel
asynchronous stochastic coordinate descent, primal (CSC) and dual (CSR), with fp64 objective /
duality-gap evaluation and distributed add / average / optimal-gamma aggregation over NCCL.

The compute lives in ``libscd.so`` (hand-written sm_100a CUDA behind the C ABI of
``include/scd.h``); ``scd`` is the ctypes binding with the same names.
"""
from .scd import (AGG, ScdError, Solver, aggregate_group, block_permutation, evaluate_group, lib,  # noqa: F401
                  load_libsvm, nccl_comm_destroy, nccl_comm_init, nccl_unique_id, partition, partition_balanced,
                  permutation, renumber,
                  transpose)

__all__ = ["Solver", "aggregate_group", "evaluate_group", "permutation", "block_permutation", "partition",
           "partition_balanced",
           "transpose", "renumber",
           "load_libsvm", "nccl_unique_id", "nccl_comm_init", "nccl_comm_destroy", "ScdError", "AGG", "lib"]
