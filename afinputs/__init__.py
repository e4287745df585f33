"""Seeded synthetic input generators shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the AutoFreeze method (no accumulation, no
norm, no Eq. 1, no percentile, no freezing rule, no cache semantics).  It only
produces the inputs both sides consume:

* segment layouts (offsets + kinds) for the BERT-base / BERT-large flat
  gradient buffers and the tiny closed-form config;
* counter-based hash values (splitmix64) for the tiny dyadic config;
* per-step synthetic gradients with the paper's workload shape
  (DESIGN.md "Input recipe");
* cache payload rows and example-id permutations.

Neither `oracle/` nor the CUDA package imports the other; both may import this.
"""
from .layouts import (SEG_PRE, SEG_POOL, SEG_HEAD, Layout, bert_layout, tiny_layout,
                      uniform_layout)
from .gen import (splitmix64, hash_u64, tiny_dyadic_ints, tiny_schedule_a, tiny_grad_step,
                  bert_grad_step, segment_rho, f32_to_bf16_bits, bf16_bits_to_f32, cache_rows,
                  rank_ids, epoch_permutation)

__all__ = [
    "SEG_PRE", "SEG_POOL", "SEG_HEAD", "Layout", "bert_layout", "tiny_layout",
    "uniform_layout", "splitmix64", "hash_u64", "tiny_dyadic_ints", "tiny_schedule_a",
    "tiny_grad_step", "bert_grad_step", "segment_rho", "f32_to_bf16_bits", "bf16_bits_to_f32",
    "cache_rows", "rank_ids", "epoch_permutation",
]
