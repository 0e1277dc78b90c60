"""Seeded synthetic inputs for the MxMoE group-GEMM (shared by tests, smoke and bench).

This module holds NO arithmetic of the method (no quantizer, GEMM, SwiGLU or
combine). It only draws inputs with the shapes and distributions of the paper's
workloads (SURVEY.md §8(d) "Synthetic inputs", recipe restated in DESIGN.md §3):

- activations x ~ N(0,1) rounded to bf16 (seed 1); optional heavy-tailed
  Student-t(3) variant with 1 % outlier channels x20;
- weights W ~ N(0, 1/K) rounded to bf16, seed 1000 + 3*e + j (j = 0 gate, 1 up, 2 down);
- routing: Zipf(s) expert popularity over a seeded permutation of ids, Gumbel-top-k
  without replacement, weights = softmax over the k selected perturbed logits
  (ties -> lower id); s = 0.8 reproduces the ">10x" activation spread;
- precision tables for every BASELINE.json config (Table 6 verbatim for Qwen1.5).

bf16 values are carried as numpy uint16 bit patterns.
"""
from .gen import (  # noqa: F401
    bf16_bits_from_f32,
    bf16_bits_to_f64,
    gen_activations,
    gen_weight,
    gen_routing,
    gen_shared_weights,
)
from .configs import (  # noqa: F401
    CONFIGS,
    LayerConfig,
    Scheme,
    get_config,
    precision_table,
    uniform_table,
)
