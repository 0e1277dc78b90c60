"""CPU ORACLE for the MxMoE mixed-precision MoE group-GEMM — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy (fp64 unless the definition fixes another
precision) implementation of what the hot path computes, written from the paper
 and the readings in DESIGN.md §2 (= SURVEY.md §8(c)). It shares no code
with the CUDA path (`paper_2505_05799_b200/`) and neither imports the other.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything in this package. The
product path never routes through it (there is no CPU fallback).

Modules
- bf16:  bf16 bit-pattern helpers (RNE from fp64, next/prev representable).
- quant: weight quantizer Q (§2.1), dequantization, storage bits,
         activation quantizer A ("dynamically quantized", P:306 symmetric).
- pack:  the native packed layout of docs/packed_format.md (S0b).
- moe:   route preparation, per-scheme linear blocks (G), the MoE block
         (Eq. 1 P:65-67 and Eq. 2), expressed as the paper's
         "sequential execution ... each expert processed individually".

Pins (what fixes each function to something other than itself) are in
tests/test_oracle_*.py and listed in DESIGN.md §4. Every function here is pinned;
none is "parity unpinned".
"""
from .bf16 import bf16_round_f64, bf16_next_up, bf16_next_down, bits_to_f64, f64_to_bits  # noqa: F401
from .quant import (  # noqa: F401
    quantize_weight,
    dequantize_weight,
    storage_bits_per_weight,
    quantize_act,
)
from .pack import pack_block, packed_size, unpack_block  # noqa: F401
from .moe import (  # noqa: F401
    route_prep,
    linear_block,
    wa_int_accumulators,
    expert_ffn,
    moe_block,
    QuantizedLayer,
    quantize_layer,
)
