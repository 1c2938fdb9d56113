"""Synthetic workload descriptions (input recipe only, no method arithmetic).

Shared by the benchmark, the tests and the oracle-driven checks: parameter-tensor
tables shaped like the paper's models (tab:models; BASELINE.json
configs) and the seeded-input conventions of DESIGN.md "Input recipe".
"""
from __future__ import annotations

# Default synthetic-input constants.
SEED = 0
GRAD_SCALE = 10          # s: gradients are int-mantissa * 2^(-23-e-s) (fp32) / 2^(-7-e-s) (bf16)
CAP_BYTES = 25 << 20     # PyTorch DDP default bucket cap, 25 MiB (reading R11)
HP = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)   # SPEC.md:342 defaults
HP_SGD = dict(lr=1e-2, momentum=0.9, weight_decay=1e-4)   # SGD-momentum (f4, reading R27)


def gpt2_small():
    """GPT-2 small (124,439,808 params, 148 tensors) in Hugging Face parameter order,
    lm_head tied to wte (so it is not a separate tensor)."""
    d, v, ctx, L = 768, 50257, 1024, 12
    t = [("wte", v * d), ("wpe", ctx * d)]
    for i in range(L):
        t += [(f"h{i}.ln_1.w", d), (f"h{i}.ln_1.b", d),
              (f"h{i}.attn.c_attn.w", d * 3 * d), (f"h{i}.attn.c_attn.b", 3 * d),
              (f"h{i}.attn.c_proj.w", d * d), (f"h{i}.attn.c_proj.b", d),
              (f"h{i}.ln_2.w", d), (f"h{i}.ln_2.b", d),
              (f"h{i}.mlp.c_fc.w", d * 4 * d), (f"h{i}.mlp.c_fc.b", 4 * d),
              (f"h{i}.mlp.c_proj.w", 4 * d * d), (f"h{i}.mlp.c_proj.b", d)]
    t += [("ln_f.w", d), ("ln_f.b", d)]
    return t


def llama3_8b():
    """Llama-3-8B (8,030,261,248 params, 291 tensors) in Hugging Face order, untied head."""
    d, v, L, kv, ff = 4096, 128256, 32, 1024, 14336
    t = [("embed_tokens", v * d)]
    for i in range(L):
        t += [(f"l{i}.q_proj", d * d), (f"l{i}.k_proj", kv * d), (f"l{i}.v_proj", kv * d),
              (f"l{i}.o_proj", d * d), (f"l{i}.gate_proj", ff * d), (f"l{i}.up_proj", ff * d),
              (f"l{i}.down_proj", d * ff), (f"l{i}.input_layernorm", d),
              (f"l{i}.post_attention_layernorm", d)]
    t += [("norm", d), ("lm_head", v * d)]
    return t


def c1():
    """BASELINE.json configs[0]: 2^20 fp32 params = 4 x 262,144; cap 1 MiB -> 4 buckets."""
    return [(f"t{i}", 262144) for i in range(4)]


def c1_ragged():
    """Ragged variant of C1 (exercises padding): P = 1,000,000."""
    return [("t0", 300001), ("t1", 250000), ("t2", 249999), ("t3", 200000)]


def numels(table):
    return [n for _, n in table]
