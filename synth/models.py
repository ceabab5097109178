"""Tensor inventories of the synthetic checkpoints (inputs only, no method arithmetic).

Shapes follow the public HuggingFace configs of the models the paper evaluates
(§Evaluation: OPT and LLaMA-2 families, all FP16), in HF
state-dict order.  Tensor-parallel shards are produced *upstream* of conversion
(SURVEY.md §8(c) Q25): column-parallel weights (q, k, v, gate, up, embed,
lm_head) split on dim 0, row-parallel weights (o, down) on dim 1, norms
replicated; shard names are ``"<hf_name>@<rank>"`` (Q14) and shard ``r`` is
placed on device ``r`` -- the "model parallelism plan" of P:462/P:541.

Global source order (the order fed to ``convert`` and the index ``e`` used by
the payload generator) is rank-major: every tensor of device 0 in HF order,
then device 1, ...
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

# dtype code table of include/sllm.h; widths per SURVEY §8(c) O1.
DTYPES = {"f16": 0, "bf16": 1, "f32": 2, "i8": 3, "u8": 4, "i64": 5,
          "i32": 6, "f64": 7, "i16": 8, "bool": 9, "f8e4m3": 10, "f8e5m2": 11}
DTYPE_WIDTH = {"f16": 2, "bf16": 2, "f32": 4, "i8": 1, "u8": 1, "i64": 8,
               "i32": 4, "f64": 8, "i16": 2, "bool": 1, "f8e4m3": 1, "f8e5m2": 1}


@dataclass(frozen=True)
class TensorSpec:
    name: str
    device: int
    dtype: str
    shape: Tuple[int, ...]

    @property
    def nbytes(self) -> int:
        return math.prod(self.shape) * DTYPE_WIDTH[self.dtype]


def toy() -> List[TensorSpec]:
    """BASELINE.json configs[0]: 2-layer transformer, d=384, FFN 1536, vocab 4096,
    256 positions, untied head, plus ``odd.vec`` [33] (66 B) and ``odd.scalar`` []
    (2 B) so the 16-byte vector tails of the kernels are exercised.  22 tensors,
    13,569,860 payload bytes."""
    d, f, v, p = 384, 1536, 4096, 256
    t = [("embed_tokens.weight", (v, d)), ("embed_positions.weight", (p, d))]
    for i in range(2):
        pre = f"layers.{i}."
        t += [(pre + "attn_norm.weight", (d,)),
              (pre + "attn.q_proj.weight", (d, d)), (pre + "attn.k_proj.weight", (d, d)),
              (pre + "attn.v_proj.weight", (d, d)), (pre + "attn.o_proj.weight", (d, d)),
              (pre + "mlp_norm.weight", (d,)),
              (pre + "mlp.fc1.weight", (f, d)), (pre + "mlp.fc2.weight", (d, f))]
    t += [("final_norm.weight", (d,)), ("lm_head.weight", (v, d)),
          ("odd.vec", (33,)), ("odd.scalar", ())]
    return [TensorSpec(n, 0, "f16", s) for n, s in t]


def opt(d: int, layers: int, ffn: int, vocab: int = 50272, pos: int = 2050,
        device: int = 0) -> List[TensorSpec]:
    """HF ``OPTForCausalLM`` state dict (lm_head tied to embed_tokens, so absent)."""
    t = [("model.decoder.embed_tokens.weight", (vocab, d)),
         ("model.decoder.embed_positions.weight", (pos, d)),
         ("model.decoder.final_layer_norm.weight", (d,)),
         ("model.decoder.final_layer_norm.bias", (d,))]
    for i in range(layers):
        pre = f"model.decoder.layers.{i}."
        for proj in ("k_proj", "v_proj", "q_proj", "out_proj"):
            t += [(pre + f"self_attn.{proj}.weight", (d, d)), (pre + f"self_attn.{proj}.bias", (d,))]
        t += [(pre + "self_attn_layer_norm.weight", (d,)), (pre + "self_attn_layer_norm.bias", (d,)),
              (pre + "fc1.weight", (ffn, d)), (pre + "fc1.bias", (ffn,)),
              (pre + "fc2.weight", (d, ffn)), (pre + "fc2.bias", (d,)),
              (pre + "final_layer_norm.weight", (d,)), (pre + "final_layer_norm.bias", (d,))]
    return [TensorSpec(n, device, "f16", s) for n, s in t]


def llama2(d: int, layers: int, ffn: int, kv: int, vocab: int = 32000, tp: int = 1) -> List[TensorSpec]:
    """HF ``LlamaForCausalLM`` state dict, sharded ``tp`` ways (see module doc)."""
    def shard(shape, dim):
        s = list(shape)
        assert s[dim] % tp == 0, (shape, dim, tp)
        s[dim] //= tp
        return tuple(s)

    full = [("model.embed_tokens.weight", (vocab, d), 0)]
    for i in range(layers):
        pre = f"model.layers.{i}."
        full += [(pre + "self_attn.q_proj.weight", (d, d), 0), (pre + "self_attn.k_proj.weight", (kv, d), 0),
                 (pre + "self_attn.v_proj.weight", (kv, d), 0), (pre + "self_attn.o_proj.weight", (d, d), 1),
                 (pre + "mlp.gate_proj.weight", (ffn, d), 0), (pre + "mlp.up_proj.weight", (ffn, d), 0),
                 (pre + "mlp.down_proj.weight", (d, ffn), 1),
                 (pre + "input_layernorm.weight", (d,), None),
                 (pre + "post_attention_layernorm.weight", (d,), None)]
    full += [("model.norm.weight", (d,), None), ("lm_head.weight", (vocab, d), 0)]
    out = []
    for r in range(tp):
        for n, s, dim in full:
            name = n if tp == 1 else f"{n}@{r}"
            out.append(TensorSpec(name, r, "f16", s if dim is None else shard(s, dim)))
    return out


def lora(base_d: int, layers: int, ffn: int, kv: int, rank: int = 32) -> List[TensorSpec]:
    """PEFT-style LoRA adapter on all 7 projections (paper P:1254)."""
    out = []
    for i in range(layers):
        pre = f"base_model.model.model.layers.{i}."
        for mod, (o, k) in (("self_attn.q_proj", (base_d, base_d)), ("self_attn.k_proj", (kv, base_d)),
                            ("self_attn.v_proj", (kv, base_d)), ("self_attn.o_proj", (base_d, base_d)),
                            ("mlp.gate_proj", (ffn, base_d)), ("mlp.up_proj", (ffn, base_d)),
                            ("mlp.down_proj", (base_d, ffn))):
            out.append(TensorSpec(pre + mod + ".lora_A.weight", 0, "f16", (rank, k)))
            out.append(TensorSpec(pre + mod + ".lora_B.weight", 0, "f16", (o, rank)))
    return out


# BASELINE.json configs -> (inventory builder, seed, description).  Seeds per SURVEY §8(d) D1.
CONFIGS = {
    "toy": (toy, 0, "toy 2-layer fp16 (22 tensors) -> 1 partition"),
    "opt-6.7b": (lambda: opt(4096, 32, 16384), 1, "OPT-6.7B-shaped fp16, 1 partition"),
    "llama2-13b-tp2": (lambda: llama2(5120, 40, 13824, 5120, tp=2), 2, "LLaMA-2-13B-shaped fp16, TP2"),
    "llama2-70b": (lambda: llama2(8192, 80, 28672, 1024, tp=1), 3, "LLaMA-2-70B-shaped fp16, 1 partition (TP1)"),
    "llama2-70b-tp8": (lambda: llama2(8192, 80, 28672, 1024, tp=8), 3, "LLaMA-2-70B-shaped fp16, TP8"),
    "llama2-70b-tp4": (lambda: llama2(8192, 80, 28672, 1024, tp=4), 3, "LLaMA-2-70B-shaped fp16, TP4"),
    "llama2-70b-tp2": (lambda: llama2(8192, 80, 28672, 1024, tp=2), 3, "LLaMA-2-70B-shaped fp16, TP2"),
    "opt-30b": (lambda: opt(7168, 48, 28672), 4, "OPT-30B-shaped fp16, 1 replicated partition"),
    "lora-70b-r32": (lambda: lora(8192, 80, 28672, 1024, 32), 5, "rank-32 LoRA adapter of LLaMA-2-70B"),
}


def model_inventory(config: str) -> Tuple[List[TensorSpec], int]:
    build, seed, _ = CONFIGS[config]
    return build(), seed


def random_inventory(rng: np.random.Generator, n_tensors: int, n_devices: int,
                     max_total: int, dtypes: Sequence[str] = tuple(DTYPES)) -> List[TensorSpec]:
    """Random checkpoint for the SPEC acceptance-1 style sweep: mixed dtypes,
    ranks 0..4 (rank 0 = scalar), sizes from a few bytes to ~max_total/n_tensors*8,
    devices drawn from a possibly sparse id set (Q15)."""
    dev_ids = sorted(rng.choice(np.arange(0, max(2 * n_devices, 1)), size=n_devices, replace=False).tolist())
    budget = max_total
    out = []
    for e in range(n_tensors):
        dt = dtypes[int(rng.integers(len(dtypes)))]
        w = DTYPE_WIDTH[dt]
        ndim = int(rng.integers(0, 5))
        cap = max(1, min(budget // w, max(1, 8 * max_total // max(n_tensors, 1) // w)))
        # log-uniform element count so tiny and large tensors both appear
        numel = int(math.exp(rng.uniform(0, math.log(cap)))) if cap > 1 else 1
        numel = max(1, min(numel, cap))
        if ndim == 0:
            shape: Tuple[int, ...] = ()
            numel = 1
        else:
            dims = [1] * ndim
            rem = numel
            for k in range(ndim - 1):
                f = int(rng.integers(1, 4))
                if rem % f == 0 and rem > 1:
                    dims[k] = f
                    rem //= f
            dims[-1] = rem
            shape = tuple(dims)
            numel = math.prod(shape)
        budget -= numel * w
        out.append(TensorSpec(f"t{e}.{dt}", int(rng.choice(dev_ids)), dt, shape))
        if budget <= 0:
            break
    return out
