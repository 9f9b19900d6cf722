"""Synthetic checkpoint layouts for the BASELINE.json configs and their synthetic
values, generated on the GPU by the counter-hash kernel `rlk_synth_normal`.

Values: base ~ N(0, 0.02^2) rounded to the dtype; expert_i = base + N(0, (sigma_i * 1e-3)^2) with
sigma_i = i + 1, so task-vector norms differ and normalisation matters.  Each tensor t draws from
seeds derived from (seed, t, stream), indexed by the flat element index, so any slice of a tensor has
the same values whichever rank generates it.
"""
from __future__ import annotations

from collections import OrderedDict

import torch

from . import _lib as L
from .core import mix64


def mlp_10m() -> "OrderedDict[str, tuple]":
    """Config 1: toy MLP state dict, 9,966,592 params (fp32)."""
    return OrderedDict([("embed", (1536, 1024)), ("fc1.w", (4096, 1024)), ("fc1.b", (4096,)),
                        ("fc2.w", (1024, 4096)), ("fc2.b", (1024,))])


def gpt_1p3b() -> "OrderedDict[str, tuple]":
    """Config 2: GPT-style 1.3B (24 layers, d 2048, ffn 8192, vocab 50304): 292 tensors, 1.316e9 params."""
    d, f, v, n = 2048, 8192, 50304, 24
    out = OrderedDict([("wte", (v, d)), ("wpe", (2048, d))])
    for i in range(n):
        p = f"h.{i}."
        out.update([(p + "ln_1.w", (d,)), (p + "ln_1.b", (d,)), (p + "attn.c_attn.w", (d, 3 * d)),
                    (p + "attn.c_attn.b", (3 * d,)), (p + "attn.c_proj.w", (d, d)), (p + "attn.c_proj.b", (d,)),
                    (p + "ln_2.w", (d,)), (p + "ln_2.b", (d,)), (p + "mlp.c_fc.w", (d, f)), (p + "mlp.c_fc.b", (f,)),
                    (p + "mlp.c_proj.w", (f, d)), (p + "mlp.c_proj.b", (d,))])
    out.update([("ln_f.w", (d,)), ("ln_f.b", (d,))])
    return out


def llama3_8b() -> "OrderedDict[str, tuple]":
    """Config 3: Llama-3-8B-shaped (32 layers, d 4096, GQA kv 1024, ffn 14336, vocab 128256):
    291 tensors, 8,030,261,248 params."""
    d, kv, f, v, n = 4096, 1024, 14336, 128256, 32
    out = OrderedDict([("model.embed_tokens.weight", (v, d))])
    for i in range(n):
        p = f"model.layers.{i}."
        out.update([(p + "self_attn.q_proj.weight", (d, d)), (p + "self_attn.k_proj.weight", (kv, d)),
                    (p + "self_attn.v_proj.weight", (kv, d)), (p + "self_attn.o_proj.weight", (d, d)),
                    (p + "mlp.gate_proj.weight", (f, d)), (p + "mlp.up_proj.weight", (f, d)),
                    (p + "mlp.down_proj.weight", (d, f)), (p + "input_layernorm.weight", (d,)),
                    (p + "post_attention_layernorm.weight", (d,))])
    out.update([("model.norm.weight", (d,)), ("lm_head.weight", (v, d))])
    return out


def longcat_560b(n_layers: int = 28) -> "OrderedDict[str, tuple]":
    """Config 4: LongCat-Flash-560B-MoE-shaped (shapes not published, this layout is
    an assumption): 28 layers x 512 experts x (gate, up: 2048x6144; down: 6144x2048) stored per expert
    matrix, + attention 4 x 6144^2, router 6144x512, norms, and 131072 x 6144 embeddings / head.
    ~5.5e11 params in ~43k tensors."""
    d, f, e, v = 6144, 2048, 512, 131072
    out = OrderedDict([("model.embed_tokens.weight", (v, d))])
    for i in range(n_layers):
        p = f"model.layers.{i}."
        out.update([(p + "input_layernorm.weight", (d,)), (p + "post_attention_layernorm.weight", (d,))])
        for m in ("q_proj", "k_proj", "v_proj", "o_proj"):
            out[p + f"self_attn.{m}.weight"] = (d, d)
        out[p + "mlp.router.weight"] = (e, d)
        for x in range(e):
            q = p + f"mlp.experts.{x}."
            out.update([(q + "gate_proj.weight", (f, d)), (q + "up_proj.weight", (f, d)), (q + "down_proj.weight", (d, f))])
    out.update([("model.norm.weight", (d,)), ("lm_head.weight", (v, d))])
    return out


LAYOUTS = {"mlp10m": mlp_10m, "gpt1p3b": gpt_1p3b, "llama8b": llama3_8b, "longcat560b": longcat_560b}


def numel(shape) -> int:
    n = 1
    for s in shape:
        n *= int(s)
    return n


def stream_seed(seed: int, tensor: int, stream: int) -> int:
    return mix64(mix64(seed * 1000003 + tensor) ^ (stream + 1))


def fill_synthetic(base: torch.Tensor, experts: list[torch.Tensor], tensor: int, j0: int = 0, seed: int = 0,
                   base_std: float = 0.02, expert_std: float = 1e-3, stream=None) -> None:
    """Fill a slice [j0, j0 + n) of tensor `tensor`: base then each expert = base + noise (on device)."""
    s = L.stream_handle(stream)
    dt = L.dtype_code(base.dtype)
    n = base.numel()
    L.call("rlk_synth_normal", L.ptr(base), dt, n, j0, stream_seed(seed, tensor, 0), base_std, None, s)
    for i, e in enumerate(experts):
        L.call("rlk_synth_normal", L.ptr(e), dt, n, j0, stream_seed(seed, tensor, i + 1), expert_std * (i + 1),
               L.ptr(base), s)
