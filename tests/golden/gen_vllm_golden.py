#!/usr/bin/env python
"""Regenerate the third-party fixtures in tests/golden/:

* vllm_tp_shards.json — an independent pin of the byte layout of
  tensor-parallel shards (DESIGN.md §3 G3/G4/G10), from vLLM; the Megatron
  grouped QKV layout is checked through vLLM's Falcon loader, which
  de-interleaves exactly that layout (falcon.py load_weights);
* hf_llama_inventory.json — the parameter inventory (names, [out, in]
  shapes, totals) of HF transformers' LlamaForCausalLM /
  LlamaForSequenceClassification (num_labels=1, the critic's scalar head) at
  the BASELINE shapes, built on the meta device.

The reference never materialises weights, so no
reference fixture pins which bytes a TP rank holds. This script takes a
third-party implementation of Megatron-style LLaMA tensor parallelism —
vLLM's weight loaders (vllm.model_executor.layers.linear.QKVParallelLinear,
MergedColumnParallelLinear, RowParallelLinear and
vocab_parallel_embedding.VocabParallelEmbedding / ParallelLMHead) — feeds them
the full logical tensors of a model (the weight function of DESIGN.md §4,
through the C oracle) and records, for every TP rank, the SHA-256 of each
parameter the loader produced. tests/test_thirdparty_layout_pin.py checks that the
shard of the same rank under a (pp1, dp1, tp) placement with the Concat
layouts ([Q_r; K_r; V_r] and [G_r; U_r]) holds exactly those bytes.

vLLM is library code in this image; it is imported only here (CPU, no GPU,
a fake TP group object), never by the product or the tests.

Usage: python tests/golden/gen_vllm_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

SEED = 11
# (name, hidden, ffn, layers, heads, kv_heads, vocab, tp degrees)
MODELS = [
    ("tiny", 256, 688, 4, 4, 2, 1024, (1, 2, 4)),  # tp4 > 2 KV heads: vLLM replicates them
    ("tiny_gqa4", 512, 1376, 2, 8, 4, 2048, (2, 4)),
]


def logical(tensor: int, rows: int, cols: int):
    """Full logical tensor `tensor` as bf16 (torch), values from the oracle."""
    import torch
    n = rows * cols
    vals = np.fromiter((O.value(SEED, tensor, i) for i in range(n)), dtype=np.uint16, count=n)
    return torch.from_numpy(vals.view(np.int16).copy()).view(torch.bfloat16).reshape(rows, cols)


def sha(t) -> str:
    import torch
    return hashlib.sha256(t.contiguous().view(torch.int16).numpy().tobytes()).hexdigest()


def falcon_deinterleave(fused, heads: int, kv: int):
    """[Q; K; V] from a Falcon / Megatron grouped fused QKV weight, computed
    by vLLM's own FalconModel.load_weights (vllm/model_executor/models/
    falcon.py) on a stub module that captures what it would load."""
    import torch.nn as nn
    from vllm.model_executor.models import falcon as F
    got = {}

    class Leaf(nn.Module):
        def __init__(self):
            super().__init__()
            self.weight = nn.Parameter(fused.new_zeros(fused.shape), requires_grad=False)
            self.weight.output_dim = 0
            self.weight.weight_loader = lambda p, w: got.__setitem__("w", w.clone())

    class Att(nn.Module):
        def __init__(self):
            super().__init__()
            self.query_key_value = Leaf()

    class Layer(nn.Module):
        def __init__(self):
            super().__init__()
            self.self_attention = Att()

    class Stub(nn.Module):
        def __init__(self):
            super().__init__()
            self.h = nn.ModuleList([Layer()])
            self.config = types.SimpleNamespace(num_attention_heads=heads, num_kv_heads=kv,
                                                new_decoder_architecture=True, multi_query=False)

    F.FalconModel.load_weights(Stub(), [("h.0.self_attention.query_key_value.weight", fused)])
    return got["w"]


def main() -> None:
    import torch
    import vllm
    import vllm.distributed.parallel_state as ps
    from vllm.model_executor.layers import linear as L
    from vllm.model_executor.layers import vocab_parallel_embedding as V

    out = {"generator": f"tests/golden/gen_vllm_golden.py with vllm {vllm.__version__}", "seed": SEED,
           "layout": "(pp1, dp1, tp) placement, qkv Concat [Q_r;K_r;V_r], gate_up Concat [G_r;U_r], KV heads replicated when tp > kv",
           "models": {}, "cases": []}
    for name, h, ffn, nl, heads, kv, vocab, tps in MODELS:
        hd = h // heads
        out["models"][name] = dict(hidden_size=h, intermediate_size=ffn, num_layers=nl, num_attention_heads=heads,
                                   num_kv_heads=kv, vocab_size=vocab)
        # canonical tensor ids (DESIGN.md §3 G12)
        full = {0: logical(0, vocab, h)}
        for l in range(nl):
            b = 1 + 9 * l
            shapes = [(1, h), (heads * hd, h), (kv * hd, h), (kv * hd, h), (h, heads * hd), (1, h), (ffn, h),
                      (ffn, h), (h, ffn)]
            for k, (r, c) in enumerate(shapes):
                full[b + k] = logical(b + k, r, c)
        full[1 + 9 * nl] = logical(1 + 9 * nl, 1, h)
        full[2 + 9 * nl] = logical(2 + 9 * nl, vocab, h)
        for tp in tps:
            for rank in range(tp):
                ps._TP = types.SimpleNamespace(rank_in_group=rank, world_size=tp)
                params = {}

                def put(pname, module, tensor_ids, loads):
                    for tid, shard_id in loads:
                        if shard_id is None:
                            module.weight_loader(module.weight, full[tid])
                        else:
                            module.weight_loader(module.weight, full[tid], shard_id)
                    params[pname] = {"tensors": tensor_ids, "shape": list(module.weight.shape),
                                     "sha256": sha(module.weight.data)}

                emb = V.VocabParallelEmbedding(vocab, h, params_dtype=torch.bfloat16)
                put("embed_tokens", emb, [0], [(0, None)])
                for l in range(nl):
                    b = 1 + 9 * l
                    params[f"layers.{l}.input_layernorm"] = {"tensors": [b], "shape": [h],
                                                             "sha256": sha(full[b].reshape(h))}
                    qkv = L.QKVParallelLinear(h, hd, heads, kv, bias=False, params_dtype=torch.bfloat16)
                    put(f"layers.{l}.qkv_proj", qkv, [b + 1, b + 2, b + 3], [(b + 1, "q"), (b + 2, "k"), (b + 3, "v")])
                    if kv % tp == 0:
                        # Megatron grouped layout of the same rank: per local KV
                        # group [its q heads; k; v]. The grouped tensor is the
                        # unique row permutation that vLLM's Falcon loader maps
                        # back onto vLLM's [Q_r; K_r; V_r]; checked here.
                        lq, lkv = heads // tp, kv // tp
                        cat = qkv.weight.data
                        q_r, k_r, v_r = cat[:lq * hd], cat[lq * hd:(lq + lkv) * hd], cat[(lq + lkv) * hd:]
                        grouped = torch.cat([q_r.reshape(lkv, lq // lkv, hd, h), k_r.reshape(lkv, 1, hd, h),
                                             v_r.reshape(lkv, 1, hd, h)], dim=1).reshape(-1, h)
                        assert torch.equal(falcon_deinterleave(grouped, lq, lkv).view(torch.int16),
                                           cat.view(torch.int16))
                        params[f"layers.{l}.qkv_proj_grouped"] = {
                            "tensors": [b + 1, b + 2, b + 3], "shape": list(grouped.shape), "sha256": sha(grouped),
                            "layout": "Megatron grouped (qkv_layout 2); verified with vLLM FalconModel.load_weights"}
                    o = L.RowParallelLinear(heads * hd, h, bias=False, params_dtype=torch.bfloat16)
                    put(f"layers.{l}.o_proj", o, [b + 4], [(b + 4, None)])
                    params[f"layers.{l}.post_attention_layernorm"] = {"tensors": [b + 5], "shape": [h],
                                                                      "sha256": sha(full[b + 5].reshape(h))}
                    gu = L.MergedColumnParallelLinear(h, [ffn, ffn], bias=False, params_dtype=torch.bfloat16)
                    put(f"layers.{l}.gate_up_proj", gu, [b + 6, b + 7], [(b + 6, 0), (b + 7, 1)])
                    dn = L.RowParallelLinear(ffn, h, bias=False, params_dtype=torch.bfloat16)
                    put(f"layers.{l}.down_proj", dn, [b + 8], [(b + 8, None)])
                params["norm"] = {"tensors": [1 + 9 * nl], "shape": [h], "sha256": sha(full[1 + 9 * nl].reshape(h))}
                head = V.ParallelLMHead(vocab, h, params_dtype=torch.bfloat16)
                put("lm_head", head, [2 + 9 * nl], [(2 + 9 * nl, None)])
                out["cases"].append({"model": name, "tp": tp, "rank": rank, "params": params})
                print(f"{name} tp{tp} rank{rank}: {len(params)} params", flush=True)
    ps._TP = None
    with open(os.path.join(HERE, "vllm_tp_shards.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


# (name, hidden, ffn, layers, heads, kv_heads, vocab, has_output_head) — PAPER.md:880-893
HF_MODELS = [
    ("llama7b", 4096, 14336, 32, 32, 8, 128256, True),
    ("llama13b", 5120, 13824, 40, 40, 40, 128256, True),
    ("llama34b_critic", 8192, 22016, 48, 64, 8, 128256, False),
    ("llama70b", 8192, 28672, 80, 64, 8, 128256, True),
    ("tiny", 256, 688, 4, 4, 2, 1024, True),
]


def gen_hf() -> None:
    import torch
    import transformers
    from transformers import LlamaConfig, LlamaForCausalLM, LlamaForSequenceClassification

    out = {"generator": f"tests/golden/gen_vllm_golden.py with transformers {transformers.__version__}",
           "models": {}}
    for name, h, ffn, nl, heads, kv, vocab, has_head in HF_MODELS:
        cfg = LlamaConfig(hidden_size=h, intermediate_size=ffn, num_hidden_layers=nl, num_attention_heads=heads,
                          num_key_value_heads=kv, vocab_size=vocab, tie_word_embeddings=False, num_labels=1)
        with torch.device("meta"):
            m = LlamaForCausalLM(cfg) if has_head else LlamaForSequenceClassification(cfg)
        params = [(n, list(p.shape)) for n, p in m.named_parameters()]
        out["models"][name] = {
            "dims": dict(hidden_size=h, intermediate_size=ffn, num_layers=nl, num_attention_heads=heads,
                         num_kv_heads=kv, vocab_size=vocab, has_output_head=has_head),
            "total_params": sum(p.numel() for p in m.parameters()),
            "non_layer": [x for x in params if ".layers." not in x[0]],
            "layer0": [x for x in params if ".layers.0." in x[0]],
            "layers": sum(1 for n, _ in params if n.endswith("input_layernorm.weight")),
        }
        print(f"hf {name}: {out['models'][name]['total_params']} params", flush=True)
    with open(os.path.join(HERE, "hf_llama_inventory.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    gen_hf()
    main()
