#!/usr/bin/env python
"""Regenerate the golden fixtures in tests/golden/.

* reference_outputs.json — outputs of the REFERENCE's own C++
  (/root/reference/proj/src/model_arith.cpp + cluster.cpp, compiled as-is by
  oracle/Makefile into oracle/_ref/librlplan_ref.so) on the inputs the path
  uses: the Appendix-A models, the tiny specs, B200 cluster shapes, meshes,
  mesh strings and error messages. Needs /root/reference (run in the build
  container); the fixture travels, the reference does not.
* weights_kat.json — known-answer values of the weight function
   from the C oracle, pinning CPU == GPU bit patterns.

spec_examples.json is transcribed by hand from SPEC.md (line-cited) and is
not generated.

Usage: python tests/golden/gen_golden.py
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

MODELS = {
    # name: (hidden, ffn, layers, heads, kv, vocab, maxpos, has_head) — PAPER.md:880-893 + tiny specs
    "llama7b": (4096, 14336, 32, 32, 8, 128256, 8192, True),
    "llama13b": (5120, 13824, 40, 40, 40, 128256, 8192, True),
    "llama34b": (8192, 22016, 48, 64, 8, 128256, 8192, True),
    "llama34b_critic": (8192, 22016, 48, 64, 8, 128256, 8192, False),
    "llama70b": (8192, 28672, 80, 64, 8, 128256, 8192, True),
    "tiny": (256, 688, 4, 4, 2, 1024, 8192, True),
    "spec_tiny": (4, 8, 1, 2, 1, 10, 16, True),
    "bad_heads": (100, 8, 1, 3, 1, 10, 16, True),
    "bad_kv": (128, 8, 1, 4, 3, 10, 16, True),
    "zero_vocab": (128, 8, 1, 4, 1, 0, 16, True),
}


class M:
    def __init__(self, name, t):
        (self.hidden_size, self.intermediate_size, self.num_layers, self.num_attention_heads, self.num_kv_heads,
         self.vocab_size, self.max_position_embeddings, self.has_output_head) = t
        self.name, self.param_bytes, self.grad_bytes, self.optimizer_bytes_per_param = name, 2, 2, 12


def reference_outputs() -> dict:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from oracle.oracle import Reference
    if not Reference.available():
        raise SystemExit("oracle/_ref/librlplan_ref.so missing: /root/reference is needed to regenerate")
    R = Reference()
    out = {"source": "reference proj/src/model_arith.cpp + cluster.cpp compiled by oracle/Makefile",
           "models": {}, "clusters": {}, "mesh_strings": {}, "bad_mesh_strings": {}, "validate_mesh": []}
    for name, t in MODELS.items():
        m = M(name, t)
        entry = {"spec": list(t)}
        pc_t, pc_f = R.param_count(m, True), R.param_count(m, False)
        entry["param_count_true"] = pc_t
        entry["param_count_false"] = pc_f
        entry["error"] = R.error() if pc_t is None else None
        if pc_t is not None:
            entry["static_param_bytes"] = list(R.static_param_bytes(m))
            entry["flops_fwd_1_1"] = R.flops(m, False, 1, 1)
            entry["flops_bwd_512_2048"] = R.flops(m, True, 512, 2048)
            entry["kv_cache_bytes_512_2048"] = R.kv_cache_bytes(m, 512, 2048)
        out["models"][name] = entry
    out["logits_bytes"] = {"128000,512,2048,2": R.logits_bytes(128000, 512, 2048, 2),
                           "128256,512,2048,2": R.logits_bytes(128256, 512, 2048, 2)}
    for nodes, gpus in [(1, 1), (1, 2), (1, 4), (1, 8), (2, 8), (8, 8)]:
        meshes = R.enumerate_meshes(nodes, gpus)
        out["clusters"][f"{nodes}x{gpus}"] = {
            "meshes": meshes,
            "devices": [R.mesh_devices(nodes, gpus, m) for m in meshes],
            "strings": [R.mesh_to_string(nodes, gpus, m) for m in meshes],
            "overlap_first_10": [[int(R.overlap(nodes, gpus, a, b)) for b in meshes[:10]] for a in meshes[:10]],
            "bandwidth": [[R.link_bandwidth(nodes, gpus, a, b) for b in range(nodes * gpus)]
                          for a in range(nodes * gpus)],
        }
    for text in ["trainer01", "trainer01:gpu[0-3]", "trainer01:gpu5", "trainer[01-02]", "trainer02:gpu[4-7]"]:
        mesh, err = R.mesh_from_string(2, 8, text)
        out["mesh_strings"][text] = list(mesh) if mesh else err
    for text in ["trainer01:gpu[1-2]", "node01", "trainer01:gpu[0-3", "trainer01x", "trainer03", "trainer01:gpu[0-2]"]:
        mesh, err = R.mesh_from_string(2, 8, text)
        out["bad_mesh_strings"][text] = err
    for mesh in [(0, 1, 0, 8), (0, 1, 1, 2), (0, 2, 0, 4), (1, 1, 4, 4), (0, 1, 0, 3), (0, 3, 0, 8), (0, 1, 6, 4)]:
        out["validate_mesh"].append([list(mesh), R.validate_mesh(2, 8, mesh)])
    return out


def weights_kat() -> dict:
    from oracle import oracle as O
    cases = []
    for seed in (0, 1, 5, 2**63 + 7, O.SEED_SPECIAL | 3, O.SEED_SPECIAL | (2**63 + 9)):
        for tensor in (0, 1, 2, 100, 723):
            for idx in (0, 1, 255, 4096, 123456789, 2**39 - 1):
                cases.append([seed, tensor, idx, O.value(seed, tensor, idx)])
    return {"function": "splitmix64(seed ^ tensor<<40 ^ index) -> bf16 bits (DESIGN.md §3; seed bit 62: special values)",
            "cases": cases}


def main() -> None:
    with open(os.path.join(HERE, "reference_outputs.json"), "w") as f:
        json.dump(reference_outputs(), f, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "weights_kat.json"), "w") as f:
        json.dump(weights_kat(), f, indent=1)
    print("wrote reference_outputs.json, weights_kat.json")


if __name__ == "__main__":
    main()
