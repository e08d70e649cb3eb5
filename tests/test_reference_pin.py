"""Pin the product's rlplan vocabulary and the CPU oracle to the reference.

reference_outputs.json holds outputs of the reference's own C++
(proj/src/model_arith.cpp + cluster.cpp compiled as-is, oracle/Makefile);
when oracle/_ref is built (this container) the live reference is compared
too. spec_examples.json holds the SPEC/PAPER known answers."""
from __future__ import annotations

import json
import math
import os

import pytest

from oracle import oracle as O
from paper_2406_14088_b200 import rlplan as P

HERE = os.path.dirname(os.path.abspath(__file__))
REF = json.load(open(os.path.join(HERE, "golden", "reference_outputs.json")))
SPEC = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))


def model(name: str) -> P.ModelSpec:
    h, i, L, heads, kv, vocab, maxpos, head = REF["models"][name]["spec"]
    return P.ModelSpec(name="ref", hidden_size=h, intermediate_size=i, num_layers=L, num_attention_heads=heads,
                       num_kv_heads=kv, vocab_size=vocab, max_position_embeddings=maxpos, has_output_head=head)


def cluster(key: str) -> P.ClusterSpec:
    n, g = map(int, key.split("x"))
    return P.ClusterSpec(n_nodes=n, gpus_per_node=g, mem_per_device=1, intra_node_bw=900e9, inter_node_bw=50e9,
                         host_to_device_bw=55e9)


@pytest.mark.parametrize("name", sorted(REF["models"]))
def test_model_arith_matches_reference(name):
    e = REF["models"][name]
    m = model(name)
    if e["error"]:
        with pytest.raises(P.ValidationError) as ex:
            P.param_count(m, True)
        assert str(ex.value) == e["error"]
        return
    assert P.param_count(m, True) == e["param_count_true"]
    assert P.param_count(m, False) == e["param_count_false"]
    assert list(P.static_param_bytes(m)) == e["static_param_bytes"]
    assert P.flops(m, P.Phase.Forward, 1, 1) == e["flops_fwd_1_1"]
    assert P.flops(m, P.Phase.Backward, 512, 2048) == e["flops_bwd_512_2048"]
    assert P.kv_cache_bytes(m, 512, 2048) == e["kv_cache_bytes_512_2048"]
    # the oracle's independent shape-summation restatement agrees too
    assert O.param_count(m, True) == e["param_count_true"]
    assert O.param_count(m, False) == e["param_count_false"]


def test_logits_bytes_matches_reference():
    for k, v in REF["logits_bytes"].items():
        assert P.logits_bytes(*map(int, k.split(","))) == v


@pytest.mark.parametrize("key", sorted(REF["clusters"]))
def test_cluster_topology_matches_reference(key):
    c = cluster(key)
    e = REF["clusters"][key]
    meshes = P.enumerate_meshes(c)
    assert [[m.node_offset, m.node_count, m.gpu_offset, m.gpu_count] for m in meshes] == e["meshes"]
    assert [m.devices(c) for m in meshes] == e["devices"]
    assert [P.mesh_to_string(m, c) for m in meshes] == e["strings"]
    assert [P.mesh_from_string(s, c) for s in e["strings"]] == meshes
    for i, a in enumerate(meshes[:10]):
        for j, b in enumerate(meshes[:10]):
            assert int(P.overlap(a, b, c)) == e["overlap_first_10"][i][j]
    n = c.device_count()
    for a in range(n):
        for b in range(n):
            assert P.link_bandwidth(c, a, b) == e["bandwidth"][a][b]
    with pytest.raises(P.ValidationError, match="device index out of range"):
        P.link_bandwidth(c, 0, n)


def test_mesh_strings_and_errors_match_reference():
    c = cluster("2x8")
    for text, want in REF["mesh_strings"].items():
        m = P.mesh_from_string(text, c)
        assert [m.node_offset, m.node_count, m.gpu_offset, m.gpu_count] == want
    for text, err in REF["bad_mesh_strings"].items():
        with pytest.raises(P.ValidationError) as ex:
            P.mesh_from_string(text, c)
        assert str(ex.value) == err
    for mesh, err in REF["validate_mesh"]:
        m = P.DeviceMesh(*mesh)
        if err is None:
            P.validate_mesh(m, c)
        else:
            with pytest.raises(P.ValidationError) as ex:
                P.validate_mesh(m, c)
            assert str(ex.value) == err


def test_spec_and_paper_known_answers():
    for e in SPEC["param_count"]:
        assert P.param_count(P.MODELS[e["model"]], e["include"]) == e["value"], e["cite"]
    assert P.param_count(P.MODELS["spec_tiny"], True) == SPEC["spec_tiny_param_count"]["value"]
    assert O.param_count(P.MODELS["spec_tiny"], True) == SPEC["spec_tiny_param_count"]["value"]
    k = SPEC["kv_cache_bytes"]
    assert P.kv_cache_bytes(P.MODELS[k["model"]], k["batch"], k["seq_len"]) == k["value"]
    for e in SPEC["logits_bytes"]:
        assert P.logits_bytes(*e["args"]) == e["value"]
    assert P.static_param_bytes(P.MODELS["llama7b"])[0] == SPEC["static_param_bytes"]["params"]
    for e in SPEC["enumerate_meshes"]:
        c = P.ClusterSpec(e["n_nodes"], e["gpus_per_node"], 1, 1.0, 1.0, 1.0)
        assert len(P.enumerate_meshes(c)) == e["count"]
    for e in SPEC["stage_layer_map"]:
        assert [list(s) for s in P.stage_layer_map(e["layers"], e["pp"])] == e["stages"]
        assert [list(s) for s in O.stage_layer_map(e["layers"], e["pp"])] == e["stages"]


def test_local_bandwidth_sentinel():
    assert math.isinf(P.local_bandwidth())
    c = P.b200_cluster(8)
    assert math.isinf(P.link_bandwidth(c, 3, 3))


@pytest.mark.skipif(not O.Reference.available(), reason="oracle/_ref not built (reference tree absent)")
def test_live_reference_agrees_with_fixture():
    """The committed fixture is what the reference produces now."""
    R = O.Reference()
    for name, e in REF["models"].items():
        h, i, L, heads, kv, vocab, maxpos, head = e["spec"]
        m = P.ModelSpec(name="ref", hidden_size=h, intermediate_size=i, num_layers=L, num_attention_heads=heads,
                        num_kv_heads=kv, vocab_size=vocab, max_position_embeddings=maxpos, has_output_head=head)
        assert R.param_count(m, True) == e["param_count_true"]
    assert len(R.enumerate_meshes(8, 8)) == len(REF["clusters"]["8x8"]["meshes"])
