"""augment over the B200 planner and cost model: the SPEC
examples, an independent edge-scan oracle on random plans, and the node
durations (SPEC estimate beside the measured B200 model)."""
from __future__ import annotations

import random

import pytest

from _helpers import placement, random_placement
from paper_2406_14088_b200 import costmodel
from paper_2406_14088_b200 import rlplan as P
from paper_2406_14088_b200.augment import Call, DataEdge, augment, total_seconds

C = P.b200_cluster(8)
MODELS = {"actor": P.MODELS["llama7b"], "critic": P.MODELS["llama34b_critic"], "ref": P.MODELS["llama7b"],
          "reward": P.MODELS["llama34b_critic"]}


def ppo(gen, train, critic=None, offload_ref=False):
    """One PPO iteration: ActorGen -> {RewardInf, RefInf,
    CriticInf} -> {ActorTrain, CriticTrain}."""
    critic = critic or train
    calls = [Call("ActorGen", "actor", gen), Call("RewardInf", "reward", critic),
             Call("RefInf", "ref", train, offload=offload_ref), Call("CriticInf", "critic", critic),
             Call("ActorTrain", "actor", train), Call("CriticTrain", "critic", critic)]
    d = 16 << 20
    edges = [DataEdge("ActorGen", x, d) for x in ("RewardInf", "RefInf", "CriticInf", "ActorTrain", "CriticTrain")]
    edges += [DataEdge(x, y, d) for x in ("RewardInf", "RefInf", "CriticInf") for y in ("ActorTrain", "CriticTrain")]
    return calls, edges


def test_one_placement_for_everything_inserts_nothing():
    """SPEC.md:425 [TRIVIAL]: all calls share one (mesh, strategy)."""
    pl = placement(8, 1, 1, 8)
    calls, edges = ppo(pl, pl)
    assert augment(calls, edges, MODELS, C) == []
    # n_microbatches does not change who holds which bytes
    pl2 = P.Placement(pl.mesh, P.ParallelStrategy(dp=1, tp=8, pp=1, n_microbatches=4))
    assert augment(ppo(pl, pl2)[0], [], MODELS, C) == []


def test_actor_gen_and_train_on_different_layouts():
    """actor generation on one layout and training on another ->
    one actor param_realloc per direction (train -> gen across the
    iteration boundary), priced by the planner and both cost models."""
    gen, train = placement(8, 1, 8, 1), placement(8, 1, 1, 8)
    calls, edges = ppo(gen, train)
    nodes = augment(calls, edges, MODELS, C)
    actor = [n for n in nodes if n.kind == "param_realloc"]
    assert sorted(n.between for n in actor) == [("ActorGen", "ActorTrain"), ("ActorTrain", "ActorGen")]
    fwd = next(n for n in actor if n.between == ("ActorTrain", "ActorGen"))
    assert fwd.spec_seconds == fwd.plan.est_time
    assert fwd.b200_seconds == pytest.approx(costmodel.estimate_seconds(fwd.plan)["seconds"])
    # tp8 -> dp8 all-gather: SPEC's bytes/bandwidth misses the ingress of every destination
    assert fwd.b200_seconds > 5 * fwd.spec_seconds
    # ActorGen's output goes to calls on the training layout: data transfers
    data = [n for n in nodes if n.kind == "data_transfer"]
    assert {n.between for n in data} == {("ActorGen", x) for x in
                                         ("RewardInf", "RefInf", "CriticInf", "ActorTrain", "CriticTrain")}
    assert total_seconds(nodes)["b200_seconds"] > 0


def test_offload_flag_parks_and_restores_parameters():
    """offload/onload nodes per offload flag, duration = param
    bytes / host_to_device_bw; B200: per-GPU shard over its own host link."""
    pl = placement(8, 1, 1, 8)
    calls, edges = ppo(pl, pl, offload_ref=True)
    nodes = augment(calls, edges, MODELS, C)
    assert [n.kind for n in nodes] == ["offload", "onload"]
    off = nodes[0]
    shard = P.MODELS["llama7b"]
    per_gpu = max(P.plan_param_realloc(shard, pl, pl, C).shard_bytes(0, d) for d in range(8))
    assert off.bytes == per_gpu
    assert off.spec_seconds == pytest.approx(per_gpu / C.host_to_device_bw)
    assert off.b200_seconds == pytest.approx(per_gpu / 55.6e9)


def _edge_scan(calls, edges, cyclic=True):
    """Independent count (SPEC.md:427 edge-scan oracle): for each model,
    adjacent calls (cyclically) whose grids or layouts differ, plus offload
    pairs, plus data edges between differing grids."""
    def key(p):
        return (p.mesh.gpu_offset, p.mesh.gpu_count, p.strategy.dp, p.strategy.tp, p.strategy.pp)
    n = 0
    models = []
    for c in calls:
        if c.model not in models:
            models.append(c.model)
    for m in models:
        seq = [c for c in calls if c.model == m]
        for i, a in enumerate(seq):
            if i + 1 == len(seq) and not cyclic:
                break
            b = seq[(i + 1) % len(seq)]
            n += 2 if a.offload else 0
            if a is not b and (key(a.placement), a.placement.qkv_layout, a.placement.gate_up_layout) != \
                    (key(b.placement), b.placement.qkv_layout, b.placement.gate_up_layout):
                n += 1
    by = {c.name: c for c in calls}
    n += sum(1 for e in edges if key(by[e.producer].placement) != key(by[e.consumer].placement))
    return n


def test_inserted_node_count_matches_edge_scan_oracle_on_random_plans():
    rng = random.Random(428)
    tiny = {"actor": P.MODELS["tiny"], "critic": P.MODELS["tiny"], "ref": P.MODELS["tiny"],
            "reward": P.MODELS["tiny"]}
    for _ in range(60):
        names = ["ActorGen", "RewardInf", "RefInf", "CriticInf", "ActorTrain", "CriticTrain"]
        owners = ["actor", "reward", "ref", "critic", "actor", "critic"]
        calls = [Call(nm, mo, random_placement(rng, tiny[mo]), offload=rng.random() < 0.2)
                 for nm, mo in zip(names, owners)]
        # data bytes divisible by every lcm(dp) on <= 8 devices
        edges = [DataEdge(a, b, 1 << 16) for a, b in rng.sample(
            [(x, y) for i, x in enumerate(names) for y in names[i + 1:]], 5)]
        cyclic = rng.random() < 0.7
        nodes = augment(calls, edges, tiny, C, cyclic=cyclic)
        assert len(nodes) == _edge_scan(calls, edges, cyclic)
        assert all(n.b200_seconds >= 0 and n.spec_seconds >= 0 for n in nodes)
