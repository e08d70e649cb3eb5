"""Host-side logic of the one-process-per-GPU path on CPU (gloo, world 2, 4
and 8 -- the 8-GPU box the pool cannot lend): every rank plans independently
and gets the identical plan and the identical policy inputs (link bottleneck
estimates, relay flag-array lengths); the push and pull work partitions over
ranks cover each delivered byte exactly once."""
from __future__ import annotations

import json
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from _helpers import config_placements
    from paper_2406_14088_b200.rlplan import BALANCED, plan_param_realloc
    from paper_2406_14088_b200.runtime import hosted_devices, link_bottleneck, relay_slots

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    result = {}
    for key in ("7b_tp8_to_dp8", "13b_pp2tp4_to_dp2tp4", "34b_pp4tp2_to_tp8_fused", "70b_pp2tp4_to_tp8"):
        m, src, dst, c = config_placements(key)
        plan = plan_param_realloc(m, src, dst, c, BALANCED)
        js = json.dumps(plan.to_json(), sort_keys=True)
        plans = [None] * world
        dist.all_gather_object(plans, js)
        n = c.device_count()
        local = hosted_devices(n, rank, world)
        host_of = [d // (n // world) for d in range(n)]
        work = {f"{mode}{h}": plan.work(local, mode, host_of if h else None) for mode in (0, 1) for h in (0, 1)}
        works = [None] * world
        dist.all_gather_object(works, work)
        total_written = plan.work(list(range(n)), 0)["written"]
        entry = {"same_plan": all(p == js for p in plans), "total": total_written}
        # RankRealloc's auto policies and relay buffers are sized from these;
        # a rank that disagreed would deadlock the flag protocol
        policy = [link_bottleneck(plan, host_of, mc, rl) for mc, rl in ((0, 0), (1, 0), (0, 1))]
        policy += [relay_slots(plan, host_of, 0, chain, star) for chain, star in ((1, 0), (0, 1), (1, 1))]
        policies = [None] * world
        dist.all_gather_object(policies, policy)
        entry["same_policy"] = all(q == policy for q in policies)
        entry["link_bottleneck"] = policy[0]
        for k in work:
            entry[f"written_{k}"] = sum(w[k]["written"] + w[k]["fanout_written"] for w in works)
            entry[f"wire_in_{k}"] = sum(w[k]["wire_in"] for w in works)
            entry[f"wire_out_{k}"] = sum(w[k]["wire_out"] for w in works)
        # hierarchical delivery never sends more over links than flat delivery
        entry["hier_saves"] = all(w["01"]["wire_in"] <= w["00"]["wire_in"] for w in works)
        result[key] = entry
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(result, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ranks_agree_and_partition_covers_plan(tmp_path, world):
    mp.spawn(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        res = json.load(open(tmp_path / f"rank{r}.json"))
        for key, v in res.items():
            assert v["same_plan"], key
            assert v["same_policy"], key
            assert v["hier_saves"], key
            for k in ("00", "01", "10", "11"):
                # every destination byte is stored exactly once across ranks and phases
                assert v[f"written_{k}"] == v["total"], (key, k)
                assert v[f"wire_in_{k}"] == v[f"wire_out_{k}"], (key, k)


def test_link_bottleneck_at_8_gpus():
    """7B tp8->dp8 with one plan device per GPU is ingress-bound: every GPU
    receives the 7 shards it does not hold (14,052,491,264 B)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _helpers import config_placements
    from paper_2406_14088_b200.rlplan import BALANCED, plan_param_realloc
    from paper_2406_14088_b200.runtime import link_bottleneck
    m, src, dst, c = config_placements("7b_tp8_to_dp8")
    plan = plan_param_realloc(m, src, dst, c, BALANCED)
    host_of = list(range(8))
    assert link_bottleneck(plan, host_of) == 14052491264
    # a relay chain cannot beat an all-gather's ingress bound
    assert link_bottleneck(plan, host_of, relay=True) == 14052491264


def test_hosted_devices_blocks():
    from paper_2406_14088_b200.runtime import hosted_devices, link_bottleneck, relay_slots
    assert hosted_devices(8, 0, 2) == [0, 1, 2, 3]
    assert hosted_devices(8, 3, 4) == [6, 7]
    with pytest.raises(ValueError):
        hosted_devices(8, 0, 3)
