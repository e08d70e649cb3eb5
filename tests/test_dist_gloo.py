"""Host-side logic of the one-process-per-GPU path on CPU (gloo, world 2):
every rank plans independently and gets the identical plan; the push and
pull work partitions over ranks cover each delivered byte exactly once."""
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
    from paper_2406_14088_b200.runtime import hosted_devices

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


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_agree_and_partition_covers_plan(tmp_path, world):
    mp.spawn(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        res = json.load(open(tmp_path / f"rank{r}.json"))
        for key, v in res.items():
            assert v["same_plan"], key
            assert v["hier_saves"], key
            for k in ("00", "01", "10", "11"):
                # every destination byte is stored exactly once across ranks and phases
                assert v[f"written_{k}"] == v["total"], (key, k)
                assert v[f"wire_in_{k}"] == v[f"wire_out_{k}"], (key, k)


def test_hosted_devices_blocks():
    from paper_2406_14088_b200.runtime import hosted_devices
    assert hosted_devices(8, 0, 2) == [0, 1, 2, 3]
    assert hosted_devices(8, 3, 4) == [6, 7]
    with pytest.raises(ValueError):
        hosted_devices(8, 0, 3)
