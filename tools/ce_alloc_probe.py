"""Copy engine into RankRealloc shard buffers vs fresh IPC buffers (diagnostics, 2 ranks):
found that cudaMalloc sizes that are not 2 MiB multiples slowed peer copy-engine writes
(551 vs 777 GB/s); rr_device_alloc now pads to whole 2 MiB pages."""
import os, sys, json, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, torch.distributed as dist
from paper_2406_14088_b200 import runtime as R
from paper_2406_14088_b200.rlplan import BALANCED
from paper_2406_14088_b200.workloads import WORKLOADS
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
w = WORKLOADS["llama13b_pp2tp4_to_dp2tp4"]
plan = w.plans(BALANCED)[0]
rr = R.RankRealloc([plan], {"a": (0, R.SRC), "b": (0, R.DST)}, [("a", "b")], rank, world, local)
ex = rr.executors[0]
stream = torch.cuda.current_stream()
host_of = [rr.owner[d] for d in range(8)]
runs = plan.ce_runs(rr.local, host_of)
out = {"runs": len(runs), "bytes": sum(u[4] for u in runs)}
def t(name, fn, nbytes, reps=4):
    best = 1e9
    for r in range(reps):
        torch.cuda.synchronize(); dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream); fn(); e.record(stream); torch.cuda.synchronize()
        if r: best = min(best, s.elapsed_time(e))
    out[name] = round(nbytes / (best * 1e6), 1)
tot = out["bytes"]
t("executor_launch", lambda: ex.launch(stream), tot)
t("memcpy_runs_direct", lambda: [R.memcpy_async(rr.ptrs["b"][d] + do, rr.ptrs["a"][s] + so, nb, 2, stream) for (s, d, so, do, nb) in runs], tot)
big = R.DeviceBuffer(local, 4 << 30)
hs = [None] * world
dist.all_gather_object(hs, big.ipc_handle())
rem = R.open_ipc(local, hs[rank ^ 1])
src0 = rr.ptrs["a"][runs[0][0]]
t("memcpy_src0_to_fresh_remote_3GB", lambda: R.memcpy_async(rem, src0, 3 << 30, 2, stream), 3 << 30)
d0 = rr.ptrs["b"][runs[0][1]]
mine = R.DeviceBuffer(local, 4 << 30)
t("memcpy_fresh_local_to_remote_dst0_3GB", lambda: R.memcpy_async(d0, mine.ptr, 3 << 30, 2, stream), 3 << 30)
t("memcpy_fresh_to_fresh_3GB", lambda: R.memcpy_async(rem, mine.ptr, 3 << 30, 2, stream), 3 << 30)
odd = R.DeviceBuffer(local, (3 << 30) + 256 * 12345)
hs2 = [None] * world
dist.all_gather_object(hs2, odd.ipc_handle())
rem2 = R.open_ipc(local, hs2[rank ^ 1])
t("memcpy_to_remote_oddsize_3GB", lambda: R.memcpy_async(rem2, mine.ptr, 3 << 30, 2, stream), 3 << 30)
if rank == 0:
    print(json.dumps(out), flush=True)
dist.barrier()
