#!/bin/bash
# One-off environment probe for the GPU box (host RAM, cores, P2P, multicast).
set -x
nproc; free -g; lscpu | head -20; nvidia-smi; nvidia-smi topo -m
python - <<'PY'
import torch, ctypes
n = torch.cuda.device_count(); print("devices", n)
for i in range(n):
    p = torch.cuda.get_device_properties(i); print(i, p.name, p.total_memory, p.multi_processor_count)
for i in range(n):
    for j in range(n):
        if i != j: print("p2p", i, j, torch.cuda.can_device_access_peer(i, j))
cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
for i in range(n):
    v = ctypes.c_int()
    # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
    cuda.cuDeviceGetAttribute(ctypes.byref(v), 132, i); print("multicast_supported", i, v.value)
PY
