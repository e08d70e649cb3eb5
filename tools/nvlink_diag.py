"""Which NVLink counters does this box expose (NVML field values, nvidia-smi)?"""
import subprocess

import pynvml as N

N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
for name in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX",
             "NVML_FI_DEV_NVLINK_LINK_COUNT", "NVML_FI_DEV_NVLINK_GET_SPEED"):
    fid = getattr(N, name, None)
    if fid is None:
        print(name, "absent")
        continue
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = N.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(name, scope, "ret", v.nvmlReturn, "val", v.value.ullVal)
        except Exception as e:
            print(name, scope, "exc", e)
for cmd in (["nvidia-smi", "nvlink", "-s", "-i", "0"], ["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"]):
    r = subprocess.run(cmd, capture_output=True, text=True)
    print(" ".join(cmd), "rc", r.returncode)
    print(r.stdout[:1500], r.stderr[:300])
