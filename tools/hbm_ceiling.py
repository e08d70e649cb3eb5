"""HBM ceilings on this B200 for the traffic mixes the reallocation kernels
generate (plumbing-only microbenchmark; torch kernels, CUDA events):
pure write (fill), pure read (sum), 1:1 copy, and our own TMA broadcast of
one source into 8 destinations (1:8 read:write, the 7B train->gen mix)."""
import json
import sys

import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    gb = 1e9
    n = 32 * 2**30  # 64 GiB of bf16
    a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    b = torch.empty(n // 4, dtype=torch.bfloat16, device="cuda")
    out = {}
    ms = timed(lambda: a.fill_(1.0))
    out["write_only_gbs"] = a.numel() * 2 / (ms * 1e-3) / gb
    ms = timed(lambda: a.zero_())
    out["write_only_zero_gbs"] = a.numel() * 2 / (ms * 1e-3) / gb
    sys.path.insert(0, ".")
    from paper_2406_14088_b200 import runtime as R
    buf = R.DeviceBuffer(0, 64 * 2**30)
    st = torch.cuda.current_stream().cuda_stream
    ms = timed(lambda: R.check(R.lib.rr_memset(buf.ptr, 0, buf.nbytes, st)))
    out["write_only_cudaMemset_gbs"] = buf.nbytes / (ms * 1e-3) / gb
    ms = timed(lambda: R.check(R.lib.rr_memset(buf.ptr, 0x3c, buf.nbytes, st)))
    out["write_only_cudaMemset_nonzero_gbs"] = buf.nbytes / (ms * 1e-3) / gb
    buf.free()
    ms = timed(lambda: a.sum(dtype=torch.float32))
    out["read_only_gbs"] = a.numel() * 2 / (ms * 1e-3) / gb
    ms = timed(lambda: a[: b.numel()].copy_(b))
    out["copy_rw_gbs"] = 2 * b.numel() * 2 / (ms * 1e-3) / gb
    # 1:8 broadcast with torch copies (8 separate copy kernels) for reference
    src = b[: b.numel() // 8]
    dsts = [a[i * src.numel():(i + 1) * src.numel()] for i in range(8)]
    ms = timed(lambda: [d.copy_(src) for d in dsts])
    out["torch_8_copies_rw_gbs"] = 16 * src.numel() * 2 / (ms * 1e-3) / gb
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    sys.exit(main())
