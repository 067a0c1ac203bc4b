"""HBM throughput vs read:write mix on this GPU (torch kernels, CUDA events): pure write (fill),
copy (1:1), 1:4 read:write (broadcast one source into 4 outputs), 4:1 (sum of 4 sources)."""
import torch
n = 256 * 1024 * 1024   # bf16 elements per buffer (512 MB)
a = [torch.randn(n, device="cuda", dtype=torch.bfloat16) for _ in range(4)]
o = [torch.empty(n, device="cuda", dtype=torch.bfloat16) for _ in range(4)]

def t(f, by, reps=10):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return by / ms / 1e6
B = 2 * n
print("fill (write only)      %.0f GB/s" % t(lambda: o[0].fill_(1.0), B))
print("copy 1:1               %.0f GB/s" % t(lambda: o[0].copy_(a[0]), 2 * B))
print("1 read : 4 writes      %.0f GB/s" % t(lambda: [x.copy_(a[0]) for x in o], 5 * B))
out = o[0]
print("4 reads : 1 write      %.0f GB/s" % t(lambda: torch.add(torch.add(a[0], a[1]), torch.add(a[2], a[3]), out=out), 7 * B))
