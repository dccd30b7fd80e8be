#!/usr/bin/env python
"""What a read-dominated stream achieves on this B200: torch reductions over
multi-GiB bf16 tensors (read-only) vs copy (read+write), CUDA events."""
import json, torch
dev = torch.device("cuda:0")
n = 4 << 30  # 4 Gi elements = 8 GiB bf16
x = torch.empty(n, dtype=torch.bfloat16, device=dev).normal_()
y = torch.empty_like(x)
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best
res = {}
res["sum_read_GBps"] = n * 2 / t(lambda: x.sum(dtype=torch.float32)) / 1e9
res["amax_read_GBps"] = n * 2 / t(lambda: x.abs().amax()) / 1e9 if False else None
res["copy_rw_GBps"] = 2 * n * 2 / t(lambda: y.copy_(x)) / 1e9
v = x.view(-1, 4096)
res["rowsum_read_GBps"] = n * 2 / t(lambda: v.sum(dim=1, dtype=torch.float32)) / 1e9
print(json.dumps(res))
