"""Host<->device copy bandwidth on the box: H2D, D2H, and both directions concurrently (pinned)."""
import json
import torch

N = 134 * 1024 * 1024 // 8
h1 = torch.empty(N, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(N, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(N, dtype=torch.float64, device="cuda")
d2 = torch.empty(N, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
B = N * 8


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


res = {"h2d_GBs": B / t(lambda: d1.copy_(h1, non_blocking=True)) / 1e9,
       "d2h_GBs": B / t(lambda: h2.copy_(d2, non_blocking=True)) / 1e9,
       "both_GBs_each": B / t(both) / 1e9}
print(json.dumps(res))
