"""Read-only HBM ceiling on this B200: torch reductions over 4 GiB (no kernel of ours)
plus a copy for reference.  Prints GB/s (best of N, CUDA events)."""
import json
import torch

x = torch.empty(2 * 1024**3, dtype=torch.bfloat16, device="cuda").normal_()
y = torch.empty_like(x)


def t(fn, bytes_, n=10):
    best = 1e9
    for _ in range(3):
        fn()
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return bytes_ / best / 1e9


res = {"sum_read_GBps": t(lambda: x.sum(dtype=torch.float32), x.numel() * 2),
       "amax_read_GBps": t(lambda: x.abs().amax() if False else torch.amax(x), x.numel() * 2),
       "copy_rw_GBps": t(lambda: y.copy_(x), x.numel() * 4)}
print(json.dumps(res))
