import os, sys, time, torch, json
def bw(n=64<<20, reps=10):
    h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device='cuda')
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    def t(fn):
        torch.cuda.synchronize(); a=time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter()-a
    h2d = t(lambda: [d.copy_(h, non_blocking=True) for _ in range(reps)])
    d2h = t(lambda: [h2.copy_(d2, non_blocking=True) for _ in range(reps)])
    def both():
        with torch.cuda.stream(s1):
            for _ in range(reps): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            for _ in range(reps): h2.copy_(d2, non_blocking=True)
    bo = t(both)
    return {"h2d_GBps": n*reps/h2d/1e9, "d2h_GBps": n*reps/d2h/1e9, "both_total_GBps": 2*n*reps/bo/1e9}
print("affinity", sorted(os.sched_getaffinity(0))[:4], "...", len(os.sched_getaffinity(0)), json.dumps(bw()))
