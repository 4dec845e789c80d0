"""evict_select alone on the `evict` config (2^20 keys, top-64k) and its straddle variant:
CUDA-event time per call (keys L2-resident from the previous call, as in the serving step),
phase timestamps of CTA 0, for a list of cooperative grid sizes (option evict_ctas; each size
in its own process).

usage: python profiles/evict_bench.py [ctas ...]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, %r)
import workloads as W, paper_2504_03651_b200 as K
K.set_option("evict_ctas", int(sys.argv[1]))
dev = torch.device("cuda", 0)
res = {}
for straddle in (False, True):
    ev = W.make_evict(straddle=straddle)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)
    keys = K.evict_keys(t(ev.state, np.uint8), t(ev.rc, np.int32), t(ev.lat, np.int32), t(ev.depth, np.int16))
    ws = torch.zeros(K.evict_select_workspace_size(len(ev.state), ev.k), dtype=torch.uint8, device=dev)
    ids = torch.empty(ev.k, dtype=torch.int32, device=dev)
    for _ in range(10):
        K.evict_select(keys, ev.k, out_ids=ids, workspace=ws, sync=False)
    torch.cuda.synchronize()
    times = []
    for _ in range(10):  # 20 back-to-back calls per event pair: host enqueue hidden
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            K.evict_select(keys, ev.k, out_ids=ids, workspace=ws, sync=False)
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) * 1e3 / 20)
    ts = ws[256:256 + 256].view(torch.int64).cpu().numpy()
    ctl = ws[256 + 256:256 + 256 + 4 * 50].view(torch.int32).cpu().numpy()
    pt = ws[768:768 + 32 * 512].view(torch.int64).view(-1, 4).cpu().numpy()
    t_end = None
    if pt[0, 3] > ts[0]:  # -DKVA_SEL_SPAN build: per-CTA large-bucket end / exit
        C = int((pt[:, 3] > ts[0]).sum())
        ex, le = (pt[:C, 3] - ts[0]) / 1e3, (pt[:C, 0] - ts[0]) / 1e3
        t_end = {"exit_max_us": round(float(ex.max()), 1), "exit_argmax": int(ex.argmax()),
                 "exit_p50_us": round(float(np.median(ex)), 1), "large_end_max_us": round(float(le.max()), 1),
                 "exit_top8": [(int(i), round(float(ex[i]), 1)) for i in np.argsort(-ex)[:8]]}
    ts = ts[ts > 0]
    times.sort()
    res["straddle" if straddle else "evict"] = {
        "us_median": times[len(times) // 2], "us_p10": times[len(times) // 10], "us_p90": times[9 * len(times) // 10],
        "phase_us": [round(float(x), 1) for x in np.diff(ts) / 1e3], "last_cta": t_end, "rounds": int(ctl[48]), "levels": int(ctl[49]),
        "records_small_large_big": [[int(ctl[l]), int(ctl[16 + l]), int(ctl[32 + l])] for l in range(int(ctl[49]) + 1)]}
# launch + teardown cost: a call with nothing evictable returns after phase 0 and one barrier
keys1 = torch.full((1 << 20,), -1, dtype=torch.int64, device=dev)
ws1 = torch.zeros(K.evict_select_workspace_size(1 << 20, 1), dtype=torch.uint8, device=dev)
ids1 = torch.empty(1, dtype=torch.int32, device=dev)
for _ in range(5):
    K.evict_select(keys1, 1, out_ids=ids1, workspace=ws1, sync=False)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    K.evict_select(keys1, 1, out_ids=ids1, workspace=ws1, sync=False)
b.record()
b.synchronize()
res["nothing_evictable_us"] = a.elapsed_time(b) * 1e3 / 50
print("RESULT " + json.dumps(res))
""" % ROOT


def main():
    sizes = sys.argv[1:] or ["0"]
    for c in sizes:
        r = subprocess.run([sys.executable, "-c", CHILD, c], capture_output=True, text=True, timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        if r.returncode != 0 or not line:
            print(json.dumps({"ctas": c, "error": (r.stdout + r.stderr)[-3000:]}))
            continue
        print(json.dumps({"ctas": c, **json.loads(line[0][7:])}))


if __name__ == "__main__":
    main()
