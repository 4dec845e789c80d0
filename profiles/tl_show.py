"""Print the last N steps of a timeline JSON (profiles/timeline.py output): kva kernels per
stream, times relative to the first kernel shown.  python profiles/tl_show.py file.json [n_events]"""
import json
import sys

ev = json.load(open(sys.argv[1]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
dev = [e for e in ev if e["stream"] != -1 and ("kva" in e["kernel"] or "Memcpy" in e["kernel"])]
dev.sort(key=lambda e: e["start_us"])
dev = dev[-n:]
t0 = dev[0]["start_us"]
for e in dev:
    name = e["kernel"].split("(")[0].replace("void kva::", "").replace("(anonymous namespace)::", "")[:60]
    print(f"s{e['stream']:<3} {e['start_us'] - t0:9.1f} {e['end_us'] - t0:9.1f} {e['end_us'] - e['start_us']:7.1f}  {name}")
