"""Summarise ncu --set full captures into profiles/ncu_summary.json (config -> kernel -> metrics)
and keep the raw metric CSV next to it.

python profiles/ncu_summarize.py OUTDIR gpurun_out/prof_<config>_<kernel>.ncu-rep ...
(bench.py reads dram_bytes_per_launch as the roofline `traffic`.)
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return None


def main():
    outdir = sys.argv[1]
    os.makedirs(outdir, exist_ok=True)
    path = os.path.join(HERE, "ncu_summary.json")
    summ = json.load(open(path)) if os.path.exists(path) else {}
    if summ and not all(isinstance(v, dict) and all(isinstance(w, dict) for w in v.values()) for v in summ.values()):
        summ = {}
    for rep in sys.argv[2:]:
        m = re.match(r"prof_(.+?)_(\w+?_kernel\w*?)\.ncu-rep$", os.path.basename(rep))
        if not m:
            print("skip", rep)
            continue
        cfg, kern = m.group(1), m.group(2)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        open(os.path.join(outdir, f"ncu_raw_{cfg}_{kern}.csv"), "w").write(raw)
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            print("empty", rep)
            continue
        h, units, vals = rows[0], rows[1], rows[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
                 "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
        d = {}
        for k, u, v in zip(h, units, vals):
            if k in KEYS and num(v) is not None:
                d[k] = num(v) * scale.get(u, 1.0)  # bytes in B, times in us
        d["units"] = "bytes: B, gpu__time_duration: us"
        d["kernel_name"] = dict(zip(h, vals)).get("Kernel Name")
        rd, wr = d.get("dram__bytes_read.sum") or 0, d.get("dram__bytes_write.sum") or 0
        d["dram_bytes_per_launch"] = rd + wr
        summ.setdefault(cfg, {})[kern] = d
        print(cfg, kern, {k: d[k] for k in ("gpu__time_duration.sum", "dram_bytes_per_launch") if k in d})
    json.dump(summ, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
