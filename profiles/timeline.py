"""GPU kernel timeline of a few bench steps via torch.profiler (CUPTI activity records):
start/end of every kernel per stream, relative to the first kernel of the last step.

python profiles/timeline.py [config] [--out file.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "llama7b"
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    e2e = "--e2e" in sys.argv
    dump_all = "--all" in sys.argv
    if e2e:  # profile the pipelined end-to-end loop (host copies) instead of the device-only one
        os.environ["KVA_BENCH_E2E_IN_PROFILE"] = "1"
    sys.argv = [sys.argv[0], "--config", cfg, "--steps", "6", "--warmup", "3", "--no-cpu-baseline",
                "--profile"] + ([] if e2e else ["--no-e2e"])
    import bench
    from torch.profiler import ProfilerActivity, profile
    args = bench.parse()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        bench.run_ours(args, 0, 1, 0)
    evs = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0:
            evs.append((e.time_range.start, e.time_range.end, e.name, getattr(e, "device_resource_id", 0)))
    evs.sort()
    mine = [x for x in evs if any(k in x[2] for k in ("kva::", "decode_", "tile_", "merge_kernel",
                                                      "append_kernel", "manager_", "evict_", "release_ids",
                                                      "Memcpy", "Memset", "elementwise", "copy"))]
    if dump_all:  # every CUDA event of the run (relative to the first)
        t00 = mine[0][0]
        allrows = [{"kernel": n.split("(")[0][-40:], "stream": s, "start_us": round(a - t00, 1),
                    "end_us": round(b - t00, 1)} for a, b, n, s in mine]
        # host runtime calls that block (> 20 us), same clock
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CPU and e.time_range.elapsed_us() > 20 and \
                    ("cuda" in e.name.lower() or "synchron" in e.name.lower() or "copy" in e.name.lower()):
                allrows.append({"kernel": "HOST " + e.name[:60], "stream": -1,
                                "start_us": round(e.time_range.start - t00, 1),
                                "end_us": round(e.time_range.end - t00, 1)})
        allrows.sort(key=lambda r: r["start_us"])
        if out:
            json.dump(allrows, open(out, "w"), indent=0)
        return
    # last step = kernels after the last append_kernel's preceding evict_keys
    starts = [i for i, x in enumerate(mine) if "manager_kernel" in x[2]] or [0]
    last = mine[starts[-1]:]
    t0 = last[0][0]
    rows = [{"kernel": n.split("(")[0][-40:], "stream": s, "start_us": round(a - t0, 1),
             "end_us": round(b - t0, 1), "dur_us": round(b - a, 1)} for a, b, n, s in last]
    # host-side runtime API calls of the same step (when each launch was ENQUEUED)
    t_end = last[-1][1]
    api = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda") and \
                t0 - 200 <= e.time_range.start <= t_end:
            api.append({"api": e.name, "start_us": round(e.time_range.start - t0, 1),
                        "dur_us": round(e.time_range.elapsed_us(), 1)})
    api.sort(key=lambda r: r["start_us"])
    rows.append({"host_api": api})
    for r in rows[:-1]:
        print(f"{r['kernel']:42s} stream={r['stream']:<4} {r['start_us']:9.1f} -> {r['end_us']:9.1f}  ({r['dur_us']:.1f} us)")
    if out:
        json.dump(rows, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
