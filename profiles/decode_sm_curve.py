"""Decode-kernel bandwidth as a function of the SMs it gets (diagnostic): kva_diag_occupy holds
N SMs on a side stream, then the decode phase of the llama7b plan runs on the remaining ones.

python profiles/decode_sm_curve.py [config] -> JSON lines {occupied, sms, us, GBps}
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402
from bench import _post_append_batch  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "llama7b"
    dev = torch.device("cuda", 0)
    wl = W.make_workload(cfg, device=dev)
    pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
    batch = _post_append_batch(K, wl, dev)
    plan = K.Plan(pool, batch)
    st = plan.stats()
    out = torch.empty(wl.q.shape, dtype=torch.bfloat16, device=dev)
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream(priority=-1)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for occ in [0, 24, 44, 54, 64, 74, 84, 104]:
        ts = []
        for i in range(6):
            torch.cuda.synchronize()
            K.diag_occupy(occ, 200 * 1024, 3_000_000, stream=side)
            torch.cuda._sleep(200000)  # let the occupying CTAs become resident
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main_s)
            plan.run(wl.q, out, phases=K.PHASE_DECODE)
            b.record(main_s)
            torch.cuda.synchronize()
            if i >= 1:
                ts.append(a.elapsed_time(b) * 1e3)
        us = statistics.median(ts)
        print(json.dumps({"occupied": occ, "sms": nsm - occ, "us": round(us, 1),
                          "GBps": round(st["decode_kv_bytes"] / us / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
