"""External yardstick for the tcgen05 tile kernel (optional; FlashInfer is called
only here): llama70b's prefill part — 2 chunks of 8,192 queries at positions [8192, 16384),
64 q / 8 kv heads x d128, causal — through this library's hybrid_attention and through
FlashInfer 0.6.11's trtllm-gen paged context attention on the SAME pool and tables.  CUDA events,
20 calls after warm-up; prints one JSON line."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / n


def main():
    dev = torch.device("cuda", 0)
    reqs = [W.ReqSpec(W.OFFLINE_PREFILL, 16384, 8192, -1) for _ in range(2)]
    wl = W.make_workload(W.custom_config("yt", 64, 8, 128, 4, reqs, []), device=dev)
    pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
    batch = K.Batch(wl.batch, dev)
    K.kv_append(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
    torch.cuda.synchronize()
    q = wl.q.to(dev)
    out = torch.empty(q.shape, dtype=torch.bfloat16, device=dev)
    plan = K.Plan(pool, batch)
    flops = plan.stats()["tile_flops"]
    res = {"shape": "2 causal chunks x 8192 queries at [8192, 16384), 64/8 heads x d128", "flops": flops,
           "ours_us": timed(lambda: plan.run(q, out))}
    try:
        import flashinfer
        from flashinfer.prefill import trtllm_batch_context_with_kv_cache
        ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
        bt = batch.table_dev[:, : 16384 // 16].contiguous().to(torch.int32)
        seq = torch.full((2,), 16384, dtype=torch.int32, device=dev)
        cq = torch.tensor([0, 8192, 16384], dtype=torch.int32, device=dev)
        ck = torch.tensor([0, 16384, 32768], dtype=torch.int32, device=dev)
        fo = torch.empty_like(out)
        fn = lambda: trtllm_batch_context_with_kv_cache(  # noqa: E731
            q, (pool.k_pool, pool.v_pool), ws, bt, seq, 8192, 16384, 1.0 / math.sqrt(128), 1.0, 2, cq, ck,
            out=fo, kv_layout="HND", causal=True)
        res["flashinfer_version"] = flashinfer.__version__
        res["flashinfer_trtllm_gen_us"] = timed(fn)
        res["max_abs_diff_vs_ours"] = float((fo.float() - out.float()).abs().max().item())
    except Exception as e:  # noqa: BLE001
        res["flashinfer_error"] = f"{type(e).__name__}: {str(e)[:300]}"
    for k in ("ours_us", "flashinfer_trtllm_gen_us"):
        if k in res:
            res[k.replace("_us", "_TFLOPs")] = flops / (res[k] * 1e-6) / 1e12
    print(json.dumps(res))


if __name__ == "__main__":
    main()
