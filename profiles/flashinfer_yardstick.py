"""External yardstick (FlashInfer "may serve as an optional external yardstick on
the same box; not the oracle and not a code source"): the decode part of the llama7b batch —
64 online decodes of 2,048 keys, 32/32 heads x d128, 16-token pages — through this library's
hybrid_attention (decode split-KV + merge) and through FlashInfer's trtllm-gen paged decode
(library kernels, called only here, never on the product path), on the SAME pool and block
tables (our [blocks][Hkv][16][d] K / V pools are its HND layout).  CUDA events, 200 calls
after warm-up; prints one JSON line.  python profiles/flashinfer_yardstick.py"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402


def timed(fn, n=200):
    for _ in range(20):
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
    reqs = [W.ReqSpec(W.ONLINE_DECODE, 2048, 1) for _ in range(64)]
    wl = W.make_workload(W.custom_config("yard", 32, 32, 128, 1, reqs, []), device=dev)
    pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
    batch = K.Batch(wl.batch, dev)
    K.kv_append(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
    torch.cuda.synchronize()
    q = wl.q.to(dev)
    out = torch.empty(q.shape, dtype=torch.bfloat16, device=dev)
    plan = K.Plan(pool, batch)
    ours_us = timed(lambda: plan.run(q, out))
    res = {"shape": "64 decodes x 2048 keys, 32/32 heads, d128, bf16 KV, 16-token pages",
           "kv_bytes": 64 * 2048 * 32 * 128 * 2 * 2, "ours_us": ours_us}
    try:
        import flashinfer
        from flashinfer.decode import trtllm_batch_decode_with_kv_cache
        ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
        bt = batch.table_dev[:, : 2048 // 16].contiguous().to(torch.int32)
        seq = torch.full((64,), 2048, dtype=torch.int32, device=dev)
        fo = torch.empty_like(out)
        fn = lambda: trtllm_batch_decode_with_kv_cache(  # noqa: E731
            q, (pool.k_pool, pool.v_pool), ws, bt, seq, 2048, bmm1_scale=1.0 / math.sqrt(128), bmm2_scale=1.0,
            out=fo, kv_layout="HND")
        res["flashinfer_version"] = flashinfer.__version__
        res["flashinfer_trtllm_gen_us"] = timed(fn)
        res["max_abs_diff_vs_ours"] = float((fo.float() - out.float()).abs().max().item())
    except Exception as e:  # noqa: BLE001
        res["flashinfer_error"] = f"{type(e).__name__}: {str(e)[:300]}"
    for k in ("ours_us", "flashinfer_trtllm_gen_us"):
        if k in res:
            res[k.replace("_us", "_GBps")] = res["kv_bytes"] / (res[k] * 1e-6) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
