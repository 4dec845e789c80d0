"""Helpers for the -m gpu parity tests: run one step through the C-ABI library on cuda:0 and
the same step through the oracle, on the same seeded inputs (workloads)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import workloads as W


def bits16(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def gpu_step(wl: W.Workload, out_dtype=torch.float32, device="cuda", want_lse=True):
    """kv_append + hybrid_attention through the library; returns a dict of device results."""
    import paper_2504_03651_b200 as K
    kp = wl.k_pool.to(device).contiguous()
    vp = wl.v_pool.to(device).contiguous()
    fb = K.free_bits_tensor(wl.free_bits, device)
    pool = K.Pool(kp, vp, fb)
    batch = K.Batch(wl.batch, device)
    K.kv_append(pool, batch, wl.k_new.to(device), wl.v_new.to(device))
    q = wl.q.to(device)
    out = torch.full(q.shape, float("nan"), dtype=out_dtype, device=device)
    lse = torch.full(q.shape[:2], float("nan"), dtype=torch.float32, device=device) if want_lse else None
    plan = K.Plan(pool, batch)
    plan.run(q, out, lse)
    torch.cuda.synchronize()
    return dict(pool=pool, batch=batch, out=out, lse=lse, k_pool=kp, v_pool=vp, free_bits=fb,
                plan=plan, q=q)


def oracle_step(wl: W.Workload):
    """The oracle's append + attention on the pre-append state (never reads GPU results)."""
    st, deficit, kp, vp, bt, fb = oracle.kv_append(wl.batch, wl.k_pool, wl.v_pool, wl.free_bits,
                                                  wl.k_new, wl.v_new)
    assert st == oracle.OK, st
    b = dict(wl.batch)
    b["block_table"] = bt
    st, out, lse = oracle.attention(b, kp, vp, wl.q)
    assert st == oracle.OK, st
    return dict(k_pool=kp, v_pool=vp, block_table=bt, free_bits=fb, out=out, lse=lse, batch=b)


def oracle_rows(wl: W.Workload, rows, heads):
    st, deficit, kp, vp, bt, fb = oracle.kv_append(wl.batch, wl.k_pool, wl.v_pool, wl.free_bits,
                                                  wl.k_new, wl.v_new)
    assert st == oracle.OK
    b = dict(wl.batch)
    b["block_table"] = bt
    st, out, lse = oracle.attention_rows(b, kp, vp, wl.q, rows, heads)
    assert st == oracle.OK
    return out, lse, bt


def assert_attention_close(out_gpu, lse_gpu, out_ref, lse_ref, bf16=False):
    """north_star tolerance: max-abs 1e-2 (fp32 output); bf16 output: 1e-2 + 2^-8|O| (H7);
    lse max-abs 1e-3."""
    o = out_gpu.float().cpu().numpy().astype(np.float64)
    assert np.isfinite(o).all(), "non-finite output"
    err = np.abs(o - out_ref)
    tol = 1e-2 + (2.0 ** -8) * np.abs(out_ref) if bf16 else 1e-2
    bad = err > tol
    assert not bad.any(), f"max err {err.max():.3e} at {np.unravel_index(err.argmax(), err.shape)}"
    if lse_gpu is not None:
        l = lse_gpu.cpu().numpy().astype(np.float64)
        lerr = np.abs(l - lse_ref)
        assert lerr.max() <= 1e-3, f"lse max err {lerr.max():.3e}"
    return float(err.max())
