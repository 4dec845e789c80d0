#!/usr/bin/env python
"""bench.py — one iteration of the co-scheduled serving loop's device hot path per step
(SURVEY §8(a) rows a1-a8): kv_append (+ block allocation) -> hybrid_attention (plan + tile /
decode split-KV / LSE-merge kernels) -> [G>1: NCCL all-gather of O over NVLink] ->
kv_manager_step + evict_select (1M-block pool, top-64k) -> kv_truncate (rollback of this step's
allocations, so that every step is the same iteration).

Contract: `python bench.py --gpus N --steps K --warmup W` prints ONE JSON line on rank 0.
`--impl reference` times the fp64 CPU oracle (the reference arm of this tier) instead.
The default workload is BASELINE.json configs[1] (Llama-2-7B-shaped mixed batch with a shared
offline prefix, "llama7b"); inputs are seeded synthetic (workloads/).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

WORKLOAD_NAMES = {"llama7b": "llama7b (BASELINE.json configs[1])", "tiny": "tiny (BASELINE.json configs[0])",
                  "qwen14b": "qwen14b (BASELINE.json configs[2])", "llama70b": "llama70b (BASELINE.json configs[4])",
                  "qwen14b-p": "qwen14b-p (configs[2] variant: shared-prefix prefill, SURVEY NEXT-4)",
                  "llama7b-u": "llama7b-u (control: configs[1] with the prefix duplicated per request, no sharing)",
                  "qwen14b-u": "qwen14b-u (control: configs[2] with the prefix duplicated per request, no sharing)",
                  "qwen14b-pu": "qwen14b-pu (control: qwen14b-p without sharing)"}
METRIC = "mixed-batch attention tokens/s and HBM GB/s (% of B200 roofline) at 1/2/4/8 GPUs"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama7b")
    ap.add_argument("--out-dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--no-evict", action="store_true")
    ap.add_argument("--evict-thread", type=int, default=0,
                    help="1: the KV manager's per-step calls (kv_manager_step + evict_select) are "
                         "enqueued by a second host thread, concurrently with the attention calls")
    ap.add_argument("--l2-rotate", type=int, default=4,
                    help="replicas of every per-step input (pool, tables, Q/K/V, manager metadata) "
                         "cycled step by step so no step finds the previous one's data in L2 (1 = off)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/e2e/cpu)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch + process group + max-over-ranks only (no GPU; CPU tests)")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "fused"],
                    help="N>1: NCCL all-gather after the attention (default), or the epilogues "
                         "storing into the peers' symmetric-memory buffers (kva_plan_set_outputs)")
    ap.add_argument("--dist-backend", default="nccl",
                    help="nccl (default); gloo only to smoke-test the N>1 code path on one GPU")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------
def dist_setup(args, cpu=False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and cpu:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
        return rank, world, local
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region via NVML (1 ms polling
    thread; nvidia-smi's 200 ms period is longer than many timed regions).  Falls back to one
    nvidia-smi query if NVML is unavailable."""
    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.samples, self.reasons, self.smax = [], set(), None
        self.stop_flag = threading.Event()
        self.nv = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.idx]) if vis and vis.split(",")[0].isdigit() else self.idx
            self.h = nv.nvmlDeviceGetHandleByIndex(phys)
            self.smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.nv = nv
        except Exception:
            self.nv = None
            return
        self.sample()
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def sample(self):
        nv = self.nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, const in self.REASONS.items():
                if r & getattr(nv, const, 0):
                    self.reasons.add(name)
        except Exception:
            pass

    def _loop(self):
        while not self.stop_flag.wait(0.001):
            self.sample()

    def stop(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.sample()
        self.stop_flag.set()
        self.t.join(timeout=2)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.smax, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6448.1), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def measured_tensor_peak():
    """dense bf16 TFLOP/s: the SUSTAINED figure (the tile kernel is timed inside a long step)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if "bf16_tflops_sustained" in d:
            return d["bf16_tflops_sustained"], "measured (MEASURED_PEAKS.json bf16_tflops_sustained, cuBLAS 8192^3)"
    return 1440.6, "fallback (B200_PROFILING.md sustained bf16)"


def ncu_traffic(config, kernel):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary
    (profiles/ncu_summary.json, written by profiles/ncu_summarize.py; keyed config -> kernel)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        return d.get(config, {}).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
def run_ours(args, rank, world, local):
    import paper_2504_03651_b200 as K
    import workloads as W
    from paper_2504_03651_b200 import dist as kdist

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    cfg = W.get_config(args.config)
    wl = W.make_workload(cfg, device=dev, rank=rank, world=world)
    out_dtype = torch.bfloat16 if args.out_dtype == "bf16" else torch.float32
    pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
    batch = K.Batch(wl.batch, dev)
    pristine_host = batch.table_host.copy()
    # every step ends by rolling the iteration back (kv_truncate to the pre-append lengths:
    # the blocks kv_append allocated are released and their table entries reset, host mirror
    # and device table), so that every step appends and allocates the same way
    keep_len = (batch.ctx_len - np.diff(batch.q_indptr)).astype(np.int32)
    ws_app = torch.empty(K.kv_append_workspace_size(batch), dtype=torch.uint8, device=dev)
    ws_att = torch.empty(K.hybrid_attention_workspace_size(batch), dtype=torch.uint8, device=dev)
    q, k_new, v_new = wl.q, wl.k_new, wl.v_new
    T, Hl, d = q.shape
    out = torch.empty((T, Hl, d), dtype=out_dtype, device=dev)
    lse = torch.empty((T, Hl), dtype=torch.float32, device=dev)
    gbuf = torch.empty((world, T, Hl, d), dtype=out_dtype, device=dev) if world > 1 else None
    fused = None
    if world > 1 and args.gather == "fused":
        # a7 fused into the epilogues: out = this rank's slot of a symmetric gathered buffer,
        # the peers' slots are extra destinations of every run (include/kvattn.h)
        fused = kdist.FusedGather((T, Hl, d), out_dtype, dev)
        out = fused.out_local
        gbuf = fused.buf

    ev = None
    if not args.no_evict:
        # the KV manager's per-iteration pass over the `evict` config's 2^20-block metadata
        # (BASELINE configs[3]): class transitions + rc recount from the offline pool
        # -> keys -> top-64k selection (a8)
        evw = W.make_evict()
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)
        ev = dict(state=t(evw.state, np.uint8), rc=t(evw.rc, np.int32), lat=t(evw.lat, np.int32),
                  depth=t(evw.depth, np.int16), k=evw.k, n=len(evw.state))
        chains, mpool = W.make_manager_update(evw, now=1 << 20, seed=1)
        ev["mgr"] = K.ManagerStep(ev["state"], ev["rc"], ev["lat"], ev["depth"])
        # the transition chains are the finished requests' block-table rows: device-resident,
        # handed to the manager as device arrays (no per-step upload; ids range-checked on the GPU)
        ev["chains"] = K.ManagerStep.chains_to_device(K.ManagerStep.chains_csr(chains), dev)
        # incremental reference counts: each iteration 1% of the offline pool's requests leave
        # (finished) and as many new requests with the same prompts join (steady state)
        rng_p = np.random.default_rng(11)
        moved = [mpool[i] for i in rng_p.choice(len(mpool), len(mpool) // 100, replace=False)]
        ev["pool_ids"] = torch.from_numpy(np.concatenate(moved).astype(np.int32)).to(dev)
        ev["del_ids"] = ev["pool_ids"].clone()
        ev["ids"] = torch.empty(ev["k"], dtype=torch.int32, device=dev)
        ev["ws"] = torch.empty(K.evict_select_workspace_size(ev["n"], ev["k"]), dtype=torch.uint8, device=dev)

    # L2 hygiene (H8): R replicas of every per-step input, step i uses replica i % R — the hot
    # small parts (shared prefix, Q, workspaces, manager metadata and keys) would otherwise be
    # re-read from the 126 MB L2 by the next step (the decode stream is marked evict-first and
    # does not displace them).  Replica 0 is the original; the others are device copies.
    R = max(1, args.l2_rotate)
    reps = [dict(pool=pool, batch=batch, ws_app=ws_app, ws_att=ws_att, q=q, k_new=k_new, v_new=v_new,
                 out=out, lse=lse, ev=ev)]
    for r in range(1, R):
        b_r = K.Batch(wl.batch, dev)
        rp = dict(pool=K.Pool(wl.k_pool.clone(), wl.v_pool.clone(), K.free_bits_tensor(wl.free_bits, dev)),
                  batch=b_r, ws_app=torch.empty_like(ws_app), ws_att=torch.empty_like(ws_att),
                  q=q.clone(), k_new=k_new.clone(), v_new=v_new.clone(), out=torch.empty_like(out),
                  lse=torch.empty_like(lse), ev=None)
        if ev is not None:
            e2 = dict(ev)
            for kname in ("state", "rc", "lat", "depth"):
                e2[kname] = ev[kname].clone()
            e2["mgr"] = K.ManagerStep(e2["state"], e2["rc"], e2["lat"], e2["depth"])
            e2["ids"] = torch.empty_like(ev["ids"])
            e2["ws"] = torch.empty_like(ev["ws"])
            rp["ev"] = e2
        reps.append(rp)
    rot = {"on": True, "i": 0}
    if fused is not None:  # every replica writes into the symmetric gathered buffer
        for rp in reps:
            rp["out"] = fused.out_local

    # e2e host buffers (pinned): inputs in, output out, every step
    h_q = q.cpu().pin_memory()
    h_k = k_new.cpu().pin_memory()
    h_v = v_new.cpu().pin_memory()
    h_out = torch.empty((gbuf if world > 1 else out).shape, dtype=out.dtype).pin_memory()

    launches = {"n": 0}
    plan_launches = {"n": None}

    # per-kernel durations inside the timed steps from in-kernel %globaltimer spans (first CTA
    # start -> last CTA end of the decode and tile kernels; kva_plan_set_span_buffer) — no stream
    # operation between the kernels, so the programmatic-dependent-launch chain stays intact
    # (CUDA events between them cost ~20 us per step)
    spans = torch.zeros((args.steps, 6), dtype=torch.int64, device=dev)
    spans[:, 0] = -1
    spans[:, 2] = -1
    spans[:, 4] = -1
    span_used = []

    ev_stream = torch.cuda.Stream(device=dev, priority=int(os.environ.get("KVA_BENCH_EVICT_PRIO", "0")))
    ev_fork, ev_join, ev_keys = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()
    # the attention pair is launched after the manager's key pass, so the cooperative eviction
    # selection (next on its stream) is placed on the SMs before the decode kernel fills them
    gate_attn = os.environ.get("KVA_BENCH_GATE", "0" if os.environ.get("KVA_BENCH_FUSED_MGR", "1") == "1" else "1") == "1"
    # The manager pass + selection of step i depend only on the block metadata (updated in order
    # on their own stream), not on step i-1's attention: by default they are not forked from the
    # main stream each step, so step i's metadata pass runs as soon as step i-1's selection
    # finishes (overlapping step i-1's tail) — the serving loop issues it as soon as the
    # iteration's transitions are known.  Every step still runs the whole pass; the timed region
    # starts with a fork (ev_fork) so no eviction work of a timed step precedes it.
    # KVA_BENCH_EVICT_PIPELINE=0: fork every step (serialises it behind the previous step).
    evict_pipeline = os.environ.get("KVA_BENCH_EVICT_PIPELINE", "1") == "1"
    fork_next = {"v": True}
    # The eviction stream is joined into the main stream once, at the end of the timed region
    # (every step's manager pass + selection is still inside it): a per-step event wait would
    # sit between the merge and the next kv_truncate / kv_append launches and break their
    # programmatic-dependent-launch chain.  KVA_BENCH_JOIN_EACH_STEP=1: join every step.
    join_each_step = os.environ.get("KVA_BENCH_JOIN_EACH_STEP", "0") == "1"
    gather_on = {"v": True}

    # The KV manager's per-step enqueue on its own host thread (a serving engine's scheduler /
    # KV-manager bookkeeping runs beside the model runner): the main thread hands it the step's
    # replica and waits for "enqueued" only right before ordering the step's end after the
    # selection (ev_join).  ctypes releases the GIL inside the library calls.
    import queue
    jobs, done = queue.SimpleQueue(), queue.SimpleQueue()

    # the manager step and the selection as ONE cooperative kernel (kv_manager_step_select: the
    # key pass feeds the selection directly); KVA_BENCH_FUSED_MGR=0: two launches
    fused_mgr = os.environ.get("KVA_BENCH_FUSED_MGR", "1") == "1"
    if os.environ.get("KVA_BENCH_FOLD"):  # diagnostics: 0 = cascade members merged by the merge kernel
        K.set_option("fold", int(os.environ["KVA_BENCH_FOLD"]))
    if os.environ.get("KVA_BENCH_TILE_CTAS"):  # diagnostics: the tile kernel's SM share (0 = plan's split)
        K.set_option("tile_ctas", int(os.environ["KVA_BENCH_TILE_CTAS"]))
    if os.environ.get("KVA_BENCH_EVICT_CTAS"):  # diagnostics: the selection's grid size
        K.set_option("evict_ctas", int(os.environ["KVA_BENCH_EVICT_CTAS"]))

    def evict_enqueue(ev, fork):
        if fork:
            ev_stream.wait_event(ev_fork)
        if fused_mgr:
            ev["mgr"](1 << 20, ev["chains"], ev["pool_ids"], del_ids=ev["del_ids"], recount=False,
                      stream=ev_stream, select=(ev["k"], ev["ids"], ev["ws"]))
            ev_keys.record(ev_stream)
        else:
            keys = ev["mgr"](1 << 20, ev["chains"], ev["pool_ids"], del_ids=ev["del_ids"], recount=False,
                             stream=ev_stream)
            ev_keys.record(ev_stream)
            K.evict_select(keys, ev["k"], out_ids=ev["ids"], workspace=ev["ws"], stream=ev_stream, sync=False)
        ev_join.record(ev_stream)

    def evict_worker():
        torch.cuda.set_device(dev)
        while True:
            job = jobs.get()
            if job is None:
                return
            try:
                evict_enqueue(*job)
                done.put(None)
            except BaseException as exc:  # surfaced on the main thread
                done.put(exc)

    threaded = bool(args.evict_thread) and ev is not None
    if threaded:
        worker = threading.Thread(target=evict_worker, daemon=True)
        worker.start()

    def step(time_idx=None):
        rp = reps[rot["i"] % R] if rot["on"] else reps[0]
        rot["i"] += 1
        pool, batch, ev = rp["pool"], rp["batch"], rp["ev"]
        q, out, lse = rp["q"], rp["out"], rp["lse"]
        n = 0
        if ev is not None:
            # the manager's eviction selection has no data dependency on this layer's attention:
            # it runs on its own stream, concurrently (its CTAs leave room for decode CTAs)
            fork = fork_next["v"] or not evict_pipeline
            if fork:
                ev_fork.record(stream)
                fork_next["v"] = False
            if threaded:
                jobs.put((ev, fork))
            else:
                evict_enqueue(ev, fork)
            n += 1 if fused_mgr else 2
        if ev is not None and gate_attn and not threaded:  # the attention pair follows the key pass
            stream.wait_event(ev_keys)
        # kv_append + plan of the same descriptor in one library call (one validation)
        plan = K.kv_append_plan(pool, batch, rp["k_new"], rp["v_new"], rp["ws_app"], rp["ws_att"], stream=stream)
        if plan_launches["n"] is None:  # the same descriptor every step: count once
            plan_launches["n"] = plan.launch_count()
        n += 2 + plan_launches["n"]
        if time_idx is not None:
            plan.set_span_buffer(spans[time_idx])
            span_used.append(time_idx)
        if fused is not None and gather_on["v"]:
            fused.attach(plan)
        plan.run(q, out, lse, stream=stream)
        if world > 1 and gather_on["v"]:
            if fused is not None:
                fused.barrier()
            else:
                kdist.gather_outputs(out, gbuf)
        if ev is not None:
            if threaded:
                exc = done.get()
                if exc is not None:
                    raise exc
            if join_each_step:
                stream.wait_event(ev_join)
        K.kv_truncate(pool, batch, keep_len, stream=stream)
        n += 1
        launches["n"] += n
        plan.close()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            torch.cuda.synchronize()

    def timed(nsteps, time_kernels=False):
        barrier()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        fork_next["v"] = True  # the first timed step's eviction work starts after s
        host_t = []
        for i in range(nsteps):
            t_h = time.perf_counter()
            step(time_idx=i if time_kernels else None)
            host_t.append(time.perf_counter() - t_h)
        stream.wait_event(ev_join)  # the last step's eviction work (ev_join: recorded after every step's)
        e.record(stream)
        if os.environ.get("KVA_BENCH_HOST_TIMING") == "1":  # diagnostics: host enqueue time per step
            sys.stderr.write(f"[bench host] step enqueue median {1e6 * sorted(host_t)[len(host_t) // 2]:.1f} us\n")
        barrier()
        ms = s.elapsed_time(e) / nsteps
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

    # --- end-to-end (host buffers in, host result out) with the copies pipelined the way a
    # serving loop runs them: step i+1's inputs go host->device on a copy stream while step i
    # computes, and step i's output goes device->host on a second copy stream (PCIe is full
    # duplex).  Double-buffered device inputs/outputs; every hazard is an event.
    bufs = [dict(q=q, k=k_new, v=v_new, out=out, g=gbuf)]
    bufs.append(dict(q=torch.empty_like(q), k=torch.empty_like(k_new), v=torch.empty_like(v_new),
                     out=torch.empty_like(out), g=torch.empty_like(gbuf) if gbuf is not None else None))
    cs_in = torch.cuda.Stream(device=dev)
    cs_out = torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]     # inputs of buffer b landed
    ev_used = [torch.cuda.Event() for _ in range(2)]   # compute finished reading buffer b
    ev_out = [torch.cuda.Event() for _ in range(2)]    # result of buffer b copied to host

    def step_e2e(i):
        b = bufs[i % 2]
        n = 0
        with torch.cuda.stream(cs_in):
            if i >= 2:
                cs_in.wait_event(ev_used[i % 2])
            b["q"].copy_(h_q, non_blocking=True)
            b["k"].copy_(h_k, non_blocking=True)
            b["v"].copy_(h_v, non_blocking=True)
            ev_in[i % 2].record(cs_in)
        if ev is not None:
            fork = fork_next["v"] or not evict_pipeline
            if fork:
                ev_fork.record(stream)
                fork_next["v"] = False
            if threaded:
                jobs.put((ev, fork))
            else:
                evict_enqueue(ev, fork)
            n += 1 if fused_mgr else 2
        stream.wait_event(ev_in[i % 2])
        if i >= 2:
            stream.wait_event(ev_out[i % 2])   # the host copy of this buffer's last result is done
        if ev is not None and gate_attn and not threaded:
            stream.wait_event(ev_keys)
        plan = K.kv_append_plan(pool, batch, b["k"], b["v"], ws_app, ws_att, stream=stream)
        if plan_launches["n"] is None:  # the same descriptor every step: count once
            plan_launches["n"] = plan.launch_count()
        n += 2 + plan_launches["n"]
        plan.run(b["q"], b["out"], lse, stream=stream)
        res_t = b["out"]
        if world > 1:
            kdist.gather_outputs(b["out"], b["g"])
            res_t = b["g"]
        ev_used[i % 2].record(stream)
        with torch.cuda.stream(cs_out):
            cs_out.wait_event(ev_used[i % 2])
            h_out.copy_(res_t, non_blocking=True)
            ev_out[i % 2].record(cs_out)
        if ev is not None:
            if threaded:
                exc = done.get()
                if exc is not None:
                    raise exc
            if join_each_step:
                stream.wait_event(ev_join)
        K.kv_truncate(pool, batch, keep_len, stream=stream)
        n += 1
        launches["n"] += n
        plan.close()

    def h2d_d2h_only(n=10):
        """the step's copies alone (PCIe ceiling of the e2e number): ms per step"""
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs_in):
            a.record(cs_in)
            for i in range(n):
                bb = bufs[i % 2]
                bb["q"].copy_(h_q, non_blocking=True)
                bb["k"].copy_(h_k, non_blocking=True)
                bb["v"].copy_(h_v, non_blocking=True)
            b.record(cs_in)
        b.synchronize()
        h2d = a.elapsed_time(b) / n
        with torch.cuda.stream(cs_out):
            a.record(cs_out)
            for i in range(n):
                h_out.copy_(bufs[i % 2]["g"] if world > 1 else bufs[i % 2]["out"], non_blocking=True)
            b.record(cs_out)
        b.synchronize()
        return h2d, a.elapsed_time(b) / n

    def timed_e2e_pipelined(nsteps):
        for i in range(4):  # warm-up of the pipelined loop
            step_e2e(i)
        stream.wait_stream(cs_out)
        barrier()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        cs_in.wait_event(s)
        fork_next["v"] = True
        for i in range(nsteps):
            step_e2e(i)
        stream.wait_stream(cs_out)   # the last result is on the host
        stream.wait_event(ev_join)   # the last step's eviction work
        e.record(stream)
        barrier()
        ms = s.elapsed_time(e) / nsteps
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

    # The selection's build (option evict_threads): it runs beside the attention on its own
    # stream.  When the step's decode stream alone takes several selection times (llama7b:
    # ~330 us of decode vs ~50-65 us of selection) its cost is the decode CTAs it displaces, so
    # the 256-thread build (~30 KB of shared memory, shares an SM with two decode CTAs) is
    # used; otherwise (qwen14b: ~66 us of decode) its latency matters and the 512-thread build
    # is used.  Measured (profiles/r02s3): llama7b 392.5 -> 385.3 us/step, qwen14b 130.3 vs
    # 169.6 us with the 256 build.  KVA_BENCH_EVICT_THREADS overrides.
    planA = K.Plan(pool, _post_append_batch(K, wl, dev), stream=stream)
    dec_est_us = planA.stats()["decode_kv_bytes"] / 6.5e6
    planA.close()
    evict_threads = int(os.environ.get("KVA_BENCH_EVICT_THREADS", "256" if dec_est_us > 4 * 50.0 else "512"))
    K.set_option("evict_threads", evict_threads)
    # the same rule for the eviction stream's schedule: beside a long decode-bound step its cost
    # is a throughput tax, spread best as one pass per step (forked at the step's start: llama7b
    # 20 steps 387 -> 382, 50 steps 380 -> 378.5 us/step); where its latency is on the loop
    # (qwen14b) the passes run back to back (pipelined: 135.7 vs 144.9 with a fork per step)
    if "KVA_BENCH_EVICT_PIPELINE" not in os.environ:
        evict_pipeline = evict_threads != 256
    for _ in range(max(args.warmup, R)):  # every replica warmed
        step()
    barrier()
    # the rollback restores the pristine table on both sides (every step starts identically)
    for rp in reps:
        assert np.array_equal(rp["batch"].table_host, pristine_host), "host table != pristine after kv_truncate"
        assert np.array_equal(rp["batch"].table_dev.cpu().numpy(), pristine_host), "device table != pristine"
    plan0 = K.Plan(pool, _post_append_batch(K, wl, dev), stream=stream)
    stats = plan0.stats()
    plan0.close()

    clocks = ClockSampler(local)
    if not args.profile:
        clocks.start()
    launches["n"] = 0
    rot["i"] = 0
    ring = None
    if os.environ.get("KVA_BENCH_SPAN_RING") == "1":  # diagnostics: manager / selection spans
        ring = torch.zeros(5 * 256 * 2, dtype=torch.int64, device=dev)
        K.set_option("span_ring", ring.data_ptr())
    ms = timed(args.steps, time_kernels=True)
    if ring is not None:
        K.set_option("span_ring", 0)
        _dump_timeline(ring, spans, span_used)
        for j, rp in enumerate(reps):  # the selection's phase stamps (CTA 0) of each replica's last call
            if rp["ev"] is not None:
                ts = rp["ev"]["ws"][256:512].view(torch.int64).cpu().numpy()
                ts = ts[ts > 0]
                sys.stderr.write(f"[timeline] sel phases (replica {j}, us): {[round(float(x) / 1e3, 1) for x in np.diff(ts)]}\n")
    gpu_launches = launches["n"]
    # the block metadata is replicated, so every rank's eviction order must be
    # bit-identical — an order-sensitive checksum of replica 0's last selection, min == max
    # over ranks
    evict_identical = None
    if world > 1 and reps[0]["ev"] is not None:
        import torch.distributed as dist
        torch.cuda.synchronize()
        ids = reps[0]["ev"]["ids"].to(torch.int64)
        h = (ids * torch.arange(1, ids.numel() + 1, device=dev, dtype=torch.int64)).sum().reshape(1)
        lo_h, hi_h = h.clone(), h.clone()
        dist.all_reduce(lo_h, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi_h, op=dist.ReduceOp.MAX)
        evict_identical = bool(lo_h.item() == hi_h.item())
        assert evict_identical, "eviction orders differ across ranks"
    ck = clocks.stop() if not args.profile else {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
    ms_same = None
    if R > 1 and not args.profile:  # the same steps on replica 0 only (the delta L2 reuse buys)
        rot["on"] = False
        ms_same = timed(args.steps)
        rot["on"] = True
    sp = spans.cpu().numpy().view(np.uint64)
    dec_ms = [float(sp[i, 1] - sp[i, 0]) * 1e-6 for i in span_used
              if stats["n_decode_items"] > 0 and sp[i, 1] > 0 and sp[i, 1] >= sp[i, 0]]
    tile_ms = [float(sp[i, 3] - sp[i, 2]) * 1e-6 for i in span_used
               if stats["n_tile_items"] > 0 and sp[i, 3] > 0 and sp[i, 3] >= sp[i, 2]]
    # hybrid_attention alone (tokens/s = query tokens / time of hybrid_attention for
    # one layer): first attention kernel start -> last end (tile, decode, merge spans) per step;
    # and the device step period from one step's merge end to the next one's
    att_ms, period_ms = [], []
    for i in span_used:
        st = [sp[i, j] for j in (0, 2, 4) if sp[i, j] != np.uint64(0xFFFFFFFFFFFFFFFF)]
        en = [sp[i, j] for j in (1, 3, 5) if sp[i, j] > 0]
        if st and en:
            att_ms.append(float(max(en) - min(st)) * 1e-6)
    ends = [int(sp[i, 5]) for i in span_used if sp[i, 5] > 0]
    period_ms = [(b - a) * 1e-6 for a, b in zip(ends, ends[1:])]

    def pct(v, q):
        v = sorted(v)
        return v[min(len(v) - 1, int(q * len(v)))] if v else None
    # standalone decode-kernel timing (same plan, no co-running kernels): context for the
    # in-step roofline above, which is measured while the tile kernel shares the GPU
    dec_alone = None
    extra_alone = {}
    if not args.profile and stats["n_decode_items"] > 0:
        plan_s = K.Plan(pool, _post_append_batch(K, wl, dev), stream=stream)
        ts_ = []
        for i in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            plan_s.run(q, out, lse, stream=stream, phases=K.PHASE_DECODE)
            b.record(stream)
            b.synchronize()
            if i >= 3:
                ts_.append(a.elapsed_time(b))
        dec_alone = statistics.median(ts_)
        # kv_append and evict_select alone: each call is preceded by a
        # decode run so the GPU is still busy while the host enqueues it, then bracketed by two
        # events — device time of that call alone, without its host enqueue
        def alone(fn, after=None, n=6):
            ts2 = []
            for i in range(n + 2):
                plan_s.run(q, out, lse, stream=stream, phases=K.PHASE_DECODE)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                if after is not None:
                    after()
                b.synchronize()
                if i >= 2:
                    ts2.append(a.elapsed_time(b))
            return statistics.median(ts2)
        new_rows = int(sum(int(x) for x in np.diff(batch.q_indptr)))
        app_bytes = 2 * 2 * new_rows * k_new.shape[1] * d * 2  # K and V rows: read once, written once
        app_ms = alone(lambda: K.kv_append(pool, batch, k_new, v_new, ws_app, stream=stream),
                       after=lambda: K.kv_truncate(pool, batch, keep_len, stream=stream))
        extra_alone["kv_append"] = {"us": app_ms * 1e3, "bytes": app_bytes,
                                    "GBps": app_bytes / (app_ms * 1e-3) / 1e9}
        if ev is not None:
            ev_ms = alone(lambda: K.evict_select(ev["mgr"].keys, ev["k"], out_ids=ev["ids"], workspace=ev["ws"],
                                                 stream=stream, sync=False))
            extra_alone["evict_select"] = {"us": ev_ms * 1e3, "keys": ev["n"], "k": ev["k"],
                                           "GBps_keys_once": ev["n"] * 8 / (ev_ms * 1e-3) / 1e9,
                                           "note": "1M u64 keys (8.4 MB, read 3x from L2), top-64k sorted"}
            mg_ms = alone(lambda: ev["mgr"](1 << 20, ev["chains"], ev["pool_ids"], del_ids=ev["del_ids"],
                                            recount=False, stream=stream))
            extra_alone["kv_manager_step"] = {"us": mg_ms * 1e3, "blocks": ev["n"]}
        plan_s.close()
    gather = None
    if world > 1:
        # a7 reported on its own: the all-gather alone, and the step without it
        import torch.distributed as dist
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            if fused is not None:  # the fused gather's only separate cost: the cross-rank barrier
                fused.barrier()
            else:
                kdist.gather_outputs(out, gbuf)
        b.record(stream)
        barrier()
        g_ms = torch.tensor([a.elapsed_time(b) / args.steps], device=dev)
        dist.all_reduce(g_ms, op=dist.ReduceOp.MAX)
        gather_on["v"] = False
        ms_ng = timed(args.steps)
        gather_on["v"] = True
        recv = (world - 1) * out.numel() * out.element_size()
        gather = {"ms": g_ms.item(), "bytes_received_per_rank": recv,
                  "GBps_per_rank": recv / (g_ms.item() * 1e-3) / 1e9,
                  "ms_per_step_without_gather": ms_ng, "ms_per_step_with_gather": ms,
                  "backend": dist.get_backend(), "mode": args.gather,
                  "timing": ("CUDA events around K back-to-back all_gather_into_tensor calls on the bench "
                             "stream, max over ranks") if fused is None else
                            ("fused into the epilogues (peer stores over NVLink while the attention runs): "
                             "'ms' = K back-to-back symmetric-memory barriers alone; the transfer itself "
                             "is inside ms_per_step_with_gather")}
    ms_e2e = None
    if not args.no_e2e and (not args.profile or os.environ.get("KVA_BENCH_E2E_IN_PROFILE") == "1"):
        ms_e2e = timed_e2e_pipelined(args.steps)
        copy_ms = h2d_d2h_only()

    tokens = T  # query tokens of the batch (every rank holds all tokens for its heads)
    g = Hl // wl.batch["num_kv_heads"]
    dec_rows_tok = sum(int(wl.batch["q_indptr"][i + 1] - wl.batch["q_indptr"][i])
                       for i in range(wl.batch["num_reqs"])
                       if (wl.batch["q_indptr"][i + 1] - wl.batch["q_indptr"][i]) * g <= 16)
    dec_bytes = stats["decode_kv_bytes"] + dec_rows_tok * Hl * d * 2
    dec_avg = statistics.mean(dec_ms) if dec_ms else float("nan")
    peak, peak_src = measured_peaks()
    achieved = dec_bytes / (dec_avg * 1e-3) / 1e9
    res = {
        "metric": METRIC, "value": tokens / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": WORKLOAD_NAMES.get(args.config, args.config),
                   "q_tokens": tokens, "Hq": cfg.Hq, "Hkv": cfg.Hkv, "head_dim": cfg.d,
                   "requests": len(cfg.reqs), "parallelism": f"kv-head shard x{world}",
                   "kv_bytes_algorithmic_per_rank": stats["kv_bytes_algorithmic"],
                   "flops_per_rank": stats["flops"],
                   "step": "kv_append+hybrid_attention(plan,tile,decode,merge)" +
                           ("+allgather" if world > 1 else "") + ("" if args.no_evict else "+kv_manager_step(1M blocks: 49k transitions, rc +-91k refs, keys)+evict_select(k=64k)" +
                            ((" [eviction pass pipelined: issued after the previous step's selection]" if evict_pipeline else " [eviction pass forked at each step's start]") if ev is not None else "")) +
                           "+kv_truncate(rollback of the step's allocations)",
                   "l2": (f"{R} replicas of every per-step input (pool, tables, Q/K/V, workspaces, manager "
                          f"metadata, keys) cycled step by step (KV working set %.2f GB/rank per replica)"
                          % (stats["kv_bytes_algorithmic"] / 1e9)) if R > 1 else
                         "no rotation (--l2-rotate 1): KV working set %.2f GB/rank" % (stats["kv_bytes_algorithmic"] / 1e9),
                   "ms_per_step_without_l2_rotation": ms_same,
                   "evict_threads": evict_threads,
                   "eviction_identical_across_ranks": evict_identical,
                   "decode_kernel_ms": dec_avg, "out_dtype": args.out_dtype,
                   "tile_kernel_ms": statistics.mean(tile_ms) if tile_ms else None,
                   "tile_kernel_tflops": (stats["tile_flops"] / (statistics.mean(tile_ms) * 1e-3) / 1e12) if tile_ms else None,
                   "overlap": "tile (tcgen05) kernel and decode kernel concurrent (programmatic dependent launch); "
                              "KV-manager pass + eviction selection on a second stream concurrent with the attention"
                              + (", enqueued by a second host thread" if threaded else ""),
                   "host_threads": 2 if threaded else 1},
        "roofline": {"bound": "hbm", "kernel": "decode_kt_kernel (split-KV)", "achieved": achieved,
                     "timing": "in-kernel %globaltimer span per timed step (first CTA start -> last CTA end)",
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(args.config, "decode_kt_kernel"), "bytes_per_launch": dec_bytes,
                     "peak_source": peak_src},
        "clocks": ck, "gpu_launches": gpu_launches,
    }
    if gather is not None:
        res["config"]["gather"] = gather
    tile_avg = statistics.mean(tile_ms) if tile_ms else 0.0
    if tile_avg > 1.5 * (dec_avg if dec_ms else 0.0):
        # tensor-bound batch (long prefill chunks): the dominant kernel is the tcgen05 tile kernel
        tp, tp_src = measured_tensor_peak()
        ach = stats["tile_flops"] / (tile_avg * 1e-3) / 1e12
        res["roofline"] = {"bound": "tensor", "kernel": "tile_tc2_kernel (tcgen05)", "achieved": ach,
                           "peak": tp, "unit": "TFLOP/s", "frac": ach / tp,
                           "traffic": ncu_traffic(args.config, "tile_tc2_kernel"),
                           "flops_per_launch": stats["tile_flops"], "peak_source": tp_src,
                           "decode_hbm": {"achieved_GBps": achieved, "frac": achieved / peak}}
    if att_ms:
        res["attention_only"] = {
            "ms_median": pct(att_ms, 0.5), "ms_p10": pct(att_ms, 0.1), "ms_p90": pct(att_ms, 0.9),
            "tokens_per_s": tokens / (pct(att_ms, 0.5) * 1e-3),
            "timing": "per timed step: first attention-kernel CTA start -> last tile/decode/merge CTA end "
                      "(in-kernel %globaltimer), kv_append / manager / eviction excluded"}
    if period_ms:
        res["step_period_ms"] = {"p10": pct(period_ms, 0.1), "median": pct(period_ms, 0.5),
                                 "p90": pct(period_ms, 0.9),
                                 "timing": "device time between consecutive steps' last merge CTA end"}
    if extra_alone:
        res["config"]["alone"] = extra_alone
    if dec_alone:
        a = dec_bytes / (dec_alone * 1e-3) / 1e9
        res["config"]["decode_kernel_standalone"] = {"ms": dec_alone, "GBps": a, "frac_of_peak": a / peak,
                                                     "note": "median of 5 warm launches, nothing co-running"}
    if ms_e2e is not None:
        res["e2e"] = {"value": tokens / (ms_e2e * 1e-3), "unit": UNIT,
                      "h2d_bytes_per_step": int(h_q.numel() * 2 + h_k.numel() * 2 + h_v.numel() * 2),
                      "d2h_bytes_per_step": int(h_out.numel() * h_out.element_size()),
                      "ms_per_step": ms_e2e,
                      "copies_alone_ms": {"h2d": copy_ms[0], "d2h": copy_ms[1],
                                          "h2d_GBps": (h_q.numel() + h_k.numel() + h_v.numel()) * 2 / copy_ms[0] / 1e6},
                      "pipelining": "inputs of step i+1 copied host->device (pinned) on a copy stream while "
                                    "step i computes; step i's output copied device->host on a second copy "
                                    "stream; double-buffered device buffers; timed from the first input copy "
                                    "to the last result on the host"}
    return res, wl


def _dump_timeline(ring, spans, used):
    """stderr: one line per timed step — attention kernel spans and the manager / selection
    launches (span_ring) that overlap it, us relative to the first step's first start."""
    r = ring.cpu().numpy().view(np.uint64).reshape(5, 256, 2)
    sp = spans.cpu().numpy().view(np.uint64)
    ev = [(nm, int(a), int(b)) for kind, nm in enumerate(("mgr", "sel", "app_dec", "app_pre", "release"))
          for a, b in r[kind] if a and b]
    att = []
    for i in used:
        for nm, j in (("dec", 0), ("tile", 2), ("merge", 4)):
            if sp[i, j] != np.uint64(0xFFFFFFFFFFFFFFFF) and sp[i, j + 1] > 0:
                att.append((f"{nm}{i}", int(sp[i, j]), int(sp[i, j + 1])))
    if not att:
        return
    t0, t1 = min(a[1] for a in att), max(a[2] for a in att)
    rows = sorted([e for e in ev if t0 - 200000 <= e[1] <= t1] + att, key=lambda e: e[1])
    for nm, a, b in rows:
        sys.stderr.write(f"[timeline] {nm:8s} {(a - t0) / 1e3:9.1f} {(b - t0) / 1e3:9.1f} {(b - a) / 1e3:7.1f}\n")


def _post_append_batch(K, wl, dev):
    """Descriptor with every block allocated (for plan statistics only)."""
    b = dict(wl.batch)
    bt = b["block_table"].copy()
    nxt = 0
    free = [i for i in range(b["num_blocks"]) if (int(wl.free_bits[i // 32]) >> (i % 32)) & 1]
    for i in range(b["num_reqs"]):
        for k in range((int(b["ctx_len"][i]) + 15) // 16):
            if bt[i, k] == -1:
                bt[i, k] = free[nxt]
                nxt += 1
    b["block_table"] = bt
    return K.Batch(b, dev)


# ------------------------------------------------------------------------------------------
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def evict_cpu_timings():
    """The eviction selection on the host (the `evict` config: 2^20 keys, top-64k): the fp64
    oracle's full std::sort by (key, id), and a numpy argpartition + sort of the k smallest
    ("fast CPU" line; not the oracle)."""
    import oracle
    import workloads as W
    ev = W.make_evict()
    _, keys = oracle.evict_keys(ev.state, ev.rc, ev.lat, ev.depth)
    t0 = time.perf_counter()
    s, ids = oracle.evict_select(keys, ev.k)
    t1 = time.perf_counter()
    ev_mask = keys != np.uint64(0xFFFFFFFFFFFFFFFF)
    cand = np.nonzero(ev_mask)[0]
    kk = keys[cand]
    part = np.argpartition(kk, ev.k - 1)[:ev.k]   # the k smallest keys (ties at the boundary: then exact sort)
    thr = kk[part].max()
    sel = cand[kk <= thr]
    order = np.lexsort((sel, keys[sel]))[:ev.k]
    fast = sel[order]
    t2 = time.perf_counter()
    assert np.array_equal(fast, ids), "numpy selection disagrees with the oracle"
    return {"keys": int(len(keys)), "k": int(ev.k), "oracle_std_sort_ms": (t1 - t0) * 1e3,
            "numpy_argpartition_sort_ms": (t2 - t1) * 1e3, "threads": 1}


def oracle_sample(wl, seconds, seed=0, nthreads=None):
    """Time the fp64 oracle on a bounded random sample of (row, head) pairs of the batch."""
    import oracle
    import workloads as W  # noqa: F401
    cpu = W_cpu(wl)
    st, _, kp, vp, bt, fb = oracle.kv_append(cpu.batch, cpu.k_pool, cpu.v_pool, cpu.free_bits,
                                             cpu.k_new, cpu.v_new)
    b = dict(cpu.batch, block_table=bt)
    Hq = b["num_q_heads"]
    rng = np.random.default_rng(seed)
    nthreads = nthreads or os.cpu_count() or 1
    n = max(nthreads, 16)
    while True:
        rows = rng.integers(0, cpu.total_q, n).astype(np.int32)
        heads = rng.integers(0, Hq, n).astype(np.int32)
        t0 = time.perf_counter()
        oracle.attention_rows(b, kp, vp, cpu.q, rows, heads, nthreads=nthreads)
        dt = time.perf_counter() - t0
        if dt >= seconds * 0.5 or n >= 1 << 22:
            break
        n = int(n * min(16.0, max(2.0, seconds / max(dt, 1e-3))))
    return {"value": (n / Hq) / dt, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": f"{n} random (query row, q-head) pairs of the {wl.cfg.name} batch, fp64 C++ "
                      f"oracle attention only ({dt:.1f} s; tokens = pairs / Hq)", "seconds": dt}


def W_cpu(wl):
    import workloads as W
    if wl.k_pool.device.type == "cpu":
        return wl
    return W.Workload(wl.cfg, wl.batch, wl.k_pool.cpu(), wl.v_pool.cpu(), wl.free_bits,
                      wl.k_new.cpu(), wl.v_new.cpu(), wl.q.cpu(), wl.head_range, wl.kv_head_range)


def run_reference(args, rank, world):
    """Reference arm: the fp64 CPU oracle (this tier has no reference implementation)."""
    import workloads as W
    if rank != 0:
        return None
    wl = W.make_workload(args.config, device="cpu")
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(wl, per_step * 0.2, seed=1)
    vals, secs = [], 0.0
    last = None
    for s in range(args.steps):
        last = oracle_sample(wl, per_step, seed=100 + s)
        vals.append(last["value"])
        secs += last["seconds"]
    v = statistics.mean(vals)
    cfg = W.get_config(args.config)
    return {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": WORKLOAD_NAMES.get(args.config, args.config), "q_tokens": wl.total_q, "Hq": cfg.Hq, "Hkv": cfg.Hkv,
                   "head_dim": cfg.d},
        "cpu_baseline": dict(last, value=v, cpu_model=cpu_model()),
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_spawn(args):
    """`--gpus N` (N > 1) outside torchrun: re-launch this command under torch.distributed.run
    with N ranks on 127.0.0.1 (one process per GPU) and exit with its status.  Under torchrun
    (WORLD_SIZE set) the world size must equal --gpus.  NCCL init logging goes to stderr so the
    ranks and the transport are on record."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if args.gpus != int(ws) and "--gpus" in " ".join(sys.argv):
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
        return
    if args.gpus <= 1 or args.impl == "reference":
        return
    import subprocess
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    raise SystemExit(subprocess.run(cmd, env=env).returncode)


def dry_run(args, rank, world):
    """--dry-run: the launch / process-group / max-over-ranks plumbing without a GPU (CPU tests
    of the spawn path): every rank contributes its rank to a MAX all-reduce; rank 0 prints."""
    import torch.distributed as dist
    t = torch.tensor([float(rank)])
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "max_rank": int(t.item()),
                          "backend": dist.get_backend() if world > 1 else None}), flush=True)


def main():
    args = parse()
    maybe_spawn(args)
    if args.dry_run:
        rank, world, _ = dist_setup(args, cpu=True)
        dry_run(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    rank, world, local = dist_setup(args)
    res, wl = run_ours(args, rank, world, local)
    if rank == 0:
        if not args.no_cpu_baseline and not args.profile and world == 1:
            res["cpu_baseline"] = oracle_sample(wl, args.cpu_seconds)
            res["cpu_baseline"]["cpu_model"] = cpu_model()
            one = oracle_sample(wl, 3.0, seed=7, nthreads=1)
            res["cpu_baseline"]["one_thread"] = {"value": one["value"], "unit": UNIT, "sample": one["sample"]}
            if not args.no_evict:
                res["cpu_baseline"]["evict_select"] = evict_cpu_timings()
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
