"""World-size-2 gloo tests of the N>1 host logic: head sharding of the seeded
workload, descriptor replication, and the output all-gather used by bench.py.  Each rank runs
the fp64 oracle on its shard as the stand-in for its device; rank 0 checks that the gathered
heads equal the G=1 oracle output bit-exactly (heads are independent, reading #9)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import workloads as W
        from paper_2504_03651_b200 import dist as kdist
        wl = W.make_workload(cfg_name, rank=rank, world=world, preappended=True)
        cfg = W.get_config(cfg_name)
        (q0, q1), (k0, k1) = kdist.head_ranges(cfg.Hq, cfg.Hkv, world, rank)
        assert (q0, q1) == wl.head_range and (k0, k1) == wl.kv_head_range
        # descriptor replicated: every rank sees the same tables
        t = torch.from_numpy(wl.batch["block_table"].astype(np.int64))
        ts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(ts, t)
        assert all(torch.equal(x, t) for x in ts)
        st, out, lse = oracle.attention(wl.batch, wl.k_pool, wl.v_pool, wl.q)
        assert st == oracle.OK
        g = kdist.gather_outputs(torch.from_numpy(out))
        if rank == 0:
            full = W.make_workload(cfg_name, preappended=True)
            st, ref, _ = oracle.attention(full.batch, full.k_pool, full.v_pool, full.q)
            got = kdist.token_major(g).numpy()
            q.put(bool(np.array_equal(got, ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name", ["tiny"])
def test_gloo_world2_sharded_gather(cfg_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, cfg_name, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in ps)
    assert q.get(timeout=5) is True


def test_head_ranges_cover_all_heads():
    from paper_2504_03651_b200.dist import head_ranges
    for Hq, Hkv in [(32, 32), (40, 8), (64, 8)]:
        for G in (1, 2, 4, 8):
            if Hkv % G:
                continue
            qs = [head_ranges(Hq, Hkv, G, r)[0] for r in range(G)]
            assert qs[0][0] == 0 and qs[-1][1] == Hq
            assert all(a[1] == b[0] for a, b in zip(qs, qs[1:]))
    with pytest.raises(ValueError):
        head_ranges(4, 4, 8, 0)


def test_bench_gpus_n_spawns_n_ranks():
    """`python bench.py --gpus 2` outside torchrun re-launches itself under
    torch.distributed.run with 2 ranks (127.0.0.1); --dry-run exercises that launch, the
    process group and the max-over-ranks reduction without a GPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["max_rank"] == 1 and d["backend"] == "gloo"
