"""KV-head sharding on the real kernels (reading #9, H9): for G = 2, 4, 8 every
rank's shard (its kv-heads and q-heads, replicated tables) is run through the library on this
GPU, one rank after another, and the head-concatenated outputs must equal the G = 1 output
BIT-EXACTLY (fixed splits, per-head independence); block tables are identical on every rank.
The NCCL all-gather that joins the shards on a multi-GPU box is a byte copy (bench.py)."""
import numpy as np
import pytest
import torch

import workloads as W

from gpu_util import gpu_step

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,worlds", [("tiny", (2, 4)), ("qwen14b", (2, 4, 8)), ("llama7b", (2, 4, 8))])
def test_shards_concatenate_to_g1_bitexact(name, worlds):
    full = gpu_step(W.make_workload(name, device="cuda"), out_dtype=torch.bfloat16)
    ref, ref_lse = full["out"].cpu(), full["lse"].cpu()
    ref_bt = full["batch"].table_dev.cpu().numpy()
    for G in worlds:
        outs, lses = [], []
        for r in range(G):
            g = gpu_step(W.make_workload(name, device="cuda", rank=r, world=G), out_dtype=torch.bfloat16)
            assert np.array_equal(g["batch"].table_dev.cpu().numpy(), ref_bt), (G, r)
            outs.append(g["out"].cpu())
            lses.append(g["lse"].cpu())
            del g
            torch.cuda.empty_cache()
        assert torch.equal(torch.cat(outs, dim=1), ref), G
        assert torch.equal(torch.cat(lses, dim=1), ref_lse), G


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_fused_gather_epilogue_stores_every_destination(out_dtype):
    """kva_plan_set_outputs (a7 fused into the epilogues): with kv-head shards G = 2 on one GPU
    and each shard's plan given the OTHER shard's slot of a second gathered buffer as an extra
    destination (what the peers' NVLink mappings are on a node), both gathered buffers end up
    bit-identical to the concatenation of the shards' own outputs — decode-direct, tile-direct
    and merged rows alike (tiny: online decodes, chunks, a shared-prefix group)."""
    import paper_2504_03651_b200 as K
    G = 2
    outs = []
    wl0 = W.make_workload("tiny", rank=0, world=G)
    T, Hl, d = wl0.q.shape
    gbufs = [torch.full((G, T, Hl, d), float("nan"), dtype=out_dtype, device="cuda") for _ in range(G)]
    for r in range(G):
        wl = W.make_workload("tiny", rank=r, world=G)
        g = gpu_step(wl, out_dtype=out_dtype)
        outs.append(g["out"])
        # rank r's run again, now storing into its slot of BOTH gathered buffers
        plan = g["plan"]
        plan.set_extra_outputs([gbufs[1 - r][r]])
        plan.run(g["q"], gbufs[r][r])
        torch.cuda.synchronize()
    for p in range(G):
        for r in range(G):
            a = gbufs[p][r].cpu().view(torch.int16 if out_dtype == torch.bfloat16 else torch.int32)
            b = outs[r].cpu().view(torch.int16 if out_dtype == torch.bfloat16 else torch.int32)
            assert torch.equal(a, b), (p, r)


def test_fused_gather_symmetric_memory_one_rank():
    """dist.FusedGather through torch symmetric memory on a 1-rank NCCL group (the API path a
    multi-GPU node uses: allocation, rendezvous, peer pointers, device-side barrier): the
    gathered buffer holds exactly the plan's output."""
    import os
    import socket
    import torch.distributed as dist
    import paper_2504_03651_b200 as K
    from paper_2504_03651_b200 import dist as kdist
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        wl = W.make_workload("tiny")
        g = gpu_step(wl, out_dtype=torch.bfloat16)
        T, Hl, d = g["out"].shape
        try:
            fg = kdist.FusedGather((T, Hl, d), torch.bfloat16, torch.device("cuda", 0))
        except Exception as e:  # symmetric memory unavailable in this build / driver
            pytest.skip(f"symmetric memory unavailable: {e}")
        assert fg.peer_ptrs == [] and fg.buf.shape == (1, T, Hl, d)
        fg.attach(g["plan"])
        g["plan"].run(g["q"], fg.out_local)
        fg.barrier()
        torch.cuda.synchronize()
        assert torch.equal(fg.buf[0].view(torch.int16), g["out"].view(torch.int16))
    finally:
        dist.destroy_process_group()
