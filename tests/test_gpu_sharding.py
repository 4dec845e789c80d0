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
