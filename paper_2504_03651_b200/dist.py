"""KV-head sharding over G ranks and the output all-gather.

Rank r holds kv-heads [r*Hkv/G, (r+1)*Hkv/G) and the matching q-heads [r*Hq/G, (r+1)*Hq/G);
block ids, tables and the batch descriptor are replicated, so kv_append, hybrid_attention and
evict_select need no communication.  The single exchange is the all-gather of O along heads
(NCCL over NVLink on GPUs; gloo in the CPU tests of this host logic).
"""
from __future__ import annotations

import torch


def head_ranges(Hq: int, Hkv: int, world: int, rank: int):
    """((q_head0, q_head1), (kv_head0, kv_head1)) owned by `rank`."""
    if Hkv % world:
        raise ValueError(f"Hkv={Hkv} does not split over {world} ranks")
    return ((rank * Hq // world, (rank + 1) * Hq // world),
            (rank * Hkv // world, (rank + 1) * Hkv // world))


def gather_outputs(out_local: torch.Tensor, gbuf: torch.Tensor | None = None, group=None):
    """All-gather O [T][Hq/G][d] of every rank into [G][T][Hq/G][d] (rank-major heads: rank r's
    block holds q-heads [r*Hq/G, (r+1)*Hq/G), so no transpose is needed on the device)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if gbuf is None:
        gbuf = torch.empty((world,) + tuple(out_local.shape), dtype=out_local.dtype,
                           device=out_local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(gbuf, out_local.contiguous(), group=group)
    else:  # gloo (CPU tests): list form
        parts = [gbuf[i] for i in range(world)]
        dist.all_gather(parts, out_local.contiguous(), group=group)
    return gbuf


def token_major(gbuf: torch.Tensor) -> torch.Tensor:
    """[G][T][Hl][d] -> [T][G*Hl][d] (a copy; for checks and for consumers needing it)."""
    G, T, Hl, d = gbuf.shape
    return gbuf.permute(1, 0, 2, 3).reshape(T, G * Hl, d)


class FusedGather:
    """a7 fused into the attention epilogues (include/kvattn.h kva_plan_set_outputs, H5): a
    symmetric-memory buffer gbuf [G][T][Hq/G][d] on every rank (torch symmetric memory, NVLink
    peer mappings); this rank's merge / tile / decode epilogues store its head block into slot
    `rank` of EVERY peer's gbuf while the attention runs, instead of an all-gather after it.
    barrier() (a device-side cross-rank barrier on the current stream) then orders the peers'
    reads.  The NCCL all_gather_into_tensor of gather_outputs() is the correctness baseline."""

    def __init__(self, local_shape, dtype, device, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        gname = (group or dist.group.WORLD).group_name
        if hasattr(symm_mem, "enable_symm_mem_for_group"):
            symm_mem.enable_symm_mem_for_group(gname)
        self.buf = symm_mem.empty((self.world,) + tuple(local_shape), dtype=dtype, device=device)
        self.hdl = symm_mem.rendezvous(self.buf, gname)
        self.out_local = self.buf[self.rank]          # this rank's own slot (the plan's `out`)
        slot_bytes = self.out_local.numel() * self.out_local.element_size()
        self.peer_ptrs = [int(self.hdl.buffer_ptrs[p]) + self.rank * slot_bytes
                          for p in range(self.world) if p != self.rank]

    def attach(self, plan):
        """Every later run of `plan` also stores into the peers' slots of this rank."""
        plan.set_extra_outputs(self.peer_ptrs)

    def barrier(self):
        """Device-side: every rank's stores issued before this point are visible after it."""
        self.hdl.barrier(channel=0)
        return self.buf
