"""Seeded synthetic inputs for the hybrid paged-attention hot path (shared by tests,
bench.py, smoke, the oracle and the CUDA path).

This module holds NO arithmetic of the method: it only draws seeded random numbers and
lays them out (block tables, pools, queries, eviction metadata) in the shapes of the
paper's workloads.  Recipe:

* Structure (block-id permutation, suffix lengths) always comes from a CPU
  ``torch.Generator`` seeded with the config seed, so it is identical on every device.
* Values are i.i.d. N(0,1) fp32 rounded to bf16 (RNE) from a generator on the target
  device, seeded with the config seed; draw order: resident K/V (prefix groups first,
  then requests in order), K_new/V_new, Q.
* Pool = ceil(1.25 x blocks used) blocks; every slot not written is NaN (poison).
* Resident positions [0, ctx - q_len) are in the pool before the step; kv_append writes
  [ctx - q_len, ctx).  Table entries of blocks that start at or after ctx - q_len are -1
  (allocated by kv_append); a partially filled last block is reused (reading #14).

Configs follow BASELINE.json ``configs`` and SURVEY.md §8(d); shapes quote Table 1
(LooGLE 91% / NExT-QA 88% prefix sharing, long offline prompts).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

BLOCK = 16

# request types (descriptor field; planning/metrics only)
ONLINE_DECODE, OFFLINE_PREFILL, OFFLINE_DECODE, ONLINE_PREFILL = 0, 1, 2, 3


@dataclass
class ReqSpec:
    type: int
    ctx: int          # KV length after this step's append
    q_len: int        # query tokens this step (= tokens appended)
    group: int = -1   # shared-prefix group, -1 = none


@dataclass
class Config:
    name: str
    Hq: int
    Hkv: int
    d: int
    seed: int
    reqs: list = field(default_factory=list)
    group_prefix_blocks: list = field(default_factory=list)
    spiky: bool = False
    group_parent: list = field(default_factory=list)  # nested groups: parent index or -1


def _cfg_tiny():
    # BASELINE config 1: 4 heads x d64; 2 online decodes ctx 256; 6 offline chunks of 64
    # sharing a 128-token prefix (chunk at [128,192), reading #30).
    reqs = [ReqSpec(ONLINE_DECODE, 256, 1) for _ in range(2)]
    reqs += [ReqSpec(OFFLINE_PREFILL, 192, 64, 0) for _ in range(6)]
    return Config("tiny", 4, 4, 64, 0, reqs, [8])


def _cfg_llama7b(shared=True):
    # BASELINE config 2: 32/32 x d128; 64 online decodes ctx 2k + 4 offline chunks of 512
    # sharing a 1,536-token prefix (reading #27).
    reqs = [ReqSpec(ONLINE_DECODE, 2048, 1) for _ in range(64)]
    reqs += [ReqSpec(OFFLINE_PREFILL, 2048, 512, 0 if shared else -1) for _ in range(4)]
    return Config("llama7b" if shared else "llama7b-u", 32, 32, 128, 1, reqs,
                  [96] if shared else [])


def _cfg_qwen14b(shared=True):
    # BASELINE config 3: 40/8 x d128; 32 online decodes ctx 2k + 256 offline decodes sharing
    # a 2k prefix with private suffixes U{32..256} incl. the new token (reading #28).
    # suffix lengths: their own CPU generator (seed 2), independent of the block permutation
    suffix = torch.randint(32, 257, (256,), generator=torch.Generator("cpu").manual_seed(2))
    reqs = [ReqSpec(ONLINE_DECODE, 2048, 1) for _ in range(32)]
    reqs += [ReqSpec(OFFLINE_DECODE, 2048 + int(s), 1, 0 if shared else -1) for s in suffix]
    return Config("qwen14b" if shared else "qwen14b-u", 40, 8, 128, 2, reqs,
                  [128] if shared else [])


def _cfg_qwen14b_prefill(shared=True):
    # SURVEY §8(f) NEXT-4, variant 3b of BASELINE config 3: the same 256 offline tasks, each
    # PREFILLING its private suffix U{32..256} (q_len = suffix) under the shared 2k prompt
    # prefix (Table 1: a shared document, private question), + 32 online decodes.
    # The cascade part is tensor-bound here (every member's suffix rows x the 2k prefix).
    suffix = torch.randint(32, 257, (256,), generator=torch.Generator("cpu").manual_seed(2))
    reqs = [ReqSpec(ONLINE_DECODE, 2048, 1) for _ in range(32)]
    reqs += [ReqSpec(OFFLINE_PREFILL, 2048 + int(s), int(s), 0 if shared else -1) for s in suffix]
    return Config("qwen14b-p" if shared else "qwen14b-pu", 40, 8, 128, 2, reqs,
                  [128] if shared else [])


def _cfg_llama70b():
    # BASELINE config 5: 64/8 x d128; 32 online decodes ctx 32k + 2 offline 8k chunks at
    # [8192, 16384) sharing an 8k prefix (reading #29).
    reqs = [ReqSpec(ONLINE_DECODE, 32768, 1) for _ in range(32)]
    reqs += [ReqSpec(OFFLINE_PREFILL, 16384, 8192, 0) for _ in range(2)]
    return Config("llama70b", 64, 8, 128, 4, reqs, [512])


CONFIGS = {
    "tiny": _cfg_tiny,
    "llama7b": lambda: _cfg_llama7b(True),
    "llama7b-u": lambda: _cfg_llama7b(False),
    "qwen14b": lambda: _cfg_qwen14b(True),
    "qwen14b-u": lambda: _cfg_qwen14b(False),
    "llama70b": _cfg_llama70b,
    "qwen14b-p": lambda: _cfg_qwen14b_prefill(True),
    "qwen14b-pu": lambda: _cfg_qwen14b_prefill(False),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]()


def custom_config(name, Hq, Hkv, d, seed, reqs, group_prefix_blocks, spiky=False, group_parent=None) -> Config:
    return Config(name, Hq, Hkv, d, seed, list(reqs), list(group_prefix_blocks), spiky, list(group_parent or []))


def _parent(cfg: Config, g: int) -> int:
    return cfg.group_parent[g] if cfg.group_parent else -1


@dataclass
class Workload:
    cfg: Config
    batch: dict          # host numpy descriptor (see oracle.attention for keys)
    k_pool: torch.Tensor  # bf16 [num_blocks][Hkv_local][16][d]  (pre-append state)
    v_pool: torch.Tensor
    free_bits: np.ndarray  # uint32 words, bit b = block b free (pre-append state)
    k_new: torch.Tensor    # bf16 [total_q][Hkv_local][d]
    v_new: torch.Tensor
    q: torch.Tensor        # bf16 [total_q][Hq_local][d]
    head_range: tuple      # (q_head0, q_head1) of the full model this rank holds
    kv_head_range: tuple

    @property
    def total_q(self):
        return int(self.batch["q_indptr"][-1])


def _blocks_used(cfg: Config):
    """Blocks the step touches: prefixes + private blocks up to ctx (incl. appended)."""
    n = sum(np_ - (cfg.group_prefix_blocks[_parent(cfg, g)] if _parent(cfg, g) >= 0 else 0)
            for g, np_ in enumerate(cfg.group_prefix_blocks))
    for r in cfg.reqs:
        start = cfg.group_prefix_blocks[r.group] * BLOCK if r.group >= 0 else 0
        n += math.ceil(r.ctx / BLOCK) - start // BLOCK
    return n


def _fill(pool, blk_ids, offs, gen, Hkv, d, device, chunk_tokens=1 << 16):
    """Write N(0,1)->bf16 rows into pool[blk, :, off, :] for the given slots, in order."""
    n = len(blk_ids)
    for s in range(0, n, chunk_tokens):
        e = min(n, s + chunk_tokens)
        vals = torch.randn((e - s, Hkv, d), generator=gen, device=device, dtype=torch.float32)
        bi = torch.as_tensor(blk_ids[s:e], device=device, dtype=torch.long)
        oi = torch.as_tensor(offs[s:e], device=device, dtype=torch.long)
        pool[bi, :, oi, :] = vals.to(torch.bfloat16)


def make_workload(cfg: Config | str, device="cpu", rank: int = 0, world: int = 1,
                  pool_scale: float = 1.25, preappended: bool = False) -> Workload:
    """Build the pre-append state of one step for ``cfg`` on ``device``.

    With world > 1, rank r keeps kv-heads [r*Hkv/G, (r+1)*Hkv/G) and the matching q-heads
    (SURVEY §8(e)); block ids, tables and the descriptor are replicated.  Values are drawn
    for the FULL model and sliced, so every G sees identical bytes.
    """
    if isinstance(cfg, str):
        cfg = get_config(cfg)
    device = torch.device(device)
    Hq, Hkv, d = cfg.Hq, cfg.Hkv, cfg.d
    if Hkv % world:
        raise ValueError(f"{cfg.name}: Hkv={Hkv} does not split over {world} ranks")
    R = len(cfg.reqs)
    used = _blocks_used(cfg)
    num_blocks = int(math.ceil(pool_scale * used))
    gs = torch.Generator("cpu").manual_seed(cfg.seed)
    perm = torch.randperm(num_blocks, generator=gs).numpy().astype(np.int32)
    nxt = 0

    max_ctx = max(r.ctx for r in cfg.reqs)
    max_blocks = math.ceil(max_ctx / BLOCK)
    table = np.full((R, max_blocks), -1, np.int32)
    # group prefixes first
    gblocks = []
    for g, np_ in enumerate(cfg.group_prefix_blocks):
        p = _parent(cfg, g)
        if p >= 0:  # nested group: the parent's blocks, then its own
            if p >= g or cfg.group_prefix_blocks[p] > np_:
                raise ValueError("group_parent must point to an earlier group with a shorter prefix")
            npp = cfg.group_prefix_blocks[p]
            gblocks.append(np.concatenate([gblocks[p][:npp], perm[nxt:nxt + np_ - npp]]))
            nxt += np_ - npp
        else:
            gblocks.append(perm[nxt:nxt + np_].copy())
            nxt += np_
    # resident private blocks per request (positions [start_private, ctx - q_len))
    for i, r in enumerate(cfg.reqs):
        npfx = cfg.group_prefix_blocks[r.group] if r.group >= 0 else 0
        table[i, :npfx] = gblocks[r.group][:npfx] if r.group >= 0 else []
        resident = r.ctx if preappended else r.ctx - r.q_len
        if r.ctx - r.q_len < npfx * BLOCK:
            raise ValueError("group member queries must follow the prefix (reading #8)")
        nres = math.ceil(resident / BLOCK)
        for b in range(npfx, nres):
            table[i, b] = perm[nxt]
            nxt += 1
    assert nxt <= num_blocks
    free = np.ones(num_blocks, bool)
    used_ids = table[table >= 0]
    free[used_ids] = False
    words = (num_blocks + 31) // 32
    free_bits = np.zeros(words, np.uint32)
    idx = np.nonzero(free)[0]
    np.bitwise_or.at(free_bits, idx // 32, (np.uint32(1) << (idx % 32).astype(np.uint32)))

    # ---- values (full model heads, then slice) ----
    gv = torch.Generator(device).manual_seed(cfg.seed)
    kvh0, kvh1 = rank * Hkv // world, (rank + 1) * Hkv // world
    qh0, qh1 = rank * Hq // world, (rank + 1) * Hq // world
    nan = float("nan")
    k_pool = torch.full((num_blocks, Hkv, BLOCK, d), nan, dtype=torch.bfloat16, device=device)
    v_pool = torch.full((num_blocks, Hkv, BLOCK, d), nan, dtype=torch.bfloat16, device=device)

    def slots(blks, n_tok, t0=0):
        ts = np.arange(t0, n_tok)
        return blks[ts // BLOCK], ts % BLOCK

    for gi, np_ in enumerate(cfg.group_prefix_blocks):
        p = _parent(cfg, gi)
        t0 = cfg.group_prefix_blocks[p] * BLOCK if p >= 0 else 0  # the parent filled its part
        bi, oi = slots(gblocks[gi], np_ * BLOCK, t0)
        _fill(k_pool, bi, oi, gv, Hkv, d, device)
        _fill(v_pool, bi, oi, gv, Hkv, d, device)
    for i, r in enumerate(cfg.reqs):
        npfx = cfg.group_prefix_blocks[r.group] if r.group >= 0 else 0
        resident = r.ctx if preappended else r.ctx - r.q_len
        if resident > npfx * BLOCK:
            bi, oi = slots(table[i], resident, npfx * BLOCK)
            _fill(k_pool, bi, oi, gv, Hkv, d, device)
            _fill(v_pool, bi, oi, gv, Hkv, d, device)
    q_indptr = np.zeros(R + 1, np.int32)
    q_indptr[1:] = np.cumsum([r.q_len for r in cfg.reqs])
    total_q = int(q_indptr[-1])
    k_new = torch.randn((total_q, Hkv, d), generator=gv, device=device).to(torch.bfloat16)
    v_new = torch.randn((total_q, Hkv, d), generator=gv, device=device).to(torch.bfloat16)
    qf = torch.randn((total_q, Hq, d), generator=gv, device=device)
    if cfg.spiky:
        qf = qf * 8.0
    q = qf.to(torch.bfloat16)

    if world > 1:
        k_pool = k_pool[:, kvh0:kvh1].contiguous()
        v_pool = v_pool[:, kvh0:kvh1].contiguous()
        k_new = k_new[:, kvh0:kvh1].contiguous()
        v_new = v_new[:, kvh0:kvh1].contiguous()
        q = q[:, qh0:qh1].contiguous()

    batch = dict(
        num_reqs=R, num_q_heads=qh1 - qh0, num_kv_heads=kvh1 - kvh0, head_dim=d,
        req_type=np.array([r.type for r in cfg.reqs], np.int32),
        q_indptr=q_indptr,
        ctx_len=np.array([r.ctx for r in cfg.reqs], np.int32),
        block_table=table,
        group_of=np.array([r.group for r in cfg.reqs], np.int32),
        group_prefix_blocks=np.array(cfg.group_prefix_blocks, np.int32),
        group_parent=np.array(cfg.group_parent, np.int32) if cfg.group_parent else None,
        num_blocks=num_blocks,
        sm_scale=0.0,
    )
    return Workload(cfg, batch, k_pool, v_pool, free_bits, k_new, v_new, q,
                    (qh0, qh1), (kvh0, kvh1))


# ---------------------------------------------------------------------------------------
# Eviction metadata (BASELINE config 4; SURVEY §8(d) `evict`)
# ---------------------------------------------------------------------------------------
EV_FREE, EV_RUNNING_ONLINE, EV_PINNED, EV_ACTIVE_OFFLINE, EV_FINISHED_ONLINE, EV_FINISHED_OFFLINE = range(6)


@dataclass
class EvictWorkload:
    state: np.ndarray   # uint8 [N]
    rc: np.ndarray      # uint32 [N]
    lat: np.ndarray     # uint32 [N]
    depth: np.ndarray   # uint16 [N]
    k: int
    run_start: np.ndarray  # per-run first index into `order`
    order: np.ndarray      # block ids of resident runs, run-major


def make_evict(n: int = 1 << 20, k: int = 1 << 16, seed: int = 3, free_frac: float = 0.10,
               mix=(0.10, 0.05, 0.40, 0.15, 0.30), run_lo: int = 16, run_hi: int = 128,
               straddle: bool = False) -> EvictWorkload:
    """1M-block pool at 90% occupancy in runs (request chains) of U{16..128} blocks.

    Run classes: running-online / pinned / active-offline (rc = min(256, Zipf(1.5))) /
    finished-online / finished-offline; lat per run U[0, 2^20); depth = position in run.
    ``straddle`` sets finished-offline to 3% so k crosses into the 0.5 class.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    if straddle:
        mix = (0.10, 0.05, 0.40, 0.42, 0.03)
    perm = rng.permutation(n).astype(np.int32)
    nfree = int(round(free_frac * n))
    state = np.zeros(n, np.uint8)
    rc = np.zeros(n, np.uint32)
    lat = np.zeros(n, np.uint32)
    depth = np.zeros(n, np.uint16)
    resident = perm[nfree:]
    lens = []
    tot = 0
    while tot < len(resident):
        L = int(rng.integers(run_lo, run_hi + 1))
        L = min(L, len(resident) - tot)
        lens.append(L)
        tot += L
    lens = np.array(lens, np.int64)
    nr = len(lens)
    classes = rng.choice(5, size=nr, p=np.array(mix) / sum(mix)) + 1   # states 1..5
    rcs = np.minimum(256, rng.zipf(1.5, size=nr)).astype(np.uint32)
    lats = rng.integers(0, 1 << 20, size=nr).astype(np.uint32)
    run_start = np.concatenate([[0], np.cumsum(lens)[:-1]])
    run_of = np.repeat(np.arange(nr), lens)
    pos = np.arange(len(resident)) - run_start[run_of]
    state[resident] = classes[run_of]
    r_rc = np.where(classes[run_of] == EV_ACTIVE_OFFLINE, rcs[run_of], 0).astype(np.uint32)
    rc[resident] = r_rc
    lat[resident] = lats[run_of]
    depth[resident] = pos.astype(np.uint16)
    return EvictWorkload(state, rc, lat, depth, k, run_start, resident)


def retouch(ev: EvictWorkload, now: int, frac: float = 0.05, seed: int = 0):
    """Between iterations: set lat = now for a random 5% of runs (LRU refresh)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nr = len(ev.run_start)
    pick = rng.choice(nr, size=max(1, int(frac * nr)), replace=False)
    ends = np.concatenate([ev.run_start[1:], [len(ev.order)]])
    for r in pick:
        ev.lat[ev.order[ev.run_start[r]:ends[r]]] = now


def make_manager_update(ev: EvictWorkload, now: int, seed: int = 0, touch_frac: float = 0.05,
                        finish_frac: float = 0.01):
    """One KV-manager iteration over the `evict` metadata: returns
    (chains, pool) with chains = [(state, ids)] (host) and pool = [ids] (the offline pool's
    prompt chains).  The pool reproduces the drawn rc exactly: an active-offline run with
    rc = r is the prefix chain of r pool requests ("how many offline requests ... will
    reuse it").  Transitions: a random touch_frac of runs keep their class with lat = now
    (LRU refresh); finish_frac of runs change class (running online -> finished online,
    pinned -> finished offline).  No method arithmetic here: only seeded choices."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nr = len(ev.run_start)
    ends = np.concatenate([ev.run_start[1:], [len(ev.order)]])
    runs = [ev.order[ev.run_start[r]:ends[r]] for r in range(nr)]
    pool = []
    for r in range(nr):
        b0 = runs[r][0]
        if ev.state[b0] == EV_ACTIVE_OFFLINE:
            pool.extend([runs[r]] * int(ev.rc[b0]))
    chains = []
    for r in rng.choice(nr, size=max(1, int(touch_frac * nr)), replace=False):
        chains.append((int(ev.state[runs[r][0]]), runs[r]))
    for r in rng.choice(nr, size=max(1, int(finish_frac * nr)), replace=False):
        s = int(ev.state[runs[r][0]])
        if s == 1:
            chains.append((4, runs[r]))
        elif s == 2:
            chains.append((5, runs[r]))
    return chains, pool
