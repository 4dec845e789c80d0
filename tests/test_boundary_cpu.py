"""Boundary tests that need no GPU: the C-ABI library loads, exports every symbol declared in
include/kvattn.h, and its host-side validation returns the contract's status codes
(SURVEY §8(b) "Errors"; reading #8) before any device work."""
import os
import re

import numpy as np
import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def K():
    import paper_2504_03651_b200 as K
    K.load()
    return K


def _header_functions():
    src = open(os.path.join(ROOT, "include", "kvattn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:kva_status|const char \*)\s*(\w+)\s*\(", src)))


def test_exports_every_header_symbol(K):
    names = _header_functions()
    assert len(names) >= 15
    lib = K.load()
    for n in names:
        assert hasattr(lib, n), n
    from paper_2504_03651_b200.kvattn import EXPORTS
    assert sorted(EXPORTS) == names


def test_version_names_sm100a(K):
    assert "sm_100a" in K.version()


def test_library_is_sm100a_cubin():
    import subprocess
    from paper_2504_03651_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _batch(K, wl, **over):
    b = dict(wl.batch)
    b.update(over)
    return K.Batch(b, None)


def test_validate_ok_and_errors(K):
    reqs = [W.ReqSpec(W.OFFLINE_PREFILL, 100, 30, 0), W.ReqSpec(W.OFFLINE_DECODE, 90, 1, 0)]
    wl = W.make_workload(W.custom_config("v", 4, 2, 64, 13, reqs, [3]), preappended=True)
    nb = wl.batch["num_blocks"]
    assert K.validate_batch(_batch(K, wl), nb, 0) == K.OK
    # queries inside the group prefix -> ERR_GROUP (reading #8)
    assert K.validate_batch(_batch(K, wl, group_prefix_blocks=np.array([7], np.int32)), nb, 0) == K.ERR_GROUP
    bt = wl.batch["block_table"].copy()
    bt[1, 0] = bt[1, 5]
    assert K.validate_batch(_batch(K, wl, block_table=bt), nb, 0) == K.ERR_GROUP
    # q_len > ctx, Hq % Hkv, head_dim, unallocated block
    assert K.validate_batch(_batch(K, wl, q_indptr=np.array([0, 101, 102], np.int32)), nb, 0) == K.ERR_INVALID
    assert K.validate_batch(_batch(K, wl, num_q_heads=3), nb, 0) == K.ERR_INVALID
    assert K.validate_batch(_batch(K, wl, head_dim=96), nb, 0) == K.ERR_UNSUPPORTED
    bt = wl.batch["block_table"].copy()
    bt[0, 6] = -1
    assert K.validate_batch(_batch(K, wl, block_table=bt), nb, 0) == K.ERR_INVALID
    assert "block_table" in K.last_error()


def test_validate_append_mode_allows_unallocated_new_blocks(K):
    wl = W.make_workload("tiny")   # pre-append: new blocks are -1
    nb = wl.batch["num_blocks"]
    assert K.validate_batch(_batch(K, wl), nb, 1) == K.OK
    assert K.validate_batch(_batch(K, wl), nb, 0) == K.ERR_INVALID  # attention needs them


def test_workspace_sizes_are_host_only(K):
    for name in ["tiny", "llama7b", "qwen14b"]:
        wl = W.make_workload(name) if name == "tiny" else None
        if wl is None:
            continue
        b = _batch(K, wl)
        assert K.hybrid_attention_workspace_size(b) > 0
        assert K.kv_append_workspace_size(b) > 0
    assert K.evict_select_workspace_size(1 << 20, 1 << 16) > (1 << 16) * 12


def test_pool_create_rejects_before_cuda(K):
    import ctypes
    from paper_2504_03651_b200.kvattn import PoolDesc
    L = K.load()
    h = ctypes.c_void_p()
    d = PoolDesc(16, 8, 1, 64, 1024, 2048, 4096, 0)  # block_size 8
    assert L.kv_pool_create(ctypes.byref(d), ctypes.byref(h)) == K.ERR_UNSUPPORTED
    d = PoolDesc(16, 16, 1, 96, 1024, 2048, 4096, 0)  # head_dim 96
    assert L.kv_pool_create(ctypes.byref(d), ctypes.byref(h)) == K.ERR_UNSUPPORTED
    assert L.evict_select(None, -1, 1, None, None, 0, None, None, 0, None) == K.ERR_INVALID


def test_product_does_not_import_oracle():
    """The product package never references oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2504_03651_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f


def test_batch_descriptor_cache_follows_rebinding(K):
    """Batch.desc() is cached (ctypes marshalling per call is host time on the hot path); a
    rebound array is picked up, an in-place write needs no rebuild (same addresses), and the
    validation result follows the data either way."""
    wl = W.make_workload("tiny", preappended=True)
    nb = wl.batch["num_blocks"]
    b = _batch(K, wl)
    d1 = b.desc()
    assert b.desc() is d1 and K.validate_batch(b, nb, 0) == K.OK
    row = b.table_host[0].copy()
    b.table_host[0, 0] = -1                       # in place: same descriptor, new verdict
    assert b.desc() is d1 and K.validate_batch(b, nb, 0) == K.ERR_INVALID
    b.table_host[0] = row
    b.ctx_len = b.ctx_len.copy()                  # rebinding: a new descriptor
    d2 = b.desc()
    assert d2 is not d1 and d2.ctx_len == b.ctx_len.ctypes.data
    assert K.validate_batch(b, nb, 0) == K.OK


def test_workspace_size_validates_groups(K):
    """*_workspace_size runs the call's descriptor checks first: a self- or cyclic parent and an
    out-of-range group_of return ERR_GROUP (the planner walks parent chains and indexes
    per-group arrays; it must never see such a descriptor)."""
    import subprocess
    import sys
    reqs = [W.ReqSpec(W.OFFLINE_DECODE, 100, 1, 0), W.ReqSpec(W.OFFLINE_DECODE, 120, 1, 1)]
    wl = W.make_workload(W.custom_config("wg", 4, 2, 64, 17, reqs, [2, 4], group_parent=[-1, 0]))
    assert K.hybrid_attention_workspace_size(_batch(K, wl)) > 0
    cases = [dict(group_parent=np.array([-1, 1], np.int32)),            # self-parented
             dict(group_parent=np.array([1, 0], np.int32)),             # cycle / later parent
             dict(group_of=np.array([0, 5], np.int32))]                 # group out of range
    code = ("import sys; sys.path.insert(0, %r); import numpy as np, workloads as W, "
            "paper_2504_03651_b200 as K\n" % ROOT +
            "reqs=[W.ReqSpec(W.OFFLINE_DECODE,100,1,0),W.ReqSpec(W.OFFLINE_DECODE,120,1,1)]\n"
            "wl=W.make_workload(W.custom_config('wg',4,2,64,17,reqs,[2,4],group_parent=[-1,0]))\n"
            "for over in %r:\n"
            "    b=dict(wl.batch); b.update({k: np.array(v, np.int32) for k, v in over.items()})\n"
            "    for f in (K.hybrid_attention_workspace_size, K.kv_append_workspace_size):\n"
            "        try:\n"
            "            f(K.Batch(b, None)); print('OK')\n"
            "        except K.KvaError as e:\n"
            "            print(e.status)\n" % [{k: v.tolist() for k, v in c.items()} for c in cases])
    # in a subprocess with a timeout: the bug this guards against was a hang
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    assert r.stdout.split() == [str(K.ERR_GROUP)] * (2 * len(cases)), r.stdout


def test_member_prefix_entries_checked_through_the_first_member(K):
    """Only a group's first member range-checks its prefix entries; another member's prefix
    entries are checked equal to them, so an out-of-range entry there is still rejected."""
    reqs = [W.ReqSpec(W.OFFLINE_DECODE, 90, 1, 0), W.ReqSpec(W.OFFLINE_DECODE, 95, 1, 0),
            W.ReqSpec(W.ONLINE_DECODE, 40, 1)]
    wl = W.make_workload(W.custom_config("m", 4, 2, 64, 15, reqs, [3]), preappended=True)
    nb = wl.batch["num_blocks"]
    assert K.validate_batch(_batch(K, wl), nb, 0) == K.OK
    for row, want in ((1, K.ERR_GROUP), (0, K.ERR_INVALID)):
        bt = wl.batch["block_table"].copy()
        bt[row, 1] = nb + 7
        assert K.validate_batch(_batch(K, wl, block_table=bt), nb, 0) == want, row


def test_options_evict_threads_fold_span_ring(K):
    """kva_set_option: evict_threads accepts 256 / 512 only; fold and span_ring round-trip."""
    try:
        for v in (256, 512):
            K.set_option("evict_threads", v)
            assert K.get_option("evict_threads") == v
        with pytest.raises(K.KvaError):
            K.set_option("evict_threads", 300)
        assert K.get_option("evict_threads") == 512
        for name, v in (("fold", 1), ("fold", 0), ("span_ring", 0)):
            K.set_option(name, v)
            assert K.get_option(name) == v
        with pytest.raises(K.KvaError):
            K.set_option("no_such_option", 1)
    finally:
        K.set_option("evict_threads", 512)
        K.set_option("fold", 0)
