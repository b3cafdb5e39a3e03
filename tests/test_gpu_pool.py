"""Device page pool: PagedKvStore's free list
(kv_store.py:103-136) on the device.  Generation reserves each slot's next
page in the seal epilogue, so a decode loop never returns to the host for a
page; an empty pool is a sticky per-slot flag the host maps to
OutOfPagesError (kv_store.py:129-132).

Bars:
  * a pool-managed decode run equals a host-managed one bit for bit in every
    logical quantity (summaries, selections, working sets, attention output);
  * live physical pages are never shared and free + owned == capacity;
  * exhaustion sets pool_oom, leaves every written page untouched (the
    zero-copy audit of kv_store.sealed_versions) and raises OutOfPagesError;
  * released pages are reused.
"""

import numpy as np
import pytest
import torch

from paper_2602_20732_b200.config import preset_config
from paper_2602_20732_b200.engine import ChessDecoder
from paper_2602_20732_b200.errors import OutOfPagesError
from paper_2602_20732_b200.state import DecodeState, Shape

pytestmark = pytest.mark.gpu

B = 16


def _shape(batch=3, n_phys=64, max_pages=40):
    return Shape(batch=batch, layers=2, kv_heads=2, q_heads=4, head_dim=64, page_size=B,
                 pages_per_chunk=4, chunks_per_grid=4, max_pages=max_pages, window_pages=2,
                 max_ws=max_pages, n_phys=n_phys)


def _cfg():
    return preset_config("aggressive", page_size=B, pages_per_chunk=4, chunks_per_grid=4, window_pages=2)


def _inputs(sh, tokens, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    k = (torch.randn((tokens, sh.batch, sh.dim), device="cuda", generator=g) / 8).to(torch.bfloat16)
    v = torch.randn((tokens, sh.batch, sh.dim), device="cuda", generator=g).to(torch.bfloat16)
    q = torch.randn((tokens, sh.batch, sh.layers, sh.q_heads, sh.head_dim), device="cuda",
                    generator=g).to(torch.bfloat16)
    lg = torch.randn((tokens, sh.batch, 1000), device="cuda", generator=g)
    return k, v, q, lg


def _run(st, cfg, inputs, tokens):
    dec = ChessDecoder(st, cfg, policy="always")
    k, v, q, lg = inputs
    outs = torch.zeros((tokens, st.shape.batch, st.shape.layers, st.shape.q_heads, st.shape.head_dim),
                       device="cuda", dtype=torch.bfloat16)
    for t in range(tokens):
        dec.step(k[t], v[t], q[t], lg[t], outs[t])
    torch.cuda.synchronize()
    return outs


def _logical_keys(st, s):
    """Written key rows of slot s in logical order: full sealed pages, then the
    first tail_fill rows of the open page (rows past fill are never written)."""
    n, fill = int(st.num_pages[s]), int(st.tail_fill[s])
    tab = st.page_table[s, :n].long()
    kp = st.k_pool[:, tab]  # [L, n, H, B, d]
    return torch.cat([kp[:, : n - 1].flatten(), kp[:, n - 1, :, :fill].flatten()])


def test_pool_run_matches_host_managed_run():
    sh = _shape()
    cfg = _cfg()
    tokens = 5 * B + 3
    inputs = _inputs(sh, tokens)

    host = DecodeState(sh)
    host.reset()
    # distinct physical runs per slot (each slot uses its first 7 entries)
    host.page_table.copy_(torch.tensor([[(s * 21 + p) % sh.n_phys for p in range(sh.max_pages)]
                                        for s in range(sh.batch)], dtype=torch.int32, device="cuda"))
    out_h = _run(host, cfg, inputs, tokens)

    dev = DecodeState(sh, page_pool=True)
    dev.reset()
    dev.pool_init()
    dev.pool_reserve(1)  # admission: the first page of every slot
    out_d = _run(dev, cfg, inputs, tokens)
    dev.check_pool()

    assert torch.equal(out_h, out_d)
    for name in ("num_pages", "tail_fill", "num_sealed", "n_semantic", "ws_len"):
        assert torch.equal(getattr(host, name), getattr(dev, name)), name
    for s in range(sh.batch):
        n = int(host.num_pages[s])
        assert torch.equal(host.page_vec64[s, :n], dev.page_vec64[s, :n])
        assert torch.equal(host.semantic[s, : int(host.n_semantic[s])], dev.semantic[s, : int(dev.n_semantic[s])])
        assert torch.equal(host.ws_logical[s], dev.ws_logical[s])
        assert torch.equal(_logical_keys(host, s), _logical_keys(dev, s))
    # ownership: every slot owns its pages [0, num_pages) plus the reserved next one
    # when its tail is full; live ids are distinct; free + owned == capacity
    owned = []
    for s in range(sh.batch):
        base, end = int(dev.pool_base[s]), int(dev.pool_end[s])
        assert base == 0 and end >= int(dev.num_pages[s])
        owned += dev.page_table[s, base:end].tolist()
    assert len(owned) == len(set(owned))
    assert dev.pool_free_count() + len(owned) == sh.n_phys


def test_pool_exhaustion_is_out_of_pages_and_leaves_pages_untouched():
    sh = _shape(batch=3, n_phys=7)
    cfg = _cfg()
    tokens = 3 * B
    k, v, q, lg = _inputs(sh, tokens, seed=1)
    st = DecodeState(sh, page_pool=True)
    st.reset()
    st.pool_init()
    st.pool_reserve(1)
    dec = ChessDecoder(st, cfg, policy="always")
    out = torch.zeros((sh.batch, sh.layers, sh.q_heads, sh.head_dim), device="cuda", dtype=torch.bfloat16)
    snapshots = {}
    for t in range(tokens):
        dec.step(k[t], v[t], q[t], lg[t], out)
        torch.cuda.synchronize()
        # zero-copy audit: a written page never changes once sealed
        for s in range(sh.batch):
            for p in range(int(st.num_sealed[s])):
                pid = int(st.page_table[s, p])
                if (s, p) not in snapshots:
                    snapshots[(s, p)] = (pid, st.k_pool[:, pid].clone(), st.v_pool[:, pid].clone())
    for (s, p), (pid, kk, vv) in snapshots.items():
        assert int(st.page_table[s, p]) == pid
        assert torch.equal(st.k_pool[:, pid], kk) and torch.equal(st.v_pool[:, pid], vv)
    # 7 pages for 3 slots x 3 pages (+ reserved next pages): someone ran out
    assert bool(st.pool_oom.any())
    assert st.pool_free_count() == 0
    with pytest.raises(OutOfPagesError):
        st.check_pool()
    # a slot that ran out never wrote past its last reserved page
    for s in range(sh.batch):
        assert int(st.num_pages[s]) <= int(st.pool_end[s])
        assert int(st.token_count[s]) <= B * int(st.pool_end[s])


def test_pool_release_and_reuse():
    sh = _shape(batch=2, n_phys=10)
    cfg = _cfg()
    tokens = 2 * B
    inputs = _inputs(sh, tokens, seed=2)
    st = DecodeState(sh, page_pool=True)
    st.reset()
    st.pool_init()
    st.pool_reserve(1)
    _run(st, cfg, inputs, tokens)
    st.check_pool()
    owned0 = st.page_table[0, : int(st.pool_end[0])].tolist()
    free_before = st.pool_free_count()
    mask = torch.tensor([1, 0], dtype=torch.uint8, device="cuda")
    st.pool_release(mask)
    st.reset(mask)
    torch.cuda.synchronize()
    assert st.pool_free_count() == free_before + len(owned0)
    assert int(st.pool_end[0]) == 0 and int(st.pool_base[0]) == 0
    # slot 0 is re-admitted and gets pages from the released set back
    st.pool_reserve(torch.tensor([3, 0], dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    got = st.page_table[0, :3].tolist()
    assert set(got) <= set(owned0)
    live1 = set(st.page_table[1, : int(st.pool_end[1])].tolist())
    assert not (set(got) & live1)
    # all-or-nothing: asking for more than is free fails without taking any
    free = st.pool_free_count()
    st.pool_reserve(torch.tensor([free + 1, 0], dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    assert st.pool_free_count() == free and bool(st.pool_oom[0])
    with pytest.raises(OutOfPagesError):
        st.check_pool()


def test_pool_requires_pool_buffers():
    st = DecodeState(_shape())
    with pytest.raises(Exception):
        st.pool_init()


def test_evict_and_admit_reuses_slot_and_pages():
    """Continuous batching on the device pool: finish slot 0 mid-run, admit a
    new sequence into it and keep decoding slot 1.  The new sequence equals a
    fresh single-sequence run fed the same tokens (summaries, selections and
    working sets bit for bit, attention within the bf16 bound), slot 1 is
    untouched by the turnover, and the evicted pages are reused."""
    from oracle import attention as attn_ref

    sh = _shape(batch=2, n_phys=40)
    cfg = _cfg()
    t1, t2 = 2 * B + 3, 3 * B + 2
    k1, v1, q1, lg1 = _inputs(sh, t1, seed=4)
    k2, v2, q2, lg2 = _inputs(sh, t2, seed=5)
    st = DecodeState(sh, page_pool=True)
    st.reset()
    st.pool_init()
    dec = ChessDecoder(st, cfg, policy="always")
    dec.admit(torch.ones(2, dtype=torch.uint8, device="cuda"))
    out = torch.zeros((sh.batch, sh.layers, sh.q_heads, sh.head_dim), device="cuda", dtype=torch.bfloat16)
    for t in range(t1):
        dec.step(k1[t], v1[t], q1[t], lg1[t], out)
    torch.cuda.synchronize()
    old_pages = set(st.page_table[0, : int(st.pool_end[0])].tolist())
    slot1_before = st.page_vec64[1].clone()
    m0 = torch.tensor([1, 0], dtype=torch.uint8, device="cuda")
    dec.evict(m0)
    dec.admit(m0)
    outs = torch.zeros((t2,) + out.shape, device="cuda", dtype=torch.bfloat16)
    for t in range(t2):
        dec.step(k2[t], v2[t], q2[t], lg2[t], outs[t])
    torch.cuda.synchronize()
    st.check_pool()
    new_pages = set(st.page_table[0, : int(st.pool_end[0])].tolist())
    assert new_pages & old_pages  # the freed pages came back to slot 0
    n1 = int(st.num_sealed[1])
    # slot 1's earlier pages did not change across the turnover
    n1_before = (t1 // B)
    assert torch.equal(st.page_vec64[1, :n1_before], slot1_before[:n1_before])
    assert n1 == (t1 + t2) // B

    # reference: the same tokens as a fresh single sequence
    sh1 = _shape(batch=1, n_phys=40)
    ref_st = DecodeState(sh1, page_pool=True)
    ref_st.reset()
    ref_st.pool_init()
    rdec = ChessDecoder(ref_st, cfg, policy="always")
    rdec.admit(torch.ones(1, dtype=torch.uint8, device="cuda"))
    routs = torch.zeros((t2, 1) + out.shape[1:], device="cuda", dtype=torch.bfloat16)
    for t in range(t2):
        rdec.step(k2[t][:1], v2[t][:1], q2[t][:1], lg2[t][:1], routs[t])
    torch.cuda.synchronize()
    for name in ("num_pages", "tail_fill", "num_sealed", "n_semantic", "ws_len"):
        assert int(getattr(st, name)[0]) == int(getattr(ref_st, name)[0]), name
    n = int(ref_st.num_sealed[0])
    assert torch.equal(st.page_vec64[0, :n], ref_st.page_vec64[0, :n])
    assert torch.equal(st.anchor[0], ref_st.anchor[0])
    assert torch.equal(st.semantic[0, : int(st.n_semantic[0])], ref_st.semantic[0, : int(ref_st.n_semantic[0])])
    assert torch.equal(st.ws_logical[0, : int(st.ws_len[0])], ref_st.ws_logical[0, : int(ref_st.ws_len[0])])
    assert torch.equal(_logical_keys(st, 0), _logical_keys(ref_st, 0))
    # attention: same math, possibly a different work split across CTAs
    a, b_ = outs[:, 0].float(), routs[:, 0].float()
    assert torch.all((a - b_).abs() <= 2.0**-7 * (b_.abs() + 2.0**-4)), (a - b_).abs().max()
