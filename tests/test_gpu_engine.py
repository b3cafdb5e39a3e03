"""The engine's concurrent step (selection of step t on a side stream next to
step t's L decode launches, working sets deferred to a flush after the join)
gives bit-identical results to the sequential step — eagerly and replayed
from a captured CUDA graph.  Selection of step t only feeds step t+1's
decode (simulate.py:157-182: a re-selection applies to the following page),
so the order inside a step is free once the block-table writes wait for the
decode to finish."""

import pytest
import torch

from paper_2602_20732_b200.config import preset_config
from paper_2602_20732_b200.engine import ChessDecoder
from paper_2602_20732_b200.state import DecodeState, Shape

pytestmark = pytest.mark.gpu

B = 16


def _state(seed):
    sh = Shape(batch=3, layers=2, kv_heads=4, q_heads=8, head_dim=64, page_size=B, pages_per_chunk=4,
               chunks_per_grid=4, max_pages=64, window_pages=2, max_ws=64, n_phys=200)
    st = DecodeState(sh)
    st.reset()
    g = torch.Generator(device="cuda").manual_seed(seed)
    st.k_pool.copy_((torch.randn(st.k_pool.shape, device="cuda", generator=g) / 8).to(torch.bfloat16))
    st.v_pool.copy_(torch.randn(st.v_pool.shape, device="cuda", generator=g).to(torch.bfloat16))
    n_ctx = 24
    st.page_table.copy_(torch.stack([torch.arange(64, dtype=torch.int32) + 64 * s for s in range(3)]).cuda() % 200)
    st.num_pages.fill_(n_ctx)
    st.tail_fill.fill_(B)
    st.token_count.fill_(n_ctx * B)
    st.sink_count.fill_(1)
    return st, n_ctx


def _inputs(sh, tokens, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    k = (torch.randn((tokens, sh.batch, sh.dim), device="cuda", generator=g) / 8).to(torch.bfloat16)
    v = torch.randn((tokens, sh.batch, sh.dim), device="cuda", generator=g).to(torch.bfloat16)
    q = torch.randn((tokens, sh.batch, sh.layers, sh.q_heads, sh.head_dim), device="cuda",
                    generator=g).to(torch.bfloat16)
    lg = torch.randn((tokens, sh.batch, 500), device="cuda", generator=g)
    return k, v, q, lg


@pytest.mark.parametrize("policy,full_scan", [("always", False), ("every_step", False), ("every_step", True)])
@pytest.mark.parametrize("graph", [False, True])
def test_concurrent_step_equals_sequential(policy, full_scan, graph):
    cfg = preset_config("aggressive", page_size=B, pages_per_chunk=4, chunks_per_grid=4, window_pages=2)
    tokens = 2 * B + 5
    runs = []
    for concurrent in (False, True):
        st, n_ctx = _state(seed=1)
        dec = ChessDecoder(st, cfg, policy=policy, concurrent_select=concurrent, full_scan=full_scan)
        dec.build_index(torch.full((3,), n_ctx, dtype=torch.int32, device="cuda"))
        dec.initial_selection()
        k, v, q, lg = _inputs(st.shape, tokens, seed=2)
        outs = torch.zeros((tokens,) + q.shape[1:], device="cuda", dtype=torch.bfloat16)
        if graph:
            # token 0 eagerly (first-launch setup outside capture), then one
            # captured step replayed on static buffers fed per token
            dec.step(k[0], v[0], q[0], lg[0], outs[0])
            sk, sv, sq, slg = k[0].clone(), v[0].clone(), q[0].clone(), lg[0].clone()
            so = torch.zeros_like(outs[0])
            g = dec.capture(sk, sv, sq, slg, so)
            for t in range(1, tokens):
                sk.copy_(k[t])
                sv.copy_(v[t])
                sq.copy_(q[t])
                slg.copy_(lg[t])
                g.replay()
                outs[t].copy_(so)
        else:
            for t in range(tokens):
                dec.step(k[t], v[t], q[t], lg[t], outs[t])
        torch.cuda.synchronize()
        runs.append((st, outs))
    (a, oa), (b, ob) = runs
    assert torch.equal(oa, ob)
    for name in ("num_pages", "num_sealed", "n_semantic", "ws_len", "semantic", "ws_logical",
                 "block_table", "ws_prov", "page_vec64", "anchor", "fire", "gen_pages"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
