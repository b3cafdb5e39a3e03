"""Model-driven decode: a random-init Llama-shaped
decoder produces each layer's K/V only after the previous layer's attention,
so the token's append is split by layer (chess_append_kv_layers).

Bars:
  * per-layer appends leave the state bit-identical to one whole-row
    chess_append_kv per token (pages, running key sums, counters, block
    tables), across page seals;
  * with every page in the working set (short sequences: the W-page window
    covers the context), the model's logits through CHESS equal a pure-torch
    dense-attention restatement of the same model within the bf16 bar;
  * the whole token (dense layers + CHESS calls + trigger + seal + selection
    + greedy argmax) replays from one CUDA graph identically to eager steps.
"""

import pytest
import torch

from paper_2602_20732_b200 import _lib
from paper_2602_20732_b200.config import preset_config
from paper_2602_20732_b200.engine import ChessDecoder
from paper_2602_20732_b200.model import LlamaChess, LlamaShape, dense_reference_step
from paper_2602_20732_b200.state import DecodeState, Shape

pytestmark = pytest.mark.gpu

MS = LlamaShape(vocab=512, hidden=256, layers=2, q_heads=8, kv_heads=2, head_dim=64, ffn=512)


def _state(batch, max_pages=16):
    sh = Shape(batch=batch, layers=MS.layers, kv_heads=MS.kv_heads, q_heads=MS.q_heads, head_dim=MS.head_dim,
               page_size=16, pages_per_chunk=4, chunks_per_grid=4, max_pages=max_pages, window_pages=4,
               max_ws=max_pages, n_phys=batch * max_pages)
    st = DecodeState(sh)
    st.reset()
    st.k_pool.zero_()
    st.v_pool.zero_()
    st.page_table.copy_(torch.arange(batch * max_pages, dtype=torch.int32, device="cuda").view(batch, max_pages))
    st.sink_count.fill_(1)
    return st


def test_append_layers_equals_append():
    batch = 3
    a, b = _state(batch), _state(batch)
    D = a.shape.dim
    per = MS.kv_heads * MS.head_dim
    g = torch.Generator(device="cuda").manual_seed(3)
    for t in range(2 * 16 + 5):
        k = torch.randn((batch, D), device="cuda", generator=g).to(torch.bfloat16)
        v = torch.randn((batch, D), device="cuda", generator=g).to(torch.bfloat16)
        _lib.call("chess_append_kv", a.ref, _lib.ptr(k), _lib.ptr(v), D, None, _lib.stream_ptr())
        for li in range(MS.layers):
            kl = k[:, li * per:(li + 1) * per].contiguous()
            vl = v[:, li * per:(li + 1) * per].contiguous()
            _lib.call("chess_append_kv_layers", b.ref, li, li + 1, _lib.ptr(kl), _lib.ptr(vl), per, None,
                      _lib.stream_ptr())
        for st in (a, b):
            _lib.call("chess_summary_seal", st.ref, _lib.stream_ptr())
    torch.cuda.synchronize()
    for name in ("k_pool", "v_pool", "key_sum", "num_pages", "tail_fill", "token_count", "num_sealed",
                 "page_vec64", "chunk_sum64", "grid_sum64", "ws_len", "block_table"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    with pytest.raises(IndexError):
        _lib.call("chess_append_kv_layers", b.ref, 1, 3, _lib.ptr(k), _lib.ptr(v), D, None, _lib.stream_ptr())


def test_model_logits_match_dense_reference():
    torch.manual_seed(0)
    batch, T = 2, 40  # 40 tokens = 2.5 pages: the 4-page window covers the context
    st = _state(batch)
    cfg = preset_config("aggressive", page_size=16, pages_per_chunk=4, chunks_per_grid=4)
    dec = ChessDecoder(st, cfg, policy="every_step")
    model = LlamaChess(MS, dec, seed=1)
    tokens = torch.randint(0, MS.vocab, (T, batch), device="cuda")
    logits = torch.empty((batch, MS.vocab), device="cuda")
    nxt = torch.empty(batch, dtype=torch.int64, device="cuda")
    cache = [(torch.empty((batch, 0, MS.kv_heads, MS.head_dim), dtype=torch.bfloat16, device="cuda"),) * 2
             for _ in range(MS.layers)]
    for t in range(T):
        model.step(tokens[t], logits, nxt)
        pos = torch.full((batch,), t, dtype=torch.int64, device="cuda")
        ref = dense_reference_step(model, cache, tokens[t], pos)
        err = (logits - ref).norm() / ref.norm()
        assert err < 2e-2, (t, float(err))
        assert torch.equal(nxt, logits.argmax(-1))
    assert int(st.token_count[0]) == T and int(st.num_sealed[0]) == T // 16


def test_model_graph_replay_equals_eager():
    batch, T = 2, 24
    runs = []
    for use_graph in (False, True):
        torch.manual_seed(0)
        st = _state(batch)
        cfg = preset_config("aggressive", page_size=16, pages_per_chunk=4, chunks_per_grid=4)
        dec = ChessDecoder(st, cfg, policy="every_step")
        model = LlamaChess(MS, dec, seed=2)
        tok = torch.zeros(batch, dtype=torch.int64, device="cuda")
        logits = torch.empty((batch, MS.vocab), device="cuda")
        nxt = torch.empty(batch, dtype=torch.int64, device="cuda")
        seq = []
        if use_graph:
            model.step(tok, logits, nxt)  # token 0 eagerly, then graph replays
            seq.append(nxt.clone())
            tok.copy_(nxt)
            g = model.capture(tok, logits, nxt)
            # capture() runs one warm-up step itself: that is token 1
            seq.append(nxt.clone())
            tok.copy_(nxt)
            for _ in range(T - 2):
                g.replay()
                seq.append(nxt.clone())
                tok.copy_(nxt)
        else:
            for _ in range(T):
                model.step(tok, logits, nxt)
                seq.append(nxt.clone())
                tok.copy_(nxt)
        torch.cuda.synchronize()
        runs.append((torch.stack(seq), st))
    (sa, a), (sb, b) = runs
    assert torch.equal(sa, sb)
    for name in ("token_count", "num_sealed", "ws_len", "block_table", "k_pool"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
