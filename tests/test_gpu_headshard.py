"""KV-head shard on one GPU: several rank states in one
process, each holding kv heads [r*H/n, (r+1)*H/n) of every layer.

The score of a summary row is a sum over the (layer, head) column slices of
the flattened key row (selection.py:62-74), so each rank's scan yields a
PARTIAL score; chess_select_partial exports it, the exchange all-gathers it
and chess_select_combine adds the partials in rank order.  Bars:
  * every rank's semantic set / working set / block table is bit-identical;
  * they equal the oracle's selection on the unsharded f64 index;
  * a full decode step of the rank states (engine.ChessDecoder with a
    HeadShardExchange whose all-gather is a thread-barrier stand-in for
    NCCL) reproduces the unsharded state's selections and block tables bit
    for bit, and its attention output head block by head block within the
    bf16 bar of the attention tests.
"""

import ctypes
import threading

import numpy as np
import pytest
import torch

from oracle import pagesel_ref as ref
from paper_2602_20732_b200 import _lib
from paper_2602_20732_b200.config import SelectionConfig, preset_config
from paper_2602_20732_b200.engine import ChessDecoder
from paper_2602_20732_b200.parallel import HeadShard, HeadShardExchange, PeerScoreExchange
from paper_2602_20732_b200.state import DecodeState, Shape

pytestmark = pytest.mark.gpu


def _levels(full_scan):
    return [3] if full_scan else [0, 1, 2]


def _select_sharded(states, cfg, full_scan, exchanges):
    """Drive the cascade level by level across in-process rank states."""
    sc = _lib.ChessSelectCfg(cfg.rho_grid, cfg.rho_chunk, cfg.rho_page, int(full_scan), 1)
    world = len(states)
    for lv in _levels(full_scan):
        for st, x in zip(states, exchanges):
            _lib.call("chess_select_partial", st.ref, ctypes.byref(sc), lv, _lib.ptr(x.partial[lv]),
                      x.ld[lv], _lib.stream_ptr())
        gathered = torch.stack([x.partial[lv] for x in exchanges])
        for st, x in zip(states, exchanges):
            _lib.call("chess_select_combine", st.ref, ctypes.byref(sc), lv, _lib.ptr(gathered),
                      world, x.ld[lv], _lib.stream_ptr())
    torch.cuda.synchronize()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("full_scan", [False, True])
@pytest.mark.parametrize("summary_dtype", ["f32", "f64"])
def test_head_shard_selection_matches_oracle(world, full_scan, summary_dtype):
    from helpers import load_vectors, read_selection, set_tables

    rng = np.random.default_rng(5 + world)
    L, H, d = 3, 8, 16
    D = L * H * d
    batch = 3
    for trial in range(6):
        cfg = SelectionConfig(pages_per_chunk=int(rng.integers(2, 9)), chunks_per_grid=int(rng.integers(2, 9)),
                              rho_grid=0.5, rho_chunk=0.2, rho_page=0.1,
                              window_pages=4, sink_pages=1)
        max_pages = 700
        states, exchanges, shards = [], [], []
        for r in range(world):
            sh = HeadShard(r, world, L, H, H, d)
            shape = Shape(batch=batch, layers=L, kv_heads=H // world, q_heads=H // world, head_dim=d,
                          page_size=cfg.page_size, pages_per_chunk=cfg.pages_per_chunk,
                          chunks_per_grid=cfg.chunks_per_grid, max_pages=max_pages,
                          window_pages=cfg.window_pages, max_ws=max_pages, n_phys=1,
                          summary_dtype=summary_dtype)
            states.append(DecodeState(shape))
            shards.append(sh)
            exchanges.append(HeadShardExchange(sh, batch, max_pages, cfg.pages_per_chunk,
                                               cfg.chunks_per_grid, "cuda", full_scan=full_scan,
                                               allgather=lambda o, i: None))
        hs = []
        for slot in range(batch):
            n = int(rng.integers(1, 650))
            rows = rng.standard_normal((n, D))
            for st, sh in zip(states, shards):
                load_vectors(st, slot, rows[:, sh.flat_columns().numpy()])
                set_tables(st, slot, n + 1, cfg.sink_pages)
            hs.append((ref.Hierarchy.from_rows(rows, cfg.pages_per_chunk, cfg.chunks_per_grid), n))
        _select_sharded(states, cfg, full_scan, exchanges)
        for slot, (h, n) in enumerate(hs):
            a, _ = ref.anchor(h.page_vectors, cfg.window_pages)
            s = [m @ a for m in (h.grid_vectors, h.chunk_vectors, h.page_vectors)]
            p2c, c2g = h.parent_maps()
            sel, _ = ref.prune(s[0], s[1], s[2], p2c, c2g, cfg.ratios)
            pages, _ = ref.working_set(sel, n + 1, cfg.window_pages, cfg.sink_pages)
            got0 = read_selection(states[0], slot)
            np.testing.assert_array_equal(got0[0], sel, err_msg=f"trial {trial} slot {slot} P={n}")
            np.testing.assert_array_equal(got0[1], pages)
            for st in states[1:]:
                got = read_selection(st, slot)
                for x, y in zip(got0, got):
                    np.testing.assert_array_equal(x, y)


def test_exchange_validation():
    cfg = preset_config("aggressive", page_size=16)
    shape = Shape(batch=2, layers=1, kv_heads=1, q_heads=1, head_dim=8, page_size=16,
                  pages_per_chunk=8, chunks_per_grid=8, max_pages=100, window_pages=4,
                  max_ws=100, n_phys=1)
    st = DecodeState(shape)
    sc = _lib.ChessSelectCfg(cfg.rho_grid, cfg.rho_chunk, cfg.rho_page, 0, 1)
    buf = torch.zeros((2, 100), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):  # conditional scan has no level 3
        _lib.call("chess_select_partial", st.ref, ctypes.byref(sc), 3, _lib.ptr(buf), 100, None)
    with pytest.raises(ValueError):  # page level needs max_pages columns
        _lib.call("chess_select_partial", st.ref, ctypes.byref(sc), 2, _lib.ptr(buf), 99, None)
    with pytest.raises(ValueError):
        _lib.call("chess_select_combine", st.ref, ctypes.byref(sc), 0, _lib.ptr(buf), 0, 100, None)


class _ThreadAllGather:
    """In-process stand-in for NCCL all_gather_into_tensor across rank threads."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.inputs = [None] * world

    def for_rank(self, rank):
        def allgather(out, inp):
            torch.cuda.current_stream().synchronize()
            self.inputs[rank] = inp
            self.barrier.wait()
            for r in range(self.world):
                if out[r].data_ptr() != self.inputs[r].data_ptr():
                    out[r].copy_(self.inputs[r])
            torch.cuda.current_stream().synchronize()
            self.barrier.wait()

        return allgather


@pytest.mark.parametrize("transport", ["nccl", "p2p", "p2p_scores"])
@pytest.mark.parametrize("world", [2, 4])
def test_head_shard_decode_step_matches_unsharded(world, transport):
    """Whole engine step: append -> L x (K4 + output gather) -> entropy ->
    seal -> level-by-level selection with the score exchange."""
    torch.manual_seed(world)
    cfg = preset_config("aggressive", page_size=16)
    L, H, Hq, d, B = 2, 8, 16, 64, 16
    batch, n_ctx, max_pages, n_phys = 2, 96, 140, 300
    full_shape = Shape(batch=batch, layers=L, kv_heads=H, q_heads=Hq, head_dim=d, page_size=B,
                       pages_per_chunk=8, chunks_per_grid=8, max_pages=max_pages, window_pages=4,
                       max_ws=max_pages, n_phys=n_phys)
    k_pool = (torch.randn((L, n_phys, H, B, d), device="cuda") / 8).to(torch.bfloat16)
    v_pool = torch.randn((L, n_phys, H, B, d), device="cuda").to(torch.bfloat16)
    # a planted direction on a few pages so the selection is not pure noise
    sig = torch.randn((L, H, d), device="cuda")
    k_pool[:, 40:44] += (0.5 * sig[:, None, :, None, :]).to(torch.bfloat16)
    table = torch.stack([torch.arange(max_pages) + 150 * s for s in range(batch)]) % n_phys

    def setup(shape, kp, vp):
        st = DecodeState(shape, kv_pool=(kp, vp))
        st.reset()
        st.page_table.copy_(table.to(torch.int32))
        st.num_pages.fill_(n_ctx)
        st.tail_fill.fill_(B)
        st.token_count.fill_(n_ctx * B)
        st.sink_count.fill_(1)
        return st

    full = setup(full_shape, k_pool.clone(), v_pool.clone())
    k_new = (torch.randn((3, batch, L, H, d), device="cuda") / 8).to(torch.bfloat16)
    v_new = torch.randn((3, batch, L, H, d), device="cuda").to(torch.bfloat16)
    q = torch.randn((3, batch, L, Hq, d), device="cuda").to(torch.bfloat16)
    logits = torch.randn((3, batch, 32000), device="cuda")
    n_now = torch.full((batch,), n_ctx, dtype=torch.int32, device="cuda")

    dec_full = ChessDecoder(full, cfg, policy="every_step")
    dec_full.build_index(n_now)
    dec_full.initial_selection()
    out_full = torch.zeros((3, batch, L, Hq, d), device="cuda", dtype=torch.bfloat16)
    for t in range(3):
        dec_full.step(k_new[t].reshape(batch, -1), v_new[t].reshape(batch, -1), q[t], logits[t], out_full[t])
    torch.cuda.synchronize()

    hk, hq = H // world, Hq // world
    group = _ThreadAllGather(world)
    results = [None] * world
    errors = []
    # p2p: the score exchange over peer pointers (here: one device, in-process
    # ranks on their own streams, so a pull really waits for another rank's push)
    # p2p also gathers the outputs from K4's epilogue; p2p_scores keeps the
    # per-layer all-gather for them
    p2p = transport != "nccl"
    xs = [PeerScoreExchange(HeadShard(r, world, L, H, Hq, d), batch, max_pages, 8, 8, "cuda",
                            allgather=group.for_rank(r), fused_outputs=transport == "p2p")
          if p2p else
          HeadShardExchange(HeadShard(r, world, L, H, Hq, d), batch, max_pages, 8, 8, "cuda",
                            allgather=group.for_rank(r))
          for r in range(world)]
    if p2p:
        for x in xs:
            x.connect_local(xs)
    streams = [torch.cuda.Stream() for _ in range(world)]

    def rank_main(r):
        try:
            with torch.cuda.stream(streams[r]):
                rank_body(r)
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            group.barrier.abort()

    def rank_body(r):
        shape = Shape(**{**full_shape.__dict__, "kv_heads": hk, "q_heads": hq})
        st = setup(shape, k_pool[:, :, r * hk:(r + 1) * hk].contiguous(),
                   v_pool[:, :, r * hk:(r + 1) * hk].contiguous())
        x = xs[r]
        dec = ChessDecoder(st, cfg, policy="every_step", exchange=x)
        dec.build_index(n_now)
        dec.initial_selection()
        out = torch.zeros((3, L, world, batch, hq, d), device="cuda", dtype=torch.bfloat16)
        for t in range(3):
            kl = k_new[t][:, :, r * hk:(r + 1) * hk].reshape(batch, -1).contiguous()
            vl = v_new[t][:, :, r * hk:(r + 1) * hk].reshape(batch, -1).contiguous()
            ql = q[t][:, :, r * hq:(r + 1) * hq].contiguous()
            dec.step(kl, vl, ql, logits[t], out[t])
        torch.cuda.synchronize()
        if p2p:
            x.check()
        results[r] = (st, out)

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    for x in xs:
        if p2p:
            x.close()
    for r, (st, out) in enumerate(results):
        for s in range(batch):
            for name in ("semantic", "ws_logical", "block_table"):
                n = int(getattr(full, "n_semantic" if name == "semantic" else "ws_len")[s])
                assert torch.equal(getattr(st, name)[s, :n], getattr(full, name)[s, :n]), (r, s, name)
        # gathered output [t, L, world, b, hq, d] -> [t, b, L, Hq, d]
        g = out.permute(0, 3, 1, 2, 4, 5).reshape(3, batch, L, Hq, d)
        # K4 splits a segment into more pieces when there are fewer heads, so the
        # merge order (not the math) differs: bf16-rounding tolerance
        err = (g.float() - out_full.float()).abs()
        assert torch.all(err <= 2.0**-7 * (out_full.float().abs() + 0.125)), (r, err.max())


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("full_scan", [False, True])
def test_peer_exchange_selection(world, full_scan):
    """chess_select_push / chess_select_pull: the all-gather fused into the
    partial scan's tail over peer pointers.  In-process ranks on their own
    streams, issued rank after rank, so every pull really waits for the other
    ranks' pushes; repeated exchanges cycle both receive buffers; the last
    rounds replay per-rank CUDA graphs.  Bars: the oracle's selection on every
    rank, bit-identical across ranks, no wait timed out."""
    from helpers import load_vectors, read_selection, set_tables

    rng = np.random.default_rng(11 + world)
    L, H, d, batch, max_pages = 2, 8, 16, 3, 500
    D = L * H * d
    cfg = SelectionConfig(pages_per_chunk=4, chunks_per_grid=5, rho_grid=0.5, rho_chunk=0.2, rho_page=0.1,
                          window_pages=4, sink_pages=1)
    states, xs, shards = [], [], []
    for r in range(world):
        sh = HeadShard(r, world, L, H, H, d)
        shape = Shape(batch=batch, layers=L, kv_heads=H // world, q_heads=H // world, head_dim=d,
                      page_size=cfg.page_size, pages_per_chunk=cfg.pages_per_chunk,
                      chunks_per_grid=cfg.chunks_per_grid, max_pages=max_pages,
                      window_pages=cfg.window_pages, max_ws=max_pages, n_phys=1)
        states.append(DecodeState(shape))
        shards.append(sh)
        xs.append(PeerScoreExchange(sh, batch, max_pages, cfg.pages_per_chunk, cfg.chunks_per_grid, "cuda",
                                    full_scan=full_scan))
    for x in xs:
        x.connect_local(xs)
    expect = []
    for slot in range(batch):
        n = int(rng.integers(1, 450))
        rows = rng.standard_normal((n, D))
        for st, sh in zip(states, shards):
            load_vectors(st, slot, rows[:, sh.flat_columns().numpy()])
            set_tables(st, slot, n + 1, cfg.sink_pages)
        h = ref.Hierarchy.from_rows(rows, cfg.pages_per_chunk, cfg.chunks_per_grid)
        a, _ = ref.anchor(h.page_vectors, cfg.window_pages)
        s = [m @ a for m in (h.grid_vectors, h.chunk_vectors, h.page_vectors)]
        p2c, c2g = h.parent_maps()
        sel, _ = ref.prune(s[0], s[1], s[2], p2c, c2g, cfg.ratios)
        expect.append((sel, ref.working_set(sel, n + 1, cfg.window_pages, cfg.sink_pages)[0]))
    torch.cuda.synchronize()
    sc = _lib.ChessSelectCfg(cfg.rho_grid, cfg.rho_chunk, cfg.rho_page, int(full_scan), 1)
    streams = [torch.cuda.Stream() for _ in range(world)]

    def run_cascade(r):
        for lv in _levels(full_scan):
            xs[r].select_level(states[r], sc, lv, streams[r].cuda_stream)

    def verify():
        torch.cuda.synchronize()
        for x in xs:
            x.check()
        for slot, (sel, pages) in enumerate(expect):
            got0 = read_selection(states[0], slot)
            np.testing.assert_array_equal(got0[0], sel)
            np.testing.assert_array_equal(got0[1], pages)
            for st in states[1:]:
                for u, v in zip(got0, read_selection(st, slot)):
                    np.testing.assert_array_equal(u, v)

    rounds = 3
    for _ in range(rounds):
        for st in states:
            st.ws_len.zero_()
            st.n_semantic.zero_()
        torch.cuda.synchronize()
        for r in range(world):
            run_cascade(r)
        verify()
    graphs = []
    for r in range(world):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(streams[r]):
            with torch.cuda.graph(g, stream=streams[r]):
                run_cascade(r)
        graphs.append(g)
    torch.cuda.synchronize()
    for _ in range(2):
        for st in states:
            st.ws_len.zero_()
            st.n_semantic.zero_()
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                graphs[r].replay()
        verify()
    for x in xs:
        for lv in x.levels:
            assert torch.all(x.gen[lv] == rounds + 2), (lv, x.gen[lv])
        x.close()
