"""The peer-memory score exchange across PROCESSES: two ranks (both on
cuda:0 — this round's boxes have one GPU) share their receive regions through
CUDA IPC handles (chess_p2p_export / chess_p2p_open, swapped over a gloo
group), then run the KV-head-sharded selection cascade with
chess_select_push / chess_select_pull.  Same bars as the in-process test:
the oracle's selection, identical on both ranks, no wait timed out.  On a
multi-GPU node the same code maps the peer GPU's memory over NVLink."""


import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _rank(rank, world, port, full_scan, q):
    import torch.distributed as dist

    from helpers import load_vectors, read_selection, set_tables
    from oracle import pagesel_ref as ref
    from paper_2602_20732_b200 import _lib
    from paper_2602_20732_b200.config import SelectionConfig
    from paper_2602_20732_b200.parallel import HeadShard, PeerScoreExchange
    from paper_2602_20732_b200.state import DecodeState, Shape

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        rng = np.random.default_rng(3)
        L, H, d, batch, max_pages = 2, 4, 16, 2, 300
        cfg = SelectionConfig(pages_per_chunk=4, chunks_per_grid=4, rho_grid=0.5, rho_chunk=0.25,
                              rho_page=0.1, window_pages=4, sink_pages=1)
        sh = HeadShard(rank, world, L, H, H, d)
        shape = Shape(batch=batch, layers=L, kv_heads=H // world, q_heads=H // world, head_dim=d,
                      page_size=cfg.page_size, pages_per_chunk=cfg.pages_per_chunk,
                      chunks_per_grid=cfg.chunks_per_grid, max_pages=max_pages,
                      window_pages=cfg.window_pages, max_ws=max_pages, n_phys=1)
        st = DecodeState(shape)
        x = PeerScoreExchange(sh, batch, max_pages, cfg.pages_per_chunk, cfg.chunks_per_grid, "cuda:0",
                              full_scan=full_scan)
        x.connect()
        expect = []
        for slot in range(batch):
            n = int(rng.integers(20, 280))
            rows = rng.standard_normal((n, L * H * d))
            load_vectors(st, slot, rows[:, sh.flat_columns().numpy()])
            set_tables(st, slot, n + 1, cfg.sink_pages)
            h = ref.Hierarchy.from_rows(rows, cfg.pages_per_chunk, cfg.chunks_per_grid)
            a, _ = ref.anchor(h.page_vectors, cfg.window_pages)
            s = [m @ a for m in (h.grid_vectors, h.chunk_vectors, h.page_vectors)]
            p2c, c2g = h.parent_maps()
            sel, _ = ref.prune(s[0], s[1], s[2], p2c, c2g, cfg.ratios)
            expect.append((sel, ref.working_set(sel, n + 1, cfg.window_pages, cfg.sink_pages)[0]))
        torch.cuda.synchronize()
        dist.barrier()
        sc = _lib.ChessSelectCfg(cfg.rho_grid, cfg.rho_chunk, cfg.rho_page, int(full_scan), 1)
        for _ in range(3):
            for lv in x.levels:
                x.select_level(st, sc, lv, _lib.stream_ptr())
            torch.cuda.synchronize()
            x.check()
            for slot, (sel, pages) in enumerate(expect):
                got = read_selection(st, slot)
                np.testing.assert_array_equal(got[0], sel)
                np.testing.assert_array_equal(got[1], pages)
        dist.barrier()  # peers are done reading before regions are closed / freed
        x.close()
        q.put((rank, "ok"))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("full_scan", [False, True])
def test_peer_exchange_across_processes(full_scan):
    _run(_rank, (full_scan,))


def _rank_step(rank, world, port, q):
    """Whole head-shard decode steps across processes: scores AND outputs over
    IPC-mapped peer memory (no collective on the data path), eager then
    replayed from a captured CUDA graph; checked against the unsharded decoder
    run in the same process."""
    import torch.distributed as dist

    from paper_2602_20732_b200.config import preset_config
    from paper_2602_20732_b200.engine import ChessDecoder
    from paper_2602_20732_b200.parallel import HeadShard, PeerScoreExchange
    from paper_2602_20732_b200.state import DecodeState, Shape

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        torch.manual_seed(0)  # identical inputs in both processes
        cfg = preset_config("aggressive", page_size=16)
        L, H, Hq, d, B = 2, 4, 8, 64, 16
        batch, n_ctx, max_pages, n_phys, T = 2, 80, 120, 260, 4
        full_shape = Shape(batch=batch, layers=L, kv_heads=H, q_heads=Hq, head_dim=d, page_size=B,
                           pages_per_chunk=8, chunks_per_grid=8, max_pages=max_pages, window_pages=4,
                           max_ws=max_pages, n_phys=n_phys)
        k_pool = (torch.randn((L, n_phys, H, B, d), device="cuda") / 8).to(torch.bfloat16)
        v_pool = torch.randn((L, n_phys, H, B, d), device="cuda").to(torch.bfloat16)
        k_new = (torch.randn((T, batch, L, H, d), device="cuda") / 8).to(torch.bfloat16)
        v_new = torch.randn((T, batch, L, H, d), device="cuda").to(torch.bfloat16)
        qs = torch.randn((T, batch, L, Hq, d), device="cuda").to(torch.bfloat16)
        logits = torch.randn((T, batch, 3000), device="cuda")
        table = (torch.stack([torch.arange(max_pages) + 130 * s for s in range(batch)]) % n_phys).to(torch.int32)
        n_now = torch.full((batch,), n_ctx, dtype=torch.int32, device="cuda")

        def setup(shape, kp, vp):
            st = DecodeState(shape, kv_pool=(kp, vp))
            st.reset()
            st.page_table.copy_(table)
            st.num_pages.fill_(n_ctx)
            st.tail_fill.fill_(B)
            st.token_count.fill_(n_ctx * B)
            st.sink_count.fill_(1)
            return st

        full = setup(full_shape, k_pool.clone(), v_pool.clone())
        dec_full = ChessDecoder(full, cfg, policy="every_step")
        dec_full.build_index(n_now)
        dec_full.initial_selection()
        out_full = torch.zeros((T, batch, L, Hq, d), device="cuda", dtype=torch.bfloat16)
        sel_full = []
        for t in range(T):
            dec_full.step(k_new[t].reshape(batch, -1), v_new[t].reshape(batch, -1), qs[t], logits[t], out_full[t])
            sel_full.append((full.ws_len.clone(), full.block_table.clone()))

        hk, hq = H // world, Hq // world
        shape = Shape(**{**full_shape.__dict__, "kv_heads": hk, "q_heads": hq})
        st = setup(shape, k_pool[:, :, rank * hk:(rank + 1) * hk].contiguous(),
                   v_pool[:, :, rank * hk:(rank + 1) * hk].contiguous())
        x = PeerScoreExchange(HeadShard(rank, world, L, H, Hq, d), batch, max_pages, 8, 8, "cuda:0")
        x.connect()
        dec = ChessDecoder(st, cfg, policy="every_step", exchange=x)
        dec.build_index(n_now)
        dec.initial_selection()
        kl = k_new[:, :, :, rank * hk:(rank + 1) * hk].reshape(T, batch, -1).contiguous()
        vl = v_new[:, :, :, rank * hk:(rank + 1) * hk].reshape(T, batch, -1).contiguous()
        ql = qs[:, :, :, rank * hq:(rank + 1) * hq].contiguous()
        out = torch.zeros((T, L, world, batch, hq, d), device="cuda", dtype=torch.bfloat16)
        sels = []
        dec.step(kl[0], vl[0], ql[0], logits[0], out[0])
        sels.append((st.ws_len.clone(), st.block_table.clone()))
        sk, sv, sq, slg = kl[0].clone(), vl[0].clone(), ql[0].clone(), logits[0].clone()
        so = torch.zeros_like(out[0])
        g = dec.capture(sk, sv, sq, slg, so)
        for t in range(1, T):
            sk.copy_(kl[t])
            sv.copy_(vl[t])
            sq.copy_(ql[t])
            slg.copy_(logits[t])
            g.replay()
            out[t].copy_(so)
            sels.append((st.ws_len.clone(), st.block_table.clone()))
        torch.cuda.synchronize()
        x.check()
        for t in range(T):
            assert torch.equal(sels[t][0], sel_full[t][0]), t
            for s in range(batch):
                n = int(sel_full[t][0][s])
                assert torch.equal(sels[t][1][s, :n], sel_full[t][1][s, :n]), (t, s)
        gathered = out.permute(0, 3, 1, 2, 4, 5).reshape(T, batch, L, Hq, d)
        err = (gathered.float() - out_full.float()).abs()
        assert torch.all(err <= 2.0**-7 * (out_full.float().abs() + 0.125)), float(err.max())
        dist.barrier()
        x.close()
        q.put((rank, "ok"))
    except Exception as e:
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_peer_decode_step_across_processes():
    _run(_rank_step, ())


def _run(fn, extra):
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    procs = [ctx.Process(target=fn, args=(r, world, port, *extra, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = {}
    while not q.empty():
        r, msg = q.get()
        res[r] = msg
    for p in procs:
        if p.is_alive():
            p.kill()
    assert res == {0: "ok", 1: "ok"}, res
