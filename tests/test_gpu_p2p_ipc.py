"""The peer-memory score exchange across PROCESSES: two ranks (both on
cuda:0 — this round's boxes have one GPU) share their receive regions through
CUDA IPC handles (chess_p2p_export / chess_p2p_open, swapped over a gloo
group), then run the KV-head-sharded selection cascade with
chess_select_push / chess_select_pull.  Same bars as the in-process test:
the oracle's selection, identical on both ranks, no wait timed out.  On a
multi-GPU node the same code maps the peer GPU's memory over NVLink."""

import os

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
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    procs = [ctx.Process(target=_rank, args=(r, world, port, full_scan, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = {}
    while not q.empty():
        r, msg = q.get()
        res[r] = msg
    for p in procs:
        if p.is_alive():
            p.kill()
    assert res == {0: "ok", 1: "ok"}, res
