"""World-size-2 gloo tests (CPU) of the multi-GPU host logic
(paper_2602_20732_b200/parallel.py): batch-shard slot ranges,
head-shard column ownership, rank-ordered partial-score sums that give every
rank the identical selection, output gathers and max-over-ranks timing."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pagesel_ref as ref
from paper_2602_20732_b200.parallel import (
    BatchShard,
    HeadShard,
    HeadShardExchange,
    allgather_sum_scores,
    gather_head_outputs,
    max_over_ranks,
)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, H, Hq, d = 3, 4, 8, 5
        sh = HeadShard(rank, world, L, H, Hq, d)
        rng = np.random.default_rng(0)
        D = L * H * d
        P, nc, ng = 37, 4, 3
        rows = rng.standard_normal((P, D))
        h_full = ref.Hierarchy.from_rows(rows, nc, ng)
        a_full, _ = ref.anchor(h_full.page_vectors, 4)
        cols = sh.flat_columns().numpy()
        # each rank: summaries + anchor over its own columns (linear in the columns)
        h_loc = ref.Hierarchy.from_rows(rows[:, cols], nc, ng)
        a_loc, _ = ref.anchor(h_loc.page_vectors, 4)
        mats = (h_loc.grid_vectors, h_loc.chunk_vectors, h_loc.page_vectors)
        partial = torch.as_tensor(np.concatenate([m @ a_loc for m in mats]))
        total = allgather_sum_scores(partial)
        G, C, _ = h_full.counts
        s = total.numpy()
        p2c, c2g = h_full.parent_maps()
        sel, _ = ref.prune(s[:G], s[G:G + C], s[G + C:], p2c, c2g, (0.5, 0.2, 0.1))
        full = np.concatenate([m @ a_full for m in (h_full.grid_vectors, h_full.chunk_vectors,
                                                     h_full.page_vectors)])
        out_local = torch.full((2, sh.local_q_heads, d), float(rank))
        gathered = gather_head_outputs(out_local)
        t = max_over_ranks(1.0 + rank)
        shard = BatchShard(rank, world, 5)
        # the engine's exchange object over the same process group
        x = HeadShardExchange(sh, 2, 37, nc, ng, "cpu")
        for lv in x.levels:
            x.partial[lv].fill_(10.0 * lv + rank)
            g = x.scores(lv)
            assert g.shape == (world, 2, x.ld[lv])
            assert all(torch.all(g[r] == 10.0 * lv + r) for r in range(world))
        buf = torch.zeros((world, 2, sh.local_q_heads, d))
        buf[rank].fill_(rank + 1.0)
        x.outputs(buf)
        assert all(torch.all(buf[r] == r + 1.0) for r in range(world))
        q.put((rank, s.tobytes(), sel.tolist(), float(np.max(np.abs(s - full))), gathered.numpy(),
               t, list(shard.slots), cols.tolist()))
    finally:
        dist.destroy_process_group()


def test_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical f64 scores and selections on every rank
    assert res[0][1] == res[1][1]
    assert res[0][2] == res[1][2]
    # the sharded sum equals the full-dimension scores to rounding
    assert res[0][3] < 1e-12
    # outputs gathered in head order
    g0 = res[0][4]
    assert g0.shape == (2, 8, 5)
    assert np.all(g0[:, :4] == 0.0) and np.all(g0[:, 4:] == 1.0)
    assert res[0][5] == res[1][5] == 2.0
    # batch shard covers every slot exactly once
    assert res[0][6] + res[1][6] == list(range(5))
    # head shard columns partition the flattened key row
    assert sorted(res[0][7] + res[1][7]) == list(range(3 * 4 * 5))


def test_shard_validation():
    with pytest.raises(ValueError):
        HeadShard(0, 3, 1, 8, 8, 4)
    assert list(BatchShard(3, 4, 128).slots) == list(range(96, 128))


def test_peer_exchange_layout():
    """Receive buffers / flags of the peer-memory score exchange: the same
    offsets on every rank (each rank maps its peers' regions at these),
    256-byte aligned blocks, no overlap."""
    from paper_2602_20732_b200.parallel import PeerScoreExchange

    for world, batch in ((1, 1), (2, 3), (8, 64)):
        ld = {0: 7, 1: 33, 2: 250}
        offs, total = PeerScoreExchange.layout(world, batch, ld)
        spans = []
        for lv, (ro, fo) in offs.items():
            assert ro % 256 == 0 and fo % 256 == 0
            spans.append((ro, ro + 2 * world * batch * ld[lv] * 8))
            spans.append((fo, fo + batch * world * 4))
        spans.sort()
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert a1 <= b0
        assert spans[-1][1] <= total
