"""K2+K3 microbenchmark: the three-level selection cascade on random
summaries of a model shape, timed with CUDA events over a captured graph.

  python tools/select_micro.py --batch 16 --pages 4096 --dim 32768
"""

import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2602_20732_b200 import _lib  # noqa: E402
from paper_2602_20732_b200.state import DecodeState, Shape  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--pages", type=int, default=4096)
    ap.add_argument("--dim", type=int, default=32768)
    ap.add_argument("--full-scan", action="store_true")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    b, P, D = args.batch, args.pages, args.dim
    sh = Shape(batch=b, layers=1, kv_heads=1, q_heads=1, head_dim=D, page_size=32, pages_per_chunk=8,
               chunks_per_grid=8, max_pages=P + 8, window_pages=4, max_ws=P + 8, n_phys=1)
    st = DecodeState(sh)
    st.reset()
    for t in (st.page_vec32, st.chunk_vec32, st.grid_vec32):
        t.normal_()
    st.anchor.normal_()
    st.num_sealed.fill_(P)
    st.num_pages.fill_(P)
    st.tail_fill.fill_(32)
    st.sink_count.fill_(1)
    cfg = _lib.ChessSelectCfg(0.5, 0.2, 0.1, int(args.full_scan), 1)
    call = lambda stream: _lib.call("chess_select", st.ref, ctypes.byref(cfg), _lib.stream_ptr(stream))
    call(None)
    torch.cuda.synchronize()
    stats = st.sel_stats[0].tolist()
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        for _ in range(args.reps):
            call(gs)
    torch.cuda.current_stream().wait_stream(gs)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (3 * args.reps)
    G, C, Pn, Ac, Ap = stats[0], stats[1], stats[2], stats[3], stats[4]
    rows = (G + C + Pn) if args.full_scan else (G + Ac + Ap)
    nbytes = b * (rows * D * 4 + D * 8)
    res = {"batch": b, "pages": P, "dim": D, "sel_stats": stats, "us": us,
           "bytes": nbytes, "GBps": nbytes / us / 1e3}
    import numpy as np
    buf = (ctypes.c_ulonglong * (4 * 256 * 8))()
    if _lib.load().chess_debug_select_trace(buf) == 0:
        tr = np.frombuffer(buf, dtype=np.uint64).reshape(4, 256, 8)[:, :148].astype(np.int64)
        t0 = tr[0, :, 0].min()
        pct = lambda x: [round(float(np.percentile((x - t0) / 1e3, p)), 1) for p in (0, 50, 100)]
        for lv in range(4):
            if tr[lv, :, 0].max() == 0:
                continue
            res[f"level{lv}"] = {"entry": pct(tr[lv, :, 0]), "first_row": pct(tr[lv, :, 2]),
                                 "items_done": pct(tr[lv, :, 3]), "exit": pct(tr[lv, :, 4]),
                                 "producer_fetch_us": float(np.mean(tr[lv, :, 5])) / 1.9e3,
                                 "producer_issue_us": float(np.mean(tr[lv, :, 6])) / 1.9e3,
                                 "producer_wait_us": float(np.mean(tr[lv, :, 7])) / 1.9e3}
        tb = (ctypes.c_ulonglong * (4 * 64 * 8))()
        if _lib.load().chess_debug_select_tail_trace(tb) == 0:
            tt = np.frombuffer(tb, dtype=np.uint64).reshape(4, 64, 8)[:, :b].astype(np.int64)
            for lv in range(3):
                d = tt[lv]
                res[f"tail{lv}_us"] = {"won": float(np.median(d[:, 1] - d[:, 0]) / 1e3),
                                       "reduce": float(np.median(d[:, 2] - d[:, 1]) / 1e3),
                                       "topk": float(np.median(d[:, 3] - d[:, 2]) / 1e3),
                                       "rest": float(np.median(d[:, 4] - d[:, 3]) / 1e3),
                                       "end_vs_level_exit": float((d[:, 4].max() - tr[lv, :, 4].max()) / 1e3)}
    sb = (ctypes.c_ulonglong * (16 * 16))()
    lib = _lib.load()
    if hasattr(lib, "chess_debug_select_small_trace") and lib.chess_debug_select_small_trace(sb) == 0:
        t = np.frombuffer(sb, dtype=np.uint64).reshape(16, 16)[:b].astype(np.int64)
        if t[:, 0].max() > 0 and t[:, 14].max() > 0:
            # select_small_kernel (rows <= 16 KB) per-slot phases, median over slots:
            # anchor, then per level: rows landed, scored, top-k, emitted; then the working set
            names = ["anchor"] + [f"L{lv}_{x}" for lv in range(3) for x in ("rows", "score", "topk", "emit")] + ["ws"]
            idx = [1] + [2 + 4 * lv + j for lv in range(3) for j in range(4)] + [14]
            prev = t[:, 0]
            ph = {}
            for nme, j in zip(names, idx):
                ph[nme] = round(float(np.median(t[:, j] - prev)) / 1e3, 2)
                prev = t[:, j]
            res["small_phases_us"] = ph
            res["small_total_us"] = round(float(np.median(t[:, 14] - t[:, 0])) / 1e3, 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
