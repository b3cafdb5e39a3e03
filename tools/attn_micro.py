"""K4 microbenchmark: one sparse-decode launch timed with CUDA events under
three block-table patterns, to separate kernel-internal limits from DRAM
access-pattern effects.

  hot     every working-set page maps to one of 64 physical pages (L2 resident)
  seq     pages consecutive in the pool
  random  pages drawn uniformly from the whole pool (the bench's pattern)

  python tools/attn_micro.py --batch 16 --ws 44 --pool-gib 40
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_20732_b200 import _lib  # noqa: E402
from paper_2602_20732_b200.state import DecodeState, Shape  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ws", type=int, default=44)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--q-heads", type=int, default=32)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--page", type=int, default=32)
    ap.add_argument("--pool-gib", type=float, default=40)
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    b, L, H, Hq, d, B = args.batch, args.layers, args.kv_heads, args.q_heads, args.head_dim, args.page
    page_bytes = L * H * B * d * 2 * 2
    n_phys = int(args.pool_gib * (1 << 30) // page_bytes)
    sh = Shape(batch=b, layers=L, kv_heads=H, q_heads=Hq, head_dim=d, page_size=B, pages_per_chunk=8,
               chunks_per_grid=8, max_pages=args.ws + 8, window_pages=4, max_ws=args.ws + 8, n_phys=n_phys)
    st = DecodeState(sh)
    st.k_pool.normal_()
    st.v_pool.normal_()
    q = torch.randn(b, L, Hq, d, device="cuda").to(torch.bfloat16)
    out = torch.zeros_like(q)
    rng = np.random.default_rng(0)
    res = {"n_phys": n_phys, "batch": b, "ws": args.ws}
    bytes_launch = b * args.ws * B * 2 * H * d * 2 + b * Hq * d * 4
    for pattern in ("hot", "seq", "random"):
        if pattern == "hot":
            bt = rng.integers(0, 64, size=(b, args.ws))
        elif pattern == "seq":
            bt = (np.arange(b * args.ws).reshape(b, args.ws) * 1) % n_phys
        else:
            bt = rng.choice(n_phys, size=(b, args.ws), replace=False)
        st.block_table[:, : args.ws] = torch.as_tensor(bt.astype(np.int32), device="cuda")
        st.ws_len.fill_(args.ws)
        st.tail_fill.fill_(B)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(3):
            for layer in range(L):
                _lib.call("chess_sparse_decode", st.ref, layer, _lib.ptr(q[:, layer]), q.stride(0),
                          _lib.ptr(out[:, layer]), out.stride(0), None, 0.088, _lib.stream_ptr())
        torch.cuda.synchronize()
        ev[0].record()
        for r in range(args.reps):
            for layer in range(L):
                _lib.call("chess_sparse_decode", st.ref, layer, _lib.ptr(q[:, layer]), q.stride(0),
                          _lib.ptr(out[:, layer]), out.stride(0), None, 0.088, _lib.stream_ptr())
        ev[1].record()
        torch.cuda.synchronize()
        us = ev[0].elapsed_time(ev[1]) * 1e3 / (args.reps * L)
        # the same launches captured in one CUDA graph (no host gaps, PDL edges)
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        per_graph = 8
        with torch.cuda.graph(graph, stream=gs):
            for r in range(per_graph):
                for layer in range(L):
                    # as the engine: every layer after the first follows another K4
                    _lib.call("chess_sparse_decode_ex", st.ref, layer, _lib.ptr(q[:, layer]), q.stride(0),
                              _lib.ptr(out[:, layer]), out.stride(0), None, 0.088,
                              _lib.ATTN_AFTER_DECODE if (r or layer) else 0, _lib.stream_ptr(gs))
        torch.cuda.current_stream().wait_stream(gs)
        graph.replay()
        torch.cuda.synchronize()
        ev[0].record()
        for r in range(5):
            graph.replay()
        ev[1].record()
        torch.cuda.synchronize()
        us_g = ev[0].elapsed_time(ev[1]) * 1e3 / (5 * per_graph * L)
        res[pattern] = {"us": us, "GBps": bytes_launch / us / 1e3, "graph_us": us_g,
                        "graph_GBps": bytes_launch / us_g / 1e3}
        # per-CTA timelines of the last two launches of the graph (layers L-2, L-1)
        import ctypes
        buf = (ctypes.c_ulonglong * (2 * 256 * 16))()
        if _lib.load().chess_debug_attn_trace(buf) == 0:
            tr = np.frombuffer(buf, dtype=np.uint64).reshape(2, 256, 16).astype(np.int64)
            ta, tb = tr[(L - 2) & 1], tr[(L - 1) & 1]
            ok_a, ok_b = ta[:, 4] > ta[:, 0], tb[:, 4] > tb[:, 0]
            if not ok_a.any() or not ok_b.any():
                print(json.dumps(res))
                continue
            t0 = ta[ok_a, 0].min()
            pct = lambda x: [round(float(np.percentile((x - t0) / 1e3, p)), 2) for p in (0, 50, 100)]
            res[pattern]["trace_us"] = {
                "prev_entry": pct(ta[ok_a, 0]), "prev_exit": pct(ta[ok_a, 4]),
                "entry": pct(tb[ok_b, 0]), "prologue": pct(tb[ok_b, 1]),
                "first_page": pct(tb[ok_b & (tb[:, 2] > 0), 2]) if (ok_b & (tb[:, 2] > 0)).any() else None,
                "consumed": pct(tb[ok_b & (tb[:, 3] > 0), 3]) if (ok_b & (tb[:, 3] > 0)).any() else None,
                "exit": pct(tb[ok_b, 4]),
                "pdl_passed": pct(tb[ok_b & (tb[:, 5] > 0), 5]) if (ok_b & (tb[:, 5] > 0)).any() else None,
                "merged": pct(tb[ok_b & (tb[:, 6] > 0), 6]) if (ok_b & (tb[:, 6] > 0)).any() else None,
                "sm_mhz": (lambda m: round(float(np.median((tb[m, 9] - tb[m, 8]) / (tb[m, 4] - tb[m, 2]) * 1e3)), 0) if m.any() else None)(ok_b & (tb[:, 8] > 0) & (tb[:, 4] > tb[:, 2])),
                "cycles_spin_write_merge_push_arrive": [int(np.median(tb[ok_b & (tb[:, i] > 0), i])) if (ok_b & (tb[:, i] > 0)).any() else None for i in range(10, 15)],
                "inbox": pct(tb[ok_b & (tb[:, 7] > 0), 7]) if (ok_b & (tb[:, 7] > 0)).any() else None}
        if pattern == "random" and _lib.load().chess_debug_attn_trace(buf) == 0:
            # per CTA of the last launch: SM id, streaming time (first page -> consumed)
            tb = np.frombuffer(buf, dtype=np.uint64).reshape(2, 256, 16).astype(np.int64)[(L - 1) & 1]
            ok = (tb[:, 3] > 0) & (tb[:, 2] > 0)
            res["per_cta"] = [[int(c), int(tb[c, 15]), round((tb[c, 3] - tb[c, 2]) / 1e3, 2),
                               round((tb[c, 4] - tb[ok, 0].min()) / 1e3, 2)] for c in np.nonzero(ok)[0]]
    res["bytes_per_launch"] = bytes_launch
    print(json.dumps(res))


if __name__ == "__main__":
    main()
