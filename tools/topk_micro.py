"""Block top-k (K3's block_topk_mark through chess_topk, one CTA) timed
alone over a captured graph: the per-level cost inside the selection tail.

  python tools/topk_micro.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2602_20732_b200 import _lib  # noqa: E402


def main():
    res = {}
    for n in (16, 64, 128, 256, 416, 1024, 4096):
        k = max(1, (n + 4) // 5)
        sc = torch.randn(n, dtype=torch.float64, device="cuda").abs() + 1.0
        out = torch.zeros(n, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(4, dtype=torch.int32, device="cuda")
        ws = torch.zeros(64 * n + 4096, dtype=torch.uint8, device="cuda")
        call = lambda s: _lib.call("chess_topk", _lib.ptr(sc), n, k, None, _lib.ptr(out), _lib.ptr(cnt), 1,
                                   _lib.ptr(ws), _lib.stream_ptr(s))
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for _ in range(20):
                call(gs)
        torch.cuda.current_stream().wait_stream(gs)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[n] = round(e0.elapsed_time(e1) * 1e3 / 100, 2)
        import ctypes
        buf = (ctypes.c_longlong * 8)()
        lib = _lib.load()
        if hasattr(lib, "chess_debug_topk_trace") and lib.chess_debug_topk_trace(buf) == 0 and buf[1]:
            res[f"{n}_cycles_keys_mark_64sync_64redpopc"] = [buf[0], buf[1], buf[2], buf[3]]
    print(json.dumps({"topk_us_per_call": res}))


if __name__ == "__main__":
    main()
