"""Selection pass at the bench's cfg3 state (planted relevance, K1b build):
time one chess_select (force_all) per summary dtype with CUDA events over a
captured graph, and report the tensor-core pass's uncertain rows per slot.

  python tools/select_tc_probe.py --dtypes f32 f16tc [--reps 10]
"""

import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_20732_b200 import _lib  # noqa: E402
from paper_2602_20732_b200.config import preset_config  # noqa: E402
from paper_2602_20732_b200.engine import ChessDecoder  # noqa: E402
from paper_2602_20732_b200.synthetic import SyntheticDecode  # noqa: E402


def probe(dt, reps, cfg_name, batch):
    wl = SyntheticDecode(cfg_name, batch=batch, gen_pages=4, ring=2, kv_budget_gib=8, summary_dtype=dt)
    st = wl.st
    cfg = preset_config("aggressive", page_size=wl.shape.page_size)
    dec = ChessDecoder(st, cfg, policy="every_step")
    wl.prefill(dec)
    sc = _lib.ChessSelectCfg(cfg.rho_grid, cfg.rho_chunk, cfg.rho_page, 0, 1)
    call = lambda stream: _lib.call("chess_select", st.ref, ctypes.byref(sc), _lib.stream_ptr(stream))
    lib = _lib.load()
    lib.chess_debug_tc_read.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32] + [ctypes.c_void_p] * 5

    def rescored():
        if dt != "f16tc":
            return 0
        m, tot = np.zeros(4, np.int32), 0
        for s in range(batch):
            _lib.check(lib.chess_debug_tc_read(st.ref, s, 0, 0, None, None, None, m.ctypes.data, None), "read")
            tot += int(m[3])
        return tot

    call(None)
    torch.cuda.synchronize()
    r0 = rescored()
    call(None)
    torch.cuda.synchronize()
    per_pass = rescored() - r0
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        for _ in range(reps):
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
    us = e0.elapsed_time(e1) * 1e3 / (3 * reps)
    stats = st.sel_stats.cpu().numpy()
    rows = int((stats[:, 0] + stats[:, 3] + stats[:, 4]).sum())
    per_level = []
    if dt == "f16tc":
        # uncertain rows per level (tensor-core pass of one level at a time)
        lib.chess_debug_select_tc_level.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
        m = np.zeros(4, np.int32)
        for level in range(3):
            _lib.check(lib.chess_debug_select_tc_level(st.ref, ctypes.byref(sc), level, None), "tc level")
            torch.cuda.synchronize()
            counts = []
            for s in range(batch):
                _lib.check(lib.chess_debug_tc_read(st.ref, s, level, 0, None, None, None, m.ctypes.data, None), "read")
                counts.append(int(m[0]))
            per_level.append(counts)
    out = {"dtype": dt, "us_per_pass": us, "rows_scanned": rows, "rescored_rows_per_pass": per_pass, "uncertain_per_level_slot": per_level,
           "dim": wl.shape.dim}
    print(json.dumps(out), flush=True)
    del g, dec, wl, st
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtypes", nargs="+", default=["f32", "f16tc"])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--batch", type=int, default=16)
    args = ap.parse_args()
    for dt in args.dtypes:
        probe(dt, args.reps, args.config, args.batch)


if __name__ == "__main__":
    main()
