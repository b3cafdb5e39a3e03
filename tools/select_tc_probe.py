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
    trace = {}
    if dt == "f16tc" and hasattr(lib, "chess_debug_select_tc_trace"):
        # trace build (CHESS_B200_LIB=.../libchess_b200_trace.so): one more pass, then
        # the per-CTA / per-slot stamps of the three tensor-core launches and the
        # rescoring launches (select_scan_kernel<double>, g_sel_trace / g_tail_trace)
        call(None)
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (3 * 256 * 4 + 3 * 64 * 12))()
        if lib.chess_debug_select_tc_trace(buf) == 0:
            a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
            ct = a[:3 * 256 * 4].reshape(3, 256, 4)[:, :148]
            tt = a[3 * 256 * 4:].reshape(3, 64, 12)[:, :batch]
            sb = (ctypes.c_ulonglong * (4 * 256 * 8))()
            tb = (ctypes.c_ulonglong * (4 * 64 * 8))()
            lib.chess_debug_select_trace(sb)
            lib.chess_debug_select_tail_trace(tb)
            sr = np.frombuffer(sb, dtype=np.uint64).astype(np.int64).reshape(4, 256, 8)[:, :148]
            rt = np.frombuffer(tb, dtype=np.uint64).astype(np.int64).reshape(4, 64, 8)[:, :batch]
            if ct[:, :, 0].max() > 0:
                t0 = ct[0, :, 0].min()
                us_ = lambda x: (x - t0) / 1e3
                pct = lambda x: [round(float(np.percentile(us_(x), p)), 1) for p in (0, 50, 100)]
                for lv in range(3):
                    e = {"tc_entry": pct(ct[lv, :, 0]), "tc_items_done": pct(ct[lv, :, 1]),
                         "tc_exit": pct(ct[lv, :, 2]),
                         "tail_start": pct(tt[lv, :, 0]), "tail_end": pct(tt[lv, :, 1]),
                         "tail_us": [round(float(x), 1) for x in np.percentile((tt[lv, :, 1] - tt[lv, :, 0]) / 1e3, (0, 50, 100))],
                         "tail_items_left": [int(x) for x in tt[lv, :, 3]],
                         # median per-phase time: norms, certify rows, T top-k, H top-k, classify+compact, emit
                         "tail_phases_us": [round(float(np.median(tt[lv, :, j] - tt[lv, :, j - 1 if j > 4 else 0])) / 1e3, 2)
                                            for j in range(4, 10)]}
                    if sr[lv, :, 0].max() > 0:
                        e["rescore_entry"] = pct(sr[lv, :, 0][sr[lv, :, 0] > 0])
                        e["rescore_exit"] = pct(sr[lv, :, 4][sr[lv, :, 4] > 0])
                        e["rescore_first_row"] = pct(sr[lv, :, 2][sr[lv, :, 2] > 0])
                        e["rescore_items_done"] = pct(sr[lv, :, 3][sr[lv, :, 3] > 0])
                        w = rt[lv][rt[lv, :, 0] > 0]
                        if len(w):
                            # per-slot rescoring tail: {flush entered, counter won, reduced, top-k, done}
                            e["rescore_tail_phases_us"] = [round(float(np.median(w[:, j] - w[:, j - 1])) / 1e3, 2)
                                                           for j in range(1, 5)]
                            e["rescore_tail_won"] = pct(w[:, 1])
                            # finish: reduced -> top-k -> flags scattered -> emitted -> done
                            e["rescore_finish_us"] = [round(float(np.median(w[:, b] - w[:, a])) / 1e3, 2)
                                                      for a, b in ((2, 3), (3, 5), (5, 6), (6, 4))]
                        v = rt[lv, :, 4][rt[lv, :, 4] > 0]
                        if v.size:
                            e["rescore_tail_end"] = pct(v)
                    trace[f"level{lv}"] = e
    out = {"dtype": dt, "us_per_pass": us, "trace": trace, "rows_scanned": rows, "rescored_rows_per_pass": per_pass, "uncertain_per_level_slot": per_level,
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
