"""Feasibility probe: the step's selection on a side stream concurrently with
the L attention launches (fork/join inside one CUDA graph), vs the two run
back to back.  Timing only — the concurrent select rewrites block tables the
attention is reading (no double buffering here), which changes which valid
pages are read but not how many.

  CHESS_ATTN_GRID=108 CHESS_SELECT_GRID=40 python tools/concurrent_probe.py --config cfg3
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2602_20732_b200.config import preset_config  # noqa: E402
from paper_2602_20732_b200.engine import ChessDecoder  # noqa: E402
from paper_2602_20732_b200.synthetic import SyntheticDecode  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    args = ap.parse_args()
    wl = SyntheticDecode(args.config, gen_pages=16, ring=2)
    sel = preset_config("aggressive", page_size=wl.B)
    dec = ChessDecoder(wl.st, sel, policy="every_step")
    wl.prefill(dec)
    k, v, q, lg = wl.step_inputs(0)
    L = wl.shape.layers
    main_s, side_s = torch.cuda.Stream(), torch.cuda.Stream()

    def seq(s):
        for layer in range(L):
            dec.attend(layer, q[:, layer], wl.out[:, layer], stream=s)
        dec.select(force_all=True, stream=s)

    def conc(s):
        ev0 = torch.cuda.Event()
        ev0.record(s)
        side_s.wait_event(ev0)
        dec.select(force_all=True, stream=side_s)
        for layer in range(L):
            dec.attend(layer, q[:, layer], wl.out[:, layer], stream=s)
        ev1 = torch.cuda.Event()
        ev1.record(side_s)
        s.wait_event(ev1)

    res = {}
    for name, fn in (("sequential", seq), ("concurrent", conc)):
        main_s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=main_s):
            for _ in range(3):
                fn(main_s)
        torch.cuda.current_stream().wait_stream(main_s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[name + "_us"] = round(e0.elapsed_time(e1) * 1e3 / 15, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
