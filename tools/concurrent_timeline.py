"""Which stream of the concurrent step finishes last?  Replays the engine's
concurrent step structure eagerly with CUDA events at the fork, at the end of
the decode chain (main stream) and at the end of the selection chain (side
stream), averaged over steps.

  python tools/concurrent_timeline.py --config cfg3
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2602_20732_b200 import _lib  # noqa: E402
from paper_2602_20732_b200.config import preset_config  # noqa: E402
from paper_2602_20732_b200.engine import ChessDecoder  # noqa: E402
from paper_2602_20732_b200.synthetic import SyntheticDecode  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    wl = SyntheticDecode(args.config, gen_pages=16, ring=2)
    sel = preset_config("aggressive", page_size=wl.B)
    dec = ChessDecoder(wl.st, sel, policy="every_step")
    wl.prefill(dec)
    k, v, q, lg = wl.step_inputs(0)
    L = wl.shape.layers
    main_s, side = torch.cuda.Stream(), dec._side
    acc = {"decode_chain_us": 0.0, "select_chain_us": 0.0, "step_us": 0.0}
    for t in range(args.steps + 3):
        with torch.cuda.stream(main_s):
            e0, e_dec, e_sel, e_end = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            dec.append(k, v, main_s)
            e0.record(main_s)
            side.wait_event(e0)
            dec.entropy_trigger(lg, None, side)
            dec.seal(side)
            dec.select(force_all=True, stream=side, defer_ws=True)
            e_sel.record(side)
            for layer in range(L):
                dec.attend(layer, q[:, layer], wl.out[:, layer], None, main_s)
            e_dec.record(main_s)
            main_s.wait_event(e_sel)
            _lib.call("chess_flush_working_sets", wl.st.ref, _lib.stream_ptr(main_s))
            e_end.record(main_s)
        torch.cuda.synchronize()
        if t >= 3:
            acc["decode_chain_us"] += e0.elapsed_time(e_dec) * 1e3 / args.steps
            acc["select_chain_us"] += e0.elapsed_time(e_sel) * 1e3 / args.steps
            acc["step_us"] += e0.elapsed_time(e_end) * 1e3 / args.steps
    print(json.dumps({k_: round(v_, 1) for k_, v_ in acc.items()}))


if __name__ == "__main__":
    main()
