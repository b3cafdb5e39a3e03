"""Focused driver for ncu: builds a model-shaped state and launches the hot
kernels a few times eagerly (no graphs) so `ncu -k regex:...` captures them.

  python tools/profile_kernels.py --config cfg3 --kv-gib 24 --reps 2
"""

import argparse
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
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--kv-gib", type=float, default=24)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--summary-dtype", default="f32")
    args = ap.parse_args()
    wl = SyntheticDecode(args.config, batch=args.batch, gen_pages=8, ring=2,
                         kv_budget_gib=args.kv_gib, summary_dtype=args.summary_dtype)
    sel = preset_config("aggressive", page_size=wl.B)
    dec = ChessDecoder(wl.st, sel, policy="every_step")
    wl.prefill(dec)
    k, v, q, lg = wl.step_inputs(0)
    torch.cuda.synchronize()
    for _ in range(args.reps):
        dec.step(k, v, q, lg, wl.out)
        for layer in range(4):
            dec.attend(layer, q[:, layer], wl.out[:, layer])
        dec.select(force_all=True)
    torch.cuda.synchronize()
    print("ws_len", wl.st.ws_len.tolist())


if __name__ == "__main__":
    main()
