"""Stage-by-stage run of the bench's decode step with a sync after every
stage (eager, then one captured graph), printing progress — locates a stage
that faults or stalls without running the whole bench.

  python tools/debug_step.py --config cfg3 --kv-gib 24
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2602_20732_b200.config import preset_config  # noqa: E402
from paper_2602_20732_b200.engine import ChessDecoder  # noqa: E402
from paper_2602_20732_b200.synthetic import SyntheticDecode  # noqa: E402


def stage(name, fn):
    t = time.time()
    fn()
    torch.cuda.synchronize()
    print(f"{name:28s} ok {1e3 * (time.time() - t):8.2f} ms", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--kv-gib", type=float, default=24)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    wl = SyntheticDecode(args.config, batch=args.batch, gen_pages=8, ring=4, kv_budget_gib=args.kv_gib)
    sel = preset_config("aggressive", page_size=wl.B)
    dec = ChessDecoder(wl.st, sel, policy="every_step")
    stage("prefill", lambda: wl.prefill(dec))
    print("ws_len", wl.st.ws_len.tolist(), "fill", wl.st.tail_fill.tolist(), flush=True)
    for t in range(args.steps):
        k, v, q, lg = wl.step_inputs(t)
        stage(f"append[{t}]", lambda: dec.append(k, v))
        for layer in range(wl.shape.layers):
            stage(f"attend[{t}][{layer}]", lambda: dec.attend(layer, q[:, layer], wl.out[:, layer]))
        stage(f"entropy[{t}]", lambda: dec.entropy_trigger(lg))
        stage(f"seal[{t}]", lambda: dec.seal())
        stage(f"select[{t}]", lambda: dec.select())
    k, v, q, lg = wl.step_inputs(0)
    g = dec.capture(k, v, q, lg, wl.out)
    for t in range(args.steps):
        stage(f"graph[{t}]", g.replay)
    print("ws_len", wl.st.ws_len.tolist(), flush=True)


if __name__ == "__main__":
    main()
