"""Where a decode step's time goes: each stage of ChessDecoder.step captured
alone in a CUDA graph (reps back to back, CUDA events on the replay stream)
next to the whole step.  Stages that mutate state (append/seal) are replayed
on a fresh state copy only as timing probes.

  python tools/step_breakdown.py --config cfg2
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


def time_graph(fn, reps=20, outer=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn(s)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(outer):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * outer)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--kv-gib", type=float, default=None)
    args = ap.parse_args()
    wl = SyntheticDecode(args.config, batch=args.batch, gen_pages=64, ring=4, kv_budget_gib=args.kv_gib)
    sel = preset_config("aggressive", page_size=wl.B)
    dec = ChessDecoder(wl.st, sel, policy="every_step")
    wl.prefill(dec)
    k, v, q, lg = wl.step_inputs(0)
    L = wl.shape.layers
    res = {"config": args.config, "batch": wl.batch}
    res["attn_layer_us"] = time_graph(lambda s: dec.attend(0, q[:, 0], wl.out[:, 0], stream=s))
    res["attn_all_layers_us"] = time_graph(
        lambda s: [dec.attend(layer, q[:, layer], wl.out[:, layer], stream=s) for layer in range(L)], reps=4)
    res["entropy_trigger_us"] = time_graph(lambda s: dec.entropy_trigger(lg, stream=s))
    res["select_us"] = time_graph(lambda s: dec.select(force_all=True, stream=s), reps=5)
    res["build_ws_us"] = time_graph(lambda s: __import__("paper_2602_20732_b200")._lib.call(
        "chess_build_working_set", wl.st.ref, __import__("paper_2602_20732_b200")._lib.stream_ptr(s)))
    # state-mutating stages: time on the live state (the step is re-run below anyway)
    res["append_us"] = time_graph(lambda s: dec.append(k, v, stream=s), reps=8, outer=1)
    res["seal_us"] = time_graph(lambda s: dec.seal(stream=s), reps=8, outer=1)
    res["step_us"] = time_graph(lambda s: dec.step(k, v, q, lg, wl.out, stream=s), reps=8, outer=2)
    print(json.dumps({k_: (round(v_, 2) if isinstance(v_, float) else v_) for k_, v_ in res.items()}))


if __name__ == "__main__":
    main()
