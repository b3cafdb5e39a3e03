"""K4 at the bench's cfg3 state under different working-set compositions.

Explains why the bench's K4 launch time depends on --steps: after a short
run the anchor is the last context window (noise), so the semantic set is
scattered; once generated pages (which carry half the planted signal) seal,
the anchor points at the signal and the semantic set is the planted,
contiguous run of pages.  Same state, same q; only block_table / ws_len
change.  Each line: us per launch (CUDA graph of 3 x 32 layers, CUDA events),
GB/s of algorithmic bytes, unique physical pages per launch.

  python tools/k4_ws_probe.py [--kv-gib 120]
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_20732_b200.config import preset_config  # noqa: E402
from paper_2602_20732_b200.engine import ChessDecoder  # noqa: E402
from paper_2602_20732_b200.synthetic import SyntheticDecode  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kv-gib", type=float, default=None)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    wl = SyntheticDecode("cfg3", batch=16, gen_pages=8, ring=2, kv_budget_gib=args.kv_gib)
    st, sh = wl.st, wl.shape
    cfg = preset_config("aggressive", page_size=sh.page_size)
    dec = ChessDecoder(st, cfg, policy="every_step")
    wl.prefill(dec)
    P, B, L, b = wl.P, wl.B, sh.layers, wl.batch
    q = wl.q_ring[0]
    rng = np.random.default_rng(0)
    init_ws = [st.ws_logical[s, : int(st.ws_len[s])].cpu().numpy() for s in range(b)]
    n = int(round(np.mean([len(w) for w in init_ws])))
    window = list(range(P - 4, P))
    pats = {"initial_selection": init_ws,
            "planted_run": [np.array(sorted({0, *wl.relevant[s], *window})) for s in range(b)],
            "random_pages": [np.array(sorted({0, *rng.choice(np.arange(1, P - 4), n - 5, replace=False), *window}))
                             for s in range(b)],
            "shifted_run": [np.array(sorted({0, *[(p + 997) % (P - 5) + 1 for p in wl.relevant[s]], *window}))
                            for s in range(b)]}
    res = {"n_phys": sh.n_phys, "aliased": wl.aliased}
    for name, wss in pats.items():
        for s, w in enumerate(wss):
            st.ws_logical[s, : len(w)] = torch.as_tensor(w, dtype=torch.int32)
            st.block_table[s, : len(w)] = torch.as_tensor(wl.table_cpu[s, w].numpy(), dtype=torch.int32)
            st.ws_len[s] = len(w)
        st.tail_fill.fill_(B)
        phys = np.concatenate([wl.table_cpu[s, w].numpy() for s, w in enumerate(wss)])
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for r in range(args.reps):
                for layer in range(L):
                    dec.attend(layer, q[:, layer], wl.out[:, layer], stream=gs, after_decode=r + layer > 0)
        torch.cuda.current_stream().wait_stream(gs)
        g.replay()
        torch.cuda.synchronize()
        times = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3 / (args.reps * L))
        us = float(np.median(times))
        rows = sum(len(w) for w in wss) * B
        byt = rows * 2 * sh.kv_heads * sh.head_dim * 2 + b * sh.q_heads * sh.head_dim * 4
        res[name] = {"us": round(us, 3), "GBps": round(byt / us / 1e3, 1), "ws_mean": float(np.mean([len(w) for w in wss])),
                     "pages": int(phys.size), "unique_pages": int(np.unique(phys).size),
                     "phys_span_mean": float(np.mean([np.ptp(wl.table_cpu[s, w].numpy()) for s, w in enumerate(wss)]))}
        del g
    print(json.dumps(res))


if __name__ == "__main__":
    main()
