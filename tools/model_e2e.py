"""Random-init Llama-3-8B decoding through CHESS at cfg3's context (SURVEY.md
§8f row 4): tokens/s of the whole model step (dense layers on cuBLAS + the
CHESS calls + trigger + seal + selection + greedy argmax), captured as one
CUDA graph, next to the CHESS-only share of the same step.

    python tools/model_e2e.py [--config cfg3] [--steps 50] [--kv-gib 100] [--policy every_step]

Prints one JSON line.  Not part of bench.py's contract (the bench measures the
hot path itself); this shows what the hot path costs inside a real model step.
The KV pool is aliased to --kv-gib (the 16 GB of weights must fit beside it).
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2602_20732_b200.config import preset_config  # noqa: E402
from paper_2602_20732_b200.engine import ChessDecoder  # noqa: E402
from paper_2602_20732_b200.model import LLAMA3_8B, LlamaChess  # noqa: E402
from paper_2602_20732_b200.synthetic import SyntheticDecode  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--kv-gib", type=float, default=100.0)
    ap.add_argument("--policy", default="every_step")
    args = ap.parse_args()
    total = args.warmup + args.steps + 2
    ring = 64
    wl = SyntheticDecode(args.config, gen_pages=(total + 2 * ring) // 32 + 8, ring=ring, seed=0,
                         kv_budget_gib=args.kv_gib)
    st, sh = wl.st, wl.shape
    st.reset()
    st.num_pages.fill_(wl.P)
    st.tail_fill.fill_(wl.B)
    st.token_count.fill_(wl.P * wl.B)
    st.sink_count.fill_(1)
    dec = ChessDecoder(st, preset_config("aggressive", page_size=sh.page_size), policy=args.policy)
    wl.prefill(dec)
    model = LlamaChess(LLAMA3_8B, dec, seed=0)
    b = sh.batch
    tok = torch.zeros(b, dtype=torch.int64, device="cuda")
    logits = torch.empty((b, LLAMA3_8B.vocab), device="cuda")
    nxt = torch.empty(b, dtype=torch.int64, device="cuda")
    model.step(tok, logits, nxt)
    g = model.capture(tok, logits, nxt)
    for _ in range(args.warmup):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / args.steps
    weight_bytes = sum(t.numel() * t.element_size() for lw in model.layers for t in lw.values())
    weight_bytes += model.lm_head.numel() * 2
    print(json.dumps({
        "workload": f"random-init Llama-3-8B decode through CHESS, {args.config} context "
                    f"({sh.max_pages * sh.page_size} max tokens), batch {b}, policy {args.policy}",
        "us_per_token_step": us,
        "tokens_per_s": b / us * 1e6,
        "weights_gb_read_per_step": weight_bytes / 1e9,
        "weights_floor_us": weight_bytes / 6554.6e9 * 1e6,
        "ws_pages_mean": float(st.ws_len.float().mean()),
        "finite_logits": bool(torch.isfinite(logits).all()),
    }))


if __name__ == "__main__":
    main()
