"""Timeline of one captured decode step: every kernel of the step graph with
its start/end relative to the step's first kernel, from CUPTI activity records
(torch.profiler) of graph replays.  Shows where the step's time goes beyond
the attention layers: the gaps between dependent kernels, the side-stream
selection next to the decode layers, and what follows the last layer.

  python tools/step_timeline.py --config cfg3 --policy every_step --steps 3
"""

import argparse
import json
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2602_20732_b200 import _lib  # noqa: E402
from paper_2602_20732_b200.config import preset_config  # noqa: E402
from paper_2602_20732_b200.engine import ChessDecoder  # noqa: E402
from paper_2602_20732_b200.synthetic import SyntheticDecode  # noqa: E402


def graph_edges(graph):
    """Edge census of a captured step graph: programmatic (PDL) vs full
    edges, and the successors of every node that has more than one."""
    from cuda.bindings import runtime as cudart

    g = graph.raw_cuda_graph()
    err, _, _, _, n = cudart.cudaGraphGetEdges_v2(g, numEdges=0)
    err, frm, to, data, n = cudart.cudaGraphGetEdges_v2(g, numEdges=n)
    kinds = {}
    for i in range(n):
        t = int(data[i].type)
        kinds[t] = kinds.get(t, 0) + 1

    def kind(nd):
        e, t = cudart.cudaGraphNodeGetType(nd)
        return str(t).split(".")[-1].replace("cudaGraphNodeType", "")

    out = {}
    for i in range(n):
        out.setdefault(int(frm[i]), []).append((kind(to[i]), int(data[i].type), int(data[i].from_port)))
    fan = [v for v in out.values() if len(v) > 1]
    return {"edges": n, "edge_types": kinds, "multi_successor_nodes": fan}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--policy", default="every_step")
    ap.add_argument("--summary-dtype", default="f16tc")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--json", default="")
    ap.add_argument("--dot", default="", help="write the step graph as DOT (cudaGraphDebugDotPrint)")
    ap.add_argument("--sequential", action="store_true", help="no side-stream selection")
    args = ap.parse_args()
    _lib.load()
    wl = SyntheticDecode(args.config, gen_pages=16, ring=8, seed=0, summary_dtype=args.summary_dtype)
    st, sh = wl.st, wl.shape
    P, B = wl.P, wl.B
    st.reset()
    st.num_pages.fill_(P)
    st.tail_fill.fill_(B)
    st.token_count.fill_(P * B)
    st.sink_count.fill_(1)
    sel = preset_config("aggressive", page_size=sh.page_size)
    dec = ChessDecoder(st, sel, policy=args.policy, thresholds=wl.tau if args.policy == "dynamic" else None,
                       concurrent_select=not args.sequential)
    wl.prefill(dec)
    pre = 4 * B
    for t in range(pre):
        k, v, q, lg = wl.step_inputs(t)
        dec.step(k, v, q, lg, wl.out)
    torch.cuda.synchronize()
    graphs = []
    for r in range(args.steps + 2):
        k, v, q, lg = wl.step_inputs(pre + r)
        graphs.append(dec.capture(k, v, q, lg, wl.out))
    print(json.dumps(graph_edges(graphs[0])))
    if args.dot:
        from cuda.bindings import runtime as cudart

        cudart.cudaGraphDebugDotPrint(graphs[0].raw_cuda_graph(), args.dot.encode(), 1 << 14)
    graphs[0].replay()
    graphs[1].replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for g in graphs[2:]:
            g.replay()
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
           and "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
    evs.sort(key=lambda e: e.time_range.start)
    # split into steps at the synchronize gaps (> 50 us idle)
    steps, cur, last_end = [], [], None
    for e in evs:
        if last_end is not None and e.time_range.start - last_end > 50:
            steps.append(cur)
            cur = []
        cur.append(e)
        last_end = max(last_end or 0, e.time_range.end)
    if cur:
        steps.append(cur)
    report = []
    for i, s in enumerate(steps):
        t0 = s[0].time_range.start
        span = max(e.time_range.end for e in s) - t0
        rows = []
        for e in s:
            m = re.search(r"(\w+_kernel)(<[^>]*>)?", e.name)
            nm = m.group(0) if m else e.name
            rows.append({"kernel": nm[:48], "start_us": round(e.time_range.start - t0, 2),
                         "dur_us": round(e.time_range.end - e.time_range.start, 2)})
        report.append({"step": i, "span_us": round(span, 2), "kernels": rows})
    for rep in report:
        print(f"# step {rep['step']}: span {rep['span_us']} us, {len(rep['kernels'])} kernels")
        prev_end = 0.0
        for r in rep["kernels"]:
            gap = r["start_us"] - prev_end
            print(f"  {r['start_us']:9.2f} +{r['dur_us']:7.2f}  gap {gap:6.2f}  {r['kernel']}")
            prev_end = max(prev_end, r["start_us"] + r["dur_us"])
    # the last step's decode-stream kernels: sum of K4 durations vs span
    last = report[-1]
    k4 = [r for r in last["kernels"] if "sparse_decode" in r["kernel"]]
    if k4:
        first, lastk = k4[0], k4[-1]
        print(json.dumps({
            "span_us": last["span_us"],
            "k4_first_start_us": first["start_us"],
            "k4_last_end_us": round(lastk["start_us"] + lastk["dur_us"], 2),
            "k4_layers": len(k4),
            "k4_window_per_layer_us": round((lastk["start_us"] + lastk["dur_us"] - first["start_us"]) / len(k4), 2),
            "after_last_k4_us": round(last["span_us"] - (lastk["start_us"] + lastk["dur_us"]), 2),
        }))
    if args.json:
        Path(args.json).write_text(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
