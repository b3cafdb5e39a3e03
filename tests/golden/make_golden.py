"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container only (it imports `pagesel` from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Every output value below is produced by the reference package's own public
functions (pagesel/__init__.py:43-86); the inputs are seeded NumPy draws that
are stored alongside, so the fixtures are self-contained.  The oracle
(oracle/pagesel_ref.py) is pinned against these files by
tests/test_oracle_golden.py, and the CUDA path is checked against the same
files by tests/test_gpu_golden.py.

Files
  hierarchy.npz    incremental finalize_page over seeded pages: page/chunk/
                   grid vectors + snapshot checksums (hierarchy.py:102-162)
  selection.npz    seeded selection instances (incl. partial tails, ties,
                   zero/negative scores): anchor, scores, hierarchical_prune,
                   oracle_flat_topk, reconstruct_working_set, gather_pages
                   (selection.py:44-140, kv_store.py:156-166)
  uncertainty.json entropy / page_uncertainty / calibrate / check_trigger
                   (uncertainty.py:22-98) on seeded distributions
  decode_loop.json run_decode_loop under every policy with the working set of
                   every generated page recorded (simulate.py:110-217)
  acceptance.json  release criteria C1-C3 (pkg/tests/test_acceptance.py:45-112)
                   and the CPU demo run of BASELINE configs[0] (seed 0, dim
                   1024, 256 pages of 16, policy always): prefill snapshot
                   checksums, working sets, budgets, recall
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _import_reference():
    if not REF_SRC.exists():
        raise SystemExit("reference tree not found; fixtures are generated in the build container")
    sys.path.insert(0, str(REF_SRC))
    import pagesel  # noqa: F401

    return pagesel


def _page(pagesel, keys, pid=0):
    page = pagesel.KvPage(pid, keys.shape[0], keys.shape[1])
    for k in keys:
        page.write(k, np.zeros_like(k))
    return page


def make_hierarchy(pagesel):
    rng = np.random.default_rng(1234)
    cases = {}
    for ci, (P, B, dim, nc, ng) in enumerate([(37, 4, 24, 3, 2), (7, 2, 5, 2, 2), (130, 8, 16, 8, 8),
                                               (1, 3, 7, 8, 8), (64, 16, 12, 4, 5)]):
        keys = rng.standard_normal((P, B, dim))
        idx = pagesel.HierarchyIndex(dim, nc, ng)
        for p in range(P):
            idx.finalize_page(_page(pagesel, keys[p], p), p)
        cases[f"c{ci}_keys"] = keys
        cases[f"c{ci}_shape"] = np.array([P, B, dim, nc, ng])
        cases[f"c{ci}_pages"] = idx.page_vectors
        cases[f"c{ci}_chunks"] = idx.chunk_vectors
        cases[f"c{ci}_grids"] = idx.grid_vectors
        snap = idx.snapshot()
        cases[f"c{ci}_snapshot"] = np.array(json.dumps(snap, sort_keys=True))
        # from_page_vectors over the same page rows (hierarchy.py:43-58)
        bulk = pagesel.HierarchyIndex.from_page_vectors(idx.page_vectors, nc, ng)
        cases[f"c{ci}_bulk_chunks"] = bulk.chunk_vectors
        cases[f"c{ci}_bulk_grids"] = bulk.grid_vectors
    cases["n_cases"] = np.array(5)
    np.savez_compressed(OUT / "hierarchy.npz", **cases)


class _Seq:
    def __init__(self, table, sinks):
        self.page_table = list(table)
        self.sink_count = sinks


def make_selection(pagesel):
    rng = np.random.default_rng(2026)
    out = {}
    n = 0

    def add(vectors, cfg, tail=None, n_table=None, sinks=None, table=None):
        nonlocal n
        P, dim = vectors.shape
        idx = pagesel.HierarchyIndex.from_page_vectors(vectors, cfg.pages_per_chunk, cfg.chunks_per_grid)
        tail_page = None
        if tail is not None:
            tail_page = pagesel.KvPage(10**6, cfg.page_size, dim)
            for k in tail:
                tail_page.write(k, np.zeros(dim))
        anchor = pagesel.compute_anchor(idx, tail_page, cfg)
        v_all, splits = idx.coalesced_matrix()
        s_g, s_c, s_p = pagesel.score_all(anchor, v_all, splits)
        sel = pagesel.hierarchical_prune(s_g, s_c, s_p, idx.page_to_chunk, idx.chunk_to_grid, cfg)
        k_flat = max(1, min(P, len(sel)))
        flat = pagesel.oracle_flat_topk(anchor, idx.page_vectors, k_flat) if P else np.zeros(0, int)
        n_tab = n_table if n_table is not None else P
        if table is None:
            table = (np.arange(n_tab) * 7 + 3) % 100003
        seq = _Seq(table, cfg.sink_pages if sinks is None else sinks)
        ws = pagesel.reconstruct_working_set(sel, seq, cfg)
        store = pagesel.PagedKvStore(1, 1)
        phys = store.gather_pages(seq, ws.pages)
        p = f"i{n}_"
        out[p + "vectors"] = vectors
        out[p + "cfg"] = np.array([cfg.page_size, cfg.pages_per_chunk, cfg.chunks_per_grid, cfg.rho_grid,
                                   cfg.rho_chunk, cfg.rho_page, cfg.window_pages, cfg.sink_pages])
        out[p + "tail"] = tail if tail is not None else np.zeros((0, dim))
        out[p + "table"] = np.asarray(table, dtype=np.int64)
        out[p + "sinks"] = np.array(seq.sink_count)
        out[p + "anchor"] = anchor.v
        out[p + "anchor_sources"] = np.asarray(anchor.source_pages, dtype=np.int64)
        out[p + "splits"] = np.asarray(splits, dtype=np.int64)
        out[p + "scores"] = np.concatenate([s_g, s_c, s_p])
        out[p + "selected"] = np.asarray(sel, dtype=np.int64)
        out[p + "flat_k"] = np.array(k_flat)
        out[p + "flat"] = np.asarray(flat, dtype=np.int64)
        out[p + "ws_pages"] = np.asarray(ws.pages, dtype=np.int64)
        prov_code = {"semantic": 1, "window": 2, "sink": 3}
        out[p + "ws_prov"] = np.asarray([prov_code[ws.provenance[i]] for i in ws.pages], dtype=np.int8)
        out[p + "ws_phys"] = np.asarray(phys, dtype=np.int64)
        n += 1

    SC = pagesel.SelectionConfig
    # random instances across presets / fan-outs / windows
    for t in range(24):
        P = int(rng.integers(1, 200))
        dim = int(rng.choice([4, 8, 16, 33]))
        preset = ["aggressive", "moderate", "conservative"][t % 3]
        cfg = pagesel.preset_config(preset, pages_per_chunk=int(rng.integers(1, 10)),
                                    chunks_per_grid=int(rng.integers(1, 10)),
                                    window_pages=int(rng.integers(1, 7)),
                                    sink_pages=int(rng.integers(0, 3)), page_size=8)
        vectors = rng.standard_normal((P, dim))
        tail = rng.standard_normal((int(rng.integers(1, 8)), dim)) if t % 4 == 1 else None
        n_table = P + (1 if tail is not None or t % 5 == 2 else 0)
        add(vectors, cfg, tail=tail, n_table=n_table)
    # heavy ties: quantised vectors, zero and negative scores (acceptance C3)
    for t in range(8):
        P = int(rng.integers(5, 200))
        dim = int(rng.choice([2, 3, 8]))
        vectors = rng.integers(-2, 3, size=(P, dim)).astype(np.float64)
        if t % 3 == 0:
            vectors[:] = 0.0
        if t % 3 == 1:
            vectors = -np.abs(vectors)
        cfg = SC(pages_per_chunk=int(rng.integers(1, 6)), chunks_per_grid=int(rng.integers(1, 6)),
                 rho_grid=float(rng.choice([0.5, 0.3, 1.0])), rho_chunk=float(rng.choice([0.2, 0.7, 1.0])),
                 rho_page=float(rng.choice([0.1, 0.5, 0.25])), window_pages=int(rng.integers(1, 5)),
                 sink_pages=int(rng.integers(0, 3)))
        add(vectors, cfg)
    # hand-derived cascade (test_selection.py:149-161 shape): 4 pages, one chunk/grid
    add(np.array([[4.0], [3.0], [2.0], [1.0]]),
        SC(pages_per_chunk=4, chunks_per_grid=1, rho_grid=1.0, rho_chunk=1.0, rho_page=0.5,
           window_pages=1, sink_pages=0))
    # a -0.0 / +0.0 tie
    add(np.array([[-0.0], [0.0], [0.0], [-0.0], [1.0]]),
        SC(pages_per_chunk=2, chunks_per_grid=2, rho_grid=1.0, rho_chunk=1.0, rho_page=0.5,
           window_pages=1, sink_pages=0))
    out["n_instances"] = np.array(n)
    np.savez_compressed(OUT / "selection.npz", **out)


def make_uncertainty(pagesel):
    rng = np.random.default_rng(77)
    rows = []
    for t in range(40):
        V = int(rng.choice([2, 8, 64, 300, 1000]))
        kind = t % 4
        if kind == 0:
            p = rng.dirichlet(np.full(V, 0.1))
        elif kind == 1:
            lam = float(rng.uniform(0.01, 0.05))
            p = np.full(V, lam / V)
            p[int(rng.integers(V))] += 1.0 - lam
        elif kind == 2:
            p = np.zeros(V)
            p[int(rng.integers(V))] = 1.0
        else:
            x = rng.standard_normal(V) * float(rng.uniform(0.5, 8.0))
            p = np.exp(x - x.max())
            p = p / p.sum()
        rows.append({"probs": p.tolist(), "entropy": pagesel.entropy(p)})
    known = {"uniform8": pagesel.entropy(np.full(8, 1 / 8)), "onehot": pagesel.entropy([0.0, 1.0, 0.0]),
             "half_quarter": pagesel.entropy([0.5, 0.25, 0.25])}
    pages = []
    for t in range(30):
        n = int(rng.integers(1, 40))
        e = (rng.gamma(2.0, 0.2, size=n)).tolist()
        u = pagesel.page_uncertainty(e)
        pages.append({"entropies": e, "mean": u.mean_entropy, "var": u.varentropy, "n": u.token_count})
    samples = [pagesel.PageUncertainty(p["mean"], p["var"], p["n"]) for p in pages]
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        th = pagesel.calibrate(samples, 0.9)
    trig = []
    for p in pages:
        u = pagesel.PageUncertainty(p["mean"], p["var"], p["n"])
        trig.append({"joint": pagesel.check_trigger(u, th, "joint"), "any": pagesel.check_trigger(u, th, "any")})
    # boundary: exactly at threshold never fires (strict)
    at = pagesel.PageUncertainty(th.tau_entropy, th.tau_varentropy, 1)
    doc = {"rows": rows, "known": known, "pages": pages,
           "calibration": {"percentile": 0.9, "tau_H": th.tau_entropy, "tau_V": th.tau_varentropy},
           "trigger": trig, "at_threshold": pagesel.check_trigger(at, th, "joint")}
    (OUT / "uncertainty.json").write_text(json.dumps(doc))


def make_decode_loop(pagesel):
    from pagesel import simulate

    runs = []
    base = dict(seed=5, dim=48, context_pages=96, page_size=8, generation_pages=12, pages_per_chunk=4,
                relevant_page_fraction=0.05, vocab=32)
    spec_cal = pagesel.WorkloadSpec(**{**base, "seed": 100, "generation_pages": 150})
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        th = pagesel.calibrate(pagesel.collect_page_uncertainties(spec_cal), 0.99)
    for policy, sched in [("never", ()), ("always", ()), ("fixed(3)", ()), ("dynamic", ((2, 2.0), (7, 2.0))),
                          ("dynamic", ())]:
        spec = pagesel.WorkloadSpec(**base, instability_schedule=sched)
        cfg = pagesel.preset_config("aggressive", page_size=8, pages_per_chunk=4, chunks_per_grid=3)
        recorded = []
        orig = simulate.reconstruct_working_set

        def rec(selected, seq, config, _orig=orig):
            ws = _orig(selected, seq, config)
            recorded.append({"pages": list(map(int, ws.pages)), "table": list(map(int, seq.page_table)),
                             "semantic": sorted(int(i) for i in selected)})
            return ws

        simulate.reconstruct_working_set = rec
        try:
            rep = pagesel.run_decode_loop(spec, cfg, policy, thresholds=th if policy == "dynamic" else None)
        finally:
            simulate.reconstruct_working_set = orig
        runs.append({
            "spec": {**base, "instability_schedule": [list(x) for x in sched]},
            "cfg": [cfg.page_size, cfg.pages_per_chunk, cfg.chunks_per_grid, cfg.rho_grid, cfg.rho_chunk,
                    cfg.rho_page, cfg.window_pages, cfg.sink_pages],
            "policy": policy,
            "tau": [th.tau_entropy, th.tau_varentropy],
            "fired": [bool(s.trigger_fired) for s in rep.steps],
            "ws_size": [s.working_set_size for s in rep.steps],
            "recall": [s.recall for s in rep.steps],
            "working_sets": recorded,
            "summary": rep.summary(),
        })
    (OUT / "decode_loop.json").write_text(json.dumps(runs))


def make_acceptance(pagesel):
    """Reference outputs of the release criteria the device must reproduce
    (pkg/tests/test_acceptance.py:45-112) and of the CPU demo run that is
    BASELINE configs[0].  Inputs are re-drawn by the tests
    with the same NumPy RNG calls, so only outputs are stored."""
    from pagesel import (HierarchyIndex, PagedKvStore, QueryAnchor, SelectionConfig, SequenceState,
                         hierarchical_prune, oracle_flat_topk, reconstruct_working_set, score_all)
    from pagesel.workload import generate_workload

    doc = {}
    # C1 (test_acceptance.py:45-65): budgets on 2048 pages, dim 32, seed 0
    rng = np.random.default_rng(0)
    index = HierarchyIndex.from_page_vectors(rng.standard_normal((2048, 32)), 8, 8)
    anchor = QueryAnchor(v=rng.standard_normal(32), source_pages=[])
    scores = score_all(anchor, *index.coalesced_matrix())
    doc["c1"] = {}
    for name in ("aggressive", "moderate", "conservative"):
        sel = hierarchical_prune(*scores, index.page_to_chunk, index.chunk_to_grid, pagesel.preset_config(name))
        doc["c1"][name] = [int(i) for i in sel]
    # C2 (test_acceptance.py:68-86): 200 flat-equivalence instances, seed 1
    rng = np.random.default_rng(1)
    c2 = []
    for _ in range(200):
        n_pages = int(rng.integers(1, 513))
        dim = int(rng.integers(8, 257))
        rho_p = float(rng.uniform(0.05, 1.0))
        index = HierarchyIndex.from_page_vectors(rng.standard_normal((n_pages, dim)), 4, 4)
        config = SelectionConfig(pages_per_chunk=4, chunks_per_grid=4, rho_grid=1.0, rho_chunk=1.0, rho_page=rho_p)
        anchor = QueryAnchor(v=rng.standard_normal(dim), source_pages=[])
        sc = score_all(anchor, *index.coalesced_matrix())
        hier = hierarchical_prune(*sc, index.page_to_chunk, index.chunk_to_grid, config)
        flat = oracle_flat_topk(anchor, index.page_vectors, math.ceil(rho_p * n_pages))
        assert np.array_equal(hier, flat)
        c2.append([int(i) for i in hier])
    doc["c2"] = c2
    # C3 (test_acceptance.py:89-112): 1000 working-set fuzz cases, seed 2
    rng = np.random.default_rng(2)
    c3 = []
    for trial in range(1000):
        n_pages = int(rng.integers(1, 128))
        sinks = int(rng.integers(0, 5))
        window = int(rng.integers(1, 9))
        config = SelectionConfig(window_pages=window, sink_pages=sinks)
        mode = trial % 3
        if mode == 0:
            scores = np.zeros(n_pages)
        elif mode == 1:
            scores = -np.abs(rng.standard_normal(n_pages))
        else:
            scores = rng.standard_normal(n_pages)
        k = int(rng.integers(0, n_pages + 1))
        selected = np.sort(np.argsort(-scores, kind="stable")[:k])
        ws = reconstruct_working_set(selected, SequenceState(page_table=list(range(n_pages)), sink_count=sinks),
                                     config)
        c3.append({"selected": [int(i) for i in selected], "pages": [int(i) for i in ws.pages],
                   "prov": [ws.provenance[p] for p in ws.pages]})
    doc["c3"] = c3
    # BASELINE configs[0] / SURVEY §8c: the CPU demo run
    spec = pagesel.WorkloadSpec(seed=0, dim=1024, context_pages=256, page_size=16, generation_pages=2)
    cfg = pagesel.preset_config("aggressive", page_size=16)
    wl = generate_workload(spec)
    store = PagedKvStore(spec.context_pages + spec.generation_pages + 1, spec.dim, page_size=16)
    seq = store.create_sequence(cfg)
    index = HierarchyIndex(spec.dim, cfg.pages_per_chunk, cfg.chunks_per_grid)
    for t in range(wl.context_keys.shape[0]):
        ev = store.append_token(seq, wl.context_keys[t], wl.context_values[t])
        if ev.sealed:
            index.finalize_page(store.page(ev.page_id), ev.logical_index)
    snap = index.snapshot()
    from pagesel import simulate

    recorded = []
    orig = simulate.reconstruct_working_set

    def rec(selected, seq, config, _orig=orig):
        ws = _orig(selected, seq, config)
        recorded.append(list(map(int, ws.pages)))
        return ws

    simulate.reconstruct_working_set = rec
    try:
        rep = pagesel.run_decode_loop(spec, cfg, "always")
    finally:
        simulate.reconstruct_working_set = orig
    doc["cfg1"] = {
        "spec": {"seed": 0, "dim": 1024, "context_pages": 256, "page_size": 16, "generation_pages": 2},
        "policy": "always",
        "prefill_snapshot": snap,
        "working_sets": recorded,
        "ws_size": [s.working_set_size for s in rep.steps],
        "budget_semantic": [s.budget_fraction_semantic for s in rep.steps],
        "recall": [s.recall for s in rep.steps],
        "summary": rep.summary(),
    }
    (OUT / "acceptance.json").write_text(json.dumps(doc))


def main():
    pagesel = _import_reference()
    make_hierarchy(pagesel)
    make_selection(pagesel)
    make_uncertainty(pagesel)
    make_decode_loop(pagesel)
    make_acceptance(pagesel)
    for f in sorted(OUT.iterdir()):
        if f.suffix in (".npz", ".json"):
            print(f"{f.name}: {f.stat().st_size} bytes")


if __name__ == "__main__":
    main()
