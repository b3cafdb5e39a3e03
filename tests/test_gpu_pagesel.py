"""The drop-in `pagesel` surface on the device, checked against the golden
fixtures produced by the reference itself (tests/golden/make_golden.py) and
the reference's own known-answer cases.  Mirrors the structure of
pkg/tests/test_hierarchy.py, test_selection.py, test_kv_store.py,
test_uncertainty.py and test_simulate.py.

Bars: index outputs, working sets, gathers, page statistics and triggers
bit-exact; f64 summaries and anchors bit-exact (same operation order as
hierarchy.py / selection.py); scores within 1e-12 relative (the reference's
dgemv has no defined summation order); entropies within 1e-12.
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2602_20732_b200 import pagesel as ps

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def _cfg(arr):
    B, nc, ng, rg, rc, rp, w, s = arr
    return ps.SelectionConfig(page_size=int(B), pages_per_chunk=int(nc), chunks_per_grid=int(ng),
                              rho_grid=float(rg), rho_chunk=float(rc), rho_page=float(rp),
                              window_pages=int(w), sink_pages=int(s))


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


# --------------------------------------------------------------- store
def test_store_seal_gather_versions():
    store = ps.PagedKvStore(4, 3, page_size=4)
    seq = store.create_sequence(ps.SelectionConfig(page_size=4, sink_pages=1))
    assert seq.sink_count == 1
    events = [store.append_token(seq, np.full(3, t), np.zeros(3)) for t in range(10)]
    assert [e.sealed for e in events].count(True) == 2 and events[3].sealed and events[7].sealed
    assert events[9].logical_index == 2
    assert store.gather_pages(seq, [0, 2]) == [seq.page_table[0], seq.page_table[2]]
    with pytest.raises(IndexError):
        store.gather_pages(seq, [3])
    with pytest.raises(ValueError):
        store.page(seq.page_table[0]).write(np.zeros(3), np.zeros(3))
    v = store.sealed_versions(seq)
    assert sorted(v.values()) == [4, 4]
    np.testing.assert_array_equal(_np(store.page(seq.page_table[1]).keys)[:, 0], [4, 5, 6, 7])


def test_store_out_of_pages():
    store = ps.PagedKvStore(1, 2, page_size=2)
    seq = store.create_sequence()
    for _ in range(2):
        store.append_token(seq, np.zeros(2), np.zeros(2))
    with pytest.raises(ps.OutOfPagesError):
        store.append_token(seq, np.zeros(2), np.zeros(2))
    with pytest.raises(ps.ConfigurationError):
        ps.PagedKvStore(0, 2)


# ----------------------------------------------------------- hierarchy
def test_hierarchy_incremental_bitwise_vs_reference():
    g = np.load(GOLD / "hierarchy.npz")
    for ci in range(int(g["n_cases"])):
        P, B, dim, nc, ng = map(int, g[f"c{ci}_shape"])
        keys = g[f"c{ci}_keys"]
        store = ps.PagedKvStore(P, dim, page_size=B)
        seq = store.create_sequence()
        idx = ps.HierarchyIndex(dim, nc, ng)
        for p in range(P):
            for r in range(B):
                ev = store.append_token(seq, keys[p, r], np.zeros(dim))
            assert ev.sealed
            pv = idx.finalize_page(store.page(ev.page_id), ev.logical_index)
            assert pv.page_logical_index == p
        np.testing.assert_array_equal(_np(idx.page_vectors), g[f"c{ci}_pages"])
        np.testing.assert_array_equal(_np(idx.chunk_vectors), g[f"c{ci}_chunks"])
        np.testing.assert_array_equal(_np(idx.grid_vectors), g[f"c{ci}_grids"])
        snap = json.loads(str(g[f"c{ci}_snapshot"]))
        assert idx.snapshot() == snap
        v_all, splits = idx.coalesced_matrix()
        assert splits == (snap["num_grids"], snap["num_chunks"], snap["num_pages"])
        np.testing.assert_array_equal(idx.page_to_chunk, np.arange(P) // nc)


def test_hierarchy_bulk_and_errors():
    g = np.load(GOLD / "hierarchy.npz")
    for ci in range(int(g["n_cases"])):
        P, B, dim, nc, ng = map(int, g[f"c{ci}_shape"])
        idx = ps.HierarchyIndex.from_page_vectors(g[f"c{ci}_pages"], nc, ng)
        np.testing.assert_array_equal(_np(idx.chunk_vectors), g[f"c{ci}_bulk_chunks"])
        np.testing.assert_array_equal(_np(idx.grid_vectors), g[f"c{ci}_bulk_grids"])
    store = ps.PagedKvStore(2, 4, page_size=2)
    seq = store.create_sequence()
    ev = store.append_token(seq, np.ones(4), np.ones(4))
    idx = ps.HierarchyIndex(4, 2, 2)
    with pytest.raises(ValueError):  # unsealed
        idx.finalize_page(store.page(ev.page_id), 0)
    ev = store.append_token(seq, np.ones(4), np.ones(4))
    with pytest.raises(ValueError):  # out of order
        idx.finalize_page(store.page(ev.page_id), 1)


def test_hierarchy_grows_past_initial_capacity():
    rng = np.random.default_rng(5)
    rows = rng.standard_normal((300, 6))
    idx = ps.HierarchyIndex(6, 3, 4)
    store = ps.PagedKvStore(300, 6, page_size=1)
    seq = store.create_sequence()
    for p in range(300):
        ev = store.append_token(seq, rows[p], rows[p])
        idx.finalize_page(store.page(ev.page_id), p)
    bulk = ps.HierarchyIndex.from_page_vectors(rows, 3, 4)
    np.testing.assert_array_equal(_np(idx.page_vectors), rows)
    np.testing.assert_allclose(_np(idx.grid_vectors), _np(bulk.grid_vectors), rtol=1e-10, atol=1e-12)


# ----------------------------------------------------------- selection
class _Seq:
    def __init__(self, table, sinks):
        self.page_table = list(table)
        self.sink_count = sinks


def test_selection_golden_instances():
    g = np.load(GOLD / "selection.npz")
    for i in range(int(g["n_instances"])):
        p = f"i{i}_"
        cfg = _cfg(g[p + "cfg"])
        vec = g[p + "vectors"]
        idx = ps.HierarchyIndex.from_page_vectors(vec, cfg.pages_per_chunk, cfg.chunks_per_grid)
        tail = g[p + "tail"]
        tail_page = None
        if len(tail):
            store = ps.PagedKvStore(1, vec.shape[1], page_size=cfg.page_size)
            seq = store.create_sequence()
            for k in tail:
                ev = store.append_token(seq, k, np.zeros_like(k))
            tail_page = store.page(ev.page_id)
        anchor = ps.compute_anchor(idx, tail_page, cfg)
        np.testing.assert_array_equal(_np(anchor.v), g[p + "anchor"], err_msg=f"instance {i}")
        assert anchor.source_pages == list(g[p + "anchor_sources"])
        v_all, splits = idx.coalesced_matrix()
        assert list(splits) == list(g[p + "splits"])
        s_g, s_c, s_p = ps.score_all(anchor, v_all, splits)
        scores = np.concatenate([_np(s_g), _np(s_c), _np(s_p)])
        ref = g[p + "scores"]
        np.testing.assert_allclose(scores, ref, rtol=1e-12, atol=1e-12 * max(1.0, np.abs(ref).max(initial=0)))
        # the cascade on the reference's own scores: exact
        G, C, _ = splits
        sel = ps.hierarchical_prune(ref[:G], ref[G:G + C], ref[G + C:], idx.page_to_chunk, idx.chunk_to_grid, cfg)
        np.testing.assert_array_equal(sel, g[p + "selected"], err_msg=f"instance {i}")
        # end to end on device scores (golden instances hold no near-ties)
        sel_dev = ps.hierarchical_prune(s_g, s_c, s_p, idx.page_to_chunk, idx.chunk_to_grid, cfg)
        np.testing.assert_array_equal(sel_dev, g[p + "selected"], err_msg=f"instance {i} (device scores)")
        flat = ps.oracle_flat_topk(anchor, idx.page_vectors, int(g[p + "flat_k"]))
        np.testing.assert_array_equal(flat, g[p + "flat"])
        seq = _Seq(g[p + "table"], int(g[p + "sinks"]))
        ws = ps.reconstruct_working_set(sel, seq, cfg)
        assert ws.pages == list(g[p + "ws_pages"])
        code = {"semantic": 1, "window": 2, "sink": 3}
        assert [code[ws.provenance[q]] for q in ws.pages] == list(g[p + "ws_prov"])
        store = ps.PagedKvStore(1, 1)
        assert store.gather_pages(seq, ws.pages) == list(g[p + "ws_phys"])


def test_selection_known_answers_and_errors():
    cfg = ps.SelectionConfig(pages_per_chunk=4, chunks_per_grid=1, rho_grid=1.0, rho_chunk=1.0, rho_page=0.5)
    p2c, c2g = np.zeros(4, int), np.zeros(1, int)
    got = ps.hierarchical_prune(np.ones(1), np.ones(1), np.array([4.0, 3.0, 2.0, 1.0]), p2c, c2g, cfg)
    assert list(got) == [0, 1]
    got = ps.hierarchical_prune(np.zeros(1), np.zeros(1), np.zeros(4), p2c, c2g, cfg)
    assert list(got) == [0, 1]
    assert len(ps.hierarchical_prune([], [], [], [], [], cfg)) == 0
    ws = ps.reconstruct_working_set([5], _Seq(range(8), 1), ps.SelectionConfig(window_pages=1))
    assert ws.pages == [0, 5, 7] and ws.provenance == {0: "sink", 5: "semantic", 7: "window"}
    idx = ps.HierarchyIndex(4, 2, 2)
    with pytest.raises(ps.EmptyContextError):
        ps.compute_anchor(idx, None, cfg)
    idx = ps.HierarchyIndex.from_page_vectors(np.eye(4), 2, 2)
    anchor = ps.compute_anchor(idx, None, cfg)
    with pytest.raises(ValueError):
        ps.score_all(anchor, np.ones((3, 5)), (1, 1, 1))
    with pytest.raises(ValueError):
        ps.oracle_flat_topk(anchor, idx.page_vectors, 5)


# --------------------------------------------------------- uncertainty
def test_uncertainty_golden():
    doc = json.loads((GOLD / "uncertainty.json").read_text())
    H = ps.entropies(np.asarray([r["probs"] for r in doc["rows"] if len(r["probs"]) == 64]))
    ref = [r["entropy"] for r in doc["rows"] if len(r["probs"]) == 64]
    np.testing.assert_allclose(_np(H), ref, rtol=1e-12, atol=1e-12)
    for r in doc["rows"]:
        assert abs(ps.entropy(r["probs"]) - r["entropy"]) <= 1e-12 * max(1.0, r["entropy"])
    assert abs(ps.entropy(np.full(8, 1 / 8)) - np.log(8)) < 1e-12
    assert ps.entropy([0.0, 1.0, 0.0]) == 0.0
    assert abs(ps.entropy([0.5, 0.25, 0.25]) - 1.5 * np.log(2)) < 1e-12
    for pg in doc["pages"]:
        u = ps.page_uncertainty(pg["entropies"])
        assert (u.mean_entropy, u.varentropy, u.token_count) == (pg["mean"], pg["var"], pg["n"])
    with pytest.raises(ValueError):
        ps.page_uncertainty([])
    with pytest.raises(ValueError):
        ps.entropy([0.5, 0.6])
    with pytest.raises(ValueError):
        ps.entropy([-0.1, 1.1])
    th = ps.TriggerThresholds(doc["calibration"]["tau_H"], doc["calibration"]["tau_V"], 0.9, len(doc["pages"]))
    for pg, t in zip(doc["pages"], doc["trigger"]):
        u = ps.PageUncertainty(pg["mean"], pg["var"], pg["n"])
        assert ps.check_trigger(u, th, "joint") == t["joint"]
        assert ps.check_trigger(u, th, "any") == t["any"]
    assert ps.check_trigger(ps.PageUncertainty(th.tau_entropy, th.tau_varentropy, 1), th) is False


# ------------------------------------------------------ decode loop
@pytest.mark.parametrize("run_idx", range(5))
def test_decode_loop_matches_reference(run_idx):
    run = json.loads((GOLD / "decode_loop.json").read_text())[run_idx]
    spec_kw = dict(run["spec"])
    sched = tuple(tuple(x) for x in spec_kw.pop("instability_schedule"))
    spec = ps.WorkloadSpec(**spec_kw, instability_schedule=sched)
    cfg = _cfg(run["cfg"])
    th = ps.TriggerThresholds(run["tau"][0], run["tau"][1], 0.99, 150) if run["policy"] == "dynamic" else None
    rep = ps.run_decode_loop(spec, cfg, run["policy"], thresholds=th)
    assert [s.trigger_fired for s in rep.steps] == run["fired"]
    assert [s.working_set_size for s in rep.steps] == run["ws_size"]
    assert rep.working_sets == [w["pages"] for w in run["working_sets"]]
    assert [s.recall for s in rep.steps] == run["recall"]
    assert rep.zero_copy_ok
    assert rep.summary()["trigger_count"] == run["summary"]["trigger_count"]


def test_calibrate_device_golden_and_random():
    """calibrate (uncertainty.py:59-83) on the device: bit-identical
    thresholds against the reference's golden calibration (ragged pages) and
    against the oracle on random streams, including heavy ties."""
    from oracle import pagesel_ref as oref

    doc = json.loads((GOLD / "uncertainty.json").read_text())
    pages = doc["pages"]
    n = max(len(pg["entropies"]) for pg in pages)
    ent = np.zeros((len(pages), n))
    for i, pg in enumerate(pages):
        ent[i, : len(pg["entropies"])] = pg["entropies"]
    counts = [len(pg["entropies"]) for pg in pages]
    th = ps.calibrate_device(ent, counts, doc["calibration"]["percentile"])
    assert (th.tau_entropy, th.tau_varentropy) == (doc["calibration"]["tau_H"], doc["calibration"]["tau_V"])
    rng = np.random.default_rng(9)
    for n_pages, B, p in ((1, 32, 0.5), (150, 32, 0.99), (1000, 16, 0.95), (4097, 32, 0.9), (300, 8, 0.3)):
        ent = rng.gamma(2.0, 0.1, size=(n_pages, B))
        if n_pages > 100:
            ent[: n_pages // 3] = 0.25  # ties across pages
        cnt = rng.integers(1, B + 1, size=n_pages)
        stats = [oref.page_stats(ent[i, : cnt[i]]) for i in range(n_pages)]
        want = oref.calibrate([s[0] for s in stats], [s[1] for s in stats], p)
        got = ps.calibrate_device(ent, cnt, p)
        assert (got.tau_entropy, got.tau_varentropy) == want, (n_pages, B, p)
    with pytest.raises(ps.CalibrationError):
        ps.calibrate_device(np.zeros((0, 4)))
    with pytest.raises(ps.CalibrationError):
        ps.calibrate_device(np.zeros((3, 4)), percentile=1.0)
