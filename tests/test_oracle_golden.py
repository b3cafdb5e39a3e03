"""Pin the CPU oracle (oracle/pagesel_ref.py) against golden vectors produced
by the reference itself (tests/golden/make_golden.py).  CPU only.

Bar: bit-exact for every integer/index output and for the f64 arithmetic the
oracle restates in the reference's operation order (page means, chunk/grid
sums, anchor, scores), plus the known answers of the reference's own tests
(test_uncertainty.py:22-31, test_selection.py:149-195, test_hierarchy.py:48-62).
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import attention as attn_ref
from oracle import pagesel_ref as ref
from paper_2602_20732_b200.config import PRESETS, SelectionConfig

GOLD = Path(__file__).resolve().parent / "golden"


def _cfg(arr):
    B, nc, ng, rg, rc, rp, w, s = arr
    return SelectionConfig(page_size=int(B), pages_per_chunk=int(nc), chunks_per_grid=int(ng),
                           rho_grid=float(rg), rho_chunk=float(rc), rho_page=float(rp),
                           window_pages=int(w), sink_pages=int(s))


@pytest.fixture(scope="module")
def hier():
    return np.load(GOLD / "hierarchy.npz")


@pytest.fixture(scope="module")
def sel():
    return np.load(GOLD / "selection.npz")


def test_hierarchy_incremental_bitwise(hier):
    for ci in range(int(hier["n_cases"])):
        P, B, dim, nc, ng = map(int, hier[f"c{ci}_shape"])
        h = ref.Hierarchy(dim, nc, ng)
        keys = hier[f"c{ci}_keys"]
        for p in range(P):
            h.fold_page(keys[p], p)
        assert np.array_equal(h.page_vectors, hier[f"c{ci}_pages"])
        assert np.array_equal(h.chunk_vectors, hier[f"c{ci}_chunks"])
        assert np.array_equal(h.grid_vectors, hier[f"c{ci}_grids"])
        snap = json.loads(str(hier[f"c{ci}_snapshot"]))
        mine = h.snapshot()
        for k in ("num_pages", "num_chunks", "num_grids", "checksum_pages", "checksum_chunks",
                  "checksum_grids"):
            assert mine[k] == snap[k], (ci, k)


def test_hierarchy_bulk_bitwise(hier):
    for ci in range(int(hier["n_cases"])):
        P, B, dim, nc, ng = map(int, hier[f"c{ci}_shape"])
        h = ref.Hierarchy.from_rows(hier[f"c{ci}_pages"], nc, ng)
        assert np.array_equal(h.chunk_vectors, hier[f"c{ci}_bulk_chunks"])
        assert np.array_equal(h.grid_vectors, hier[f"c{ci}_bulk_grids"])
        # incremental == batch within 1e-10 (test_hierarchy.py:79-91)
        np.testing.assert_allclose(h.grid_vectors, hier[f"c{ci}_grids"], rtol=1e-10, atol=1e-12)


def test_hierarchy_order_error():
    h = ref.Hierarchy(4, 2, 2)
    h.fold(np.zeros(4), 0)
    with pytest.raises(ValueError):
        h.fold(np.zeros(4), 2)


def test_selection_instances_bitwise(sel):
    for i in range(int(sel["n_instances"])):
        p = f"i{i}_"
        cfg = _cfg(sel[p + "cfg"])
        vec = sel[p + "vectors"]
        tail = sel[p + "tail"]
        h = ref.Hierarchy.from_rows(vec, cfg.pages_per_chunk, cfg.chunks_per_grid)
        a, src = ref.anchor(h.page_vectors, cfg.window_pages, tail if len(tail) else None)
        assert np.array_equal(a, sel[p + "anchor"]), i
        assert list(src) == list(sel[p + "anchor_sources"])
        v_all, splits = h.coalesced()
        assert list(splits) == list(sel[p + "splits"])
        s = ref.score(v_all, a)
        assert np.array_equal(s, sel[p + "scores"]), i
        g, c, _ = splits
        p2c, c2g = h.parent_maps()
        got, _ = ref.prune(s[:g], s[g:g + c], s[g + c:], p2c, c2g, cfg.ratios)
        assert np.array_equal(got, sel[p + "selected"]), i
        flat = ref.flat_topk(a, h.page_vectors, int(sel[p + "flat_k"]))
        assert np.array_equal(flat, sel[p + "flat"]), i
        table = list(sel[p + "table"])
        pages, prov = ref.working_set(got, len(table), cfg.window_pages, int(sel[p + "sinks"]))
        assert pages == list(sel[p + "ws_pages"]), i
        code = {"semantic": 1, "window": 2, "sink": 3}
        assert [code[prov[q]] for q in pages] == list(sel[p + "ws_prov"])
        assert ref.gather(table, pages) == list(sel[p + "ws_phys"])


def test_known_answer_cascade_and_ties():
    # test_selection.py:149-161: S_p=[4,3,2,1], rho=(1,1,.5) -> {0,1}
    p2c, c2g = np.zeros(4, int), np.zeros(1, int)
    got, _ = ref.prune(np.array([1.0]), np.array([1.0]), np.array([4.0, 3.0, 2.0, 1.0]), p2c, c2g,
                       (1.0, 1.0, 0.5))
    assert list(got) == [0, 1]
    # all-zero tie -> lower indices (test_selection.py:185-195)
    got, _ = ref.prune(np.zeros(1), np.zeros(1), np.zeros(4), p2c, c2g, (1.0, 1.0, 0.5))
    assert list(got) == [0, 1]
    # working-set union example (test_selection.py:242-246)
    pages, prov = ref.working_set([5], 8, 1, 1)
    assert pages == [0, 5, 7] and prov == {0: "sink", 5: "semantic", 7: "window"}


def test_uncertainty_golden():
    doc = json.loads((GOLD / "uncertainty.json").read_text())
    for r in doc["rows"]:
        assert ref.entropy(r["probs"]) == r["entropy"]
    k = doc["known"]
    assert abs(k["uniform8"] - np.log(8)) < 1e-12 and k["onehot"] == 0.0
    assert abs(k["half_quarter"] - 1.5 * np.log(2)) < 1e-12
    means, vars_ = [], []
    for pg in doc["pages"]:
        m, v, n = ref.page_stats(pg["entropies"])
        assert (m, v, n) == (pg["mean"], pg["var"], pg["n"])
        means.append(m)
        vars_.append(v)
    cal = doc["calibration"]
    th = ref.calibrate(means, vars_, cal["percentile"])
    assert th == (cal["tau_H"], cal["tau_V"])
    for pg, t in zip(doc["pages"], doc["trigger"]):
        assert ref.check_trigger(pg["mean"], pg["var"], *th, "joint") == t["joint"]
        assert ref.check_trigger(pg["mean"], pg["var"], *th, "any") == t["any"]
    assert ref.check_trigger(th[0], th[1], *th) is False and doc["at_threshold"] is False


def test_uncertainty_errors():
    with pytest.raises(ValueError):
        ref.entropy([0.5, 0.6])
    with pytest.raises(ValueError):
        ref.entropy([-0.1, 1.1])
    with pytest.raises(ValueError):
        ref.page_stats([])


def _policy(p):
    if p.startswith("fixed("):
        return ("fixed", int(p[6:-1]))
    return (p, None)


def test_decode_loop_golden():
    runs = json.loads((GOLD / "decode_loop.json").read_text())
    for run in runs:
        spec = dict(run["spec"])
        sched = tuple(tuple(x) for x in spec.pop("instability_schedule"))
        load = ref.workload(**spec, instability_schedule=sched)
        cfg = _cfg(run["cfg"])
        tau = run["tau"] if run["policy"] == "dynamic" else None
        steps, fired = ref.decode_loop(load, cfg, _policy(run["policy"]), tau)
        assert [s.trigger_fired for s in steps] == run["fired"], run["policy"]
        assert [s.working_set_size for s in steps] == run["ws_size"]
        assert [s.recall for s in steps] == run["recall"]
        assert [s.working_set for s in steps] == [w["pages"] for w in run["working_sets"]]


def test_attention_restatement_vs_dense():
    """The attention oracle is unpinned by the reference (simulate.py:186 only
    counts ops); check it against an independent dense formulation."""
    rng = np.random.default_rng(3)
    n_phys, H, B, d, Hq = 9, 2, 4, 8, 4
    K = rng.standard_normal((n_phys, H, B, d))
    V = rng.standard_normal((n_phys, H, B, d))
    q = rng.standard_normal((2, Hq, d))
    bt = np.array([[3, 1, 7, 0], [5, 2, 0, 0]])
    wl, fill = np.array([4, 2]), np.array([3, 1])
    o, lse = attn_ref.sparse_decode(q, K, V, bt, wl, fill, 0.3)
    for s in range(2):
        toks_k, toks_v = [], []
        for i in range(wl[s]):
            n = fill[s] if i == wl[s] - 1 else B
            toks_k.append(K[bt[s, i], :, :n])
            toks_v.append(V[bt[s, i], :, :n])
        Ks, Vs = np.concatenate(toks_k, axis=1), np.concatenate(toks_v, axis=1)
        for h in range(Hq):
            z = Ks[h // 2] @ q[s, h] * 0.3
            w = np.exp(z) / np.exp(z).sum()
            np.testing.assert_allclose(o[s, h], w @ Vs[h // 2], rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(lse[s, h], np.log(np.exp(z).sum()), rtol=1e-12)


def test_attention_bf16_bound_covers_kernel_rounding():
    """oracle/attention.bf16_bound holds for an emulation of K4's rounding
    (fp32 scores and exp, P rounded to bf16 for the PV product, fp32 l from
    unrounded p, bf16 output) — including one-page working sets."""
    import torch

    from oracle import attention as attn

    rng = np.random.default_rng(3)
    bf = lambda x: torch.as_tensor(x, dtype=torch.float32).to(torch.bfloat16).double().numpy()
    worst = 0.0
    for trial in range(40):
        B, d, hkv, grp = 32, 64, 2, 4
        n_phys = 12
        ws = int(rng.integers(1, 5))
        fill = int(rng.integers(1, B + 1))
        kp = bf(rng.standard_normal((n_phys, hkv, B, d)) * rng.choice([0.5, 1.0, 3.0]))
        vp = bf(rng.standard_normal((n_phys, hkv, B, d)))
        q = bf(rng.standard_normal((1, hkv * grp, d)))
        bt = [rng.choice(n_phys, size=ws, replace=False)]
        scale = 1.0 / np.sqrt(d)
        o_ref, _ = attn.sparse_decode(q, kp, vp, bt, [ws], [fill], scale)
        tol = attn.bf16_bound(q, kp, vp, bt, [ws], [fill], scale, o_ref)
        for h in range(hkv):
            K = attn.gather_tokens(kp, bt[0], ws, fill, h).astype(np.float32)
            V = attn.gather_tokens(vp, bt[0], ws, fill, h).astype(np.float32)
            for g in range(grp):
                qh = h * grp + g
                z = (K @ q[0, qh].astype(np.float32)) * np.float32(scale)
                p = np.exp(z - z.max()).astype(np.float32)
                o = (bf(p).astype(np.float32) @ V) / p.sum(dtype=np.float32)
                err = np.abs(bf(o) - o_ref[0, qh])
                assert np.all(err <= tol[0, qh]), (trial, (err / tol[0, qh]).max())
                worst = max(worst, float((err / tol[0, qh]).max()))
    assert worst > 0.05  # the bound is not vacuous


# ------------------------------------------------------ acceptance criteria + cfg1 demo run
def _acceptance():
    return json.loads((GOLD / "acceptance.json").read_text())


def c2_instances():
    """Inputs of test_acceptance.py:68-86, re-drawn with the same RNG calls."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        n_pages = int(rng.integers(1, 513))
        dim = int(rng.integers(8, 257))
        rho_p = float(rng.uniform(0.05, 1.0))
        rows = rng.standard_normal((n_pages, dim))
        a = rng.standard_normal(dim)
        yield rows, a, rho_p


def c3_instances():
    """Inputs of test_acceptance.py:89-112 (sinks, window, scores, k)."""
    rng = np.random.default_rng(2)
    for trial in range(1000):
        n_pages = int(rng.integers(1, 128))
        sinks = int(rng.integers(0, 5))
        window = int(rng.integers(1, 9))
        mode = trial % 3
        if mode == 0:
            scores = np.zeros(n_pages)
        elif mode == 1:
            scores = -np.abs(rng.standard_normal(n_pages))
        else:
            scores = rng.standard_normal(n_pages)
        k = int(rng.integers(0, n_pages + 1))
        yield n_pages, sinks, window, scores, k


def test_acceptance_c1_c2_c3_oracle():
    doc = _acceptance()
    rng = np.random.default_rng(0)
    h = ref.Hierarchy.from_rows(rng.standard_normal((2048, 32)), 8, 8)
    a = rng.standard_normal(32)
    v_all, (g, c, p) = h.coalesced()
    s = v_all @ a
    p2c, c2g = h.parent_maps()
    for name in ("aggressive", "moderate", "conservative"):
        sel, _ = ref.prune(s[:g], s[g:g + c], s[g + c:], p2c, c2g, PRESETS[name])
        assert sel.tolist() == doc["c1"][name], name
    for (rows, a, rho_p), want in zip(c2_instances(), doc["c2"]):
        h = ref.Hierarchy.from_rows(rows, 4, 4)
        v_all, (g, c, p) = h.coalesced()
        s = v_all @ a
        p2c, c2g = h.parent_maps()
        hier, _ = ref.prune(s[:g], s[g:g + c], s[g + c:], p2c, c2g, (1.0, 1.0, rho_p))
        flat = ref.flat_topk(a, h.page_vectors, int(np.ceil(rho_p * rows.shape[0])))
        assert hier.tolist() == want == flat.tolist()
    for (n, sinks, window, scores, k), want in zip(c3_instances(), doc["c3"]):
        sel = np.sort(ref.top_k(scores, k))
        assert sel.tolist() == want["selected"]
        pages, prov = ref.working_set(sel, n, window, sinks)
        assert pages == want["pages"] and [prov[q] for q in pages] == want["prov"]


def test_cfg1_demo_run_oracle():
    """BASELINE configs[0]: the reference CPU demo (seed 0, dim 1024, 256 pages
    of 16, policy always) — prefill snapshot checksums, working sets, budgets."""
    run = _acceptance()["cfg1"]
    load = ref.workload(**run["spec"])
    cfg = SelectionConfig(page_size=16)
    B = 16
    h = ref.Hierarchy(1024, cfg.pages_per_chunk, cfg.chunks_per_grid)
    for q in range(run["spec"]["context_pages"]):
        h.fold_page(load["context_keys"][q * B:(q + 1) * B], q)
    assert h.snapshot() == run["prefill_snapshot"]
    steps, _ = ref.decode_loop(load, cfg, ("always", None))
    assert [s.working_set for s in steps] == run["working_sets"]
    assert [s.working_set_size for s in steps] == run["ws_size"]
    assert [s.budget_fraction_semantic for s in steps] == run["budget_semantic"]
    assert [s.recall for s in steps] == run["recall"]
