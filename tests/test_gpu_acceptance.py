"""The reference's release criteria and its CPU demo run, through the device
shim (the drop-in `pagesel` mirror whose numeric work runs in
libchess_b200.so), against outputs the reference itself produced
(tests/golden/acceptance.json, made by tests/golden/make_golden.py):

  C1  budget arithmetic on 2048 pages, every preset  (test_acceptance.py:45-65)
  C2  200 random flat-equivalence instances           (test_acceptance.py:68-86)
  C3  1000 working-set safety fuzz cases              (test_acceptance.py:89-112)
  cfg1  BASELINE configs[0], the reference CPU demo run (seed 0, dim 1024,
        256 context pages of 16, policy always): prefill snapshot checksums,
        per-page working sets, semantic budgets, recall

Bar: index outputs bit-exact; f64 summaries bit-exact (checksums).
"""

import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2602_20732_b200 import _lib
from paper_2602_20732_b200 import pagesel as ps
from test_oracle_golden import c2_instances, c3_instances

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def doc():
    return json.loads((GOLD / "acceptance.json").read_text())


def test_c1_budgets(doc):
    rng = np.random.default_rng(0)
    index = ps.HierarchyIndex.from_page_vectors(rng.standard_normal((2048, 32)), 8, 8)
    anchor = ps.QueryAnchor(v=rng.standard_normal(32), source_pages=[])
    scores = ps.score_all(anchor, *index.coalesced_matrix())
    for name in ("aggressive", "moderate", "conservative"):
        sel = ps.hierarchical_prune(*scores, index.page_to_chunk, index.chunk_to_grid, ps.preset_config(name))
        assert [int(i) for i in sel] == doc["c1"][name], name


def test_c2_flat_equivalence(doc):
    for (rows, a, rho_p), want in zip(c2_instances(), doc["c2"]):
        n = rows.shape[0]
        index = ps.HierarchyIndex.from_page_vectors(rows, 4, 4)
        cfg = ps.SelectionConfig(pages_per_chunk=4, chunks_per_grid=4, rho_grid=1.0, rho_chunk=1.0, rho_page=rho_p)
        anchor = ps.QueryAnchor(v=a, source_pages=[])
        s = ps.score_all(anchor, *index.coalesced_matrix())
        hier = ps.hierarchical_prune(*s, index.page_to_chunk, index.chunk_to_grid, cfg)
        flat = ps.oracle_flat_topk(anchor, index.page_vectors, int(np.ceil(rho_p * n)))
        assert [int(i) for i in hier] == want == [int(i) for i in flat], n


def test_c3_safety_fuzz(doc):
    """Top-k on the device (chess_topk, ties to the lower index) feeding the
    device working set (chess_working_set via reconstruct_working_set)."""
    ws_buf = torch.empty(16 * 128, dtype=torch.uint8, device="cuda")
    idx = torch.empty(128, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    for (n, sinks, window, scores, k), want in zip(c3_instances(), doc["c3"]):
        sc = torch.as_tensor(scores, dtype=torch.float64, device="cuda")
        _lib.call("chess_topk", _lib.ptr(sc), n, k, None, _lib.ptr(idx), _lib.ptr(cnt), 1, _lib.ptr(ws_buf),
                  _lib.stream_ptr())
        sel = idx[: int(cnt.item())].cpu().tolist()
        assert sel == want["selected"]
        cfg = ps.SelectionConfig(window_pages=window, sink_pages=sinks)
        ws = ps.reconstruct_working_set(np.asarray(sel, dtype=np.int64),
                                        ps.SequenceState(page_table=list(range(n)), sink_count=sinks), cfg)
        assert list(ws.pages) == want["pages"]
        assert [ws.provenance[p] for p in ws.pages] == want["prov"]


def test_cfg1_demo_run(doc):
    run = doc["cfg1"]
    spec = ps.WorkloadSpec(**run["spec"])
    cfg = ps.preset_config("aggressive", page_size=16)
    wl = ps.generate_workload(spec)
    store = ps.PagedKvStore(spec.context_pages + spec.generation_pages + 1, spec.dim, page_size=16)
    seq = store.create_sequence(cfg)
    index = ps.HierarchyIndex(spec.dim, cfg.pages_per_chunk, cfg.chunks_per_grid)
    for t in range(wl.context_keys.shape[0]):
        ev = store.append_token(seq, wl.context_keys[t], wl.context_values[t])
        if ev.sealed:
            index.finalize_page(store.page(ev.page_id), ev.logical_index)
    assert index.snapshot() == run["prefill_snapshot"]
    rep = ps.run_decode_loop(spec, cfg, run["policy"])
    assert rep.working_sets == run["working_sets"]
    assert [s.working_set_size for s in rep.steps] == run["ws_size"]
    assert [s.budget_fraction_semantic for s in rep.steps] == run["budget_semantic"]
    assert [s.recall for s in rep.steps] == run["recall"]
    summ = rep.summary()
    for key in ("steps", "trigger_count", "mean_recall", "mean_budget_semantic", "zero_copy_ok"):
        assert summ[key] == run["summary"][key], key


def test_prune_workspace_exact_size_large():
    """chess_prune at thousands of pages writes nothing past
    chess_prune_workspace_bytes (a canary region after the exact size)."""
    rng = np.random.default_rng(3)
    P = 4096
    h = ps.HierarchyIndex.from_page_vectors(rng.standard_normal((P, 64)), 8, 8)
    anchor = ps.QueryAnchor(v=rng.standard_normal(64), source_pages=[])
    s_g, s_c, s_p = ps.score_all(anchor, *h.coalesced_matrix())
    G, Cn = s_g.numel(), s_c.numel()
    need = _lib.load().chess_prune_workspace_bytes(G, Cn, P)
    assert need == 16 * (G + Cn + P) + 4 * (G + Cn)
    buf = torch.full((need + 65536,), 0xA5, dtype=torch.uint8, device="cuda")
    out = torch.empty(P, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(3, dtype=torch.int32, device="cuda")
    p2c = torch.as_tensor(np.asarray(h.page_to_chunk), dtype=torch.int64, device="cuda")
    c2g = torch.as_tensor(np.asarray(h.chunk_to_grid), dtype=torch.int64, device="cuda")
    cfg = ps.preset_config("aggressive")
    _lib.call("chess_prune", _lib.ptr(s_g), G, _lib.ptr(s_c), Cn, _lib.ptr(s_p), P, _lib.ptr(p2c), _lib.ptr(c2g),
              cfg.rho_grid, cfg.rho_chunk, cfg.rho_page, _lib.ptr(out), _lib.ptr(cnt), _lib.ptr(buf), _lib.stream_ptr())
    torch.cuda.synchronize()
    assert bool((buf[need:] == 0xA5).all()), "prune wrote past its workspace"
    want = ps.hierarchical_prune(s_g, s_c, s_p, h.page_to_chunk, h.chunk_to_grid, cfg)
    assert out[: int(cnt[0])].cpu().tolist() == [int(i) for i in want]
