"""Tensor-core selection (summary_dtype 3, k_select_tc.cuh) parity.

The tcgen05 pass scores fp16 mirrors of the summary rows and certifies every
candidate against each level's cut; the rows it cannot certify are rescored
exactly from the f64 rows.  The bar is therefore the f64 one:
selected index sets, working sets and block tables identical to the oracle
cascade on f64 scores (selection.py:62-111) and to the device f64 scan.

The certificates themselves are tested directly: for every candidate of
every level, lo <= (exact f64 score) <= hi, certainly-in rows are selected
and certainly-out rows are not; and with fp16-exact rows and anchor (so the
only error left is the tensor core's f32 accumulation) the observed error
stays inside the un-inflated accumulation model the bound uses.
"""

import ctypes as C
import math

import numpy as np
import pytest
import torch

from oracle import pagesel_ref as ref
from paper_2602_20732_b200 import _lib
from paper_2602_20732_b200.config import SelectionConfig, preset_config

pytestmark = pytest.mark.gpu

GAMMA_MODEL = 18.0 * 2.0**-22  # kGammaTc before its 4x inflation


def _lib_dbg():
    lib = _lib.load()
    lib.chess_debug_select_tc_level.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
    lib.chess_debug_tc_read.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32] + [C.c_void_p] * 5
    return lib


def _scfg(cfg, force_all=True):
    return _lib.ChessSelectCfg(cfg.rho_grid, cfg.rho_chunk, cfg.rho_page, 0, int(force_all))


def _select(st, cfg):
    sc = _scfg(cfg)
    _lib.call("chess_select", st.ref, C.byref(sc), _lib.stream_ptr())
    torch.cuda.synchronize()


def _rows(rng, kind, n, dim):
    if kind == "gauss":
        return rng.standard_normal((n, dim))
    if kind == "planted":  # workload.py-style: a few rows share a strong direction
        r = rng.standard_normal((n, dim)) / math.sqrt(dim)
        sig = rng.standard_normal(dim)
        sig /= np.linalg.norm(sig)
        hot = rng.choice(n, size=max(1, n // 50), replace=False)
        r[hot] += 4.0 * sig
        r[-4:] += 2.0 * sig  # the window drives the anchor towards the signal
        return r
    if kind == "dups":  # exact duplicate rows -> exact score ties at the cut
        base = rng.standard_normal((max(1, n // 4), dim))
        return base[rng.integers(0, base.shape[0], size=n)]
    if kind == "wide":  # dynamic range beyond fp16: overflow rows go uncertain
        r = rng.standard_normal((n, dim))
        r *= 10.0 ** rng.integers(-6, 6, size=(n, 1))
        return r
    if kind == "tiny":  # fp16 subnormal territory
        return rng.standard_normal((n, dim)) * 1e-7
    raise ValueError(kind)


def _instances(rng, n):
    kinds = ["gauss", "planted", "dups", "wide", "tiny"]
    for t in range(n):
        P = int(rng.integers(1, 900))
        dim = int(rng.choice([2112, 2560, 4096, 8192]))
        nc = int(rng.choice([8, 8, 16]))
        ng = int(rng.choice([8, 8, 16]))
        rhos = [float(rng.choice([1.0, 0.5, 0.2, 0.1, float(rng.uniform(0.05, 1.0))])) for _ in range(3)]
        cfg = SelectionConfig(pages_per_chunk=nc, chunks_per_grid=ng, rho_grid=rhos[0], rho_chunk=rhos[1],
                              rho_page=rhos[2], window_pages=int(rng.integers(1, 9)),
                              sink_pages=int(rng.integers(0, 4)))
        yield P, dim, cfg, kinds[t % len(kinds)]


def _oracle(h, cfg):
    a, _ = ref.anchor(h.page_vectors, cfg.window_pages)
    s = [m @ a for m in (h.grid_vectors, h.chunk_vectors, h.page_vectors)]
    p2c, c2g = h.parent_maps()
    return ref.prune(s[0], s[1], s[2], p2c, c2g, cfg.ratios)


def test_tc_selection_equals_f64():
    """End to end: f16tc selection == f64 oracle == device f64 scan, on
    Gaussian, planted, duplicate-row (exact ties), fp16-overflow and
    fp16-subnormal summaries, fan-outs 8 and 16."""
    from helpers import index_state, load_vectors, read_selection, set_tables

    rng = np.random.default_rng(21)
    for P, dim, cfg, kind in _instances(rng, 20):
        st = index_state(3, dim, 900, cfg, summary_dtype="f16tc")
        st64 = index_state(3, dim, 900, cfg, summary_dtype="f64")
        hs = []
        for slot in range(3):
            n = max(1, P - 41 * slot)
            rows = _rows(rng, kind, n, dim)
            load_vectors(st, slot, rows)
            load_vectors(st64, slot, rows)
            set_tables(st, slot, n + slot, cfg.sink_pages)
            set_tables(st64, slot, n + slot, cfg.sink_pages)
            hs.append((ref.Hierarchy.from_rows(rows, cfg.pages_per_chunk, cfg.chunks_per_grid), n))
        _select(st, cfg)
        _select(st64, cfg)
        for slot, (h, n) in enumerate(hs):
            sel, info = _oracle(h, cfg)
            sem, ws, bt, prov = read_selection(st, slot)
            msg = f"P={n} dim={dim} kind={kind} cfg={cfg}"
            np.testing.assert_array_equal(sem, sel, err_msg=msg)
            sem64, ws64, bt64, prov64 = read_selection(st64, slot)
            np.testing.assert_array_equal(sem, sem64, err_msg=msg)
            np.testing.assert_array_equal(ws, ws64, err_msg=msg)
            np.testing.assert_array_equal(bt, bt64, err_msg=msg)
            np.testing.assert_array_equal(prov, prov64, err_msg=msg)
            stats = st.sel_stats[slot].cpu().numpy()
            G, Cn, Pn = h.counts
            assert tuple(stats[:5]) == (G, Cn, Pn, info["active_c"], info["active_p"]), msg
        del st, st64
    torch.cuda.empty_cache()


def test_tc_selection_large_candidate_sets():
    """Candidate lists around and above the tail's shared-memory capacity
    (1024): the certification thresholds come from a bitonic sort of the
    bound keys up to 1024 candidates and from the radix top-k above it; both
    must give the f64 selection."""
    from helpers import index_state, load_vectors, read_selection, set_tables

    rng = np.random.default_rng(33)
    cases = [(1024, "dups", (1.0, 1.0, 0.3)), (1025, "planted", (1.0, 1.0, 0.1)),
             (2600, "gauss", (1.0, 1.0, 0.05)), (2600, "dups", (1.0, 0.9, 0.5)), (1900, "wide", (1.0, 1.0, 0.2))]
    for P, kind, rhos in cases:
        cfg = SelectionConfig(pages_per_chunk=8, chunks_per_grid=8, rho_grid=rhos[0], rho_chunk=rhos[1],
                              rho_page=rhos[2], window_pages=4, sink_pages=1)
        dim = 2112
        st = index_state(2, dim, P + 8, cfg, summary_dtype="f16tc")
        hs = []
        for slot in range(2):
            n = P - 7 * slot
            rows = _rows(rng, kind, n, dim)
            load_vectors(st, slot, rows)
            set_tables(st, slot, n + slot, cfg.sink_pages)
            hs.append((ref.Hierarchy.from_rows(rows, cfg.pages_per_chunk, cfg.chunks_per_grid), n))
        _select(st, cfg)
        for slot, (h, n) in enumerate(hs):
            sel, info = _oracle(h, cfg)
            sem, ws, bt, prov = read_selection(st, slot)
            np.testing.assert_array_equal(sem, sel, err_msg=f"P={n} kind={kind} rhos={rhos}")
        del st
    torch.cuda.empty_cache()


def test_tc_mirror_rows_and_bounds():
    """mirror16_kernel: fp16 rows are the round-to-nearest images of the f64
    rows; the stash holds ||v - h|| and ||h|| rounded up (within 2^-19)."""
    from helpers import index_state, load_vectors, set_tables

    rng = np.random.default_rng(3)
    cfg = preset_config("aggressive")
    st = index_state(2, 2112, 300, cfg, summary_dtype="f16tc")
    for slot in range(2):
        rows = _rows(rng, "wide" if slot else "gauss", 260, 2112)
        load_vectors(st, slot, rows)
        set_tables(st, slot, 260, 1)
    torch.cuda.synchronize()
    for which, m64 in enumerate((st.grid_vec64, st.chunk_vec64, st.page_vec64)):
        h, stash = st.mirror16(which)
        n = (5, 33, 260)[which]
        for slot in range(2):
            v = m64[slot, :n].cpu().numpy()
            hh = h[slot, :n].cpu().numpy()
            np.testing.assert_array_equal(hh, v.astype(np.float16))
            hd = hh.astype(np.float64)
            with np.errstate(invalid="ignore", over="ignore"):
                err = np.sqrt(((v - hd) ** 2).sum(axis=1))
                nrm = np.sqrt((hd**2).sum(axis=1))
            got = stash[slot, :n].cpu().numpy()
            fin = np.isfinite(err)
            assert np.all(got[fin, 0] >= err[fin]) and np.all(got[fin, 0] <= err[fin] * (1 + 2.0**-19) + 1e-300)
            assert np.all(np.isinf(got[~fin, 0]))
            finn = np.isfinite(nrm)
            assert np.all(got[finn, 1] >= nrm[finn]) and np.all(got[finn, 1] <= nrm[finn] * (1 + 2.0**-19))


def _level_rows(h, level):
    return (h.grid_vectors, h.chunk_vectors, h.page_vectors)[level]


def test_tc_certified_intervals_hold():
    """Every candidate of every level: lo <= exact f64 score <= hi; class 1
    rows are kept and class 0 rows are not (the oracle's kept sets)."""
    from helpers import index_state, load_vectors, set_tables

    lib = _lib_dbg()
    rng = np.random.default_rng(8)
    cfg = SelectionConfig(rho_grid=0.5, rho_chunk=0.2, rho_page=0.1)
    P, dim, B = 3000, 4096, 3
    st = index_state(B, dim, P, cfg, summary_dtype="f16tc")
    hs = []
    for slot in range(B):
        rows = _rows(rng, ("gauss", "planted", "dups")[slot], P, dim)
        load_vectors(st, slot, rows)
        set_tables(st, slot, P, 1)
        hs.append(ref.Hierarchy.from_rows(rows, 8, 8))
    _select(st, cfg)  # leaves every level's candidate list in the workspace
    n_checked = n_unc = 0
    worst = 0.0
    for level in range(3):
        sc = _scfg(cfg)
        _lib.check(lib.chess_debug_select_tc_level(st.ref, C.byref(sc), level, _lib.stream_ptr()), "tc level")
        torch.cuda.synchronize()
        for slot, h in enumerate(hs):
            a, _ = ref.anchor(h.page_vectors, cfg.window_pages)
            sel, info = _oracle(h, cfg)
            G, Cn, Pn = h.counts
            n = (G, info["active_c"], info["active_p"])[level]
            lo, hi = np.zeros(n), np.zeros(n)
            cls, cand, meta = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(4, np.int32)
            _lib.check(lib.chess_debug_tc_read(st.ref, slot, level, n, lo.ctypes.data, hi.ctypes.data,
                                               cls.ctypes.data, meta.ctypes.data, cand.ctypes.data), "read")
            ids = np.arange(n) if level == 0 else cand
            exact = _level_rows(h, level)[ids] @ a
            k = math.ceil(cfg.ratios[level] * n)
            if k >= n:
                continue
            assert np.all(lo <= exact) and np.all(exact <= hi), f"level {level} slot {slot}"
            half = (hi - lo) / 2
            worst = max(worst, float(np.max(np.abs(exact - (hi + lo) / 2) / half)))
            kept = set(sel.tolist()) if level == 2 else set(info["kept_g" if level == 0 else "kept_c"])
            for i, c in zip(ids.tolist(), cls.tolist()):
                if c == 1:
                    assert i in kept
                elif c == 0:
                    assert i not in kept
            n_checked += n
            n_unc += int((cls == 2).sum())
    print(f"tc certificates: {n_checked} candidates, {n_unc} uncertain, max |err|/bound {worst:.3e}")
    assert n_unc < n_checked // 4


def test_tc_accumulation_error_model():
    """fp16-exact rows and a one-page window (anchor = an fp16-exact row, so
    lo = rem = err = 0): what is left of |exact - approx| is the tensor
    core's f32 accumulation, which must stay within the model 18*2^-22 of
    sum |a||h| per window that kGammaTc inflates 4x."""
    from helpers import index_state, load_vectors, set_tables

    lib = _lib_dbg()
    rng = np.random.default_rng(17)
    cfg = SelectionConfig(rho_grid=0.5, rho_chunk=0.5, rho_page=0.5, window_pages=1)
    P, dim = 2048, 8192
    st = index_state(1, dim, P, cfg, summary_dtype="f16tc")
    mant = 1.0 + rng.integers(0, 1024, size=(P, dim)) / 1024.0
    expo = rng.integers(-8, 8, size=(P, dim)).astype(np.float64)
    rows = np.where(rng.random((P, dim)) < 0.5, -1.0, 1.0) * mant * 2.0**expo
    assert np.array_equal(rows.astype(np.float16).astype(np.float64), rows)
    # page_size 1 keeps page vectors = rows; chunk/grid centroids are not
    # fp16-exact, so only the page level (level 2) isolates the accumulation
    load_vectors(st, 0, rows)
    set_tables(st, 0, P, 1)
    _select(st, cfg)
    h = ref.Hierarchy.from_rows(rows, 8, 8)
    sc = _scfg(cfg)
    _lib.check(lib.chess_debug_select_tc_level(st.ref, C.byref(sc), 2, _lib.stream_ptr()), "tc level")
    torch.cuda.synchronize()
    _, info = _oracle(h, cfg)
    n = info["active_p"]
    lo, hi, cand = np.zeros(n), np.zeros(n), np.zeros(n, np.int32)
    _lib.check(lib.chess_debug_tc_read(st.ref, 0, 2, n, lo.ctypes.data, hi.ctypes.data, None, None,
                                       cand.ctypes.data), "read")
    a = rows[-1]
    exact = rows[cand] @ a
    approx = (lo + hi) / 2
    mag = np.abs(rows[cand]) @ np.abs(a)
    ratio = np.abs(exact - approx) / mag
    print(f"tensor-core f32 accumulation: max |err| / sum|a h| = {ratio.max():.3e} "
          f"(model {GAMMA_MODEL:.3e} per window, {n} rows)")
    assert ratio.max() <= GAMMA_MODEL


def test_tc_select_at_bench_cfg5_state():
    """cfg5's state (Llama-3-70B shape: D = 80 x 8 x 128 = 81920, 40 slices
    of 2048; P = 4096; batch 8), where the bench also runs the tensor-core
    selection: every slot's selection equals the f64 cascade."""
    from paper_2602_20732_b200.engine import ChessDecoder
    from paper_2602_20732_b200.synthetic import SyntheticDecode

    wl = SyntheticDecode("cfg5", batch=8, gen_pages=4, ring=2, kv_budget_gib=8, summary_dtype="f16tc")
    st, sh = wl.st, wl.shape
    cfg = preset_config("aggressive", page_size=sh.page_size)
    dec = ChessDecoder(st, cfg, policy="every_step")
    wl.prefill(dec)
    P, D = wl.P, sh.dim
    Cn = math.ceil(P / 8)
    G = math.ceil(Cn / 8)
    p2c, c2g = np.arange(P) // 8, np.arange(Cn) // 8
    for s in range(8):
        sc = [torch.mv(m[s, :n, :D], st.anchor[s, :D]).cpu().numpy()
              for m, n in ((st.grid_vec64, G), (st.chunk_vec64, Cn), (st.page_vec64, P))]
        sel, _ = ref.prune(sc[0], sc[1], sc[2], p2c, c2g, cfg.ratios)
        sem = st.semantic[s, : int(st.n_semantic[s])].cpu().numpy()
        np.testing.assert_array_equal(sem, sel, err_msg=f"slot {s}")
    del wl, st, dec
    torch.cuda.empty_cache()


def test_tc_select_at_bench_cfg3_state():
    """The bench's headline state (cfg3: D = 32768, P = 4096, batch 16,
    planted relevance, built by K1b) with fp16 tensor-core scoring: every
    slot's selection equals the oracle cascade on f64 scores of the f64
    summary rows (torch f64 GEMV)."""
    from paper_2602_20732_b200.engine import ChessDecoder
    from paper_2602_20732_b200.synthetic import SyntheticDecode

    wl = SyntheticDecode("cfg3", batch=16, gen_pages=4, ring=2, kv_budget_gib=8, summary_dtype="f16tc")
    st, sh = wl.st, wl.shape
    cfg = preset_config("aggressive", page_size=sh.page_size)
    dec = ChessDecoder(st, cfg, policy="every_step")
    wl.prefill(dec)
    P, D = wl.P, sh.dim
    Cn = math.ceil(P / 8)
    G = math.ceil(Cn / 8)
    p2c, c2g = np.arange(P) // 8, np.arange(Cn) // 8
    for s in range(16):
        sc = [torch.mv(m[s, :n, :D], st.anchor[s, :D]).cpu().numpy()
              for m, n in ((st.grid_vec64, G), (st.chunk_vec64, Cn), (st.page_vec64, P))]
        sel, info = ref.prune(sc[0], sc[1], sc[2], p2c, c2g, cfg.ratios)
        sem = st.semantic[s, : int(st.n_semantic[s])].cpu().numpy()
        np.testing.assert_array_equal(sem, sel, err_msg=f"slot {s}")
        stats = st.sel_stats[s].cpu().numpy()
        assert tuple(stats[:5]) == (G, Cn, P, info["active_c"], info["active_p"])
        pages, _ = ref.working_set(sel, P, cfg.window_pages, 1)
        np.testing.assert_array_equal(st.ws_logical[s, : int(st.ws_len[s])].cpu().numpy(), pages)
        np.testing.assert_array_equal(st.block_table[s, : len(pages)].cpu().numpy(), wl.table_cpu[s, pages].numpy())
    # the engine's overlapped step runs the same pass with deferred working
    # sets on fewer CTAs (96 of 148): identical selections, working sets after
    # the flush
    want = st.semantic.clone(), st.n_semantic.clone(), st.ws_logical.clone(), st.block_table.clone()
    st.semantic.fill_(-1)
    dec.select(force_all=True, defer_ws=True)
    _lib.call("chess_flush_working_sets", st.ref, _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(st.n_semantic, want[1])
    for s in range(16):
        n = int(want[1][s])
        assert torch.equal(st.semantic[s, :n], want[0][s, :n]), s
    assert torch.equal(st.ws_logical, want[2]) and torch.equal(st.block_table, want[3])
    del wl, st, dec
    torch.cuda.empty_cache()
