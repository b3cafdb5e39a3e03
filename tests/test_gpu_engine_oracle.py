"""The benchmarked product path — engine.ChessDecoder.step, one decode token
for the whole batch — against the oracle's page-granular decode loop
(oracle.pagesel_ref.decode_loop, a restatement of simulate.py:110-217 pinned
to the reference's own decode-loop goldens by tests/test_oracle_golden.py).

Per slot, a reference WorkloadSpec stream (workload.py:96-137: planted
relevant pages, generated keys carrying half the signal, an instability
schedule) drives the engine token by token at the cfg1 model shape (2 layers,
8 kv heads, head_dim 64: D = 1024, pages of 16).  Keys and values are stored
as bf16, so the oracle is fed the same bf16-rounded rows; the per-token
entropies are the reference's entropy(probs) (uncertainty.py:22-31), injected
through chess_record_entropy.

At every generated page, for never / always / fixed(3) / dynamic (thresholds
calibrated on a stable stream, uncertainty.py:59-83), sequential and
concurrent step, eager and CUDA-graph replay:
  * trigger decision fire[s]                          == oracle (bit-exact)
  * semantic set after the page's (re)selection       == oracle
  * working set + provenance at the seal, and again when the next page opens
    (the window counts the open tail, selection.py:131)  == oracle
  * block table                                        == page_table[ws] (gather)
f64 summaries and the tensor-core path (f16tc) are exact end to end; f32 mirrors are compared to the oracle
scoring the device's own f32 mirror rows (the selection kernel's parity bar,
tests/test_gpu_select.py).
"""

import math
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import attention as attn_ref
from oracle import pagesel_ref as ref
from paper_2602_20732_b200 import _lib
from paper_2602_20732_b200.config import preset_config
from paper_2602_20732_b200.engine import ChessDecoder
from paper_2602_20732_b200.state import DecodeState, Shape

pytestmark = pytest.mark.gpu

L, H, HQ, HD, B = 2, 8, 8, 64, 16  # cfg1 (BASELINE configs[0]) model shape
D = L * H * HD
P_CTX, G_PAGES, BATCH = 96, 10, 2
SCHEDULES = [((2, 2.0), (5, 2.0), (8, 3.0)), ((4, 2.0),)]
_LAST_STATE = [None]  # the state of the last decode-loop test (for path checks)
NAMES = {1: "semantic", 2: "window", 3: "sink"}


def _bf16(x):
    return torch.as_tensor(x, dtype=torch.float64).to(torch.bfloat16)


def _thresholds():
    """calibrate(collect_page_uncertainties(stable spec), 0.99) restated."""
    stable = ref.workload(seed=100, dim=64, context_pages=8, page_size=B, generation_pages=150, vocab=64)
    means, var = [], []
    for g in range(150):
        m, v, _ = ref.page_stats([ref.entropy(r) for r in stable["gen_probs"][g * B:(g + 1) * B]])
        means.append(m)
        var.append(v)
    return ref.calibrate(means, var, 0.99)


def _loads():
    loads = []
    for s in range(BATCH):
        w = ref.workload(seed=10 + s, dim=D, context_pages=P_CTX, page_size=B, generation_pages=G_PAGES,
                         instability_schedule=SCHEDULES[s], pages_per_chunk=8, vocab=64)
        # the device stores bf16 rows: feed the oracle the same rounded keys
        for k in ("context_keys", "context_values", "gen_keys", "gen_values"):
            w[k + "_bf16"] = _bf16(w[k])
            w[k] = w[k + "_bf16"].double().numpy()
        loads.append(w)
    return loads


def _policy_tuple(policy):
    if policy.startswith("fixed("):
        return ("fixed", int(policy[6:-1]))
    return (policy, None)


def _rows_to_pool(rows):
    """[n, D] rows (flattened (layer, kv_head, d)) -> [L, H, n, d]."""
    return rows.reshape(rows.shape[0], L, H, HD).permute(1, 2, 0, 3)


def _make_state(loads, summary_dtype, table):
    max_pages = P_CTX + G_PAGES + 2
    sh = Shape(batch=BATCH, layers=L, kv_heads=H, q_heads=HQ, head_dim=HD, page_size=B, pages_per_chunk=8,
               chunks_per_grid=8, max_pages=max_pages, window_pages=4, max_ws=max_pages,
               n_phys=BATCH * max_pages, summary_dtype=summary_dtype)
    st = DecodeState(sh)
    st.reset()
    st.k_pool.zero_()
    st.v_pool.zero_()
    for s, w in enumerate(loads):
        ck = _rows_to_pool(w["context_keys_bf16"]).cuda()
        cv = _rows_to_pool(w["context_values_bf16"]).cuda()
        for p in range(P_CTX):
            ph = int(table[s, p])
            st.k_pool[:, ph] = ck[:, :, p * B:(p + 1) * B]
            st.v_pool[:, ph] = cv[:, :, p * B:(p + 1) * B]
    st.page_table.copy_(torch.as_tensor(table, dtype=torch.int32))
    st.num_pages.fill_(P_CTX)
    st.tail_fill.fill_(B)
    st.token_count.fill_(P_CTX * B)
    st.sink_count.fill_(1)
    return st


def _device_ws(st, s):
    n = int(st.ws_len[s])
    return (st.ws_logical[s, :n].cpu().tolist(), st.block_table[s, :n].cpu().tolist(),
            [NAMES[int(x)] for x in st.ws_prov[s, :n].cpu().tolist()])


def _oracle_with_mirrors(st, s, cfg, sealed):
    """Oracle cascade over the device's f32 mirror rows (kernel-isolated bar)."""
    h = ref.Hierarchy(D, 8, 8)
    h.pages = list(st.page_vec64[s, :sealed, :D].cpu().numpy())
    G, C = math.ceil(math.ceil(sealed / 8) / 8), math.ceil(sealed / 8)
    a, _ = ref.anchor(h.page_vectors, cfg.window_pages)
    mats = (st.grid_vec32[s, :G, :D].double().cpu().numpy(), st.chunk_vec32[s, :C, :D].double().cpu().numpy(),
            st.page_vec32[s, :sealed, :D].double().cpu().numpy())
    sc = [m @ a for m in mats]
    p2c, c2g = np.arange(sealed) // 8, np.arange(C) // 8
    sel, _ = ref.prune(sc[0], sc[1], sc[2], p2c, c2g, cfg.ratios)
    return [int(i) for i in sel]


@pytest.mark.parametrize("summary_dtype", ["f64", "f32", "f16tc"])
@pytest.mark.parametrize("mode", ["sequential", "concurrent", "graph"])
@pytest.mark.parametrize("policy", ["never", "always", "fixed(3)", "dynamic"])
def test_engine_decode_matches_oracle_loop(policy, mode, summary_dtype):
    if summary_dtype != "f64" and mode != "concurrent":
        pytest.skip("mirrors: the benched (concurrent) mode only")
    # f16tc selects exactly what the f64 scores give (certified fp16 scan +
    # f64 rescoring; at D = 1024 the rows are short and go straight to f64)
    exact = summary_dtype in ("f64", "f16tc")
    cfg = preset_config("aggressive", page_size=B)
    tau = _thresholds() if policy == "dynamic" else None
    loads = _loads()
    rng = np.random.default_rng(7)
    max_pages = P_CTX + G_PAGES + 2
    table = rng.permutation(BATCH * max_pages).reshape(BATCH, max_pages)
    st = _make_state(loads, summary_dtype, table)
    _LAST_STATE[0] = st

    th = SimpleNamespace(tau_entropy=tau[0], tau_varentropy=tau[1]) if tau else None
    dec = ChessDecoder(st, cfg, policy=policy, thresholds=th,
                       concurrent_select=mode != "sequential")
    dec.build_index(torch.full((BATCH,), P_CTX, dtype=torch.int32, device="cuda"))
    dec.initial_selection()
    torch.cuda.synchronize()

    # oracle: the page loop per slot, plus the post-prefill selection
    want = []
    for s, w in enumerate(loads):
        steps, fired = ref.decode_loop(w, cfg, _policy_tuple(policy), tau)
        h = ref.Hierarchy(D, 8, 8)
        for p in range(P_CTX):
            h.fold_page(w["context_keys"][p * B:(p + 1) * B], p)
        init = list(range(P_CTX)) if policy == "never" else [int(i) for i in ref.select_for_index(h, cfg)[0]]
        want.append((steps, set(fired), init))
        assert st.n_semantic[s].item() == len(init)
        got = st.semantic[s, : len(init)].cpu().tolist()
        if exact or policy == "never":
            assert got == init, (s, "initial selection")
        else:
            assert got == _oracle_with_mirrors(st, s, cfg, P_CTX), (s, "initial selection")

    # per-token inputs
    g = torch.Generator(device="cuda").manual_seed(3)
    T = G_PAGES * B
    q_all = torch.randn((T, BATCH, L, HQ, HD), device="cuda", generator=g).to(torch.bfloat16)
    k_all = torch.stack([_rows_to_flat(w["gen_keys_bf16"]) for w in loads], dim=1).cuda()  # [T, b, D]
    v_all = torch.stack([_rows_to_flat(w["gen_values_bf16"]) for w in loads], dim=1).cuda()
    ent_all = torch.tensor([[ref.entropy(w["gen_probs"][t]) for w in loads] for t in range(T)],
                           dtype=torch.float64, device="cuda")
    out = torch.zeros((BATCH, L, HQ, HD), device="cuda", dtype=torch.bfloat16)
    graph = None
    if mode == "graph":
        sk, sv, sq, se = k_all[0].clone(), v_all[0].clone(), q_all[0].clone(), ent_all[0].clone()

    exp_sem = [w[2] for w in want]  # semantic set in effect per slot
    for t in range(T):
        gp, r = divmod(t, B)
        if mode == "graph" and t > 0:
            if graph is None:
                graph = dec.capture(sk, sv, sq, None, out, entropies=se)
            sk.copy_(k_all[t])
            sv.copy_(v_all[t])
            sq.copy_(q_all[t])
            se.copy_(ent_all[t])
            graph.replay()
        else:
            dec.step(k_all[t], v_all[t], q_all[t], None, out, entropies=ent_all[t])
        torch.cuda.synchronize()
        for s in range(BATCH):
            steps, fired, init = want[s]
            tab = table[s].tolist()
            if r == 0:
                # the page just opened: the window counts the open tail
                pages, prov = ref.working_set(exp_sem[s], P_CTX + gp + 1, cfg.window_pages, 1)
                ws, bt, pv = _device_ws(st, s)
                assert ws == pages, (s, t, "ws at page open")
                assert bt == ref.gather(tab, pages)
                assert pv == [prov[p] for p in pages]
            if r == B - 1:
                step = steps[gp]
                sealed = P_CTX + gp + 1
                assert bool(st.fire[s].item()) == (gp in fired) == step.trigger_fired, (s, gp, "fire")
                if policy == "never":
                    exp_sem[s] = list(range(sealed))
                elif gp in fired:
                    exp_sem[s] = step.semantic if exact else _oracle_with_mirrors(st, s, cfg, sealed)
                if exact:
                    assert exp_sem[s] == step.semantic
                n_sem = int(st.n_semantic[s])
                assert st.semantic[s, :n_sem].cpu().tolist() == exp_sem[s], (s, gp, "semantic")
                pages, prov = ref.working_set(exp_sem[s], sealed, cfg.window_pages, 1)
                if exact:
                    assert pages == step.working_set
                ws, bt, pv = _device_ws(st, s)
                assert ws == pages, (s, gp, "working set")
                assert bt == ref.gather(tab, pages)
                assert pv == [prov[p] for p in pages]
    # the triggers actually exercise the cadence
    if policy == "dynamic":
        assert 0 < sum(len(w[1]) for w in want) < BATCH * G_PAGES
    # and the last token's attention over the final working sets (bf16 bound)
    kp = st.k_pool.double().cpu().numpy()
    vp = st.v_pool.double().cpu().numpy()
    bt = st.block_table.cpu().numpy()
    wl = st.ws_len.cpu().numpy()
    fills = st.tail_fill.cpu().numpy()
    q_last = (sq if mode == "graph" else q_all[T - 1])
    for layer in range(L):
        ql = q_last[:, layer].double().cpu().numpy()
        o_ref, _ = attn_ref.sparse_decode(ql, kp[layer], vp[layer], bt, wl, fills, 1.0 / math.sqrt(HD))
        tol = attn_ref.bf16_bound(ql, kp[layer], vp[layer], bt, wl, fills, 1.0 / math.sqrt(HD), o_ref)
        assert np.all(np.abs(out[:, layer].double().cpu().numpy() - o_ref) <= tol)


def _rows_to_flat(rows_bf16):
    return rows_bf16.reshape(rows_bf16.shape[0], D)


@pytest.mark.parametrize("policy", ["always", "dynamic"])
def test_engine_decode_tensor_core_scan_matches_oracle(policy):
    """The same product-path check at a key width whose summary rows go
    through the tensor-core scan (4 layers x 8 kv heads x head_dim 128: D =
    4096, f64 rows of 32 KB > the 16 KB short-row path): the overlapped
    engine step with fp16 tcgen05 scoring and exact f64 rescoring selects,
    triggers and builds working sets exactly as the f64 oracle decode loop."""
    global L, H, HQ, HD, D
    saved = (L, H, HQ, HD, D)
    L, H, HQ, HD = 4, 8, 8, 128
    D = L * H * HD
    try:
        test_engine_decode_matches_oracle_loop(policy, "concurrent", "f16tc")
        # the tensor-core tail ran: it records each slot's page-level candidate count
        import ctypes as C
        lib = _lib.load()
        lib.chess_debug_tc_read.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32] + [C.c_void_p] * 5
        meta = np.zeros(4, np.int32)
        st = _LAST_STATE[0]
        for s in range(BATCH):
            _lib.check(lib.chess_debug_tc_read(st.ref, s, 0, 0, None, None, None, meta.ctypes.data, None), "tc_read")
            assert meta[2] > 0, (s, meta)
    finally:
        L, H, HQ, HD, D = saved
        _LAST_STATE[0] = None
