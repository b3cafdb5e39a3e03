"""Parity of K1 (append + seal, bulk build), K4 (sparse decode) and K5
(entropy + trigger) against the oracle."""

import ctypes

import os

import numpy as np
import pytest
import torch

from oracle import attention as attn_ref
from oracle import pagesel_ref as ref
from paper_2602_20732_b200 import _lib
from paper_2602_20732_b200.state import DecodeState, Shape

pytestmark = pytest.mark.gpu


def _shape(**kw):
    base = dict(batch=2, layers=2, kv_heads=2, q_heads=4, head_dim=64, page_size=16,
                pages_per_chunk=2, chunks_per_grid=2, max_pages=24, window_pages=2,
                max_ws=24, n_phys=64, summary_dtype="f32")
    base.update(kw)
    base["max_ws"] = max(base["max_ws"], base["max_pages"])
    return Shape(**base)


def _flat_to_pool_rows(k_flat, shape):
    """[D] flattened (layer, head, d) -> [L, H, d]."""
    return k_flat.reshape(shape.layers, shape.kv_heads, shape.head_dim)


@pytest.mark.parametrize("ptab_seed", [0, 1])
def test_append_seal_incremental_bitwise(ptab_seed):
    sh = _shape()
    st = DecodeState(sh)
    st.reset()
    rng = np.random.default_rng(ptab_seed)
    perm = rng.permutation(sh.n_phys).astype(np.int32)
    for s in range(sh.batch):
        st.page_table[s, : sh.max_pages] = torch.as_tensor(perm[s * 24 : s * 24 + 24])
        st.sink_count[s] = 1
    T = 5 * sh.page_size + 5
    keys = torch.randn(T, sh.batch, sh.dim, device="cuda").to(torch.bfloat16)
    vals = torch.randn(T, sh.batch, sh.dim, device="cuda").to(torch.bfloat16)
    for t in range(T):
        _lib.call("chess_append_kv", st.ref, _lib.ptr(keys[t]), _lib.ptr(vals[t]), sh.dim, None, _lib.stream_ptr())
        _lib.call("chess_summary_seal", st.ref, _lib.stream_ptr())
    torch.cuda.synchronize()
    B = sh.page_size
    k64 = keys.double().cpu().numpy()
    v64 = vals.double().cpu().numpy()
    for s in range(sh.batch):
        assert int(st.token_count[s]) == T
        assert int(st.num_pages[s]) == 6 and int(st.tail_fill[s]) == 5
        assert int(st.num_sealed[s]) == 5
        h = ref.Hierarchy(sh.dim, sh.pages_per_chunk, sh.chunks_per_grid)
        for p in range(5):
            h.fold_page(k64[p * B : (p + 1) * B, s], p)
        P, C, G = 5, 3, 2
        np.testing.assert_array_equal(st.page_vec64[s, :P, : sh.dim].cpu().numpy(), h.page_vectors)
        np.testing.assert_array_equal(st.chunk_sum64[s, :C, : sh.dim].cpu().numpy(), np.asarray(h.c_sum))
        np.testing.assert_array_equal(st.grid_sum64[s, :G, : sh.dim].cpu().numpy(), np.asarray(h.g_sum))
        np.testing.assert_array_equal(st.chunk_vec64[s, :C, : sh.dim].cpu().numpy(), h.chunk_vectors)
        np.testing.assert_array_equal(st.grid_vec64[s, :G, : sh.dim].cpu().numpy(), h.grid_vectors)
        np.testing.assert_array_equal(
            st.page_vec32[s, :P, : sh.dim].cpu().numpy(), h.page_vectors.astype(np.float32)
        )
        a, _ = ref.anchor(h.page_vectors, sh.window_pages)
        np.testing.assert_array_equal(st.anchor[s, : sh.dim].cpu().numpy(), a)
        # running sum of the open tail = sum of its 5 rows
        tail = k64[5 * B : 5 * B + 5, s]
        acc = tail[0].copy()
        for r in tail[1:]:
            acc = acc + r
        np.testing.assert_array_equal(st.key_sum[s, : sh.dim].cpu().numpy(), acc)
        # pool payload (zero-copy: rows land in the physical page of the table)
        table = st.page_table[s, :6].cpu().numpy()
        kp = st.k_pool.double().cpu().numpy()
        for t in range(T):
            p, r = divmod(t, B)
            rows = _flat_to_pool_rows(k64[t, s], sh)
            np.testing.assert_array_equal(kp[:, table[p], :, r, :], rows)
        # working set after the last page open: window (2) + sink (1), no semantic
        n = int(st.ws_len[s])
        pages, _ = ref.working_set([], 6, sh.window_pages, 1)
        np.testing.assert_array_equal(st.ws_logical[s, :n].cpu().numpy(), pages)


def test_bulk_build_matches_incremental():
    sh = _shape(batch=2, max_pages=40, n_phys=100)
    st = DecodeState(sh)
    st.reset()
    rng = np.random.default_rng(4)
    st.k_pool.copy_(torch.randn(st.k_pool.shape, device="cuda").to(torch.bfloat16))
    n_pages = [37, 12]
    for s in range(2):
        tab = rng.permutation(sh.n_phys)[: sh.max_pages].astype(np.int32)
        st.page_table[s] = torch.as_tensor(tab)
        st.num_pages[s] = n_pages[s]
        st.tail_fill[s] = sh.page_size
    n_dev = torch.tensor(n_pages, dtype=torch.int32, device="cuda")
    _lib.call("chess_summary_build", st.ref, _lib.ptr(n_dev), _lib.stream_ptr())
    torch.cuda.synchronize()
    kp = st.k_pool.double().cpu().numpy()  # [L, n_phys, H, B, d]
    for s in range(2):
        tab = st.page_table[s].cpu().numpy()
        h = ref.Hierarchy(sh.dim, sh.pages_per_chunk, sh.chunks_per_grid)
        for p in range(n_pages[s]):
            page = kp[:, tab[p]]  # [L, H, B, d]
            rows = np.transpose(page, (2, 0, 1, 3)).reshape(sh.page_size, sh.dim)
            h.fold_page(rows, p)
        G, C, P = h.counts
        np.testing.assert_array_equal(st.page_vec64[s, :P, : sh.dim].cpu().numpy(), h.page_vectors)
        np.testing.assert_array_equal(st.chunk_vec64[s, :C, : sh.dim].cpu().numpy(), h.chunk_vectors)
        np.testing.assert_array_equal(st.grid_vec64[s, :G, : sh.dim].cpu().numpy(), h.grid_vectors)
        np.testing.assert_array_equal(st.grid_sum64[s, :G, : sh.dim].cpu().numpy(), np.asarray(h.g_sum))
        a, _ = ref.anchor(h.page_vectors, sh.window_pages)
        np.testing.assert_array_equal(st.anchor[s, : sh.dim].cpu().numpy(), a)
        assert int(st.num_sealed[s]) == P


ATTN_CASES = [
    # (head_dim, q_heads, kv_heads, page, batch, ws_lens, fills)
    (128, 32, 8, 32, 3, [1, 5, 17], [1, 32, 13]),
    (128, 64, 8, 32, 2, [9, 3], [7, 32]),
    (64, 8, 8, 16, 2, [9, 4], [16, 3]),
    (128, 32, 8, 32, 16, [47] * 16, [32, 1, 5, 31] * 4),
    # batch x kv_heads > SMs: stream-K split segments, two CTAs per SM
    (128, 32, 8, 32, 24, [1, 2, 3, 5, 8, 13, 21, 34] * 3, [32, 1, 17, 9] * 6),
    # tensor-core K4 shapes: pages of 16 (8-page groups), GQA 1 and 2, a
    # piece-mode split (b x kv_heads < SMs without cluster mode under CHESS_ATTN_TC=2)
    (128, 32, 8, 16, 4, [1, 9, 30, 64], [16, 3, 9, 1]),
    (128, 8, 8, 32, 18, [3, 4, 7, 12, 40, 2] * 3, [5, 32, 16, 17, 2, 31] * 3),
    (128, 16, 8, 32, 6, [11, 1, 23, 4, 64, 6], [13, 7, 32, 30, 15, 1]),
]


@pytest.mark.parametrize("case", ATTN_CASES)
def test_sparse_decode_vs_fp64(case):
    hd, hq, hkv, B, b, ws_lens, fills = case
    L = 2
    n_phys = 4 * max(ws_lens) * b + 8
    sh = Shape(batch=b, layers=L, kv_heads=hkv, q_heads=hq, head_dim=hd, page_size=B,
               pages_per_chunk=8, chunks_per_grid=8, max_pages=64, window_pages=4,
               max_ws=64, n_phys=n_phys)
    st = DecodeState(sh)
    g = torch.Generator(device="cuda").manual_seed(7)
    st.k_pool.copy_(torch.randn(st.k_pool.shape, device="cuda", generator=g).to(torch.bfloat16))
    st.v_pool.copy_(torch.randn(st.v_pool.shape, device="cuda", generator=g).to(torch.bfloat16))
    rng = np.random.default_rng(1)
    for s in range(b):
        bt = rng.choice(n_phys, size=ws_lens[s], replace=False).astype(np.int32)
        st.block_table[s, : ws_lens[s]] = torch.as_tensor(bt)
        st.ws_len[s] = ws_lens[s]
        st.tail_fill[s] = fills[s]
    q = torch.randn(b, L, hq, hd, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.zeros(b, L, hq, hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(L, b, hq, device="cuda", dtype=torch.float32)
    scale = 1.0 / np.sqrt(hd)
    for l in range(L):
        _lib.call("chess_sparse_decode", st.ref, l, _lib.ptr(q[:, l]), q.stride(0),
                  _lib.ptr(out[:, l]), out.stride(0), _lib.ptr(lse[l]), scale, _lib.stream_ptr())
    torch.cuda.synchronize()
    kp = st.k_pool.double().cpu().numpy()
    vp = st.v_pool.double().cpu().numpy()
    bt = st.block_table.cpu().numpy()
    for l in range(L):
        o_ref, lse_ref = attn_ref.sparse_decode(
            q[:, l].double().cpu().numpy(), kp[l], vp[l], bt, ws_lens, fills, scale
        )
        o = out[:, l].double().cpu().numpy()
        # bf16 P / bf16 output: |err| <= 2^-8 (sum p|v| + |ref|)  (oracle/attention.bf16_bound)
        tol = attn_ref.bf16_bound(q[:, l].double().cpu().numpy(), kp[l], vp[l], bt, ws_lens, fills, scale, o_ref)
        assert np.all(np.abs(o - o_ref) <= tol), np.max(np.abs(o - o_ref) / tol)
        np.testing.assert_allclose(lse[l].double().cpu().numpy(), lse_ref, rtol=0, atol=2e-4)


@pytest.mark.skipif(os.environ.get("CHESS_ATTN_TC") is not None, reason="already an alternate path")
@pytest.mark.parametrize("tc", ["1", "2"], ids=["tcgen05_piece_streamk", "tcgen05_everywhere"])
def test_attention_paths_in_subprocess(tc):
    """K4 has two consumers: mma.sync (default) and tcgen05 (k_attn_tc.cuh,
    head_dim 128, opt-in: CHESS_ATTN_TC=1 where cluster mode is not chosen, 2
    everywhere).  Re-run the attention parity cases with the tensor-core one."""
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_kernels.py"), "-k", "sparse_decode_vs_fp64"],
                       env=dict(os.environ, CHESS_ATTN_TC=tc), capture_output=True, text=True,
                       cwd=os.path.dirname(here), timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_entropy_logits_and_trigger_bitwise_stats():
    B = 16
    sh = _shape(batch=4, page_size=B)
    st = DecodeState(sh)
    st.reset()
    V = 32000
    cfg = _lib.ChessTriggerCfg()
    cfg.policy = _lib.POLICY_DYNAMIC
    cfg.mode = 0
    cfg.tau_entropy = 2.0
    cfg.tau_varentropy = 0.5
    g = torch.Generator(device="cuda").manual_seed(3)
    Hs = []
    for t in range(B):
        scale = torch.tensor([0.1, 1.0, 5.0, 30.0], device="cuda").unsqueeze(1)
        logits = (torch.randn(4, V, device="cuda", generator=g) * scale).float()
        if t % 3 == 0:
            logits[0] = -1e30
            logits[0, 5] = 0.0  # one-hot: H = 0
        st.sealed.fill_(1 if t == B - 1 else 0)
        Hout = torch.zeros(4, dtype=torch.float64, device="cuda")
        _lib.call("chess_entropy_trigger", st.ref, _lib.ptr(logits), V, logits.stride(0),
                  ctypes.byref(cfg), _lib.ptr(Hout), _lib.stream_ptr())
        torch.cuda.synchronize()
        for s in range(4):
            assert abs(Hout[s].item() - ref.entropy_from_logits(logits[s].double().cpu().numpy())) <= 1e-5
        Hs.append(Hout.cpu().numpy())
    ring = st.ent_ring.cpu().numpy()
    stats = st.page_stats.cpu().numpy()
    fire = st.fire.cpu().numpy()
    for s in range(4):
        np.testing.assert_array_equal(ring[s], np.array([h[s] for h in Hs]))
        mean, var, _ = ref.page_stats(ring[s])
        assert stats[s, 0] == mean and stats[s, 1] == var  # bit-exact (NumPy order)
        assert bool(fire[s]) == ref.check_trigger(mean, var, 2.0, 0.5)
    assert st.gen_pages.cpu().tolist() == [1, 1, 1, 1]


@pytest.mark.parametrize("vocab", [1, 7, 4099, 128256, 600000])
def test_entropy_logits_vocab_sizes_and_masks(vocab):
    """Entropy from logits at the Llama-3 vocabulary (and ragged / tiny /
    over-sized vocabularies) with -inf-masked entries: |dH| <= 1e-4 nats
    (SURVEY §8c), split count chosen by the kernel."""
    rows = 5
    g = torch.Generator(device="cuda").manual_seed(vocab)
    logits = torch.randn(rows, vocab, device="cuda", generator=g) * torch.tensor(
        [0.01, 1.0, 4.0, 20.0, 1.0], device="cuda").unsqueeze(1)
    if vocab > 3:
        logits[4, ::3] = -float("inf")  # masked vocabulary entries
        logits[3, : vocab // 2] = -1e30
    H = torch.zeros(rows, dtype=torch.float64, device="cuda")
    nbytes = _lib.load().chess_entropy_workspace_bytes(rows)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    _lib.call("chess_entropy_logits", _lib.ptr(logits), rows, vocab, logits.stride(0), _lib.ptr(H),
              _lib.ptr(ws), _lib.stream_ptr())
    torch.cuda.synchronize()
    for r in range(rows):
        want = ref.entropy_from_logits(logits[r].double().cpu().numpy())
        assert abs(H[r].item() - want) <= 1e-4, (r, H[r].item(), want)
