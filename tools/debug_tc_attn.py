"""Debug: one tensor-core K4 parity case, per (slot, q head) error ratio vs the fp64 restatement."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
from oracle import attention as attn_ref
from paper_2602_20732_b200 import _lib
from paper_2602_20732_b200.state import DecodeState, Shape

if "--pre" in sys.argv:
    import test_gpu_kernels as tk
    for case in tk.ATTN_CASES[:3]:
        tk.test_sparse_decode_vs_fp64(case)
    print("pre cases ok")
hd, hq, hkv, B, b = 128, 32, 8, 32, 16
ws_lens, fills = [47] * 16, [32, 1, 5, 31] * 4
if len(sys.argv) > 1 and sys.argv[1] == "uniform":
    fills = [32] * 16
L = 2
n_phys = 4 * max(ws_lens) * b + 8
sh = Shape(batch=b, layers=L, kv_heads=hkv, q_heads=hq, head_dim=hd, page_size=B, pages_per_chunk=8,
           chunks_per_grid=8, max_pages=64, window_pages=4, max_ws=64, n_phys=n_phys)
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
scale = 1.0 / np.sqrt(hd)
kp = st.k_pool.double().cpu().numpy()
vp = st.v_pool.double().cpu().numpy()
btn = st.block_table.cpu().numpy()
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    out = torch.zeros(b, L, hq, hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(L, b, hq, device="cuda", dtype=torch.float32)
    for l in range(L):
        _lib.call("chess_sparse_decode", st.ref, l, _lib.ptr(q[:, l]), q.stride(0),
                  _lib.ptr(out[:, l]), out.stride(0), _lib.ptr(lse[l]), scale, _lib.stream_ptr())
    torch.cuda.synchronize()
    for l in range(L):
        ql = q[:, l].double().cpu().numpy()
        o_ref, lse_ref = attn_ref.sparse_decode(ql, kp[l], vp[l], btn, ws_lens, fills, scale)
        tol = attn_ref.bf16_bound(ql, kp[l], vp[l], btn, ws_lens, fills, scale, o_ref)
        o = out[:, l].double().cpu().numpy()
        r = np.abs(o - o_ref) / tol  # [b, hq, hd]
        bad = np.argwhere(r.max(axis=2) > 1)
        print(f"rep {rep} layer {l}: max ratio {r.max():.2f}, bad (slot, qhead) {len(bad)}: {bad[:40].tolist()}")
        if len(bad):
            # does the error look like one page's contribution missing / doubled?
            s_, h_ = bad[0]
            kvh = h_ // (hq // hkv)
            print("   fills of bad slots:", sorted(set(int(fills[x]) for x in bad[:, 0])), "per-slot max ratio:",
                  np.round(r.max(axis=(1, 2)), 2).tolist())
        if len(bad):
            s_, h_ = bad[0]
            print("   d ratios of first bad:", np.round(r[s_, h_, :16], 2).tolist(), "lse err", float(np.abs(lse[l].cpu().numpy() - lse_ref)[s_, h_]))
        print("   lse max err", float(np.abs(lse[l].double().cpu().numpy() - lse_ref).max()))
