"""Re-run one attention parity case and report where the device output
differs most from the fp64 restatement (debug aid for K4 work splits)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import attention as attn_ref  # noqa: E402
from paper_2602_20732_b200 import _lib  # noqa: E402
from paper_2602_20732_b200.state import DecodeState, Shape  # noqa: E402


def main():
    hd, hq, hkv, B, b = 128, 32, 8, 32, 24
    ws_lens = [1, 2, 3, 5, 8, 13, 21, 34] * 3
    fills = [32, 1, 17, 9] * 6
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
    out = torch.zeros(b, L, hq, hd, device="cuda", dtype=torch.bfloat16)
    scale = 1.0 / np.sqrt(hd)
    for l in range(L):
        _lib.call("chess_sparse_decode", st.ref, l, _lib.ptr(q[:, l]), q.stride(0), _lib.ptr(out[:, l]),
                  out.stride(0), None, scale, _lib.stream_ptr())
    torch.cuda.synchronize()
    kp, vp = st.k_pool.double().cpu().numpy(), st.v_pool.double().cpu().numpy()
    bt = st.block_table.cpu().numpy()
    for l in range(L):
        o_ref, _ = attn_ref.sparse_decode(q[:, l].double().cpu().numpy(), kp[l], vp[l], bt, ws_lens, fills, scale)
        o = out[:, l].double().cpu().numpy()
        err = np.abs(o - o_ref) / (np.abs(o_ref) + 0.125)
        bad = np.argwhere(err > 2.0 ** -7)
        print(f"layer {l} CPS={os.environ.get('CHESS_ATTN_CPS', 'auto')}: max rel {err.max():.4g}, bad {len(bad)}")
        slots = sorted(set(int(x[0]) for x in bad))
        for s in slots[:8]:
            heads = sorted(set(int(x[1]) for x in bad if x[0] == s))
            print(f"  slot {s} ws {ws_lens[s]} fill {fills[s]} heads {heads[:8]} max {err[s].max():.3g}")


if __name__ == "__main__":
    main()
