"""Per-group timeline of the tensor-core K4 (CHESS_TRACE build):
  CHESS_B200_LIB=paper_2602_20732_b200/libchess_b200_trace.so python tools/tc_attn_timeline.py [hot|random]
Events per group (clock64, us from CTA start of group 0's K issue):
  Kiss K issued, K K landed, S S read by softmax, P P published, Viss V issued, V V landed, PV PV issued, O O folded"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_20732_b200 import _lib  # noqa: E402
from paper_2602_20732_b200.state import DecodeState, Shape  # noqa: E402

pattern = sys.argv[1] if len(sys.argv) > 1 else "hot"
b, L, H, Hq, d, B, ws = 16, 2, 8, 32, 128, 32, 46
page_bytes = L * H * B * d * 2 * 2
n_phys = int(20 * (1 << 30) // page_bytes)
sh = Shape(batch=b, layers=L, kv_heads=H, q_heads=Hq, head_dim=d, page_size=B, pages_per_chunk=8,
           chunks_per_grid=8, max_pages=ws + 8, window_pages=4, max_ws=ws + 8, n_phys=n_phys)
st = DecodeState(sh)
st.k_pool.normal_()
st.v_pool.normal_()
q = torch.randn(b, L, Hq, d, device="cuda").to(torch.bfloat16)
out = torch.zeros_like(q)
rng = np.random.default_rng(0)
bt = rng.integers(0, 64, size=(b, ws)) if pattern == "hot" else rng.choice(n_phys, size=(b, ws), replace=False)
st.block_table[:, :ws] = torch.as_tensor(bt.astype(np.int32), device="cuda")
st.ws_len.fill_(ws)
st.tail_fill.fill_(B)
for _ in range(5):
    for layer in range(L):
        _lib.call("chess_sparse_decode", st.ref, layer, _lib.ptr(q[:, layer]), q.stride(0),
                  _lib.ptr(out[:, layer]), out.stride(0), None, 0.088, _lib.stream_ptr())
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8 * 16 * 8))()
assert _lib.load().chess_debug_attn_tc_trace(buf) == 0
tr = np.frombuffer(buf, dtype=np.uint64).reshape(8, 16, 8).astype(np.int64)
names = ["K", "S", "P", "V", "PV", "O", "Kiss", "Viss"]
order = [6, 0, 1, 2, 7, 3, 4, 5]
ghz = 1.965
for c in range(3):
    t0 = tr[c, 0, 6]
    print(f"CTA {c} (us since group 0 K issue)")
    print("  g  " + " ".join(f"{names[e]:>6}" for e in order))
    for j in range(12):
        print(f"  {j:2d} " + " ".join(f"{(tr[c, j, e] - t0) / ghz / 1e3:6.2f}" for e in order))
