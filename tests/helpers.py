"""Shared builders for the GPU parity tests (device state <-> oracle)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import pagesel_ref as ref
from paper_2602_20732_b200 import _lib
from paper_2602_20732_b200.state import DecodeState, Shape


def index_state(batch, dim, max_pages, cfg, summary_dtype="f32", max_ws=None, layers=1, kv_heads=1, q_heads=1, n_phys=1):
    head_dim = dim // (layers * kv_heads)
    shape = Shape(
        batch=batch, layers=layers, kv_heads=kv_heads, q_heads=q_heads, head_dim=head_dim,
        page_size=cfg.page_size, pages_per_chunk=cfg.pages_per_chunk,
        chunks_per_grid=cfg.chunks_per_grid, max_pages=max_pages,
        window_pages=cfg.window_pages, max_ws=max_ws or max_pages, n_phys=n_phys,
        summary_dtype=summary_dtype,
    )
    return DecodeState(shape)


def load_vectors(st: DecodeState, slot: int, rows: np.ndarray):
    """K1c from_page_vectors for one slot (host f64 rows)."""
    dev = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.float64), device=st.device)
    _lib.call("chess_summary_from_vectors", st.ref, slot, _lib.ptr(dev), rows.shape[0],
              dev.stride(0) if rows.shape[0] else st.shape.dim, _lib.stream_ptr())
    torch.cuda.synchronize()


def set_tables(st: DecodeState, slot: int, n_pages: int, sinks: int, table=None):
    if table is None:
        table = np.arange(n_pages, dtype=np.int32) * 7 + 3  # distinct physical ids
    st.page_table[slot, :n_pages] = torch.as_tensor(np.asarray(table, dtype=np.int32), device=st.device)
    st.num_pages[slot] = n_pages
    st.sink_count[slot] = sinks
    st.tail_fill[slot] = st.shape.page_size
    return np.asarray(table)


def read_selection(st: DecodeState, slot: int):
    n_sem = int(st.n_semantic[slot])
    sem = st.semantic[slot, :n_sem].cpu().numpy()
    n_ws = int(st.ws_len[slot])
    ws = st.ws_logical[slot, :n_ws].cpu().numpy()
    bt = st.block_table[slot, :n_ws].cpu().numpy()
    prov = st.ws_prov[slot, :n_ws].cpu().numpy()
    return sem, ws, bt, prov
