"""Device-resident batched decode state (the buffers behind a ChessState).

Every buffer is a torch CUDA tensor owned here; the C-ABI struct only holds
their addresses (include/chess_b200.h: "the caller owns all device buffers").
Layouts are documented in the header and DESIGN.md §"Data layout in HBM".
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import torch

from . import _lib


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


@dataclass(frozen=True)
class Shape:
    batch: int
    layers: int
    kv_heads: int
    q_heads: int
    head_dim: int
    page_size: int
    pages_per_chunk: int
    chunks_per_grid: int
    max_pages: int
    window_pages: int
    max_ws: int
    n_phys: int
    summary_dtype: str = "f32"  # "f32"/"bf16" mirrors scanned, "f64", or "f16tc"
    # ("f16tc": fp16 mirrors scored on tcgen05 with certified bounds, rows near
    # each level's cut rescored from f64 -> the f64 selection, k_select_tc.cuh)

    @property
    def dim(self) -> int:
        return self.layers * self.kv_heads * self.head_dim

    @property
    def ld(self) -> int:
        # bf16 mirror rows must be 16-byte multiples for the scan's bulk copies;
        # the tensor-core scan reads 64-element K blocks
        if self.summary_dtype == "f16tc":
            return _round_up(self.dim, 64)
        return _round_up(self.dim, 8 if self.summary_dtype == "bf16" else 4)

    @property
    def max_chunks(self) -> int:
        return math.ceil(self.max_pages / self.pages_per_chunk)

    @property
    def max_grids(self) -> int:
        return math.ceil(self.max_chunks / self.chunks_per_grid)


SUMMARY_DTYPES = {"f32": 0, "f64": 1, "bf16": 2, "f16tc": 3}


class DecodeState:
    """Allocates and owns every buffer of a ChessState for `shape`."""

    def __init__(self, shape: Shape, device="cuda", kv_pool=None, page_pool=False):
        self.shape = s = shape
        self.device = torch.device(device)
        dev = self.device
        b, ld = s.batch, s.ld
        i32 = dict(dtype=torch.int32, device=dev)
        f64 = dict(dtype=torch.float64, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        u8 = dict(dtype=torch.uint8, device=dev)
        if kv_pool is None:
            kv_shape = (s.layers, s.n_phys, s.kv_heads, s.page_size, s.head_dim)
            self.k_pool = torch.empty(kv_shape, dtype=torch.bfloat16, device=dev)
            self.v_pool = torch.empty(kv_shape, dtype=torch.bfloat16, device=dev)
        else:
            self.k_pool, self.v_pool = kv_pool
        self.page_table = torch.zeros((b, s.max_pages), **i32)
        self.num_pages = torch.zeros(b, **i32)
        self.tail_fill = torch.zeros(b, **i32)
        self.token_count = torch.zeros(b, dtype=torch.int64, device=dev)
        self.sink_count = torch.zeros(b, **i32)
        self.sealed = torch.zeros(b, **u8)
        self.num_sealed = torch.zeros(b, **i32)
        self.page_vec64 = torch.zeros((b, s.max_pages, ld), **f64)
        self.chunk_sum64 = torch.zeros((b, s.max_chunks, ld), **f64)
        self.grid_sum64 = torch.zeros((b, s.max_grids, ld), **f64)
        self.chunk_vec64 = torch.zeros((b, s.max_chunks, ld), **f64)
        self.grid_vec64 = torch.zeros((b, s.max_grids, ld), **f64)
        if s.summary_dtype in ("f32", "bf16", "f16tc"):
            # f16tc: fp16 rows + {err, nrm} stash inside the f32 row pitch
            mdt = dict(f32) if s.summary_dtype != "bf16" else dict(dtype=torch.bfloat16, device=dev)
            self.page_vec32 = torch.zeros((b, s.max_pages, ld), **mdt)
            self.chunk_vec32 = torch.zeros((b, s.max_chunks, ld), **mdt)
            self.grid_vec32 = torch.zeros((b, s.max_grids, ld), **mdt)
        else:
            self.page_vec32 = self.chunk_vec32 = self.grid_vec32 = None
        self.key_sum = torch.zeros((b, ld), **f64)
        self.anchor = torch.zeros((b, ld), **f64)
        self.semantic = torch.zeros((b, s.max_pages), **i32)
        self.n_semantic = torch.zeros(b, **i32)
        self.sel_stats = torch.zeros((b, 8), **i32)
        self.ws_logical = torch.zeros((b, s.max_ws), **i32)
        self.block_table = torch.zeros((b, s.max_ws), **i32)
        self.ws_prov = torch.zeros((b, s.max_ws), dtype=torch.int8, device=dev)
        self.ws_len = torch.zeros(b, **i32)
        self.ent_ring = torch.zeros((b, s.page_size), **f64)
        self.ent_count = torch.zeros(b, **i32)
        self.gen_pages = torch.zeros(b, **i32)
        self.page_stats = torch.zeros((b, 2), **f64)
        self.fire = torch.zeros(b, **u8)
        self.trigger_count = torch.zeros(b, **i32)
        # optional device page pool (kv_store.py:103-136 free list on the device)
        if page_pool:
            self.pool_free = torch.zeros(s.n_phys, **i32)
            self.pool_top = torch.zeros(1, **i32)
            self.pool_base = torch.zeros(b, **i32)
            self.pool_end = torch.zeros(b, **i32)
            self.pool_oom = torch.zeros(b, **u8)
        else:
            self.pool_free = self.pool_top = self.pool_base = self.pool_end = self.pool_oom = None

        self.c = _lib.ChessState()
        d = self.c.d
        d.batch, d.layers, d.kv_heads, d.q_heads = b, s.layers, s.kv_heads, s.q_heads
        d.head_dim, d.page_size = s.head_dim, s.page_size
        d.pages_per_chunk, d.chunks_per_grid = s.pages_per_chunk, s.chunks_per_grid
        d.max_pages, d.window_pages, d.max_ws = s.max_pages, s.window_pages, s.max_ws
        d.summary_dtype = SUMMARY_DTYPES[s.summary_dtype]
        d.dim, d.ld, d.n_phys = s.dim, ld, s.n_phys
        lib = _lib.load()
        _lib.check(lib.chess_validate_dims(C.byref(d)), "validate_dims")
        nbytes = lib.chess_workspace_bytes(C.byref(d))
        self.workspace = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        for name in _lib.STATE_POINTERS:
            setattr(self.c, name, _lib.ptr(getattr(self, name)))
        self.c.workspace_bytes = nbytes
        self.ref = C.byref(self.c)

    # ------------------------------------------------------------------
    def reset(self, mask=None, stream=None):
        _lib.call("chess_reset_slots", self.ref, _lib.ptr(mask), _lib.stream_ptr(stream))

    # ------------------------------------------------------------------
    # device page pool
    # ------------------------------------------------------------------
    def pool_init(self, ids=None, stream=None):
        """Free list := ids (default: every physical page), kv_store.py:117-120."""
        if ids is None:
            ids = torch.arange(self.shape.n_phys, dtype=torch.int32, device=self.device)
        ids = torch.as_tensor(ids, dtype=torch.int32, device=self.device).contiguous()
        self._pool_ids = ids  # kept alive until the (async) copy ran
        _lib.call("chess_pool_init", self.ref, _lib.ptr(ids), int(ids.numel()), _lib.stream_ptr(stream))

    def pool_reserve(self, counts, stream=None):
        """Slot s takes counts[s] pages into its page table (admission)."""
        c = torch.as_tensor(counts, dtype=torch.int32, device=self.device).reshape(-1)
        if c.numel() == 1 and self.shape.batch > 1:
            c = c.expand(self.shape.batch)
        c = c.contiguous()
        self._pool_counts = c
        _lib.call("chess_pool_reserve", self.ref, _lib.ptr(c), _lib.stream_ptr(stream))

    def pool_release(self, mask=None, stream=None):
        _lib.call("chess_pool_release", self.ref, _lib.ptr(mask), _lib.stream_ptr(stream))

    def pool_free_count(self) -> int:
        return int(self.pool_top.item())

    def check_pool(self):
        """Raise OutOfPagesError (kv_store.py:129-132) if an allocation failed."""
        from .errors import OutOfPagesError

        if self.pool_oom is not None and bool(self.pool_oom.any()):
            slots = torch.nonzero(self.pool_oom).flatten().tolist()
            raise OutOfPagesError(f"device page pool exhausted ({self.shape.n_phys} pages); slots {slots}")

    def scan_matrices(self):
        """(grid, chunk, page) matrices the selection scan reads."""
        if self.shape.summary_dtype in ("f32", "bf16"):
            return self.grid_vec32, self.chunk_vec32, self.page_vec32
        return self.grid_vec64, self.chunk_vec64, self.page_vec64

    def mirror16(self, which: int):
        """f16tc: (fp16 rows [b, rows, ld], stash f64 [b, rows, 2] = {err, nrm})
        of the grid (0), chunk (1) or page (2) matrix (mirror16_kernel)."""
        m = (self.grid_vec32, self.chunk_vec32, self.page_vec32)[which]
        ld = self.shape.ld
        return m.view(torch.float16)[..., :ld], m.view(torch.float64)[..., ld // 4: ld // 4 + 2]

    def bytes_allocated(self) -> int:
        tot = 0
        for v in self.__dict__.values():
            if isinstance(v, torch.Tensor):
                tot += v.numel() * v.element_size()
        return tot
