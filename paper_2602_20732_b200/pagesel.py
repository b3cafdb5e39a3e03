"""Drop-in, device-backed mirror of the reference `pagesel` hot-path API.

Same public names, argument meanings and exceptions as
/root/reference/pkg/src/pagesel (__init__.py:43-86) for the decode hot path:
the paged KV store, the hierarchy index, the selector, the uncertainty
trigger and the page-granular decode loop.  Every numeric operation runs in
libchess_b200.so (sm_100a) through the C-ABI; there is no CPU fallback — a
missing library raises NativeLibraryError on first use.

Array conventions: inputs may be NumPy arrays / lists (copied to the device)
or CUDA torch tensors (used in place).  Matrices produced by the store and
the index (page keys, page/chunk/grid vectors, coalesced matrix, anchors,
scores) are CUDA float64 tensors; index outputs (selected pages, working
sets) are host integers like the reference returns, which costs one small
device->host read per call.  The batched, sync-free fast path for serving is
`engine.ChessDecoder` over a `state.DecodeState`.

Scalar-only logic with no array arithmetic — `check_trigger` (strict
comparisons), `calibrate` (nearest-rank percentiles over a host sample) and
the thresholds JSON I/O — stays on the host as in the reference; it is
offline or O(1) work.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import math
import threading
import warnings
from collections import deque
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from . import _lib
from .config import PRESETS, SelectionConfig, preset_config  # noqa: F401
from .errors import (  # noqa: F401
    CalibrationError,
    ConfigurationError,
    EmptyContextError,
    OutOfPagesError,
    PageSelError,
)
from .state import DecodeState, Shape
from .workload import Workload, WorkloadSpec, generate_workload  # noqa: F401

NORMALIZATION_TOL = 1e-9


def _device(device=None) -> torch.device:
    return torch.device(device if device is not None else "cuda")


def _f64(x, device=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(_device(device))
        return t.to(torch.float64).contiguous()
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=_device(device)).contiguous()


def _i64(x, device=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=_device(device) if not x.is_cuda else x.device, dtype=torch.int64).contiguous()
    return torch.as_tensor(np.asarray(x, dtype=np.int64).reshape(-1), device=_device(device))


def _i32(x, device=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=_device(device) if not x.is_cuda else x.device, dtype=torch.int32).contiguous()
    return torch.as_tensor(np.asarray(x, dtype=np.int64).reshape(-1).astype(np.int32), device=_device(device))


def _sp():
    return _lib.stream_ptr()


def _checksum(matrix: torch.Tensor) -> str:
    arr = matrix.detach().cpu().numpy() if isinstance(matrix, torch.Tensor) else np.asarray(matrix)
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:16]


# =============================================================================
# Paged KV store (kv_store.py:20-174)
# =============================================================================
@dataclass
class AppendEvent:
    sealed: bool
    page_id: int
    logical_index: int


class ReadOnlyRows(torch.Tensor):
    """A CUDA view whose writes raise ValueError, like the reference's
    read-only NumPy views of a page's rows (kv_store.py:52-65): item
    assignment and in-place ops raise, views of it stay read-only, and
    computed results are plain tensors.  `copy()` and `__array__` give host
    NumPy arrays, so `np.array_equal(page.keys, first)` works as there."""

    @classmethod
    def __torch_function__(cls, func, types, args=(), kwargs=None):
        name = getattr(func, "__name__", "")
        if name == "__setitem__" or (name.endswith("_") and not name.startswith("_")):
            raise ValueError("assignment destination is read-only")
        with torch._C.DisableTorchFunctionSubclass():
            out = func(*args, **(kwargs or {}))
        src = args[0] if args and isinstance(args[0], torch.Tensor) else None
        if isinstance(out, torch.Tensor) and not isinstance(out, ReadOnlyRows):
            shares = src is not None and out.numel() and src.numel() and \
                out.untyped_storage().data_ptr() == src.untyped_storage().data_ptr()
            if shares:
                out = out.as_subclass(ReadOnlyRows)
        return out

    def copy(self):
        return self.detach().cpu().numpy().copy()

    def __array__(self, dtype=None, copy=None):
        a = self.detach().cpu().numpy()
        return a.astype(dtype) if dtype is not None else a


class KvPage:
    """One physical page of the device pool (kv_store.py:29-74).  `keys` /
    `values` are read-only CUDA float64 views of the filled rows."""

    def __init__(self, store, page_id, slot=None):
        self._store = store
        self.page_id = page_id
        self._slot = page_id if slot is None else slot  # row block of the pool
        self.page_size = store.page_size
        self.fill = 0
        self.version = 0

    @property
    def sealed(self):
        return self.fill == self.page_size

    def write(self, key, value):
        if self.sealed:
            raise ValueError(f"page {self.page_id} is sealed")
        self._store._keys[self._slot, self.fill].copy_(_f64(key, self._store.device))
        self._store._values[self._slot, self.fill].copy_(_f64(value, self._store.device))
        self.fill += 1
        self.version += 1

    @property
    def keys(self) -> torch.Tensor:
        return self._store._keys[self._slot, : self.fill].as_subclass(ReadOnlyRows)

    @property
    def values(self) -> torch.Tensor:
        return self._store._values[self._slot, : self.fill].as_subclass(ReadOnlyRows)

    def dump(self):
        return {
            "page_id": self.page_id,
            "fill": self.fill,
            "keys": self.keys.copy().ravel().tolist(),
            "values": self.values.copy().ravel().tolist(),
        }


@dataclass
class SequenceState:
    page_table: list = field(default_factory=list)
    token_count: int = 0
    sink_count: int = 0


class PagedKvStore:
    """Fixed pool of physical pages in HBM; host free list under a lock
    (kv_store.py:103-136), payloads written straight into device memory."""

    def __init__(self, capacity_pages, dim, page_size=32, device=None):
        if capacity_pages < 1:
            raise ConfigurationError(f"store capacity must be >= 1 page, got {capacity_pages}")
        self.capacity_pages = capacity_pages
        self.dim = dim
        self.page_size = page_size
        self.device = _device(device)
        self._keys = torch.zeros((capacity_pages, page_size, dim), dtype=torch.float64, device=self.device)
        self._values = torch.zeros_like(self._keys)
        self._pages = {}
        self._free = deque(range(capacity_pages))
        self._lock = threading.Lock()

    def create_sequence(self, config=None):
        return SequenceState(sink_count=config.sink_pages if config is not None else 0)

    def _allocate(self):
        with self._lock:
            if not self._free:
                raise OutOfPagesError(f"page pool exhausted ({self.capacity_pages} pages)")
            pid = self._free.popleft()
        page = KvPage(self, pid)
        self._pages[pid] = page
        return page

    def page(self, page_id):
        return self._pages[page_id]

    def append_token(self, seq, key, value):
        if not seq.page_table or self._pages[seq.page_table[-1]].sealed:
            page = self._allocate()
            seq.page_table.append(page.page_id)
        else:
            page = self._pages[seq.page_table[-1]]
        page.write(key, value)
        seq.token_count += 1
        return AppendEvent(sealed=page.sealed, page_id=page.page_id, logical_index=len(seq.page_table) - 1)

    def gather_pages(self, seq, logical_indices):
        """Physical ids of the given logical positions (kv_store.py:156-166),
        looked up on the device by the gather kernel."""
        idx = np.asarray(list(logical_indices), dtype=np.int64)
        if idx.size == 0:
            return []
        table = _i32(seq.page_table if seq.page_table else [0], self.device)
        out = torch.empty(idx.size, dtype=torch.int32, device=self.device)
        err = torch.full((1,), np.iinfo(np.int32).max, dtype=torch.int32, device=self.device)
        _lib.call("chess_gather_pages", _lib.ptr(table), len(seq.page_table), _lib.ptr(_i64(idx, self.device)),
                  int(idx.size), _lib.ptr(out), _lib.ptr(err), _sp())
        bad = int(err.item())
        if bad != np.iinfo(np.int32).max:
            raise IndexError(f"logical index {int(idx[bad - 1])} out of range for "
                             f"{len(seq.page_table)}-page table")
        return [int(x) for x in out.cpu().tolist()]

    def sealed_versions(self, seq):
        return {pid: self._pages[pid].version for pid in seq.page_table if self._pages[pid].sealed}


def page_from_record(record, page_size, dim, device=None):
    """Rebuild a KvPage from a dump() record (kv_store.py:67-74, test-fixture
    path): a standalone page holding the record's rows, keeping its page_id."""
    store = PagedKvStore(1, dim, page_size=page_size, device=device)
    page = KvPage(store, record["page_id"], slot=0)
    store._free.clear()
    store._pages[page.page_id] = page
    keys = np.asarray(record["keys"], dtype=np.float64).reshape(record["fill"], dim)
    values = np.asarray(record["values"], dtype=np.float64).reshape(record["fill"], dim)
    for k, v in zip(keys, values):
        page.write(k, v)
    return page


def dump_pages(pages, path):
    with open(path, "w") as fh:
        for page in pages:
            fh.write(json.dumps(page.dump()) + "\n")


# =============================================================================
# Hierarchy index (hierarchy.py:26-174)
# =============================================================================
@dataclass
class PageVector:
    v: torch.Tensor
    page_logical_index: int


class HierarchyIndex:
    """Page / chunk / grid centroid matrices in HBM, maintained by the K1
    fold kernel in the reference's f64 operation order (bit-identical)."""

    _INITIAL_PAGES = 64

    def __init__(self, dim, pages_per_chunk, chunks_per_grid, device=None):
        if pages_per_chunk < 1 or chunks_per_grid < 1:
            raise ConfigurationError("hierarchy fan-outs must be >= 1")
        self.dim = dim
        self.pages_per_chunk = pages_per_chunk
        self.chunks_per_grid = chunks_per_grid
        self.device = _device(device)
        self._n = 0
        self._st = None
        if dim > 0:
            self._st = self._make_state(self._INITIAL_PAGES)

    def _make_state(self, max_pages):
        shape = Shape(batch=1, layers=1, kv_heads=1, q_heads=1, head_dim=self.dim, page_size=1,
                      pages_per_chunk=self.pages_per_chunk, chunks_per_grid=self.chunks_per_grid,
                      max_pages=max_pages, window_pages=1, max_ws=max_pages, n_phys=1, summary_dtype="f64")
        st = DecodeState(shape, device=self.device)
        st.reset()
        return st

    def _grow(self):
        old = self._st
        new = self._make_state(2 * old.shape.max_pages)
        P, Cn, G = self.num_pages, self.num_chunks, self.num_grids
        new.page_vec64[:, :P].copy_(old.page_vec64[:, :P])
        for name, n in (("chunk_sum64", Cn), ("chunk_vec64", Cn), ("grid_sum64", G), ("grid_vec64", G)):
            getattr(new, name)[:, :n].copy_(getattr(old, name)[:, :n])
        new.num_sealed.copy_(old.num_sealed)
        self._st = new

    @classmethod
    def from_page_vectors(cls, rows, pages_per_chunk, chunks_per_grid, device=None):
        """Direct build from page vectors (hierarchy.py:43-58), device K1c."""
        rows = _f64(rows, device)
        n = rows.shape[0] if rows.dim() == 2 else 0
        dim = rows.shape[1] if rows.dim() == 2 and rows.numel() else 0
        index = cls(dim, pages_per_chunk, chunks_per_grid, device)
        if n == 0 or dim == 0:
            return index
        cap = cls._INITIAL_PAGES
        while cap < n:
            cap *= 2
        if cap != index._st.shape.max_pages:
            index._st = index._make_state(cap)
        _lib.call("chess_summary_from_vectors", index._st.ref, 0, _lib.ptr(rows), n, rows.stride(0), _sp())
        index._n = n
        return index

    @property
    def num_pages(self):
        return self._n

    @property
    def num_chunks(self):
        return math.ceil(self._n / self.pages_per_chunk)

    @property
    def num_grids(self):
        return math.ceil(self.num_chunks / self.chunks_per_grid)

    def _rows(self, mat, n):
        if n == 0 or self._st is None:
            return torch.zeros((0, self.dim), dtype=torch.float64, device=self.device)
        return mat[0, :n, : self.dim]

    @property
    def page_vectors(self) -> torch.Tensor:
        return self._rows(self._st.page_vec64 if self._st else None, self.num_pages)

    @property
    def chunk_vectors(self) -> torch.Tensor:
        return self._rows(self._st.chunk_vec64 if self._st else None, self.num_chunks)

    @property
    def grid_vectors(self) -> torch.Tensor:
        return self._rows(self._st.grid_vec64 if self._st else None, self.num_grids)

    @property
    def page_to_chunk(self):
        return np.arange(self.num_pages) // self.pages_per_chunk

    @property
    def chunk_to_grid(self):
        return np.arange(self.num_chunks) // self.chunks_per_grid

    def finalize_page(self, page, logical_index):
        """Fold a sealed page (Eq.1 mean + chunk/grid update, hierarchy.py:102-136)."""
        if not page.sealed:
            raise ValueError("only sealed pages can be finalized")
        if logical_index != self.num_pages:
            raise ValueError(f"pages finalize in order: expected index {self.num_pages}, got {logical_index}")
        keys = page.keys if isinstance(page.keys, torch.Tensor) else _f64(page.keys, self.device)
        keys = _f64(keys, self.device)
        if self._st is None:
            raise ValueError("a zero-dimensional index cannot hold pages")
        if self._n == self._st.shape.max_pages:
            self._grow()
        _lib.call("chess_summary_fold", self._st.ref, 0, _lib.ptr(keys), _lib.F64, keys.shape[0],
                  keys.stride(0), _sp())
        self._n += 1
        return PageVector(v=self._st.page_vec64[0, logical_index, : self.dim], page_logical_index=logical_index)

    def coalesced_matrix(self):
        g, c, p = self.num_grids, self.num_chunks, self.num_pages
        if p == 0:
            return torch.zeros((0, self.dim), dtype=torch.float64, device=self.device), (0, 0, 0)
        return torch.cat([self.grid_vectors, self.chunk_vectors, self.page_vectors], dim=0), (g, c, p)

    def snapshot(self):
        return {
            "pages_per_chunk": self.pages_per_chunk,
            "chunks_per_grid": self.chunks_per_grid,
            "num_pages": self.num_pages,
            "num_chunks": self.num_chunks,
            "num_grids": self.num_grids,
            "checksum_pages": _checksum(self.page_vectors),
            "checksum_chunks": _checksum(self.chunk_vectors),
            "checksum_grids": _checksum(self.grid_vectors),
        }

    def snapshot_json(self):
        return json.dumps(self.snapshot(), sort_keys=True)


def rebuild_from_scratch(pages, config, device=None):
    dim = pages[0].keys.shape[1] if pages else 0
    index = HierarchyIndex(dim, config.pages_per_chunk, config.chunks_per_grid, device)
    for i, page in enumerate(pages):
        index.finalize_page(page, i)
    return index


# =============================================================================
# Selector (selection.py:19-159)
# =============================================================================
@dataclass
class QueryAnchor:
    v: torch.Tensor
    source_pages: list

    def checksum(self):
        return _checksum(self.v)


@dataclass
class WorkingSet:
    pages: list
    provenance: dict = field(default_factory=dict)

    def __len__(self):
        return len(self.pages)

    def __contains__(self, idx):
        return idx in self.provenance


def _mean_rows(rows: torch.Tensor, n: int, dim: int, ld: int) -> torch.Tensor:
    out = torch.empty(dim, dtype=torch.float64, device=rows.device)
    _lib.call("chess_mean_rows", _lib.ptr(rows), _lib.F64, n, dim, ld, _lib.ptr(out), _sp())
    return out


def compute_anchor(index, tail, config):
    """Eq.3 (selection.py:44-59): mean of the last min(W, n) page vectors; a
    non-empty unsealed tail is one more page pooled over its filled rows."""
    n = index.num_pages
    sources = list(range(n))
    tail_vec = None
    if tail is not None and tail.fill > 0 and not tail.sealed:
        tk = _f64(tail.keys, index.device)
        tail_vec = _mean_rows(tk, tk.shape[0], index.dim, tk.stride(0))
        sources.append(n)
    total = len(sources)
    if total == 0:
        raise EmptyContextError("no tokens to anchor on")
    w = min(config.window_pages, total)
    if tail_vec is None:
        pv = index._st.page_vec64[0]
        v = _mean_rows(pv[n - w:], w, index.dim, pv.stride(0))
    else:
        win = torch.empty((w, index.dim), dtype=torch.float64, device=index.device)
        if w > 1:
            win[: w - 1].copy_(index.page_vectors[n - (w - 1):])
        win[w - 1].copy_(tail_vec)
        v = _mean_rows(win, w, index.dim, index.dim)
    return QueryAnchor(v=v, source_pages=sources[-w:])


def score_all(anchor, v_all, split_points):
    """Alg.1 line 3 / Eq.4 (selection.py:62-74): one f64 GEMV, split into views."""
    g, c, p = split_points
    dev = anchor.v.device if isinstance(anchor.v, torch.Tensor) else None
    v_all = _f64(v_all, dev)
    if v_all.shape[0] == 0:
        e = torch.zeros(0, dtype=torch.float64, device=v_all.device)
        return e, e, e
    a = _f64(anchor.v, v_all.device)
    if v_all.shape[1] != a.shape[0]:
        raise ValueError(f"dimension mismatch: matrix has {v_all.shape[1]} columns, anchor has {a.shape[0]}")
    scores = torch.empty(v_all.shape[0], dtype=torch.float64, device=v_all.device)
    _lib.call("chess_score_rows", _lib.ptr(v_all), _lib.F64, v_all.shape[0], v_all.shape[1], v_all.stride(0),
              _lib.ptr(a), _lib.ptr(scores), _sp())
    return scores[:g], scores[g:g + c], scores[g + c:]


def hierarchical_prune(s_g, s_c, s_p, page_to_chunk, chunk_to_grid, config):
    """Masked top-k cascade (selection.py:91-111) in one device launch; returns
    the kept logical pages in increasing order."""
    dev = s_p.device if isinstance(s_p, torch.Tensor) and s_p.is_cuda else None
    sg, sc, sp = _f64(s_g, dev), _f64(s_c, dev), _f64(s_p, dev)
    G, Cn, P = sg.numel(), sc.numel(), sp.numel()
    if P == 0:
        return np.zeros(0, dtype=np.intp)
    p2c, c2g = _i64(page_to_chunk, sp.device), _i64(chunk_to_grid, sp.device)
    out = torch.empty(P, dtype=torch.int32, device=sp.device)
    cnt = torch.zeros(3, dtype=torch.int32, device=sp.device)
    ws = torch.empty(_lib.load().chess_prune_workspace_bytes(G, Cn, P), dtype=torch.uint8, device=sp.device)
    _lib.call("chess_prune", _lib.ptr(sg), G, _lib.ptr(sc), Cn, _lib.ptr(sp), P, _lib.ptr(p2c), _lib.ptr(c2g),
              config.rho_grid, config.rho_chunk, config.rho_page, _lib.ptr(out), _lib.ptr(cnt), _lib.ptr(ws), _sp())
    k = int(cnt[0].item())
    return out[:k].cpu().numpy().astype(np.intp)


def oracle_flat_topk(anchor, v_p, k):
    """Exhaustive top-k pages by affinity (selection.py:114-123)."""
    dev = anchor.v.device if isinstance(anchor.v, torch.Tensor) else None
    v_p = _f64(v_p, dev)
    n = v_p.shape[0]
    if k > n:
        raise ValueError(f"k={k} exceeds page count {n}")
    if k <= 0 or n == 0:
        return np.zeros(0, dtype=np.intp)
    s_p = score_all(anchor, v_p, (0, 0, n))[2].contiguous()
    idx = torch.empty(n, dtype=torch.int32, device=v_p.device)
    cnt = torch.zeros(1, dtype=torch.int32, device=v_p.device)
    ws = torch.empty(16 * n + 64, dtype=torch.uint8, device=v_p.device)
    _lib.call("chess_topk", _lib.ptr(s_p), n, int(k), None, _lib.ptr(idx), _lib.ptr(cnt), 1, _lib.ptr(ws), _sp())
    return idx[: int(cnt.item())].cpu().numpy().astype(np.intp)


_PROV = {1: "semantic", 2: "window", 3: "sink"}


def reconstruct_working_set(selected, seq, config):
    """Semantic ∪ window ∪ sinks, sorted, provenance sink > window > semantic
    (selection.py:126-140), computed by the working-set kernel."""
    n = len(seq.page_table)
    if config.window_pages < 1:
        raise ConfigurationError("window_pages must be >= 1")
    sel = np.asarray(selected, dtype=np.int64).reshape(-1)
    sel = sel[(sel >= 0) & (sel < n)] if n else sel[:0]
    if n == 0:
        return WorkingSet(pages=[], provenance={})
    dev = _device()
    sel_d = _i32(sel if sel.size else np.zeros(1), dev)
    pages = torch.empty(n, dtype=torch.int32, device=dev)
    prov = torch.empty(n, dtype=torch.int8, device=dev)
    length = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("chess_working_set", _lib.ptr(sel_d), int(sel.size), n, config.window_pages, seq.sink_count,
              None, _lib.ptr(pages), _lib.ptr(prov), None, _lib.ptr(length), _sp())
    m = int(length.item())
    pg = pages[:m].cpu().tolist()
    pv = prov[:m].cpu().tolist()
    return WorkingSet(pages=pg, provenance={p: _PROV[t] for p, t in zip(pg, pv)})


def trace_record(step, anchor, index, selected_g, selected_c, working_set):
    semantic = [p for p, tag in working_set.provenance.items() if tag == "semantic"]
    return {
        "step": step,
        "anchor_checksum": anchor.checksum(),
        "counts": {"G": index.num_grids, "C": index.num_chunks, "P": index.num_pages,
                   "selected_g": int(selected_g), "selected_c": int(selected_c), "selected_p": len(semantic)},
        "working_set": working_set.pages,
        "provenance": {str(k): v for k, v in sorted(working_set.provenance.items())},
    }


# =============================================================================
# Uncertainty (uncertainty.py:22-124)
# =============================================================================
def entropies(prob_rows) -> torch.Tensor:
    """Batched entropy of every row (nats); raises like `entropy` on a bad row."""
    p = _f64(prob_rows)
    if p.dim() == 1:
        p = p.unsqueeze(0)
    rows, n = p.shape
    if n == 0:
        raise ValueError("distribution sums to 0.0, not 1")
    out = torch.empty(rows, dtype=torch.float64, device=p.device)
    flags = torch.zeros(rows, dtype=torch.int32, device=p.device)
    _lib.call("chess_entropy_probs", _lib.ptr(p), rows, n, p.stride(0), _lib.ptr(out), _lib.ptr(flags), _sp())
    f = int(flags.max().item()) if rows else 0
    if f & 1:
        raise ValueError("probabilities must be non-negative")
    if f & 2:
        bad = int(torch.nonzero(flags & 2)[0, 0])
        raise ValueError(f"distribution sums to {float(p[bad].sum())}, not 1")
    return out


def entropy(probs):
    """Shannon entropy in nats, 0 ln 0 := 0 (uncertainty.py:22-31)."""
    return float(entropies(probs)[0].item())


@dataclass
class PageUncertainty:
    mean_entropy: float
    varentropy: float
    token_count: int


def page_uncertainty(entropies_):
    """Mean and population variance of a page's entropies (uncertainty.py:41-48),
    NumPy pairwise summation order on the device."""
    if len(entropies_) == 0:
        raise ValueError("page has no generated tokens")
    e = _f64(entropies_).reshape(-1)
    out = torch.empty(2, dtype=torch.float64, device=e.device)
    _lib.call("chess_page_uncertainty", _lib.ptr(e), e.numel(), _lib.ptr(out), _sp())
    m, v = out.cpu().tolist()
    return PageUncertainty(mean_entropy=m, varentropy=v, token_count=e.numel())


@dataclass
class TriggerThresholds:
    tau_entropy: float
    tau_varentropy: float
    percentile: float
    sample_count: int


def _nearest_rank(sorted_values, percentile):
    rank = math.ceil(percentile * len(sorted_values))
    return float(sorted_values[max(rank, 1) - 1])


def calibrate(samples, percentile=0.99):
    """Independent nearest-rank percentiles (uncertainty.py:59-83); offline, host."""
    if not samples:
        raise CalibrationError("cannot calibrate on an empty sample")
    if not 0.0 < percentile < 1.0:
        raise CalibrationError(f"percentile must be in (0, 1), got {percentile}")
    if percentile >= 0.99 and len(samples) < 100:
        warnings.warn(f"only {len(samples)} calibration pages for percentile {percentile}; "
                      "thresholds will be coarse", stacklevel=2)
    means = np.sort([s.mean_entropy for s in samples])
    variances = np.sort([s.varentropy for s in samples])
    return TriggerThresholds(_nearest_rank(means, percentile), _nearest_rank(variances, percentile),
                             percentile, len(samples))


def calibrate_device(entropies, counts=None, percentile=0.99, device=None):
    """calibrate (uncertainty.py:59-83) from raw per-token entropy streams on
    the device: page_uncertainty of every page (NumPy pairwise order, so the
    statistics are bit-identical to the host ones) and the independent
    nearest-rank percentiles, in two kernels.  entropies: [pages, n] (array or
    tensor, f64); counts: entries per page (default n each).  Returns the same
    TriggerThresholds as calibrate(page_uncertainty(...) per page)."""
    e = torch.as_tensor(entropies, dtype=torch.float64, device=_device(device)).contiguous()
    if e.dim() != 2 or e.shape[0] == 0:
        raise CalibrationError("cannot calibrate on an empty sample")
    if not 0.0 < percentile < 1.0:
        raise CalibrationError(f"percentile must be in (0, 1), got {percentile}")
    n_pages = int(e.shape[0])
    if percentile >= 0.99 and n_pages < 100:
        warnings.warn(f"only {n_pages} calibration pages for percentile {percentile}; "
                      "thresholds will be coarse", stacklevel=2)
    if counts is None:
        c = torch.full((n_pages,), e.shape[1], dtype=torch.int32, device=e.device)
    else:
        c = torch.as_tensor(counts, dtype=torch.int32, device=e.device).contiguous()
        if bool((c < 1).any()) or bool((c > e.shape[1]).any()):
            raise ValueError("page has no generated tokens")
    out = torch.empty(2, dtype=torch.float64, device=e.device)
    ws = torch.empty(_lib.load().chess_calibrate_workspace_bytes(n_pages), dtype=torch.uint8, device=e.device)
    _lib.call("chess_calibrate", _lib.ptr(e), _lib.ptr(c), n_pages, e.stride(0), float(percentile),
              _lib.ptr(out), _lib.ptr(ws), _sp())
    tau = out.cpu().tolist()
    return TriggerThresholds(tau[0], tau[1], percentile, n_pages)


def check_trigger(u, thresholds, mode="joint"):
    """Strict joint / any test (uncertainty.py:86-98)."""
    high_h = u.mean_entropy > thresholds.tau_entropy
    high_v = u.varentropy > thresholds.tau_varentropy
    if mode == "joint":
        return high_h and high_v
    if mode == "any":
        return high_h or high_v
    raise ValueError(f"unknown trigger mode {mode!r}")


def save_thresholds(thresholds, path, created_from=""):
    with open(path, "w") as fh:
        json.dump({"percentile": thresholds.percentile, "tau_H": thresholds.tau_entropy,
                   "tau_V": thresholds.tau_varentropy, "sample_count": thresholds.sample_count,
                   "created_from": created_from}, fh, indent=2)


def load_thresholds(path):
    with open(path) as fh:
        data = json.load(fh)
    return TriggerThresholds(data["tau_H"], data["tau_V"], data["percentile"], data["sample_count"])


# =============================================================================
# Page-granular decode loop (simulate.py:28-226)
# =============================================================================
@dataclass
class StepRecord:
    step: int
    working_set_size: int
    budget_fraction_semantic: float
    budget_fraction_total: float
    recall: float
    precision: float
    trigger_fired: bool
    selection_ops: int
    attention_ops: int


@dataclass
class RunReport:
    steps: list = field(default_factory=list)
    trigger_count: int = 0
    mean_recall: float = 0.0
    mean_precision: float = 0.0
    mean_budget_semantic: float = 0.0
    mean_budget_total: float = 0.0
    mean_inter_trigger_gap: float = 0.0
    zero_copy_ok: bool = True
    working_sets: list = field(default_factory=list, repr=False)

    def summary(self):
        keys = ("trigger_count", "mean_recall", "mean_precision", "mean_budget_semantic", "mean_budget_total",
                "mean_inter_trigger_gap", "zero_copy_ok")
        return {"steps": len(self.steps), **{k: getattr(self, k) for k in keys}}

    def write_jsonl(self, path):
        with open(path, "w") as fh:
            for rec in self.steps:
                fh.write(json.dumps(asdict(rec)) + "\n")


def parse_policy(policy):
    if isinstance(policy, tuple):
        return policy
    if policy in ("dynamic", "never", "always"):
        return (policy, None)
    if isinstance(policy, str) and policy.startswith("fixed(") and policy.endswith(")"):
        interval = int(policy[6:-1])
        if interval < 1:
            raise ConfigurationError("fixed interval must be >= 1 page")
        return ("fixed", interval)
    raise ConfigurationError(f"unknown policy {policy!r}; expected dynamic, never, always or fixed(N)")


def page_entropies(probs_block):
    return entropies(probs_block).cpu().tolist()


def collect_page_uncertainties(spec):
    load = generate_workload(spec)
    B = spec.page_size
    return [page_uncertainty(entropies(load.gen_probs[g * B:(g + 1) * B]))
            for g in range(spec.generation_pages)]


def run_decode_loop(spec, config, policy, thresholds=None, trigger_mode="joint", device=None):
    """Prefill + page-by-page generation under a trigger policy
    (simulate.py:110-217), every store/index/selector/uncertainty step on
    the device.  The report additionally carries each page's working set."""
    kind, interval = parse_policy(policy)
    if kind == "dynamic" and thresholds is None:
        raise ConfigurationError("policy 'dynamic' needs calibrated thresholds")
    if spec.page_size != config.page_size:
        raise ConfigurationError("workload and selection page sizes differ")
    if spec.pages_per_chunk != config.pages_per_chunk:
        raise ConfigurationError("workload and selection chunk fan-outs differ")
    dev = _device(device)
    load = generate_workload(spec)
    B = config.page_size
    store = PagedKvStore(spec.context_pages + spec.generation_pages + 1, spec.dim, B, dev)
    seq = store.create_sequence(config)
    index = HierarchyIndex(spec.dim, config.pages_per_chunk, config.chunks_per_grid, dev)
    sealed_at = {}

    def append_block(keys, values):
        kd, vd = _f64(keys, dev), _f64(values, dev)
        for i in range(kd.shape[0]):
            ev = store.append_token(seq, kd[i], vd[i])
            if ev.sealed:
                index.finalize_page(store.page(ev.page_id), ev.logical_index)
                sealed_at[ev.page_id] = store.page(ev.page_id).version

    def run_selection():
        anchor = compute_anchor(index, None, config)
        v_all, splits = index.coalesced_matrix()
        s_g, s_c, s_p = score_all(anchor, v_all, splits)
        sel = hierarchical_prune(s_g, s_c, s_p, index.page_to_chunk, index.chunk_to_grid, config)
        return sel, v_all.shape[0] * (spec.dim + 1)

    append_block(load.context_keys, load.context_values)
    pending = 0
    if kind == "never":
        semantic = np.arange(index.num_pages)
    else:
        semantic, pending = run_selection()
    report = RunReport()
    fired_pages = []
    for g in range(spec.generation_pages):
        lo, hi = g * B, (g + 1) * B
        append_block(load.gen_keys[lo:hi], load.gen_values[lo:hi])
        stats = page_uncertainty(entropies(load.gen_probs[lo:hi]))
        if kind == "never":
            fired = False
        elif kind == "always":
            fired = True
        elif kind == "fixed":
            fired = (g + 1) % interval == 0
        else:
            fired = check_trigger(stats, thresholds, mode=trigger_mode)
        ops, pending = pending, 0
        if fired:
            semantic, o = run_selection()
            ops += o
            fired_pages.append(g)
        sealed = index.num_pages
        if kind == "never":
            semantic = np.arange(sealed)
        ws = reconstruct_working_set(semantic, seq, config)
        report.working_sets.append(list(ws.pages))
        rel = load.relevant_pages
        hits = len(rel & set(ws.pages))
        report.steps.append(StepRecord(
            step=g, working_set_size=len(ws),
            budget_fraction_semantic=min(1.0, len(semantic) / sealed),
            budget_fraction_total=min(1.0, len(ws) / sealed),
            recall=hits / len(rel) if rel else 1.0,
            precision=hits / len(ws) if len(ws) else 0.0,
            trigger_fired=fired, selection_ops=ops,
            attention_ops=B * 2 * len(ws) * B * spec.dim))
    report.zero_copy_ok = all(store.page(pid).version == v for pid, v in sealed_at.items())
    if report.steps:
        report.mean_recall = float(np.mean([s.recall for s in report.steps]))
        report.mean_precision = float(np.mean([s.precision for s in report.steps]))
        report.mean_budget_semantic = float(np.mean([s.budget_fraction_semantic for s in report.steps]))
        report.mean_budget_total = float(np.mean([s.budget_fraction_total for s in report.steps]))
    report.trigger_count = len(fired_pages)
    report.mean_inter_trigger_gap = spec.generation_pages / max(1, len(fired_pages))
    return report


def selection_overhead_profile(report):
    sel = sum(s.selection_ops for s in report.steps)
    attn = sum(s.attention_ops for s in report.steps)
    return 0.0 if sel + attn == 0 else sel / (sel + attn)
