"""Multi-GPU partitioning of the CHESS decode path.

One process per GPU; torch.distributed (NCCL on the box, gloo in the CPU
tests) for the plumbing.

Batch shard (cfg4): sequences are independent units (selection, attention,
entropy and trigger are all per sequence), so rank r owns a
contiguous slot range and there is NO data-path collective; the bench reports
weak scaling with the max-over-ranks time.

KV-head shard (cfg5): rank r holds kv heads [r*H/n, (r+1)*H/n) of every
layer, so its flattened key slice is D_r = L * (H/n) * d and its summary rows
give PARTIAL Eq.4 scores (the score is a sum over (layer, head) slices,
selection.py:62-74).  Every level of the cascade all-gathers the partial
scores and sums them in rank order, so every rank holds bit-identical f64
scores and takes the identical top-k; attention outputs of the local query
heads are all-gathered per layer.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class BatchShard:
    rank: int
    world: int
    global_batch: int

    @property
    def slots(self) -> range:
        """Contiguous slot range of this rank (remainder spread over the first ranks)."""
        q, r = divmod(self.global_batch, self.world)
        lo = self.rank * q + min(self.rank, r)
        return range(lo, lo + q + (1 if self.rank < r else 0))


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    layers: int
    kv_heads: int
    q_heads: int
    head_dim: int

    def __post_init__(self):
        if self.kv_heads % self.world:
            raise ValueError(f"kv_heads={self.kv_heads} not divisible by world={self.world}")

    @property
    def local_kv_heads(self) -> int:
        return self.kv_heads // self.world

    @property
    def local_q_heads(self) -> int:
        return self.q_heads // self.world

    @property
    def kv_head_range(self) -> range:
        n = self.local_kv_heads
        return range(self.rank * n, (self.rank + 1) * n)

    @property
    def local_dim(self) -> int:
        return self.layers * self.local_kv_heads * self.head_dim

    def flat_columns(self) -> torch.Tensor:
        """Columns of the reference's flattened (layer, head, d) key row that
        this rank owns (kv_store.py:35 layout), in local order."""
        L, H, d, n = self.layers, self.kv_heads, self.head_dim, self.local_kv_heads
        cols = []
        for layer in range(L):
            base = (layer * H + self.rank * n) * d
            cols.append(torch.arange(base, base + n * d))
        return torch.cat(cols)


class HeadShardExchange:
    """The two exchange steps of the KV-head-sharded decode path on NCCL.

    (1) Scores: every level of the cascade (grids -> chunks of kept grids ->
        pages of kept chunks) runs `chess_select_partial` on the rank's own
        columns, all-gathers the f64 partial scores [batch, ld_level] into
        [world, batch, ld_level], and `chess_select_combine` adds them in rank
        order, so every rank takes the identical top-k and builds the
        identical working set / block table (selection.py:62-111).
    (2) Outputs: K4 writes the rank's query heads straight into its slot of
        the per-layer gather buffer [world, batch, H_q/n, d]; an in-place
        all-gather completes it (rank-major head blocks: global head
        r*H_q/n + j is [r, :, j]).

    Buffers are allocated once, so the exchange is CUDA-graph capturable.
    `allgather` is injectable: the single-GPU tests drive several rank
    states in one process through a local stand-in.
    """

    def __init__(self, shard: "HeadShard", batch: int, max_pages: int, pages_per_chunk: int,
                 chunks_per_grid: int, device, group=None, full_scan=False, allgather=None):
        import math

        self.shard, self.world, self.rank, self.group = shard, shard.world, shard.rank, group
        mc = math.ceil(max_pages / pages_per_chunk)
        mg = math.ceil(mc / chunks_per_grid)
        caps = {0: mg, 1: mc, 2: max_pages, 3: mg + mc + max_pages}
        self.levels = [3] if full_scan else [0, 1, 2]
        f64 = dict(dtype=torch.float64, device=device)
        self.ld = {lv: caps[lv] for lv in self.levels}
        self.partial = {lv: torch.zeros((batch, self.ld[lv]), **f64) for lv in self.levels}
        self.gathered = {lv: torch.zeros((self.world, batch, self.ld[lv]), **f64) for lv in self.levels}
        self._allgather = allgather or self._nccl_allgather

    def _nccl_allgather(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        if self.world == 1 and not dist.is_initialized():
            if out.data_ptr() != inp.data_ptr():
                out[0].copy_(inp)
            return
        # output as [world * rows, ...] (rank blocks concatenated on dim 0)
        dist.all_gather_into_tensor(out.view(-1, *inp.shape[1:]), inp, group=self.group)

    def select_level(self, state, cfg, level, stream_ptr) -> None:
        """One cascade level: partial scan -> all-gather -> rank-ordered combine."""
        import ctypes as C

        from . import _lib

        _lib.call("chess_select_partial", state.ref, C.byref(cfg), level, _lib.ptr(self.partial[level]),
                  self.ld[level], stream_ptr)
        gathered = self.scores(level)
        _lib.call("chess_select_combine", state.ref, C.byref(cfg), level, _lib.ptr(gathered), self.world,
                  self.ld[level], stream_ptr)

    def scores(self, level: int) -> torch.Tensor:
        self._allgather(self.gathered[level], self.partial[level])
        return self.gathered[level]

    def outputs(self, gather_buf: torch.Tensor) -> torch.Tensor:
        """gather_buf [world, batch, H_q/n, d]; this rank's block is filled."""
        self._allgather(gather_buf, gather_buf[self.rank])
        return gather_buf


class PeerScoreExchange(HeadShardExchange):
    """The score exchange of the KV-head shard over peer memory (NVLink).

    Each level is two launches instead of partial -> NCCL all-gather ->
    combine: `chess_select_push` is the partial scan whose tail stores the
    rank's partial rows straight into every rank's receive buffer through
    peer-mapped pointers and release-stores a per-(slot, source) flag;
    `chess_select_pull` waits on its own flags, sums the rows in rank order
    (bit-identical across ranks, as the NCCL path) and finishes the level.
    The all-gather is thereby fused into the scan's epilogue: no collective
    launch, no host involvement, graph capturable (generations on device).

    Memory: one `chess_p2p_alloc` region per rank (cudaMalloc, so its IPC
    handle maps the whole region), per level recv f64 [2][world][batch][ld]
    then flags u32 [batch][world], 256-byte aligned; the same offsets on
    every rank.
    `connect(group)` shares the IPC handles over torch.distributed (any
    backend) and opens the peers' regions; `connect_local(xs)` wires
    in-process rank objects (single-GPU tests).

    Outputs (fused_outputs=True): K4's epilogue stores each output row of the
    rank's query heads into its block of every rank's output region
    (chess_sparse_decode_gather), and one chess_gather_finish per step
    publishes / waits / copies (a two-phase flag barrier) — no per-layer
    all-gather; step counters live on the device, so graph replays work.
    """

    def __init__(self, shard, batch, max_pages, pages_per_chunk, chunks_per_grid, device,
                 group=None, full_scan=False, allgather=None, fused_outputs=True):
        import ctypes as C

        from . import _lib

        super().__init__(shard, batch, max_pages, pages_per_chunk, chunks_per_grid, device, group=group,
                         full_scan=full_scan, allgather=allgather)
        self.batch, self.device = batch, torch.device(device)
        # per-layer output gather fused into K4's epilogue (chess_sparse_decode_gather)
        self.fused_outputs = bool(fused_outputs)
        self.out_elems = (shard.layers * self.world * batch * shard.local_q_heads * shard.head_dim
                          if self.fused_outputs else 0)
        self.offsets, self.nbytes = self.layout(self.world, batch, self.ld, self.out_elems)
        base = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("chess_p2p_alloc", self.nbytes, C.byref(base))
        self.base = base.value
        self._opened = []
        self.gen = {lv: torch.zeros(batch, dtype=torch.int32, device=self.device) for lv in self.levels}
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.px = None

    @staticmethod
    def layout(world: int, batch: int, ld: dict, out_elems: int = 0) -> tuple[dict, int]:
        """{level: (recv offset, flags offset)} (+ {"out": (output region
        offset, output flags offset)} when out_elems, the bf16 elements of the
        output region) and the region size (bytes)."""
        def up(x):
            return (x + 255) // 256 * 256

        off, out = 0, {}
        for lv in sorted(ld):
            recv = off
            flags = up(recv + 2 * world * batch * ld[lv] * 8)
            off = up(flags + batch * world * 4)
            out[lv] = (recv, flags)
        if out_elems:
            region = off
            flags = up(region + out_elems * 2)
            off = up(flags + world * 4)
            out["out"] = (region, flags)
        return out, off

    def connect_local(self, exchanges) -> None:
        self._wire([x.base for x in exchanges])

    def connect(self, group=None) -> None:
        import ctypes as C

        from . import _lib

        if self.world == 1:
            self._wire([self.base])
            return
        h = C.create_string_buffer(64)
        _lib.call("chess_p2p_export", C.c_void_p(self.base), h)
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h.raw), group=group if group is not None else self.group)
        bases = []
        for r, hb in enumerate(handles):
            if r == self.rank:
                bases.append(self.base)
                continue
            p = C.c_void_p()
            with torch.cuda.device(self.device):
                _lib.call("chess_p2p_open", C.create_string_buffer(hb, 64), C.byref(p))
            self._opened.append(p.value)
            bases.append(p.value)
        self._wire(bases)

    def _wire(self, bases) -> None:
        import ctypes as C

        from . import _lib

        if len(bases) != self.world:
            raise ValueError(f"{len(bases)} peer regions for world {self.world}")
        self.px, self._ptrs = {}, {}
        for lv in self.levels:
            ro, fo = self.offsets[lv]
            recv = torch.tensor([b + ro for b in bases], dtype=torch.int64, device=self.device)
            flags = torch.tensor([b + fo for b in bases], dtype=torch.int64, device=self.device)
            self._ptrs[lv] = (recv, flags)
            self.px[lv] = _lib.ChessPeerExchange(
                self.world, self.rank, self.ld[lv], recv.data_ptr(), flags.data_ptr(),
                self.base + ro, self.base + fo, self.gen[lv].data_ptr(), self.err.data_ptr())
        if self.fused_outputs:
            ro, fo = self.offsets["out"]
            self._regions = (C.c_void_p * self.world)(*[b + ro for b in bases])
            oflags = torch.tensor([b + fo for b in bases], dtype=torch.int64, device=self.device)
            self.out_gen = torch.zeros(2, dtype=torch.int32, device=self.device)
            self._ptrs["out"] = (oflags,)
            self.po = _lib.ChessPeerOutputs(self.world, self.rank, self._regions, oflags.data_ptr(),
                                            self.base + fo, self.out_gen.data_ptr(), self.err.data_ptr())

    def attend(self, state, layer, q, out, lse, scale, stream_ptr, after_decode=False) -> None:
        """K4 for one layer: output rows into `out` (this rank's [layer, rank]
        block, [b, H_q/n, d] contiguous) and into every peer's region."""
        import ctypes as C

        from . import _lib

        _lib.call("chess_sparse_decode_gather", state.ref, layer, _lib.ptr(q), q.stride(0), _lib.ptr(out),
                  out.stride(0), _lib.ptr(lse), scale, _lib.ATTN_AFTER_DECODE if after_decode else 0,
                  C.byref(self.po), stream_ptr)

    def finish_outputs(self, state, out, stream_ptr) -> None:
        """Publish this rank's step, wait for every rank's, copy the peers'
        blocks into `out` [L, world, b, H_q/n, d] (contiguous)."""
        import ctypes as C

        from . import _lib

        if out is not None and (not out.is_contiguous() or out.numel() != self.out_elems):
            raise ValueError("finish_outputs: out must be a contiguous [L, world, b, H_q/n, d] buffer")
        _lib.call("chess_gather_finish", state.ref, C.byref(self.po), _lib.ptr(out), stream_ptr)

    def select_level(self, state, cfg, level, stream_ptr) -> None:
        import ctypes as C

        from . import _lib

        if self.px is None:
            raise RuntimeError("PeerScoreExchange not connected (connect / connect_local)")
        px = C.byref(self.px[level])
        _lib.call("chess_select_push", state.ref, C.byref(cfg), level, px, stream_ptr)
        _lib.call("chess_select_pull", state.ref, C.byref(cfg), level, px, stream_ptr)

    def check(self) -> None:
        """Raise if a pull wait timed out (a peer never pushed)."""
        if int(self.err.item()):
            raise RuntimeError("peer score exchange: a pull wait timed out (ranks out of step?)")

    def close(self) -> None:
        from . import _lib

        for p in self._opened:
            _lib.call("chess_p2p_close", p)
        self._opened = []
        if self.base:
            _lib.call("chess_p2p_free", self.base)
            self.base = None


def allgather_sum_scores(partial: torch.Tensor, group=None) -> torch.Tensor:
    """Sum of every rank's partial f64 scores, added in rank order so all
    ranks hold bit-identical results (the cascade then selects identically)."""
    world = dist.get_world_size(group)
    if world == 1:
        return partial.clone()
    parts = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(parts, partial.contiguous(), group=group)
    total = parts[0].clone()
    for p in parts[1:]:
        total += p
    return total


def gather_head_outputs(out_local: torch.Tensor, group=None) -> torch.Tensor:
    """[b, H_q/n, d] per rank -> [b, H_q, d] in head order."""
    world = dist.get_world_size(group)
    if world == 1:
        return out_local
    parts = [torch.empty_like(out_local) for _ in range(world)]
    dist.all_gather(parts, out_local.contiguous(), group=group)
    return torch.cat(parts, dim=1)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (bench timing rule: device time, max over ranks)."""
    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
