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

    def scores(self, level: int) -> torch.Tensor:
        self._allgather(self.gathered[level], self.partial[level])
        return self.gathered[level]

    def outputs(self, gather_buf: torch.Tensor) -> torch.Tensor:
        """gather_buf [world, batch, H_q/n, d]; this rank's block is filled."""
        self._allgather(gather_buf, gather_buf[self.rank])
        return gather_buf


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
