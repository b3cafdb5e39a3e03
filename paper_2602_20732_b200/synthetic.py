"""Synthetic model-shaped decode workloads for the bench and the GPU tests.

Shapes are BASELINE.json's configs.  Inputs follow the reference's planted-
relevance recipe (workload.py:96-137) restated per head slice, on device:

  * keys: per (token, layer, kv head) unit-norm random d-vectors; on ~1% of
    each sequence's context pages (clustered, chunk-aligned, workload.py:72-86)
    a per-sequence unit signal direction (per head slice) is added with
    strength 4.0; generated keys carry 0.5x the signal (workload.py:111-113);
  * values, queries: N(0, 1) bf16;
  * logits: log of the one-hot/uniform mixture (workload.py:89-93) with
    lambda ~ U(0.01, 0.05); scheduled instability pages alternate
    lambda = 1 - e^-2 on odd tokens (workload.py:116-126).

KV capacity: at full layer count the context KV of cfg3/cfg4/cfg5 exceeds one
B200's HBM, so logical context pages alias onto a smaller physical pool.
Every page a steady-state working set holds — the sink, the planted relevant
run, the last context pages (window) and every generated page — gets a
dedicated physical page, so working sets of different slots never share a
page (no L2 hits between slots inside one attention launch); only the
remaining background context pages alias, onto the rest of the pool
(phys = n_dedicated + (slot*P + p) mod n_background).  Bytes reported are the
logical bytes read; the pool stays far larger than L2 (126 MB).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .state import DecodeState, Shape

CONFIGS = {
    # name: model shape, context tokens, page size, batch, vocab
    "cfg1": dict(layers=2, kv_heads=8, q_heads=8, head_dim=64, ctx=4096, page=16, batch=1, vocab=32000),
    "cfg2": dict(layers=32, kv_heads=8, q_heads=32, head_dim=128, ctx=32768, page=32, batch=1, vocab=128256),
    "cfg3": dict(layers=32, kv_heads=8, q_heads=32, head_dim=128, ctx=131072, page=32, batch=16, vocab=128256),
    "cfg4": dict(layers=32, kv_heads=8, q_heads=32, head_dim=128, ctx=32768, page=32, batch=128, vocab=128256),
    "cfg5": dict(layers=80, kv_heads=8, q_heads=64, head_dim=128, ctx=131072, page=32, batch=8, vocab=128256),
}

DESCRIPTIONS = {
    "cfg1": "tiny Llama-style (2 layers, 8 heads, head_dim 64), 4K context, page 16, 1% KV",
    "cfg2": "Llama-3-8B shape (32 q / 8 kv heads, head_dim 128), 32K context, batch 1, 1% KV",
    "cfg3": "Llama-3-8B shape, 128K context, batch 16, 1% KV, backtracking enabled",
    "cfg4": "Llama-3-8B shape, 32K context, batch 128 (batch-sharded)",
    "cfg5": "Llama-3-70B shape (64 q / 8 kv heads), 128K context, batch 8",
}

GIB = 1 << 30


def mixture_entropy(lam, vocab):
    """Closed-form entropy (nats) of the workload.py:89-93 mixture."""
    q = lam / vocab
    top = 1.0 - lam + q
    return -(top * np.log(top) + (vocab - 1) * q * np.log(q))


def calibrate_thresholds(vocab, page, pages=200, seed=100, percentile=0.99):
    """Offline calibration on a stable stream (uncertainty.py:59-83 recipe):
    nearest-rank percentiles of page mean entropy and varentropy."""
    rng = np.random.default_rng(seed)
    lam = rng.uniform(0.01, 0.05, size=(pages, page))
    h = mixture_entropy(lam, vocab)
    means = h.mean(axis=1)
    var = ((h - means[:, None]) ** 2).mean(axis=1)

    def nr(v):
        v = np.sort(v)
        return float(v[max(math.ceil(percentile * len(v)), 1) - 1])

    return nr(means), nr(var)


@dataclass
class Thresholds:
    tau_entropy: float
    tau_varentropy: float


class SyntheticDecode:
    """Device state + input rings for one model-shaped config."""

    def __init__(self, cfg_name="cfg3", batch=None, gen_pages=128, ring=64, seed=0,
                 device="cuda", summary_dtype="f32", kv_budget_gib=None, unstable_every=2,
                 window=4, nc=8, ng=8, head_shard=None, page_size=None):
        c = dict(CONFIGS[cfg_name])
        if page_size is not None:  # page-size sweep (32 default, 16 swept)
            c["page"] = page_size
        if head_shard is not None:
            # KV-head shard: this rank's kv / q heads of every layer
            _, world = head_shard
            if c["kv_heads"] % world or c["q_heads"] % world:
                raise ValueError(f"{cfg_name}: heads not divisible by world={world}")
            c["kv_heads"] //= world
            c["q_heads"] //= world
        self.head_shard = head_shard
        self.name = cfg_name
        self.c = c
        b = batch if batch is not None else c["batch"]
        B = c["page"]
        P = c["ctx"] // B
        self.P, self.B, self.batch = P, B, b
        L, H, d = c["layers"], c["kv_heads"], c["head_dim"]
        page_bytes = L * H * B * d * 2 * 2  # K+V, all layers
        max_pages = P + gen_pages
        shape0 = Shape(batch=b, layers=L, kv_heads=H, q_heads=c["q_heads"], head_dim=d,
                       page_size=B, pages_per_chunk=nc, chunks_per_grid=ng, max_pages=max_pages,
                       window_pages=window, max_ws=max_pages, n_phys=1, summary_dtype=summary_dtype)
        dim = shape0.dim
        mc, mg = shape0.max_chunks, shape0.max_grids
        state_bytes = b * dim * 8 * (max_pages + 2 * mc + 2 * mg + 4)
        if summary_dtype in ("f32", "bf16", "f16tc"):  # f16tc: fp16 rows in f32-pitch buffers
            state_bytes += b * dim * (2 if summary_dtype == "bf16" else 4) * (max_pages + mc + mg)
        free, total = torch.cuda.mem_get_info(device)
        ring_bytes = ring * b * (c["vocab"] * 4 + L * c["q_heads"] * d * 2 * 2 + dim * 4)
        budget = kv_budget_gib * GIB if kv_budget_gib else free - state_bytes - ring_bytes - 12 * GIB
        need_phys = b * P + b * gen_pages
        n_phys = int(min(need_phys, max(budget // page_bytes, b * gen_pages + 64)))
        self.n_gen_phys = b * gen_pages
        self.n_ctx_phys = n_phys - self.n_gen_phys
        self.aliased = self.n_ctx_phys < b * P
        self.shape = Shape(**{**shape0.__dict__, "n_phys": n_phys})
        torch.manual_seed(seed)
        self.gen = torch.Generator(device=device).manual_seed(seed)
        self.st = DecodeState(self.shape, device=device)
        self.st.reset()
        self.device = self.st.device
        self._fill_tables()
        self._fill_kv(seed)
        self.vocab = c["vocab"]
        self.tau = Thresholds(*calibrate_thresholds(self.vocab, B))
        self.ring = ring
        self.unstable_every = unstable_every
        self._make_inputs(ring)

    # ------------------------------------------------------------------
    DEDICATED_TAIL = 8  # last context pages with dedicated physical pages (>= the window)

    def _fill_tables(self):
        b, P, B = self.batch, self.P, self.B
        st = self.st
        mp = self.shape.max_pages
        # planted relevant pages: ceil(1%) clustered, chunk-aligned (workload.py:72-86)
        rng = np.random.default_rng(1234)
        n_rel = max(1, round(0.01 * P))
        self.relevant = []
        nc = self.shape.pages_per_chunk
        for s in range(b):
            n_starts = max(1, (P - n_rel) // nc + 1)
            start = min(int(rng.integers(n_starts)) * nc, P - n_rel)
            self.relevant.append(list(range(start, start + n_rel)))
        tab = torch.empty((b, mp), dtype=torch.int64)
        ar = torch.arange(P, dtype=torch.int64)
        g = mp - P
        if not self.aliased:
            for s in range(b):
                tab[s, :P] = s * P + ar
        else:
            ded = [sorted({0, *self.relevant[s], *range(max(0, P - self.DEDICATED_TAIL), P)}) for s in range(b)]
            n_ded = sum(len(d_) for d_ in ded)
            n_bg = self.n_ctx_phys - n_ded
            if n_bg < 1:
                raise ValueError("KV pool too small for the dedicated working-set pages")
            nxt = 0
            for s in range(b):
                tab[s, :P] = n_ded + (s * P + ar) % n_bg
                d_ = torch.as_tensor(ded[s], dtype=torch.int64)
                tab[s, d_] = nxt + torch.arange(len(ded[s]))
                nxt += len(ded[s])
        for s in range(b):
            tab[s, P:] = self.n_ctx_phys + s * g + torch.arange(g)
        st.page_table.copy_(tab.to(torch.int32))
        st.num_pages.fill_(P)
        st.tail_fill.fill_(B)
        st.token_count.fill_(P * B)
        st.sink_count.fill_(1)
        self.table_cpu = tab

    def _fill_kv(self, seed):
        s = self.shape
        L, H, B, d = s.layers, s.kv_heads, s.page_size, s.head_dim
        st = self.st
        g = self.gen
        self.signal = torch.randn((self.batch, L, H, d), device=self.device, generator=g)
        self.signal /= self.signal.norm(dim=-1, keepdim=True)
        rel_phys = [self.table_cpu[s_, rel].to(self.device) for s_, rel in enumerate(self.relevant)]
        chunk = max(1, (1 << 28) // (H * B * d))  # pages per generation chunk (~1 GiB f32)
        for l in range(L):
            for p0 in range(0, s.n_phys, chunk):
                p1 = min(s.n_phys, p0 + chunk)
                k = torch.randn((p1 - p0, H, B, d), device=self.device, generator=g)
                k /= k.norm(dim=-1, keepdim=True)
                st.k_pool[l, p0:p1].copy_(k)
                st.v_pool[l, p0:p1].copy_(torch.randn((p1 - p0, H, B, d), device=self.device, generator=g))
            for s_ in range(self.batch):
                ph = rel_phys[s_]
                kk = st.k_pool[l, ph].float() + 4.0 * self.signal[s_, l][:, None, :]
                st.k_pool[l, ph] = kk.to(torch.bfloat16)
        del k

    def _make_inputs(self, ring):
        s, b = self.shape, self.batch
        g, dev = self.gen, self.device
        L, H, Hq, d = s.layers, s.kv_heads, s.q_heads, s.head_dim
        k = torch.randn((ring, b, L, H, d), device=dev, generator=g)
        k /= k.norm(dim=-1, keepdim=True)
        k += 2.0 * self.signal.unsqueeze(0)
        self.k_ring = k.reshape(ring, b, s.dim).to(torch.bfloat16)
        self.v_ring = torch.randn((ring, b, s.dim), device=dev, generator=g).to(torch.bfloat16)
        self.q_ring = torch.randn((ring, b, L, Hq, d), device=dev, generator=g).to(torch.bfloat16)
        V = self.vocab
        rng = np.random.default_rng(99)
        self.logit_ring = torch.empty((ring, b, V), device=dev, dtype=torch.float32)
        self.unstable_pages = 0
        for r in range(ring):
            page, t = divmod(r, self.B)
            unstable = self.unstable_every > 0 and page % self.unstable_every == self.unstable_every - 1
            lam = rng.uniform(0.01, 0.05, size=b)
            if unstable and t % 2 == 1:
                lam[:] = min(0.98, 1.0 - math.exp(-2.0))
            top = rng.integers(V, size=b)
            row = torch.log(torch.as_tensor(lam / V, dtype=torch.float32)).to(dev)
            self.logit_ring[r] = row[:, None].expand(b, V)
            p_top = torch.log(torch.as_tensor(1.0 - lam + lam / V, dtype=torch.float32)).to(dev)
            self.logit_ring[r, torch.arange(b, device=dev), torch.as_tensor(top, device=dev)] = p_top
        self.out = torch.zeros((b, L, Hq, d), device=dev, dtype=torch.bfloat16)

    # ------------------------------------------------------------------
    def prefill(self, decoder):
        n = torch.full((self.batch,), self.P, dtype=torch.int32, device=self.device)
        decoder.build_index(n)
        decoder.initial_selection()
        torch.cuda.synchronize()

    def step_inputs(self, r):
        r %= self.ring
        return self.k_ring[r], self.v_ring[r], self.q_ring[r], self.logit_ring[r]
