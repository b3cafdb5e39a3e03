"""TEST INFRASTRUCTURE ONLY — NumPy restatement of the pagesel hot path.

Each function cites the reference lines it restates
(/root/reference/pkg/src/pagesel/...).  Arithmetic is float64 in the same
operation order as the reference, so on identical inputs the outputs are
bit-identical to pagesel (pinned by tests/test_oracle_golden.py against
vectors generated from the reference itself).
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# hierarchy.py — Eq.1 page means, chunk running sums, grid sums of centroids
# ---------------------------------------------------------------------------


def page_mean(keys) -> np.ndarray:
    """Eq.1 pooling: f64 mean of the page's key rows (hierarchy.py:115)."""
    return np.asarray(keys).astype(np.float64).mean(axis=0)


def checksum16(matrix) -> str:
    """hierarchy.py:16-17 / selection.py:24-25 checksum format."""
    return hashlib.sha256(np.ascontiguousarray(matrix).tobytes()).hexdigest()[:16]


class Hierarchy:
    """Three-level centroid index (hierarchy.py:26-146).

    State is kept exactly as the reference keeps it: page rows, chunk sums +
    counts, grid sums (of chunk centroids) + counts; centroids are divided
    out on read (hierarchy.py:78-92).
    """

    def __init__(self, dim, n_c, n_g):
        self.dim, self.n_c, self.n_g = dim, n_c, n_g
        self.pages: list = []
        self.c_sum: list = []
        self.c_cnt: list = []
        self.g_sum: list = []
        self.g_cnt: list = []

    # hierarchy.py:102-136
    def fold(self, v, logical_index=None):
        if logical_index is not None and logical_index != len(self.pages):
            raise ValueError(
                f"pages finalize in order: expected index {len(self.pages)}, got {logical_index}"
            )
        p = len(self.pages)
        self.pages.append(v)
        c, g = p // self.n_c, (p // self.n_c) // self.n_g
        if c == len(self.c_sum):  # first page of a new chunk
            self.c_sum.append(v.copy())
            self.c_cnt.append(1)
            cen = self.c_sum[c] / self.c_cnt[c]
            if g == len(self.g_sum):
                self.g_sum.append(cen.copy())
                self.g_cnt.append(1)
            else:
                self.g_sum[g] += cen
                self.g_cnt[g] += 1
        else:  # grid tracks the change of this chunk's centroid
            before = self.c_sum[c] / self.c_cnt[c]
            self.c_sum[c] += v
            self.c_cnt[c] += 1
            after = self.c_sum[c] / self.c_cnt[c]
            self.g_sum[g] += after - before
        return v

    def fold_page(self, keys, logical_index=None):
        return self.fold(page_mean(keys), logical_index)

    # hierarchy.py:43-58
    @classmethod
    def from_rows(cls, rows, n_c, n_g):
        rows = np.asarray(rows, dtype=np.float64)
        h = cls(rows.shape[1] if rows.size else 0, n_c, n_g)
        h.pages = list(rows)
        for lo in range(0, rows.shape[0], n_c):
            grp = rows[lo : lo + n_c]
            h.c_sum.append(grp.sum(axis=0))
            h.c_cnt.append(grp.shape[0])
        cv = h.chunk_vectors
        for lo in range(0, cv.shape[0], n_g):
            grp = cv[lo : lo + n_g]
            h.g_sum.append(grp.sum(axis=0))
            h.g_cnt.append(grp.shape[0])
        return h

    @property
    def page_vectors(self):
        return np.asarray(self.pages) if self.pages else np.zeros((0, self.dim))

    @property
    def chunk_vectors(self):
        if not self.c_sum:
            return np.zeros((0, self.dim))
        return np.asarray(self.c_sum) / np.asarray(self.c_cnt, dtype=np.float64)[:, None]

    @property
    def grid_vectors(self):
        if not self.g_sum:
            return np.zeros((0, self.dim))
        return np.asarray(self.g_sum) / np.asarray(self.g_cnt, dtype=np.float64)[:, None]

    @property
    def counts(self):
        return (len(self.g_sum), len(self.c_sum), len(self.pages))

    def parent_maps(self):
        """page_to_chunk, chunk_to_grid (hierarchy.py:94-100)."""
        g, c, p = self.counts
        return np.arange(p) // self.n_c, np.arange(c) // self.n_g

    def coalesced(self):
        """[V_g; V_c; V_p] and (G, C, P) (hierarchy.py:138-146)."""
        g, c, p = self.counts
        if p == 0:
            return np.zeros((0, self.dim)), (0, 0, 0)
        return np.concatenate([self.grid_vectors, self.chunk_vectors, self.page_vectors]), (g, c, p)

    def snapshot(self):
        g, c, p = self.counts
        return {
            "pages_per_chunk": self.n_c,
            "chunks_per_grid": self.n_g,
            "num_pages": p,
            "num_chunks": c,
            "num_grids": g,
            "checksum_pages": checksum16(self.page_vectors),
            "checksum_chunks": checksum16(self.chunk_vectors),
            "checksum_grids": checksum16(self.grid_vectors),
        }


# ---------------------------------------------------------------------------
# selection.py — anchor, scoring, masked top-k cascade, working set
# ---------------------------------------------------------------------------


def anchor(page_vectors, window, tail_keys=None):
    """Eq.3 (selection.py:44-59): mean of the last min(W, n) page vectors;
    a non-empty unsealed tail counts as one more page (mean over its rows)."""
    vecs = list(np.asarray(page_vectors, dtype=np.float64))
    src = list(range(len(vecs)))
    if tail_keys is not None and len(tail_keys) > 0:
        vecs.append(np.asarray(tail_keys).astype(np.float64).mean(axis=0))
        src.append(len(src))
    if not vecs:
        raise LookupError("no tokens to anchor on")
    w = min(window, len(vecs))
    return np.asarray(vecs[-w:]).mean(axis=0), src[-w:]


def score(v_all, a):
    """Eq.4 / Alg.1 line 3 (selection.py:62-74): one GEMV."""
    return np.asarray(v_all) @ np.asarray(a)


def top_k(scores, k, active=None):
    """selection.py:77-88: best k among active, ties to the lower index."""
    scores = np.asarray(scores)
    cand = np.flatnonzero(active) if active is not None else np.arange(len(scores))
    if k <= 0 or cand.size == 0:
        return np.zeros(0, dtype=np.intp)
    order = np.argsort(-scores[cand], kind="stable")
    return cand[order[: min(k, cand.size)]]


def prune(s_g, s_c, s_p, p2c, c2g, rhos):
    """hierarchical_prune (selection.py:91-111).  Returns (pages sorted,
    level detail dict with kept grids/chunks and active counts)."""
    rg, rc, rp = rhos
    n_g, n_p = len(s_g), len(s_p)
    info = {"kept_g": [], "kept_c": [], "active_c": 0, "active_p": 0}
    if n_p == 0:
        return np.zeros(0, dtype=np.intp), info
    keep_g = top_k(s_g, math.ceil(rg * n_g))
    gmask = np.zeros(n_g, dtype=bool)
    gmask[keep_g] = True
    act_c = gmask[np.asarray(c2g)]
    keep_c = top_k(s_c, math.ceil(rc * act_c.sum()), act_c)
    cmask = np.zeros(len(s_c), dtype=bool)
    cmask[keep_c] = True
    act_p = cmask[np.asarray(p2c)]
    keep_p = top_k(s_p, math.ceil(rp * act_p.sum()), act_p)
    info.update(
        kept_g=sorted(int(i) for i in keep_g),
        kept_c=sorted(int(i) for i in keep_c),
        active_c=int(act_c.sum()),
        active_p=int(act_p.sum()),
    )
    return np.sort(keep_p), info


def flat_topk(a, v_p, k):
    """oracle_flat_topk (selection.py:114-123)."""
    n = v_p.shape[0]
    if k > n:
        raise ValueError(f"k={k} exceeds page count {n}")
    if k <= 0 or n == 0:
        return np.zeros(0, dtype=np.intp)
    order = np.argsort(-(v_p @ a), kind="stable")
    return np.sort(order[:k])


def working_set(selected, n_pages, window, sinks):
    """reconstruct_working_set (selection.py:126-140): sorted pages and
    provenance with priority sink > window > semantic."""
    prov = {int(i): "semantic" for i in selected}
    for i in range(max(0, n_pages - window), n_pages):
        prov[i] = "window"
    for i in range(min(sinks, n_pages)):
        prov[i] = "sink"
    return sorted(prov), prov


def gather(page_table, logical):
    """gather_pages (kv_store.py:156-166)."""
    out = []
    for i in logical:
        if not 0 <= i < len(page_table):
            raise IndexError(f"logical index {i} out of range for {len(page_table)}-page table")
        out.append(page_table[i])
    return out


def select_for_index(h: Hierarchy, cfg, n_table=None, sinks=None, tail_keys=None):
    """One engine selection pass (simulate.py:135-143) + working set."""
    a, _ = anchor(h.page_vectors, cfg.window_pages, tail_keys)
    v_all, (g, c, p) = h.coalesced()
    s = score(v_all, a)
    p2c, c2g = h.parent_maps()
    sel, info = prune(s[:g], s[g : g + c], s[g + c :], p2c, c2g, cfg.ratios)
    info["scores"] = (s[:g], s[g : g + c], s[g + c :])
    info["anchor"] = a
    return sel, info


# ---------------------------------------------------------------------------
# uncertainty.py — entropy, page statistics, calibration, trigger
# ---------------------------------------------------------------------------

NORMALIZATION_TOL = 1e-9


def entropy(probs):
    """uncertainty.py:22-31 (nats, 0 ln 0 = 0)."""
    p = np.asarray(probs, dtype=np.float64)
    if np.any(p < 0):
        raise ValueError("probabilities must be non-negative")
    tot = p.sum()
    if abs(tot - 1.0) > NORMALIZATION_TOL:
        raise ValueError(f"distribution sums to {tot}, not 1")
    nz = p[p > 0]
    return float(-np.sum(nz * np.log(nz)))


def entropy_from_logits(logits):
    """Entropy of softmax(logits) in f64 (the reference takes probabilities;
    the device takes logits — SURVEY.md §8c(ii))."""
    x = np.asarray(logits, dtype=np.float64)
    e = np.exp(x - x.max())
    p = e / e.sum()
    nz = p[p > 0]
    return float(-np.sum(nz * np.log(nz)))


def page_stats(entropies):
    """page_uncertainty (uncertainty.py:41-48): mean, population variance."""
    if len(entropies) == 0:
        raise ValueError("page has no generated tokens")
    e = np.asarray(entropies, dtype=np.float64)
    mean = float(e.mean())
    return mean, float(np.mean((e - mean) ** 2)), len(e)


def calibrate(means, variances, percentile=0.99):
    """Independent nearest-rank percentiles (uncertainty.py:59-83)."""
    if len(means) == 0:
        raise ValueError("cannot calibrate on an empty sample")

    def nr(vals):
        vals = np.sort(vals)
        r = math.ceil(percentile * len(vals))
        return float(vals[max(r, 1) - 1])

    return nr(means), nr(variances)


def check_trigger(mean, var, tau_h, tau_v, mode="joint"):
    """uncertainty.py:86-98 (strict inequalities)."""
    hi_h, hi_v = mean > tau_h, var > tau_v
    if mode == "joint":
        return hi_h and hi_v
    if mode == "any":
        return hi_h or hi_v
    raise ValueError(f"unknown trigger mode {mode!r}")


# ---------------------------------------------------------------------------
# workload.py — synthetic planted-relevance workload (same RNG call order)
# ---------------------------------------------------------------------------


def _unit(rng, n, dim):
    x = rng.standard_normal((n, dim))
    return x / np.linalg.norm(x, axis=1, keepdims=True)


def workload(seed=0, dim=256, context_pages=128, relevant_page_fraction=0.02,
             clustering="clustered", signal_strength=4.0, generation_pages=16,
             instability_schedule=(), gen_signal_factor=0.5, page_size=32,
             pages_per_chunk=8, vocab=64):
    """generate_workload (workload.py:96-137) restated; returns a dict."""
    rng = np.random.default_rng(seed)
    signal = _unit(rng, 1, dim)[0]
    # _place_relevant (workload.py:72-86)
    n_rel = round(relevant_page_fraction * context_pages)
    if relevant_page_fraction > 0:
        n_rel = max(n_rel, 1)
    n_rel = min(n_rel, context_pages)
    if n_rel == 0:
        relevant = frozenset()
    elif clustering == "scattered":
        relevant = frozenset(int(i) for i in rng.choice(context_pages, size=n_rel, replace=False))
    else:
        n_starts = max(1, (context_pages - n_rel) // pages_per_chunk + 1)
        start = min(int(rng.integers(n_starts)) * pages_per_chunk, context_pages - n_rel)
        relevant = frozenset(range(start, start + n_rel))
    n_ctx = context_pages * page_size
    ck = _unit(rng, n_ctx, dim)
    cv = _unit(rng, n_ctx, dim)
    for p in relevant:
        ck[p * page_size : (p + 1) * page_size] += signal_strength * signal
    n_gen = generation_pages * page_size
    gk = _unit(rng, n_gen, dim) + (gen_signal_factor * signal_strength) * signal
    gv = _unit(rng, n_gen, dim)
    unstable = {int(p): float(s) for p, s in instability_schedule}
    probs = np.zeros((n_gen, vocab))
    for g in range(generation_pages):
        shift = unstable.get(g)
        for t in range(page_size):
            lam = rng.uniform(0.01, 0.05)
            if shift is not None and t % 2 == 1:
                lam = min(0.98, 1.0 - np.exp(-shift))
            top = int(rng.integers(vocab))
            row = np.full(vocab, lam / vocab)
            row[top] += 1.0 - lam
            probs[g * page_size + t] = row
    return {
        "context_keys": ck, "context_values": cv, "gen_keys": gk, "gen_values": gv,
        "gen_probs": probs, "relevant": relevant, "signal": signal,
    }


# ---------------------------------------------------------------------------
# simulate.py — the page-granular decode loop
# ---------------------------------------------------------------------------


@dataclass
class Step:
    step: int
    working_set_size: int
    budget_fraction_semantic: float
    budget_fraction_total: float
    recall: float
    precision: float
    trigger_fired: bool
    selection_ops: int
    attention_ops: int
    working_set: list = field(default_factory=list)
    semantic: list = field(default_factory=list)
    provenance: dict = field(default_factory=dict)


def decode_loop(load, cfg, policy, tau=None, trigger_mode="joint", dim=None):
    """run_decode_loop (simulate.py:110-217) restated over a workload dict.
    policy: ('never'|'always'|'fixed'|'dynamic', interval)."""
    kind, interval = policy
    B = cfg.page_size
    dim = dim if dim is not None else load["context_keys"].shape[1]
    h = Hierarchy(dim, cfg.pages_per_chunk, cfg.chunks_per_grid)
    n_ctx_pages = load["context_keys"].shape[0] // B
    n_gen_pages = load["gen_keys"].shape[0] // B

    def select():
        sel, _ = select_for_index(h, cfg)
        v_all, _ = h.coalesced()
        return sel, v_all.shape[0] * (dim + 1)

    for p in range(n_ctx_pages):
        h.fold_page(load["context_keys"][p * B : (p + 1) * B], p)
    pending = 0
    if kind == "never":
        semantic = np.arange(len(h.pages))
    else:
        semantic, pending = select()
    steps, fired_pages = [], []
    for g in range(n_gen_pages):
        h.fold_page(load["gen_keys"][g * B : (g + 1) * B], len(h.pages))
        ents = [entropy(r) for r in load["gen_probs"][g * B : (g + 1) * B]]
        mean, var, _ = page_stats(ents)
        if kind == "never":
            fired = False
        elif kind == "always":
            fired = True
        elif kind == "fixed":
            fired = (g + 1) % interval == 0
        else:
            fired = check_trigger(mean, var, tau[0], tau[1], trigger_mode)
        ops, pending = pending, 0
        if fired:
            semantic, o = select()
            ops += o
            fired_pages.append(g)
        sealed = len(h.pages)
        if kind == "never":
            semantic = np.arange(sealed)
        pages, prov = working_set(semantic, sealed, cfg.window_pages, cfg.sink_pages)
        rel = load["relevant"]
        hits = len(rel & set(pages))
        steps.append(Step(
            step=g,
            working_set_size=len(pages),
            budget_fraction_semantic=min(1.0, len(semantic) / sealed),
            budget_fraction_total=min(1.0, len(pages) / sealed),
            recall=hits / len(rel) if rel else 1.0,
            precision=hits / len(pages) if pages else 0.0,
            trigger_fired=bool(fired),
            selection_ops=int(ops),
            attention_ops=B * 2 * len(pages) * B * dim,
            working_set=list(pages),
            semantic=[int(i) for i in semantic],
            provenance=dict(prov),
        ))
    return steps, fired_pages
