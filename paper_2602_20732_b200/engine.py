"""Batched device decode engine: the per-token CHESS step on one stream.

One decode token for every slot of the batch:

    append (a1)  ->  L x sparse paged decode (K4)  ->  entropy + trigger (K5)
                 ->  summary seal (K1, slots whose tail just sealed)
                 ->  selection cascade (K2+K3, slots whose trigger fired)

This is the device form of simulate.run_decode_loop's page loop
(simulate.py:157-182) at token granularity: the trigger is evaluated when a
generated page seals, reselection (backtracking) runs for the slots that
fired, and the working set / block table is refreshed whenever the page
table grows (selection.py:126-140).  Every stage is a C-ABI call; the whole
step is capturable as one CUDA graph (no host sync inside).
"""

from __future__ import annotations

import contextlib
import ctypes as C
import math

import torch

from . import _lib
from .config import SelectionConfig
from .state import DecodeState


def _on(stream):
    """Make `stream` torch's current stream (collectives run on it)."""
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def parse_policy(policy):
    """('never'|'always'|'fixed'|'dynamic'|'every_step', interval) (simulate.py:78-91)."""
    from .errors import ConfigurationError

    if isinstance(policy, tuple):
        return policy
    if policy in ("dynamic", "never", "always", "every_step"):
        return (policy, None)
    if isinstance(policy, str) and policy.startswith("fixed(") and policy.endswith(")"):
        interval = int(policy[6:-1])
        if interval < 1:
            raise ConfigurationError("fixed interval must be >= 1 page")
        return ("fixed", interval)
    raise ConfigurationError(
        f"unknown policy {policy!r}; expected dynamic, never, always or fixed(N)"
    )


_POLICY_CODE = {
    "never": _lib.POLICY_NEVER,
    "always": _lib.POLICY_ALWAYS,
    "fixed": _lib.POLICY_FIXED,
    "dynamic": _lib.POLICY_DYNAMIC,
    "every_step": _lib.POLICY_EVERY_STEP,
}


class ChessDecoder:
    def __init__(
        self,
        state: DecodeState,
        config: SelectionConfig,
        policy="dynamic",
        thresholds=None,
        trigger_mode="joint",
        full_scan=False,
        softmax_scale=None,
        exchange=None,
        concurrent_select=None,
    ):
        from .errors import ConfigurationError

        self.state = state
        self.config = config
        s = state.shape
        if config.page_size != s.page_size:
            raise ConfigurationError("state and selection page sizes differ")
        if (config.pages_per_chunk, config.chunks_per_grid) != (s.pages_per_chunk, s.chunks_per_grid):
            raise ConfigurationError("state and selection fan-outs differ")
        if config.window_pages != s.window_pages:
            raise ConfigurationError("state and selection window differ")
        kind, interval = parse_policy(policy)
        if kind == "dynamic" and thresholds is None:
            raise ConfigurationError("policy 'dynamic' needs calibrated thresholds")
        if trigger_mode not in ("joint", "any"):
            raise ValueError(f"unknown trigger mode {trigger_mode!r}")
        self.kind = kind
        self.sel_cfg = _lib.ChessSelectCfg(
            config.rho_grid, config.rho_chunk, config.rho_page, 1 if full_scan else 0, 0
        )
        self.sel_cfg_all = _lib.ChessSelectCfg(
            config.rho_grid, config.rho_chunk, config.rho_page, 1 if full_scan else 0, 1
        )
        # defer_ws twins: the pass leaves working sets pending (concurrent step)
        self.sel_cfg_defer = _lib.ChessSelectCfg(
            config.rho_grid, config.rho_chunk, config.rho_page, 1 if full_scan else 0, 0, 1
        )
        self.sel_cfg_all_defer = _lib.ChessSelectCfg(
            config.rho_grid, config.rho_chunk, config.rho_page, 1 if full_scan else 0, 1, 1
        )
        self.trig_cfg = _lib.ChessTriggerCfg()
        self.trig_cfg.policy = _POLICY_CODE[kind]
        self.trig_cfg.interval = interval or 1
        self.trig_cfg.mode = 0 if trigger_mode == "joint" else 1
        if thresholds is not None:
            self.trig_cfg.tau_entropy = thresholds.tau_entropy
            self.trig_cfg.tau_varentropy = thresholds.tau_varentropy
        self.scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(s.head_dim)
        self.graph = None
        # KV-head shard (parallel.HeadShardExchange): selection runs level by
        # level around the partial-score all-gather; outputs are gathered per layer
        self.exchange = exchange
        if exchange is not None and exchange.levels != ([3] if full_scan else [0, 1, 2]):
            raise ConfigurationError("exchange and decoder disagree on full_scan")
        # Selection of step t only feeds step t+1's decode, so it can run on a
        # side stream concurrently with step t's L decode launches (it fills
        # the SMs and HBM left idle at layer boundaries); its working-set /
        # block-table writes are deferred to chess_flush_working_sets after the
        # join.  Not with a head-shard exchange: two streams of NCCL calls per
        # rank could interleave differently across ranks.
        if concurrent_select is None:
            concurrent_select = exchange is None
        if concurrent_select and exchange is not None:
            raise ConfigurationError("concurrent selection cannot be combined with a head-shard exchange")
        self.concurrent_select = bool(concurrent_select)
        self._side = torch.cuda.Stream(device=state.device) if self.concurrent_select else None

    # ------------------------------------------------------------------
    # prefill: KV rows already in the pool, page tables/counters set
    # ------------------------------------------------------------------
    def build_index(self, n_pages: torch.Tensor, stream=None):
        """K1b: index pages [0, n_pages[s]) of every slot (prefill)."""
        _lib.call("chess_summary_build", self.state.ref, _lib.ptr(n_pages), _lib.stream_ptr(stream))

    # ------------------------------------------------------------------
    # continuous batching: slot eviction / admission (device page pool)
    # ------------------------------------------------------------------
    def evict(self, mask, stream=None):
        """Finish the sequences in `mask` (u8 [batch]): their pool pages go
        back to the free list and the slots are reset (kv_store.py:103-136)."""
        st = self.state
        if st.pool_free is not None:
            st.pool_release(mask, stream)
        st.reset(mask, stream)

    def admit(self, mask, stream=None):
        """Open fresh sequences in the (reset) slots of `mask`: reserve each
        one's first page from the pool; tokens then enter through step()."""
        st = self.state
        counts = mask.to(torch.int32)
        if st.pool_free is not None:
            st.pool_reserve(counts, stream)
        st.sink_count.masked_fill_(mask.bool(), self.config.sink_pages)

    def select(self, force_all=False, stream=None, defer_ws=False):
        if defer_ws:
            cfg = self.sel_cfg_all_defer if force_all else self.sel_cfg_defer
        else:
            cfg = self.sel_cfg_all if force_all else self.sel_cfg
        x = self.exchange
        if x is None:
            _lib.call("chess_select", self.state.ref, C.byref(cfg), _lib.stream_ptr(stream))
            return
        sp = _lib.stream_ptr(stream)
        with _on(stream):
            self._select_levels(cfg, sp)

    def _select_levels(self, cfg, sp):
        x = self.exchange
        for lv in x.levels:
            x.select_level(self.state, cfg, lv, sp)

    def initial_selection(self, stream=None):
        """Post-prefill selection (simulate.py:147-151); 'never' keeps every page."""
        if self.kind == "never":
            st = self.state
            n = st.num_sealed
            ar = torch.arange(st.shape.max_pages, device=st.device, dtype=torch.int32)
            st.semantic.copy_(ar.unsqueeze(0).expand_as(st.semantic))
            st.n_semantic.copy_(n)
            _lib.call("chess_build_working_set", st.ref, _lib.stream_ptr(stream))
        else:
            self.select(force_all=True, stream=stream)

    # ------------------------------------------------------------------
    # one decode token for the whole batch
    # ------------------------------------------------------------------
    def append(self, k_new, v_new, stream=None):
        _lib.call(
            "chess_append_kv", self.state.ref, _lib.ptr(k_new), _lib.ptr(v_new),
            k_new.stride(0), None, _lib.stream_ptr(stream),
        )

    def attend(self, layer, q, out, lse=None, stream=None, after_decode=False):
        """K4 for one layer: q/out [batch, q_heads, head_dim] (batch stride may be padded).

        after_decode: the previous kernel on `stream` writes none of the state
        K4 reads (another K4, or a collective on the outputs), so K4's prologue
        and first page loads may overlap it (CHESS_ATTN_AFTER_DECODE).  False
        after an append, whose writes K4 must wait for."""
        _lib.call(
            "chess_sparse_decode_ex", self.state.ref, layer, _lib.ptr(q), q.stride(0),
            _lib.ptr(out), out.stride(0), _lib.ptr(lse), self.scale,
            _lib.ATTN_AFTER_DECODE if after_decode else 0, _lib.stream_ptr(stream),
        )

    def entropy_trigger(self, logits, entropy_out=None, stream=None):
        _lib.call(
            "chess_entropy_trigger", self.state.ref, _lib.ptr(logits), logits.shape[1],
            logits.stride(0), C.byref(self.trig_cfg), _lib.ptr(entropy_out),
            _lib.stream_ptr(stream),
        )

    def record_entropy(self, entropies, stream=None):
        """K5b: per-slot f64 entropies (computed by the caller from its
        probabilities, simulate.py:160-161) into the open pages' entropy
        rings; page statistics, trigger and policy at seal as with logits."""
        _lib.call("chess_record_entropy", self.state.ref, _lib.ptr(entropies), None,
                  C.byref(self.trig_cfg), _lib.stream_ptr(stream))

    def _uncertainty(self, logits, entropies, entropy_out, stream):
        if entropies is not None:
            self.record_entropy(entropies, stream)
        else:
            self.entropy_trigger(logits, entropy_out, stream)

    def seal(self, stream=None):
        _lib.call("chess_summary_seal", self.state.ref, _lib.stream_ptr(stream))

    def step(self, k_new, v_new, q, logits, out, lse=None, entropy_out=None, stream=None, entropies=None):
        """k_new/v_new [b, D] bf16; q/out [b, L, H_q, d] bf16; logits [b, V] f32;
        lse (optional) f32 [L, b, H_q].  entropies (optional, f64 [b]): the
        token's entropies when the caller holds probabilities instead of
        logits (logits is then ignored, chess_record_entropy).

        Head shard (self.exchange set): D, H_q are this rank's; `out` is the
        per-layer gather buffer [L, world, b, H_q, d] — K4 writes the rank's
        block and the exchange all-gathers it after every layer, or (a
        PeerScoreExchange with fused_outputs) K4 stores the block into every
        rank's region and one chess_gather_finish per step fills `out`."""
        x = self.exchange
        self.append(k_new, v_new, stream)
        if self.concurrent_select and self.kind != "never":
            self._step_concurrent(q, logits, out, lse, entropy_out, stream, entropies)
            return
        if x is not None and getattr(x, "fused_outputs", False):
            # outputs gathered by K4's peer stores; one publish/wait/copy per step
            sp = _lib.stream_ptr(stream)
            for layer in range(self.state.shape.layers):
                x.attend(self.state, layer, q[:, layer], out[layer, x.rank], None if lse is None else lse[layer],
                         self.scale, sp, after_decode=layer > 0)
            x.finish_outputs(self.state, out, sp)
        else:
            for layer in range(self.state.shape.layers):
                o = out[:, layer] if x is None else out[layer, x.rank]
                self.attend(layer, q[:, layer], o, None if lse is None else lse[layer], stream,
                            after_decode=layer > 0)
                if x is not None:
                    with _on(stream):
                        x.outputs(out[layer])
        self._uncertainty(logits, entropies, entropy_out, stream)
        self.seal(stream)
        if self.kind != "never":
            self.select(force_all=False, stream=stream)

    def _step_concurrent(self, q, logits, out, lse, entropy_out, stream, entropies=None):
        """fork { side: entropy+trigger -> seal -> selection (working sets
        deferred) || main: L x decode }, join, flush the pending working sets.
        Same results as the sequential order: the decode reads only KV, q and
        the block table, none of which the side stream writes before the
        flush."""
        cur = stream if stream is not None else torch.cuda.current_stream()
        fork = torch.cuda.Event()
        fork.record(cur)
        side = self._side
        side.wait_event(fork)
        self._uncertainty(logits, entropies, entropy_out, side)
        self.seal(side)
        self.select(force_all=False, stream=side, defer_ws=True)
        for layer in range(self.state.shape.layers):
            self.attend(layer, q[:, layer], out[:, layer], None if lse is None else lse[layer], cur,
                        after_decode=layer > 0)
        join = torch.cuda.Event()
        join.record(side)
        cur.wait_event(join)
        _lib.call("chess_flush_working_sets", self.state.ref, _lib.stream_ptr(cur))

    # ------------------------------------------------------------------
    def capture(self, k_new, v_new, q, logits, out, lse=None, entropy_out=None, entropies=None):
        """Capture `step` on static buffers as one CUDA graph (the graph
        definition is kept, so its nodes and edges can be inspected)."""
        g = torch.cuda.CUDAGraph(keep_graph=True)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self.step(k_new, v_new, q, logits, out, lse, entropy_out, stream=s, entropies=entropies)
        torch.cuda.current_stream().wait_stream(s)
        g.instantiate()
        self.graph = g
        return g
