"""Random-init Llama-shaped decoder driving the CHESS decode path with real
logits (the paper's nanoVLLM role).

The dense parts (RMSNorm, QKV / o_proj / SwiGLU MLP / lm_head GEMMs, RoPE)
are plain torch ops on bf16 weights (cuBLAS: the model is the CALLER of the
hot path, not part of it).  Per layer the CHESS calls are the ones a serving
engine makes: `chess_append_kv_layers` writes the layer's new K/V row into
the tail page (the layer-0 call opens pages and publishes the counters), and
`chess_sparse_decode` (K4) attends over the slot's working set.  After the
last layer the logits feed `chess_entropy_trigger`, the tail page seals and
the selection runs for the slots that fired (simulate.py:157-182), so the
next token's decode uses the new working set.  Greedy argmax picks the next
token on the device, so a whole token is one capturable CUDA graph.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib
from .engine import ChessDecoder


@dataclass(frozen=True)
class LlamaShape:
    vocab: int
    hidden: int
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    rope_theta: float = 500000.0
    eps: float = 1e-5


LLAMA3_8B = LlamaShape(vocab=128256, hidden=4096, layers=32, q_heads=32, kv_heads=8, head_dim=128, ffn=14336)


class LlamaChess:
    """Weights + one decode token for the whole batch through a ChessDecoder."""

    def __init__(self, shape: LlamaShape, decoder: ChessDecoder, seed: int = 0):
        st = decoder.state.shape
        if (st.layers, st.q_heads, st.kv_heads, st.head_dim) != (shape.layers, shape.q_heads, shape.kv_heads,
                                                                 shape.head_dim):
            raise ValueError("model and decode state disagree on (layers, q_heads, kv_heads, head_dim)")
        self.shape, self.dec, self.state = shape, decoder, decoder.state
        dev = self.state.device
        g = torch.Generator(device=dev).manual_seed(seed)
        bf = dict(dtype=torch.bfloat16, device=dev)
        s = shape

        def w(rows, cols):
            # fan-in scaled normal init, generated in bf16-sized slabs
            t = torch.empty((rows, cols), **bf)
            t.normal_(0.0, 1.0 / math.sqrt(rows), generator=g)
            return t

        qkv = (s.q_heads + 2 * s.kv_heads) * s.head_dim
        self.embed = w(s.vocab, s.hidden) * math.sqrt(s.vocab / s.hidden)
        self.layers = []
        for _ in range(s.layers):
            self.layers.append(dict(
                wqkv=w(s.hidden, qkv), wo=w(s.q_heads * s.head_dim, s.hidden),
                wgu=w(s.hidden, 2 * s.ffn), wd=w(s.ffn, s.hidden),
                n1=torch.ones(s.hidden, **bf), n2=torch.ones(s.hidden, **bf)))
        self.norm = torch.ones(s.hidden, **bf)
        self.lm_head = w(s.hidden, s.vocab)
        half = s.head_dim // 2
        self.inv_freq = 1.0 / (s.rope_theta ** (torch.arange(half, device=dev, dtype=torch.float32) / half))

    def _rms(self, x, wgt):
        return torch.nn.functional.rms_norm(x, (x.shape[-1],), wgt, self.shape.eps)

    def _rope_tables(self, pos):
        """cos/sin [b, 1, d] of the rotate-half form, once per token step."""
        ang = pos.float()[:, None] * self.inv_freq[None, :]
        ang = torch.cat([ang, ang], dim=-1)[:, None, :]
        return ang.cos(), ang.sin()

    @staticmethod
    def _rope(x, cs):
        # x [b, H, d] bf16 (rotate-half convention)
        cos, sin = cs
        xf = x.float()
        h = xf.shape[-1] // 2
        rot = torch.cat([-xf[..., h:], xf[..., :h]], dim=-1)
        return (xf * cos + rot * sin).to(torch.bfloat16)

    def step(self, tokens, logits_out, next_tokens, stream=None):
        """tokens [b] int64 (device) -> logits_out [b, V] f32, next_tokens [b]
        (greedy).  One decode token for every slot; everything on `stream`
        (default: current), no host sync."""
        s, st, dec = self.shape, self.state, self.dec
        b = st.shape.batch
        sp = _lib.stream_ptr(stream)
        cs = self._rope_tables(st.token_count)  # position of the new token = tokens so far
        x = self.embed[tokens]
        hq, hk, d = s.q_heads * s.head_dim, s.kv_heads * s.head_dim, s.head_dim
        for li, lw in enumerate(self.layers):
            h = self._rms(x, lw["n1"])
            qkv = h @ lw["wqkv"]
            # q and k rotated together: [b, H_q + H_kv, d]
            qk = self._rope(qkv[:, :hq + hk].view(b, s.q_heads + s.kv_heads, d), cs)
            q = qk[:, :s.q_heads]
            k = qk[:, s.q_heads:].reshape(b, hk).contiguous()  # k and v share one row stride
            v = qkv[:, hq + hk:].contiguous()
            _lib.call("chess_append_kv_layers", st.ref, li, li + 1, _lib.ptr(k), _lib.ptr(v), k.stride(0), None, sp)
            o = torch.empty((b, s.q_heads, d), dtype=torch.bfloat16, device=x.device)
            dec.attend(li, q, o, None, stream)
            x = torch.addmm(x, o.view(b, hq), lw["wo"])
            h = self._rms(x, lw["n2"])
            gu = h @ lw["wgu"]
            x = torch.addmm(x, torch.nn.functional.silu(gu[:, :s.ffn]) * gu[:, s.ffn:], lw["wd"])
        logits_out.copy_((self._rms(x, self.norm) @ self.lm_head).float())
        next_tokens.copy_(logits_out.argmax(-1))
        dec.entropy_trigger(logits_out, None, stream)
        dec.seal(stream)
        if dec.kind != "never":
            dec.select(force_all=False, stream=stream)

    def capture(self, tokens, logits_out, next_tokens):
        """One decode token as a CUDA graph on static buffers."""
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.step(tokens, logits_out, next_tokens, stream=s)  # warm-up (allocator, cuBLAS handles)
            with torch.cuda.graph(g, stream=s):
                self.step(tokens, logits_out, next_tokens, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        return g


def dense_reference_step(model: LlamaChess, kv_cache, tokens, pos):
    """Pure-torch fp32-attention restatement of one model step over a dense
    per-slot K/V cache (test oracle while the working set is every page, e.g.
    contexts the W-page window covers): kv_cache = list per layer of (K [b, T, H_kv, d], V)
    bf16, extended in place by one position.  Returns logits [b, V] f32."""
    s = model.shape
    b = tokens.shape[0]
    hq, hk, d = s.q_heads * s.head_dim, s.kv_heads * s.head_dim, s.head_dim
    gq = s.q_heads // s.kv_heads
    cs = model._rope_tables(pos)
    x = model.embed[tokens]
    for li, lw in enumerate(model.layers):
        h = model._rms(x, lw["n1"])
        qkv = h @ lw["wqkv"]
        q = model._rope(qkv[:, :hq].view(b, s.q_heads, d), cs)
        k = model._rope(qkv[:, hq:hq + hk].view(b, s.kv_heads, d), cs)
        v = qkv[:, hq + hk:].view(b, s.kv_heads, d)
        K, V = kv_cache[li]
        K = torch.cat([K, k[:, None]], dim=1)
        V = torch.cat([V, v[:, None]], dim=1)
        kv_cache[li] = (K, V)
        Kf = K.float().repeat_interleave(gq, dim=2)  # [b, T, Hq, d]
        Vf = V.float().repeat_interleave(gq, dim=2)
        sc = torch.einsum("bhd,bthd->bht", q.float(), Kf) / math.sqrt(d)
        p = torch.softmax(sc, dim=-1)
        o = torch.einsum("bht,bthd->bhd", p, Vf).to(torch.bfloat16)
        x = x + o.reshape(b, hq) @ lw["wo"]
        h = model._rms(x, lw["n2"])
        gu = h @ lw["wgu"]
        x = x + (torch.nn.functional.silu(gu[:, :s.ffn]) * gu[:, s.ffn:]) @ lw["wd"]
    return (model._rms(x, model.norm) @ model.lm_head).float()
