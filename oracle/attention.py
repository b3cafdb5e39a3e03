"""TEST INFRASTRUCTURE ONLY — fp64 restatement of sparse paged decode.

The reference never computes attention (simulate.py:186 only counts
B*2*|WS|*B*D ops); the paper runs FlashInfer paged decode over the
reconstructed working set.  This restatement defines the
semantics the CUDA kernel (K4) must match:

  * tokens are the working-set pages in increasing logical order
    (selection.py:126-140, SPEC.md "positional order"), each contributing its
    first `fill` rows — rows >= fill are never read; only the
    last working-set page (the tail) can be partially filled;
  * GQA: query head h attends with kv head h // (H_q / H_kv);
  * o = softmax(q K^T * scale) V, computed in float64 from the bf16 inputs.

Parity for attention is therefore pinned by this restatement, not by the
reference; the tolerance is `bf16_bound` below.
"""

from __future__ import annotations

import numpy as np


def gather_tokens(pool_layer, block_row, ws_len, tail_fill, kv_head):
    """[tokens, d] rows of one (slot, layer, kv head) in working-set order.
    pool_layer: [n_phys, H_kv, B, d]."""
    B = pool_layer.shape[2]
    rows = []
    for i in range(ws_len):
        n = tail_fill if i == ws_len - 1 else B
        rows.append(pool_layer[block_row[i], kv_head, :n, :])
    return np.concatenate(rows, axis=0).astype(np.float64)


def sparse_decode(q, k_pool_layer, v_pool_layer, block_table, ws_len, tail_fill, scale):
    """q: [b, H_q, d]; pools: [n_phys, H_kv, B, d]; returns (o [b,H_q,d], lse [b,H_q])
    in float64 (lse is the natural-log log-sum-exp of the scaled scores)."""
    q = np.asarray(q, dtype=np.float64)
    b, hq, d = q.shape
    hkv = k_pool_layer.shape[1]
    grp = hq // hkv
    out = np.zeros((b, hq, d))
    lse = np.zeros((b, hq))
    for s in range(b):
        n = int(ws_len[s])
        if n == 0:
            continue
        for h in range(hkv):
            K = gather_tokens(k_pool_layer, block_table[s], n, int(tail_fill[s]), h)
            V = gather_tokens(v_pool_layer, block_table[s], n, int(tail_fill[s]), h)
            for g in range(grp):
                qh = h * grp + g
                z = (K @ q[s, qh]) * scale
                m = z.max()
                e = np.exp(z - m)
                out[s, qh] = (e @ V) / e.sum()
                lse[s, qh] = m + np.log(e.sum())
    return out, lse


def bf16_bound(q, k_pool_layer, v_pool_layer, block_table, ws_len, tail_fill, scale, o_ref):
    """Per-element error bound of a bf16-P / fp32-accumulate / bf16-output
    decode kernel against the fp64 result o_ref:

        |o - o_ref| <= (1 + 2^-6) * 2^-8 * (sum_i p_i |v_i| + |o_ref|)

    bf16 carries 8 significant bits, so round-to-nearest is within 2^-8
    relative.  P enters the PV product rounded to bf16, which moves the
    weighted mean by <= 2^-8 * sum_i p_i |v_i| (the normaliser l is
    accumulated from the unrounded p); the output is rounded to bf16
    (<= 2^-8 |o|); the 2^-6 margin covers fp32 accumulation and the
    online-softmax rescaling.  sum_i p_i |v_i| is the same attention run on
    |V|."""
    o_abs, _ = sparse_decode(q, k_pool_layer, np.abs(v_pool_layer), block_table, ws_len, tail_fill, scale)
    return (1.0 + 2.0 ** -6) * 2.0 ** -8 * (o_abs + np.abs(o_ref))
