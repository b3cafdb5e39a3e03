// k_attn.cu — K4 sparse paged decode attention over the CHESS block table.
//
// Not present in the reference: pagesel only counts attention work
// (simulate.py:186, B*2*|WS|*B*D).  The paper runs FlashInfer's paged decode
// over the reconstructed context; oracle restated in
// oracle/attention.py (fp64 softmax(q K^T / sqrt(d)) V over the working set
// in increasing logical order, rows >= fill never read — SPEC.md:29).
//
// B200 design:
//  * stream-K split: the (slot, kv-head, page) units of one layer are cut
//    into equal contiguous ranges, one per persistent CTA (2 per SM), so every
//    SM streams the same number of pages (+-1) regardless of |WS| skew;
//  * a producer warp walks its range and issues cp.async.bulk (TMA 1-D bulk)
//    copies of each page's K and V tile (8 KB each at B=32, d=128; only the
//    filled rows of the tail page) into an NSTAGE-deep shared-memory ring
//    guarded by mbarriers; 4 consumer warps compute;
//  * GQA: one CTA pass serves all q heads of a kv head, so every K/V byte is
//    read from HBM exactly once per layer;
//  * QK^T: lanes split d, a warp transpose-reduce turns 32 (token, head)
//    partials into 32 finished scores with 31 shuffles; online softmax in
//    exp2 domain; PV: lanes own d pairs;
//  * segments cut by CTA boundaries are merged by the last CTA to finish
//    (atomic counter), in CTA order — deterministic.
#include "common.cuh"

namespace chess {

namespace {

constexpr int kConsumerWarps = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct AttnArgs {
  const __nv_bfloat16* k_layer;  // pool base of this layer
  const __nv_bfloat16* v_layer;
  const __nv_bfloat16* q;
  int64_t q_stride;
  __nv_bfloat16* out;
  int64_t out_stride;
  float* lse;
  float scale_log2;  // softmax_scale * log2(e)
};

template <int HD, int GQ, int B>
struct Cfg {
  static constexpr int kEPL = HD / 32;                       // d elements per lane (QK)
  static constexpr int kTPW = B / kConsumerWarps;            // tokens per warp (QK)
  static constexpr int kNPass = (kTPW * GQ <= 32) ? kTPW : 32 / GQ;  // tokens per pass
  static constexpr int kPasses = kTPW / kNPass;
  static constexpr int kNV = kNPass * GQ;                    // values per transpose-reduce
  static constexpr int kPairs = HD / 2;                      // PV: d pairs
  static constexpr int kNG = (kConsumerWarps * 32) / kPairs; // PV token groups
  static constexpr int kTileBytes = B * HD * 2;
  static constexpr int kStages = (96 * 1024) / (2 * kTileBytes) < 16 ? (96 * 1024) / (2 * kTileBytes) : 16;
  static constexpr int kGQP = GQ < 4 ? 4 : GQ;               // padded P row
};

template <int HD, int GQ, int B>
struct Smem {
  using C = Cfg<HD, GQ, B>;
  alignas(128) __nv_bfloat16 k[C::kStages][B * HD];
  alignas(128) __nv_bfloat16 v[C::kStages][B * HD];
  float S[GQ][B];
  alignas(16) float P[B][C::kGQP];
  float A[GQ];
  float ml[GQ][2];
  alignas(16) float red[C::kNG][GQ][HD];
  uint64_t full[C::kStages];
  uint64_t empty[C::kStages];
  int prefix[kMaxBatch + 1];
  int last_flag;
};

__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}

// Unit walk: units of one layer are (segment sg = s*H + h, page i < ws_len[s]).
struct Walker {
  int s, h, i;      // current slot, kv head, page index within WS
  int wslen;
  int64_t seg_begin;  // first unit of the current segment
};

__device__ __forceinline__ int64_t cta_of_unit(int64_t u, int64_t N, int nC) {
  return ((u + 1) * nC + N - 1) / N - 1;
}

template <int HD, int GQ, int B>
__global__ void __launch_bounds__(kThreads, 1)
    sparse_decode_kernel(ChessState st, Workspace ws, AttnArgs args) {
  using C = Cfg<HD, GQ, B>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem<HD, GQ, B>& sm = *reinterpret_cast<Smem<HD, GQ, B>*>(smem_raw);
  const ChessDims& d = st.d;
  const int H = d.kv_heads;
  const int nb = d.batch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  pdl_wait();

  // prefix of ws_len over slots (units = H * prefix)
  if (threadIdx.x < 32) {
    int run = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int s = b0 + lane;
      int x = s < nb ? st.ws_len[s] : 0;
      int incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (s < nb) sm.prefix[s] = run + incl - x;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) sm.prefix[nb] = run;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();

  const int64_t N = (int64_t)H * sm.prefix[nb];
  // every participating CTA owns >= 1 unit, so the CTAs covering a segment
  // are exactly [cta_of_unit(first), cta_of_unit(last)] (merge count below)
  const int nC = (int)min((int64_t)gridDim.x, N);
  const int c = blockIdx.x;
  if (c >= nC) return;
  const int64_t u_begin = (int64_t)c * N / nC;
  const int64_t u_end = (int64_t)(c + 1) * N / nC;
  if (u_begin >= u_end) return;

  // locate the first unit
  Walker wk;
  {
    const int64_t slot_units = u_begin / H;  // not exact: find s with H*prefix[s] <= u_begin
    (void)slot_units;
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if ((int64_t)H * sm.prefix[mid] <= u_begin) lo = mid; else hi = mid;
    }
    // skip empty slots
    while (lo < nb - 1 && (int64_t)H * sm.prefix[lo + 1] <= u_begin) ++lo;
    wk.s = lo;
    wk.wslen = st.ws_len[lo];
    const int64_t r = u_begin - (int64_t)H * sm.prefix[lo];
    wk.h = (int)(r / wk.wslen);
    wk.i = (int)(r - (int64_t)wk.h * wk.wslen);
    wk.seg_begin = (int64_t)H * sm.prefix[lo] + (int64_t)wk.h * wk.wslen;
  }
  auto advance = [&](Walker& w) {
    if (++w.i >= w.wslen) {
      w.seg_begin += w.wslen;
      w.i = 0;
      if (++w.h >= H) {
        w.h = 0;
        do {
          ++w.s;
        } while (w.s < nb && st.ws_len[w.s] == 0);
        if (w.s < nb) w.wslen = st.ws_len[w.s];
      }
    }
  };
  const int64_t n_units = u_end - u_begin;

  if (warp == kConsumerWarps) {
    // ===================== producer =====================
    if (lane == 0) {
      Walker w = wk;
      for (int64_t k = 0; k < n_units; ++k) {
        const int stage = (int)(k % C::kStages);
        const uint32_t ph = (uint32_t)((k / C::kStages) & 1);
        mbar_wait(&sm.empty[stage], ph ^ 1u);
        const int64_t phys = st.block_table[(int64_t)w.s * d.max_ws + w.i];
        const int rows = (w.i == w.wslen - 1) ? st.tail_fill[w.s] : B;
        const uint32_t bytes = (uint32_t)rows * HD * 2;
        const int64_t off = ((phys * H + w.h) * B) * HD;
        mbar_arrive_expect_tx(&sm.full[stage], 2 * bytes);
        tma_load_1d(sm.k[stage], args.k_layer + off, bytes, &sm.full[stage]);
        tma_load_1d(sm.v[stage], args.v_layer + off, bytes, &sm.full[stage]);
        advance(w);
      }
    }
    return;
  }

  // ===================== consumers =====================
  const int ctid = threadIdx.x;  // 0..127
  float q[GQ][C::kEPL];
  float m_run[(GQ + 3) / 4], l_run[(GQ + 3) / 4];
  float o[GQ][2];
  const int dp = ctid % C::kPairs, tg = ctid / C::kPairs;

  auto load_q = [&](const Walker& w) {
    const __nv_bfloat16* qp = args.q + (int64_t)w.s * args.q_stride + (int64_t)w.h * GQ * HD;
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
#pragma unroll
      for (int e = 0; e < C::kEPL; ++e)
        q[g][e] = bf2f(qp[g * HD + lane * C::kEPL + e]) * args.scale_log2;
    }
#pragma unroll
    for (int j = 0; j < (GQ + 3) / 4; ++j) {
      m_run[j] = -INFINITY;
      l_run[j] = 0.f;
    }
#pragma unroll
    for (int g = 0; g < GQ; ++g) o[g][0] = o[g][1] = 0.f;
  };

  Walker w = wk;
  load_q(w);
  for (int64_t k = 0; k < n_units; ++k) {
    const int stage = (int)(k % C::kStages);
    const uint32_t ph = (uint32_t)((k / C::kStages) & 1);
    const int valid = (w.i == w.wslen - 1) ? st.tail_fill[w.s] : B;
    mbar_wait(&sm.full[stage], ph);
    const __nv_bfloat16* Kt = sm.k[stage];
    const __nv_bfloat16* Vt = sm.v[stage];

    // ---- QK^T: lanes split d, transpose-reduce over (token, head) ----
#pragma unroll
    for (int pass = 0; pass < C::kPasses; ++pass) {
      const int t0 = warp * C::kTPW + pass * C::kNPass;
      float val[C::kNV];
#pragma unroll
      for (int tt = 0; tt < C::kNPass; ++tt) {
        float kf[C::kEPL];
        const __nv_bfloat16* kr = Kt + (t0 + tt) * HD + lane * C::kEPL;
        if constexpr (C::kEPL == 4) {
          const uint2 raw = *reinterpret_cast<const uint2*>(kr);
          const float2 a = bf2x2f(raw.x), b = bf2x2f(raw.y);
          kf[0] = a.x; kf[1] = a.y; kf[2] = b.x; kf[3] = b.y;
        } else {
          const uint32_t raw = *reinterpret_cast<const uint32_t*>(kr);
          const float2 a = bf2x2f(raw);
          kf[0] = a.x; kf[1] = a.y;
        }
#pragma unroll
        for (int g = 0; g < GQ; ++g) {
          float x = 0.f;
#pragma unroll
          for (int e = 0; e < C::kEPL; ++e) x = fmaf(q[g][e], kf[e], x);
          val[tt * GQ + g] = x;
        }
      }
      int cnt = C::kNV;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        if (cnt > 1) {
          const int half = cnt >> 1;
          const bool upper = lane & off;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i < half) {
              const float send = upper ? val[i] : val[half + i];
              const float keep = upper ? val[half + i] : val[i];
              val[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
          }
          cnt = half;
        } else {
          val[0] += __shfl_xor_sync(0xffffffffu, val[0], off);
        }
      }
      constexpr int kLogNV = (C::kNV >= 32) ? 5 : (C::kNV >= 16) ? 4 : (C::kNV >= 8) ? 3 : (C::kNV >= 4) ? 2 : (C::kNV >= 2) ? 1 : 0;
      constexpr int kShift = 5 - kLogNV;
      if ((lane & ((1 << kShift) - 1)) == 0) {
        const int vi = lane >> kShift;
        const int tt = vi / GQ, g = vi - (vi / GQ) * GQ;
        const int t = t0 + tt;
        float sc = val[0];
        if (t >= valid || sc != sc) sc = -INFINITY;
        sm.S[g][t] = sc;
      }
    }
    consumer_sync();

    // ---- online softmax (warp w owns heads w, w+4, ...) ----
#pragma unroll
    for (int j = 0; j < (GQ + 3) / 4; ++j) {
      const int g = warp + 4 * j;
      if (g < GQ) {
        const float sc = lane < B ? sm.S[g][lane] : -INFINITY;
        float mx = sc;
#pragma unroll
        for (int o2 = 16; o2 >= 1; o2 >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
        const float m_new = fmaxf(m_run[j], mx);
        const float alpha = exp2f(m_run[j] - m_new);
        const float p = exp2f(sc - m_new);
        float ps = p;
#pragma unroll
        for (int o2 = 16; o2 >= 1; o2 >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o2);
        l_run[j] = l_run[j] * alpha + ps;
        m_run[j] = m_new;
        if (lane < B) sm.P[lane][g] = p;
        if (lane == 0) sm.A[g] = alpha;
      }
    }
    consumer_sync();

    // ---- PV: thread owns d pair dp, token group tg ----
    {
#pragma unroll
      for (int g = 0; g < GQ; ++g) {
        const float a = sm.A[g];
        o[g][0] *= a;
        o[g][1] *= a;
      }
      for (int t = tg; t < valid; t += C::kNG) {
        const float2 vf = bf2x2f(*reinterpret_cast<const uint32_t*>(Vt + t * HD + 2 * dp));
        if constexpr (GQ % 4 == 0) {
#pragma unroll
          for (int g4 = 0; g4 < GQ; g4 += 4) {
            const float4 p4 = *reinterpret_cast<const float4*>(&sm.P[t][g4]);
            o[g4 + 0][0] = fmaf(p4.x, vf.x, o[g4 + 0][0]);
            o[g4 + 0][1] = fmaf(p4.x, vf.y, o[g4 + 0][1]);
            o[g4 + 1][0] = fmaf(p4.y, vf.x, o[g4 + 1][0]);
            o[g4 + 1][1] = fmaf(p4.y, vf.y, o[g4 + 1][1]);
            o[g4 + 2][0] = fmaf(p4.z, vf.x, o[g4 + 2][0]);
            o[g4 + 2][1] = fmaf(p4.z, vf.y, o[g4 + 2][1]);
            o[g4 + 3][0] = fmaf(p4.w, vf.x, o[g4 + 3][0]);
            o[g4 + 3][1] = fmaf(p4.w, vf.y, o[g4 + 3][1]);
          }
        } else {
#pragma unroll
          for (int g = 0; g < GQ; ++g) {
            const float p = sm.P[t][g];
            o[g][0] = fmaf(p, vf.x, o[g][0]);
            o[g][1] = fmaf(p, vf.y, o[g][1]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[stage]);

    // ---- segment flush ----
    const bool seg_end = (w.i == w.wslen - 1) || (k == n_units - 1);
    if (seg_end) {
      // reduce token groups
#pragma unroll
      for (int g = 0; g < GQ; ++g) {
        sm.red[tg][g][2 * dp] = o[g][0];
        sm.red[tg][g][2 * dp + 1] = o[g][1];
      }
#pragma unroll
      for (int j = 0; j < (GQ + 3) / 4; ++j) {
        const int g = warp + 4 * j;
        if (g < GQ && lane == 0) {
          sm.ml[g][0] = m_run[j];
          sm.ml[g][1] = l_run[j];
        }
      }
      consumer_sync();
      const int64_t sg_units_begin = w.seg_begin;
      const int64_t sg_units_end = w.seg_begin + w.wslen;
      const bool whole = (sg_units_begin >= u_begin) && (sg_units_end <= u_end);
      const int sg = w.s * H + w.h;
      for (int idx = ctid; idx < GQ * HD; idx += kConsumerWarps * 32) {
        const int g = idx / HD, e = idx - g * HD;
        float x = sm.red[0][g][e];
#pragma unroll
        for (int t2 = 1; t2 < C::kNG; ++t2) x += sm.red[t2][g][e];
        sm.red[0][g][e] = x;
      }
      consumer_sync();
      if (whole) {
        for (int idx = ctid; idx < GQ * HD; idx += kConsumerWarps * 32) {
          const int g = idx / HD, e = idx - g * HD;
          const float val = sm.red[0][g][e] / sm.ml[g][1];
          args.out[(int64_t)w.s * args.out_stride + ((int64_t)w.h * GQ + g) * HD + e] = __float2bfloat16(val);
        }
        if (args.lse && ctid < GQ)
          args.lse[(int64_t)w.s * d.q_heads + w.h * GQ + ctid] = (sm.ml[ctid][0] + log2f(sm.ml[ctid][1])) * kLn2;
      } else {
        // partial slot (sg + c) ; layout [GQ][HD + 2]
        float* slot = ws.attn_part + (int64_t)(sg + c) * GQ * (HD + 2);
        for (int idx = ctid; idx < GQ * HD; idx += kConsumerWarps * 32) {
          const int g = idx / HD, e = idx - g * HD;
          slot[g * (HD + 2) + e] = sm.red[0][g][e];
        }
        if (ctid < GQ) {
          slot[ctid * (HD + 2) + HD] = sm.ml[ctid][0];
          slot[ctid * (HD + 2) + HD + 1] = sm.ml[ctid][1];
        }
        __threadfence();
        consumer_sync();
        const int c_first = (int)cta_of_unit(sg_units_begin, N, nC);
        const int c_last = (int)cta_of_unit(sg_units_end - 1, N, nC);
        if (ctid == 0) {
          const int prev = atomicAdd(&ws.attn_done[sg], 1);
          sm.last_flag = (prev == c_last - c_first);
        }
        consumer_sync();
        if (sm.last_flag) {
          __threadfence();
          for (int idx = ctid; idx < GQ * HD; idx += kConsumerWarps * 32) {
            const int g = idx / HD, e = idx - g * HD;
            float M = -INFINITY;
            for (int cc = c_first; cc <= c_last; ++cc)
              M = fmaxf(M, __ldcg(ws.attn_part + (int64_t)(sg + cc) * GQ * (HD + 2) + g * (HD + 2) + HD));
            float L = 0.f, O = 0.f;
            for (int cc = c_first; cc <= c_last; ++cc) {
              const float* sl = ws.attn_part + (int64_t)(sg + cc) * GQ * (HD + 2) + g * (HD + 2);
              const float f = exp2f(__ldcg(sl + HD) - M);
              L = fmaf(__ldcg(sl + HD + 1), f, L);
              O = fmaf(__ldcg(sl + e), f, O);
            }
            args.out[(int64_t)w.s * args.out_stride + ((int64_t)w.h * GQ + g) * HD + e] = __float2bfloat16(O / L);
            if (args.lse && e == 0)
              args.lse[(int64_t)w.s * d.q_heads + w.h * GQ + g] = (M + log2f(L)) * kLn2;
          }
          if (ctid == 0) ws.attn_done[sg] = 0;
        }
      }
      consumer_sync();
      advance(w);
      if (k + 1 < n_units) load_q(w);
    } else {
      advance(w);
    }
  }
}

template <int HD, int GQ, int B>
int launch_inst(const ChessState& st, const Workspace& ws, const AttnArgs& args, int nctas,
                cudaStream_t stream) {
  using S = Smem<HD, GQ, B>;
  const size_t smem = sizeof(S);
  static bool configured = false;
  auto kfn = sparse_decode_kernel<HD, GQ, B>;
  if (!configured) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kfn, st, ws, args);
  return check_launch("sparse_decode");
}

}  // namespace

int attn_ctas_for(const ChessDims& d) {
  (void)d;
  return 2 * num_sms();
}

int launch_sparse_decode(const ChessState& st, const Workspace& ws, int layer, const void* q,
                         int64_t q_stride, void* out, int64_t out_stride, float* lse,
                         float softmax_scale, cudaStream_t stream) {
  const ChessDims& d = st.d;
  AttnArgs a;
  const int64_t layer_elems = d.n_phys * d.kv_heads * (int64_t)d.page_size * d.head_dim;
  a.k_layer = reinterpret_cast<const __nv_bfloat16*>(st.k_pool) + layer * layer_elems;
  a.v_layer = reinterpret_cast<const __nv_bfloat16*>(st.v_pool) + layer * layer_elems;
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.q_stride = q_stride;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.out_stride = out_stride;
  a.lse = lse;
  a.scale_log2 = softmax_scale * kLog2e;
  const int gq = d.q_heads / d.kv_heads;
  const int nctas = ws.attn_ctas;
#define CHESS_ATTN_CASE(HD_, GQ_, B_)                                        \
  if (d.head_dim == HD_ && gq == GQ_ && d.page_size == B_)                   \
    return launch_inst<HD_, GQ_, B_>(st, ws, a, nctas, stream);
  CHESS_ATTN_CASE(128, 4, 32)
  CHESS_ATTN_CASE(128, 8, 32)
  CHESS_ATTN_CASE(128, 4, 16)
  CHESS_ATTN_CASE(128, 8, 16)
  CHESS_ATTN_CASE(128, 1, 32)
  CHESS_ATTN_CASE(128, 1, 16)
  CHESS_ATTN_CASE(64, 1, 16)
  CHESS_ATTN_CASE(64, 1, 32)
  CHESS_ATTN_CASE(64, 4, 16)
  CHESS_ATTN_CASE(64, 4, 32)
  CHESS_ATTN_CASE(64, 8, 32)
#undef CHESS_ATTN_CASE
  return fail(CHESS_ERR_UNSUPPORTED, "sparse_decode: no kernel for head_dim=%d gqa=%d page=%d",
              d.head_dim, gq, d.page_size);
}

}  // namespace chess
