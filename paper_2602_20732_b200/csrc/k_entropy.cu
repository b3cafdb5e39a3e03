// k_entropy.cu — K5: per-token entropy from logits, page uncertainty and the
// backtracking trigger.
//
// Reference:
//   entropy            uncertainty.py:22-31   -sum p ln p (nats), 0 ln 0 := 0
//   page_uncertainty   uncertainty.py:41-48   mean + population variance
//   check_trigger      uncertainty.py:86-98   strict joint / any
//   policy cadence     simulate.py:163-170    never/always/fixed(N)/dynamic
// The reference consumes probabilities; the device consumes the step's fp32
// logits and computes H(softmax(logits)) in one HBM pass: online per-thread
// (max, sum e, sum e*(x-max)), merged in a fixed tree per CTA and per row.
// Page statistics use NumPy's pairwise summation order so decisions are
// bit-identical given identical per-token entropies.
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace chess {

namespace {

constexpr int kNT = 256;

struct EntArgs {
  const float* logits;
  int64_t vocab;
  int64_t ld;
  double* out;         // optional per-row entropy
  ChessTriggerCfg cfg; // used when with_state
};


// Page statistics + trigger + policy for slot s (thread 0 only).
__device__ void page_trigger(const ChessState& st, const ChessTriggerCfg& cfg, int s) {
  const int B = st.d.page_size;
  double* ring = st.ent_ring + (int64_t)s * B;
  const int n = min(st.ent_count[s], B);
  uint8_t fire = 0;
  if (cfg.policy == CHESS_POLICY_EVERY_STEP) fire = 1;
  if (st.sealed[s] && n > 0) {
    // np.mean: pairwise sum / n ; var = mean((e - mean)**2)
    const double mean = __ddiv_rn(np_pairwise_sum(ring, n, 1), (double)n);
    const double var = __ddiv_rn(np_pairwise(
                                     [=](int i) {
                                       const double dlt = __dsub_rn(ring[i], mean);
                                       return __dmul_rn(dlt, dlt);
                                     },
                                     n),
                                 (double)n);
    st.page_stats[2 * s] = mean;
    st.page_stats[2 * s + 1] = var;
    const int g = st.gen_pages[s];
    switch (cfg.policy) {
      case CHESS_POLICY_NEVER:
        // no selection ever runs: the semantic set is every sealed page
        // (simulate.py:179-180), read from the arange the initial selection
        // stored; the next page-open rebuilds the working set with it
        fire = 0;
        st.n_semantic[s] = st.num_sealed[s] + 1;
        break;
      case CHESS_POLICY_ALWAYS: fire = 1; break;
      case CHESS_POLICY_FIXED: fire = ((g + 1) % cfg.interval) == 0; break;
      case CHESS_POLICY_DYNAMIC: {
        const bool hh = mean > cfg.tau_entropy;
        const bool hv = var > cfg.tau_varentropy;
        fire = cfg.mode == 0 ? (hh && hv) : (hh || hv);
        break;
      }
      default: fire = 1; break;
    }
    st.gen_pages[s] = g + 1;
    if (fire && st.trigger_count) st.trigger_count[s] += 1u;
  }
  st.fire[s] = fire;
}

// (m, S, T) with S = sum e^(x-m), T = sum e^(x-m) (x-m): merge two partial
// triples (float factors; the |dH| bar is 1e-4 nats)
struct MST {
  float m, S, T;
};
__device__ __forceinline__ MST mst_merge(MST a, MST b) {
  if (b.S == 0.f) return a;
  if (a.S == 0.f) return b;
  const float mn = fmaxf(a.m, b.m);
  const float da = a.m - mn, db = b.m - mn;
  const float fa = exp2f(da * 1.4426950408889634f), fb = exp2f(db * 1.4426950408889634f);
  MST r;
  r.m = mn;
  r.T = fmaf(a.S, da, a.T) * fa + fmaf(b.S, db, b.T) * fb;
  r.S = a.S * fa + b.S * fb;
  return r;
}
__device__ __forceinline__ MST mst_shfl_xor(MST v, int o) {
  MST r;
  r.m = __shfl_xor_sync(0xffffffffu, v.m, o);
  r.S = __shfl_xor_sync(0xffffffffu, v.S, o);
  r.T = __shfl_xor_sync(0xffffffffu, v.T, o);
  return r;
}

constexpr int kEntVec = 8;  // float4 per thread per chunk (held in registers)

// grid: (splits, rows).  One HBM pass: each thread keeps an online (m, S, T)
// over register-resident chunks of its slice, the CTA merges its threads in a
// fixed shuffle tree, and the last CTA of a row merges the row's split
// partials (one per lane, fixed tree) into H = ln S - T/S.  with_state:
// append H to the slot's entropy ring and run the page trigger when the tail
// just sealed.
template <bool kWithState>
__global__ void __launch_bounds__(kNT) entropy_kernel(ChessState st, Workspace ws, EntArgs a) {
  __shared__ MST s_w[kNT / 32];
  __shared__ int s_last;
  const int r = blockIdx.y;
  const int split = blockIdx.x;
  const int nsplit = gridDim.x;
  const int64_t per = ((a.vocab + nsplit - 1) / nsplit + 3) & ~int64_t(3);
  const int64_t lo = min(a.vocab, per * split), hi = min(a.vocab, lo + per);
  const float* row = a.logits + (int64_t)r * a.ld;
  const bool vec = ((a.ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.logits) & 15) == 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  MST t = {-INFINITY, 0.f, 0.f};
  // fold N register values into the thread's running (m, S, T)
  auto absorb = [&](const float (&v)[4 * kEntVec], auto n_const) {
    constexpr int N = decltype(n_const)::value;
    float cm = -INFINITY;
#pragma unroll
    for (int i = 0; i < N; ++i) cm = fmaxf(cm, v[i]);
    if (cm == -INFINITY) return;
    const float mn = fmaxf(t.m, cm);
    if (t.S != 0.f && mn > t.m) {  // rescale the running sums to the new max
      const float d = t.m - mn, f = exp2f(d * 1.4426950408889634f);
      t.T = fmaf(t.S, d, t.T) * f;
      t.S *= f;
    }
    t.m = mn;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const float dx = v[i] - mn;
      const float e = exp2f(dx * 1.4426950408889634f);
      if (e > 0.f) {
        t.S += e;
        t.T = fmaf(e, dx, t.T);
      }
    }
  };
  if (vec) {
    constexpr int kChunk = 4 * kEntVec * kNT;
    for (int64_t c0 = lo; c0 < hi; c0 += kChunk) {
      float v[4 * kEntVec];
#pragma unroll
      for (int q = 0; q < kEntVec; ++q) {
        const int64_t i = c0 + 4 * ((int64_t)q * kNT + threadIdx.x);
        float4 x = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        if (i + 3 < hi) {
          x = __ldcs(reinterpret_cast<const float4*>(row + i));
        } else if (i < hi) {
          x.x = row[i];
          if (i + 1 < hi) x.y = row[i + 1];
          if (i + 2 < hi) x.z = row[i + 2];
        }
        v[4 * q] = x.x;
        v[4 * q + 1] = x.y;
        v[4 * q + 2] = x.z;
        v[4 * q + 3] = x.w;
      }
      absorb(v, std::integral_constant<int, 4 * kEntVec>{});
    }
  } else {
    for (int64_t i = lo + threadIdx.x; i < hi; i += kNT) {
      float v[4 * kEntVec];
      v[0] = row[i];
      absorb(v, std::integral_constant<int, 1>{});
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) t = mst_merge(t, mst_shfl_xor(t, o));
  if (lane == 0) s_w[warp] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    MST c = s_w[0];
    for (int w = 1; w < kNT / 32; ++w) c = mst_merge(c, s_w[w]);
    double* part = ws.ent_part + ((int64_t)r * kEntSplit + split) * 3;
    part[0] = (double)c.m;
    part[1] = (double)c.S;
    part[2] = (double)c.T;
    fence_acq_rel_gpu();
    const int prev = atomicAdd(&ws.ent_done[r], 1);
    s_last = (prev == nsplit - 1);
  }
  __syncthreads();
  if (!s_last || warp != 0) return;
  fence_acq_rel_gpu();
  // warp 0 merges the row's split partials: lane i owns splits i and i + 32
  // (both loaded in one round trip, merged in that order)
  static_assert(kEntSplit <= 64, "entropy merge holds two partials per lane");
  MST c = {-INFINITY, 0.f, 0.f};
  {
    double pv[2][3];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int q = lane + 32 * j;
      const double* part = ws.ent_part + ((int64_t)r * kEntSplit + q) * 3;
#pragma unroll
      for (int e = 0; e < 3; ++e) pv[j][e] = q < nsplit ? __ldcg(part + e) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (lane + 32 * j < nsplit) c = mst_merge(c, MST{(float)pv[j][0], (float)pv[j][1], (float)pv[j][2]});
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) c = mst_merge(c, mst_shfl_xor(c, o));
  if (lane != 0) return;
  ws.ent_done[r] = 0;
  // H = ln S - T/S  (p = e^(x-m)/S, ln p = (x-m) - ln S)
  double H = log((double)c.S) - (double)c.T / (double)c.S;
  if (H < 0.0) H = 0.0;
  if (a.out) a.out[r] = H;
  if constexpr (kWithState) {
    const int B = st.d.page_size;
    const int pos = st.ent_count[r];
    if (pos < B) st.ent_ring[(int64_t)r * B + pos] = H;
    st.ent_count[r] = pos + 1;
    page_trigger(st, a.cfg, r);
  }
}

// CTAs per row: one CTA per SM over all rows for small batches, and slices
// of at most 4 register chunks per thread.  (Two per SM, the round-1 choice,
// measured the same: cfg3 8.7 vs 8.5 us in the step timeline, step 769.3 vs
// 770.6 us; one per SM leaves more room to the kernels running beside it.)
int ent_splits(int64_t rows, int64_t vocab) {
  const int64_t by_gpu = (int64_t)num_sms() / std::max<int64_t>(rows, 1);
  const int64_t by_vocab = (vocab + 4 * 4 * kEntVec * kNT - 1) / (4 * 4 * kEntVec * kNT);
  return (int)std::min<int64_t>(kEntSplit, std::max<int64_t>({(int64_t)4, by_gpu, by_vocab}));
}

// record given entropies + trigger, one thread per slot
__global__ void record_entropy_kernel(ChessState st, const double* H, const uint8_t* active,
                                      ChessTriggerCfg cfg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= st.d.batch || (active && !active[s])) return;
  const int B = st.d.page_size;
  const int pos = st.ent_count[s];
  if (pos < B) st.ent_ring[(int64_t)s * B + pos] = H[s];
  st.ent_count[s] = pos + 1;
  page_trigger(st, cfg, s);
}

// entropy over probability rows (uncertainty.py:22-31), one CTA per row.
__global__ void __launch_bounds__(kNT) entropy_probs_kernel(const double* probs, int64_t n,
                                                            int64_t ld, double* out,
                                                            int32_t* flags) {
  __shared__ double s_w[kNT / 32];
  __shared__ int s_neg;
  const double* p = probs + (int64_t)blockIdx.x * ld;
  if (threadIdx.x == 0) s_neg = 0;
  __syncthreads();
  double h = 0.0;
  int neg = 0;
  for (int64_t i = threadIdx.x; i < n; i += kNT) {
    const double x = p[i];
    if (x < 0.0) neg = 1;
    if (x > 0.0) h = fma(x, log(x), h);
  }
  if (neg) atomicOr(&s_neg, 1);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) h += shfl_xor_d(h, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = h;
  __syncthreads();
  if (threadIdx.x == 0) {
    double hh = s_w[0];
    for (int w = 1; w < kNT / 32; ++w) hh += s_w[w];
    // p.sum() in NumPy's pairwise order (validation threshold is 1e-9)
    const double total = np_pairwise_sum(p, (int)n, 1);
    int f = s_neg ? 1 : 0;
    if (fabs(total - 1.0) > 1e-9) f |= 2;
    flags[blockIdx.x] = f;
    out[blockIdx.x] = -hh;
  }
}

__global__ void page_uncertainty_kernel(const double* e, int n, double* out) {
  if (threadIdx.x != 0) return;
  const double mean = __ddiv_rn(np_pairwise_sum(e, n, 1), (double)n);
  const double var = __ddiv_rn(np_pairwise(
                                   [=](int i) {
                                     const double dlt = __dsub_rn(e[i], mean);
                                     return __dmul_rn(dlt, dlt);
                                   },
                                   n),
                               (double)n);
  out[0] = mean;
  out[1] = var;
}

// calibrate: page statistics, one thread per page (NumPy pairwise order)
__global__ void calib_stats_kernel(const double* e, const int32_t* counts, int n_pages, int64_t ld,
                                   double* means, double* vars) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pages) return;
  const double* row = e + (int64_t)p * ld;
  const int n = counts[p];
  const double mean = __ddiv_rn(np_pairwise_sum(row, n, 1), (double)n);
  const double var = __ddiv_rn(np_pairwise(
                                   [=](int i) {
                                     const double dlt = __dsub_rn(row[i], mean);
                                     return __dmul_rn(dlt, dlt);
                                   },
                                   n),
                               (double)n);
  means[p] = mean;
  vars[p] = var;
}

// nearest rank r (1-based) of x[0..n): the r-th smallest is the minimum of
// the n - r + 1 largest (block radix top-k, K3's block_topk_mark).
// blockIdx.x 0: means -> out[0], 1: variances -> out[1].
__global__ void __launch_bounds__(kNT) calib_rank_kernel(const double* vals, int n, int r,
                                                         uint64_t* keys, int* kept, double* out) {
  __shared__ int s_hist[256];
  __shared__ int s_scr[64];
  __shared__ double s_min[kNT / 32];
  const double* x = vals + (int64_t)blockIdx.x * n;
  uint64_t* k = keys + (int64_t)blockIdx.x * n;
  int* kp = kept + (int64_t)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += kNT) k[i] = score_key(x[i]);
  __syncthreads();
  block_topk_mark<kNT>(k, n, n - r + 1, kp, s_hist, s_scr);
  double m = INFINITY;
  for (int i = threadIdx.x; i < n; i += kNT)
    if (kp[i]) m = fmin(m, x[i]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = s_min[0];
    for (int w = 1; w < kNT / 32; ++w) v = fmin(v, s_min[w]);
    out[blockIdx.x] = v;
  }
}

}  // namespace

size_t calibrate_workspace_bytes(int n) { return (size_t)n * (2 * 8 + 2 * 8 + 2 * 4) + 256; }

int launch_calibrate(const double* e, const int32_t* counts, int n, int64_t ld, int rank, double* out,
                     void* workspace, cudaStream_t stream) {
  uint8_t* w = reinterpret_cast<uint8_t*>(workspace);
  double* vals = reinterpret_cast<double*>(w);                     // [2][n]: means, vars
  uint64_t* keys = reinterpret_cast<uint64_t*>(w + (size_t)n * 16);  // [2][n]
  int* kept = reinterpret_cast<int*>(w + (size_t)n * 32);            // [2][n]
  calib_stats_kernel<<<(n + 127) / 128, 128, 0, stream>>>(e, counts, n, ld, vals, vals + n);
  int rc = check_launch("calibrate_stats");
  if (rc) return rc;
  calib_rank_kernel<<<2, kNT, 0, stream>>>(vals, n, rank, keys, kept, out);
  return check_launch("calibrate_rank");
}

int launch_entropy_trigger(const ChessState& st, const Workspace& ws, const float* logits,
                           int64_t vocab, int64_t ld, const ChessTriggerCfg& cfg, double* out,
                           cudaStream_t stream) {
  EntArgs a{logits, vocab, ld, out, cfg};
  entropy_kernel<true><<<dim3(ent_splits(st.d.batch, vocab), st.d.batch), kNT, 0, stream>>>(st, ws, a);
  return check_launch("entropy_trigger");
}

int launch_record_entropy(const ChessState& st, const double* H, const uint8_t* active,
                          const ChessTriggerCfg& cfg, cudaStream_t stream) {
  record_entropy_kernel<<<(st.d.batch + 127) / 128, 128, 0, stream>>>(st, H, active, cfg);
  return check_launch("record_entropy");
}

int launch_entropy_logits(const Workspace& ws, const float* logits, int64_t rows, int64_t vocab,
                          int64_t ld, double* out, cudaStream_t stream) {
  EntArgs a{logits, vocab, ld, out, ChessTriggerCfg{}};
  ChessState dummy{};
  entropy_kernel<false><<<dim3(ent_splits(rows, vocab), (unsigned)rows), kNT, 0, stream>>>(dummy, ws, a);
  return check_launch("entropy_logits");
}

int launch_entropy_probs(const double* probs, int64_t rows, int64_t n, int64_t ld, double* out,
                         int32_t* flags, cudaStream_t stream) {
  if (rows == 0) return CHESS_OK;
  entropy_probs_kernel<<<(unsigned)rows, kNT, 0, stream>>>(probs, n, ld, out, flags);
  return check_launch("entropy_probs");
}

int launch_page_uncertainty(const double* e, int n, double* out, cudaStream_t stream) {
  page_uncertainty_kernel<<<1, 32, 0, stream>>>(e, n, out);
  return check_launch("page_uncertainty");
}

}  // namespace chess
