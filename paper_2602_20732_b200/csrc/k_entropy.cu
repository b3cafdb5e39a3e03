// k_entropy.cu — K5: per-token entropy from logits, page uncertainty and the
// backtracking trigger.
//
// Reference:
//   entropy            uncertainty.py:22-31   -sum p ln p (nats), 0 ln 0 := 0
//   page_uncertainty   uncertainty.py:41-48   mean + population variance
//   check_trigger      uncertainty.py:86-98   strict joint / any
//   policy cadence     simulate.py:163-170    never/always/fixed(N)/dynamic
// The reference consumes probabilities; the device consumes the step's fp32
// logits and computes H(softmax(logits)) in one HBM pass: per CTA slice
// (max, sum e, sum e*(x-max)) with f64 accumulation, merged in fixed order.
// Page statistics use NumPy's pairwise summation order so decisions are
// bit-identical given identical per-token entropies.
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

__device__ __forceinline__ void merge_msT(double& M, double& S, double& T, double m2, double s2,
                                          double t2) {
  if (s2 == 0.0) return;
  if (S == 0.0) {
    M = m2; S = s2; T = t2;
    return;
  }
  const double Mn = fmax(M, m2);
  const double f1 = exp(M - Mn), f2 = exp(m2 - Mn);
  T = (T + S * (M - Mn)) * f1 + (t2 + s2 * (m2 - Mn)) * f2;
  S = S * f1 + s2 * f2;
  M = Mn;
}

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
      case CHESS_POLICY_NEVER: fire = 0; break;
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
  }
  st.fire[s] = fire;
}

// grid: (kEntSplit, rows).  with_state: append H to the slot's entropy ring and
// run the page trigger when the tail just sealed.
template <bool kWithState>
__global__ void __launch_bounds__(kNT) entropy_kernel(ChessState st, Workspace ws, EntArgs a) {
  __shared__ double s_red[3][kNT / 32];
  __shared__ int s_last;
  const int r = blockIdx.y;
  const int split = blockIdx.x;
  const int nsplit = gridDim.x;
  const int64_t per = ((a.vocab + nsplit - 1) / nsplit + 3) & ~int64_t(3);
  const int64_t lo = min(a.vocab, per * split), hi = min(a.vocab, lo + per);
  const float* row = a.logits + (int64_t)r * a.ld;
  const bool vec = ((a.ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.logits) & 15) == 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  // pass 1: max
  float mx = -INFINITY;
  if (vec) {
    for (int64_t i = lo + 4 * threadIdx.x; i < hi; i += 4 * kNT) {
      if (i + 3 < hi) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(row + i));
        mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
      } else {
        for (int64_t j = i; j < hi; ++j) mx = fmaxf(mx, row[j]);
      }
    }
  } else {
    for (int64_t i = lo + threadIdx.x; i < hi; i += kNT) mx = fmaxf(mx, row[i]);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_red[0][warp] = mx;
  __syncthreads();
  float M = s_red[0][0];
  for (int w = 1; w < kNT / 32; ++w) M = fmaxf(M, s_red[0][w]);
  __syncthreads();

  // pass 2 (slice is L1/L2 resident): sum e^(x-M), sum e^(x-M) (x-M) in f64
  double S = 0.0, T = 0.0;
  const double Md = (double)M;
  auto acc = [&](float x) {
    const double dx = (double)x - Md;
    const double e = (double)expf((float)dx);
    S += e;
    T = fma(e, dx, T);
  };
  if (M > -INFINITY) {
    if (vec) {
      for (int64_t i = lo + 4 * threadIdx.x; i < hi; i += 4 * kNT) {
        if (i + 3 < hi) {
          const float4 v = *reinterpret_cast<const float4*>(row + i);
          acc(v.x); acc(v.y); acc(v.z); acc(v.w);
        } else {
          for (int64_t j = i; j < hi; ++j) acc(row[j]);
        }
      }
    } else {
      for (int64_t i = lo + threadIdx.x; i < hi; i += kNT) acc(row[i]);
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    S += shfl_xor_d(S, o);
    T += shfl_xor_d(T, o);
  }
  if (lane == 0) {
    s_red[1][warp] = S;
    s_red[2][warp] = T;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double Sb = s_red[1][0], Tb = s_red[2][0];
    for (int w = 1; w < kNT / 32; ++w) {
      Sb += s_red[1][w];
      Tb += s_red[2][w];
    }
    double* part = ws.ent_part + ((int64_t)r * kEntSplit + split) * 3;
    part[0] = (double)M;
    part[1] = Sb;
    part[2] = Tb;
    fence_acq_rel_gpu();
    const int prev = atomicAdd(&ws.ent_done[r], 1);
    s_last = (prev == nsplit - 1);
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  fence_acq_rel_gpu();
  ws.ent_done[r] = 0;
  double Mt = 0.0, St = 0.0, Tt = 0.0;
  for (int q = 0; q < nsplit; ++q) {
    const double* part = ws.ent_part + ((int64_t)r * kEntSplit + q) * 3;
    merge_msT(Mt, St, Tt, __ldcg(part), __ldcg(part + 1), __ldcg(part + 2));
  }
  // H = ln S - T/S  (p = e^(x-M)/S, ln p = (x-M) - ln S)
  double H = log(St) - Tt / St;
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

}  // namespace

int launch_entropy_trigger(const ChessState& st, const Workspace& ws, const float* logits,
                           int64_t vocab, int64_t ld, const ChessTriggerCfg& cfg, double* out,
                           cudaStream_t stream) {
  EntArgs a{logits, vocab, ld, out, cfg};
  entropy_kernel<true><<<dim3(kEntSplit, st.d.batch), kNT, 0, stream>>>(st, ws, a);
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
  entropy_kernel<false><<<dim3(kEntSplit, (unsigned)rows), kNT, 0, stream>>>(dummy, ws, a);
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
