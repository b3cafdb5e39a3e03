// k_select_tc.cuh — K2 on tensor cores: certified fp16 scoring (tcgen05 +
// TMA) with exact f64 rescoring of the rows near each level's cut
// (summary_dtype 3).  Included by k_select.cu inside namespace chess::{anon}.
//
// Reference: selection.py:62-111 (score_all = V_all @ anchor, then the masked
// top-k cascade).  The selection this path produces is the one the f64 scores
// give (the f64 scan, summary_dtype 1) — it is NOT an approximation:
//
//  1. mirror16_kernel (k_index.cu) keeps h = fp16(v) of every f64 summary row
//     v plus err = ||v - h||_2 and nrm = ||h||_2 (rounded up).
//  2. anchor_prep_kernel splits the f64 anchor a, per 2048-element slice q,
//     into a power-of-two scale 2^k_q and two fp16 vectors hi, lo with
//     a*2^k_q = hi + lo + rem, written as the MMA's B operand (N = 8 rows:
//     hi, lo, six zero rows; 128B-swizzled atoms), and the slice sums of
//     a^2, (rem 2^-k_q)^2 and ((|hi|+|lo|) 2^-k_q)^2.
//  3. select_tc_kernel streams the candidate rows' fp16 mirrors with 3-D
//     tensor TMA (one box = 8 consecutive rows x 4 K blocks of 64) into a
//     shared-memory ring; one thread issues tcgen05.mma (M = 128 rows =
//     16 row groups, N = 8, K = 16, fp16 x fp16 -> f32 in TMEM) per K step;
//     each stage (256 elements) is its own accumulation window, read back by
//     four epilogue warps with tcgen05.ld and summed in f64:
//        approx = sum_q 2^-k_q sum_w (D[:, 0] + D[:, 1])
//     |true - approx| <= A err + (Rem + gamma Sp) nrm + slack
//     (A = ||a||, Rem = ||rem||, Sp = || |hi|+|lo| ||, by Cauchy-Schwarz;
//     gamma bounds the f32 accumulation of one 16-MMA window, see kGammaTc).
//  4. The level's tail certifies each candidate against the cut: with
//     T = k-th largest lower bound and H = (k+1)-th largest upper bound, a
//     row with hi < T is certainly out, lo > H certainly in; the rest are
//     "uncertain" and are rescored from the f64 rows by select_scan_kernel
//     <double> in rescore mode (the same kernel and slice order as the f64
//     scan, so the same f64 scores), whose tail keeps the best k - #in of
//     them (ties to the lower index) — selection.py:77-88 exactly.
// Bytes: 2 B per element of every candidate row plus 8 B per element of the
// (few) uncertain rows, against 4 B (f32 mirrors) or 8 B (f64) per element.

constexpr int kTcGroups = 16;                          // 8-row groups per M = 128 tile
constexpr int kTcSliceKb = kScanSliceBytes / 8 / 64;   // 32 K blocks = the f64 scan slice
constexpr int kTcStageA = kTcGroups * kTcKbs * 1024;   // 64 KB of rows
constexpr int kTcStageB = kTcKbs * 1024;               // 4 KB of anchor atoms
constexpr int kTcStageBytes = kTcStageA + kTcStageB;
#ifndef CHESS_TC_ACC
#define CHESS_TC_ACC 8
#endif
// as many stages as fit beside the tail's static shared memory (13.7 KB),
// the barriers and the per-slot tables of kMaxBatch slots (<= 16 stages)
constexpr int kTcStagesRaw = 209000 / kTcStageBytes;
constexpr int kTcStages = kTcStagesRaw > 16 ? 16 : kTcStagesRaw;
constexpr int kTcAcc = CHESS_TC_ACC;                   // TMEM accumulation windows in flight
constexpr int kTcTmemCols = kTcAcc * 8 <= 32 ? 32 : (kTcAcc * 8 <= 64 ? 64 : (kTcAcc * 8 <= 128 ? 128 : 256));
static_assert(kTcStages >= 2, "tensor-core scan ring too shallow");
constexpr int kTcCTA = kNT + 64;                       // 8 epilogue/tail warps + TMA warp + MMA warp
constexpr int kTcProducerWarp = kWarps, kTcMmaWarp = kWarps + 1;
constexpr uint32_t kTcIdesc = tc::idesc_f16(128, 8, 0);
// f32 accumulation error of one window (16 MMAs of K = 16, exact fp16
// products): modelled as <= 2 ulp (2^-22) of the running magnitude per MMA
// step, i.e. 18 * 2^-22 * sum|products|, and inflated 4x: 18 * 2^-20.
constexpr double kGammaTc = 18.0 * 0x1p-20;

struct TcTile {
  int s, n, g0, ng, slice;
};

// Debug timeline (trace build only, chess_debug_select_tc_trace): per CTA of
// the last tensor-core launch of each level {entry, items done, exit, tails
// run}, and per slot {tail start, tail end, CTA, items left in that CTA's
// range when it won the slot}.
__device__ unsigned long long g_tc_trace[3][256][4];
__device__ unsigned long long g_tc_tail[3][64][12];
// tail phase stamps [4..9]: norms, rows certified, T, H, classified, emitted
__device__ __forceinline__ void tc_tail_stamp(int lv, int s, int which) {
  if (kTrace && threadIdx.x == 0 && s < 64) g_tc_tail[lv][s][which] = global_ns();
}

// tiles of one slot's level: groups of 8 candidates, spread evenly over
// ceil(groups / 16) tiles
__device__ __forceinline__ int tc_tiles(int n) {
  const int groups = (n + 7) / 8;
  return (groups + kTcGroups - 1) / kTcGroups;
}

// ---------------------------------------------------------------------------
// anchor split + B-operand atoms, grid (n_slices, batch), 256 threads: each
// thread owns one 16-byte chunk (8 elements) of one K block of the slice.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) anchor_prep_kernel(ChessState st, Workspace ws, SelParams prm) {
  const int s = blockIdx.y, q = blockIdx.x;
  if (!fired(st, prm, s) || st.num_sealed[s] == 0) return;
  const ChessDims& d = st.d;
  const int nsl = ws.n_slices;
  const int nkb = (int)(d.ld / 64);
  const int kb = q * kTcSliceKb + (threadIdx.x >> 3);
  const int c = threadIdx.x & 7;
  double v[8];
  const double* a = st.anchor + (int64_t)s * d.ld + (int64_t)kb * 64 + c * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = kb < nkb ? a[i] : 0.0;
  double m = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) m = fmax(m, fabs(v[i]));
  __shared__ double s_red[3][8];
  __shared__ double s_m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_red[0][threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = 0.0;
    for (int w = 0; w < 8; ++w) mm = fmax(mm, s_red[0][w]);
    s_m = mm;
  }
  __syncthreads();
  // 2^k brings the slice's largest |a| into [2^14, 2^15) (fp16 max 65504)
  const double mm = s_m;
  const int k = (mm > 0.0 && isfinite(mm)) ? 14 - ilogb(mm) : 0;
  double sa = 0.0, sr = 0.0, sp = 0.0;
  uint32_t hw[4], lw[4];
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    __half hh[2], ll[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double x = ldexp(v[i + t], k);
      hh[t] = __double2half(x);
      const double r1 = x - (double)__half2float(hh[t]);  // exact
      ll[t] = __double2half(r1);
      const double hv = (double)__half2float(hh[t]), lv = (double)__half2float(ll[t]);
      const double rem = ldexp(r1 - lv, -k);  // exact
      const double spl = ldexp(fabs(hv) + fabs(lv), -k);
      sa = __fma_rn(v[i + t], v[i + t], sa);
      sr = __fma_rn(rem, rem, sr);
      sp = __fma_rn(spl, spl, sp);
    }
    hw[i / 2] = (uint32_t)__half_as_ushort(hh[0]) | ((uint32_t)__half_as_ushort(hh[1]) << 16);
    lw[i / 2] = (uint32_t)__half_as_ushort(ll[0]) | ((uint32_t)__half_as_ushort(ll[1]) << 16);
  }
  if (kb < ws.nkb_pad) {
    // 128B-swizzled atom: row r, 16-byte chunk c at r*128 + ((c ^ r) * 16)
    uint8_t* atom = ws.anc_tile + ((int64_t)s * ws.nkb_pad + kb) * 1024;
    *reinterpret_cast<uint4*>(atom + 0 * 128 + ((c ^ 0) << 4)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(atom + 1 * 128 + ((c ^ 1) << 4)) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
#pragma unroll
    for (int r = 2; r < 8; ++r) *reinterpret_cast<uint4*>(atom + r * 128 + ((c ^ r) << 4)) = make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    sp += __shfl_xor_sync(0xffffffffu, sp, o);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    s_red[0][threadIdx.x >> 5] = sa;
    s_red[1][threadIdx.x >> 5] = sr;
    s_red[2][threadIdx.x >> 5] = sp;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += s_red[threadIdx.x][w];
    ws.anc_stats[((int64_t)s * nsl + q) * 4 + threadIdx.x] = t;
  }
  if (threadIdx.x == 0) ws.anc_exp[(int64_t)s * nsl + q] = k;
}

// ---------------------------------------------------------------------------
// Emit one level from its keep flags (candidate order): next level's
// candidates (children of the kept parents) or, at the page level, the
// semantic set + working set + block table.  Same bookkeeping as
// select_tail_topk (sel_stats, defer_ws).
// ---------------------------------------------------------------------------
__device__ void tc_emit_level(const ChessState& st, const Workspace& ws, const SelParams& prm, int s, int lv,
                              int m, const int* kept, TailSmem& sm) {
  const ChessDims& d = st.d;
  const int64_t mr = max_rows(d);
  const LevelShape sh = shape_of(st, s);
  int* stats = st.sel_stats + 8 * s;
  int* plist = ws.plist + (int64_t)s * mr;
  const int* cand = lv == 0 ? nullptr : ws.cand + ((int64_t)s * 3 + lv) * mr;
  int kcount;
  if (lv < 2) {
    const int fan = lv == 0 ? d.chunks_per_grid : d.pages_per_chunk;
    kcount = block_compact<kNT>(kept, m, plist, sm.scratch, [&](int i) { return cand ? cand[i] : i; });
    block_sync<kNT>();
    const int total_children = lv == 0 ? sh.C : sh.P;
    int* out = ws.cand + ((int64_t)s * 3 + lv + 1) * mr;
    expand_children(plist, kcount, fan, total_children, out, &ws.cand_n[4 * s + lv + 1]);
    if (threadIdx.x == 0) {
      stats[5 + lv] = kcount;
      stats[3 + lv] = (kcount > 0) ? (kcount - 1) * fan + min(fan, total_children - plist[kcount - 1] * fan) : 0;
    }
  } else {
    int32_t* sem = st.semantic + (int64_t)s * d.max_pages;
    kcount = block_compact<kNT>(kept, m, sem, sm.scratch, [&](int i) { return cand[i]; });
    if (threadIdx.x == 0) {
      st.n_semantic[s] = kcount;
      stats[7] = kcount;
      stats[0] = sh.G;
      stats[1] = sh.C;
      stats[2] = sh.P;
    }
  }
  block_sync<kNT>();
  __threadfence_block();
  if (lv == 2) {
    if (prm.defer_ws) {
      if (threadIdx.x == 0) ws.ws_pending[s] = 1;
    } else {
      block_build_ws<kNT>(st, s, sm.scratch);
    }
  }
}

// stash {err, nrm} of candidate row `id` of level `lv` (mirror16_kernel)
__device__ __forceinline__ const double* tc_row_stash(const ChessState& st, int s, int lv, int id) {
  const ChessDims& d = st.d;
  const int64_t rows = lv == 0 ? max_grids(d) : (lv == 1 ? max_chunks(d) : (int64_t)d.max_pages);
  const float* base = lv == 0 ? st.grid_vec32 : (lv == 1 ? st.chunk_vec32 : st.page_vec32);
  const float* row = base + ((int64_t)s * rows + id) * d.ld;
  return reinterpret_cast<const double*>(reinterpret_cast<const uint8_t*>(row) + 2 * d.ld);
}

// Tail of one slot's level after the tensor-core scan: reduce the slice
// partials (fixed order), certify every candidate against the cut, then
// either emit the level (nothing uncertain) or list the uncertain positions
// for the exact rescoring launch.
__device__ void tc_tail(const ChessState& st, const Workspace& ws, const SelParams& prm, int s, int lv, int n,
                        TailSmem& sm, double* s_norm) {
  const ChessDims& d = st.d;
  const int64_t mr = max_rows(d);
  const int nsl = ws.n_slices;
  double* lo_v = ws.scores + (int64_t)s * mr;
  double* part = ws.part + (int64_t)s * mr * nsl;
  const int* cand = lv == 0 ? nullptr : ws.cand + ((int64_t)s * 3 + lv) * mr;
  const bool in_smem = n <= kTailCap;
  uint64_t* keys = in_smem ? sm.keys : ws.keys + (int64_t)s * mr;
  int* kept = in_smem ? sm.kept : ws.kept + (int64_t)s * mr;
  int* cls = ws.cls + (int64_t)s * mr;
  int* meta = ws.unc_meta + 4 * s;
  // slice sums of the anchor statistics in slice order: the slices' loads in
  // parallel (one round trip, staged in sm.keys before it holds keys), the
  // sums by thread 0
  double* s_st = reinterpret_cast<double*>(sm.keys);
  const bool par_norm = 3 * nsl <= kTailCap;
  if (par_norm) {
    for (int q = threadIdx.x; q < nsl; q += kNT) {
      const double* t = ws.anc_stats + ((int64_t)s * nsl + q) * 4;
      s_st[3 * q] = __ldcg(t);
      s_st[3 * q + 1] = __ldcg(t + 1);
      s_st[3 * q + 2] = __ldcg(t + 2);
    }
    block_sync<kNT>();
  }
  if (threadIdx.x == 0) {
    double a2 = 0.0, r2 = 0.0, p2 = 0.0;
    for (int q = 0; q < nsl; ++q) {
      const double* t = par_norm ? s_st + 3 * q : nullptr;
      const double* g = ws.anc_stats + ((int64_t)s * nsl + q) * 4;
      a2 += par_norm ? t[0] : __ldcg(g);
      r2 += par_norm ? t[1] : __ldcg(g + 1);
      p2 += par_norm ? t[2] : __ldcg(g + 2);
    }
    s_norm[0] = sqrt(a2) * (1.0 + 0x1p-20);
    s_norm[1] = sqrt(r2) * (1.0 + 0x1p-20);
    s_norm[2] = sqrt(p2) * (1.0 + 0x1p-20);
  }
  block_sync<kNT>();
  tc_tail_stamp(lv, s, 4);
  const double A = s_norm[0], Rem = s_norm[1], Sp = s_norm[2];
  const int k = (int)ceil(prm.rho[lv] * (double)n);  // selection.py:98, 103, 108
  if (k >= n) {
    for (int i = threadIdx.x; i < n; i += kNT) kept[i] = 1;
    if (threadIdx.x == 0) meta[0] = 0;
    block_sync<kNT>();
    tc_emit_level(st, ws, prm, s, lv, n, kept, sm);
    return;
  }
  // intervals [lo, hi] around the certified approximate score (lo in
  // ws.scores, over the row's err stash; hi in the row's first slice
  // partial, consumed).  Two rows per thread iteration with every load issued
  // before use: the 16 slice partials of each row and the {err, nrm} the
  // scan's slice-0 epilogue gathered (ws.scores / ws.keys at the position).
  // Up to kTailCap candidates the bound keys also go to shared memory as
  // conservative 32-bit keys (lo rounded down, hi rounded up, below).
  uint32_t* k32 = reinterpret_cast<uint32_t*>(sm.keys);  // [0, 1024) lo, [1024, 2048) hi
  const double* nrm_v = reinterpret_cast<const double*>(ws.keys) + (int64_t)s * mr;
  for (int i0 = threadIdx.x; i0 < n; i0 += 2 * kNT) {
    const int i1 = i0 + kNT;
    const bool has1 = i1 < n;
    const int j1 = has1 ? i1 : i0;
    double* pr0 = part + (int64_t)i0 * nsl;
    double* pr1 = part + (int64_t)j1 * nsl;
    const double err0 = __ldcg(lo_v + i0), nrm0 = __ldcg(nrm_v + i0);
    const double err1 = __ldcg(lo_v + j1), nrm1 = __ldcg(nrm_v + j1);
    double acc0 = 0.0, acc1 = 0.0;
    for (int q0 = 0; q0 < nsl; q0 += 16) {
      double v0[16], v1[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        v0[q] = q0 + q < nsl ? __ldcg(pr0 + q0 + q) : 0.0;
        v1[q] = q0 + q < nsl ? __ldcg(pr1 + q0 + q) : 0.0;
      }
      acc0 = q0 ? __dadd_rn(acc0, v0[0]) : v0[0];
      acc1 = q0 ? __dadd_rn(acc1, v1[0]) : v1[0];
#pragma unroll
      for (int q = 1; q < 16; ++q)
        if (q0 + q < nsl) {
          acc0 = __dadd_rn(acc0, v0[q]);
          acc1 = __dadd_rn(acc1, v1[q]);
        }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (r == 1 && !has1) break;
      const double acc = r ? acc1 : acc0, err = r ? err1 : err0, nrm = r ? nrm1 : nrm0;
      const int i = r ? i1 : i0;
      const double e = A * err + (Rem + kGammaTc * Sp) * nrm + 0x1p-38 * (A * (nrm + err) + Sp * nrm);
      double lo = acc - e, hi = acc + e;
      if (!(isfinite(acc) && isfinite(e))) {
        lo = -INFINITY;
        hi = INFINITY;
      }
      lo_v[i] = lo;
      (r ? pr1 : pr0)[0] = hi;
      if (in_smem) {
        k32[i] = float_key(__double2float_rd(lo));
        k32[kTailCap + i] = float_key(__double2float_ru(hi));
      } else {
        keys[i] = score_key(lo);
      }
    }
  }
  block_sync<kNT>();
  tc_tail_stamp(lv, s, 5);
  double Tv, Hv;  // classification thresholds: Tv <= T, Hv >= H
  if (in_smem) {
    // T = k-th largest lower bound, H = (k+1)-th largest upper bound: only
    // their values matter, and any Tv <= T, Hv >= H keeps the classification
    // sound (fewer rows certain, the rest rescored exactly).  Both key arrays
    // are sorted together (bitonic, one barrier per stage) as 32-bit keys of
    // lo rounded down and hi rounded up, so Tv <= T and Hv >= H.
    const int np2 = n <= 2 ? 2 : 1 << (32 - __clz(n - 1));
    for (int i = n + threadIdx.x; i < np2; i += kNT) {
      k32[i] = 0u;
      k32[kTailCap + i] = 0u;
    }
    block_sync<kNT>();
    block_sort2_desc_u32<kNT>(k32, k32 + kTailCap, np2);
    Tv = k > 0 ? (double)float_of_key(k32[k - 1]) : INFINITY;  // k = 0: every row is out
    Hv = (double)float_of_key(k32[kTailCap + k]);
    tc_tail_stamp(lv, s, 6);
    block_sync<kNT>();
  } else {
    // T = k-th largest lower bound
    block_topk_mark<kNT>(keys, n, k, kept, sm.hist, sm.scratch);
    uint64_t tk = ~0ull;
    for (int i = threadIdx.x; i < n; i += kNT)
      if (kept[i]) tk = min(tk, keys[i]);
    for (int o = 16; o > 0; o >>= 1) tk = min(tk, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)tk, o));
    __shared__ unsigned long long s_tk[kWarps];
    if ((threadIdx.x & 31) == 0) s_tk[threadIdx.x >> 5] = tk;
    block_sync<kNT>();
    uint64_t T = ~0ull;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) T = min(T, (uint64_t)s_tk[w]);
    tc_tail_stamp(lv, s, 6);
    block_sync<kNT>();
    // H = (k+1)-th largest upper bound
    for (int i = threadIdx.x; i < n; i += kNT) keys[i] = score_key(part[(int64_t)i * nsl]);
    block_sync<kNT>();
    block_topk_mark<kNT>(keys, n, k + 1, kept, sm.hist, sm.scratch);
    uint64_t hk = ~0ull;
    for (int i = threadIdx.x; i < n; i += kNT)
      if (kept[i]) hk = min(hk, keys[i]);
    for (int o = 16; o > 0; o >>= 1) hk = min(hk, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)hk, o));
    if ((threadIdx.x & 31) == 0) s_tk[threadIdx.x >> 5] = hk;
    block_sync<kNT>();
    uint64_t H = ~0ull;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) H = min(H, (uint64_t)s_tk[w]);
    Tv = T == ~0ull ? INFINITY : double_of_key(T);
    Hv = double_of_key(H);
  }
  tc_tail_stamp(lv, s, 7);
  // classify: 1 certainly in (lo > H), 2 uncertain (hi >= T), 0 out
  int n_in = 0;
  for (int i = threadIdx.x; i < n; i += kNT) {
    const double lo = lo_v[i], hi = __ldcg(part + (int64_t)i * nsl);
    const int c = lo > Hv ? 1 : (hi >= Tv ? 2 : 0);
    cls[i] = c;
    kept[i] = c == 2;
    n_in += c == 1;
  }
  for (int o = 16; o > 0; o >>= 1) n_in += __shfl_xor_sync(0xffffffffu, n_in, o);
  __shared__ int s_nin[kWarps];
  if ((threadIdx.x & 31) == 0) s_nin[threadIdx.x >> 5] = n_in;
  block_sync<kNT>();
  n_in = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) n_in += s_nin[w];
  int* unc = ws.unc + (int64_t)s * mr;
  const int n_unc = block_compact<kNT>(kept, n, unc, sm.scratch, [](int i) { return i; });
  block_sync<kNT>();
  if (threadIdx.x == 0) {
    meta[0] = n_unc;
    meta[1] = k - n_in;
    meta[2] = n;
    meta[3] += n_unc;  // cumulative rows rescored (diagnostics, chess_debug_select_rescored)
  }
  tc_tail_stamp(lv, s, 8);
  if (n_unc == 0) {
    for (int i = threadIdx.x; i < n; i += kNT) kept[i] = cls[i] == 1;
    block_sync<kNT>();
    tc_emit_level(st, ws, prm, s, lv, n, kept, sm);
  }
  tc_tail_stamp(lv, s, 9);
}

// Tail of the rescoring launch: exact f64 scores of the uncertain rows are in
// ws.scores[s][0 .. n_unc); keep the best k - #in of them (ties to the lower
// position = lower id), add the certainly-in rows, emit the level.
__device__ void tc_rescore_finish(const ChessState& st, const Workspace& ws, const SelParams& prm, int s, int lv,
                                  TailSmem& sm) {
  const int64_t mr = max_rows(st.d);
  const int* meta = ws.unc_meta + 4 * s;
  const int n_unc = meta[0], k_rem = meta[1], m = meta[2];
  const double* sc = ws.scores + (int64_t)s * mr;
  const int* unc = ws.unc + (int64_t)s * mr;
  const int* cls = ws.cls + (int64_t)s * mr;
  const bool in_smem = m <= kTailCap;
  uint64_t* keys = in_smem ? sm.keys : ws.keys + (int64_t)s * mr;
  int* kept = in_smem ? sm.kept : ws.kept + (int64_t)s * mr;
  for (int i = threadIdx.x; i < n_unc; i += kNT) keys[i] = score_key(sc[i]);
  block_sync<kNT>();
  block_topk_mark<kNT>(keys, n_unc, k_rem, kept, sm.hist, sm.scratch);
  tail_trace(lv, s, 3);
  // kept[0..n_unc) -> flags in candidate order (uncertain positions ascend)
  for (int i = threadIdx.x; i < n_unc; i += kNT) keys[i] = kept[i];
  block_sync<kNT>();
  for (int i = threadIdx.x; i < m; i += kNT) kept[i] = cls[i] == 1;
  block_sync<kNT>();
  for (int i = threadIdx.x; i < n_unc; i += kNT)
    if (keys[i]) kept[unc[i]] = 1;
  block_sync<kNT>();
  tail_trace(lv, s, 5);
  tc_emit_level(st, ws, prm, s, lv, m, kept, sm);
  tail_trace(lv, s, 6);
}

// ---------------------------------------------------------------------------
// the tensor-core scan (one launch per level 0..2).  Warps 0-7: epilogue
// (warps 0-3 read TMEM lanes 0-127) and per-slot tails; warp 8: TMA
// producer; warp 9: TMEM owner + MMA issuer.  Items are (slot, tile of <= 16
// row groups, 2048-element slice), contiguous per CTA.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTcCTA, 1) select_tc_kernel(ChessState st, Workspace ws, SelParams prm, int level,
                                                              const __grid_constant__ CUtensorMap map_g,
                                                              const __grid_constant__ CUtensorMap map_c,
                                                              const __grid_constant__ CUtensorMap map_p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)kTcStages * kTcStageBytes);
  uint64_t* empty = full + kTcStages;
  uint64_t* tfull = empty + kTcStages;
  uint64_t* tempty = tfull + kTcAcc;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + kTcAcc);
  int* s_prefix = reinterpret_cast<int*>(s_tmem + 4);  // [batch + 1]
  int* s_rows = s_prefix + st.d.batch + 1;           // [batch]
  __shared__ TailSmem sm;
  __shared__ int s_last;
  __shared__ double s_norm[4];
  const ChessDims& d = st.d;
  const int nb = d.batch;
  const int nsl = ws.n_slices;
  const int nkb = (int)(d.ld / 64);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (kTrace && threadIdx.x == 0 && blockIdx.x < 256) {
    g_tc_trace[level][blockIdx.x][0] = global_ns();
    g_tc_trace[level][blockIdx.x][3] = 0;
  }

  if (warp == 0) {
    int run = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int s = b0 + lane;
      int items = 0;
      if (s < nb) {
        const int n = level_rows(st, ws, prm, s, level);
        s_rows[s] = n;
        items = n > 0 ? tc_tiles(n) * nsl : 0;
      }
      int incl = items;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (s < nb) s_prefix[s] = run + incl - items;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_prefix[nb] = run;
  } else if (warp == kTcProducerWarp && lane == 0) {
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kTcAcc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  } else if (warp == kTcMmaWarp) {
    tc::tmem_alloc<kTcTmemCols>(s_tmem);
    tc::fence_before();
  }
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *s_tmem;
  const int total = s_prefix[nb];
  const int it_begin = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int it_end = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  auto slot_of = [&](int it) {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_prefix[mid] <= it) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  auto decode = [&](int it, int s) {
    TcTile p;
    p.s = s;
    p.n = s_rows[s];
    const int groups = (p.n + 7) / 8;
    const int tiles = tc_tiles(p.n);
    const int gpt = (groups + tiles - 1) / tiles;
    const int local = it - s_prefix[s];
    const int t = local / nsl;
    p.slice = local - t * nsl;
    p.g0 = t * gpt;
    p.ng = min(gpt, groups - p.g0);
    return p;
  };
  auto stages_of = [&](int slice) {
    const int kbs = min(kTcSliceKb, nkb - slice * kTcSliceKb);
    return (kbs + kTcKbs - 1) / kTcKbs;
  };

  if (warp == kTcProducerWarp) {
    // ===================== TMA producer =====================
    const CUtensorMap* map = level == 0 ? &map_g : (level == 1 ? &map_c : &map_p);
    const int64_t lvl_rows = level == 0 ? max_grids(d) : (level == 1 ? max_chunks(d) : (int64_t)d.max_pages);
    const int64_t mr = max_rows(d);
    int k = 0;
    for (int it = it_begin; it < it_end; ++it) {
      const int s = slot_of(it);
      const TcTile p = decode(it, s);
      // first row of this lane's group (groups are 8 consecutive ids)
      int row = 0;
      if (lane < p.ng) {
        const int pos0 = 8 * (p.g0 + lane);
        const int id0 = level == 0 ? pos0 : __ldcg(&ws.cand[((int64_t)s * 3 + level) * mr + pos0]);
        row = (int)((int64_t)s * lvl_rows + id0);
      }
      const int nst = stages_of(p.slice);
      const uint32_t bytes = (uint32_t)(p.ng * kTcKbs * 1024 + kTcStageB);
      for (int j = 0; j < nst; ++j, ++k) {
        const int stage = k % kTcStages;
        const uint32_t ph = (uint32_t)((k / kTcStages) & 1);
        if (lane == 0) {
          mbar_wait(&empty[stage], ph ^ 1u);
          mbar_arrive_expect_tx(&full[stage], bytes);
        }
        __syncwarp();
        uint8_t* sb = ring + (size_t)stage * kTcStageBytes;
        const int kb0 = p.slice * kTcSliceKb + j * kTcKbs;
        if (lane < p.ng) tc::tma_load_3d(sb + lane * (kTcKbs * 1024), map, 0, row, kb0, &full[stage]);
        if (lane == 31)
          tma_load_1d(sb + kTcStageA, ws.anc_tile + ((int64_t)s * ws.nkb_pad + kb0) * 1024, kTcStageB, &full[stage]);
      }
    }
  } else if (warp == kTcMmaWarp) {
    // ===================== MMA issuer =====================
    int k = 0, w = 0;
    for (int it = it_begin; it < it_end; ++it) {
      const int nst = stages_of(decode(it, slot_of(it)).slice);
      for (int j = 0; j < nst; ++j, ++k, ++w) {
        const int stage = k % kTcStages;
        const int b = w % kTcAcc;
        mbar_wait(&tempty[b], (uint32_t)(((w / kTcAcc) & 1) ^ 1));
        mbar_wait(&full[stage], (uint32_t)((k / kTcStages) & 1));
        tc::fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(ring + (size_t)stage * kTcStageBytes);
          const uint64_t adesc = tc::sw128_desc(sa, kTcKbs * 1024);
          const uint64_t bdesc = tc::sw128_desc(sa + kTcStageA, 1024);
#pragma unroll
          for (int kb = 0; kb < kTcKbs; ++kb)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t off = (uint64_t)((kb * 1024 + kk * 32) >> 4);
              tc::mma_f16_ss(tmem + (uint32_t)(b * 8), adesc + off, bdesc + off, kTcIdesc, (kb | kk) != 0);
            }
          tc::commit(&empty[stage]);
          tc::commit(&tfull[b]);
        }
        __syncwarp();
      }
    }
  } else {
    // ===================== epilogue + tails (warps 0-7) =====================
    if (level == 0 && blockIdx.x == 0) handle_empty_slots(st, ws, prm, sm);
    const int64_t mr = max_rows(d);
    int s = -1, contributed = 0, w = 0;
    auto flush = [&](int s_done) {
      block_sync<kNT>();
      if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        const int items_s = s_prefix[s_done + 1] - s_prefix[s_done];
        const int prev = atomicAdd(&ws.sel_done[s_done], contributed);
        s_last = (prev + contributed == items_s);
      }
      block_sync<kNT>();
      if (s_last) {
        fence_acq_rel_gpu();
        if (kTrace && threadIdx.x == 0 && s_done < 64) {
          g_tc_tail[level][s_done][0] = global_ns();
          g_tc_tail[level][s_done][2] = blockIdx.x;
          g_tc_tail[level][s_done][3] = (unsigned long long)(it_end - s_prefix[s_done + 1] > 0 ? it_end - s_prefix[s_done + 1] : 0);
        }
        tc_tail(st, ws, prm, s_done, level, s_rows[s_done], sm, s_norm);
        if (kTrace && threadIdx.x == 0 && s_done < 64) {
          g_tc_tail[level][s_done][1] = global_ns();
          if (blockIdx.x < 256) g_tc_trace[level][blockIdx.x][3] += 1;
        }
        if (threadIdx.x == 0) ws.sel_done[s_done] = 0;
        block_sync<kNT>();
      }
    };
    for (int it = it_begin; it < it_end; ++it) {
      if (s < 0 || it >= s_prefix[s + 1]) {
        if (s >= 0) flush(s);
        s = slot_of(it);
        contributed = 0;
      }
      const TcTile p = decode(it, s);
      const int nst = stages_of(p.slice);
      if (warp < 4) {
        // slice-0 items also gather their rows' {err, nrm} stash (mirror16)
        // into compact per-position arrays for the tail (ws.scores and ws.keys
        // of the slot are free during the level's scan): the loads are issued
        // here and land while the MMAs run
        const int r = 32 * warp + lane;  // M row = 8 * group + row in group
        const int pos = 8 * p.g0 + r;
        const bool valid = r < 8 * p.ng && pos < p.n;
        const bool own_stash = valid && p.slice == 0;
        double st_err = 0.0, st_nrm = 0.0;
        if (own_stash) {
          const int id = level == 0 ? pos : __ldcg(&ws.cand[((int64_t)s * 3 + level) * mr + pos]);
          const double* sp = tc_row_stash(st, s, level, id);
          st_err = sp[0];
          st_nrm = sp[1];
        }
        double acc = 0.0;
        for (int j = 0; j < nst; ++j, ++w) {
          const int b = w % kTcAcc;
          mbar_wait(&tfull[b], (uint32_t)((w / kTcAcc) & 1));
          tc::fence_after();
          float c0, c1;
          tc::tmem_ld_x2(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(b * 8), c0, c1);
          tc::fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
          acc = j ? __dadd_rn(acc, __dadd_rn((double)c0, (double)c1)) : __dadd_rn((double)c0, (double)c1);
        }
        if (valid) {
          const int kx = ws.anc_exp[(int64_t)s * nsl + p.slice];
          ws.part[((int64_t)s * mr + pos) * nsl + p.slice] = ldexp(acc, -kx);
        }
        if (own_stash) {
          ws.scores[(int64_t)s * mr + pos] = st_err;
          reinterpret_cast<double*>(ws.keys)[(int64_t)s * mr + pos] = st_nrm;
        }
      }
      ++contributed;
    }
    if (s >= 0) flush(s);
    if (kTrace && threadIdx.x == 0 && blockIdx.x < 256) g_tc_trace[level][blockIdx.x][1] = global_ns();
  }
  __syncthreads();
  if (warp == kTcMmaWarp) {
    tc::fence_after();
    tc::tmem_dealloc<kTcTmemCols>(tmem);
  }
  if (kTrace && threadIdx.x == 0 && blockIdx.x < 256) g_tc_trace[level][blockIdx.x][2] = global_ns();
}
