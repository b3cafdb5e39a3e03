// k_select.cu — K2 anchor scoring + K3 coarse-to-fine masked top-k cascade.
//
// Reference: selection.py:44-140
//   score_all           :62-74   scores = V_all @ anchor (one GEMV)
//   _top_k              :77-88   top ceil(rho*active), ties -> lower index
//   hierarchical_prune  :91-111  grids -> chunks of kept grids -> pages
//   reconstruct_working_set :126-140, gather_pages kv_store.py:156-166
//
// Design: the scan is a batched GEMV that is HBM-bound at
// 0.25-0.5 flop/B, far below the tcgen05 ridge, so it runs on the FP64 pipe:
// f32 (or f64) summary rows x f64 anchor, accumulated in f64.  The
// conditional scan only scores children of kept parents, which is
// output-identical to Alg.1's full scan (a masked top-k can never keep a
// child of a pruned parent); `full_scan` keeps the literal one-GEMV variant.
//
// Work decomposition: an item is (slot, 8 candidate rows, 16 KB row slice).
// Persistent CTAs stride over items; per-(row, slice) partials land in the
// workspace and the last CTA to finish a slot's items (atomic counter) reduces
// them in fixed slice order (deterministic), runs the radix top-k and writes
// the next level's candidate list, or — at the page level — the semantic set,
// working set and block table.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"

namespace chess {

namespace {

constexpr int kNT = kScanThreads;
constexpr int kWarps = kNT / 32;

__device__ __forceinline__ int slot_pages(const ChessState& st, int s) { return st.num_sealed[s]; }

struct LevelShape {
  int P, C, G;
};
__device__ __forceinline__ LevelShape shape_of(const ChessState& st, int s) {
  LevelShape sh;
  sh.P = st.num_sealed[s];
  sh.C = (sh.P + st.d.pages_per_chunk - 1) / st.d.pages_per_chunk;
  sh.G = (sh.C + st.d.chunks_per_grid - 1) / st.d.chunks_per_grid;
  return sh;
}

__device__ __forceinline__ bool fired(const ChessState& st, const SelParams& prm, int s) {
  return prm.force_all || (st.fire != nullptr && st.fire[s] != 0);
}

// number of candidate rows of slot s at this level
__device__ __forceinline__ int level_rows(const ChessState& st, const Workspace& ws,
                                          const SelParams& prm, int s, int level) {
  if (!fired(st, prm, s)) return 0;
  const LevelShape sh = shape_of(st, s);
  if (sh.P == 0) return 0;
  if (prm.rescore) return ws.unc_meta[4 * s];  // uncertain rows of the tensor-core pass
  if (level == 0) return sh.G;
  if (level == 3) return sh.G + sh.C + sh.P;
  return ws.cand_n[4 * s + level];
}

template <typename T>
__device__ __forceinline__ const T* level_row_ptr(const ChessState& st, const Workspace& ws, int s,
                                                  int level, int i, const LevelShape& sh);

template <>
__device__ __forceinline__ const float* level_row_ptr<float>(const ChessState& st,
                                                             const Workspace& ws, int s, int level,
                                                             int i, const LevelShape& sh) {
  const ChessDims& d = st.d;
  const int64_t mr = max_rows(d);
  int which, row;
  if (level == 3) {
    which = i < sh.G ? 0 : (i < sh.G + sh.C ? 1 : 2);
    row = which == 0 ? i : (which == 1 ? i - sh.G : i - sh.G - sh.C);
  } else {
    which = level;
    row = level == 0 ? i : __ldcg(&ws.cand[((int64_t)s * 3 + level) * mr + i]);  // may be this launch's
  }
  if (which == 0) return st.grid_vec32 + ((int64_t)s * max_grids(d) + row) * d.ld;
  if (which == 1) return st.chunk_vec32 + ((int64_t)s * max_chunks(d) + row) * d.ld;
  return st.page_vec32 + ((int64_t)s * d.max_pages + row) * d.ld;
}

template <>
__device__ __forceinline__ const double* level_row_ptr<double>(const ChessState& st,
                                                               const Workspace& ws, int s,
                                                               int level, int i,
                                                               const LevelShape& sh) {
  const ChessDims& d = st.d;
  const int64_t mr = max_rows(d);
  int which, row;
  if (level == 3) {
    which = i < sh.G ? 0 : (i < sh.G + sh.C ? 1 : 2);
    row = which == 0 ? i : (which == 1 ? i - sh.G : i - sh.G - sh.C);
  } else {
    which = level;
    row = level == 0 ? i : __ldcg(&ws.cand[((int64_t)s * 3 + level) * mr + i]);  // may be this launch's
  }
  if (which == 0) return st.grid_vec64 + ((int64_t)s * max_grids(d) + row) * d.ld;
  if (which == 1) return st.chunk_vec64 + ((int64_t)s * max_chunks(d) + row) * d.ld;
  return st.page_vec64 + ((int64_t)s * d.max_pages + row) * d.ld;
}

template <>
__device__ __forceinline__ const __nv_bfloat16* level_row_ptr<__nv_bfloat16>(
    const ChessState& st, const Workspace& ws, int s, int level, int i, const LevelShape& sh) {
  // bf16 mirrors live in the *_vec32 buffers (summary_dtype 2)
  const ChessDims& d = st.d;
  const int64_t mr = max_rows(d);
  int which, row;
  if (level == 3) {
    which = i < sh.G ? 0 : (i < sh.G + sh.C ? 1 : 2);
    row = which == 0 ? i : (which == 1 ? i - sh.G : i - sh.G - sh.C);
  } else {
    which = level;
    row = level == 0 ? i : __ldcg(&ws.cand[((int64_t)s * 3 + level) * mr + i]);
  }
  const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(
      which == 0 ? st.grid_vec32 : (which == 1 ? st.chunk_vec32 : st.page_vec32));
  const int64_t rows = which == 0 ? max_grids(d) : (which == 1 ? max_chunks(d) : (int64_t)d.max_pages);
  return base + ((int64_t)s * rows + row) * d.ld;
}

// ---------------------------------------------------------------------------
// tail: reduce partials, top-k, emit next level (block-wide, one slot)
// ---------------------------------------------------------------------------
constexpr int kTailCap = 1024;  // candidates whose keys / flags stay in shared memory

// Debug: per slot of the last launch of each level, tail timeline
// {flush entered, counter won, scores reduced, level-0 top-k, done}.
__device__ unsigned long long g_tail_trace[4][64][8];
__device__ __forceinline__ void tail_trace(int level, int s, int which) {
  if (kTrace && threadIdx.x == 0 && s < 64) g_tail_trace[level][s][which] = global_ns();
}
struct TailSmem {
  int hist[256];
  int scratch[64];
  uint64_t keys[kTailCap];
  int kept[kTailCap];
};

__device__ void expand_children(const int* parents, int m, int fan, int total_children, int* out,
                                int* out_n) {
  // all parents except possibly the globally last have exactly `fan` children
  int count = 0;
  if (m > 0) {
    const int last = parents[m - 1];
    count = (m - 1) * fan + min(fan, total_children - last * fan);
  }
  for (int idx = threadIdx.x; idx < count; idx += kNT) {
    const int r = idx / fan, c = idx - r * fan;
    out[idx] = parents[r] * fan + c;
  }
  if (threadIdx.x == 0) *out_n = count;
}

__device__ void select_tail_topk(const ChessState& st, const Workspace& ws, const SelParams& prm,
                                 int s, int level, int n, TailSmem& sm);
__device__ void tc_rescore_finish(const ChessState& st, const Workspace& ws, const SelParams& prm, int s, int lv,
                                  TailSmem& sm);

// Tail of one slot's level: fixed-order slice reduction of the partials into
// ws.scores[s] (or, head-shard exchange mode, into prm.xout), then the top-k.
__device__ void select_tail(const ChessState& st, const Workspace& ws, const SelParams& prm, int s,
                            int level, int n, TailSmem& sm) {
  const int64_t mr = max_rows(st.d);
  const int ns = ws.n_slices;
  double* sc = ws.scores + (int64_t)s * mr;
  const double* part = ws.part + (int64_t)s * mr * ns;

  // peer-memory export: receive-slot base of this (gen, rank, slot) in every
  // rank's buffer, loaded once (the stores below could alias the arrays)
  double* xdst[kMaxPeers];
  if (prm.xpeer) {
    const int64_t off0 = (((int64_t)(__ldcg(prm.xgen + s) & 1u) * prm.xworld + prm.xrank) * st.d.batch + s) * prm.xld;
#pragma unroll
    for (int p = 0; p < kMaxPeers; ++p) xdst[p] = p < prm.xworld ? prm.xpeer[p] + off0 : nullptr;
  }
  // fixed-order reduction over slices (deterministic); the slice partials of
  // a row are loaded together (one round trip) when ns <= 16
  for (int i = threadIdx.x; i < n; i += kNT) {
    const double* pr = part + (int64_t)i * ns;
    // 16 slice partials per round trip, added in slice order
    double acc = 0.0;
    for (int q0 = 0; q0 < ns; q0 += 16) {
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = q0 + q < ns ? __ldcg(pr + q0 + q) : 0.0;
      if (q0 == 0) acc = v[0];
      else acc = __dadd_rn(acc, v[0]);
#pragma unroll
      for (int q = 1; q < 16; ++q)
        if (q0 + q < ns) acc = __dadd_rn(acc, v[q]);
    }
    if (prm.xpeer) {
      // peer-memory all-gather fused into the scan: this rank's partial row
      // goes straight into every rank's receive slot (NVLink stores)
#pragma unroll
      for (int p = 0; p < kMaxPeers; ++p)
        if (p < prm.xworld) xdst[p][i] = acc;
    } else if (prm.xout) {
      prm.xout[(int64_t)s * prm.xld + i] = acc;
    } else {
      sc[i] = acc;
    }
  }
  block_sync<kNT>();
  tail_trace(level, s, 2);
  if (prm.xpeer) {
    // every thread's stores precede thread 0's system-scope release store
    // (bar.sync above; release is cumulative), which publishes the row
    if (threadIdx.x == 0) {
      const uint32_t g = __ldcg(prm.xgen + s) + 1u;
      for (int p = 0; p < prm.xworld; ++p) st_release_sys(prm.xflag[p] + s * prm.xworld + prm.xrank, g);
    }
    return;
  }
  if (prm.xout) return;  // head shard: exchange, then select_combine_kernel finishes the level
  if (prm.rescore) {
    tc_rescore_finish(st, ws, prm, s, level, sm);
    return;
  }
  select_tail_topk(st, ws, prm, s, level, n, sm);
}

// Top-k cascade of one tail from the reduced scores ws.scores[s] (candidate
// order of `level`): keys, ceil-in-double k, radix top-k, then next-level
// candidates or — at the page level — semantic set + working set.
__device__ void select_tail_topk(const ChessState& st, const Workspace& ws, const SelParams& prm,
                                 int s, int level, int n, TailSmem& sm) {
  const ChessDims& d = st.d;
  const int64_t mr = max_rows(d);
  double* sc = ws.scores + (int64_t)s * mr;
  // keys / kept flags of every level pass fit in smem unless the full-scan
  // candidate count is large
  const bool in_smem = n <= kTailCap;  // n bounds every level's candidate count
  uint64_t* keys = in_smem ? sm.keys : ws.keys + (int64_t)s * mr;
  int* kept = in_smem ? sm.kept : ws.kept + (int64_t)s * mr;
  int* plist = ws.plist + (int64_t)s * mr;
  const LevelShape sh = shape_of(st, s);
  int* stats = st.sel_stats + 8 * s;

  // level order to run in this tail
  const int lv_begin = level == 3 ? 0 : level;
  const int lv_end = level == 3 ? 3 : level + 1;
  int* cand1 = ws.cand + ((int64_t)s * 3 + 1) * mr;
  int* cand2 = ws.cand + ((int64_t)s * 3 + 2) * mr;
  for (int lv = lv_begin; lv < lv_end; ++lv) {
    // candidate count and ids at this level
    int m;
    const int* cand = nullptr;
    if (lv == 0) {
      m = sh.G;
    } else {
      m = ws.cand_n[4 * s + lv];
      cand = lv == 1 ? cand1 : cand2;
    }
    // keys of the candidates
    for (int i = threadIdx.x; i < m; i += kNT) {
      double v;
      if (level == 3) {
        const int id = cand ? cand[i] : i;
        const int off = lv == 0 ? 0 : (lv == 1 ? sh.G : sh.G + sh.C);
        v = sc[off + id];
      } else {
        v = sc[i];
      }
      keys[i] = score_key(v);
    }
    block_sync<kNT>();
    // ceil in double (selection.py:98, 103, 108)
    const int k = (int)ceil(prm.rho[lv] * (double)m);
    block_topk_mark<kNT>(keys, m, k, kept, sm.hist, sm.scratch);
    if (lv == lv_begin) tail_trace(level, s, 3);
    const int fan = lv == 0 ? d.chunks_per_grid : d.pages_per_chunk;
    int kcount;
    if (lv < 2) {
      kcount = block_compact<kNT>(kept, m, plist, sm.scratch,
                                  [&](int i) { return cand ? cand[i] : i; });
      block_sync<kNT>();
      const int total_children = lv == 0 ? sh.C : sh.P;
      int* out = lv == 0 ? cand1 : cand2;
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
  }
  if (lv_end == 3) {
    if (prm.defer_ws) {  // the block table is being read by a concurrent decode
      if (threadIdx.x == 0) ws.ws_pending[s] = 1;
    } else {
      block_build_ws<kNT>(st, s, sm.scratch);
    }
  }
}

// slots that fired with an empty index: empty semantic set + WS refresh
__device__ void handle_empty_slots(const ChessState& st, const Workspace& ws, const SelParams& prm,
                                   TailSmem& sm) {
  for (int s = 0; s < st.d.batch; ++s) {
    if (!fired(st, prm, s) || st.num_sealed[s] != 0) continue;
    if (threadIdx.x == 0) {
      st.n_semantic[s] = 0;
      ws.cand_n[4 * s + 1] = 0;
      ws.cand_n[4 * s + 2] = 0;
      for (int i = 0; i < 8; ++i) st.sel_stats[8 * s + i] = 0;
    }
    block_sync<kNT>();
    if (prm.defer_ws) {
      if (threadIdx.x == 0) ws.ws_pending[s] = 1;
    } else {
      block_build_ws<kNT>(st, s, sm.scratch);
    }
  }
}

// ---------------------------------------------------------------------------
// the scan kernel (one launch per level; level 3 = Alg.1 full scan)
//
// Warp 8 is a TMA producer: one cp.async.bulk per (candidate row, 16 KB
// slice) into a 192 KB shared-memory ring (12 x 16 KB stages).
// Warps 0-7 consume: each thread owns 8 elements of the slice (conflict-free
// 16-byte LDS), multiplies by its f64 anchor registers, and the 8 row
// partials of an item are transpose-reduced across the warp and then across
// warps in fixed order.  The producer runs ahead across item boundaries and
// through the per-slot tails, so HBM never idles on the epilogues.
// ---------------------------------------------------------------------------
constexpr int kScanCTA = kNT + 32;  // 8 consumer warps + 1 producer warp
// Experiment knobs (co-residency with the decode kernel): TMA ring size and
// the min-blocks launch bound (2 caps registers at 113/thread).
#ifndef CHESS_SCAN_RING_KB
#define CHESS_SCAN_RING_KB 192
#endif
#ifndef CHESS_SCAN_MINB
#define CHESS_SCAN_MINB 1
#endif

// Debug timeline (chess_debug_select_trace): per CTA of the last launch of
// each level, {entry, prologue, first row, items done, exit, wait cycles of
// warp 0, rows consumed}.
__device__ unsigned long long g_sel_trace[4][256][8];
__device__ __forceinline__ void sel_trace(int level, int which, unsigned long long v) {
  if (kTrace && blockIdx.x < 256) g_sel_trace[level][blockIdx.x][which] = v;
}

template <typename T>
struct ScanCfg {
  static constexpr int kSlice = kScanSliceBytes / (int)sizeof(T);   // elements per row slice
  static constexpr int kStageBytes = kScanSliceBytes;
  static constexpr int kStages = (CHESS_SCAN_RING_KB * 1024) / kStageBytes;
  static constexpr int kVec = 16 / (int)sizeof(T);                // elements per 16-B chunk
  static constexpr int kPerThread = kSlice / kNT;                  // elements per thread
  static constexpr int kGroups = kPerThread / kVec;                // chunks per thread
  __device__ static int off(int v) { return (v * kNT + (int)threadIdx.x) * kVec; }
};

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ double to_f(double x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return bf2f(x); }

// acc += a[kVec*v ..] . (16-byte chunk of the row at shared address ad), in f64
template <typename T>
__device__ __forceinline__ void fma_chunk(double& acc, const double* a, int v, uint32_t ad) {
  constexpr int kVec = 16 / (int)sizeof(T);
  if constexpr (sizeof(T) == 4) {
    const float4 f = lds_f4(ad);
    acc = __fma_rn(a[kVec * v + 0], (double)f.x, acc);
    acc = __fma_rn(a[kVec * v + 1], (double)f.y, acc);
    acc = __fma_rn(a[kVec * v + 2], (double)f.z, acc);
    acc = __fma_rn(a[kVec * v + 3], (double)f.w, acc);
  } else if constexpr (sizeof(T) == 8) {
    const double2 f = lds_d2(ad);
    acc = __fma_rn(a[kVec * v + 0], f.x, acc);
    acc = __fma_rn(a[kVec * v + 1], f.y, acc);
  } else {  // bf16 mirrors
    const uint4 w = lds_u4(ad);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = bf2x2f(ws[q]);
      acc = __fma_rn(a[kVec * v + 2 * q], (double)f.x, acc);
      acc = __fma_rn(a[kVec * v + 2 * q + 1], (double)f.y, acc);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kScanCTA, CHESS_SCAN_MINB) select_scan_kernel(ChessState st, Workspace ws,
                                                                  SelParams prm, int level) {
  using SC = ScanCfg<T>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)SC::kStages * SC::kStageBytes);
  uint64_t* empty = full + SC::kStages;
  int* s_prefix = reinterpret_cast<int*>(empty + SC::kStages);  // [batch + 1]
  int* s_rows = s_prefix + st.d.batch + 1;                       // [batch] candidate rows
  __shared__ double s_wpart[2][kScanRows][kWarps];
  __shared__ TailSmem sm;
  __shared__ int s_last;
  const ChessDims& d = st.d;
  const int nb = d.batch;
  const int nsl = ws.n_slices;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    sel_trace(level, 0, global_ns());
    sel_trace(level, 5, 0);
    sel_trace(level, 6, 0);
    sel_trace(level, 7, 0);
  }

  // per-slot item counts -> prefix (warp 0), barrier init (lane 0)
  if (warp == 0) {
    int run = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int s = b0 + lane;
      int items = 0;
      if (s < nb) {
        const int n = level_rows(st, ws, prm, s, level);
        s_rows[s] = n;
        items = ((n + kScanRows - 1) / kScanRows) * nsl;
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
    if (lane == 0) {
      s_prefix[nb] = run;
      for (int i = 0; i < SC::kStages; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], kWarps);
      }
      fence_barrier_init();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) sel_trace(level, 1, global_ns());
  // contiguous item range per CTA; within a slot items are ordered
  // (slice, row block) so a CTA reuses one anchor slice across row blocks.
  const int total = s_prefix[nb];
  const int it_begin = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int it_end = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  auto slot_of = [&](int it) {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_prefix[mid] <= it) lo = mid; else hi = mid;
    }
    return lo;
  };
  struct ItemPos {
    int s, n, r0, rows, slice;
  };
  auto decode = [&](int it, int s) {
    ItemPos p;
    p.s = s;
    p.n = s_rows[s];
    const int nrb = (p.n + kScanRows - 1) / kScanRows;
    const int local = it - s_prefix[s];
    p.slice = local / nrb;
    const int rb = local - p.slice * nrb;
    p.r0 = rb * kScanRows;
    p.rows = min(kScanRows, p.n - p.r0);
    return p;
  };

  if (warp == kWarps) {
    // ===================== TMA producer =====================
    // Ops are (item, row) pairs, 8 per item (rows past the item's count are
    // skipped).  The 32 lanes resolve the source rows of 4 items with one
    // coalesced round of candidate-id loads, prefetched one batch ahead, and
    // lane 0 then issues their bulk copies back to back.
    const int n_ops = (it_end - it_begin) * kScanRows;
    auto fetch = [&](int base, const T*& src, uint32_t& bytes) {
      src = nullptr;
      bytes = 0;
      const int op = base + lane;
      if (op < n_ops) {
        const int it = it_begin + op / kScanRows;
        const int r = op % kScanRows;
        const int s = slot_of(it);
        const ItemPos p = decode(it, s);
        if (r < p.rows) {
          const LevelShape sh = shape_of(st, s);
          const int64_t ebase = (int64_t)p.slice * SC::kSlice;
          bytes = (uint32_t)(min((int64_t)SC::kSlice, d.ld - ebase) * sizeof(T));
          // rescore mode: the row is the level candidate at an uncertain position
          const int ci = prm.rescore ? __ldcg(&ws.unc[(int64_t)s * max_rows(d) + p.r0 + r]) : p.r0 + r;
          src = level_row_ptr<T>(st, ws, s, level, ci, sh) + ebase;
        }
      }
    };
    const T* cur_src;
    uint32_t cur_bytes;
    const T* nxt_src = nullptr;
    uint32_t nxt_bytes = 0;
    long long t_fetch = 0, t_issue = 0, t_wait = 0;
    long long tq = clock64();
    fetch(0, cur_src, cur_bytes);
    int k = 0;
    for (int base = 0; base < n_ops; base += 32) {
      if (base + 32 < n_ops) fetch(base + 32, nxt_src, nxt_bytes);
      const long long tq1 = clock64();
      t_fetch += tq1 - tq;
      tq = tq1;
      // 4 items per batch; the lanes of an item issue their rows in parallel
      const uint32_t valid = __ballot_sync(0xffffffffu, cur_bytes != 0);
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        const uint32_t grp = (valid >> (8 * q)) & 0xffu;
        if (grp == 0) continue;
        const int r = lane - 8 * q;
        if (r >= 0 && r < 8 && ((grp >> r) & 1u)) {
          const int kr = k + r;
          const int stage = kr % SC::kStages;
          const uint32_t ph = (uint32_t)((kr / SC::kStages) & 1);
          const long long tw = clock64();
          mbar_wait(&empty[stage], ph ^ 1u);
          if (r == 0) t_wait += clock64() - tw;
          if (prm.mode == 2) {
            mbar_arrive(&full[stage]);
          } else {
            mbar_arrive_expect_tx(&full[stage], cur_bytes);
            tma_load_1d(ring + (size_t)stage * SC::kStageBytes, cur_src, cur_bytes, &full[stage]);
          }
        }
        k += __popc(grp);
        __syncwarp();
      }
      const long long tq2 = clock64();
      t_issue += tq2 - tq;
      tq = tq2;
      cur_src = nxt_src;
      cur_bytes = nxt_bytes;
    }
    t_wait = __shfl_sync(0xffffffffu, t_wait, 0);
    if (lane == 0) {
      sel_trace(level, 5, t_fetch);
      sel_trace(level, 6, t_issue);
      sel_trace(level, 7, t_wait);
    }
    return;
  }

  // ===================== consumers =====================
  if ((level == 0 || level == 3) && blockIdx.x == 0 && !prm.rescore) handle_empty_slots(st, ws, prm, sm);
  int k = 0, buf = 0;
  int s = -1, contributed = 0, a_slice = -1;
  double a[SC::kPerThread];
  bool in[SC::kGroups];
  bool all_in = true;
  auto flush = [&](int s_done) {
    // one release per (CTA, slot) run: publishes this CTA's partials
    const unsigned long long tf = global_ns();
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
      if (kTrace && threadIdx.x == 0 && s_done < 64) g_tail_trace[level][s_done][0] = tf;
      tail_trace(level, s_done, 1);
      select_tail(st, ws, prm, s_done, level, s_rows[s_done], sm);
      tail_trace(level, s_done, 4);
      if (threadIdx.x == 0) ws.sel_done[s_done] = 0;
      block_sync<kNT>();
    }
  };
  for (int it = it_begin; it < it_end; ++it) {
    if (s < 0 || it >= s_prefix[s + 1]) {
      if (s >= 0) flush(s);
      s = slot_of(it);
      contributed = 0;
      a_slice = -1;
    }
    const ItemPos p = decode(it, s);
    const int64_t ebase = (int64_t)p.slice * SC::kSlice;
    if (p.slice != a_slice) {  // anchor slice (f64) in registers; zero beyond ld
      a_slice = p.slice;
      const double* anc = st.anchor + (int64_t)s * d.ld + ebase;
#pragma unroll
      all_in = ebase + SC::kSlice <= d.ld;
      for (int v = 0; v < SC::kGroups; ++v) {
        const int o = SC::off(v);
        in[v] = ebase + o < d.ld;
#pragma unroll
        for (int e = 0; e < SC::kVec; e += 2) {
          double2 x = make_double2(0.0, 0.0);
          if (in[v]) x = *reinterpret_cast<const double2*>(anc + o + e);
          a[v * SC::kVec + e] = x.x;
          a[v * SC::kVec + e + 1] = x.y;
        }
      }
    }
    // all rows of the item first, then 8 independent dot-product chains
    double acc[kScanRows];
#pragma unroll
    for (int r = 0; r < kScanRows; ++r) {
      acc[r] = 0.0;
      if (r < p.rows) {
        const int kr = k + r;
        mbar_wait(&full[kr % SC::kStages], (uint32_t)((kr / SC::kStages) & 1));
        if (kr == 0 && threadIdx.x == 0) sel_trace(level, 2, global_ns());
      }
    }
    if (prm.mode != 1) {
      // shared-window addresses of the item's rows (explicit ld.shared)
      uint32_t rowa[kScanRows];
#pragma unroll
      for (int r = 0; r < kScanRows; ++r)
        rowa[r] = smem_u32(ring) + (uint32_t)(((k + r) % SC::kStages) * SC::kStageBytes);
      if (p.rows == kScanRows && all_in) {
        // fast path: full item, full slice — no predication
#pragma unroll
        for (int v = 0; v < SC::kGroups; ++v) {
#pragma unroll
          for (int r = 0; r < kScanRows; ++r) {
            fma_chunk<T>(acc[r], a, v, rowa[r] + (uint32_t)(SC::off(v) * sizeof(T)));
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v < SC::kGroups; ++v) {
          if (in[v]) {
#pragma unroll
            for (int r = 0; r < kScanRows; ++r) {
              if (r < p.rows) {
                fma_chunk<T>(acc[r], a, v, rowa[r] + (uint32_t)(SC::off(v) * sizeof(T)));
              }
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < kScanRows; ++r)
        if (r < p.rows) mbar_arrive(&empty[(k + r) % SC::kStages]);
    }
    k += p.rows;
    // warp transpose-reduce of 8 row partials: 4+2+1 exchanges, then 2 xor adds.
    {
      const bool b4 = lane & 16;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double send = b4 ? acc[i] : acc[4 + i];
        const double keep = b4 ? acc[4 + i] : acc[i];
        acc[i] = keep + shfl_xor_d(send, 16);
      }
      const bool b3 = lane & 8;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double send = b3 ? acc[i] : acc[2 + i];
        const double keep = b3 ? acc[2 + i] : acc[i];
        acc[i] = keep + shfl_xor_d(send, 8);
      }
      const bool b2 = lane & 4;
      {
        const double send = b2 ? acc[0] : acc[1];
        const double keep = b2 ? acc[1] : acc[0];
        acc[0] = keep + shfl_xor_d(send, 4);
      }
      acc[0] += shfl_xor_d(acc[0], 2);
      acc[0] += shfl_xor_d(acc[0], 1);
      const int row = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      if ((lane & 3) == 0) s_wpart[buf][row][warp] = acc[0];
    }
    block_sync<kNT>();  // double-buffered s_wpart: one barrier per item
    if ((int)threadIdx.x < p.rows) {
      double x = s_wpart[buf][threadIdx.x][0];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) x = __dadd_rn(x, s_wpart[buf][threadIdx.x][w]);
      ws.part[((int64_t)s * max_rows(d) + p.r0 + threadIdx.x) * nsl + p.slice] = x;
    }
    buf ^= 1;
    ++contributed;
  }
  if (threadIdx.x == 0) sel_trace(level, 3, global_ns());
  if (s >= 0) flush(s);
  if (threadIdx.x == 0) sel_trace(level, 4, global_ns());
}

// ---------------------------------------------------------------------------
// Dataflow cascade (conditional scan, one launch for all three levels).
//
// Items are (level, slot, slice, row block) in level-major, slot-minor order;
// each (level, slot) gets an UPPER BOUND of row blocks known at launch
// (level 1 <= k_g*N_g children, level 2 <= ceil(rho_c*that)*N_c), so the item
// space is static while the actual candidate counts are produced by the
// tails.  CTAs grab items from a global counter; an item of level l >= 1 of
// slot s waits (producer side) until slot s's level l-1 tail has published
// its candidates (flow_lvl[s] >= l, release/acquire at gpu scope).  Rows past
// the actual count make an item empty; every item, empty or not, counts
// towards its (level, slot) completion and the CTA that completes it runs the
// tail (same select_tail as the per-level kernel).  Level l+1 of early slots
// therefore streams while later slots are still finishing level l, and there
// is one launch/prologue instead of three.  Measured slower than the
// per-level kernel so far (see launch_select); opt-in with CHESS_SELECT_FLOW=1.
//
// Completions are counted per (CTA, level, slot) run and flushed when the
// next descriptor belongs to another (level, slot), at the end, or when the
// producer is about to block on a dependency (a FLUSH descriptor) — so a
// CTA never sits on the last contribution a tail it waits for needs.
// Deadlock freedom: items are grabbed in level order and a tail depends only
// on items of its own level, which never wait on later levels.
// ---------------------------------------------------------------------------
constexpr int kSmallRowBytes = 16384;  // rows up to this size use select_small_kernel
constexpr int kSmallCand = 1024;       // select_small_kernel: candidates per level kept in shared memory
constexpr int kSmallStageBytes = 128 * 1024;  // select_small_kernel: candidate rows staged per batch
constexpr int kDescRing = 8;
constexpr int kFlowMaxBatch = 256;  // per-slot scheduler tables live in shared memory
constexpr int kDescEnd = -1, kDescFlush = -2;
struct FlowDesc {
  int s, level, r0, rows, slice;  // rows: >= 0 item rows, kDescEnd, kDescFlush
};

__device__ __forceinline__ int flow_row_bound(const ChessState& st, const SelParams& prm, int s,
                                              int level) {
  if (!fired(st, prm, s)) return 0;
  const LevelShape sh = shape_of(st, s);
  if (sh.P == 0) return 0;
  if (level == 0) return sh.G;
  // ceil in double, as the tail's k (selection.py:98, 103)
  const int kg = (int)ceil(prm.rho[0] * (double)sh.G);
  const int r1 = min(sh.C, kg * st.d.chunks_per_grid);
  if (level == 1) return r1;
  const int kc = (int)ceil(prm.rho[1] * (double)r1);
  return min(sh.P, kc * st.d.pages_per_chunk);
}

template <typename T>
__global__ void __launch_bounds__(kScanCTA, 1) select_flow_kernel(ChessState st, Workspace ws,
                                                                  SelParams prm) {
  using SC = ScanCfg<T>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)SC::kStages * SC::kStageBytes);
  uint64_t* empty = full + SC::kStages;
  uint64_t* dfull = empty + SC::kStages;
  uint64_t* dempty = dfull + kDescRing;
  FlowDesc* desc = reinterpret_cast<FlowDesc*>(dempty + kDescRing);
  int* s_pre = reinterpret_cast<int*>(desc + kDescRing);  // [3 * batch + 1]
  int* s_ready = s_pre + 3 * st.d.batch + 1;               // [batch] levels seen published (producer)
  int* s_nrb = s_ready + st.d.batch;                       // [3][batch] row blocks (upper bound)
  int* s_n = s_nrb + 3 * st.d.batch;                       // [3][batch] actual rows (once published)
  __shared__ double s_wpart[2][kScanRows][kWarps];
  __shared__ TailSmem sm;
  __shared__ int s_last;
  const ChessDims& d = st.d;
  const int nb = d.batch;
  const int nsl = ws.n_slices;
  const int64_t mr = max_rows(d);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* next = ws.flow;
  int* done = ws.flow + 1;           // [3][batch]
  int* lvl = ws.flow + 1 + 3 * nb;   // [batch]

  // item prefix over (level, slot): upper-bound row blocks x slices
  if (warp == 0) {
    int run = 0;
    for (int l = 0; l < 3; ++l) {
      for (int b0 = 0; b0 < nb; b0 += 32) {
        const int s = b0 + lane;
        const int nrb = s < nb ? (flow_row_bound(st, prm, s, l) + kScanRows - 1) / kScanRows : 0;
        const int items = nrb * nsl;
        if (s < nb) {
          s_nrb[l * nb + s] = nrb;
          if (l == 0) s_n[s] = shape_of(st, s).G;
        }
        int incl = items;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (s < nb) s_pre[l * nb + s] = run + incl - items;
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    for (int s = lane; s < nb; s += 32) s_ready[s] = 0;
    if (lane == 0) {
      s_pre[3 * nb] = run;
      for (int i = 0; i < SC::kStages; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], kWarps);
      }
      for (int i = 0; i < kDescRing; ++i) {
        mbar_init(&dfull[i], 1);
        mbar_init(&dempty[i], kWarps);
      }
      fence_barrier_init();
    }
  }
  __syncthreads();
  const int total = s_pre[3 * nb];
  auto items_of = [&](int idx) { return s_pre[idx + 1] - s_pre[idx]; };

  if (warp == kWarps) {
    // ===================== producer: grab, resolve, issue =====================
    int k = 0, di = 0;
    auto post = [&](const FlowDesc& x) {
      const int slot = di % kDescRing;
      if (lane == 0) {
        mbar_wait(&dempty[slot], (uint32_t)(((di / kDescRing) & 1) ^ 1));
        desc[slot] = x;
        mbar_arrive(&dfull[slot]);
      }
      __syncwarp();
      ++di;
    };
    // Items are grabbed kGrab at a time: consecutive items of a (level, slot)
    // share a slice (slice-major order), so the consumers' anchor slice stays
    // in registers across a grab and the counter is hit once per kGrab items.
    // Within a grab, groups of 4 items resolve their 32 row pointers in one
    // round of loads (lane 8q + r: item q, row r) before any TMA is issued.
    // The grab size follows the level the counter was last seen in (guided
    // self-scheduling): a quarter of an even share, so a short level (the
    // grids) still spreads over every CTA.
    int grab_of[3];
#pragma unroll
    for (int l = 0; l < 3; ++l)
      grab_of[l] = max(1, min(16, (s_pre[(l + 1) * nb] - s_pre[l * nb]) / (4 * (int)gridDim.x)));
    int seen_level = 0;
    bool finished = false;
    while (!finished) {
      const int kGrab = grab_of[seen_level];
      int it0 = 0;
      if (lane == 0) it0 = atomicAdd(next, kGrab);
      it0 = __shfl_sync(0xffffffffu, it0, 0);
      seen_level = it0 >= s_pre[2 * nb] ? 2 : (it0 >= s_pre[nb] ? 1 : 0);
      for (int g0 = 0; g0 < kGrab && !finished; g0 += 4) {
        int q_s[4], q_level[4], q_r0[4], q_rows[4], q_slice[4];
        int nq = 0;
        for (int q = 0; q < 4 && g0 + q < kGrab; ++q) {
          const int it = it0 + g0 + q;
          if (it >= total) {
            finished = true;
            break;
          }
          int lo = 0, hi = 3 * nb;  // last idx with s_pre[idx] <= it
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_pre[mid] <= it) lo = mid; else hi = mid;
          }
          const int level = lo / nb, s = lo - level * nb;
          if (level > 0 && s_ready[s] < level) {
            int ready = 0;
            if (lane == 0) ready = ld_acquire_gpu(&lvl[s]) >= level;
            ready = __shfl_sync(0xffffffffu, ready, 0);
            __syncwarp();  // order the lanes' candidate reads after lane 0's acquire
            if (!ready) {
              post(FlowDesc{0, 0, 0, kDescFlush, 0});  // consumers publish pending completions first
              if (lane == 0) {
                const uint64_t t0 = global_ns();
                uint32_t polls = 0;
                while (ld_acquire_gpu(&lvl[s]) < level) {
                  if ((++polls & 1023u) == 0 && global_ns() - t0 > 4000000000ull) {
                    printf("chess: select dataflow wait timed out (block %d slot %d level %d)\n", blockIdx.x, s, level);
                    asm volatile("trap;");
                  }
                }
              }
              __syncwarp();
            }
            if (lane == 0) {
              s_ready[s] = level;
              s_n[level * nb + s] = __ldcg(&ws.cand_n[4 * s + level]);
            }
            __syncwarp();
          }
          const int n = s_n[level * nb + s];
          const int nrb = s_nrb[lo];
          const int local = it - s_pre[lo];
          q_s[q] = s;
          q_level[q] = level;
          q_slice[q] = local / nrb;
          q_r0[q] = (local - q_slice[q] * nrb) * kScanRows;
          q_rows[q] = max(0, min(kScanRows, n - q_r0[q]));
          ++nq;
        }
        // one round of row-pointer loads for the group
        const int mq = lane >> 3, mr_ = lane & 7;
        const T* src = nullptr;
        uint32_t bytes = 0;
        if (mq < nq) {
          int qs = 0, ql = 0, qr0 = 0, qrows = 0, qsl = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q == mq) {
              qs = q_s[q]; ql = q_level[q]; qr0 = q_r0[q]; qrows = q_rows[q]; qsl = q_slice[q];
            }
          if (mr_ < qrows) {
            const int64_t ebase = (int64_t)qsl * SC::kSlice;
            bytes = (uint32_t)(min((int64_t)SC::kSlice, d.ld - ebase) * sizeof(T));
            const LevelShape none = {0, 0, 0};  // only the full scan's level 3 needs the shape
            src = level_row_ptr<T>(st, ws, qs, ql, qr0 + mr_, none) + ebase;
          }
        }
        for (int q = 0; q < nq; ++q) {
          post(FlowDesc{q_s[q], q_level[q], q_r0[q], q_rows[q], q_slice[q]});
          if (mq == q && src) {
            const int kr = k + mr_;
            const int stage = kr % SC::kStages;
            mbar_wait(&empty[stage], (uint32_t)(((kr / SC::kStages) & 1) ^ 1));
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_1d(ring + (size_t)stage * SC::kStageBytes, src, bytes, &full[stage]);
          }
          k += q_rows[q];
          __syncwarp();
        }
      }
    }
    post(FlowDesc{0, 0, 0, kDescEnd, 0});
    return;
  }

  // ===================== consumers =====================
  if (blockIdx.x == 0) handle_empty_slots(st, ws, prm, sm);
  int k = 0, di = 0, buf = 0;
  int a_s = -1, a_slice = -1;
  int run_idx = -1, run_cnt = 0;  // pending completions of (level, slot) index run_idx
  double a[SC::kPerThread];
  bool in[SC::kGroups];
  bool all_in = true;
  auto flush = [&]() {
    if (run_idx < 0) return;
    block_sync<kNT>();
    if (threadIdx.x == 0) {
      fence_acq_rel_gpu();
      const int prev = atomicAdd(&done[run_idx], run_cnt);
      s_last = (prev + run_cnt == items_of(run_idx));
    }
    block_sync<kNT>();
    if (s_last) {
      fence_acq_rel_gpu();
      const int level = run_idx / nb, s = run_idx - level * nb;
      const int n = level == 0 ? shape_of(st, s).G : __ldcg(&ws.cand_n[4 * s + level]);
      if (n > 0) select_tail(st, ws, prm, s, level, n, sm);
      if (threadIdx.x == 0 && level < 2) {
        fence_acq_rel_gpu();
        st_release_gpu(&lvl[s], level + 1);
      }
      block_sync<kNT>();
    }
    run_idx = -1;
    run_cnt = 0;
  };
  for (;;) {
    const int slot = di % kDescRing;
    mbar_wait(&dfull[slot], (uint32_t)((di / kDescRing) & 1));
    const FlowDesc x = desc[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&dempty[slot]);
    ++di;
    if (x.rows < 0) {
      flush();
      if (x.rows == kDescEnd) break;
      continue;
    }
    const int idx = x.level * nb + x.s;
    if (idx != run_idx) {
      flush();
      run_idx = idx;
    }
    ++run_cnt;
    if (x.rows == 0) continue;
    const int64_t ebase = (int64_t)x.slice * SC::kSlice;
    if (x.s != a_s || x.slice != a_slice) {  // anchor slice (f64) in registers; zero beyond ld
      a_s = x.s;
      a_slice = x.slice;
      const double* anc = st.anchor + (int64_t)x.s * d.ld + ebase;
      all_in = ebase + SC::kSlice <= d.ld;
#pragma unroll
      for (int v = 0; v < SC::kGroups; ++v) {
        const int o = SC::off(v);
        in[v] = ebase + o < d.ld;
#pragma unroll
        for (int e = 0; e < SC::kVec; e += 2) {
          double2 y = make_double2(0.0, 0.0);
          if (in[v]) y = *reinterpret_cast<const double2*>(anc + o + e);
          a[v * SC::kVec + e] = y.x;
          a[v * SC::kVec + e + 1] = y.y;
        }
      }
    }
    double acc[kScanRows];
#pragma unroll
    for (int r = 0; r < kScanRows; ++r) {
      acc[r] = 0.0;
      if (r < x.rows) {
        const int kr = k + r;
        mbar_wait(&full[kr % SC::kStages], (uint32_t)((kr / SC::kStages) & 1));
      }
    }
    {
      uint32_t rowa[kScanRows];
#pragma unroll
      for (int r = 0; r < kScanRows; ++r)
        rowa[r] = smem_u32(ring) + (uint32_t)(((k + r) % SC::kStages) * SC::kStageBytes);
#pragma unroll
      for (int v = 0; v < SC::kGroups; ++v) {
        if (all_in || in[v]) {
#pragma unroll
          for (int r = 0; r < kScanRows; ++r) {
            if (r < x.rows) {
              fma_chunk<T>(acc[r], a, v, rowa[r] + (uint32_t)(SC::off(v) * sizeof(T)));
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < kScanRows; ++r)
        if (r < x.rows) mbar_arrive(&empty[(k + r) % SC::kStages]);
    }
    k += x.rows;
    {  // warp transpose-reduce of 8 row partials (as in select_scan_kernel)
      const bool b4 = lane & 16;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double send = b4 ? acc[i] : acc[4 + i];
        const double keep = b4 ? acc[4 + i] : acc[i];
        acc[i] = keep + shfl_xor_d(send, 16);
      }
      const bool b3 = lane & 8;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double send = b3 ? acc[i] : acc[2 + i];
        const double keep = b3 ? acc[2 + i] : acc[i];
        acc[i] = keep + shfl_xor_d(send, 8);
      }
      const bool b2 = lane & 4;
      {
        const double send = b2 ? acc[0] : acc[1];
        const double keep = b2 ? acc[1] : acc[0];
        acc[0] = keep + shfl_xor_d(send, 4);
      }
      acc[0] += shfl_xor_d(acc[0], 2);
      acc[0] += shfl_xor_d(acc[0], 1);
      const int row = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      if ((lane & 3) == 0) s_wpart[buf][row][warp] = acc[0];
    }
    block_sync<kNT>();
    if ((int)threadIdx.x < x.rows) {
      double y = s_wpart[buf][threadIdx.x][0];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) y = __dadd_rn(y, s_wpart[buf][threadIdx.x][w]);
      ws.part[((int64_t)x.s * mr + x.r0 + threadIdx.x) * nsl + x.slice] = y;
    }
    buf ^= 1;
  }
}

// ---------------------------------------------------------------------------
// Small-index cascade: one CTA per slot runs all three levels (no inter-CTA
// hand-offs).  For short summary rows (<= 16 KB: the reference's CPU-demo
// shape, D = 1024) the per-level launches, cross-CTA partial reductions and
// tails of the streaming kernel cost far more than the bytes; here each warp
// scores whole rows (lanes stride the row, fixed shuffle tree in f64) and the
// same select_tail_topk runs between levels.
// ---------------------------------------------------------------------------
// Debug timeline (trace build, chess_debug_select_small_trace): per slot of
// the last select_small_kernel launch {entry, anchor staged, then per level
// {rows landed, scored, top-k, emitted}, exit}.
__device__ unsigned long long g_small_trace[16][16];
__device__ __forceinline__ void small_trace(int s, int which) {
  if (kTrace && threadIdx.x == 0 && s < 16) g_small_trace[s][which] = global_ns();
}

template <typename T>
__global__ void __launch_bounds__(kNT) select_small_kernel(ChessState st, Workspace ws, SelParams prm) {
  __shared__ TailSmem sm;
  const int s = blockIdx.x;
  small_trace(s, 0);
  if (!fired(st, prm, s)) return;
  const ChessDims& d = st.d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const LevelShape sh = shape_of(st, s);
  if (sh.P == 0) {  // as handle_empty_slots, for this slot
    if (threadIdx.x == 0) {
      st.n_semantic[s] = 0;
      ws.cand_n[4 * s + 1] = 0;
      ws.cand_n[4 * s + 2] = 0;
      for (int i = 0; i < 8; ++i) st.sel_stats[8 * s + i] = 0;
    }
    block_sync<kNT>();
    if (prm.defer_ws) {
      if (threadIdx.x == 0) ws.ws_pending[s] = 1;
    } else {
      block_build_ws<kNT>(st, s, sm.scratch);
    }
    return;
  }
  // the anchor once into shared memory (rows here are <= 16 KB: <= 4096
  // elements of f32 / 2048 of f64; dynamic shared memory, d.dim doubles)
  extern __shared__ double s_anc[];
  const double* anc_g = st.anchor + (int64_t)s * d.ld;
  for (int j = threadIdx.x; j < d.dim; j += kNT) s_anc[j] = anc_g[j];
  block_sync<kNT>();
  small_trace(s, 1);
  const int64_t mr = max_rows(d);
  double* sc = ws.scores + (int64_t)s * mr;
  // dot product of one summary row with the anchor by one warp: the plain
  // j = lane, lane + 32, ... FMA chain (exact f64 parity, signed zeros
  // included), with the row loads of 16 steps issued before their FMAs (one
  // memory latency per 512 elements instead of one per 32)
  auto dot = [&](const T* row) {
    double acc = 0.0;
    for (int j0 = lane; j0 < d.dim; j0 += 32 * 16) {
      using V = decltype(to_f(row[0]));  // f32 (f32 / bf16 mirrors) or f64 rows
      V r[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int j = j0 + 32 * k;
        r[k] = j < d.dim ? to_f(row[j]) : V(0);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int j = j0 + 32 * k;
        if (j < d.dim) acc = __fma_rn(s_anc[j], (double)r[k], acc);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += shfl_xor_d(acc, o);
    return acc;
  };
  if (sh.G > kTailCap || sh.C > kSmallCand || sh.P > kSmallCand) {
    // large index: the shared tail (candidates and scores in global memory)
    for (int level = 0; level < 3; ++level) {
      const int n = level == 0 ? sh.G : ws.cand_n[4 * s + level];
      for (int i = warp; i < n; i += kNT / 32) {
        const double acc = dot(level_row_ptr<T>(st, ws, s, level, i, sh));
        if (lane == 0) sc[i] = acc;
      }
      block_sync<kNT>();
      select_tail_topk(st, ws, prm, s, level, n, sm);
      block_sync<kNT>();
    }
    return;
  }
  // Every level's candidates, keys and kept parents stay in shared memory:
  // the global round trips of the shared tail (scores written and read back,
  // candidate counts, candidate ids behind each row pointer) were most of a
  // cfg1 pass.  Global candidate lists / counts / scores are still written
  // (write-only) for the debug readers.
  __shared__ int s_cand[kSmallCand];
  __shared__ int s_plist[kSmallCand];
  __shared__ int s_cnt;
  // a level's candidate rows are staged into shared memory (after the
  // anchor) in batches of bulk copies: one memory latency per batch instead
  // of one per row and warp (cfg1: every level is one batch)
  __shared__ uint64_t s_rbar;
  uint8_t* s_rows = reinterpret_cast<uint8_t*>(s_anc + ((d.dim + 15) & ~15));
  const uint32_t row_bytes = (uint32_t)(((int64_t)d.dim * sizeof(T) + 15) & ~15);
  const int batch_rows = (int)(kSmallStageBytes / row_bytes);
  if (threadIdx.x == 0) {
    mbar_init(&s_rbar, 1);
    fence_barrier_init();
  }
  block_sync<kNT>();
  uint32_t rphase = 0;
  int* stats = st.sel_stats + 8 * s;
  int m = sh.G;
  for (int lv = 0; lv < 3; ++lv) {
    // rows of this level (level_row_ptr's layout: f64 rows in *_vec64, f32 /
    // bf16 mirrors in the *_vec32 buffers)
    const void* b64 = lv == 0 ? (const void*)st.grid_vec64 : (lv == 1 ? (const void*)st.chunk_vec64 : (const void*)st.page_vec64);
    const void* b32 = lv == 0 ? (const void*)st.grid_vec32 : (lv == 1 ? (const void*)st.chunk_vec32 : (const void*)st.page_vec32);
    const int64_t lrows = lv == 0 ? max_grids(d) : (lv == 1 ? max_chunks(d) : (int64_t)d.max_pages);
    const T* base = reinterpret_cast<const T*>(sizeof(T) == 8 ? b64 : b32) + (int64_t)s * lrows * d.ld;
    for (int b0 = 0; b0 < m; b0 += batch_rows) {
      const int nr = min(batch_rows, m - b0);
      if (warp == 0) {
        // warp 0 issues the batch's bulk copies, one row per lane per round
        if (lane == 0) mbar_arrive_expect_tx(&s_rbar, (uint32_t)nr * row_bytes);
        __syncwarp();
        for (int r = lane; r < nr; r += 32) {
          const int id = lv == 0 ? b0 + r : s_cand[b0 + r];
          tma_load_1d(s_rows + (size_t)r * row_bytes, base + (int64_t)id * d.ld, row_bytes, &s_rbar);
        }
      }
      mbar_wait(&s_rbar, rphase);
      rphase ^= 1u;
      if (b0 == 0) small_trace(s, 2 + 4 * lv);
      // batches of more than two rows per warp: four rows per warp at once,
      // four independent FMA chains, each in the same per-row order as dot()
      // (so the same scores), interleaved to hide the f64 FMA latency a
      // one-row chain exposes.  Measured on the cfg1 shape (tools/select_micro.py
      // trace build): 32 rows 2.94 -> 2.14 us, but 4 and 16 rows slower than
      // one chain per row (0.67 -> 1.66, 1.50 -> 2.02 us), so those keep dot().
      if (nr <= 2 * (kNT / 32)) {
        for (int r = warp; r < nr; r += kNT / 32) {
          const double acc = dot(reinterpret_cast<const T*>(s_rows + (size_t)r * row_bytes));
          if (lane == 0) {
            sm.keys[b0 + r] = score_key(acc);
            sc[b0 + r] = acc;
          }
        }
      } else
      for (int r0 = warp; r0 < nr; r0 += 4 * (kNT / 32)) {
        constexpr int kR = 4;
        double acc[kR];
        const T* rp[kR];
#pragma unroll
        for (int q = 0; q < kR; ++q) {
          const int r = min(r0 + q * (kNT / 32), nr - 1);
          rp[q] = reinterpret_cast<const T*>(s_rows + (size_t)r * row_bytes);
          acc[q] = 0.0;
        }
        for (int j0 = lane; j0 < d.dim; j0 += 32 * 8) {
          using V = decltype(to_f(rp[0][0]));
          V v[kR][8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int j = j0 + 32 * k;
#pragma unroll
            for (int q = 0; q < kR; ++q) v[q][k] = j < d.dim ? to_f(rp[q][j]) : V(0);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int j = j0 + 32 * k;
            if (j < d.dim) {
              const double a = s_anc[j];
#pragma unroll
              for (int q = 0; q < kR; ++q) acc[q] = __fma_rn(a, (double)v[q][k], acc[q]);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kR; ++q) {
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) acc[q] += shfl_xor_d(acc[q], o);
        }
        if (lane == 0) {
#pragma unroll
          for (int q = 0; q < kR; ++q) {
            const int r = r0 + q * (kNT / 32);
            if (r < nr) {
              sm.keys[b0 + r] = score_key(acc[q]);
              sc[b0 + r] = acc[q];
            }
          }
        }
      }
      block_sync<kNT>();  // the staging buffer is refilled by the next batch
    }
    small_trace(s, 3 + 4 * lv);
    const int k = (int)ceil(prm.rho[lv] * (double)m);  // selection.py:98, 103, 108
    block_topk_mark<kNT>(sm.keys, m, k, sm.kept, sm.hist, sm.scratch);
    small_trace(s, 4 + 4 * lv);
    if (lv < 2) {
      const int kcount = block_compact<kNT>(sm.kept, m, s_plist, sm.scratch,
                                            [&](int i) { return lv == 0 ? i : s_cand[i]; });
      block_sync<kNT>();
      const int fan = lv == 0 ? d.chunks_per_grid : d.pages_per_chunk;
      const int total_children = lv == 0 ? sh.C : sh.P;
      expand_children(s_plist, kcount, fan, total_children, s_cand, &s_cnt);
      block_sync<kNT>();
      m = s_cnt;
      int* gc = ws.cand + ((int64_t)s * 3 + lv + 1) * mr;
      for (int i = threadIdx.x; i < m; i += kNT) gc[i] = s_cand[i];
      if (threadIdx.x == 0) {
        ws.cand_n[4 * s + lv + 1] = m;
        stats[5 + lv] = kcount;
        stats[3 + lv] = m;
      }
    } else {
      int32_t* sem = st.semantic + (int64_t)s * d.max_pages;
      const int kcount = block_compact<kNT>(sm.kept, m, sem, sm.scratch, [&](int i) { return s_cand[i]; });
      if (threadIdx.x == 0) {
        st.n_semantic[s] = kcount;
        stats[7] = kcount;
        stats[0] = sh.G;
        stats[1] = sh.C;
        stats[2] = sh.P;
      }
    }
    block_sync<kNT>();
    small_trace(s, 5 + 4 * lv);
  }
  __threadfence_block();
  if (prm.defer_ws) {  // the block table is being read by a concurrent decode
    if (threadIdx.x == 0) ws.ws_pending[s] = 1;
  } else {
    block_build_ws<kNT>(st, s, sm.scratch);
  }
  small_trace(s, 14);
}

// ---------------------------------------------------------------------------
// KV-head shard: finish one level from every rank's exported
// partial scores.  gathered = [world][batch][xld] (rank-major, the layout of
// an all-gather of each rank's xout); the partials are added in rank order so
// every rank holds bit-identical scores and takes the identical top-k.  One
// CTA per slot; slots that did not fire (or have no candidates) exit.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kNT) select_combine_kernel(ChessState st, Workspace ws,
                                                             SelParams prm, int level,
                                                             const double* gathered, int world) {
  __shared__ TailSmem sm;
  const int s = blockIdx.x;
  const int n = level_rows(st, ws, prm, s, level);
  if (n == 0) return;
  const int64_t mr = max_rows(st.d);
  const int64_t rstride = (int64_t)st.d.batch * prm.xld;
  const double* g = gathered + (int64_t)s * prm.xld;
  double* sc = ws.scores + (int64_t)s * mr;
  for (int i = threadIdx.x; i < n; i += kNT) {
    double acc = __ldcg(g + i);
    for (int r = 1; r < world; ++r) acc = __dadd_rn(acc, __ldcg(g + r * rstride + i));
    sc[i] = acc;
  }
  block_sync<kNT>();
  select_tail_topk(st, ws, prm, s, level, n, sm);
}

// Receive side of the peer-memory transport (chess_select_pull): wait for
// every rank's flag of this slot to reach gen + 1 (acquire, system scope),
// add the rows of receive buffer (gen & 1) in rank order, advance gen, top-k.
// Two buffers suffice: a rank writes generation g + 2 into the buffer of g
// only after its pull of g + 1, which needs this rank's push of g + 1, which
// stream order places after this pull of g.  A wait longer than 10 s sets
// *err (the host raises) instead of hanging the device.
__global__ void __launch_bounds__(kNT) select_pull_kernel(ChessState st, Workspace ws, SelParams prm,
                                                          int level, const double* recv,
                                                          const uint32_t* flags, uint32_t* gen,
                                                          int32_t* err) {
  __shared__ TailSmem sm;
  const int s = blockIdx.x;
  const int n = level_rows(st, ws, prm, s, level);
  if (n == 0) return;
  const int world = prm.xworld;
  const uint32_t g = gen[s];
  if (threadIdx.x < world) {
    const uint32_t* f = flags + s * world + threadIdx.x;
    const uint64_t t0 = global_ns();
    uint32_t polls = 0;
    // wrap-safe "flag >= g + 1"
    while ((int32_t)(ld_acquire_sys(f) - (g + 1u)) < 0) {
      if ((++polls & 255u) == 0 && global_ns() - t0 > 10000000000ull) {
        atomicExch(err, 1);
        break;
      }
    }
  }
  block_sync<kNT>();
  const int64_t mr = max_rows(st.d);
  const int64_t rstride = (int64_t)st.d.batch * prm.xld;
  const double* b = recv + ((int64_t)(g & 1u) * world * st.d.batch + s) * prm.xld;
  double* sc = ws.scores + (int64_t)s * mr;
  for (int i = threadIdx.x; i < n; i += kNT) {
    double acc = __ldcg(b + i);
    for (int r = 1; r < world; ++r) acc = __dadd_rn(acc, __ldcg(b + r * rstride + i));
    sc[i] = acc;
  }
  block_sync<kNT>();
  if (threadIdx.x == 0) gen[s] = g + 1u;
  select_tail_topk(st, ws, prm, s, level, n, sm);
}

// ---------------------------------------------------------------------------
// generic function-level kernels
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ double as_d(const T* p, int64_t i) { return (double)p[i]; }
template <>
__device__ __forceinline__ double as_d<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return (double)bf2f(p[i]);
}

// score_all: one CTA per row, fixed-order f64 block reduction.
template <typename T>
__global__ void __launch_bounds__(256) score_rows_kernel(const T* rows, int64_t dim, int64_t ld,
                                                         const double* anchor, double* scores) {
  __shared__ double s_w[8];
  const int64_t r = blockIdx.x;
  const T* row = rows + r * ld;
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < dim; j += 256) acc = __fma_rn(anchor[j], as_d(row, j), acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += shfl_xor_d(acc, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = s_w[0];
    for (int w = 1; w < 8; ++w) x = __dadd_rn(x, s_w[w]);
    scores[r] = x;
  }
}

// hierarchical_prune with arbitrary maps (selection.py:91-111); one CTA.
__global__ void __launch_bounds__(kNT) prune_kernel(const double* s_g, int G, const double* s_c,
                                                    int C, const double* s_p, int P,
                                                    const int64_t* p2c, const int64_t* c2g,
                                                    double rg, double rc, double rp,
                                                    int32_t* out_pages, int32_t* out_count,
                                                    uint8_t* wsb) {
  __shared__ TailSmem sm;
  const int N = G + C + P;
  uint64_t* keys = reinterpret_cast<uint64_t*>(wsb);
  int* kept = reinterpret_cast<int*>(wsb + 8 * (size_t)N);
  int* cand = kept + N;
  int* mask = cand + N;  // [G + C] masks of kept grids, kept chunks
  if (P == 0) {
    if (threadIdx.x == 0) out_count[0] = out_count[1] = out_count[2] = 0;
    return;
  }
  for (int lv = 0; lv < 3; ++lv) {
    const int n_lv = lv == 0 ? G : (lv == 1 ? C : P);
    const double* sc = lv == 0 ? s_g : (lv == 1 ? s_c : s_p);
    // active candidates ascending
    auto active = [&](int i) -> int {
      if (lv == 0) return 1;
      if (lv == 1) return mask[c2g[i]];
      return mask[G + p2c[i]];
    };
    int m = 0;
    for (int base = 0; base < n_lv; base += kNT) {
      const int i = base + threadIdx.x;
      const int f = (i < n_lv) ? active(i) : 0;
      int tot;
      const int pos = block_exclusive_scan<kNT>(f, sm.scratch, &tot);
      if (f) cand[m + pos] = i;
      m += tot;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += kNT) keys[i] = score_key(sc[cand[i]]);
    __syncthreads();
    const double rho = lv == 0 ? rg : (lv == 1 ? rc : rp);
    const int k = (int)ceil(rho * (double)m);
    block_topk_mark<kNT>(keys, m, k, kept, sm.hist, sm.scratch);
    if (lv < 2) {
      int* mk = mask + (lv == 0 ? 0 : G);
      for (int i = threadIdx.x; i < n_lv; i += kNT) mk[i] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < m; i += kNT)
        if (kept[i]) mk[cand[i]] = 1;
    } else {
      const int cnt = block_compact<kNT>(kept, m, out_pages, sm.scratch, [&](int i) { return cand[i]; });
      if (threadIdx.x == 0) out_count[0] = cnt;
    }
    __syncthreads();
  }
  // kept grid / chunk counts
  int ng = 0, nc = 0;
  for (int i = threadIdx.x; i < G; i += kNT) ng += mask[i];
  for (int i = threadIdx.x; i < C; i += kNT) nc += mask[G + i];
  int tot;
  block_exclusive_scan<kNT>(ng, sm.scratch, &tot);
  if (threadIdx.x == 0) out_count[1] = tot;
  block_exclusive_scan<kNT>(nc, sm.scratch, &tot);
  if (threadIdx.x == 0) out_count[2] = tot;
}

// masked top-k (selection.py:77-88 / oracle_flat_topk :114-123); one CTA.
__device__ long long g_topk_trace[8];  // debug (trace build): phase cycles of the last topk_kernel
__global__ void __launch_bounds__(kNT) topk_kernel(const double* scores, int n, int k,
                                                   const uint8_t* active, int32_t* out_idx,
                                                   int32_t* out_count, int sorted, uint8_t* wsb) {
  __shared__ TailSmem sm;
  uint64_t* keys = reinterpret_cast<uint64_t*>(wsb);
  int* kept = reinterpret_cast<int*>(wsb + 8 * (size_t)n);
  int* const cand = kept + n;
  int m = 0;
  for (int base = 0; base < n; base += kNT) {
    const int i = base + threadIdx.x;
    const int f = (i < n) ? (active ? (active[i] != 0) : 1) : 0;
    int tot;
    const int pos = block_exclusive_scan<kNT>(f, sm.scratch, &tot);
    if (f) cand[m + pos] = i;
    m += tot;
  }
  __syncthreads();
  const long long tk0 = clock64();
  if (m <= kTailCap) {  // keys and flags in shared memory, as in the scan tail
    keys = sm.keys;
    kept = sm.kept;
  }
  for (int i = threadIdx.x; i < m; i += kNT) keys[i] = score_key(scores[cand[i]]);
  __syncthreads();
  const long long tk1 = clock64();
  block_topk_mark<kNT>(keys, m, k, kept, sm.hist, sm.scratch);
  const long long tk2 = clock64();
  if (kTrace) {
    // calibration: 64 named-barrier syncs, 64 bar.red.popc
    const long long tb0 = clock64();
    for (int i = 0; i < 64; ++i) block_sync<kNT>();
    const long long tb1 = clock64();
    int acc = 0;
    for (int i = 0; i < 64; ++i) {
      int c;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\tbar.red.popc.u32 %0, 1, %1, p;\n\t}"
                   : "=r"(c) : "n"(kNT), "r"((int)((threadIdx.x + i) & 1)) : "memory");
      acc += c;
    }
    const long long tb2 = clock64();
    if (threadIdx.x == 0) {
      g_topk_trace[0] = tk1 - tk0;
      g_topk_trace[1] = tk2 - tk1;
      g_topk_trace[2] = tb1 - tb0;
      g_topk_trace[3] = tb2 - tb1 + (acc == -1);
    }
  }
  const int cnt = min(max(k, 0), m);
  if (sorted) {
    block_compact<kNT>(kept, m, out_idx, sm.scratch, [&](int i) { return cand[i]; });
  } else {
    // descending score order, ties by index: rank among kept entries
    for (int i = threadIdx.x; i < m; i += kNT) {
      if (!kept[i]) continue;
      int rank = 0;
      for (int j = 0; j < m; ++j)
        if (kept[j] && (keys[j] > keys[i] || (keys[j] == keys[i] && j < i))) ++rank;
      out_idx[rank] = cand[i];
    }
  }
  if (threadIdx.x == 0) out_count[0] = cnt;
}

// reconstruct_working_set for arbitrary (unsorted, duplicated) selections.
__global__ void __launch_bounds__(kNT) working_set_kernel(const int32_t* selected, int n_sel,
                                                          int n_pages, int window, int sinks,
                                                          const int32_t* page_table,
                                                          int32_t* out_pages, int8_t* out_prov,
                                                          int32_t* out_phys, int32_t* out_len) {
  extern __shared__ int8_t s_tag[];
  __shared__ int s_scr[48];
  for (int i = threadIdx.x; i < n_pages; i += kNT) s_tag[i] = CHESS_PROV_NONE;
  __syncthreads();
  for (int i = threadIdx.x; i < n_sel; i += kNT) {
    const int p = selected[i];
    if (p >= 0 && p < n_pages) s_tag[p] = CHESS_PROV_SEMANTIC;
  }
  __syncthreads();
  for (int i = max(0, n_pages - window) + (int)threadIdx.x; i < n_pages; i += kNT)
    s_tag[i] = CHESS_PROV_WINDOW;
  __syncthreads();
  for (int i = threadIdx.x; i < min(sinks, n_pages); i += kNT) s_tag[i] = CHESS_PROV_SINK;
  __syncthreads();
  int count = 0;
  for (int base = 0; base < n_pages; base += kNT) {
    const int i = base + threadIdx.x;
    const int f = (i < n_pages && s_tag[i] != CHESS_PROV_NONE) ? 1 : 0;
    int tot;
    const int pos = block_exclusive_scan<kNT>(f, s_scr, &tot);
    if (f) {
      out_pages[count + pos] = i;
      out_prov[count + pos] = s_tag[i];
      if (out_phys) out_phys[count + pos] = page_table ? page_table[i] : i;
    }
    count += tot;
  }
  if (threadIdx.x == 0) *out_len = count;
}

__global__ void gather_pages_kernel(const int32_t* table, int n_pages, const int64_t* idx, int n,
                                    int32_t* out, int32_t* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p = idx[i];
  if (p < 0 || p >= n_pages) {
    atomicMin(err, i + 1);
    out[i] = -1;
  } else {
    out[i] = table[p];
  }
}

#include "k_select_tc.cuh"

}  // namespace

// ---------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------
template <typename T>
static int launch_scan(const ChessState& st, const Workspace& ws, const SelParams& prm, int level,
                       cudaStream_t stream, int grid_default = 0) {
  using SC = ScanCfg<T>;
  const size_t smem = 128 + (size_t)SC::kStages * SC::kStageBytes + 2 * SC::kStages * 8 +
                      (size_t)(2 * st.d.batch + 1) * sizeof(int);
  static bool configured = false;
  if (!configured) {
    const size_t smem_max = 128 + (size_t)SC::kStages * SC::kStageBytes + 2 * SC::kStages * 8 +
                            (size_t)(2 * kMaxBatch + 1) * sizeof(int);
    cudaFuncSetAttribute(select_scan_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    configured = true;
  }
  static const int grid_override = getenv("CHESS_SELECT_GRID") ? atoi(getenv("CHESS_SELECT_GRID")) : 0;  // debug
  // Next to a concurrent decode at small batch (its cluster grid is a
  // quarter of the SMs or less: cfg2) the scan does best on 64 CTAs: cfg2
  // step 115-117 us at 24..64 against 122 at 148 (profiles/r02/select_grid_sweep.txt).
  const bool small_batch_overlap = prm.defer_ws && st.d.batch * st.d.kv_heads * 4 <= num_sms();
  const int grid = grid_override > 0 ? grid_override
                   : grid_default > 0 ? grid_default
                   : small_batch_overlap ? std::max(1, num_sms() * 64 / 148) : num_sms();
  select_scan_kernel<T><<<grid, kScanCTA, smem, stream>>>(st, ws, prm, level);
  return check_launch("select_scan");
}

template <typename T>
static size_t flow_smem(int batch) {
  using SC = ScanCfg<T>;
  return 128 + (size_t)SC::kStages * SC::kStageBytes + 2 * SC::kStages * 8 + 2 * kDescRing * 8 +
         kDescRing * sizeof(FlowDesc) + (size_t)(10 * batch + 1) * sizeof(int);
}

template <typename T>
static int launch_flow(const ChessState& st, const Workspace& ws, const SelParams& prm,
                       cudaStream_t stream) {
  const size_t smem = flow_smem<T>(st.d.batch);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(select_flow_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)flow_smem<T>(kFlowMaxBatch));
    configured = true;
  }
  // scheduler counters start at zero every call (a memset node under capture)
  cudaMemsetAsync(ws.flow, 0, (size_t)(1 + 4 * st.d.batch) * sizeof(int32_t), stream);
  select_flow_kernel<T><<<num_sms(), kScanCTA, smem, stream>>>(st, ws, prm);
  return check_launch("select_flow");
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D view of one level's fp16 mirror rows (summary_dtype 3): (64 elements,
// rows, K blocks) with strides (f32 row pitch 4*ld B, 128 B); a box
// (64, 8, kTcKbs) is 8 consecutive rows x 4 K blocks, landing as
// [K block][8 rows][128 B] with 128B swizzle = four MMA atoms of one group.
static int make_mirror_map(CUtensorMap* m, const float* base, int64_t rows, const ChessDims& d) {
  auto fn = encode_fn();
  if (!fn) return fail(CHESS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(d.ld / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)d.ld * 4, 128};
  cuuint32_t box[3] = {64, 8, (cuuint32_t)kTcKbs};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<float*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHESS_ERR_CUDA, "cuTensorMapEncodeTiled (mirror) failed (%d)", (int)r);
  return CHESS_OK;
}

static size_t tc_smem(int batch) {
  return 1024 + (size_t)kTcStages * kTcStageBytes + (size_t)(2 * kTcStages + 2 * kTcAcc) * 8 + 16 +
         (size_t)(2 * batch + 1) * sizeof(int);
}

// summary_dtype 3: anchor split, then per level the tensor-core scan and the
// exact f64 rescoring of its uncertain rows (k_select_tc.cuh)
static int launch_select_tc(const ChessState& st, const Workspace& ws, const SelParams& prm, cudaStream_t stream) {
  const ChessDims& d = st.d;
  anchor_prep_kernel<<<dim3((unsigned)ws.n_slices, (unsigned)d.batch), 256, 0, stream>>>(st, ws, prm);
  int rc = check_launch("anchor_prep");
  if (rc) return rc;
  CUtensorMap mg, mc, mp;
  if ((rc = make_mirror_map(&mg, st.grid_vec32, (int64_t)d.batch * max_grids(d), d))) return rc;
  if ((rc = make_mirror_map(&mc, st.chunk_vec32, (int64_t)d.batch * max_chunks(d), d))) return rc;
  if ((rc = make_mirror_map(&mp, st.page_vec32, (int64_t)d.batch * d.max_pages, d))) return rc;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(select_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem(kMaxBatch));
    if ((rc = check_launch("select_tc smem attribute"))) return rc;
    configured = true;
  }
  SelParams pr = prm;
  pr.rescore = 1;
  // Next to a concurrent decode (defer_ws: the engine's overlapped step) the
  // scan and rescoring launches run on 96 of 148 CTAs: measured on the cfg3 step (two runs each,
  // profiles/r02/select_grid_sweep.txt) 775.6 us at 96 against 791.1 at 148,
  // 779-782 at 80-88 / 104-112 and 797 at 64-72; the pass alone is faster
  // on every SM (328 vs 373 us), which is what a standalone selection gets.
  static const int grid_override = getenv("CHESS_SELECT_GRID") ? atoi(getenv("CHESS_SELECT_GRID")) : 0;  // A/B
  // With more segments than SMs the decode runs two CTAs per SM (stream-K)
  // and the scan does best on 72 (cfg4: 2034 us at 72, 2058 at 64, 2083 at 96,
  // 2097 at 148, 2148 at 48).
  const int segs = d.batch * d.kv_heads;
  const int share = segs > num_sms() ? 72 : 96;
  const int grid = grid_override > 0 ? grid_override : (prm.defer_ws ? std::max(1, num_sms() * share / 148) : num_sms());
  for (int level = 0; level < 3; ++level) {
    select_tc_kernel<<<grid, kTcCTA, tc_smem(d.batch), stream>>>(st, ws, prm, level, mg, mc, mp);
    if ((rc = check_launch("select_tc"))) return rc;
    if ((rc = launch_scan<double>(st, ws, pr, level, stream, grid))) return rc;
  }
  return CHESS_OK;
}

// Debug / test entry: anchor split + the tensor-core scan of ONE level,
// without the exact rescoring, so a test can read the certified intervals
// (chess_debug_tc_read) before the next launch consumes them.
int launch_select_tc_level(const ChessState& st, const Workspace& ws, const SelParams& prm, int level,
                           cudaStream_t stream) {
  const ChessDims& d = st.d;
  anchor_prep_kernel<<<dim3((unsigned)ws.n_slices, (unsigned)d.batch), 256, 0, stream>>>(st, ws, prm);
  int rc = check_launch("anchor_prep");
  if (rc) return rc;
  CUtensorMap mg, mc, mp;
  if ((rc = make_mirror_map(&mg, st.grid_vec32, (int64_t)d.batch * max_grids(d), d))) return rc;
  if ((rc = make_mirror_map(&mc, st.chunk_vec32, (int64_t)d.batch * max_chunks(d), d))) return rc;
  if ((rc = make_mirror_map(&mp, st.page_vec32, (int64_t)d.batch * d.max_pages, d))) return rc;
  cudaFuncSetAttribute(select_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem(kMaxBatch));
  select_tc_kernel<<<num_sms(), kTcCTA, tc_smem(d.batch), stream>>>(st, ws, prm, level, mg, mc, mp);
  return check_launch("select_tc");
}

// persistent scan: one CTA per SM (192 KB TMA ring each), one launch per level
int launch_select(const ChessState& st, const Workspace& ws, const SelParams& prm, int /*grid*/,
                  cudaStream_t stream) {
  // Dataflow cascade (one launch), opt-in: CHESS_SELECT_FLOW=1.  Parity-green
  // (tests/test_gpu_select.py, test_gpu_pagesel.py, test_gpu_headshard.py) but
  // measured slower than three per-level launches (tools/select_micro.py:
  // cfg3 378 vs 308 us, cfg2 45 vs 38 us) — kept for further work.
  static const int flow_env = getenv("CHESS_SELECT_FLOW") ? atoi(getenv("CHESS_SELECT_FLOW")) : 0;
  // tensor-core scan (summary_dtype 3) for the conditional cascade over long
  // rows; full scans, head-shard exchanges and short rows use the exact f64 path
  const bool tc_path = st.d.summary_dtype == kSummaryTc && !prm.full_scan && !prm.xout && !prm.xpeer &&
                       st.d.ld * summary_elem_bytes(st.d.summary_dtype) > kSmallRowBytes;
  if (tc_path) return launch_select_tc(st, ws, prm, stream);
  if (flow_env && !prm.full_scan && !prm.xout && !prm.xpeer && prm.mode == 0 && st.d.batch <= kFlowMaxBatch)
    return st.d.summary_dtype == 0 ? launch_flow<float>(st, ws, prm, stream)
           : st.d.summary_dtype == 2 ? launch_flow<__nv_bfloat16>(st, ws, prm, stream)
                                     : launch_flow<double>(st, ws, prm, stream);
  // short rows: the whole cascade of a slot in one CTA (CHESS_SELECT_SMALL=0 to A/B)
  static const int small_env = getenv("CHESS_SELECT_SMALL") ? atoi(getenv("CHESS_SELECT_SMALL")) : 1;
  if (small_env && !prm.full_scan && !prm.xout && !prm.xpeer && prm.mode == 0 &&
      st.d.ld * summary_elem_bytes(st.d.summary_dtype) <= kSmallRowBytes) {
    // dynamic shared memory: the slot's anchor (d.dim doubles, <= 64 KB) and
    // the row staging buffer
    const size_t dyn = (size_t)((st.d.dim + 15) & ~15) * sizeof(double) + kSmallStageBytes;
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(select_small_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSmallRowBytes * 2 + kSmallStageBytes);
      cudaFuncSetAttribute(select_small_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSmallRowBytes * 4 + kSmallStageBytes);
      cudaFuncSetAttribute(select_small_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSmallRowBytes + kSmallStageBytes);
      configured = true;
    }
    if (st.d.summary_dtype == 0)
      select_small_kernel<float><<<st.d.batch, kNT, dyn, stream>>>(st, ws, prm);
    else if (st.d.summary_dtype == 2)
      select_small_kernel<__nv_bfloat16><<<st.d.batch, kNT, dyn, stream>>>(st, ws, prm);
    else
      select_small_kernel<double><<<st.d.batch, kNT, dyn, stream>>>(st, ws, prm);
    return check_launch("select_small");
  }
  const int nlev = prm.full_scan ? 1 : 3;
  for (int li = 0; li < nlev; ++li) {
    const int level = prm.full_scan ? 3 : li;
    const int rc = st.d.summary_dtype == 0   ? launch_scan<float>(st, ws, prm, level, stream)
                   : st.d.summary_dtype == 2 ? launch_scan<__nv_bfloat16>(st, ws, prm, level, stream)
                                             : launch_scan<double>(st, ws, prm, level, stream);
    if (rc) return rc;
  }
  return CHESS_OK;
}

// head shard: the scan of one level with its tail exporting partial scores
int launch_select_partial(const ChessState& st, const Workspace& ws, const SelParams& prm,
                          int level, cudaStream_t stream) {
  return st.d.summary_dtype == 0   ? launch_scan<float>(st, ws, prm, level, stream)
         : st.d.summary_dtype == 2 ? launch_scan<__nv_bfloat16>(st, ws, prm, level, stream)
                                   : launch_scan<double>(st, ws, prm, level, stream);
}

int launch_select_combine(const ChessState& st, const Workspace& ws, const SelParams& prm,
                          int level, const double* gathered, int world, cudaStream_t stream) {
  select_combine_kernel<<<st.d.batch, kNT, 0, stream>>>(st, ws, prm, level, gathered, world);
  return check_launch("select_combine");
}

int launch_select_pull(const ChessState& st, const Workspace& ws, const SelParams& prm, int level,
                       const double* recv, const uint32_t* flags, uint32_t* gen, int32_t* err,
                       cudaStream_t stream) {
  select_pull_kernel<<<st.d.batch, kNT, 0, stream>>>(st, ws, prm, level, recv, flags, gen, err);
  return check_launch("select_pull");
}

int launch_build_ws_all(const ChessState& st, cudaStream_t stream);

int launch_score_rows(const void* rows, int dtype, int64_t n, int64_t dim, int64_t ld,
                      const double* anchor, double* scores, cudaStream_t stream) {
  if (n == 0) return CHESS_OK;
  if (dtype == CHESS_F64)
    score_rows_kernel<double><<<(unsigned)n, 256, 0, stream>>>((const double*)rows, dim, ld, anchor, scores);
  else if (dtype == CHESS_F32)
    score_rows_kernel<float><<<(unsigned)n, 256, 0, stream>>>((const float*)rows, dim, ld, anchor, scores);
  else
    score_rows_kernel<__nv_bfloat16><<<(unsigned)n, 256, 0, stream>>>((const __nv_bfloat16*)rows, dim, ld, anchor, scores);
  return check_launch("score_rows");
}

int launch_prune(const double* s_g, int G, const double* s_c, int C, const double* s_p, int P,
                 const int64_t* p2c, const int64_t* c2g, double rg, double rc, double rp,
                 int32_t* out_pages, int32_t* out_count, void* workspace, cudaStream_t stream) {
  prune_kernel<<<1, kNT, 0, stream>>>(s_g, G, s_c, C, s_p, P, p2c, c2g, rg, rc, rp, out_pages,
                                      out_count, (uint8_t*)workspace);
  return check_launch("prune");
}

int launch_topk(const double* scores, int n, int k, const uint8_t* active, int32_t* out_idx,
                int32_t* out_count, int sorted, void* workspace, cudaStream_t stream) {
  topk_kernel<<<1, kNT, 0, stream>>>(scores, n, k, active, out_idx, out_count, sorted,
                                     (uint8_t*)workspace);
  return check_launch("topk");
}

int launch_working_set(const int32_t* selected, int n_sel, int n_pages, int window, int sinks,
                       const int32_t* page_table, int32_t* out_pages, int8_t* out_prov,
                       int32_t* out_phys, int32_t* out_len, cudaStream_t stream) {
  const size_t smem = (size_t)n_pages + 16;
  if (smem > 200 * 1024) return fail(CHESS_ERR_UNSUPPORTED, "working_set: %d pages too many", n_pages);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(working_set_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  working_set_kernel<<<1, kNT, smem, stream>>>(selected, n_sel, n_pages, window, sinks, page_table,
                                               out_pages, out_prov, out_phys, out_len);
  return check_launch("working_set");
}

int launch_gather_pages(const int32_t* table, int n_pages, const int64_t* idx, int n, int32_t* out,
                        int32_t* err, cudaStream_t stream) {
  if (n == 0) return CHESS_OK;
  gather_pages_kernel<<<(n + 255) / 256, 256, 0, stream>>>(table, n_pages, idx, n, out, err);
  return check_launch("gather_pages");
}

namespace {
__global__ void __launch_bounds__(256) build_ws_kernel(ChessState st) {
  __shared__ int s_scr[64];
  block_build_ws<256>(st, blockIdx.x, s_scr);
}
}  // namespace

namespace {
__global__ void __launch_bounds__(256) flush_ws_kernel(ChessState st, Workspace ws) {
  __shared__ int s_scr[64];
  const int s = blockIdx.x;
  if (!ws.ws_pending[s]) return;
  block_build_ws<256>(st, s, s_scr);
  if (threadIdx.x == 0) ws.ws_pending[s] = 0;
}
}  // namespace

int launch_flush_ws(const ChessState& st, const Workspace& ws, cudaStream_t stream) {
  flush_ws_kernel<<<st.d.batch, 256, 0, stream>>>(st, ws);
  return check_launch("flush_working_sets");
}

int launch_build_ws_all(const ChessState& st, cudaStream_t stream) {
  build_ws_kernel<<<st.d.batch, 256, 0, stream>>>(st);
  return check_launch("build_working_set");
}

}  // namespace chess

extern "C" int chess_debug_topk_trace(long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, chess::g_topk_trace, sizeof(chess::g_topk_trace)) == cudaSuccess ? 0 : 8;
}

extern "C" int chess_debug_select_trace(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, chess::g_sel_trace, sizeof(chess::g_sel_trace)) == cudaSuccess ? 0 : 8;
}

// trace build: [3][256][4] per-CTA stamps of the tensor-core scan, then [3][64][12] per-slot tails
extern "C" int chess_debug_select_tc_trace(unsigned long long* host_out) {
  if (cudaMemcpyFromSymbol(host_out, chess::g_tc_trace, sizeof(chess::g_tc_trace)) != cudaSuccess) return 8;
  return cudaMemcpyFromSymbol(host_out + 3 * 256 * 4, chess::g_tc_tail, sizeof(chess::g_tc_tail)) == cudaSuccess ? 0 : 8;
}

extern "C" int chess_debug_select_small_trace(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, chess::g_small_trace, sizeof(chess::g_small_trace)) == cudaSuccess ? 0 : 8;
}

extern "C" int chess_debug_select_tail_trace(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, chess::g_tail_trace, sizeof(chess::g_tail_trace)) == cudaSuccess ? 0 : 8;
}
