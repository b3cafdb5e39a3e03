// k_index.cu — KV append (a1) and the hierarchy summary builder (K1/K1b/K1c).
//
// Reference semantics:
//   append_token            kv_store.py:141-154  (tail write, seal event)
//   finalize_page           hierarchy.py:102-136 (Eq.1 page mean, chunk running
//                                                  sum, grid delta update)
//   rebuild_from_scratch    hierarchy.py:165-174 (= finalize_page in order)
//   from_page_vectors       hierarchy.py:43-58   (direct group sums)
//   compute_anchor          selection.py:44-59   (mean of last W page vectors)
// All per-element f64 arithmetic uses explicit _rn intrinsics in the
// reference's operation order, so the f64 state is bit-identical to pagesel's
// given identical keys.  The f32 matrices are rounded mirrors used only by the
// selection scan.
#include <algorithm>

#include <cuda_fp16.h>

#include "common.cuh"

namespace chess {

namespace {

constexpr int kNT = 256;

// D index j -> element offset inside the KV pool for page `phys`, row `row`.
__device__ __forceinline__ int64_t pool_offset(const ChessDims& d, int64_t j, int64_t phys,
                                               int row) {
  const int64_t hd = d.head_dim;
  const int64_t lh = j / hd;  // = l*H + h
  const int64_t e = j - lh * hd;
  const int64_t l = lh / d.kv_heads;
  const int64_t h = lh - l * d.kv_heads;
  return (((l * d.n_phys + phys) * d.kv_heads + h) * d.page_size + row) * hd + e;
}

// Anchor = mean of the last min(W, n) f64 page vectors (selection.py:57-59;
// numpy axis-0 reduction is sequential over rows).
__device__ __forceinline__ double anchor_elem(const double* pv64, int64_t ld, int n, int W,
                                              int64_t j) {
  const int w = min(W, n);
  double acc = pv64[(int64_t)(n - w) * ld + j];
  for (int i = n - w + 1; i < n; ++i) acc = __dadd_rn(acc, pv64[(int64_t)i * ld + j]);
  return __ddiv_rn(acc, (double)w);
}

// finalize_page's per-element update of chunk/grid sums for logical page p
// with page vector v (hierarchy.py:118-135).  Counts are positional.
struct FoldOut {
  double csum, gsum;
  int ccnt, gcnt;
};
__device__ __forceinline__ FoldOut fold_page(double v, int p, int Nc, int Ng, double csum_prev,
                                             double gsum_prev) {
  FoldOut o;
  const int c = p / Nc;
  const int g = c / Ng;
  const int pos_in_chunk = p - c * Nc;
  const int pos_in_grid = c - g * Ng;
  if (pos_in_chunk == 0) {
    o.csum = v;
    o.ccnt = 1;
    const double centroid = __ddiv_rn(o.csum, 1.0);
    if (pos_in_grid == 0) {
      o.gsum = centroid;
    } else {
      o.gsum = __dadd_rn(gsum_prev, centroid);
    }
    o.gcnt = pos_in_grid + 1;
  } else {
    const int cnt = pos_in_chunk;  // children before this page
    const double old_c = __ddiv_rn(csum_prev, (double)cnt);
    o.csum = __dadd_rn(csum_prev, v);
    o.ccnt = cnt + 1;
    const double cen = __ddiv_rn(o.csum, (double)o.ccnt);
    o.gsum = __dadd_rn(gsum_prev, __dsub_rn(cen, old_c));
    o.gcnt = pos_in_grid + 1;
  }
  return o;
}

// ---------------------------------------------------------------------------
// reset
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// device page pool (kv_store.py:103-136): a stack of free physical ids.
// ---------------------------------------------------------------------------
// Slot s takes `cnt` pages into page_table[s][pool_end ..), all or none (CAS
// loop on the stack top: no spurious failure under contention).  One thread.
__device__ bool pool_take(const ChessState& st, int s, int cnt) {
  const ChessDims& d = st.d;
  int end = st.pool_end[s];
  const int np = st.num_pages[s];
  if (end < np) {  // entries before num_pages were filled by the caller
    st.pool_base[s] = np;
    end = np;
  }
  if (cnt <= 0) return true;
  if (end + cnt > d.max_pages) {
    st.pool_oom[s] = 1;
    return false;
  }
  int top = atomicAdd(st.pool_top, 0);
  for (;;) {
    if (top < cnt) {
      st.pool_oom[s] = 1;
      return false;
    }
    const int seen = atomicCAS(st.pool_top, top, top - cnt);
    if (seen == top) break;
    top = seen;
  }
  int32_t* row = st.page_table + (int64_t)s * d.max_pages;
  for (int i = 0; i < cnt; ++i) row[end + i] = st.pool_free[top - 1 - i];
  st.pool_end[s] = end + cnt;
  return true;
}

__global__ void pool_init_kernel(ChessState st, const int32_t* ids, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    st.pool_free[i] = ids[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *st.pool_top = n;
}

__global__ void pool_reserve_kernel(ChessState st, const int32_t* counts) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= st.d.batch) return;
  pool_take(st, s, counts[s]);
}

// one CTA per slot: push the slot's pool pages back
__global__ void pool_release_kernel(ChessState st, const uint8_t* mask) {
  __shared__ int s_pos;
  const int s = blockIdx.x;
  if (mask && !mask[s]) return;
  const int base = st.pool_base[s], end = st.pool_end[s];
  const int n = end - base;
  if (n > 0) {
    if (threadIdx.x == 0) s_pos = atomicAdd(st.pool_top, n);
    __syncthreads();
    const int32_t* row = st.page_table + (int64_t)s * st.d.max_pages;
    for (int i = threadIdx.x; i < n; i += blockDim.x) st.pool_free[s_pos + i] = row[base + i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st.pool_base[s] = 0;
    st.pool_end[s] = 0;
    st.pool_oom[s] = 0;
  }
}

__global__ void reset_kernel(ChessState st, const uint8_t* mask) {
  const int s = blockIdx.x;
  if (mask && !mask[s]) return;
  const ChessDims& d = st.d;
  const int64_t ld = d.ld;
  for (int64_t j = threadIdx.x; j < ld; j += blockDim.x) {
    st.key_sum[(int64_t)s * ld + j] = 0.0;
    st.anchor[(int64_t)s * ld + j] = 0.0;
  }
  if (threadIdx.x == 0) {
    st.num_pages[s] = 0;
    st.tail_fill[s] = 0;
    st.token_count[s] = 0;
    st.sealed[s] = 0;
    st.num_sealed[s] = 0;
    st.n_semantic[s] = 0;
    st.ws_len[s] = 0;
    st.ent_count[s] = 0;
    st.gen_pages[s] = 0;
    st.fire[s] = 0;
    if (st.trigger_count) st.trigger_count[s] = 0;
    st.page_stats[2 * s] = 0.0;
    st.page_stats[2 * s + 1] = 0.0;
    for (int i = 0; i < 8; ++i) st.sel_stats[8 * s + i] = 0;
  }
}

// ---------------------------------------------------------------------------
// append (kv_store.py:141-154) + running key sum + WS refresh on page open
// grid: (ceil(D / (kNT*8)), batch)
// ---------------------------------------------------------------------------
// Columns [col0, col0 + ncols) of the flattened (layer, head, d) row; k_rows
// / v_rows hold just those columns.  post == 0 (the token's first call, the
// whole row for chess_append_kv): slot/row from the pre-append counters,
// which the last CTA then publishes.  post == 1 (later layer ranges of the
// same token, chess_append_kv_layers): the counters are already published,
// so the token's row is tail_fill - 1 of the last page and nothing else moves.
__global__ void __launch_bounds__(kNT) append_kernel(ChessState st, const __nv_bfloat16* k_rows,
                                                     const __nv_bfloat16* v_rows,
                                                     int64_t row_stride, const uint8_t* active,
                                                     int32_t* done, int64_t col0, int64_t ncols,
                                                     int post) {
  __shared__ int s_scratch[48];
  __shared__ int s_last;
  // The decode layer that follows (K4, launched with programmatic stream
  // serialization) may launch now: it executes griddepcontrol.wait before it
  // reads any state this kernel writes, so only its launch latency overlaps.
  pdl_launch_dependents();
  const int s = blockIdx.y;
  if (active && !active[s]) return;
  const ChessDims& d = st.d;
  const int B = d.page_size;
  // The token's columns and their running key sums do not depend on the
  // counters: load them first, so that the counter reads, these loads and
  // the key-sum reads share one memory round trip (the stores below would
  // otherwise keep the key-sum loads behind them).
  const int64_t cend_ = col0 + ncols;
  const int64_t j0_ = col0 + ((int64_t)blockIdx.x * kNT + threadIdx.x) * 8;
  const bool vec = (d.head_dim % 8) == 0 && (row_stride % 8) == 0 && (d.ld % 2) == 0;
  uint4 kv_pre = make_uint4(0, 0, 0, 0), vv_pre = kv_pre;
  double2 ks_pre[4];
  if (vec && j0_ < cend_) {
    kv_pre = __ldcs(reinterpret_cast<const uint4*>(k_rows + (int64_t)s * row_stride - col0 + j0_));
    vv_pre = __ldcs(reinterpret_cast<const uint4*>(v_rows + (int64_t)s * row_stride - col0 + j0_));
    const double2* k2 = reinterpret_cast<const double2*>(st.key_sum + (int64_t)s * d.ld + j0_);
#pragma unroll
    for (int q = 0; q < 4; ++q) ks_pre[q] = k2[q];
  }
  const int np = st.num_pages[s];
  const int fill = st.tail_fill[s];
  bool open_new;
  int slot, row;
  if (post) {
    if (st.pool_free && st.pool_oom[s]) return;  // the token's first call was refused
    open_new = fill == 1;
    slot = np - 1;
    row = fill - 1;
  } else {
    open_new = (np == 0) || (fill >= B);
    if (st.pool_free && open_new && st.pool_end[s] <= np) {
      // device pool: the page this token opens was never reserved (pool empty)
      if (blockIdx.x == 0 && threadIdx.x == 0) st.pool_oom[s] = 1;
      return;
    }
    slot = open_new ? np : np - 1;
    row = open_new ? 0 : fill;
  }
  const int64_t phys = st.page_table[(int64_t)s * d.max_pages + slot];
  const __nv_bfloat16* kr = k_rows + (int64_t)s * row_stride - col0;
  const __nv_bfloat16* vr = v_rows + (int64_t)s * row_stride - col0;
  double* ks = st.key_sum + (int64_t)s * d.ld;
  __nv_bfloat16* kp = reinterpret_cast<__nv_bfloat16*>(st.k_pool);
  __nv_bfloat16* vp = reinterpret_cast<__nv_bfloat16*>(st.v_pool);
  const int64_t cend = col0 + ncols;

  const int64_t j0 = col0 + ((int64_t)blockIdx.x * kNT + threadIdx.x) * 8;
  if (j0 < cend) {
    if (vec) {
      const int64_t off = pool_offset(d, j0, phys, row);
      *reinterpret_cast<uint4*>(kp + off) = kv_pre;
      *reinterpret_cast<uint4*>(vp + off) = vv_pre;
      const uint32_t w[4] = {kv_pre.x, kv_pre.y, kv_pre.z, kv_pre.w};
      double2* k2 = reinterpret_cast<double2*>(ks + j0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = bf2x2f(w[q]);
        double2 o;
        o.x = open_new ? (double)f.x : __dadd_rn(ks_pre[q].x, (double)f.x);
        o.y = open_new ? (double)f.y : __dadd_rn(ks_pre[q].y, (double)f.y);
        k2[q] = o;
      }
    } else {
      for (int q = 0; q < 8; ++q) {
        const int64_t j = j0 + q;
        if (j >= cend) break;
        const int64_t off = pool_offset(d, j, phys, row);
        kp[off] = kr[j];
        vp[off] = vr[j];
        const double f = (double)bf2f(kr[j]);
        ks[j] = open_new ? f : __dadd_rn(ks[j], f);
      }
    }
  }
  if (post) return;
  // last CTA of this slot publishes the new counters (all CTAs read the
  // pre-state above before incrementing).
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    const int prev = atomicAdd(&done[s], 1);
    s_last = (prev == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  fence_acq_rel_gpu();
  if (threadIdx.x == 0) {
    done[s] = 0;
    st.num_pages[s] = open_new ? np + 1 : np;
    st.tail_fill[s] = row + 1;
    st.token_count[s] += 1;
    st.sealed[s] = (row + 1 == B) ? 1 : 0;
    if (open_new) st.ent_count[s] = 0;
  }
  __syncthreads();
  if (open_new) block_build_ws<kNT>(st, s, s_scratch);
}

// ---------------------------------------------------------------------------
// K1 seal: fold the just-sealed tail page of each slot (hierarchy.py:102-136)
// grid: (ceil(ld / kNT), batch); one element per thread.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kNT) seal_kernel(ChessState st, int32_t* done, int32_t* pend) {
  __shared__ int s_last;
  const int s = blockIdx.y;
  if (!st.sealed[s]) {
    if (pend && blockIdx.x == 0 && threadIdx.x == 0) pend[s] = 0;  // no fp16 mirror rows owed
    return;
  }
  const ChessDims& d = st.d;
  const int64_t ld = d.ld;
  const int P = st.num_sealed[s];  // logical index of the sealing page
  const int Nc = d.pages_per_chunk, Ng = d.chunks_per_grid;
  const int c = P / Nc, g = c / Ng;
  const int64_t mc = max_chunks(d), mg = max_grids(d);
  const int64_t j = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (j < ld) {
    double* pv64 = st.page_vec64 + (int64_t)s * d.max_pages * ld;
    double* cs64 = st.chunk_sum64 + ((int64_t)s * mc + c) * ld;
    double* gs64 = st.grid_sum64 + ((int64_t)s * mg + g) * ld;
    double* ks = st.key_sum + (int64_t)s * ld;
    // Eq.1: page vector = mean of the B key rows (hierarchy.py:115)
    const double v = (j < d.dim) ? __ddiv_rn(ks[j], (double)d.page_size) : 0.0;
    pv64[(int64_t)P * ld + j] = v;
    const FoldOut o = fold_page(v, P, Nc, Ng, cs64[j], gs64[j]);
    cs64[j] = o.csum;
    gs64[j] = o.gsum;
    const double cen_c = __ddiv_rn(o.csum, (double)o.ccnt);
    const double cen_g = __ddiv_rn(o.gsum, (double)o.gcnt);
    st.chunk_vec64[((int64_t)s * mc + c) * ld + j] = cen_c;
    st.grid_vec64[((int64_t)s * mg + g) * ld + j] = cen_g;
    store_mirror(st.page_vec32, ((int64_t)s * d.max_pages + P) * ld + j, v, d.summary_dtype);
    store_mirror(st.chunk_vec32, ((int64_t)s * mc + c) * ld + j, cen_c, d.summary_dtype);
    store_mirror(st.grid_vec32, ((int64_t)s * mg + g) * ld + j, cen_g, d.summary_dtype);
    // Eq.3 anchor over the sealed pages (engine passes tail=None, simulate.py:136)
    st.anchor[(int64_t)s * ld + j] = anchor_elem(pv64, ld, P + 1, d.window_pages, j);
    ks[j] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    const int prev = atomicAdd(&done[s], 1);
    s_last = (prev == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    done[s] = 0;
    if (pend) pend[s] = P + 1;  // mirror16_kernel refreshes this page's rows
    st.num_sealed[s] = P + 1;
    st.sealed[s] = 0;
    // device pool: the slot's next append opens page num_pages — reserve it now
    if (st.pool_free && st.pool_end[s] <= st.num_pages[s]) pool_take(st, s, 1);
  }
}

// ---------------------------------------------------------------------------
// K1d fold given rows (function-level finalize_page)
// grid: (ceil(ld / kNT)); one element per thread
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ double ld_elem(const T* p) { return (double)(*p); }
template <>
__device__ __forceinline__ double ld_elem<__nv_bfloat16>(const __nv_bfloat16* p) {
  return (double)bf2f(*p);
}

template <typename T>
__global__ void __launch_bounds__(kNT) fold_rows_kernel(ChessState st, int s, const T* rows,
                                                        int n_rows, int64_t row_stride,
                                                        int32_t* done, int32_t* pend) {
  __shared__ int s_last;
  const ChessDims& d = st.d;
  const int64_t ld = d.ld;
  const int P = st.num_sealed[s];
  const int Nc = d.pages_per_chunk, Ng = d.chunks_per_grid;
  const int c = P / Nc, g = c / Ng;
  const int64_t mc = max_chunks(d), mg = max_grids(d);
  const int64_t j = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (j < ld) {
    double v = 0.0;
    if (j < d.dim) {
      if (d.dim == 1 && n_rows >= 8 && sizeof(T) == 8) {
        v = np_pairwise_sum(reinterpret_cast<const double*>(rows), n_rows, (int)row_stride);
      } else {
        for (int i = 0; i < n_rows; ++i) {
          const double x = ld_elem(rows + (int64_t)i * row_stride + j);
          v = i ? __dadd_rn(v, x) : x;
        }
      }
      v = __ddiv_rn(v, (double)n_rows);
    }
    double* pv64 = st.page_vec64 + (int64_t)s * d.max_pages * ld;
    double* cs64 = st.chunk_sum64 + ((int64_t)s * mc + c) * ld;
    double* gs64 = st.grid_sum64 + ((int64_t)s * mg + g) * ld;
    pv64[(int64_t)P * ld + j] = v;
    const FoldOut o = fold_page(v, P, Nc, Ng, cs64[j], gs64[j]);
    cs64[j] = o.csum;
    gs64[j] = o.gsum;
    const double cen_c = __ddiv_rn(o.csum, (double)o.ccnt);
    const double cen_g = __ddiv_rn(o.gsum, (double)o.gcnt);
    st.chunk_vec64[((int64_t)s * mc + c) * ld + j] = cen_c;
    st.grid_vec64[((int64_t)s * mg + g) * ld + j] = cen_g;
    store_mirror(st.page_vec32, ((int64_t)s * d.max_pages + P) * ld + j, v, d.summary_dtype);
    store_mirror(st.chunk_vec32, ((int64_t)s * mc + c) * ld + j, cen_c, d.summary_dtype);
    store_mirror(st.grid_vec32, ((int64_t)s * mg + g) * ld + j, cen_g, d.summary_dtype);
    st.anchor[(int64_t)s * ld + j] = anchor_elem(pv64, ld, P + 1, d.window_pages, j);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    const int prev = atomicAdd(&done[s], 1);
    s_last = (prev == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    done[s] = 0;
    if (pend) pend[s] = P + 1;
    st.num_sealed[s] = P + 1;
  }
}

// ---------------------------------------------------------------------------
// K1m: fp16 mirror rows + certified row bounds (summary_dtype 3).
// The tensor-core scan (k_select_tc.cuh) scores h = fp16(v) (round to
// nearest) of every f64 summary row v; its certificates need, per row,
//   err = ||v - h||_2  and  nrm = ||h||_2
// (both rounded up), kept in the row's stash right after its ld halves (the
// mirror buffers have the f32 row pitch, 4*ld bytes).  One CTA per (row,
// slot); fixed thread partition and reduction tree, so the bounds are
// deterministic.  An fp16 overflow makes err infinite: the row is then
// always rescored exactly, never mis-certified.
// mode 0: the page pend[s]-1 just sealed and its chunk and grid (3 CTAs);
// mode 1: every row of the slot's sealed index (bulk builds).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) mirror16_kernel(ChessState st, const int32_t* pend, int only_seq, int mode) {
  const int s = only_seq >= 0 ? only_seq : blockIdx.y;
  const ChessDims& d = st.d;
  const int Nc = d.pages_per_chunk, Ng = d.chunks_per_grid;
  int which, row;
  if (mode == 0) {
    const int P = pend[s] - 1;
    if (P < 0) return;
    which = blockIdx.x;
    row = which == 0 ? P : (which == 1 ? P / Nc : P / Nc / Ng);
  } else {
    const int n = st.num_sealed[s];
    const int C = (n + Nc - 1) / Nc, G = (C + Ng - 1) / Ng;
    const int r = blockIdx.x;
    if (r < n) which = 0, row = r;
    else if (r < n + C) which = 1, row = r - n;
    else if (r < n + C + G) which = 2, row = r - n - C;
    else return;
  }
  const int64_t rows = which == 0 ? (int64_t)d.max_pages : (which == 1 ? max_chunks(d) : max_grids(d));
  const int64_t ri = (int64_t)s * rows + row;
  const double* src = (which == 0 ? st.page_vec64 : (which == 1 ? st.chunk_vec64 : st.grid_vec64)) + ri * d.ld;
  float* mrow = (which == 0 ? st.page_vec32 : (which == 1 ? st.chunk_vec32 : st.grid_vec32)) + ri * d.ld;
  __half* dst = reinterpret_cast<__half*>(mrow);
  double e2 = 0.0, n2 = 0.0;
  for (int64_t j = (int64_t)threadIdx.x * 4; j < d.ld; j += 256 * 4) {
    const double2 a = *reinterpret_cast<const double2*>(src + j);
    const double2 b = *reinterpret_cast<const double2*>(src + j + 2);
    const double v[4] = {a.x, a.y, b.x, b.y};
    __half h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h[q] = __double2half(v[q]);
      const double hd = (double)__half2float(h[q]);
      const double dl = v[q] - hd;
      e2 = __fma_rn(dl, dl, e2);
      n2 = __fma_rn(hd, hd, n2);
    }
    uint2 w;
    w.x = (uint32_t)__half_as_ushort(h[0]) | ((uint32_t)__half_as_ushort(h[1]) << 16);
    w.y = (uint32_t)__half_as_ushort(h[2]) | ((uint32_t)__half_as_ushort(h[3]) << 16);
    *reinterpret_cast<uint2*>(dst + j) = w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    n2 += __shfl_xor_sync(0xffffffffu, n2, o);
  }
  __shared__ double s_e[8], s_n[8];
  if ((threadIdx.x & 31) == 0) {
    s_e[threadIdx.x >> 5] = e2;
    s_n[threadIdx.x >> 5] = n2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = 0.0, n = 0.0;
    for (int w = 0; w < 8; ++w) {
      e += s_e[w];
      n += s_n[w];
    }
    // sums of <= 2^31 non-negative terms: relative error < 2^-21 is far
    // inside the (1 + 2^-20) inflation; sqrt is correctly rounded
    double* stash = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(mrow) + 2 * d.ld);
    stash[0] = sqrt(e) * (1.0 + 0x1p-20);
    stash[1] = sqrt(n) * (1.0 + 0x1p-20);
  }
}

// ---------------------------------------------------------------------------
// K1b bulk build from the KV pool = finalize_page over pages [0, n) in order.
// grid: (ceil(ld / (kNT*2)), n_grids_max, batch); each thread owns 2 elements
// and walks every page of one grid sequentially (exact finalize_page order).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kNT) build_kernel(ChessState st, const int32_t* n_pages) {
  const int s = blockIdx.z;
  const int g = blockIdx.y;
  const ChessDims& d = st.d;
  const int n = n_pages[s];
  const int Nc = d.pages_per_chunk, Ng = d.chunks_per_grid;
  const int pages_per_grid = Nc * Ng;
  const int p_begin = g * pages_per_grid;
  if (p_begin >= n) return;
  const int p_end = min(n, p_begin + pages_per_grid);
  const int64_t ld = d.ld;
  const int64_t mc = max_chunks(d), mg = max_grids(d);
  const int B = d.page_size;
  const int64_t j0 = ((int64_t)blockIdx.x * kNT + threadIdx.x) * 2;
  if (j0 >= ld) return;
  const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(st.k_pool);
  const int32_t* pt = st.page_table + (int64_t)s * d.max_pages;
  double* pv64 = st.page_vec64 + (int64_t)s * d.max_pages * ld;
  const bool pair_ok = (d.head_dim % 2) == 0;
  double csum[2] = {0.0, 0.0}, gsum[2] = {0.0, 0.0};
  for (int p = p_begin; p < p_end; ++p) {
    const int64_t phys = pt[p];
    double v[2];
    // Eq.1: sequential f64 sum over the page's B rows, then / B
    if (pair_ok && j0 + 1 < d.dim) {
      const int64_t off = pool_offset(d, j0, phys, 0);
      double a0 = 0.0, a1 = 0.0;
      for (int t = 0; t < B; ++t) {
        const float2 f = bf2x2f(*reinterpret_cast<const uint32_t*>(kp + off + (int64_t)t * d.head_dim));
        a0 = t ? __dadd_rn(a0, (double)f.x) : (double)f.x;
        a1 = t ? __dadd_rn(a1, (double)f.y) : (double)f.y;
      }
      v[0] = __ddiv_rn(a0, (double)B);
      v[1] = __ddiv_rn(a1, (double)B);
    } else {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t j = j0 + q;
        double a = 0.0;
        if (j < d.dim) {
          const int64_t off = pool_offset(d, j, phys, 0);
          for (int t = 0; t < B; ++t) {
            const double f = (double)bf2f(kp[off + (int64_t)t * d.head_dim]);
            a = t ? __dadd_rn(a, f) : f;
          }
          a = __ddiv_rn(a, (double)B);
        }
        v[q] = a;
      }
    }
    const int c = p / Nc;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t j = j0 + q;
      if (j >= ld) break;
      pv64[(int64_t)p * ld + j] = v[q];
      store_mirror(st.page_vec32, ((int64_t)s * d.max_pages + p) * ld + j, v[q], d.summary_dtype);
      const FoldOut o = fold_page(v[q], p, Nc, Ng, csum[q], gsum[q]);
      csum[q] = o.csum;
      gsum[q] = o.gsum;
      // write chunk state after its last page in range, grid after each page
      if ((p + 1) % Nc == 0 || p + 1 == p_end) {
        const double cen = __ddiv_rn(o.csum, (double)o.ccnt);
        st.chunk_sum64[((int64_t)s * mc + c) * ld + j] = o.csum;
        st.chunk_vec64[((int64_t)s * mc + c) * ld + j] = cen;
        store_mirror(st.chunk_vec32, ((int64_t)s * mc + c) * ld + j, cen, d.summary_dtype);
      }
      if (p + 1 == p_end) {
        const double gc = __ddiv_rn(o.gsum, (double)o.gcnt);
        st.grid_sum64[((int64_t)s * mg + g) * ld + j] = o.gsum;
        st.grid_vec64[((int64_t)s * mg + g) * ld + j] = gc;
        store_mirror(st.grid_vec32, ((int64_t)s * mg + g) * ld + j, gc, d.summary_dtype);
      }
    }
  }
}

// Epilogue of K1b / K1c: anchor, running tail key sum, counters.
// grid: (ceil(ld / kNT), batch)
__global__ void __launch_bounds__(kNT) build_finish_kernel(ChessState st, const int32_t* n_pages,
                                                           int only_seq) {
  const int s = only_seq >= 0 ? only_seq : blockIdx.y;
  const ChessDims& d = st.d;
  const int n = n_pages[only_seq >= 0 ? 0 : s];
  const int64_t ld = d.ld;
  const int64_t j = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (j < ld) {
    const double* pv64 = st.page_vec64 + (int64_t)s * d.max_pages * ld;
    st.anchor[(int64_t)s * ld + j] = n > 0 ? anchor_elem(pv64, ld, n, d.window_pages, j) : 0.0;
    // open tail (pages beyond the index): running sum of its filled rows
    double ks = 0.0;
    const int np = st.num_pages[s];
    const int fill = st.tail_fill[s];
    if (only_seq < 0 && np == n + 1 && fill < d.page_size && j < d.dim) {
      const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(st.k_pool);
      const int64_t phys = st.page_table[(int64_t)s * d.max_pages + n];
      const int64_t off = pool_offset(d, j, phys, 0);
      for (int t = 0; t < fill; ++t) {
        const double f = (double)bf2f(kp[off + (int64_t)t * d.head_dim]);
        ks = t ? __dadd_rn(ks, f) : f;
      }
    }
    if (only_seq < 0) st.key_sum[(int64_t)s * ld + j] = ks;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st.num_sealed[s] = n;
    st.sealed[s] = 0;
  }
}

// ---------------------------------------------------------------------------
// K1c from_page_vectors (hierarchy.py:43-58): chunk sums = sequential sum of
// <= N_c f64 page rows; grid sums = sequential sum of <= N_g chunk centroids.
// grid: (ceil(ld / kNT), n_chunks) then (ceil(ld/kNT), n_grids)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kNT) from_vectors_pages(ChessState st, int s, const double* rows,
                                                          int n, int64_t row_stride) {
  const ChessDims& d = st.d;
  const int64_t ld = d.ld;
  const int c = blockIdx.y;
  const int Nc = d.pages_per_chunk;
  const int p0 = c * Nc, p1 = min(n, p0 + Nc);
  const int64_t j = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (j >= ld) return;
  const int64_t mc = max_chunks(d);
  double* pv64 = st.page_vec64 + (int64_t)s * d.max_pages * ld;
  double acc = 0.0;
  for (int p = p0; p < p1; ++p) {
    const double v = j < d.dim ? rows[(int64_t)p * row_stride + j] : 0.0;
    pv64[(int64_t)p * ld + j] = v;
    store_mirror(st.page_vec32, ((int64_t)s * d.max_pages + p) * ld + j, v, d.summary_dtype);
    acc = (p == p0) ? v : __dadd_rn(acc, v);
  }
  if (d.dim == 1 && p1 - p0 >= 8) acc = np_pairwise_sum(pv64 + (int64_t)p0 * ld + j, p1 - p0, (int)ld);
  const double cen = __ddiv_rn(acc, (double)(p1 - p0));
  st.chunk_sum64[((int64_t)s * mc + c) * ld + j] = acc;
  st.chunk_vec64[((int64_t)s * mc + c) * ld + j] = cen;
  store_mirror(st.chunk_vec32, ((int64_t)s * mc + c) * ld + j, cen, d.summary_dtype);
}

__global__ void __launch_bounds__(kNT) from_vectors_grids(ChessState st, int s, int n_chunks) {
  const ChessDims& d = st.d;
  const int64_t ld = d.ld;
  const int g = blockIdx.y;
  const int Ng = d.chunks_per_grid;
  const int c0 = g * Ng, c1 = min(n_chunks, c0 + Ng);
  const int64_t j = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (j >= ld) return;
  const int64_t mc = max_chunks(d), mg = max_grids(d);
  const double* cv = st.chunk_vec64 + (int64_t)s * mc * ld;
  double acc = 0.0;
  for (int c = c0; c < c1; ++c) acc = (c == c0) ? cv[(int64_t)c * ld + j] : __dadd_rn(acc, cv[(int64_t)c * ld + j]);
  if (d.dim == 1 && c1 - c0 >= 8) acc = np_pairwise_sum(cv + (int64_t)c0 * ld + j, c1 - c0, (int)ld);
  const double cen = __ddiv_rn(acc, (double)(c1 - c0));
  st.grid_sum64[((int64_t)s * mg + g) * ld + j] = acc;
  st.grid_vec64[((int64_t)s * mg + g) * ld + j] = cen;
  store_mirror(st.grid_vec32, ((int64_t)s * mg + g) * ld + j, cen, d.summary_dtype);
}

// ---------------------------------------------------------------------------
// mean of rows (page pooling / anchor window), reference order
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ double load_as_double(const T* p) { return (double)(*p); }
template <>
__device__ __forceinline__ double load_as_double<__nv_bfloat16>(const __nv_bfloat16* p) {
  return (double)bf2f(*p);
}

template <typename T>
__global__ void mean_rows_kernel(const T* rows, int64_t n, int64_t dim, int64_t ld, double* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= dim) return;
  double acc = 0.0;
  if (dim == 1 && n >= 8 && sizeof(T) == 8) {
    acc = np_pairwise_sum(reinterpret_cast<const double*>(rows) + j, (int)n, (int)ld);
  } else {
    for (int64_t i = 0; i < n; ++i) {
      const double v = load_as_double(rows + i * ld + j);
      acc = i ? __dadd_rn(acc, v) : v;
    }
  }
  out[j] = __ddiv_rn(acc, (double)n);
}

}  // namespace

// ---------------------------------------------------------------------------
// launch wrappers (called from capi.cu)
// ---------------------------------------------------------------------------
int launch_reset(const ChessState& st, const uint8_t* mask, cudaStream_t stream) {
  reset_kernel<<<st.d.batch, 256, 0, stream>>>(st, mask);
  return check_launch("reset_slots");
}

int launch_pool_init(const ChessState& st, const int32_t* ids, int n, cudaStream_t stream) {
  pool_init_kernel<<<std::max(1, std::min(148, (n + 255) / 256)), 256, 0, stream>>>(st, ids, n);
  return check_launch("pool_init");
}

int launch_pool_reserve(const ChessState& st, const int32_t* counts, cudaStream_t stream) {
  pool_reserve_kernel<<<(st.d.batch + 127) / 128, 128, 0, stream>>>(st, counts);
  return check_launch("pool_reserve");
}

int launch_pool_release(const ChessState& st, const uint8_t* mask, cudaStream_t stream) {
  pool_release_kernel<<<st.d.batch, 128, 0, stream>>>(st, mask);
  return check_launch("pool_release");
}

int launch_append(const ChessState& st, const Workspace& ws, const void* k_rows, const void* v_rows,
                  int64_t row_stride, const uint8_t* active, cudaStream_t stream, int64_t col0,
                  int64_t ncols, int post) {
  if (ncols < 0) ncols = st.d.dim;
  const int64_t per = (int64_t)kNT * 8;
  dim3 grid((unsigned)((ncols + per - 1) / per), st.d.batch);
  append_kernel<<<grid, kNT, 0, stream>>>(st, reinterpret_cast<const __nv_bfloat16*>(k_rows),
                                          reinterpret_cast<const __nv_bfloat16*>(v_rows),
                                          row_stride, active, ws.append_done, col0, ncols, post);
  return check_launch("append_kv");
}

int launch_seal(const ChessState& st, const Workspace& ws, cudaStream_t stream) {
  dim3 grid((unsigned)((st.d.ld + kNT - 1) / kNT), st.d.batch);
  const bool tcs = st.d.summary_dtype == kSummaryTc;
  seal_kernel<<<grid, kNT, 0, stream>>>(st, ws.seal_done, tcs ? ws.mirror_pend : nullptr);
  int rc = check_launch("summary_seal");
  if (rc || !tcs) return rc;
  mirror16_kernel<<<dim3(3, st.d.batch), 256, 0, stream>>>(st, ws.mirror_pend, -1, 0);
  return check_launch("mirror16");
}

int launch_fold(const ChessState& st, const Workspace& ws, int seq, const void* rows, int dtype,
                int n_rows, int64_t row_stride, cudaStream_t stream) {
  const unsigned grid = (unsigned)((st.d.ld + kNT - 1) / kNT);
  const bool tcs = st.d.summary_dtype == kSummaryTc;
  int32_t* pend = tcs ? ws.mirror_pend : nullptr;
  if (dtype == CHESS_F64)
    fold_rows_kernel<double><<<grid, kNT, 0, stream>>>(st, seq, (const double*)rows, n_rows, row_stride, ws.seal_done, pend);
  else if (dtype == CHESS_F32)
    fold_rows_kernel<float><<<grid, kNT, 0, stream>>>(st, seq, (const float*)rows, n_rows, row_stride, ws.seal_done, pend);
  else
    fold_rows_kernel<__nv_bfloat16><<<grid, kNT, 0, stream>>>(st, seq, (const __nv_bfloat16*)rows, n_rows, row_stride, ws.seal_done, pend);
  int rc = check_launch("summary_fold");
  if (rc || !tcs) return rc;
  mirror16_kernel<<<dim3(3, 1), 256, 0, stream>>>(st, ws.mirror_pend, seq, 0);
  return check_launch("mirror16");
}

int launch_build(const ChessState& st, const int32_t* n_pages, cudaStream_t stream) {
  const int64_t per = (int64_t)kNT * 2;
  dim3 grid((unsigned)((st.d.ld + per - 1) / per), (unsigned)max_grids(st.d), st.d.batch);
  build_kernel<<<grid, kNT, 0, stream>>>(st, n_pages);
  int rc = check_launch("summary_build");
  if (rc) return rc;
  dim3 g2((unsigned)((st.d.ld + kNT - 1) / kNT), st.d.batch);
  build_finish_kernel<<<g2, kNT, 0, stream>>>(st, n_pages, -1);
  rc = check_launch("summary_build_finish");
  if (rc || st.d.summary_dtype != kSummaryTc) return rc;
  mirror16_kernel<<<dim3((unsigned)max_rows(st.d), st.d.batch), 256, 0, stream>>>(st, nullptr, -1, 1);
  return check_launch("mirror16");
}

int launch_from_vectors(const ChessState& st, int seq, const double* rows, int n,
                        int64_t row_stride, const int32_t* n_dev, cudaStream_t stream) {
  const ChessDims& d = st.d;
  const int nc = (n + d.pages_per_chunk - 1) / d.pages_per_chunk;
  const int ng = (nc + d.chunks_per_grid - 1) / d.chunks_per_grid;
  const unsigned gx = (unsigned)((d.ld + kNT - 1) / kNT);
  if (n > 0) {
    from_vectors_pages<<<dim3(gx, nc), kNT, 0, stream>>>(st, seq, rows, n, row_stride);
    int rc = check_launch("from_vectors_pages");
    if (rc) return rc;
    from_vectors_grids<<<dim3(gx, ng), kNT, 0, stream>>>(st, seq, nc);
    rc = check_launch("from_vectors_grids");
    if (rc) return rc;
  }
  build_finish_kernel<<<dim3(gx, 1), kNT, 0, stream>>>(st, n_dev, seq);
  int rc = check_launch("from_vectors_finish");
  if (rc || d.summary_dtype != kSummaryTc) return rc;
  mirror16_kernel<<<dim3((unsigned)max_rows(d), 1), 256, 0, stream>>>(st, nullptr, seq, 1);
  return check_launch("mirror16");
}

int launch_mean_rows(const void* rows, int dtype, int64_t n, int64_t dim, int64_t ld, double* out,
                     cudaStream_t stream) {
  const unsigned grid = (unsigned)((dim + 255) / 256);
  if (dtype == CHESS_F64)
    mean_rows_kernel<double><<<grid, 256, 0, stream>>>((const double*)rows, n, dim, ld, out);
  else if (dtype == CHESS_F32)
    mean_rows_kernel<float><<<grid, 256, 0, stream>>>((const float*)rows, n, dim, ld, out);
  else
    mean_rows_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>((const __nv_bfloat16*)rows, n, dim,
                                                              ld, out);
  return check_launch("mean_rows");
}

}  // namespace chess
