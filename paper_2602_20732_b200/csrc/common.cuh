// common.cuh — shared device helpers for the CHESS B200 kernels (sm_100a).
//
// Contents: error plumbing for the C-ABI, bf16 helpers, mbarrier +
// cp.async.bulk (TMA 1-D bulk copy) PTX wrappers, f64 helpers that reproduce
// NumPy's summation orders bit-for-bit, the orderable score key used by every
// top-k (ties to the lower index, selection.py:77-88), and a block-wide radix
// select.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>

#include "../../include/chess_b200.h"

namespace chess {

// ---------------------------------------------------------------------------
// host-side error plumbing
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);
int check_launch(const char* what);
int num_sms();

__host__ __device__ inline int64_t max_chunks(const ChessDims& d) {
  return (d.max_pages + d.pages_per_chunk - 1) / d.pages_per_chunk;
}
__host__ __device__ inline int64_t max_grids(const ChessDims& d) {
  return (max_chunks(d) + d.chunks_per_grid - 1) / d.chunks_per_grid;
}
__host__ __device__ inline int64_t max_rows(const ChessDims& d) { return d.max_pages + max_chunks(d) + max_grids(d); }

// ---------------------------------------------------------------------------
// workspace layout (carved from ChessState::workspace, see capi.cu)
// ---------------------------------------------------------------------------
// Elements of one (row, slice) scan work unit: 16 KB of summary row per
// bulk copy (f32 mirrors: 4096, f64 rows: 2048), so a ring of 12 stages
// holds 1.5 items of 8 rows.
constexpr int kScanSliceBytes = 16384;
// summary_dtype: 0 f32 mirrors, 1 f64 (no mirrors), 2 bf16 mirrors,
// 3 fp16 mirrors scored on tcgen05 with certified bounds + exact f64
// rescoring of the rows near each level's cut (k_select_tc.cuh).  For 3 the
// element size below is that of the rows the exact (rescoring / short-row)
// scan reads: f64.
constexpr int kSummaryTc = 3;
#ifndef CHESS_TC_KBS
#define CHESS_TC_KBS 4
#endif
constexpr int kTcKbs = CHESS_TC_KBS;  // 64-element K blocks per tensor-core scan stage
__host__ __device__ constexpr int summary_elem_bytes(int summary_dtype) {
  return summary_dtype == 0 ? 4 : (summary_dtype == 2 ? 2 : 8);
}
__host__ __device__ constexpr int scan_slice(int summary_dtype) { return kScanSliceBytes / summary_elem_bytes(summary_dtype); }
constexpr int kScanRows = 8;       // rows per work item
constexpr int kScanThreads = 256;
constexpr int kMaxBatch = 1024;

// Debug timelines (per-CTA globaltimer stamps read by tools/*_micro.py).
// Off in the product build: the stamps are global stores that every later
// release fence in the kernel would have to wait for.  build.py builds a
// separate libchess_b200_trace.so with -DCHESS_TRACE=1.
#ifndef CHESS_TRACE
#define CHESS_TRACE 0
#endif
constexpr bool kTrace = CHESS_TRACE != 0;

struct Workspace {
  int32_t* sel_done;     // [batch]
  int32_t* ws_pending;   // [batch] working set owed by a defer_ws selection pass
  int32_t* flow;         // select dataflow scheduler: [0] next item, [1 .. 3b] items done per
                         // (level, slot), [1+3b .. 1+4b] levels finished per slot
  int32_t* cand;         // [batch][3][max_rows]  candidate row ids per level
  int32_t* cand_n;       // [batch][4]            candidate counts (levels 0..2, full)
  double* scores;        // [batch][max_rows]     reduced scores of the current level
  uint64_t* keys;        // [batch][max_rows]
  double* part;          // [batch][max_rows][n_slices]
  int32_t* kept;         // [batch][max_rows]
  int32_t* plist;        // [batch][max_rows]  kept parents (ascending)
  int32_t* attn_done;    // [batch*kv_heads]
  float* attn_part;      // [(batch*kv_heads + attn_ctas)][q_per_kv][head_dim + 2]
  int32_t* ent_done;     // [batch]
  double* ent_part;      // [batch][kEntSplit][3]
  int32_t* append_done;  // [batch]
  int32_t* seal_done;    // [batch]
  // summary_dtype 3 (tensor-core scan, k_select_tc.cuh)
  int32_t* mirror_pend;  // [batch] 1 + page sealed by the last seal/fold (0: none)
  uint8_t* anc_tile;     // [batch][nkb_pad][1024] anchor hi/lo as swizzled fp16 B atoms
  double* anc_stats;     // [batch][n_slices][4] per-slice sum a^2, sum rem^2, sum (|hi|+|lo|)^2
  int32_t* anc_exp;      // [batch][n_slices] power-of-two scale of the slice's anchor
  int32_t* cls;          // [batch][max_rows] certification: 0 out, 1 certainly in, 2 uncertain
  int32_t* unc;          // [batch][max_rows] candidate positions to rescore exactly
  int32_t* unc_meta;     // [batch][4] uncertain count, seats left for them, candidates
  int32_t nkb_pad;       // 64-element K blocks per row, padded to the stage size
  int32_t attn_ctas;
  int32_t n_slices;
};

constexpr int kEntSplit = 64;  // max CTAs per logit row (entropy split partials)
constexpr int kAttnCtasMax = 320;               // attention CTAs (<= 2 per SM)
constexpr int kAttnWarpsMax = kAttnCtasMax * 8; // stream-K warps (partial slots)

size_t workspace_layout(const ChessDims& d, void* base, Workspace* ws);

// head-shard output gather over peer memory (chess_sparse_decode_gather)
constexpr int kMaxPeers = 8;
struct PeerOut {
  __nv_bfloat16* peer_out[kMaxPeers - 1];  // this rank's block in every other rank's region
  int n_peer;
};

struct SelParams {
  double rho[3];
  int32_t full_scan;
  int32_t force_all;
  int32_t mode;  // debug (CHESS_SELECT_MODE): 0 normal, 1 no math, 2 no loads
  int32_t defer_ws;  // leave working sets to chess_flush_working_sets (concurrent step)
  int32_t rescore;   // summary_dtype 3: exact f64 pass over the level's uncertain rows
  // KV-head shard: when set, the level's tail stops after the
  // fixed-order slice reduction and exports this rank's PARTIAL scores to
  // xout[slot * xld + candidate]; select_combine_kernel finishes the level.
  double* xout;
  int64_t xld;
  // Peer-memory transport of the same exchange (chess_select_push): the tail
  // stores the partial row straight into every peer's receive buffer
  // xpeer[p][(gen&1)][xrank][slot][xld] over NVLink and release-stores
  // xflag[p][slot * xworld + xrank] = gen + 1 (gen = xgen[slot]).
  double* const* xpeer;
  uint32_t* const* xflag;
  const uint32_t* xgen;
  int32_t xrank, xworld;
};

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }

__device__ __forceinline__ float2 bf2x2f(uint32_t packed) {
  float2 r;
  r.x = __uint_as_float(packed << 16);
  r.y = __uint_as_float(packed & 0xffff0000u);
  return r;
}

// write a scanned-summary mirror element (the *_vec32 buffers hold f32 rows
// for summary_dtype 0 and bf16 rows for 2; f64 scans read the f64 rows)
// (summary_dtype 3: the fp16 mirror and its row bounds are written by
// mirror16_kernel from the finished f64 rows, k_index.cu)
__device__ __forceinline__ void store_mirror(float* base, int64_t i, double v, int summary_dtype) {
  if (summary_dtype == 0) base[i] = (float)v;
  else if (summary_dtype == 2) reinterpret_cast<__nv_bfloat16*>(base)[i] = __double2bfloat16(v);
}

// Orderable key for f64 scores: larger score -> larger key.  -0.0 is
// canonicalised to +0.0 (NumPy compares them equal, stable order decides) and
// NaN sorts below -inf (argsort of -scores puts NaN last).
__device__ __forceinline__ uint64_t score_key(double s) {
  if (s != s) return 0ull;
  if (s == 0.0) s = 0.0;
  uint64_t b = (uint64_t)__double_as_longlong(s);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
// inverse of score_key on non-NaN values
__device__ __forceinline__ double double_of_key(uint64_t k) {
  const uint64_t b = (k & 0x8000000000000000ull) ? (k ^ 0x8000000000000000ull) : ~k;
  return __longlong_as_double((long long)b);
}
// order-preserving 32-bit key of a float (-0 and +0 equal, NaN lowest) and its inverse
__device__ __forceinline__ uint32_t float_key(float f) {
  if (f != f) return 0u;
  if (f == 0.0f) f = 0.0f;
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float float_of_key(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
}

// NumPy pairwise summation of a contiguous f64 vector (numpy
// DOUBLE_pairwise_sum, blocks of 8 accumulators up to 128 elements).  Used for
// page statistics (uncertainty.py:41-48 -> np.mean) so device results are
// bit-identical to the reference given identical inputs.
template <typename F>
__device__ __forceinline__ double np_pairwise_leaf(F at, int off, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, at(off + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = at(off + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], at(off + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, at(off + i));
  return res;
}

// Non-recursive evaluation of NumPy's pairwise tree (n > 128 splits at
// n2 = n/2 rounded down to a multiple of 8) with an explicit stack.
template <typename F>
__device__ double np_pairwise(F at, int n) {
  if (n <= 128) return np_pairwise_leaf(at, 0, n);
  int st_off[40], st_n[40], st_phase[40];
  double st_left[40];
  int sp = 0;
  st_off[0] = 0; st_n[0] = n; st_phase[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    const int off = st_off[sp], m = st_n[sp];
    if (m <= 128) {
      ret = np_pairwise_leaf(at, off, m);
      --sp;
      continue;
    }
    int m2 = m / 2;
    m2 -= m2 % 8;
    if (st_phase[sp] == 0) {  // descend left
      st_phase[sp] = 1;
      ++sp;
      st_off[sp] = off; st_n[sp] = m2; st_phase[sp] = 0;
    } else if (st_phase[sp] == 1) {  // left done -> descend right
      st_left[sp] = ret;
      st_phase[sp] = 2;
      ++sp;
      st_off[sp] = off + m2; st_n[sp] = m - m2; st_phase[sp] = 0;
    } else {  // both done
      ret = __dadd_rn(st_left[sp], ret);
      --sp;
    }
  }
  return ret;
}

__device__ __forceinline__ double np_pairwise_sum(const double* a, int n, int stride) {
  return np_pairwise([=](int i) { return a[(int64_t)i * stride]; }, n);
}

// ---------------------------------------------------------------------------
// mbarrier + TMA bulk copy (cp.async.bulk) wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
#ifdef CHESS_MBAR_TEST_WAIT
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
#else
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
#endif
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline that never completes (lost TMA transaction,
// protocol bug) traps after ~4 s of wall time instead of hanging the device;
// the trap surfaces as a CUDA error at the next synchronisation.
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = global_ns();
  uint32_t polls = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++polls & 1023u) == 0 && global_ns() - t0 > 4000000000ull) {
      printf("chess: mbarrier wait timed out (block %d thread %d parity %u)\n", blockIdx.x,
             threadIdx.x, parity);
      asm volatile("trap;");
    }
  }
}
// ---- thread-block clusters / DSMEM ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32x2(uint32_t addr, float a, float b) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
// asynchronous 8-byte store into another CTA's shared memory that completes
// `bytes` of the transaction count of that CTA's mbarrier (no release fence:
// the consumer's mbarrier phase completion makes the data visible)
__device__ __forceinline__ void st_async_f32x2(uint32_t cluster_addr, float a, float b,
                                               uint32_t cluster_bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(
          cluster_addr),
      "f"(a), "f"(b), "r"(cluster_bar)
      : "memory");
}
// arrive on an mbarrier in another CTA of the cluster, releasing this
// thread's prior (DSMEM) writes at cluster scope
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar_addr)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint64_t t0 = global_ns();
  uint32_t polls = 0;
  while (!mbar_try_wait_cluster(bar, parity)) {
    if ((++polls & 1023u) == 0 && global_ns() - t0 > 4000000000ull) {
      printf("chess: cluster mbarrier wait timed out (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      asm volatile("trap;");
    }
  }
}

// 1-D bulk global->shared copy completing on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// GPU-scope acquire/release fence: orders this thread's prior global writes
// before (and later reads after) a flag/counter handshake between CTAs.  Far
// cheaper than __threadfence() (fence.sc.gpu + L1 invalidate, SASS ERRBAR +
// CCTL.IVALL), which showed up as microseconds per split-K merge.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// system scope (peer GPU memory over NVLink)
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// explicit shared-window vector loads (a generic pointer into dynamic smem
// after alignment arithmetic compiles to LD.E, not LDS)
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ double2 lds_d2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

// Programmatic dependent launch controls (griddepcontrol, sm_90+).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ double shfl_xor_d(double v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// Named barrier 1 over the first NT threads: the block helpers below run on a
// CTA's compute warps while a producer warp (if any) keeps streaming.
template <int NT>
__device__ __forceinline__ void block_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

// ---------------------------------------------------------------------------
// block-wide helpers (blockDim.x == NT, multiple of 32)
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int v, int* smem_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  block_sync<NT>();
  if (warp == 0) {
    int w = (lane < NT / 32) ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) smem_warp[lane] = w;
  }
  block_sync<NT>();
  int base = warp > 0 ? smem_warp[warp - 1] : 0;
  *total = smem_warp[NT / 32 - 1];
  block_sync<NT>();
  return base + x - v;
}

// Block-wide bitonic sort of two arrays of n2 (a power of two, >= 2) 32-bit
// keys in shared memory, both descending, side by side: log2(n2)(log2(n2)+1)/2
// compare-exchange stages, one barrier each for both arrays.
template <int NT>
__device__ void block_sort2_desc_u32(uint32_t* a, uint32_t* b, int n2) {
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (n2 >> 1); t += NT) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool desc = (i & size) == 0;
        const uint32_t x = a[i], y = a[j], u = b[i], v = b[j];
        if (desc ? (x < y) : (x > y)) {
          a[i] = y;
          a[j] = x;
        }
        if (desc ? (u < v) : (u > v)) {
          b[i] = v;
          b[j] = u;
        }
      }
      block_sync<NT>();
    }
  }
}

constexpr int kRankTopkMax = 64;  // rank-count top-k up to this many candidates

// Block-wide top-k selection over n keys (keys[i] = score_key(score), entries
// in increasing index order).  Marks keep[i] = 1 for exactly min(k, n)
// entries: all keys above the k-th largest key, plus the lowest-index entries
// equal to it (ties to the lower index, selection.py:77-88).  Radix select
// over the differing digits of 8 bits.  smem: 256 ints hist + 40 ints scratch.
template <int NT>
__device__ void block_topk_mark(const uint64_t* keys, int n, int k, int* keep, int* s_hist,
                                int* s_scratch) {
  if (k >= n) {
    for (int i = threadIdx.x; i < n; i += NT) keep[i] = 1;
    block_sync<NT>();
    return;
  }
  if (k <= 0) {
    for (int i = threadIdx.x; i < n; i += NT) keep[i] = 0;
    block_sync<NT>();
    return;
  }
  if (n <= kRankTopkMax) {
    // tiny candidate sets: keep[i] = rank_i < k, rank_i = #{j: key_j > key_i,
    // or equal and j < i} (the stable argsort order, ties to the lower index)
    for (int i = threadIdx.x; i < n; i += NT) {
      const uint64_t ki = keys[i];
      int rank = 0;
#pragma unroll 4
      for (int j = 0; j < n; ++j) {
        const uint64_t kj = keys[j];
        rank += (kj > ki || (kj == ki && j < i)) ? 1 : 0;
      }
      keep[i] = rank < k ? 1 : 0;
    }
    block_sync<NT>();
    return;
  }
  // Radix select.  Digits above the first byte where the smallest and largest
  // key differ are common to every key and skipped; histogram increments are
  // warp-aggregated (match.any), so equal digits do not serialise on one bin.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t kmin = ~0ull, kmax = 0ull;
  for (int i = threadIdx.x; i < n; i += NT) {
    const uint64_t x = keys[i];
    kmin = x < kmin ? x : kmin;
    kmax = x > kmax ? x : kmax;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
    kmin = a < kmin ? a : kmin;
    kmax = b > kmax ? b : kmax;
  }
  uint64_t* s_mm = reinterpret_cast<uint64_t*>(s_hist);  // [NT/32][2] (hist is reset below)
  if (lane == 0) {
    s_mm[2 * warp] = kmin;
    s_mm[2 * warp + 1] = kmax;
  }
  block_sync<NT>();
  uint64_t gmin = s_mm[0], gmax = s_mm[1];
  for (int w = 1; w < NT / 32; ++w) {
    gmin = s_mm[2 * w] < gmin ? s_mm[2 * w] : gmin;
    gmax = s_mm[2 * w + 1] > gmax ? s_mm[2 * w + 1] : gmax;
  }
  block_sync<NT>();
  const uint64_t diff = gmin ^ gmax;
  if (diff == 0) {  // every key equal: the k lowest indices
    for (int i = threadIdx.x; i < n; i += NT) keep[i] = i < k ? 1 : 0;
    block_sync<NT>();
    return;
  }
  const int top_shift = ((63 - __clzll((long long)diff)) / 8) * 8;
  uint64_t mask = top_shift == 56 ? 0ull : ~0ull << (top_shift + 8);
  uint64_t prefix = gmax & mask;
  int kk = k;  // how many still to take among keys matching prefix
  bool bin_taken = false;  // early exit: the k-th key's bin holds exactly kk keys
  for (int shift = top_shift; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += NT) s_hist[b] = 0;
    block_sync<NT>();
    for (int i0 = 0; i0 < n; i0 += NT) {
      const int i = i0 + threadIdx.x;
      const uint64_t key = i < n ? keys[i] : 0ull;
      const bool in = i < n && (key & mask) == prefix;
      const unsigned active = __ballot_sync(0xffffffffu, in);
      if (in) {
        const int digit = (int)((key >> shift) & 255);
        const unsigned peers = __match_any_sync(active, digit);
        if (lane == __ffs(peers) - 1) atomicAdd(&s_hist[digit], __popc(peers));
      }
    }
    block_sync<NT>();
    if (threadIdx.x < 32) {
      // lane l owns bins [255-8l-7, 255-8l] (descending digit order)
      int c[8];
      int tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = s_hist[255 - (lane * 8 + j)];
        tot += c[j];
      }
      int incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int excl = incl - tot;  // count of keys in higher digits (owned by lower lanes)
      // find digit where cumulative count reaches kk
      int found_digit = -1, above = 0;
      if (excl < kk && incl >= kk) {
        int run = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (found_digit < 0) {
            if (run + c[j] >= kk) {
              found_digit = 255 - (lane * 8 + j);
              above = run;
            } else {
              run += c[j];
            }
          }
        }
        s_scratch[0] = found_digit;
        s_scratch[1] = above;
        s_scratch[2] = s_hist[found_digit];
      }
    }
    block_sync<NT>();
    const int digit = s_scratch[0];
    kk -= s_scratch[1];
    const int in_bin = s_scratch[2];
    prefix |= ((uint64_t)digit) << shift;
    mask |= 0xFFull << shift;
    block_sync<NT>();
    if (in_bin == kk) {  // every key of the bin is kept: no lower digits needed
      bin_taken = true;
      break;
    }
  }
  if (bin_taken) {
    for (int i = threadIdx.x; i < n; i += NT) keep[i] = (keys[i] & mask) >= prefix ? 1 : 0;
    block_sync<NT>();
    return;
  }
  // prefix == k-th largest key T; take all keys > T and the first kk keys == T.
  const uint64_t T = prefix;
  int taken_eq = 0;
  for (int base = 0; base < n; base += NT) {
    int i = base + threadIdx.x;
    uint64_t key = i < n ? keys[i] : 0ull;
    int eq = (i < n && key == T) ? 1 : 0;
    int tot;
    int pos = block_exclusive_scan<NT>(eq, s_scratch + 8, &tot);
    if (i < n) keep[i] = (key > T) || (eq && (taken_eq + pos) < kk);
    taken_eq += tot;
  }
  block_sync<NT>();
}

// Working set of slot s from its sorted semantic list + window + sinks, then
// gathered through the page table into the block table (selection.py:126-140,
// kv_store.py:156-166).  Sorted output falls out of the region structure:
// [0, ns) sinks | semantic in [ns, w0) | [max(w0, ns), n) window.
template <int NT>
__device__ void block_build_ws(const ChessState& st, int s, int* s_scratch) {
  const ChessDims& d = st.d;
  const int n = st.num_pages[s];
  const int ns = min(st.sink_count[s], n);
  const int w0 = max(0, n - d.window_pages);
  const int c0 = max(w0, ns);
  const int32_t* sem = st.semantic + (int64_t)s * d.max_pages;
  // sem is sorted: lo = #entries < ns, hi = max(lo, #entries < w0), counted
  // in parallel (one round of loads instead of two dependent binary searches)
  const int nsem = st.n_semantic[s];
  int c_ns = 0, c_w0 = 0;
  for (int i = threadIdx.x; i < nsem; i += NT) {
    const int v = sem[i];
    c_ns += v < ns ? 1 : 0;
    c_w0 += v < w0 ? 1 : 0;
  }
  int t_ns, t_w0;
  block_exclusive_scan<NT>(c_ns, s_scratch, &t_ns);
  block_exclusive_scan<NT>(c_w0, s_scratch, &t_w0);
  const int lo = t_ns, hi = max(t_ns, t_w0);
  int total = ns + (hi - lo) + (n - c0);
  const int cap = d.max_ws;
  int32_t* wl = st.ws_logical + (int64_t)s * cap;
  int32_t* bt = st.block_table + (int64_t)s * cap;
  int8_t* pv = st.ws_prov + (int64_t)s * cap;
  const int32_t* pt = st.page_table + (int64_t)s * d.max_pages;
  for (int i = threadIdx.x; i < total && i < cap; i += NT) {
    int lp;
    int8_t tag;
    if (i < ns) {
      lp = i;
      tag = CHESS_PROV_SINK;
    } else if (i < ns + (hi - lo)) {
      lp = sem[lo + i - ns];
      tag = CHESS_PROV_SEMANTIC;
    } else {
      lp = c0 + (i - ns - (hi - lo));
      tag = CHESS_PROV_WINDOW;
    }
    wl[i] = lp;
    bt[i] = pt[lp];
    pv[i] = tag;
  }
  if (threadIdx.x == 0) st.ws_len[s] = min(total, cap);
  block_sync<NT>();
}

// Ordered compaction: out[pos] = idx_of(i) for keep[i] != 0, i ascending.
template <int NT, typename F>
__device__ int block_compact(const int* keep, int n, int* out, int* s_scratch, F idx_of) {
  int count = 0;
  for (int base = 0; base < n; base += NT) {
    int i = base + threadIdx.x;
    int f = (i < n && keep[i]) ? 1 : 0;
    int tot;
    int pos = block_exclusive_scan<NT>(f, s_scratch, &tot);
    if (f) out[count + pos] = idx_of(i);
    count += tot;
  }
  return count;
}

}  // namespace chess
