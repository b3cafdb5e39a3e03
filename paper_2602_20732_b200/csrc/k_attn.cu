// k_attn.cu — K4 sparse paged decode attention over the CHESS block table.
//
// Not present in the reference: pagesel only counts attention work
// (simulate.py:186, B*2*|WS|*B*D).  The paper runs FlashInfer's paged decode
// over the reconstructed context; oracle restated in
// oracle/attention.py (fp64 softmax(q K^T * scale) V over the working set in
// increasing logical order; rows >= fill never contribute).
//
// B200 design — HBM-bound, one persistent CTA per SM:
//  * work list = every (slot, kv head, working-set page) of the layer, laid
//    out segment by segment (segment = one (slot, kv head)).  Three modes:
//    cluster-merge (segments * 2 <= SMs: each segment split over a 2- or
//    4-CTA thread-block cluster, peer states pushed into the leader's smem
//    with st.async); piece (segments <= CTAs: k = floor(G/segments) pieces
//    of >= 4 pages, no merge when k = 1 — cfg3); stream-K (more segments,
//    two CTAs per SM: CTA c owns pages [c*N/G, (c+1)*N/G), split segments
//    merged by the last CTA);
//  * the last warp is the TMA producer: block-table ids of 32 pages come from
//    one coalesced load (prefetched a batch ahead); pages go out in runs of
//    3 whose 4-D tensor loads (128B swizzle, one box per K or V tile) are
//    issued by lanes in parallel into an S-stage ring of K+V page tiles; each
//    piece's GQA q rows go through a 2-slot q ring; the first run is issued
//    before griddepcontrol.wait so it overlaps the previous kernel;
//  * 4 consumer warps take pages round-robin: S^T = K q^T and O^T += V^T P^T
//    with mma.sync m16n8k16 (tokens as M; P^T via movmatrix, never in smem),
//    online softmax per head in registers;
//  * piece states are merged asynchronously by the last consumer warp to
//    arrive (warp order); a split segment is merged by the last CTA to finish
//    it (atomic counter), in CTA order — deterministic.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"

namespace chess {

namespace {

// Consumer warps per CTA (build-time knob) and CTAs per SM (CPS, a template
// parameter chosen per launch).  Measured on B200 (tools/attn_micro.py,
// graph-replayed, profiles/r01/attn_micro/): 4 consumers x 1 CTA (13-stage
// ring) 19.1 us at cfg3 vs 19.8 with 8 consumers.  Two co-resident CTAs per
// SM (6-stage rings) lose when segments <= SMs (cfg3 19.6 us, cfg5 17.5 vs
// 14.5) but win in the stream-K regime (batch x kv_heads > SMs: cfg4 48.3 vs
// 51.2 us, b=32 32.6 vs 36.4): layer l+1's CTAs start in the freed half of
// each SM while layer l drains.
#ifndef CHESS_ATTN_CONSUMERS
#define CHESS_ATTN_CONSUMERS 4
#endif
// Pages per producer TMA run (<= 8: 4 lanes per page).  A run is issued only
// once all its stages are free, so long runs make the producer wait for the
// slowest consumer; measured (profiles/r01/attn_micro/sweep_producer_run.txt):
// 8 -> 3 pages: cfg3 19.0 -> 18.25 us, cfg5 14.5 -> 13.0 us, cfg4 unchanged;
// 1 page is slower (21.3 us).
#ifndef CHESS_ATTN_RUN
#define CHESS_ATTN_RUN 3
#endif
// q fragments: when a cluster-mode CTA's whole piece fits in the ring, its
// consumers read q from global right after their own griddepcontrol.wait
// (b=1 layer 4.25 -> 3.8 us).  Otherwise the producer's 2-slot smem q ring
// stays: it also holds the producer's K/V run-ahead behind the PDL wait
// (direct q for long pieces: cfg3 18.3 -> 20.4 us, cfg5 13.0 -> 13.8 us;
// profiles/r01/attn_micro/sweep_qdirect.txt).
#ifndef CHESS_ATTN_QDIRECT
#define CHESS_ATTN_QDIRECT 1
#endif
constexpr int kConsumers = CHESS_ATTN_CONSUMERS;
constexpr int kMaxCtasPerSm = 2;
constexpr int kAttnMaxBatch = 256;  // per-slot tables live in smem
constexpr int kMinPiece = 4;  // piece mode: pages per piece >= 4 (bounds the merge fan-in)
constexpr int kThreads = (kConsumers + 1) * 32;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
// per-CTA dynamic smem budget at CPS CTAs per SM, minus reserved + static smem
#ifndef CHESS_ATTN_SMEM_KB  // experiment knob: cap the per-CTA budget (co-residency studies)
#define CHESS_ATTN_SMEM_KB 228
#endif
__host__ __device__ constexpr int smem_budget(int cps) {
  return (cps == 1 && CHESS_ATTN_SMEM_KB < 228 ? CHESS_ATTN_SMEM_KB : 228) * 1024 / cps - 1024 - 256;
}

struct AttnArgs {
  const __nv_bfloat16* q;
  int64_t q_stride;
  __nv_bfloat16* out;
  int64_t out_stride;
  float* lse;
  float scale_log2;  // softmax_scale * log2(e)
  int layer;
  int cl;    // cluster-merge mode: CTAs per segment (= cluster size), 0 = off
  int prefetch;  // pages past the first run prefetched into L2 before the PDL wait
  // Head-shard output gather over peer memory (chess_sparse_decode_gather):
  // every output row is also stored at the same offset from peer_out[p]
  // (this rank's block in peer p's region, NVLink stores).
  __nv_bfloat16* peer_out[kMaxPeers - 1];
  int n_peer;
  int early;  // 1: the previous kernel on the stream is a K4 (CHESS_ATTN_AFTER_DECODE), which
              // writes none of the state the prologue reads, so the prologue and the first
              // K/V loads may run before griddepcontrol.wait; 0: wait first (e.g. after an
              // append, which writes the tail row, tail_fill and the block table)
  int mode;  // debug (CHESS_ATTN_MODE): 0 normal, 1 loads only (no math), 2 math only (no K/V loads), 5 exit at entry, 6 exit after the prologue, 7 force stream-K, 8 no PDL wait (timing only: ignores the previous kernel)
  int next_pf;  // pages of the CTA's range prefetched into L2 for layer + 1 once its own loads are issued
  // (New fields go here, at the end: inserting next_pf before peer_out moved
  // the parameter offsets and changed the cluster instance's code generation,
  // 178 -> 167 registers, cfg2 K4 3.1 -> 3.4 us; A/B in profiles/r02/k4_next_layer_prefetch.txt.)
};

// one bf16 pair of an output row, to this rank's buffer and (PEERS: the
// head-shard gather instance of K4) every peer's.  A compile-time switch: the
// predicated peer stores kept their addresses live across the unrolled
// epilogue (+10 registers in the cluster instance, 0.3-2.8% per step) even
// with no peers.  Constant indices only: a runtime index into the
// kernel-parameter array would copy AttnArgs to the local stack.
template <bool PEERS>
__device__ __forceinline__ void out_pair(const AttnArgs& a, __nv_bfloat16* orow, float x, float y) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(x, y);
  *reinterpret_cast<__nv_bfloat162*>(orow) = v;
  if constexpr (PEERS) {
    const int64_t off = orow - a.out;
#pragma unroll
    for (int p = 0; p < kMaxPeers - 1; ++p)
      if (p < a.n_peer) *reinterpret_cast<__nv_bfloat162*>(a.peer_out[p] + off) = v;
  }
}

// Debug timeline (read by chess_debug_attn_trace): per CTA globaltimer stamps
// {entry, prologue done, first page ready, consumers done, exit}, kept for
// the last launch of each layer parity.
// Stamps go to shared memory and are flushed by the last consumer warp at
// exit, so they never sit in front of the kernel's release fences.
__device__ unsigned long long g_attn_trace[2][256][16];
__shared__ unsigned long long s_trace[16];
__shared__ int s_trace_warps;
__device__ __forceinline__ void trace(int which, int /*layer*/) {
  if (kTrace && threadIdx.x == 0) s_trace[which] = global_ns();
}
__device__ __forceinline__ void trace_max(int which) {
  if (kTrace) atomicMax(&s_trace[which], (unsigned long long)global_ns());
}

// Cluster size cap (inbox slots = cap - 1).  Measured (profiles/r01/attn_micro/
// sweep_cluster_cap.txt): b=1 ws16 4.3 us at 4 vs 5.3 at 8 (2-page pieces spend
// more on merging than they save on streaming); b=4 8.6 at 4 vs 8.3 at 2.
#ifndef CHESS_ATTN_CLMAX_CT
#define CHESS_ATTN_CLMAX_CT 4
#endif
constexpr int kMaxCluster = CHESS_ATTN_CLMAX_CT;  // compile-time knob (build.py --define=CHESS_ATTN_CLMAX_CT=8)

// XC: cluster-merge variant (piece mode with one segment per thread-block
// cluster): the leader CTA owns an inbox for the other CTAs' piece states.
template <int HD, int GQ, int B, bool XC = false, int CPS = 1>
struct Cfg {
  static constexpr int kCB = HD / 64;                  // 128-byte column blocks
  static constexpr int kPageBytes = B * HD * 2;        // K (or V) bytes of a page
  static constexpr int kStageBytes = 2 * kPageBytes;
  static constexpr int kRow = HD + 4;                  // state row: o[HD], m, l, pad
  static constexpr int kStateBytes = kConsumers * GQ * kRow * 4;
  static constexpr int kQBytes = GQ * HD * 2;          // one GQA group's q rows (bf16)
  static constexpr int kQSlots = 2;
  static constexpr int kTables = (kAttnMaxBatch + 1) * 4 * 4;
  static constexpr int kXBytes = XC ? (kMaxCluster - 1) * GQ * kRow * 4 : 0;  // leader's inbox
  static constexpr int kMisc = kTables + 64 * 8 + 64 + 1024;  // tables, barriers, counters, align
  static constexpr int kStagesRaw =
      (smem_budget(CPS) - kStateBytes - kQSlots * kQBytes - kXBytes - kMisc) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 32 ? 32 : kStagesRaw;
  static constexpr int kMT = B / 16;                   // QK m-tiles (16 tokens each)
  static constexpr int kKS = HD / 16;                  // QK k-steps over d
  static constexpr int kDT = HD / 16;                  // PV m-tiles (16 d each)
  static constexpr int kPK = B / 16;                   // PV k-steps (16 tokens each)
  static constexpr int kEPL = GQ * HD / 32;            // merge: state elements per lane
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + kStateBytes +
                                  kQSlots * kQBytes + kXBytes + (2 * kStages + 2 * kQSlots + 3) * 8 +
                                  64 + kTables;
  static_assert(kStages >= 4, "ring too shallow");
  static_assert(GQ <= 8, "one GQA group per n8 tile");
  static_assert(kEPL >= 2 && kEPL % 2 == 0 && HD % kEPL == 0, "merge lane mapping");
};

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
// 8x8 b16 register transpose across the warp
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// L2 prefetch of one tensor box (no shared-memory destination, no barrier)
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// 128B-swizzled address of 16-byte chunk `chunk` (0..HD/8-1) of page row `row`
// inside one K or V page tile laid out as [HD/64 column blocks][B rows][128 B].
template <int B>
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + (uint32_t)((chunk >> 3) * (B * 128) + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
}

// named barrier 2 over the consumer warps only
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 2, %0;" ::"n"(kConsumers * 32) : "memory");
}

// The producer's "pages issued" counter: atomic acquire / release on shared
// memory (an atomic is never a data race, so compute-sanitizer racecheck has
// nothing to report on the handoff).
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("atom.acquire.cta.shared::cta.or.b32 %0, [%1], 0;" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  int old;
  asm volatile("atom.release.cta.shared::cta.exch.b32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  (void)old;
}

// Consumer math layout ("tokens as M"): per page, S^T = K q^T with the
// page's tokens as the MMA M dimension (16 per tile), the GQA group's q heads
// as N (8, padded) and d as K; then O^T += V^T P^T with d as M, heads as N
// and tokens as K.  The S^T accumulator of an 8-token block is exactly the
// P^T B-fragment after one movmatrix transpose, so P never touches smem.
// Per 32-token page: 2x8 + 8x2 = 32 HMMA (half of the heads-as-M layout).
//
// Synchronisation: consumers block only on data.
//  * K/V ring: full/empty mbarriers per stage.  A stage is shared by
//    different consumer warps, so before waiting on page j's full barrier a
//    consumer checks the producer's `issued` counter (> j): page j issued
//    implies page j-S was consumed, so the parity test cannot alias an older
//    phase of the stage.
//  * q ring (2 slots): the producer bulk-copies each piece's GQA q rows next
//    to the piece's first page; consumers release a slot after reading it.
//  * piece states: each consumer warp drops its (m, l, o) into a state slot
//    and moves on; the last warp to arrive (smem atomic) merges the 8 states
//    in warp order and writes the output, or the split-segment partial and the
//    cross-CTA combine.  The slot is reopened via `st_next`.
//
// Cluster-merge variant (XC, args.cl > 1; segments * cl <= SMs): segment
// (slot, kv head) number blockIdx.x / cl is split into cl near-equal pieces,
// one per CTA of a thread-block cluster.  Each non-leader CTA pushes its
// merged piece state into the leader's shared-memory inbox over DSMEM and
// arrives on the leader's mbarrier (release.cluster); the leader merges the
// states in cluster-rank order.  This replaces the split-segment path's
// global partials + fences + atomics (~3 us of round trips) on small batches.
template <int HD, int GQ, int B, bool XC, int CPS, bool PEERS>
__global__ void __launch_bounds__(kThreads, CPS)
    sparse_decode_kernel(ChessState st, Workspace ws, AttnArgs args,
                         const __grid_constant__ CUtensorMap kmap,
                         const __grid_constant__ CUtensorMap vmap) {
  using C = Cfg<HD, GQ, B, XC, CPS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  float* stv = reinterpret_cast<float*>(ring + (size_t)C::kStages * C::kStageBytes);
  uint8_t* qbuf = reinterpret_cast<uint8_t*>(stv + kConsumers * GQ * C::kRow);
  float* xst = reinterpret_cast<float*>(qbuf + C::kQSlots * C::kQBytes);  // [cl-1][GQ][kRow] (XC)
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xst) + C::kXBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* qfull = empty + C::kStages;
  uint64_t* qempty = qfull + C::kQSlots;
  uint64_t* xbar = qempty + C::kQSlots;                    // leader's inbox barrier (XC)
  uint64_t* stbar = xbar + 1;                               // piece states written (kConsumers arrivals)
  uint64_t* slotfree = stbar + 1;                            // piece states read by the merger (1 arrival)
  int* ctr = reinterpret_cast<int*>(slotfree + 1);           // [0] issued, [1] st_cnt
  int* prefix = ctr + 16;                                   // [nb + 1] pages before slot s
  int* s_np = prefix + kAttnMaxBatch + 1;                   // [nb] pages per segment of slot s
  int* s_fill = s_np + kAttnMaxBatch;                        // [nb] valid rows of the last page
  int* ppre = s_fill + kAttnMaxBatch;                        // [nb + 1] pieces before slot s (piece mode)
  const ChessDims& d = st.d;
  const int H = d.kv_heads;
  const int nb = d.batch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == kConsumers * 32) {
    prefetch_tmap(&kmap);
    prefetch_tmap(&vmap);
  }
  trace(0, args.layer);
  if (kTrace && threadIdx.x == 0) {
#pragma unroll
    for (int i = 1; i < 16; ++i) s_trace[i] = 0;
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    s_trace[15] = smid;  // which SM ran this CTA (per-CTA studies, tools/attn_micro.py)
    s_trace_warps = 0;
    if (blockIdx.x < 256)
      for (int i = 0; i < 16; ++i) g_attn_trace[args.layer & 1][blockIdx.x][i] = 0;
  }
  if (args.mode == 5) return;  // debug: launch overhead only
  // After another K4 (args.early), everything up to the q load reads state
  // that was final before the previous kernel started (KV pool, block table,
  // ws_len, fill), so the prologue, the block-table fetch and the first K/V
  // TMA loads overlap the previous kernel's tail under PDL; griddepcontrol.wait
  // guards the q reads and every write (out, lse, split partials, counters).
  // Any other predecessor (an append writes the token's K/V row, tail_fill and
  // the block table) may not have made its writes visible before the wait, so
  // the kernel waits before reading anything.
  if (!args.early && args.mode != 8) pdl_wait();
  // pages per segment: np = ws_len - 1 + (fill > 0); prefix over slots (x H)
  if (warp == 0) {
    int run = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int s = b0 + lane;
      int np = 0, fill = 0;
      if (s < nb) {
        const int wl = st.ws_len[s];
        fill = min(st.tail_fill[s], B);
        if (wl > 0) np = wl - 1 + (fill > 0 ? 1 : 0);
        s_np[s] = np;
        s_fill[s] = fill > 0 ? fill : B;
      }
      const int x = np * H;
      int incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (s < nb) prefix[s] = run + incl - x;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) prefix[nb] = run;
    // piece mode (segments <= CTAs): every segment of np pages is split into
    // k_s = min(k, np) near-equal pieces, k = floor(G / segments), one piece
    // per CTA; piece prefix over slots.
    const int G0 = min((int)gridDim.x, run);
    int nseg = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int s = b0 + lane;
      nseg += __popc(__ballot_sync(0xffffffffu, s < nb && s_np[s] > 0)) * H;
    }
    const int kp = (args.mode != 7 && nseg > 0 && nseg <= G0) ? G0 / nseg : 0;  // 0: stream-K mode
    int prun = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int s = b0 + lane;
      const int x = (s < nb) ? min(kp, (s_np[s] + kMinPiece - 1) / kMinPiece) * H : 0;
      int incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (s < nb) ppre[s] = prun + incl - x;
      prun += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      ppre[nb] = prun;
      ctr[3] = kp;
    }
  } else if (warp == kConsumers && lane == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < C::kQSlots; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], kConsumers);
    }
    if (XC) {
      // inbox: one local arrival + the peers' st.async bytes (o rows, m, l)
      mbar_init(xbar, 1);
      mbar_arrive_expect_tx(xbar, (uint32_t)(args.cl - 1) * (uint32_t)(GQ * (HD + 2) * 4));
    }
    ctr[0] = 0;
    mbar_init(stbar, kConsumers * 32);
    mbar_init(slotfree, 32);
    ctr[1] = 0;
    fence_barrier_init();
  }
  __syncthreads();
  // the leader's inbox barrier is initialised before any peer can arrive on it
  if (XC) cluster_sync_all();
  trace(1, args.layer);
  pdl_launch_dependents();

  if (args.mode == 6) return;  // debug: launch + prologue
  const int N = prefix[nb];
  const int kp = ctr[3];
  // stream-K: CTA c owns pages [c*N/G, (c+1)*N/G), G = min(grid, N).
  // piece mode: CTA c owns piece c of the segment-aligned split.
  const int G = kp > 0 ? ppre[nb] : min((int)gridDim.x, N);
  const int c = blockIdx.x;
  int u_begin, u_end;
  int cs = 0, ch = 0;  // XC: this cluster's segment
  if (XC) {
    const int seg = c / args.cl, cr = c - seg * args.cl;
    cs = seg / H;
    ch = seg - cs * H;
    if (cs >= nb) return;
    const int np = s_np[cs];
    if (np == 0) return;  // the whole cluster has nothing to do
    const int base = prefix[cs] + ch * np;
    u_begin = base + (int)((int64_t)cr * np / args.cl);
    u_end = base + (int)((int64_t)(cr + 1) * np / args.cl);
  } else if (c >= G) {
    return;
  } else if (kp > 0) {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (ppre[mid] <= c) lo = mid; else hi = mid;
    }
    const int np = s_np[lo], ks = min(kp, (np + kMinPiece - 1) / kMinPiece);
    const int r = c - ppre[lo], h = r / ks, idx = r - h * ks;
    const int base = prefix[lo] + h * np;
    u_begin = base + (int)((int64_t)idx * np / ks);
    u_end = base + (int)((int64_t)(idx + 1) * np / ks);
  } else {
    u_begin = (int)((int64_t)c * N / G);
    u_end = (int)((int64_t)(c + 1) * N / G);
  }

  const bool qdirect = CHESS_ATTN_QDIRECT && XC && (u_end - u_begin) <= C::kStages;
  // global page index u -> (slot, head, page within segment)
  auto locate = [&](int u, int& s, int& h, int& p) {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (prefix[mid] <= u) lo = mid; else hi = mid;
    }
    s = lo;
    const int r = u - prefix[lo];
    h = r / s_np[lo];
    p = r - h * s_np[lo];
  };

  if (warp == kConsumers) {
    // ===================== TMA producer =====================
    const int n = u_end - u_begin;
    // lane -> page base+lane: first pool row of (page, head); piece-start tag
    auto fetch = [&](int base, int& row0, int& tag) {
      row0 = 0;
      tag = -1;
      if (base + lane < n) {
        int s, h, p;
        locate(u_begin + base + lane, s, h, p);
        const int pid = __ldg(st.block_table + (int64_t)s * d.max_ws + p);
        row0 = (pid * H + h) * B;
        if (p == 0 || base + lane == 0) tag = s * 256 + h;
      }
    };
    int cur_row, cur_tag, nxt_row = 0, nxt_tag = -1;
    fetch(0, cur_row, cur_tag);
    int qk = 0;
    for (int base = 0; base < n; base += 32) {
      if (base + 32 < n) fetch(base + 32, nxt_row, nxt_tag);
      const int cnt = min(32, n - base);
      // Pages go out in runs of <= 8 that never cross a piece start; a run
      // that begins a piece first sends that piece's q rows (q ring order =
      // page order, so the 2-slot q ring cannot deadlock).  Within a run,
      // lane 4p+b issues box b of page p: the TMA issues run in parallel.
      const uint32_t starts = __ballot_sync(0xffffffffu, cur_tag >= 0);
      constexpr int kRun = C::kStages < CHESS_ATTN_RUN ? C::kStages : CHESS_ATTN_RUN;  // distinct stages within a run
      for (int c0 = 0; c0 < cnt;) {
        const uint32_t later = starts & ~((2u << c0) - 1u);  // starts after c0
        const int nxt_start = later ? __ffs(later) - 1 : 32;
        const int c1 = min(min(c0 + kRun, cnt), nxt_start);
        const bool first_run = qk == 0 && base == 0 && c0 == 0;
        auto issue_q = [&](int at) {
          const int tag = __shfl_sync(0xffffffffu, cur_tag, at);
          if (qk == 0 && args.prefetch > 0 && args.mode != 2) {
            // Before waiting on the previous grid, pull this CTA's next pages
            // (after the first run, which is already in flight) into L2, so
            // HBM streams through the previous layer's drain and this
            // layer's ring refills hit L2.  Rows of pages 0..31 are in
            // cur_row, 32..63 in nxt_row (fetched a batch ahead).
            const int lim = min(n, kRun + args.prefetch);
            if (lane >= kRun && lane < lim) {
              tma_prefetch_4d(&kmap, 0, cur_row, 0, args.layer);
              tma_prefetch_4d(&vmap, 0, cur_row, 0, args.layer);
            }
            if (32 + lane < lim) {
              tma_prefetch_4d(&kmap, 0, nxt_row, 0, args.layer);
              tma_prefetch_4d(&vmap, 0, nxt_row, 0, args.layer);
            }
          }
          if (lane == 0) {
            if (qk == 0 && args.mode != 8) pdl_wait();
            const int qs = qk & 1;
            mbar_wait(&qempty[qs], (uint32_t)(((qk >> 1) & 1) ^ 1));
            mbar_arrive_expect_tx(&qfull[qs], (uint32_t)C::kQBytes);
            const __nv_bfloat16* qsrc = args.q + (int64_t)(tag >> 8) * args.q_stride + (int64_t)(tag & 255) * GQ * HD;
            tma_load_1d(qbuf + qs * C::kQBytes, qsrc, (uint32_t)C::kQBytes, &qfull[qs]);
          }
          ++qk;
        };
        // the kernel's first q load waits for the previous grid (PDL); the
        // first run of K/V pages is issued before it so it overlaps that wait
        if (!qdirect && ((starts >> c0) & 1u) && !first_run) issue_q(c0);
        const int pg = lane >> 2, bx = lane & 3;
        const int i = c0 + pg;
        const int row0 = __shfl_sync(0xffffffffu, cur_row, min(i, 31));
        const bool live = i < c1;
        const int j = base + i;
        const int stg = j % C::kStages;
        const uint32_t ph = (uint32_t)((j / C::kStages) & 1);
        if (live && bx == 0) {
          mbar_wait(&empty[stg], ph ^ 1u);
          if (args.mode == 2) mbar_arrive(&full[stg]);
          else mbar_arrive_expect_tx(&full[stg], (uint32_t)C::kStageBytes);
        }
        __syncwarp();
        if (live && args.mode != 2 && bx < 2) {  // lane 4p: K tile, 4p+1: V tile
          const uint32_t dst = smem_u32(ring + (size_t)stg * C::kStageBytes) + bx * C::kPageBytes;
          tma_load_4d(dst, bx ? &vmap : &kmap, 0, row0, 0, args.layer, smem_u32(&full[stg]));
        }
        __syncwarp();
        if (lane == 0) st_release_cta(&ctr[0], base + c1);
        if (!qdirect && first_run) issue_q(0);
        c0 = c1;
      }
      cur_row = nxt_row;
      cur_tag = nxt_tag;
    }
    // Every layer's launch walks the same block table with the same work
    // split, so this CTA's first pages are the next layer's first pages on the
    // same position: once this layer's loads are all issued (the ring only
    // drains from here), pull the next layer's first tiles into L2 so that
    // layer's start hits L2 instead of HBM (an L2 hint: no data dependency).
    if constexpr (!XC) {  // piece mode only (the work split of the cluster instance differs)
      if (args.next_pf > 0 && args.layer + 1 < d.layers && n > 0) {
        int row0, tag;
        fetch(0, row0, tag);
        if (lane < min(args.next_pf, min(n, 32))) {
          tma_prefetch_4d(&kmap, 0, row0, 0, args.layer + 1);
          tma_prefetch_4d(&vmap, 0, row0, 0, args.layer + 1);
        }
      }
    }
    return;
  }

  // ===================== consumers =====================
  const int g = lane >> 2, t = lane & 3;
  const int lr = lane & 7, lm = lane >> 3;  // ldmatrix: row in matrix, matrix index
  int u = u_begin, k = 0;
  bool once = XC;  // XC: exactly one piece per CTA, possibly empty (np < cl)
  while (u < u_end || once) {
    once = false;
    int s, h, p0;
    if (XC) {
      s = cs;
      h = ch;
      p0 = u - (prefix[s] + h * s_np[s]);
    } else {
      locate(u, s, h, p0);
    }
    const int np = s_np[s];
    const int seg_begin = prefix[s] + h * np;
    const int seg_end = seg_begin + np;
    const int piece_end = min(seg_end, u_end);
    const int piece_n = piece_end - u;
    const int j0 = u - u_begin;  // CTA-local index of the piece's first page
    const int last_fill = s_fill[s];

    // q^T B-fragments from the q ring: b[ks][0] = q[g][16ks+2t..], b[ks][1] = q[g][16ks+8+2t..]
    uint32_t qb[C::kKS][2];
    if (qdirect && piece_n > 0) {
      if (k == 0 && args.mode != 8) pdl_wait();  // q comes from the previous grid
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(
          args.q + (int64_t)s * args.q_stride + ((int64_t)h * GQ + (g < GQ ? g : 0)) * HD);
#pragma unroll
      for (int ks = 0; ks < C::kKS; ++ks) {
        qb[ks][0] = g < GQ ? __ldg(qrow + (ks * 16 + 2 * t) / 2) : 0u;
        qb[ks][1] = g < GQ ? __ldg(qrow + (ks * 16 + 8 + 2 * t) / 2) : 0u;
      }
    } else if (piece_n > 0) {
      const int qs = k & 1;
      mbar_wait(&qfull[qs], (uint32_t)((k >> 1) & 1));
      const uint8_t* qrow = qbuf + qs * C::kQBytes + g * HD * 2;
#pragma unroll
      for (int ks = 0; ks < C::kKS; ++ks) {
        if (g < GQ) {
          qb[ks][0] = *reinterpret_cast<const uint32_t*>(qrow + (ks * 16 + 2 * t) * 2);
          qb[ks][1] = *reinterpret_cast<const uint32_t*>(qrow + (ks * 16 + 8 + 2 * t) * 2);
        } else {
          qb[ks][0] = qb[ks][1] = 0u;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
    }
    // O^T accumulators: o[dt] = rows d 16dt+g (+8), cols heads 2t, 2t+1
    float o[C::kDT][4];
#pragma unroll
    for (int dt = 0; dt < C::kDT; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};  // heads 2t, 2t+1

    for (int i = warp; i < piece_n; i += kConsumers) {
      const int j = j0 + i;
      const int valid = (p0 + i == np - 1) ? last_fill : B;
      const int stage = j % C::kStages;
      const uint32_t phase = (uint32_t)((j / C::kStages) & 1);
      if (lane == 0) {
        while (ld_acquire_cta(&ctr[0]) <= j) {
        }
      }
      __syncwarp();
      mbar_wait(&full[stage], phase);
      if (j == 0 && warp == 0) {
        trace(2, args.layer);
        if (kTrace && lane == 0) s_trace[8] = clock64();
      }
      const uint32_t kst = smem_u32(ring + (size_t)stage * C::kStageBytes);
      const uint32_t vst = kst + C::kPageBytes;
      if (args.mode != 1) {
        // ---- S^T = K q^T : tokens (M) x heads (N) ----
        float sc[C::kMT][4];
#pragma unroll
        for (int mt = 0; mt < C::kMT; ++mt) sc[mt][0] = sc[mt][1] = sc[mt][2] = sc[mt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < C::kKS; ++ks) {
#pragma unroll
          for (int mt = 0; mt < C::kMT; ++mt) {
            uint32_t a[4];
            ldsm_x4(swz<B>(kst, 16 * mt + lr + 8 * (lm & 1), 2 * ks + (lm >> 1)), a);
            mma_bf16(sc[mt], a, qb[ks][0], qb[ks][1]);
          }
        }
        // ---- online softmax per head (2t, 2t+1) over tokens 16mt + g (+8) ----
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int mt = 0; mt < C::kMT; ++mt) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int tok = 16 * mt + g + 8 * (r >> 1);
            const float x = sc[mt][r] * args.scale_log2;
            sc[mt][r] = (tok < valid && x == x) ? x : -INFINITY;
            mx[r & 1] = fmaxf(mx[r & 1], sc[mt][r]);
          }
        }
        float alpha[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 4));
          mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 8));
          mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 16));
          const float m_new = fmaxf(m_run[e], mx[e]);
          alpha[e] = exp2f(m_run[e] - m_new);
          m_run[e] = m_new;
        }
        float ps[2] = {0.f, 0.f};
#pragma unroll
        for (int mt = 0; mt < C::kMT; ++mt) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            sc[mt][r] = exp2f(sc[mt][r] - m_run[r & 1]);
            ps[r & 1] += sc[mt][r];
          }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          ps[e] += __shfl_xor_sync(0xffffffffu, ps[e], 4);
          ps[e] += __shfl_xor_sync(0xffffffffu, ps[e], 8);
          ps[e] += __shfl_xor_sync(0xffffffffu, ps[e], 16);
          l_run[e] = l_run[e] * alpha[e] + ps[e];
        }
#pragma unroll
        for (int dt = 0; dt < C::kDT; ++dt) {
          o[dt][0] *= alpha[0];
          o[dt][1] *= alpha[1];
          o[dt][2] *= alpha[0];
          o[dt][3] *= alpha[1];
        }
        // ---- O^T += V^T P^T : d (M) x heads (N), tokens as K ----
#pragma unroll
        for (int kk = 0; kk < C::kPK; ++kk) {
          // P^T fragment of tokens 16kk..16kk+15 (b0: +0..7, b1: +8..15)
          const uint32_t pb0 = movm_t(pack_bf16(sc[kk][0], sc[kk][1]));
          const uint32_t pb1 = movm_t(pack_bf16(sc[kk][2], sc[kk][3]));
          // V rows >= valid may hold never-written data: zero this thread's
          // A-fragment halves for those tokens so 0 * garbage cannot poison O.
          uint32_t vm0 = 0xffffffffu, vm1 = 0xffffffffu;
          if (valid < B) {
            const int t0 = 16 * kk + 2 * t;
            vm0 = (t0 < valid ? 0x0000ffffu : 0u) | (t0 + 1 < valid ? 0xffff0000u : 0u);
            vm1 = (t0 + 8 < valid ? 0x0000ffffu : 0u) | (t0 + 9 < valid ? 0xffff0000u : 0u);
          }
#pragma unroll
          for (int dt = 0; dt < C::kDT; ++dt) {
            uint32_t a[4];
            ldsm_x4_t(swz<B>(vst, 16 * kk + lr + 8 * (lm >> 1), 2 * dt + (lm & 1)), a);
            a[0] &= vm0;
            a[1] &= vm0;
            a[2] &= vm1;
            a[3] &= vm1;
            mma_bf16(o[dt], a, pb0, pb1);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
    }
    if (piece_end == u_end && warp == 0) trace(3, args.layer);

    // ---- hand this warp's piece state to the merge slot ----
    if (k == 0 && args.mode != 8) pdl_wait();
    if (k == 0 && lane == 0) trace_max(5);  // debug timeline: last warp past the PDL wait
    const long long ck0 = kTrace ? clock64() : 0;
    // the state slots are free once the previous piece's merger read them
    if (k > 0) mbar_wait(slotfree, (uint32_t)((k - 1) & 1));
    const long long ck1 = kTrace ? clock64() : 0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int hh = 2 * t + e;
      if (hh < GQ) {
        float* pr = stv + (warp * GQ + hh) * C::kRow;
        if (g == 0) {
          pr[HD] = m_run[e];
          pr[HD + 1] = l_run[e];
        }
#pragma unroll
        for (int dt = 0; dt < C::kDT; ++dt) {
          pr[16 * dt + g] = o[dt][e];
          pr[16 * dt + g + 8] = o[dt][2 + e];
        }
      }
    }
    __syncwarp();
    // A CTA whose range is exactly one piece (cluster mode; piece mode with
    // one whole segment per CTA, as cfg3) has every consumer warp here and
    // nothing left to stream: instead of one warp merging all four states,
    // each merges a quarter of the (head, d) elements and writes it (piece
    // mode), or pushes it to the cluster leader (whose warps then finish
    // their quarters over the peers' states).
    const bool one_piece = XC || (u_begin == seg_begin && u_end == seg_end);
    if constexpr (C::kEPL % (2 * kConsumers) == 0) if (one_piece) {
      consumer_sync();
      constexpr int kQ = GQ * HD / kConsumers, kE = kQ / 32;
      const int e0 = warp * kQ + lane * kE;
      const int hh = e0 / HD, el = e0 % HD;
      float M = -INFINITY, L = 0.f, acc[kE];
#pragma unroll
      for (int e = 0; e < kE; ++e) acc[e] = 0.f;
#pragma unroll
      for (int w = 0; w < kConsumers; ++w) M = fmaxf(M, stv[(w * GQ + hh) * C::kRow + HD]);
#pragma unroll
      for (int w = 0; w < kConsumers; ++w) {
        const float* pr = stv + (w * GQ + hh) * C::kRow;
        const float f = pr[HD] == -INFINITY ? 0.f : exp2f(pr[HD] - M);
        L = fmaf(pr[HD + 1], f, L);
#pragma unroll
        for (int e = 0; e < kE; e += 2) {
          const float2 x = *reinterpret_cast<const float2*>(pr + el + e);
          acc[e] = fmaf(x.x, f, acc[e]);
          acc[e + 1] = fmaf(x.y, f, acc[e + 1]);
        }
      }
      const int cr = XC ? c % args.cl : 0;
      if (XC && cr != 0) {
        const uint32_t rx = mapa_shared(smem_u32(xst + ((cr - 1) * GQ + hh) * C::kRow), 0);
        const uint32_t rb = mapa_shared(smem_u32(xbar), 0);
#pragma unroll
        for (int e = 0; e < kE; e += 2) st_async_f32x2(rx + (uint32_t)(el + e) * 4u, acc[e], acc[e + 1], rb);
        if (el == 0) st_async_f32x2(rx + (uint32_t)HD * 4u, M, L, rb);
      } else {
        const int ncl = XC ? args.cl : 1;
        if (XC) mbar_wait_cluster(xbar, 0);
        float Mx = M;
        for (int r = 1; r < ncl; ++r) Mx = fmaxf(Mx, xst[((r - 1) * GQ + hh) * C::kRow + HD]);
        const float f0 = M == -INFINITY ? 0.f : exp2f(M - Mx);
        float Lx = L * f0;
#pragma unroll
        for (int e = 0; e < kE; ++e) acc[e] *= f0;
        for (int r = 1; r < ncl; ++r) {
          const float* pr = xst + ((r - 1) * GQ + hh) * C::kRow;
          const float f = pr[HD] == -INFINITY ? 0.f : exp2f(pr[HD] - Mx);
          Lx = fmaf(pr[HD + 1], f, Lx);
#pragma unroll
          for (int e = 0; e < kE; e += 2) {
            const float2 x = *reinterpret_cast<const float2*>(pr + el + e);
            acc[e] = fmaf(x.x, f, acc[e]);
            acc[e + 1] = fmaf(x.y, f, acc[e + 1]);
          }
        }
        const float inv = 1.f / Lx;
        __nv_bfloat16* orow = args.out + (int64_t)s * args.out_stride + ((int64_t)h * GQ + hh) * HD + el;
#pragma unroll
        for (int e = 0; e < kE; e += 2)
          out_pair<PEERS>(args, orow + e, acc[e] * inv, acc[e + 1] * inv);
        if (args.lse && el == 0) args.lse[(int64_t)s * d.q_heads + h * GQ + hh] = (Mx + log2f(Lx)) * kLn2;
      }
      u = piece_end;
      ++k;
      continue;
    }
    // Piece-state handoff: every warp arrives on stbar (release) after its
    // state stores; the last to arrive (shared counter) merges after waiting
    // on stbar (acquire) and frees the slots through slotfree.  mbarrier
    // phases make the ordering explicit (compute-sanitizer racecheck models
    // them; the earlier fence + atomic handoff it could not see).
    int last = 0;
    mbar_arrive(stbar);  // every lane: its own state stores are released
    if (lane == 0) last = atomicAdd(&ctr[1], 1) == kConsumers - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    const long long ck2 = kTrace ? clock64() : 0;
    if (last) {
      // ---- this warp merges the piece (warp order, deterministic) ----
      mbar_wait(stbar, (uint32_t)(k & 1));
      const int hh = (lane * C::kEPL) / HD, el = (lane * C::kEPL) % HD;
      float M = -INFINITY, L = 0.f, acc[C::kEPL];
#pragma unroll
      for (int e = 0; e < C::kEPL; ++e) acc[e] = 0.f;
#pragma unroll
      for (int w = 0; w < kConsumers; ++w) M = fmaxf(M, stv[(w * GQ + hh) * C::kRow + HD]);
#pragma unroll
      for (int w = 0; w < kConsumers; ++w) {
        const float* pr = stv + (w * GQ + hh) * C::kRow;
        const float f = pr[HD] == -INFINITY ? 0.f : exp2f(pr[HD] - M);
        L = fmaf(pr[HD + 1], f, L);
        if constexpr (C::kEPL % 4 == 0) {
#pragma unroll
          for (int e = 0; e < C::kEPL; e += 4) {
            const float4 x = *reinterpret_cast<const float4*>(pr + el + e);
            acc[e] = fmaf(x.x, f, acc[e]);
            acc[e + 1] = fmaf(x.y, f, acc[e + 1]);
            acc[e + 2] = fmaf(x.z, f, acc[e + 2]);
            acc[e + 3] = fmaf(x.w, f, acc[e + 3]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < C::kEPL; e += 2) {
            const float2 x = *reinterpret_cast<const float2*>(pr + el + e);
            acc[e] = fmaf(x.x, f, acc[e]);
            acc[e + 1] = fmaf(x.y, f, acc[e + 1]);
          }
        }
      }
      // the slot is free again once the states are in registers
      if (lane == 0) atomicExch(&ctr[1], 0);
      mbar_arrive(slotfree);  // every lane of the merger: its reads are done
      if (lane == 0) trace_max(6);
      const long long ck3 = kTrace ? clock64() : 0;
      if (kTrace && lane == 0) {
        s_trace[10] = ck1 - ck0;
        s_trace[11] = ck2 - ck1;
        s_trace[12] = ck3 - ck2;
      }
      const bool whole = seg_begin >= u_begin && seg_end <= u_end;
      const int sg = s * H + h;
      __nv_bfloat16* orow = args.out + (int64_t)s * args.out_stride + ((int64_t)h * GQ + hh) * HD + el;
      float* lse = args.lse ? args.lse + (int64_t)s * d.q_heads + h * GQ + hh : nullptr;
      if (XC) {
        const int cr = c % args.cl;  // == %cluster_ctarank (1-D clusters of consecutive CTAs)
        if (cr != 0) {
          // push (o, m, l) of this piece into the leader's inbox slot cr-1
          // (st.async completes bytes on the leader's inbox mbarrier)
          const uint32_t rx = mapa_shared(smem_u32(xst + ((cr - 1) * GQ + hh) * C::kRow), 0);
          const uint32_t rb = mapa_shared(smem_u32(xbar), 0);
#pragma unroll
          for (int e = 0; e < C::kEPL; e += 2) st_async_f32x2(rx + (uint32_t)(el + e) * 4u, acc[e], acc[e + 1], rb);
          if (el == 0) st_async_f32x2(rx + (uint32_t)HD * 4u, M, L, rb);
          if (kTrace && lane == 0) s_trace[13] = clock64() - ck3;
        } else {
          // leader: own state first, then the peers in cluster-rank order
          mbar_wait_cluster(xbar, 0);
          if (lane == 0) trace_max(7);
          float Mx = M;
          for (int r = 1; r < args.cl; ++r) Mx = fmaxf(Mx, xst[((r - 1) * GQ + hh) * C::kRow + HD]);
          const float f0 = M == -INFINITY ? 0.f : exp2f(M - Mx);
          float Lx = L * f0;
#pragma unroll
          for (int e = 0; e < C::kEPL; ++e) acc[e] *= f0;
          for (int r = 1; r < args.cl; ++r) {
            const float* pr = xst + ((r - 1) * GQ + hh) * C::kRow;
            const float f = pr[HD] == -INFINITY ? 0.f : exp2f(pr[HD] - Mx);
            Lx = fmaf(pr[HD + 1], f, Lx);
#pragma unroll
            for (int e = 0; e < C::kEPL; e += 2) {
              const float2 x = *reinterpret_cast<const float2*>(pr + el + e);
              acc[e] = fmaf(x.x, f, acc[e]);
              acc[e + 1] = fmaf(x.y, f, acc[e + 1]);
            }
          }
          const float inv = 1.f / Lx;
#pragma unroll
          for (int e = 0; e < C::kEPL; e += 2)
            out_pair<PEERS>(args, orow + e, acc[e] * inv, acc[e + 1] * inv);
          if (lse && el == 0) *lse = (Mx + log2f(Lx)) * kLn2;
        }
      } else if (whole) {
        const float inv = 1.f / L;
#pragma unroll
        for (int e = 0; e < C::kEPL; e += 2)
          out_pair<PEERS>(args, orow + e, acc[e] * inv, acc[e + 1] * inv);
        if (lse && el == 0) *lse = (M + log2f(L)) * kLn2;
      } else {
        // split segment: partial (2*cta + which), which = 0 for the CTA's first piece
        const int which = (u == u_begin) ? 0 : 1;
        float* slot = ws.attn_part + ((int64_t)(2 * c + which) * GQ + hh) * C::kRow;
#pragma unroll
        for (int e = 0; e < C::kEPL; ++e) slot[el + e] = acc[e];
        if (el == 0) {
          slot[HD] = M;
          slot[HD + 1] = L;
        }
        int c_first, c_last;
        if (kp > 0) {  // the segment's pieces sit on consecutive CTAs
          const int ks = min(kp, (np + kMinPiece - 1) / kMinPiece);
          c_first = ppre[s] + h * ks;
          c_last = c_first + ks - 1;
        } else {
          c_first = (int)(((int64_t)(seg_begin + 1) * G + N - 1) / N) - 1;
          c_last = (int)(((int64_t)seg_end * G + N - 1) / N) - 1;
        }
        fence_acq_rel_gpu();
        __syncwarp();
        int fin = 0;
        if (lane == 0) fin = atomicAdd(&ws.attn_done[sg], 1) == (c_last - c_first);
        fin = __shfl_sync(0xffffffffu, fin, 0);
        if (fin) {
          fence_acq_rel_gpu();
          // pieces in chunks whose loads are all in flight together
          constexpr int kPieces = C::kEPL >= 32 ? 2 : (C::kEPL >= 16 ? 4 : 8);
          const int npieces = c_last - c_first + 1;
          float Mx = -INFINITY, Lx = 0.f, ax[C::kEPL];
#pragma unroll
          for (int e = 0; e < C::kEPL; ++e) ax[e] = 0.f;
          for (int p0c = 0; p0c < npieces; p0c += kPieces) {
            float mv[kPieces], lv[kPieces], xv[kPieces][C::kEPL];
#pragma unroll
            for (int q = 0; q < kPieces; ++q) {
              mv[q] = -INFINITY;
              lv[q] = 0.f;
              if (p0c + q < npieces) {
                const int cc = c_first + p0c + q;
                const int ub = (int)((int64_t)cc * N / G);
                const int wh = (kp > 0 || max(seg_begin, ub) == ub) ? 0 : 1;
                const float* pr = ws.attn_part + ((int64_t)(2 * cc + wh) * GQ + hh) * C::kRow;
                const float2 ml = __ldcg(reinterpret_cast<const float2*>(pr + HD));
                mv[q] = ml.x;
                lv[q] = ml.y;
#pragma unroll
                for (int e = 0; e < C::kEPL; e += 2) {
                  const float2 x = __ldcg(reinterpret_cast<const float2*>(pr + el + e));
                  xv[q][e] = x.x;
                  xv[q][e + 1] = x.y;
                }
              }
            }
            float Mn = Mx;
#pragma unroll
            for (int q = 0; q < kPieces; ++q) Mn = fmaxf(Mn, mv[q]);
            const float rs = Mx == -INFINITY ? 0.f : exp2f(Mx - Mn);
            Lx *= rs;
#pragma unroll
            for (int e = 0; e < C::kEPL; ++e) ax[e] *= rs;
            Mx = Mn;
#pragma unroll
            for (int q = 0; q < kPieces; ++q) {
              const float f = mv[q] == -INFINITY ? 0.f : exp2f(mv[q] - Mx);
              Lx = fmaf(lv[q], f, Lx);
#pragma unroll
              for (int e = 0; e < C::kEPL; ++e) ax[e] = fmaf(p0c + q < npieces ? xv[q][e] : 0.f, f, ax[e]);
            }
          }
          const float inv = 1.f / Lx;
#pragma unroll
          for (int e = 0; e < C::kEPL; e += 2)
            out_pair<PEERS>(args, orow + e, ax[e] * inv, ax[e + 1] * inv);
          if (lse && el == 0) *lse = (Mx + log2f(Lx)) * kLn2;
          if (lane == 0) ws.attn_done[sg] = 0;
        }
      }
    }
    u = piece_end;
    ++k;
  }
  // exit stamp: the last consumer warp to finish (merges included)
  if (kTrace && lane == 0) {
    trace_max(4);
    atomicMax(&s_trace[9], (unsigned long long)clock64());
    if (atomicAdd(&s_trace_warps, 1) == kConsumers - 1 && blockIdx.x < 256)
      for (int i = 0; i < 16; ++i) g_attn_trace[args.layer & 1][blockIdx.x][i] = s_trace[i];
  }
}

#include "k_attn_tc.cuh"

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 3-D view [layers][n_phys*kv_heads*page][head_dim] of a KV pool; boxes of
// 64 columns x one page of rows with 128-byte swizzle.
// 4-D view of a KV pool: (64 columns, pool rows, HD/64 column blocks,
// layers) with strides (2 B, HD*2 B, 128 B, pool bytes).  One box
// (64, B, HD/64, 1) is a whole (page, head) K or V tile, landing in smem as
// [column block][B rows][128 B] with 128B swizzle — one TMA op per tile.
// cb_box = 1 (tensor-core K4): one box per (page, column block), so a
// group's pages land column block by column block.
int make_kv_map(CUtensorMap* m, const void* base, const ChessDims& d, int cb_box = 0) {
  auto fn = encode_fn();
  if (!fn) return fail(CHESS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t rows = (cuuint64_t)d.n_phys * d.kv_heads * d.page_size;
  cuuint64_t dims[4] = {64, rows, (cuuint64_t)d.head_dim / 64, (cuuint64_t)d.layers};
  cuuint64_t strides[3] = {(cuuint64_t)d.head_dim * 2, 128, rows * d.head_dim * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)d.page_size, (cuuint32_t)(cb_box ? cb_box : d.head_dim / 64), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHESS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return CHESS_OK;
}

template <int HD, int GQ, int B>
int launch_cluster(const ChessState& st, const Workspace& ws, const AttnArgs& args, int segs,
                   cudaStream_t stream) {
  using C = Cfg<HD, GQ, B, true>;
  // smem attributes of both instances set by cluster_size_for
  auto kfn = args.n_peer ? sparse_decode_kernel<HD, GQ, B, true, 1, true>
                         : sparse_decode_kernel<HD, GQ, B, true, 1, false>;
  CUtensorMap km, vm;
  int rc = make_kv_map(&km, st.k_pool, st.d);
  if (rc) return rc;
  rc = make_kv_map(&vm, st.v_pool, st.d);
  if (rc) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(segs * args.cl);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = args.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool no_pdl = getenv("CHESS_ATTN_NOPDL") != nullptr;  // debug A/B
  cfg.numAttrs = no_pdl ? 1 : 2;
  cudaLaunchKernelEx(&cfg, kfn, st, ws, args, km, vm);
  return check_launch("sparse_decode(cluster)");
}

template <int HD, int GQ, int B>
int cluster_size_for(int segs);

// Largest cluster size (8, 4, 2) whose clusters can all be co-resident for
// `segs` segments, or 0 (no cluster mode: batch * kv_heads > SMs / 2).
template <int HD, int GQ, int B>
int cluster_size_for(int segs) {
  static int max_active[kMaxCluster + 1] = {};
  static bool probed = false;
  auto kfn = sparse_decode_kernel<HD, GQ, B, true, 1, false>;
  using C = Cfg<HD, GQ, B, true>;
  if (!probed) {
    // Load every instance of this shape now (first launch of the shape):
    // with CUDA's lazy module loading a kernel's first launch can wait for
    // running kernels, so a first launch of the peer-store instance while a
    // peer-exchange wait spins on the same device (in-process multi-rank
    // runs) would stall until the wait times out.
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, sparse_decode_kernel<HD, GQ, B, true, 1, false>);
    cudaFuncGetAttributes(&fa, sparse_decode_kernel<HD, GQ, B, true, 1, true>);
    cudaFuncGetAttributes(&fa, sparse_decode_kernel<HD, GQ, B, false, 1, false>);
    cudaFuncGetAttributes(&fa, sparse_decode_kernel<HD, GQ, B, false, 1, true>);
    cudaFuncGetAttributes(&fa, sparse_decode_kernel<HD, GQ, B, false, 2, false>);
    cudaFuncGetAttributes(&fa, sparse_decode_kernel<HD, GQ, B, false, 2, true>);
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    cudaFuncSetAttribute(sparse_decode_kernel<HD, GQ, B, true, 1, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    for (int cl = 2; cl <= kMaxCluster; cl *= 2) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cl * 8);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = C::kSmem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cl;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kfn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
      }
      max_active[cl] = n;
    }
    probed = true;
  }
  static const bool off = getenv("CHESS_ATTN_CLUSTER") && atoi(getenv("CHESS_ATTN_CLUSTER")) == 0;  // A/B
  if (off || segs <= 0) return 0;
  static const int cl_cap = getenv("CHESS_ATTN_CLMAX") ? atoi(getenv("CHESS_ATTN_CLMAX")) : kMaxCluster;  // A/B
  for (int cl = std::min(kMaxCluster, cl_cap); cl >= 2; cl /= 2)
    if (segs <= max_active[cl] && segs * cl <= num_sms()) return cl;
  return 0;
}

template <int HD, int GQ, int B, int CPS>
int launch_grid(const ChessState& st, const Workspace& ws, const AttnArgs& args, int nctas,
                cudaStream_t stream);

// Tensor-core K4 (k_attn_tc.cuh): one CTA per SM, piece mode / stream-K.
template <int GQ, int B>
int launch_tc(const ChessState& st, const Workspace& ws, const AttnArgs& args, int nctas, cudaStream_t stream) {
  static bool configured = false;
  auto kfn = args.n_peer ? sparse_decode_tc_kernel<GQ, B, true> : sparse_decode_tc_kernel<GQ, B, false>;
  if (!configured) {
    cudaFuncAttributes fa;  // load both instances now (see cluster_size_for)
    cudaFuncGetAttributes(&fa, sparse_decode_tc_kernel<GQ, B, true>);
    cudaFuncGetAttributes(&fa, sparse_decode_tc_kernel<GQ, B, false>);
    cudaFuncSetAttribute(sparse_decode_tc_kernel<GQ, B, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)tca::kSmem);
    cudaFuncSetAttribute(sparse_decode_tc_kernel<GQ, B, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)tca::kSmem);
    configured = true;
  }
  CUtensorMap km, vm;
  int rc = make_kv_map(&km, st.k_pool, st.d, 1);
  if (rc) return rc;
  rc = make_kv_map(&vm, st.v_pool, st.d, 1);
  if (rc) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::min(nctas, num_sms()));
  cfg.blockDim = dim3(tca::kThreads);
  cfg.dynamicSmemBytes = tca::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool no_pdl = getenv("CHESS_ATTN_NOPDL") != nullptr;  // debug A/B
  cfg.numAttrs = no_pdl ? 0 : 1;
  cudaLaunchKernelEx(&cfg, kfn, st, ws, args, km, vm);
  return check_launch("sparse_decode_tc");
}

template <int HD, int GQ, int B>
int launch_inst(const ChessState& st, const Workspace& ws, const AttnArgs& args_in, int nctas,
                cudaStream_t stream) {
  AttnArgs args = args_in;
  const int segs = st.d.batch * st.d.kv_heads;
  args.cl = args.mode == 7 ? 0 : cluster_size_for<HD, GQ, B>(segs);
  // next-layer L2 prefetch (see the producer): piece mode only, where CTA c
  // owns the same segment piece in every layer.  Measured (profiles/r02/
  // k4_next_layer_prefetch.txt): cfg3 K4 18.18 -> 17.8 us, dynamic step
  // 614.6 -> 602.8 us, headline neutral; stream-K (cfg4, two CTAs per SM)
  // 47.5 -> 48.6 us and cluster mode (cfg2, cfg5) neutral or worse: off there.
  static const int next_pf_env = getenv("CHESS_ATTN_NEXTPF") ? atoi(getenv("CHESS_ATTN_NEXTPF")) : -1;  // A/B
  args.next_pf = next_pf_env >= 0 ? next_pf_env : (args.cl == 0 && segs <= num_sms() ? 8 : 0);
  // CHESS_ATTN_TC: 0 (default) mma.sync consumer; 1 tensor-core consumer
  // (k_attn_tc.cuh) wherever cluster mode is not chosen; 2 everywhere.
  // Measured on B200 (profiles/r02/k4_tc/): a tcgen05.mma of kind::f16 costs
  // ~150 cycles whatever N (8..128) and M (64, 128) are, so the decode shape
  // (N = GQA heads = 4-8) runs the tensor pipe at ~1/30 of its rate; QK + PV
  // take 4 MMAs per 32-token page = ~600 cycles per page, above the mma.sync
  // consumer's ~500: cfg3 K4 18.96 vs 18.01 us, cfg5 20.8 vs 11.6, cfg4 54.7
  // vs 45.7, cfg2 12.4 vs 3.2.
  static const int tc_env = getenv("CHESS_ATTN_TC") ? atoi(getenv("CHESS_ATTN_TC")) : 0;
  if constexpr (HD == 128 && (B == 16 || B == 32))
    if (tc_env && args.mode == 0 && (tc_env == 2 || args.cl == 0)) return launch_tc<GQ, B>(st, ws, args, nctas, stream);
  if (args.cl) return launch_cluster<HD, GQ, B>(st, ws, args, segs, stream);
  // stream-K regime: two CTAs per SM over half-depth rings
  static const int cps_env = getenv("CHESS_ATTN_CPS") ? atoi(getenv("CHESS_ATTN_CPS")) : 0;  // A/B
  const int cps = cps_env ? cps_env : (segs > num_sms() ? 2 : 1);
  if (cps == 2) return launch_grid<HD, GQ, B, 2>(st, ws, args, std::min(nctas, 2 * num_sms()), stream);
  return launch_grid<HD, GQ, B, 1>(st, ws, args, std::min(nctas, num_sms()), stream);
}

template <int HD, int GQ, int B, int CPS>
int launch_grid(const ChessState& st, const Workspace& ws, const AttnArgs& args, int nctas,
                cudaStream_t stream) {
  using C = Cfg<HD, GQ, B, false, CPS>;
  const size_t smem = C::kSmem;
  static bool configured = false;
  auto kfn = args.n_peer ? sparse_decode_kernel<HD, GQ, B, false, CPS, true>
                         : sparse_decode_kernel<HD, GQ, B, false, CPS, false>;
  if (!configured) {
    cudaFuncSetAttribute(sparse_decode_kernel<HD, GQ, B, false, CPS, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sparse_decode_kernel<HD, GQ, B, false, CPS, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  CUtensorMap km, vm;
  int rc = make_kv_map(&km, st.k_pool, st.d);
  if (rc) return rc;
  rc = make_kv_map(&vm, st.v_pool, st.d);
  if (rc) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool no_pdl = getenv("CHESS_ATTN_NOPDL") != nullptr;  // debug A/B
  cfg.numAttrs = no_pdl ? 0 : 1;
  cudaLaunchKernelEx(&cfg, kfn, st, ws, args, km, vm);
  return check_launch("sparse_decode");
}

}  // namespace

int attn_ctas_for(const ChessDims& d) {
  (void)d;
  return kMaxCtasPerSm * num_sms();
}

int launch_sparse_decode(const ChessState& st, const Workspace& ws, int layer, const void* q,
                         int64_t q_stride, void* out, int64_t out_stride, float* lse,
                         float softmax_scale, uint32_t flags, cudaStream_t stream, const PeerOut* po) {
  const ChessDims& d = st.d;
  AttnArgs a;
  a.early = (flags & CHESS_ATTN_AFTER_DECODE) ? 1 : 0;
  a.n_peer = 0;
  if (po) {
    a.n_peer = po->n_peer;
    for (int p = 0; p < po->n_peer; ++p) a.peer_out[p] = po->peer_out[p];
  }
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.q_stride = q_stride;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.out_stride = out_stride;
  a.lse = lse;
  a.scale_log2 = softmax_scale * kLog2e;
  a.layer = layer;
  static const int dbg_mode = getenv("CHESS_ATTN_MODE") ? atoi(getenv("CHESS_ATTN_MODE")) : 0;
  a.mode = dbg_mode;
  a.cl = 0;
  // measured (tools/attn_prefetch_sweep.sh): 16 pages -1% at cfg3, worse at
  // cfg4/cfg5 and beyond 16 pages (the prefetches evict the running layer)
  static const int prefetch = getenv("CHESS_ATTN_PREFETCH") ? atoi(getenv("CHESS_ATTN_PREFETCH")) : 0;
  a.prefetch = prefetch;
  a.next_pf = -1;  // set per mode in launch_inst
  const int gq = d.q_heads / d.kv_heads;
  static const int grid_env = getenv("CHESS_ATTN_GRID") ? atoi(getenv("CHESS_ATTN_GRID")) : 0;  // experiments
  const int nctas = grid_env > 0 ? std::min(grid_env, ws.attn_ctas) : ws.attn_ctas;
  if ((reinterpret_cast<uintptr_t>(q) & 15) || (q_stride & 7))
    return fail(CHESS_ERR_UNSUPPORTED, "sparse_decode: q must be 16-byte aligned with q_stride %% 8 == 0");
  if (d.kv_heads > 255 || d.batch > kAttnMaxBatch)
    return fail(CHESS_ERR_UNSUPPORTED, "sparse_decode: kv_heads must be <= 255 and batch <= %d", kAttnMaxBatch);
#define CHESS_ATTN_CASE(HD_, GQ_, B_)                                        \
  if (d.head_dim == HD_ && gq == GQ_ && d.page_size == B_)                   \
    return launch_inst<HD_, GQ_, B_>(st, ws, a, nctas, stream);
  CHESS_ATTN_CASE(128, 4, 32)
  CHESS_ATTN_CASE(128, 8, 32)
  CHESS_ATTN_CASE(128, 4, 16)
  CHESS_ATTN_CASE(128, 8, 16)
  CHESS_ATTN_CASE(128, 1, 32)
  CHESS_ATTN_CASE(128, 1, 16)
  CHESS_ATTN_CASE(128, 2, 32)
  CHESS_ATTN_CASE(64, 1, 16)
  CHESS_ATTN_CASE(64, 1, 32)
  CHESS_ATTN_CASE(64, 2, 16)
  CHESS_ATTN_CASE(64, 4, 16)
  CHESS_ATTN_CASE(64, 4, 32)
  CHESS_ATTN_CASE(64, 8, 32)
#undef CHESS_ATTN_CASE
  return fail(CHESS_ERR_UNSUPPORTED, "sparse_decode: no kernel for head_dim=%d gqa=%d page=%d",
              d.head_dim, gq, d.page_size);
}

// End of a step's peer-memory output gather, a two-phase barrier on
// per-source flags (system scope; value 2g+1 = "step g written", 2g+2 =
// "step g copied out", g = steps finished on this rank): CTA 0 publishes
// "written" (stream order puts it after this rank's K4 launches), every CTA
// waits for all ranks' "written", copies the peers' blocks of this rank's
// region into `out` (K4 stored the own blocks there directly); the
// last CTA publishes "copied" and waits for every rank's "copied" before the
// kernel ends, so no rank's next-step K4 can overwrite a region a peer has
// not copied yet.  One region (no double buffer) and no device read in K4.
__device__ __forceinline__ void wait_flags(const uint32_t* f, int world, uint32_t target, int32_t* err) {
  if (threadIdx.x < world) {
    const uint64_t t0 = global_ns();
    uint32_t polls = 0;
    while ((int32_t)(ld_acquire_sys(f + threadIdx.x) - target) < 0) {
      if ((++polls & 255u) == 0 && global_ns() - t0 > 10000000000ull) {
        atomicExch(err, 1);
        break;
      }
    }
  }
}

__global__ void __launch_bounds__(256) gather_finish_kernel(uint32_t* const* flags, uint32_t* my_flags,
                                                            int world, int rank, uint32_t* gen,
                                                            int32_t* err, const __nv_bfloat16* region,
                                                            int64_t elems, int64_t blk, __nv_bfloat16* out) {
  __shared__ uint32_t s_g;
  __shared__ int s_last;
  if (threadIdx.x == 0) s_g = __ldcg(gen);
  __syncthreads();
  const uint32_t g = s_g;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < world; ++p) st_release_sys(flags[p] + rank, 2u * g + 1u);
  }
  wait_flags(my_flags, world, 2u * g + 1u, err);
  __syncthreads();
  if (out && world > 1) {
    // the peers' blocks only: K4 wrote this rank's own blocks into `out`
    const uint4* src = reinterpret_cast<const uint4*>(region);
    uint4* dst = reinterpret_cast<uint4*>(out);
    const int64_t n = elems / 8, bv = blk / 8;  // elems, blk % 8 == 0 (checked by the caller)
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
      if ((int)((i / bv) % world) != rank) dst[i] = __ldcg(src + i);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(gen + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x == 0) {
    __threadfence();
    for (int p = 0; p < world; ++p) st_release_sys(flags[p] + rank, 2u * g + 2u);
  }
  wait_flags(my_flags, world, 2u * g + 2u, err);
  if (threadIdx.x == 0) {
    gen[1] = 0;
    gen[0] = g + 1u;
  }
}

int launch_gather_finish(uint32_t* const* flags, uint32_t* my_flags, int world, int rank, uint32_t* gen,
                         int32_t* err, const void* region, int64_t elems, int64_t blk, void* out,
                         cudaStream_t stream) {
  const int64_t v = elems / 8;
  const int grid = world == 1 ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(2 * num_sms(), (v + 255) / 256));
  gather_finish_kernel<<<grid, 256, 0, stream>>>(flags, my_flags, world, rank, gen, err,
                                                 reinterpret_cast<const __nv_bfloat16*>(region), elems, blk,
                                                 reinterpret_cast<__nv_bfloat16*>(out));
  return check_launch("gather_finish");
}

}  // namespace chess

// Debug only (not part of include/chess_b200.h): copy the per-CTA timeline of
// the last sparse_decode launch of each layer parity, [2][256][16] u64 (ns; [8],[9] SM clocks).
// tensor-core K4 per-group timeline (CHESS_TRACE builds; [8 CTAs][16 groups][8 events] clock64)
extern "C" int chess_debug_attn_tc_trace(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, chess::g_tca_trace, sizeof(chess::g_tca_trace)) == cudaSuccess ? 0 : 8;
}

extern "C" int chess_debug_attn_trace(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, chess::g_attn_trace, sizeof(chess::g_attn_trace)) == cudaSuccess ? 0 : 8;
}
