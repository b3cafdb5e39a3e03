// k_attn_tc.cuh — K4 with a tcgen05 consumer (head_dim 128).  Included by
// k_attn.cu inside namespace chess::{anon}; same inputs, outputs, work
// partition (piece mode / stream-K) and split-segment merge as
// sparse_decode_kernel, oracle oracle/attention.py (fp64 softmax(q K^T) V over
// the working set, rows >= fill excluded).
//
// Work unit: a GROUP of 128 tokens = 128/B consecutive working-set pages of
// one segment (slot, kv head).  Per group:
//   QK   S[128 tok][8] = K[128 tok][128 d] . q^T     tcgen05 M=128 N=8 K=16 x8,
//        A = K tile K-major SW128 ([cb][128 rows][128 B], one TMA box per
//        (page, cb)), B = the GQA group's q rows (K-major SW128, rows >= GQ 0)
//   softmax   4 warps, thread t = token t: tcgen05.ld of its S row, group max
//        per head (9-shuffle transpose-reduce + 4-warp smem exchange), online
//        (m, l) per head, P^T row t stored as 16 B (8 heads bf16)
//   PV   O_g^T[128 d][8] = V^T . P^T                  tcgen05 M=128 N=8, one
//        MMA per 16 valid tokens, A = V tile MN-major SW128 (lbo = 16 KB cb
//        stride, sbo = 1 KB), B = P MN-major no-swizzle (lbo = 128 B)
//   correction   thread t = d row t: acc[h] = acc[h] * alpha_g[h] + O_g[t][h]
//        (each group's PV writes a fresh TMEM accumulator; the rescale of the
//        running output happens in registers, no TMEM read-modify-write)
// Roles (12 warps): 0-3 softmax (S -> P, running max / sum; thread t = token
// t of the group), 4-7 correction + epilogue (thread t = d row t of O), 8 / 9
// TMA producers of the K / V tiles (3-stage ring; K and V released
// separately, a stage's K refills as soon as its QK is done), 10 QK issuer
// (TMEM owner), 11 PV issuer.  S, P and O are 4-deep (TMEM 64 columns), so
// the QK of group g+3, the softmax of g+1 and the PV + correction of g run
// at once; nothing waits on an MMA's latency except through data.  All
// hand-offs are mbarriers (TMA complete_tx, tcgen05.commit, per-warp
// arrivals); the rescale factors of each group and the piece's (m, l) pass
// from the softmax to the correction warps through shared memory.
// Layouts verified on B200 by tools/tc_attn_probe.cu (profiles/r02/tc_attn_layout_probe.txt).

namespace tca {

constexpr int kHD = 128;
constexpr int kGT = 128;                    // tokens per group
constexpr int kStages = 3;
constexpr int kKBytes = kGT * kHD * 2;      // 32 KB: one K (or V) group tile
constexpr int kStageBytes = 2 * kKBytes;
constexpr int kCbStride = kGT * 128;        // 16 KB between the two 64-column blocks
constexpr int kQBytes = 2 * 8 * 128;        // [cb][8 rows][128 B]
constexpr int kPBytes = kGT * 16;           // [token][8 heads] bf16
constexpr int kNB = 4;                      // S / P / O / alpha buffers in flight
constexpr int kSoftmax = 4;                 // softmax warps
constexpr int kCorr = 4;                    // first correction warp
constexpr int kProducer = 8, kVProducer = 9, kMma = 10, kPvMma = 11;
constexpr int kThreads = 12 * 32;
constexpr int kTmemCols = 64;               // S[4] at cols 0..31, O[4] at 32..63
constexpr int kRow = kHD + 4;               // split-partial row: o[HD], m, l, pad
constexpr uint32_t kIdQK = tc::idesc_f16_major(128, 8, 1, 0, 0);
constexpr uint32_t kIdPV = tc::idesc_f16_major(128, 8, 1, 1, 1);
constexpr int kNumBars = 4 * kStages + 8 * kNB + 6;
constexpr int kAlphaBytes = kNB * 8 * 4;    // rescale factors per buffered group
constexpr int kLmBytes = 2 * 16 * 4;        // per piece (k & 1): m[8], l[8]
constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 2 * kQBytes + kNB * kPBytes + 96 * 4 + kAlphaBytes +
                         kLmBytes + (size_t)(4 * kAttnMaxBatch + 2 + 4) * 4 + kNumBars * 8 + 64;

__device__ __forceinline__ void softmax_sync() { asm volatile("bar.sync 3, 128;" ::: "memory"); }
__device__ __forceinline__ void corr_sync() { asm volatile("bar.sync 4, 128;" ::: "memory"); }
__device__ __forceinline__ void sts_u4(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// max / sum over the 128 softmax threads of 8 values each (fixed order):
// transpose-reduce inside the warp (lane ends up with head (lane >> 2) & 7),
// then the 4 warps' rows through shared memory.
template <bool MAX>
__device__ __forceinline__ void reduce128(const float (&x)[8], float (&out)[8], float* red) {
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 3;
  auto op = [](float a, float b) { return MAX ? fmaxf(a, b) : a + b; };
  float y[4], z[2], w;
  const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float keep = u16 ? x[i + 4] : x[i], send = u16 ? x[i] : x[i + 4];
    y[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 16));
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float keep = u8 ? y[i + 2] : y[i], send = u8 ? y[i] : y[i + 2];
    z[i] = op(keep, __shfl_xor_sync(0xffffffffu, send, 8));
  }
  {
    const float keep = u4 ? z[1] : z[0], send = u4 ? z[0] : z[1];
    w = op(keep, __shfl_xor_sync(0xffffffffu, send, 4));
  }
  w = op(w, __shfl_xor_sync(0xffffffffu, w, 2));
  w = op(w, __shfl_xor_sync(0xffffffffu, w, 1));
  const uint32_t ra = smem_u32(red);
  if ((lane & 3) == 0) sts_f32(ra + (uint32_t)(warp * 8 + (lane >> 2)) * 4u, w);
  softmax_sync();
  float4 a0 = lds_f4(ra), a1 = lds_f4(ra + 16);
#pragma unroll
  for (int q = 1; q < kSoftmax; ++q) {
    const float4 b0 = lds_f4(ra + 32 * q), b1 = lds_f4(ra + 32 * q + 16);
    a0 = make_float4(op(a0.x, b0.x), op(a0.y, b0.y), op(a0.z, b0.z), op(a0.w, b0.w));
    a1 = make_float4(op(a1.x, b1.x), op(a1.y, b1.y), op(a1.z, b1.z), op(a1.w, b1.w));
  }
  out[0] = a0.x, out[1] = a0.y, out[2] = a0.z, out[3] = a0.w;
  out[4] = a1.x, out[5] = a1.y, out[6] = a1.z, out[7] = a1.w;
}

// One group of the CTA's work, produced identically by every role.
struct Group {
  int s, h, pg0, npg, nvalid;  // slot, kv head, first page (in segment), pages, valid tokens
  bool first, last;            // first / last group of its piece
  int seg_begin, seg_end;      // the segment's global page range
  int piece_begin;             // global index of the piece's first page
};

}  // namespace tca

// Debug timeline (CHESS_TRACE builds, read by chess_debug_attn_tc_trace):
// clock64 stamps per (CTA < 8, group < 16, event): 0 K landed (QK issuer),
// 1 S read (softmax), 2 P published, 3 V landed (PV issuer), 4 PV issued,
// 5 O folded (correction), 6 K issued (producer), 7 V issued (producer).
__device__ unsigned long long g_tca_trace[8][16][8];
__device__ __forceinline__ void tca_stamp(int j, int ev) {
  if (kTrace && blockIdx.x < 8 && j < 16) g_tca_trace[blockIdx.x][j][ev] = clock64();
}

template <int GQ, int B, bool PEERS>
__global__ void __launch_bounds__(tca::kThreads, 1)
    sparse_decode_tc_kernel(ChessState st, Workspace ws, AttnArgs args, const __grid_constant__ CUtensorMap kmap,
                            const __grid_constant__ CUtensorMap vmap) {
  using namespace tca;
  constexpr int kGP = kGT / B;  // pages per group
  static_assert(GQ <= 8 && kGT % B == 0, "tc attention shape");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qbuf = ring + (size_t)kStages * kStageBytes;
  uint8_t* pbuf = qbuf + 2 * kQBytes;
  float* red = reinterpret_cast<float*>(pbuf + kNB * kPBytes);  // [2][32] max, [32] sum (softmax warps)
  float* alph = red + 96;                                        // [kNB][8] rescale factors
  float* lm = alph + kNB * 8;                                    // [2][m 8, l 8]
  int* prefix = reinterpret_cast<int*>(lm + 32);                 // [nb + 1]
  int* s_np = prefix + kAttnMaxBatch + 1;                        // [nb]
  int* s_fill = s_np + kAttnMaxBatch;                            // [nb]
  int* ppre = s_fill + kAttnMaxBatch;                            // [nb + 1]
  int* misc = ppre + kAttnMaxBatch + 1;                          // [0] kp, [1] tmem, [2] merge flag
  uint64_t* bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(misc + 4) + 7) & ~uintptr_t(7));
  uint64_t* kfull = bars;
  uint64_t* kempty = kfull + kStages;
  uint64_t* vfull = kempty + kStages;
  uint64_t* vempty = vfull + kStages;
  uint64_t* sfull = vempty + kStages;  // [kNB] each below
  uint64_t* sempty = sfull + kNB;
  uint64_t* pfull = sempty + kNB;
  uint64_t* pempty = pfull + kNB;
  uint64_t* ofull = pempty + kNB;
  uint64_t* oempty = ofull + kNB;
  uint64_t* afull = oempty + kNB;      // alpha[j % kNB] written
  uint64_t* aempty = afull + kNB;      // ... and read
  uint64_t* qfull = aempty + kNB;      // [2]
  uint64_t* lfull = qfull + 2;         // [2] piece (m, l) written
  uint64_t* lempty = lfull + 2;        // [2] ... and read
  const ChessDims& d = st.d;
  const int H = d.kv_heads;
  const int nb = d.batch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == kProducer * 32) prefetch_tmap(&kmap);
  if (threadIdx.x == kVProducer * 32) prefetch_tmap(&vmap);
  // see sparse_decode_kernel: only after another K4 may the prologue and the
  // first K/V loads run ahead of griddepcontrol.wait
  if (!args.early) pdl_wait();
  if (warp == 0) {
    // pages per segment (np = ws_len - 1 + (fill > 0)), page and piece prefixes
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
    const int G0 = min((int)gridDim.x, run);
    int nseg = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int s = b0 + lane;
      nseg += __popc(__ballot_sync(0xffffffffu, s < nb && s_np[s] > 0)) * H;
    }
    const int kp = (nseg > 0 && nseg <= G0) ? G0 / nseg : 0;  // 0: stream-K
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
      misc[0] = kp;
    }
  } else if (warp == kProducer && lane == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&kfull[i], 1);
      mbar_init(&kempty[i], 1);
      mbar_init(&vfull[i], 1);
      mbar_init(&vempty[i], 1);
    }
    for (int i = 0; i < kNB; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], kSoftmax);
      mbar_init(&pfull[i], kSoftmax);
      mbar_init(&pempty[i], 1);
      mbar_init(&ofull[i], 1);
      mbar_init(&oempty[i], 4);
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&lfull[i], 1);
      mbar_init(&lempty[i], 4);
    }
    fence_barrier_init();
  } else if (warp == kMma) {
    tc::tmem_alloc<kTmemCols>(reinterpret_cast<uint32_t*>(&misc[1]));
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  pdl_launch_dependents();
  const uint32_t tmem = static_cast<uint32_t>(misc[1]);

  const int N = prefix[nb];
  const int kp = misc[0];
  const int G = kp > 0 ? ppre[nb] : min((int)gridDim.x, N);
  const int c = blockIdx.x;
  int u_begin = 0, u_end = 0;
  if (c < G) {
    if (kp > 0) {
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
  }
  // cursor over the CTA's groups (identical in every role)
  int cu = u_begin, c_piece_end = u_begin, cs = 0, ch = 0, cp = 0, cnp = 0, c_seg_begin = 0, c_piece_begin = 0;
  auto next = [&](Group& g) -> bool {
    if (cu >= u_end) return false;
    g.first = false;
    if (cu == c_piece_end) {
      int lo = 0, hi = nb;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (prefix[mid] <= cu) lo = mid; else hi = mid;
      }
      cs = lo;
      cnp = s_np[lo];
      const int r = cu - prefix[lo];
      ch = r / cnp;
      cp = r - ch * cnp;
      c_seg_begin = prefix[lo] + ch * cnp;
      c_piece_end = min(c_seg_begin + cnp, u_end);
      c_piece_begin = cu;
      g.first = true;
    }
    g.s = cs;
    g.h = ch;
    g.pg0 = cp;
    g.npg = min(kGP, c_piece_end - cu);
    g.nvalid = (cp + g.npg == cnp) ? (g.npg - 1) * B + s_fill[cs] : g.npg * B;
    g.seg_begin = c_seg_begin;
    g.seg_end = c_seg_begin + cnp;
    g.piece_begin = c_piece_begin;
    cu += g.npg;
    cp += g.npg;
    g.last = cu == c_piece_end;
    return true;
  };

  if (warp == kProducer || warp == kVProducer) {
    // ===================== TMA producers (K warp, V warp) =====================
    // Separate warps so a group's K tile (free once its QK is done) is never
    // queued behind the V tile of an earlier group (free only after its PV).
    // Lane 2p + cb issues the box of (page p, column block cb); the next
    // group's page ids are loaded before this group's waits.
    const bool is_v = warp == kVProducer;
    uint64_t* full = is_v ? vfull : kfull;
    uint64_t* empty = is_v ? vempty : kempty;
    const CUtensorMap* map = is_v ? &vmap : &kmap;
    Group g, gn;
    bool have = next(g);
    auto row_of = [&](const Group& x) {
      int r = 0;
      if (lane < 2 * x.npg) {
        const int pid = __ldg(st.block_table + (int64_t)x.s * d.max_ws + x.pg0 + (lane >> 1));
        r = (pid * H + x.h) * B;
      }
      return r;
    };
    int row0 = have ? row_of(g) : 0;
    for (int j = 0; have; ++j) {
      const bool have_n = next(gn);
      const int row0n = have_n ? row_of(gn) : 0;
      const int stage = j % kStages;
      const uint32_t ph = (uint32_t)((j / kStages) & 1);
      const uint32_t dst = smem_u32(ring + (size_t)stage * kStageBytes + (is_v ? kKBytes : 0)) +
                           (uint32_t)((lane & 1) * kCbStride + (lane >> 1) * B * 128);
      if (lane == 0) {
        mbar_wait(&empty[stage], ph ^ 1u);
        mbar_arrive_expect_tx(&full[stage], (uint32_t)(g.npg * B * kHD * 2));
      }
      __syncwarp();
      if (lane < 2 * g.npg) tma_load_4d(dst, map, 0, row0, lane & 1, args.layer, smem_u32(&full[stage]));
      if (lane == 0) tca_stamp(j, is_v ? 7 : 6);
      g = gn;
      row0 = row0n;
      have = have_n;
    }
  } else if (warp == kMma) {
    // ===================== QK issuer =====================
    Group g;
    int j = 0, k = -1;
    while (next(g)) {
      if (g.first) {
        ++k;
        mbar_wait(&qfull[k & 1], (uint32_t)((k >> 1) & 1));
      }
      const int stage = j % kStages, nb_ = j % kNB;
      mbar_wait(&kfull[stage], (uint32_t)((j / kStages) & 1));
      if (lane == 0) tca_stamp(j, 0);
      mbar_wait(&sempty[nb_], (uint32_t)(((j / kNB) & 1) ^ 1));
      tc::fence_after();
      if (lane == 0) {
        const uint32_t a = smem_u32(ring + (size_t)stage * kStageBytes);
        const uint32_t b = smem_u32(qbuf + (k & 1) * kQBytes);
#pragma unroll
        for (int ks = 0; ks < kHD / 16; ++ks) {
          const uint32_t off = (uint32_t)((ks >> 2) * kCbStride + (ks & 3) * 32);
          const uint32_t offb = (uint32_t)((ks >> 2) * 1024 + (ks & 3) * 32);
          tc::mma_f16_ss(tmem + (uint32_t)(nb_ * 8), tc::smem_desc(a + off, 16, 1024, 2),
                         tc::smem_desc(b + offb, 16, 1024, 2), kIdQK, ks != 0);
        }
        tc::commit(&kempty[stage]);
        tc::commit(&sfull[nb_]);
      }
      __syncwarp();
      ++j;
    }
  } else if (warp == kPvMma) {
    // ===================== PV issuer =====================
    Group g;
    int j = 0;
    while (next(g)) {
      const int stage = j % kStages, nb_ = j % kNB;
      const uint32_t ph = (uint32_t)((j / kNB) & 1);
      mbar_wait(&vfull[stage], (uint32_t)((j / kStages) & 1));
      if (lane == 0) tca_stamp(j, 3);
      mbar_wait(&pfull[nb_], ph);
      mbar_wait(&oempty[nb_], ph ^ 1u);
      tc::fence_after();
      if (lane == 0) tca_stamp(j, 4);
      // V rows of the last MMA's 16 tokens at or past `nvalid` (rows past the
      // tail page's fill) may hold never-written data: zero them so that
      // 0 * garbage cannot poison O (P is 0 there)
      const int vz0 = g.nvalid, vz1 = (g.nvalid + 15) & ~15;
      if (vz1 > vz0) {
        const uint32_t vb = smem_u32(ring + (size_t)stage * kStageBytes + kKBytes);
        for (int i = lane; i < (vz1 - vz0) * 16; i += 32) {
          const int row = vz0 + (i >> 4), cb = (i >> 3) & 1, q = i & 7;
          sts_u4(vb + (uint32_t)(cb * kCbStride + row * 128 + q * 16), make_uint4(0, 0, 0, 0));
        }
        fence_proxy_async();
        __syncwarp();
      }
      if (lane == 0) {
        const uint32_t a = smem_u32(ring + (size_t)stage * kStageBytes + kKBytes);
        const uint32_t b = smem_u32(pbuf + nb_ * kPBytes);
        const int nks = (g.nvalid + 15) >> 4;
        for (int ks = 0; ks < nks; ++ks)
          tc::mma_f16_ss(tmem + 32u + (uint32_t)(nb_ * 8), tc::smem_desc(a + ks * 2048, kCbStride, 1024, 2),
                         tc::smem_desc(b + ks * 256, 128, 2048, 0), kIdPV, ks != 0);
        tc::commit(&vempty[stage]);
        tc::commit(&pempty[nb_]);
        tc::commit(&ofull[nb_]);
      }
      __syncwarp();
      ++j;
    }
  } else if (warp < kCorr) {
    // ===================== softmax (warps 0-3) =====================
    const int t = threadIdx.x;  // token of the group (S row)
    const uint32_t tl = tmem + ((uint32_t)(32 * warp) << 16);
    bool waited = !args.early;
    float m_run[8], l_part[8];
    Group g;
    int j = 0, k = -1;
    while (next(g)) {
      const int nb_ = j % kNB;
      const uint32_t ph = (uint32_t)((j / kNB) & 1);
      if (g.first) {
        ++k;
        if (!waited) {
          pdl_wait();  // q comes from the previous grid
          waited = true;
        }
        // the GQA group's q rows -> K-major SW128 [cb][8 rows][128 B]; rows >= GQ zero
        {
          const int r = t >> 4, cc = t & 15;
          uint4 v = make_uint4(0, 0, 0, 0);
          if (r < GQ)
            v = __ldg(reinterpret_cast<const uint4*>(args.q + (int64_t)g.s * args.q_stride + ((int64_t)g.h * GQ + r) * kHD) + cc);
          sts_u4(smem_u32(qbuf + (k & 1) * kQBytes + (cc >> 3) * 1024 + r * 128 + (((cc & 7) ^ r) << 4)), v);
        }
        fence_proxy_async();
        softmax_sync();
        if (t == 0) mbar_arrive(&qfull[k & 1]);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          m_run[e] = -INFINITY;
          l_part[e] = 0.f;
        }
      }
      // ---- S row t ----
      mbar_wait(&sfull[nb_], ph);
      if (t == 0) tca_stamp(j, 1);
      tc::fence_after();
      float x[8];
      tc::tmem_ld_x8(tl + (uint32_t)(nb_ * 8), x);
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[nb_]);
      const bool valid = t < g.nvalid;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float y = x[e] * args.scale_log2;
        x[e] = (valid && y == y) ? y : -INFINITY;
      }
      float gm[8];
      reduce128<true>(x, gm, red + (j & 1) * 32);
      float alpha[8], p[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float m_new = fmaxf(m_run[e], gm[e]);
        alpha[e] = m_new == -INFINITY ? 1.f : exp2f(m_run[e] - m_new);
        p[e] = x[e] == -INFINITY ? 0.f : exp2f(x[e] - m_new);
        l_part[e] = fmaf(l_part[e], alpha[e], p[e]);
        m_run[e] = m_new;
      }
      // ---- rescale factors of this group for the correction warps ----
      if (t == 0) {
        mbar_wait(&aempty[nb_], ph ^ 1u);
        const uint32_t aa = smem_u32(alph + nb_ * 8);
        sts_u4(aa, make_uint4(__float_as_uint(alpha[0]), __float_as_uint(alpha[1]), __float_as_uint(alpha[2]),
                              __float_as_uint(alpha[3])));
        sts_u4(aa + 16, make_uint4(__float_as_uint(alpha[4]), __float_as_uint(alpha[5]), __float_as_uint(alpha[6]),
                                   __float_as_uint(alpha[7])));
        mbar_arrive(&afull[nb_]);
      }
      // ---- P^T row t (bf16) ----
      mbar_wait(&pempty[nb_], ph ^ 1u);
      sts_u4(smem_u32(pbuf + nb_ * kPBytes + t * 16),
             make_uint4(pack_bf16(p[0], p[1]), pack_bf16(p[2], p[3]), pack_bf16(p[4], p[5]), pack_bf16(p[6], p[7])));
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull[nb_]);
      if (t == 0) tca_stamp(j, 2);
      if (g.last) {
        // piece (m, l) for the correction warps' epilogue
        float L[8];
        reduce128<false>(l_part, L, red + 64);
        if (t == 0) {
          mbar_wait(&lempty[k & 1], (uint32_t)(((k >> 1) & 1) ^ 1));
          const uint32_t la = smem_u32(lm + (k & 1) * 16);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            sts_f32(la + 4u * e, m_run[e]);
            sts_f32(la + 32u + 4u * e, L[e]);
          }
          mbar_arrive(&lfull[k & 1]);
        }
      }
      ++j;
    }
  } else if (warp < kCorr + 4) {
    // ===================== correction + epilogue (warps 4-7) =====================
    const int t = threadIdx.x - kCorr * 32;  // d row of O
    const uint32_t tl = tmem + ((uint32_t)(32 * (warp - kCorr)) << 16);
    bool waited = !args.early;
    float acc[8];
    Group g;
    int j = 0, k = -1;
    while (next(g)) {
      const int nb_ = j % kNB;
      const uint32_t ph = (uint32_t)((j / kNB) & 1);
      if (g.first) {
        ++k;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
      }
      mbar_wait(&ofull[nb_], ph);
      if (t == 0) tca_stamp(j, 5);
      tc::fence_after();
      float o8[8];
      tc::tmem_ld_x8(tl + 32u + (uint32_t)(nb_ * 8), o8);
      tc::fence_before();
      mbar_wait(&afull[nb_], ph);
      const uint32_t aa = smem_u32(alph + nb_ * 8);
      const float4 a0 = lds_f4(aa), a1 = lds_f4(aa + 16);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&oempty[nb_]);
        mbar_arrive(&aempty[nb_]);
      }
      acc[0] = fmaf(acc[0], a0.x, o8[0]);
      acc[1] = fmaf(acc[1], a0.y, o8[1]);
      acc[2] = fmaf(acc[2], a0.z, o8[2]);
      acc[3] = fmaf(acc[3], a0.w, o8[3]);
      acc[4] = fmaf(acc[4], a1.x, o8[4]);
      acc[5] = fmaf(acc[5], a1.y, o8[5]);
      acc[6] = fmaf(acc[6], a1.z, o8[6]);
      acc[7] = fmaf(acc[7], a1.w, o8[7]);
      if (g.last) {
        // ---- piece epilogue ----
        if (!waited) {
          pdl_wait();  // every write of this kernel comes after the previous grid
          waited = true;
        }
        mbar_wait(&lfull[k & 1], (uint32_t)((k >> 1) & 1));
        float M[8], L[8];
        {
          const uint32_t la = smem_u32(lm + (k & 1) * 16);
          const float4 m0 = lds_f4(la), m1 = lds_f4(la + 16), l0 = lds_f4(la + 32), l1 = lds_f4(la + 48);
          M[0] = m0.x, M[1] = m0.y, M[2] = m0.z, M[3] = m0.w, M[4] = m1.x, M[5] = m1.y, M[6] = m1.z, M[7] = m1.w;
          L[0] = l0.x, L[1] = l0.y, L[2] = l0.z, L[3] = l0.w, L[4] = l1.x, L[5] = l1.y, L[6] = l1.z, L[7] = l1.w;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&lempty[k & 1]);
        const bool whole = g.seg_begin >= u_begin && g.seg_end <= u_end;
        const int s = g.s, h = g.h;
        if (whole) {
#pragma unroll
          for (int hh = 0; hh < GQ; ++hh) {
            const float v = acc[hh] / L[hh];
            const float w = __shfl_down_sync(0xffffffffu, v, 1);
            __nv_bfloat16* orow = args.out + (int64_t)s * args.out_stride + ((int64_t)h * GQ + hh) * kHD;
            if ((t & 1) == 0) out_pair<PEERS>(args, orow + t, v, w);
            if (args.lse && t == 0) args.lse[(int64_t)s * d.q_heads + h * GQ + hh] = (M[hh] + log2f(L[hh])) * kLn2;
          }
        } else {
          // split segment: partial (2c + which), which = 0 for the CTA's first piece
          const int which = g.piece_begin == u_begin ? 0 : 1;
#pragma unroll
          for (int hh = 0; hh < GQ; ++hh) {
            float* slot = ws.attn_part + ((int64_t)(2 * c + which) * GQ + hh) * kRow;
            slot[t] = acc[hh];
            if (t == 0) {
              slot[kHD] = M[hh];
              slot[kHD + 1] = L[hh];
            }
          }
          const int np = g.seg_end - g.seg_begin;
          int c_first, c_last;
          if (kp > 0) {  // the segment's pieces sit on consecutive CTAs
            const int ks = min(kp, (np + kMinPiece - 1) / kMinPiece);
            c_first = ppre[s] + h * ks;
            c_last = c_first + ks - 1;
          } else {
            c_first = (int)(((int64_t)(g.seg_begin + 1) * G + N - 1) / N) - 1;
            c_last = (int)(((int64_t)g.seg_end * G + N - 1) / N) - 1;
          }
          fence_acq_rel_gpu();
          corr_sync();
          if (t == 0) misc[2] = atomicAdd(&ws.attn_done[s * H + h], 1) == (c_last - c_first);
          corr_sync();
          if (misc[2]) {
            fence_acq_rel_gpu();
#pragma unroll
            for (int hh = 0; hh < GQ; ++hh) {
              float Mx = -INFINITY, Lx = 0.f, ax = 0.f;
              for (int cc = c_first; cc <= c_last; ++cc) {
                const int ub = (int)((int64_t)cc * N / G);
                const int wh = (kp > 0 || max(g.seg_begin, ub) == ub) ? 0 : 1;
                const float* pr = ws.attn_part + ((int64_t)(2 * cc + wh) * GQ + hh) * kRow;
                const float mv = __ldcg(pr + kHD), lv = __ldcg(pr + kHD + 1), xv = __ldcg(pr + t);
                const float Mn = fmaxf(Mx, mv);
                const float f0 = Mx == -INFINITY ? 0.f : exp2f(Mx - Mn);
                const float f1 = mv == -INFINITY ? 0.f : exp2f(mv - Mn);
                Lx = Lx * f0 + lv * f1;
                ax = ax * f0 + xv * f1;
                Mx = Mn;
              }
              const float v = ax / Lx;
              const float w = __shfl_down_sync(0xffffffffu, v, 1);
              __nv_bfloat16* orow = args.out + (int64_t)s * args.out_stride + ((int64_t)h * GQ + hh) * kHD;
              if ((t & 1) == 0) out_pair<PEERS>(args, orow + t, v, w);
              if (args.lse && t == 0) args.lse[(int64_t)s * d.q_heads + h * GQ + hh] = (Mx + log2f(Lx)) * kLn2;
            }
            if (t == 0) ws.attn_done[s * H + h] = 0;
          }
          corr_sync();  // misc[2] is reused by the next piece
        }
      }
      ++j;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == kMma) {
    tc::fence_after();
    tc::tmem_dealloc<kTmemCols>(tmem);
  }
}
