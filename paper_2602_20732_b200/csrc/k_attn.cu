// k_attn.cu — K4 sparse paged decode attention over the CHESS block table.
//
// Not present in the reference: pagesel only counts attention work
// (simulate.py:186, B*2*|WS|*B*D).  The paper runs FlashInfer's paged decode
// over the reconstructed context; oracle restated in
// oracle/attention.py (fp64 softmax(q K^T / sqrt(d)) V over the working set
// in increasing logical order; rows >= fill never contribute).
//
// B200 design:
//  * unit of work = 16 tokens of one (slot, kv head, page); the units of a
//    layer are cut into equal contiguous ranges, one per WARP (stream-K over
//    8 warps x 148 SMs), so every warp streams the same bytes (+-1 unit);
//  * every warp is its own producer: lane 0 issues 2-D TMA tensor loads
//    (cp.async.bulk.tensor, 128B swizzle, 8-row boxes) of the unit's K and V
//    into a private 3-stage shared-memory ring guarded by mbarriers — no
//    CTA-wide barrier anywhere in the main loop;
//  * QK^T and PV run on the tensor cores with mma.sync m16n8k16 (bf16 in,
//    fp32 accumulate): the GQA group's q heads fill the M=16 rows, tokens are
//    N (QK) / K (PV); ldmatrix reads the swizzled tiles conflict-free and the
//    S accumulator fragments are reused in registers as the P operand;
//  * segments split across warps are merged by the last warp to finish
//    (atomic counter), in warp order — deterministic.
#include <cudaTypedefs.h>

#include "common.cuh"

namespace chess {

namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kThreads = kWarpsPerCta * 32;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct AttnArgs {
  const __nv_bfloat16* q;
  int64_t q_stride;
  __nv_bfloat16* out;
  int64_t out_stride;
  float* lse;
  float scale_log2;  // softmax_scale * log2(e)
  int layer;
};

template <int HD, int GQ, int B>
struct Cfg {
  static constexpr int kUT = 16;                     // tokens per unit
  static constexpr int kUPP = B / kUT;               // units per page
  static constexpr int kHalves = HD / 64;            // 128-byte column boxes
  static constexpr int kUnitBytes = kUT * HD * 2;    // K (or V) bytes of a unit
  static constexpr int kStageBytes = 2 * kUnitBytes;
  static constexpr int kStages = HD == 128 ? 3 : 6;  // per warp
  static constexpr int kNT = HD / 8;                 // PV n-tiles
  static constexpr int kKS = HD / 16;                // QK k-steps
  static constexpr size_t kSmem = (size_t)kWarpsPerCta * kStages * kStageBytes + 1024 /*align*/ +
                                  kWarpsPerCta * kStages * 8 + (kMaxBatch + 1) * 4;
};

__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
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

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// swizzled (128B) address of 16-byte chunk `chunk` (0..HD/8-1) of tile row `row`
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + (uint32_t)((chunk >> 3) * (16 * 128) + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
}

struct Unit {
  int s, h, j;   // slot, kv head, unit index within the segment
  int ups;       // units in this segment
  int64_t seg_begin;
};

template <int HD, int GQ, int B>
__global__ void __launch_bounds__(kThreads, 1)
    sparse_decode_kernel(ChessState st, Workspace ws, AttnArgs args,
                         const __grid_constant__ CUtensorMap kmap,
                         const __grid_constant__ CUtensorMap vmap) {
  using C = Cfg<HD, GQ, B>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stages = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + (size_t)kWarpsPerCta * C::kStages * C::kStageBytes);
  int* prefix = reinterpret_cast<int*>(bars + kWarpsPerCta * C::kStages);
  const ChessDims& d = st.d;
  const int H = d.kv_heads;
  const int nb = d.batch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  pdl_wait();
  // units per slot: H * ((ws_len-1)*UPP + ceil(fill/16)); prefix over slots
  if (warp == 0) {
    int run = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int s = b0 + lane;
      int x = 0;
      if (s < nb) {
        const int wl = st.ws_len[s];
        if (wl > 0) x = H * ((wl - 1) * C::kUPP + (st.tail_fill[s] + C::kUT - 1) / C::kUT);
      }
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
  }
  __syncthreads();
  pdl_launch_dependents();

  const int64_t N = prefix[nb];
  const int64_t NW = min((int64_t)gridDim.x * kWarpsPerCta, N);
  const int64_t gw = (int64_t)blockIdx.x * kWarpsPerCta + warp;
  if (gw >= NW) return;
  const int64_t u_begin = gw * N / NW, u_end = (gw + 1) * N / NW;
  const int n_units = (int)(u_end - u_begin);

  uint8_t* my_stages = stages + (size_t)warp * C::kStages * C::kStageBytes;
  uint64_t* my_bars = bars + warp * C::kStages;
  if (lane == 0) {
    for (int i = 0; i < C::kStages; ++i) mbar_init(&my_bars[i], 1);
    fence_barrier_init();
  }
  __syncwarp();

  // ---- unit walker ----
  auto locate = [&](int64_t u) {
    int lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (prefix[mid] <= u) lo = mid; else hi = mid;
    }
    Unit x;
    x.s = lo;
    const int wl = st.ws_len[lo];
    x.ups = (wl - 1) * C::kUPP + (st.tail_fill[lo] + C::kUT - 1) / C::kUT;
    const int64_t r = u - prefix[lo];
    x.h = (int)(r / x.ups);
    x.j = (int)(r - (int64_t)x.h * x.ups);
    x.seg_begin = prefix[lo] + (int64_t)x.h * x.ups;
    return x;
  };
  auto advance = [&](Unit& x) {
    if (++x.j >= x.ups) {
      x.seg_begin += x.ups;
      x.j = 0;
      if (++x.h >= H) {
        x.h = 0;
        do {
          ++x.s;
        } while (x.s < nb && st.ws_len[x.s] == 0);
        if (x.s < nb)
          x.ups = (st.ws_len[x.s] - 1) * C::kUPP + (st.tail_fill[x.s] + C::kUT - 1) / C::kUT;
      }
    }
  };
  auto unit_rows = [&](const Unit& x) {
    const int page = x.j / C::kUPP;
    const int half = x.j - page * C::kUPP;
    const int wl = st.ws_len[x.s];
    const int fill = (page == wl - 1) ? st.tail_fill[x.s] : B;
    return min(C::kUT, fill - half * C::kUT);
  };

  // ---- producer (lane 0): TMA loads of unit x into stage ----
  auto issue = [&](const Unit& x, int stage) {
    const int page = x.j / C::kUPP;
    const int half = x.j - page * C::kUPP;
    const int valid = unit_rows(x);
    const int nrb = valid > 8 ? 2 : 1;
    const int64_t phys = st.block_table[(int64_t)x.s * d.max_ws + page];
    const int row0 = (int)((phys * H + x.h) * B + half * C::kUT);
    const uint32_t bar = smem_u32(&my_bars[stage]);
    const uint32_t kdst = smem_u32(my_stages + (size_t)stage * C::kStageBytes);
    const uint32_t vdst = kdst + C::kUnitBytes;
    mbar_arrive_expect_tx(&my_bars[stage], (uint32_t)(2 * C::kHalves * nrb * 1024));
#pragma unroll
    for (int hb = 0; hb < C::kHalves; ++hb) {
      for (int rb = 0; rb < nrb; ++rb) {
        const uint32_t off = hb * (C::kUT * 128) + rb * 1024;
        tma_load_3d(kdst + off, &kmap, hb * 64, row0 + rb * 8, args.layer, bar);
        tma_load_3d(vdst + off, &vmap, hb * 64, row0 + rb * 8, args.layer, bar);
      }
    }
  };

  Unit cu = locate(u_begin);
  {
    Unit pu = cu;
    if (lane == 0) {
      for (int k = 0; k < C::kStages && k < n_units; ++k) {
        issue(pu, k);
        advance(pu);
      }
    }
  }
  Unit pu = cu;  // producer cursor (lane 0 only meaningful), kStages ahead
  for (int k = 0; k < C::kStages && k < n_units; ++k) advance(pu);

  // ---- consumer state ----
  const int g = lane >> 2, t = lane & 3;
  uint32_t qa[C::kKS][2];
  float o[C::kNT][4];
  float m_run, l_run;
  auto load_q = [&](const Unit& x) {
    const __nv_bfloat16* qp = args.q + (int64_t)x.s * args.q_stride + ((int64_t)x.h * GQ + g) * HD;
#pragma unroll
    for (int kk = 0; kk < C::kKS; ++kk) {
      if (g < GQ) {
        qa[kk][0] = *reinterpret_cast<const uint32_t*>(qp + kk * 16 + 2 * t);
        qa[kk][1] = *reinterpret_cast<const uint32_t*>(qp + kk * 16 + 8 + 2 * t);
      } else {
        qa[kk][0] = qa[kk][1] = 0u;
      }
    }
#pragma unroll
    for (int nt = 0; nt < C::kNT; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    m_run = -INFINITY;
    l_run = 0.f;
  };
  load_q(cu);

  const int mr = lane & 7, mm = lane >> 3;  // ldmatrix row / matrix of this lane
  for (int k = 0; k < n_units; ++k) {
    const int stage = k % C::kStages;
    const uint32_t parity = (uint32_t)((k / C::kStages) & 1);
    const int valid = unit_rows(cu);
    mbar_wait(&my_bars[stage], parity);
    uint8_t* kst_p = my_stages + (size_t)stage * C::kStageBytes;
    const uint32_t kst = smem_u32(kst_p);
    const uint32_t vst = kst + C::kUnitBytes;
    if (valid < C::kUT) {
      // rows >= valid hold stale / never-written data: zero V so P*V stays finite
      for (int idx = lane; idx < (C::kUT - valid) * C::kHalves * 8; idx += 32) {
        const int r = valid + idx / (C::kHalves * 8);
        const int ch = idx % (C::kHalves * 8);
        *reinterpret_cast<uint4*>(kst_p + C::kUnitBytes + (swz(0, r, ch))) = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
    }

    // ---- S = Q K^T (16 q rows x 16 tokens) ----
    float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kp = 0; kp < C::kKS / 2; ++kp) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t b[4];
        ldsm_x4(swz(kst, 8 * j + mr, 4 * kp + mm), b);
        mma_bf16(sacc[j], qa[2 * kp][0], 0u, qa[2 * kp][1], 0u, b[0], b[1]);
        mma_bf16(sacc[j], qa[2 * kp + 1][0], 0u, qa[2 * kp + 1][1], 0u, b[2], b[3]);
      }
    }
    // ---- online softmax over this unit's tokens (row g) ----
    float sv[4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = 8 * j + 2 * t + e;
        const float x = sacc[j][e] * args.scale_log2;
        sv[2 * j + e] = (tok < valid && x == x) ? x : -INFINITY;
      }
    }
    float mx = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    const float alpha = exp2f(m_run - m_new);
    float p[4], ps = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      p[e] = exp2f(sv[e] - m_new);
      ps += p[e];
    }
    ps += __shfl_xor_sync(0xffffffffu, ps, 1);
    ps += __shfl_xor_sync(0xffffffffu, ps, 2);
    l_run = l_run * alpha + ps;
    m_run = m_new;
#pragma unroll
    for (int nt = 0; nt < C::kNT; ++nt) {
      o[nt][0] *= alpha;
      o[nt][1] *= alpha;
    }
    const uint32_t pa0 = pack_bf16(p[0], p[1]);
    const uint32_t pa2 = pack_bf16(p[2], p[3]);
    // ---- O += P V ----
#pragma unroll
    for (int np = 0; np < C::kNT / 2; ++np) {
      uint32_t v[4];
      ldsm_x4_t(swz(vst, ((mm & 1) << 3) + mr, 2 * np + (mm >> 1)), v);
      mma_bf16(o[2 * np], pa0, 0u, pa2, 0u, v[0], v[1]);
      mma_bf16(o[2 * np + 1], pa0, 0u, pa2, 0u, v[2], v[3]);
    }
    __syncwarp();
    // refill this stage with the unit kStages ahead
    if (k + C::kStages < n_units) {
      if (lane == 0) {
        fence_proxy_async();
        issue(pu, stage);
      }
      advance(pu);
    }

    // ---- segment flush ----
    const bool seg_end = (cu.j == cu.ups - 1) || (k == n_units - 1);
    if (seg_end) {
      const int64_t sb = cu.seg_begin, se = cu.seg_begin + cu.ups;
      const bool whole = sb >= u_begin && se <= u_end;
      const int sg = cu.s * H + cu.h;
      const int64_t qrow = (int64_t)cu.s * args.out_stride + (int64_t)cu.h * GQ * HD;
      if (whole) {
        if (g < GQ) {
          const float inv = 1.f / l_run;
#pragma unroll
          for (int nt = 0; nt < C::kNT; ++nt) {
            *reinterpret_cast<__nv_bfloat162*>(args.out + qrow + g * HD + nt * 8 + 2 * t) =
                __floats2bfloat162_rn(o[nt][0] * inv, o[nt][1] * inv);
          }
          if (args.lse && t == 0)
            args.lse[(int64_t)cu.s * d.q_heads + cu.h * GQ + g] = (m_run + log2f(l_run)) * kLn2;
        }
      } else {
        // partial slot (sg + gw): O [GQ][HD+4] (16-B aligned rows), m at +HD, l at +HD+1
        constexpr int kRow = HD + 4;
        float* slot = ws.attn_part + (int64_t)(sg + gw) * GQ * kRow;
        if (g < GQ) {
#pragma unroll
          for (int nt = 0; nt < C::kNT; ++nt)
            *reinterpret_cast<float2*>(slot + g * kRow + nt * 8 + 2 * t) = make_float2(o[nt][0], o[nt][1]);
          if (t == 0) {
            slot[g * kRow + HD] = m_run;
            slot[g * kRow + HD + 1] = l_run;
          }
        }
        __syncwarp();
        const int64_t w_first = ((sb + 1) * NW + N - 1) / N - 1;
        const int64_t w_last = (se * NW + N - 1) / N - 1;
        int last = 0;
        if (lane == 0) {
          __threadfence();
          last = atomicAdd(&ws.attn_done[sg], 1) == (int)(w_last - w_first);
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          __threadfence();
          // merge in warp order: per head M = max m_w, L = sum l_w 2^(m_w - M);
          // each lane owns EPL consecutive elements of one head.
          const float* base = ws.attn_part + (sg + w_first) * GQ * kRow;
          const int nsl = (int)(w_last - w_first + 1);
          float M[GQ], L[GQ];
#pragma unroll
          for (int gg = 0; gg < GQ; ++gg) {
            float mx = -INFINITY;
            for (int w2 = lane; w2 < nsl; w2 += 32) mx = fmaxf(mx, __ldcg(base + (int64_t)w2 * GQ * kRow + gg * kRow + HD));
#pragma unroll
            for (int o2 = 16; o2 >= 1; o2 >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
            float sum = 0.f;
            for (int w2 = lane; w2 < nsl; w2 += 32) {
              const float* sl = base + (int64_t)w2 * GQ * kRow + gg * kRow;
              sum += __ldcg(sl + HD + 1) * exp2f(__ldcg(sl + HD) - mx);
            }
#pragma unroll
            for (int o2 = 16; o2 >= 1; o2 >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o2);
            M[gg] = mx;
            L[gg] = sum;
          }
          constexpr int kEPL = GQ * HD / 32;
          const int e0 = lane * kEPL;
          const int gl = e0 / HD, el = e0 - gl * HD;
          float Mg = M[0], Lg = L[0];
#pragma unroll
          for (int gg = 1; gg < GQ; ++gg)
            if (gl == gg) { Mg = M[gg]; Lg = L[gg]; }
          float acc[kEPL];
#pragma unroll
          for (int e = 0; e < kEPL; ++e) acc[e] = 0.f;
          for (int w2 = 0; w2 < nsl; ++w2) {
            const float* sl = base + (int64_t)w2 * GQ * kRow + gl * kRow;
            const float f = exp2f(__ldcg(sl + HD) - Mg);
#pragma unroll
            for (int e = 0; e < kEPL; e += 2) {
              const float2 x = __ldcg(reinterpret_cast<const float2*>(sl + el + e));
              acc[e] = fmaf(x.x, f, acc[e]);
              acc[e + 1] = fmaf(x.y, f, acc[e + 1]);
            }
          }
          const float inv = 1.f / Lg;
#pragma unroll
          for (int e = 0; e < kEPL; e += 2)
            *reinterpret_cast<__nv_bfloat162*>(args.out + qrow + gl * HD + el + e) =
                __floats2bfloat162_rn(acc[e] * inv, acc[e + 1] * inv);
          if (args.lse && el == 0)
            args.lse[(int64_t)cu.s * d.q_heads + cu.h * GQ + gl] = (Mg + log2f(Lg)) * kLn2;
          if (lane == 0) ws.attn_done[sg] = 0;
        }
      }
      advance(cu);
      if (k + 1 < n_units) load_q(cu);
    } else {
      advance(cu);
    }
  }
}

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

// 3-D view [layers][n_phys*kv_heads*page][head_dim] of a KV pool; 8-row x
// 64-column boxes with 128-byte swizzle.
int make_kv_map(CUtensorMap* m, const void* base, const ChessDims& d) {
  auto fn = encode_fn();
  if (!fn) return fail(CHESS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t rows = (cuuint64_t)d.n_phys * d.kv_heads * d.page_size;
  cuuint64_t dims[3] = {(cuuint64_t)d.head_dim, rows, (cuuint64_t)d.layers};
  cuuint64_t strides[2] = {(cuuint64_t)d.head_dim * 2, rows * d.head_dim * 2};
  cuuint32_t box[3] = {64, 8, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHESS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return CHESS_OK;
}

template <int HD, int GQ, int B>
int launch_inst(const ChessState& st, const Workspace& ws, const AttnArgs& args, int nctas,
                cudaStream_t stream) {
  using C = Cfg<HD, GQ, B>;
  const size_t smem = C::kSmem;
  static bool configured = false;
  auto kfn = sparse_decode_kernel<HD, GQ, B>;
  if (!configured) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kfn, st, ws, args, km, vm);
  return check_launch("sparse_decode");
}

}  // namespace

int attn_ctas_for(const ChessDims& d) {
  (void)d;
  return num_sms();
}

int launch_sparse_decode(const ChessState& st, const Workspace& ws, int layer, const void* q,
                         int64_t q_stride, void* out, int64_t out_stride, float* lse,
                         float softmax_scale, cudaStream_t stream) {
  const ChessDims& d = st.d;
  AttnArgs a;
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.q_stride = q_stride;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.out_stride = out_stride;
  a.lse = lse;
  a.scale_log2 = softmax_scale * kLog2e;
  a.layer = layer;
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
