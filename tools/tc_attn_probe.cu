// tc_attn_probe.cu — checks the shared-memory operand layouts the tensor-core
// decode attention (K4 tcgen05 consumer) relies on, one MMA form at a time,
// against a host reference.  Standalone (no library):
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -o tools/tc_attn_probe tools/tc_attn_probe.cu -lcuda
//   ./tools/tc_attn_probe
//
//  QK : S[128 tok][8] = K[128 tok][128 d] . q[8][128 d]^T
//       A = K  K-major SW128 ([cb][128 rows][128 B]),  B = q K-major SW128 ([cb][8 rows][128 B])
//  PV : O^T[128 d][8] = V^T[128 d][128 tok] . P^T
//       A = V  MN-major SW128 ([cb][128 tok][128 B]: d contiguous), LBO = cb stride, SBO = 8-row stride
//       B = P  MN-major no-swizzle (token t, head h at t*16 + 2h) or K-major SW128 ([tb][8 h][128 B])
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cstdint>

#include "../paper_2602_20732_b200/csrc/tc.cuh"

using namespace chess;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fffu);
  d |= (uint64_t)((lbo >> 4) & 0x3fffu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fffu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc(int M, int N, int amaj, int bmaj) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// swizzled byte offset of 16-byte chunk c of 128-byte row r (1024-aligned atoms)
__device__ __forceinline__ uint32_t sw(int r, int c) { return (uint32_t)(r * 128 + (((c ^ (r & 7)) & 7) << 4)); }

struct Args {
  const __nv_bfloat16* K;  // [128][128]
  const __nv_bfloat16* q;  // [8][128]
  const __nv_bfloat16* V;  // [128][128]
  const __nv_bfloat16* P;  // [128 tok][8]
  float* S;                // [128][8]
  float* O;                // [128 d][8]
  int form;                // 0: QK; 1: PV (P interleave); 2: PV (P K-major SW128); 3: QK with M = 64
  uint32_t lbo_a, sbo_a, lbo_b, sbo_b;
};

__global__ void __launch_bounds__(128) probe(Args a) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = sm;             // 32 KB
  uint8_t* Bq = sm + 32768;    // 2 KB (q / P)
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // stage operands
  if (a.form == 3) {
    for (int i = t; i < 64 * 16; i += 128) {  // K rows 0..63: [cb][64 rows][128 B]
      const int r = i / 16, c = i % 16, cb = c / 8;
      *reinterpret_cast<uint4*>(A + cb * 8192 + sw(r, c & 7)) = *reinterpret_cast<const uint4*>(a.K + r * 128 + c * 8);
    }
    for (int i = t; i < 8 * 16; i += 128) {
      const int r = i / 16, c = i % 16, cb = c / 8;
      *reinterpret_cast<uint4*>(Bq + cb * 1024 + sw(r, c & 7)) = *reinterpret_cast<const uint4*>(a.q + r * 128 + c * 8);
    }
  } else if (a.form == 0) {
    for (int i = t; i < 128 * 16; i += 128) {  // K: row r, chunk c (16 chunks of 8 elems)
      const int r = i / 16, c = i % 16, cb = c / 8;
      *reinterpret_cast<uint4*>(A + cb * 16384 + sw(r, c & 7)) = *reinterpret_cast<const uint4*>(a.K + r * 128 + c * 8);
    }
    for (int i = t; i < 8 * 16; i += 128) {
      const int r = i / 16, c = i % 16, cb = c / 8;
      *reinterpret_cast<uint4*>(Bq + cb * 1024 + sw(r, c & 7)) = *reinterpret_cast<const uint4*>(a.q + r * 128 + c * 8);
    }
  } else {
    for (int i = t; i < 128 * 16; i += 128) {  // V: token r, d-chunk c
      const int r = i / 16, c = i % 16, cb = c / 8;
      *reinterpret_cast<uint4*>(A + cb * 16384 + sw(r, c & 7)) = *reinterpret_cast<const uint4*>(a.V + r * 128 + c * 8);
    }
    if (a.form == 1) {
      // token t: 8 heads, 16 B at t*16
      *reinterpret_cast<uint4*>(Bq + t * 16) = *reinterpret_cast<const uint4*>(a.P + t * 8);
    } else {
      // K-major SW128: [tb = t/64][8 head rows][128 B of 64 tokens]
      for (int h = 0; h < 8; ++h) {
        const int tb = t / 64, tt = t % 64;
        *reinterpret_cast<__nv_bfloat16*>(Bq + tb * 1024 + h * 128 + ((((tt >> 3) ^ h) & 7) << 4) + (tt & 7) * 2) =
            a.P[t * 8 + h];
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    tc::tmem_alloc<32>(&tm);
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tm;
  if (t == 0) {
    const uint32_t sa = su32(A), sb = su32(Bq);
    if (a.form == 3) {
      const uint32_t id = idesc(64, 8, 0, 0);
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t off = (ks / 4) * 8192 + (ks % 4) * 32;
        const uint32_t offb = (ks / 4) * 1024 + (ks % 4) * 32;
        tc::mma_f16_ss(tmem, desc(sa + off, 16, 1024, 2), desc(sb + offb, 16, 1024, 2), id, ks != 0);
      }
    } else if (a.form == 0) {
      const uint32_t id = idesc(128, 8, 0, 0);
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t off = (ks / 4) * 16384 + (ks % 4) * 32;
        const uint32_t offb = (ks / 4) * 1024 + (ks % 4) * 32;
        tc::mma_f16_ss(tmem, desc(sa + off, a.lbo_a, a.sbo_a, 2), desc(sb + offb, a.lbo_b, a.sbo_b, 2), id, ks != 0);
      }
    } else {
      const uint32_t id = idesc(128, 8, 1, a.form == 1 ? 1 : 0);
      for (int ks = 0; ks < 8; ++ks) {  // 16 tokens per MMA
        const uint32_t offa = ks * 2048;  // 2 groups of 8 token rows
        uint64_t bd;
        if (a.form == 1) bd = desc(sb + ks * 256, a.lbo_b, a.sbo_b, 0);
        else bd = desc(sb + (ks / 4) * 1024 + (ks % 4) * 32, a.lbo_b, a.sbo_b, 2);
        tc::mma_f16_ss(tmem + 8, desc(sa + offa, a.lbo_a, a.sbo_a, 2), bd, id, ks != 0);
      }
    }
    tc::commit(&bar);
  }
  __syncwarp();
  // wait
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(su32(&bar))
          : "memory");
    }
  }
  tc::fence_after();
  uint32_t r[8];
  const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + ((a.form == 0 || a.form == 3) ? 0u : 8u);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  float* out = (a.form == 0 || a.form == 3) ? a.S : a.O;
  for (int j = 0; j < 8; ++j) out[t * 8 + j] = __uint_as_float(r[j]);
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc<32>(tmem);
  }
}

// MMA latency: `reps` rounds of {8 MMAs (M128 N8 K16) into `nacc` accumulators, commit, wait}
__global__ void __launch_bounds__(128) mma_latency(int nacc, int reps, long long* cycles, int nmma = 8, int slot = -1, int N = 8, int M = 128) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 65536 / 16; i += 128) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tc::tmem_alloc<256>(&tm);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tm;
  if (t == 0) {
    const uint32_t sa = su32(sm), sb = su32(sm + 32768);
    const uint32_t id = idesc(M, N, 0, 0);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int ks = 0; ks < nmma; ++ks) {
        const int acc = ks % nacc;
        const uint32_t off = ((ks / 4) & 1) * 16384 + (ks % 4) * 32;
        tc::mma_f16_ss(tmem + acc * 8, desc(sa + off, 16, 1024, 2), desc(sb + ((ks / 4) & 1) * 1024 + (ks % 4) * 32, 16, 1024, 2), id, ks >= nacc);
      }
      tc::commit(&bar);
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(su32(&bar)), "r"(r & 1)
            : "memory");
      }
    }
    cycles[slot >= 0 ? slot : nacc] = (clock64() - t0) / reps;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc<256>(tmem);
  }
}

static float bf(const __nv_bfloat16& x) { return __bfloat162float(x); }

int main() {
  srand(1);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  std::vector<__nv_bfloat16> K(128 * 128), q(8 * 128), V(128 * 128), P(128 * 8);
  for (auto& x : K) x = __float2bfloat16(rnd());
  for (auto& x : q) x = __float2bfloat16(rnd());
  for (auto& x : V) x = __float2bfloat16(rnd());
  for (auto& x : P) x = __float2bfloat16(rnd());
  std::vector<double> Sref(128 * 8), Oref(128 * 8);
  for (int i = 0; i < 128; ++i)
    for (int h = 0; h < 8; ++h) {
      double s = 0;
      for (int k = 0; k < 128; ++k) s += (double)bf(K[i * 128 + k]) * bf(q[h * 128 + k]);
      Sref[i * 8 + h] = s;
    }
  for (int dd = 0; dd < 128; ++dd)
    for (int h = 0; h < 8; ++h) {
      double s = 0;
      for (int tk = 0; tk < 128; ++tk) s += (double)bf(V[tk * 128 + dd]) * bf(P[tk * 8 + h]);
      Oref[dd * 8 + h] = s;
    }
  __nv_bfloat16 *dK, *dq, *dV, *dP;
  float *dS, *dO;
  cudaMalloc(&dK, K.size() * 2);
  cudaMalloc(&dq, q.size() * 2);
  cudaMalloc(&dV, V.size() * 2);
  cudaMalloc(&dP, P.size() * 2);
  cudaMalloc(&dS, 128 * 8 * 4);
  cudaMalloc(&dO, 128 * 8 * 4);
  cudaMemcpy(dK, K.data(), K.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  struct V_ {
    const char* name;
    int form;
    uint32_t la, sa, lb, sb;
  } vs[] = {
      {"QK  A:K-major SW128 (lbo 16, sbo 1024)  B:K-major SW128", 0, 16, 1024, 16, 1024},
      {"PV  A:MN SW128 lbo=16K sbo=1K  B:MN interleave lbo=128 sbo=2048", 1, 16384, 1024, 128, 2048},
      {"PV  A:MN SW128 lbo=1K sbo=16K  B:MN interleave lbo=128 sbo=2048", 1, 1024, 16384, 128, 2048},
      {"PV  A:MN SW128 lbo=16K sbo=1K  B:MN interleave lbo=2048 sbo=128", 1, 16384, 1024, 2048, 128},
      {"PV  A:MN SW128 lbo=1K sbo=16K  B:MN interleave lbo=2048 sbo=128", 1, 1024, 16384, 2048, 128},
      {"PV  A:MN SW128 lbo=16K sbo=1K  B:K-major SW128", 2, 16384, 1024, 16, 1024},
      {"PV  A:MN SW128 lbo=1K sbo=16K  B:K-major SW128", 2, 1024, 16384, 16, 1024},
  };
  int ok_all = 1;
  {
    long long* dc;
    cudaMalloc(&dc, 16 * 8);
    cudaFuncSetAttribute(mma_latency, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    for (int nacc : {1, 2, 4, 8}) mma_latency<<<1, 128, 80 * 1024>>>(nacc, 200, dc);
    cudaDeviceSynchronize();
    long long hc[16];
    cudaMemcpy(hc, dc, 16 * 8, cudaMemcpyDeviceToHost);
    printf("MMA round trip (8 x M128N8K16 + commit + wait), cycles: 1 acc %lld, 2 acc %lld, 4 acc %lld, 8 acc %lld\n",
           hc[1], hc[2], hc[4], hc[8]);
    int ns[6] = {1, 2, 4, 8, 16, 32};
    for (int i = 0; i < 6; ++i) mma_latency<<<1, 128, 80 * 1024>>>(1, 200, dc, ns[i], i, 8);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, dc, 16 * 8, cudaMemcpyDeviceToHost);
    printf("N=8 round trip vs MMAs per round: 1: %lld 2: %lld 4: %lld 8: %lld 16: %lld 32: %lld\n", hc[0], hc[1], hc[2], hc[3], hc[4], hc[5]);
    for (int i = 0; i < 6; ++i) mma_latency<<<1, 128, 80 * 1024>>>(1, 200, dc, ns[i], i, 32);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, dc, 16 * 8, cudaMemcpyDeviceToHost);
    printf("N=32 round trip vs MMAs per round: 1: %lld 2: %lld 4: %lld 8: %lld 16: %lld 32: %lld\n", hc[0], hc[1], hc[2], hc[3], hc[4], hc[5]);
    int nn[6] = {8, 16, 64, 128, 256, 0};
    for (int i = 0; i < 5; ++i) mma_latency<<<1, 128, 80 * 1024>>>(1, 200, dc, 16, i, nn[i], 128);
    mma_latency<<<1, 128, 80 * 1024>>>(1, 200, dc, 16, 5, 8, 64);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, dc, 16 * 8, cudaMemcpyDeviceToHost);
    printf("16 MMAs M=128 by N: 8: %lld 16: %lld 64: %lld 128: %lld 256: %lld | M=64 N=8: %lld\n", hc[0], hc[1], hc[2], hc[3], hc[4], hc[5]);
  }
  {
    // M = 64: where does row i of S land in TMEM (lane, column)?
    Args a{dK, dq, dV, dP, dS, dO, 3, 16, 1024, 16, 1024};
    cudaMemset(dS, 0, 128 * 8 * 4);
    probe<<<1, 128, 40 * 1024>>>(a);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("M=64 probe failed\n"); return 1; }
    std::vector<float> got(128 * 8);
    cudaMemcpy(got.data(), dS, 128 * 8 * 4, cudaMemcpyDeviceToHost);
    printf("M=64 QK: TMEM lane of S row i (col 0) [first 64 rows]:");
    int okm = 1;
    for (int i = 0; i < 64; ++i) {
      int where = -1;
      for (int ln = 0; ln < 128; ++ln)
        if (fabs(got[ln * 8] - Sref[i * 8]) <= 1e-3 * (1 + fabs(Sref[i * 8]))) { where = ln; break; }
      printf(" %d", where);
      if (where >= 0) for (int h = 0; h < 8; ++h) okm &= fabs(got[where * 8 + h] - Sref[i * 8 + h]) <= 1e-3 * (1 + fabs(Sref[i * 8 + h]));
      else okm = 0;
    }
    printf("\nM=64 QK rows found with all 8 columns in one lane: %s\n", okm ? "yes" : "no");
  }
  for (auto& v : vs) {
    Args a{dK, dq, dV, dP, dS, dO, v.form, v.la, v.sa, v.lb, v.sb};
    cudaMemset(dS, 0, 128 * 8 * 4);
    cudaMemset(dO, 0, 128 * 8 * 4);
    probe<<<1, 128, 40 * 1024>>>(a);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%-70s CUDA error %s\n", v.name, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> got(128 * 8);
    cudaMemcpy(got.data(), v.form == 0 ? dS : dO, 128 * 8 * 4, cudaMemcpyDeviceToHost);
    const auto& ref = v.form == 0 ? Sref : Oref;
    double mx = 0, mref = 0;
    for (int i = 0; i < 128 * 8; ++i) {
      mx = fmax(mx, fabs(got[i] - ref[i]));
      mref = fmax(mref, fabs(ref[i]));
    }
    const bool ok = mx <= 1e-3 * mref;
    printf("%-70s max|err| %.3e (max|ref| %.3e) %s\n", v.name, mx, mref, ok ? "OK" : "MISMATCH");
    if (v.form == 0) ok_all &= ok;
  }
  return ok_all ? 0 : 2;
}
