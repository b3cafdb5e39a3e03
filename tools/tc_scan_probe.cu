// tc_scan_probe.cu — operand layout of the tensor-core summary scan with the
// summary rows as the MMA's N dimension: A = one 8-row x 128-byte anchor atom
// (row 0 = hi, row 1 = lo, rows 2-7 = 0) re-read for every 8-row group of
// M = 128 by a zero stride-byte-offset; B = 256 summary rows, K-major SW128 in
// 8-row groups 1 KB apart.  Checks D[lane 32q + 0][n] = hi . row_n and
// D[lane 32q + 1][n] = lo . row_n for every quadrant q.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -o tools/tc_scan_probe tools/tc_scan_probe.cu -lcuda
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cstdint>

#include "../paper_2602_20732_b200/csrc/tc.cuh"

using namespace chess;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t sw(int r, int c) { return (uint32_t)(r * 128 + (((c ^ (r & 7)) & 7) << 4)); }

__global__ void __launch_bounds__(128) probe(const __half* anc, const __half* rows, float* D, int N) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* B = sm;            // 32 groups x 1 KB
  uint8_t* A = sm + 32768;    // 1 KB atom
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < N * 8; i += 128) {  // row r, chunk c (8 chunks of 8 fp16 = 64 elements)
    const int r = i / 8, c = i % 8, g = r / 8, rr = r % 8;
    *reinterpret_cast<uint4*>(B + g * 1024 + sw(rr, c)) = *reinterpret_cast<const uint4*>(rows + r * 64 + c * 8);
  }
  if (t < 64) {
    const int r = t / 8, c = t % 8;
    *reinterpret_cast<uint4*>(A + sw(r, c)) = *reinterpret_cast<const uint4*>(anc + r * 64 + c * 8);
  }
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
    const uint32_t id = tc::idesc_f16(128, N, 0);
    for (int kk = 0; kk < 4; ++kk)
      tc::mma_f16_ss(tmem, tc::smem_desc(su32(A) + kk * 32, 16, 0, 2), tc::smem_desc(su32(B) + kk * 32, 16, 1024, 2), id,
                     kk != 0);
    tc::commit(&bar);
  }
  __syncwarp();
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(&bar))
        : "memory");
  }
  tc::fence_after();
  for (int c0 = 0; c0 < N; c0 += 8) {
    float v[8];
    tc::tmem_ld_x8(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
    for (int j = 0; j < 8; ++j) D[t * 256 + c0 + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc<256>(tmem);
  }
}

int main() {
  srand(3);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  int ok = 1;
  for (int N : {256, 104, 8}) {
    std::vector<__half> anc(8 * 64), rows(256 * 64);
    for (int i = 0; i < 8 * 64; ++i) anc[i] = __float2half(i < 128 ? rnd() : 0.f);
    for (auto& x : rows) x = __float2half(rnd());
    __half *da, *dr;
    float* dD;
    cudaMalloc(&da, anc.size() * 2);
    cudaMalloc(&dr, rows.size() * 2);
    cudaMalloc(&dD, 128 * 256 * 4);
    cudaMemcpy(da, anc.data(), anc.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dr, rows.data(), rows.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 128 * 256 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    probe<<<1, 128, 40 * 1024>>>(da, dr, dD, N);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed N=%d\n", N); return 1; }
    std::vector<float> D(128 * 256);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double mx = 0, mref = 0;
    for (int q = 0; q < 4; ++q)
      for (int ar = 0; ar < 2; ++ar)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int k = 0; k < 64; ++k) ref += (double)__half2float(anc[ar * 64 + k]) * __half2float(rows[n * 64 + k]);
          mx = fmax(mx, fabs(D[(32 * q + ar) * 256 + n] - ref));
          mref = fmax(mref, fabs(ref));
        }
    const bool good = mx <= 1e-3 * mref;
    printf("N=%3d: A atom (sbo 0) x B rows: max|err| %.3e (max|ref| %.3e) %s\n", N, mx, mref, good ? "OK" : "MISMATCH");
    ok &= good;
  }
  return ok ? 0 : 2;
}
