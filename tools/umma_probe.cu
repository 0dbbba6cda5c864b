// umma_probe.cu — one-CTA probe of the tensor-core blur building blocks (k_tc):
// block-Toeplitz descriptors (SS MMA, row pass), in-place fp16 hi/lo split in TMEM and
// the TMEM-A MMA (TS, column pass).  Compares D1 and D2 with f64 host sums.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2108_12050_b200/csrc tools/umma_probe.cu -o tools/umma_probe
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "tc_plan.h"
#include "umma.cuh"

using namespace mhfd;

__device__ __forceinline__ void mbar_init_(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(umma::smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait_(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(umma::smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// X: S x S int (values -128..127); tab: the level's [hi | lo] pair block
__global__ void __launch_bounds__(512, 1) probe(const int* X, int S, const uint8_t* tab, int tab_bytes, int c0, int K,
                                                float* d1, float* d2) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* B1 = sm;                                   // S x S fp16 canonical K-major
  uint8_t* T = B1 + (size_t)S * S * 2;                // table
  uint64_t* bar = reinterpret_cast<uint64_t*>(T + ((tab_bytes + 15) & ~15));
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int SBO1 = (S / 8) * 128;
  for (int i = tid; i < S * S; i += 512) {
    const int r = i / S, k = i % S;
    __half h = __int2half_rn(X[i]);
    *reinterpret_cast<__half*>(B1 + (r / 8) * SBO1 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) = h;
  }
  for (int i = tid; i < tab_bytes / 4; i += 512) reinterpret_cast<uint32_t*>(T)[i] = reinterpret_cast<const uint32_t*>(tab)[i];
  if (tid == 0) { mbar_init_(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) umma::tmem_alloc(tslot, 512);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tbase = *tslot;
  const int npairs = K / 8 + 14;
  const int E1 = K / 8 - 2;
  const uint32_t thi = umma::smem_addr(T), tlo = thi + npairs * 256;
  const uint32_t b1 = umma::smem_addr(B1) + (c0 / 8) * SBO1 + (c0 / 8) * 128;
  if (tid == 0) {
    const uint32_t id = umma::idesc_f16(128, K);
    for (int j = 0; j < K / 16; ++j) {
      const uint64_t bd = umma::desc_kmajor(b1 + 256 * j, 128, SBO1);
      umma::mma_ss(tbase, umma::desc_kmajor(thi + (E1 - 2 * j) * 256, 128, 256), bd, id, j > 0);
      umma::mma_ss(tbase, umma::desc_kmajor(tlo + (E1 - 2 * j) * 256, 128, 256), bd, id, 1);
    }
    umma::commit(bar);
  }
  mbar_wait_(bar, 0);
  umma::fence_after();
  const int q = warp & 3, wg = warp >> 2;
  const uint32_t lane_addr = tbase + ((uint32_t)(32 * q) << 16);
  const int c = 32 * q + (tid & 31);
  // dump D1 and split in place (chunks j = wg, wg+4, ...)
  for (int j = wg; j < K / 16; j += 4) {
    uint32_t r[16];
    umma::ld16(lane_addr + 16 * j, r);
    umma::wait_ld();
    uint32_t h[8], l[8];
#pragma unroll
    for (int u = 0; u < 16; ++u) d1[(size_t)c * K + 16 * j + u] = __uint_as_float(r[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float y0 = __uint_as_float(r[2 * u]) * (1.f / kTcWScale), y1 = __uint_as_float(r[2 * u + 1]) * (1.f / kTcWScale);
      const __half h0 = __float2half_rn(y0), h1 = __float2half_rn(y1);
      const __half l0 = __float2half_rn(y0 - __half2float(h0)), l1 = __float2half_rn(y1 - __half2float(h1));
      h[u] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
      l[u] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
    }
    umma::st8(lane_addr + 16 * j, h);
    umma::st8(lane_addr + 16 * j + 8, l);
  }
  umma::wait_st();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  if (tid == 0) {
    const uint32_t id = umma::idesc_f16(128, 128);
    for (int j = 0; j < K / 16; ++j) {
      const uint64_t bh = umma::desc_kmajor(thi + (E1 - 2 * j) * 256, 128, 256);
      const uint64_t bl = umma::desc_kmajor(tlo + (E1 - 2 * j) * 256, 128, 256);
      umma::mma_ts(tbase + 256, tbase + 16 * j, bh, id, j > 0);
      umma::mma_ts(tbase + 256, tbase + 16 * j, bl, id, 1);
      umma::mma_ts(tbase + 256, tbase + 16 * j + 8, bh, id, 1);
    }
    umma::commit(bar);
  }
  mbar_wait_(bar, 1);
  umma::fence_after();
  for (int j = wg; j < 8; j += 4) {
    uint32_t r[16];
    umma::ld16(lane_addr + 256 + 16 * j, r);
    umma::wait_ld();
#pragma unroll
    for (int u = 0; u < 16; ++u) d2[(size_t)c * 128 + 16 * j + u] = __uint_as_float(r[u]);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tbase, 512);
}

int main() {
  const int nlev = 11;
  int R[nlev];
  double t[nlev];
  std::vector<std::vector<double>> w(nlev);
  for (int i = 0; i < nlev; ++i) {
    t[i] = 1.0 + 0.9 * i;
    R[i] = (int)std::ceil(5.0 * t[i]);
    double sum = 0;
    for (int d = -R[i]; d <= R[i]; ++d) sum += std::exp(-d * d / (2 * t[i] * t[i]));
    for (int d = -R[i]; d <= R[i]; ++d) w[i].push_back(std::exp(-d * d / (2 * t[i] * t[i])) / sum);
  }
  TcPlan P;
  if (!tc_plan_build(P, nlev, R, t)) { printf("plan failed\n"); return 1; }
  printf("S=%d H0=%d tab_bytes=%d max_level_bytes=%d\n", P.S, P.H0, P.tab_bytes, P.max_level_bytes);
  std::vector<uint8_t> tab(P.tab_bytes);
  tc_fill_tables(P, w, tab.data());
  const int S = P.S;
  std::vector<int> X(S * S);
  srand(1);
  for (auto& v : X) v = (rand() % 256) - 128;
  int *dX; uint8_t* dT; float *dd1, *dd2;
  cudaMalloc(&dX, S * S * 4);
  cudaMalloc(&dT, P.tab_bytes);
  cudaMalloc(&dd1, 128 * 256 * 4);
  cudaMalloc(&dd2, 128 * 128 * 4);
  cudaMemcpy(dX, X.data(), S * S * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dT, tab.data(), P.tab_bytes, cudaMemcpyHostToDevice);
  int fails = 0;
  for (int i : {0, 3, 10}) {
    const TcLevel& L = P.lev[i];
    const int lb = 2 * L.npairs * 256;
    const size_t smem = (size_t)S * S * 2 + lb + 64;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<<<1, 512, smem>>>(dX, S, dT + L.tab_off, lb, L.c0, L.K, dd1, dd2);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("level %d: CUDA error %s\n", i, cudaGetErrorString(e)); return 2; }
    std::vector<float> h1(128 * L.K), h2(128 * 128);
    cudaMemcpy(h1.data(), dd1, 128 * L.K * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), dd2, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    // reference: Rx[c][n] = sum_d w[d] X[c0+n][c0 + c + s + R + d]  (times 2^12)
    double e1 = 0, m1 = 0, e2 = 0, m2 = 0;
    std::vector<double> rx(128 * L.K);
    for (int c = 0; c < 128; ++c)
      for (int n = 0; n < L.K; ++n) {
        double acc = 0;
        for (int d = -L.R; d <= L.R; ++d) {
          const int k = c + L.s + L.R + d;
          if (k < L.K && L.c0 + n < S) acc += w[i][d + L.R] * X[(L.c0 + n) * S + L.c0 + k];
        }
        rx[c * L.K + n] = acc;
        e1 = fmax(e1, fabs(acc * kTcWScale - h1[c * L.K + n]));
        m1 = fmax(m1, fabs(acc * kTcWScale));
      }
    for (int c = 0; c < 128; ++c)
      for (int m = 0; m < 128; ++m) {
        double acc = 0;
        for (int d = -L.R; d <= L.R; ++d) {
          const int k = m + L.s + L.R + d;
          if (k < L.K) acc += w[i][d + L.R] * rx[c * L.K + k];
        }
        e2 = fmax(e2, fabs(acc * kTcWScale - h2[c * 128 + m]));
        m2 = fmax(m2, fabs(acc * kTcWScale));
      }
    printf("level %d R=%d c0=%d s=%d K=%d: D1 max err %.3e (max |D1| %.3e, rel %.2e)  D2 max err %.3e (max %.3e, rel %.2e)\n",
           i, L.R, L.c0, L.s, L.K, e1, m1, e1 / m1, e2, m2, e2 / m2);
    printf("   sample D1[0][0] gpu %.6f ref %.6f   D2[5][7] gpu %.6f\n", h1[0], rx[0] * kTcWScale, h2[5 * 128 + 7]);
    if (!(e1 / m1 < 1e-6 && e2 / m2 < 1e-6)) ++fails;
  }
  printf(fails ? "PROBE FAIL\n" : "PROBE OK\n");
  return fails ? 3 : 0;
}
