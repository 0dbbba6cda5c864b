// ubench_umma.cu — issue-rate microbenchmark of tcgen05.mma kind::f16 (M = 128, K = 16) on
// every SM: cycles per MMA for SS (A, B in shared memory) and TS (A in TMEM) against N,
// alone and with 16 warps loading TMEM (tcgen05.ld) or storing shared memory at the same
// time.  The model behind k_tc's schedule comes from these numbers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2108_12050_b200/csrc tools/ubench_umma.cu -o tools/ubench_umma
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#include "umma.cuh"

using namespace mhfd;

// whole-warp issue: one elected lane executes the MMA (no per-MMA ELECT loop)
__device__ __forceinline__ void mma_ss_w(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(id)
      : "memory");
}
__device__ __forceinline__ void mma_ts_w(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}\n" ::"r"(d), "r"(a), "l"(b), "r"(id)
      : "memory");
}

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

// mode: 0 SS, 1 TS.  load: 0 none, 1 tcgen05.ld x16 loop, 2 st.shared loop, 3 tcgen05.st loop
// ksteps: distinct A/B slices cycled through (different smem addresses per MMA)
__global__ void __launch_bounds__(544, 1) ub(int mode, int N, int reps, int load, int nd, int niss, long long* out_cyc,
                                             unsigned long long* out_ld) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;                    // 8 slices x 4 KB
  uint8_t* B = sm + 8 * 4096;         // 8 slices x (N x 32 B) <= 8 x 8 KB
  uint8_t* junk = B + 8 * 8192;       // 32 KB scratch for the st.shared load
  uint64_t* bar = reinterpret_cast<uint64_t*>(junk + 32768);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  volatile int* done = reinterpret_cast<volatile int*>(tslot + 1);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  for (int i = tid; i < (8 * 4096 + 8 * 8192) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) {
    mbar_init_(bar, 1);
    mbar_init_(bar + 1, 1);
    *done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc(tslot, 512);
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tm = *tslot;
  if (warp == 16 || (niss == 2 && warp == 15)) {
    const int wi = warp == 16 ? 0 : 1;
    const uint32_t id = umma::idesc_f16(128, N);
    const uint32_t a0 = umma::smem_addr(A), b0 = umma::smem_addr(B);
    uint64_t da[8], db[8];
    uint32_t dd[8], at[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      da[u] = umma::desc_kmajor(a0 + u * 4096, 128, 256);
      db[u] = umma::desc_kmajor(b0 + u * 8192, 128, 256);
      dd[u] = tm + (uint32_t)(((u % nd) * niss + wi) * N);
      at[u] = tm + 448 + 8 * (u & 3);
    }
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (mode == 0) mma_ss_w(dd[u], da[u], db[u], id);
        else mma_ts_w(dd[u], at[u], db[u], id);
      }
    if (lane == 0) umma::commit(&bar[wi]);
    __syncwarp();
    mbar_wait_(&bar[wi], 0);
    if (niss == 2) asm volatile("bar.sync 2, 64;" ::: "memory");
    const long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < reps / 8 / niss; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (mode == 0) mma_ss_w(dd[u], da[u], db[u], id);
        else mma_ts_w(dd[u], at[u], db[u], id);
      }
    if (lane == 0) umma::commit(&bar[wi]);
    __syncwarp();
    mbar_wait_(&bar[wi], 1);
    const long long t1 = clock64();
    if (lane == 0) {
      if (wi == 0) out_cyc[blockIdx.x] = t1 - t0;
      else out_cyc[148 + blockIdx.x] = t1 - t0;
      *done = 1;
    }
  } else if (load && warp != 15) {
    const int q = warp & 3;
    const uint32_t base = tm + ((uint32_t)(32 * q) << 16) + 384 + 16 * (warp >> 2) % 128;
    unsigned long long n = 0;
    uint32_t acc = 0;
    while (!*done) {
      if (load == 1) {
        uint32_t r[16];
        umma::ld16(base, r);
        umma::wait_ld();
#pragma unroll
        for (int u = 0; u < 16; ++u) acc += r[u];
        n += 16 * 32 * 4;
      } else if (load == 2) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          reinterpret_cast<uint4*>(junk)[(warp * 32 + lane + 512 * u) & 2047] = make_uint4(acc, n, u, 0);
        n += 8 * 16 * 32;
      } else {
        uint32_t r[8] = {acc, 1, 2, 3, 4, 5, 6, 7};
        umma::st8(base, r);
        umma::wait_st();
        n += 8 * 32 * 4;
      }
    }
    if (acc == 12345u) out_ld[0] = 0;
    if (lane == 0) atomicAdd(&out_ld[blockIdx.x], n);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 512);
}

int main() {
  const int reps = 4096, grid = 148;
  long long* dc;
  unsigned long long* dl;
  cudaMalloc(&dc, 2 * grid * 8);
  cudaMalloc(&dl, grid * 8);
  const int smem = 8 * 4096 + 8 * 8192 + 32768 + 64;
  cudaFuncSetAttribute(ub, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("mode  N  issuers  cyc/MMA(median, all MMAs of the SM)  floor N/2\n");
  for (int mode = 0; mode < 2; ++mode)
    for (int N : {32, 64, 128, 192, 256})
      for (int niss : {1, 2}) {
        if (niss * N > (mode ? 448 : 512)) continue;
        cudaMemset(dc, 0, 2 * grid * 8);
        ub<<<grid, 544, smem>>>(mode, N, reps, 0, 1, niss, dc, dl);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<long long> c(2 * grid), m(grid);
        cudaMemcpy(c.data(), dc, 2 * grid * 8, cudaMemcpyDeviceToHost);
        for (int b = 0; b < grid; ++b) m[b] = std::max(c[b], c[grid + b]);
        std::sort(m.begin(), m.end());
        printf("%s  %3d  %d   %8.1f      %5.1f\n", mode ? "TS" : "SS", N, niss, (double)m[grid / 2] / reps, N / 2.0);
      }
  return 0;
}
