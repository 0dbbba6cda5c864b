// Microbenchmark 2: FFMA vs FFMA2 with weights in vector registers / uniform registers,
// no extra instructions in the loop body (weights preloaded).  sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float cw[64];

template <int V, int NACC>
__global__ void __launch_bounds__(256) k(float* out, int iters, float s0) {
  float x[NACC], acc[NACC], wr[16];
#pragma unroll
  for (int k = 0; k < NACC; ++k) { x[k] = s0 + (threadIdx.x + k) * 1e-6f; acc[k] = 0.f; }
#pragma unroll
  for (int k = 0; k < 16; ++k) wr[k] = s0 * (0.5f + threadIdx.x * 1e-9f + k * 1e-3f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const float w = (V == 0 || V == 2) ? wr[u] : cw[u];
      if (V <= 1) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) acc[k] = fmaf(x[k], w, acc[k]);
      } else {
        const float2 w2 = make_float2(w, w);
#pragma unroll
        for (int k = 0; k < NACC; k += 2) {
          float2 a = make_float2(acc[k], acc[k + 1]);
          a = __ffma2_rn(make_float2(x[k], x[k + 1]), w2, a);
          acc[k] = a.x; acc[k + 1] = a.y;
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NACC; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V, int NACC>
double run(float* out, int blocks, int iters) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<V, NACC><<<blocks, 256>>>(out, 2, 1.f);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  k<V, NACC><<<blocks, 256>>>(out, iters, 1.f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return (double)blocks * 256 * iters * 16 * NACC / (ms * 1e-3) / 1e12;
}

int main() {
  float h[64]; for (int i = 0; i < 64; ++i) h[i] = 0.25f + i * 1e-3f;
  cudaMemcpyToSymbol(cw, h, sizeof(h));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sms * 8 * 256 * sizeof(float));
  for (int occ : {2, 4, 8}) {
    int blocks = sms * occ;
    int iters = 20000 * 8 / occ;
    double r[8];
    for (int rep = 0; rep < 2; ++rep) {
      r[0] = run<0, 8>(out, blocks, iters); r[1] = run<1, 8>(out, blocks, iters);
      r[2] = run<2, 8>(out, blocks, iters); r[3] = run<3, 8>(out, blocks, iters);
      r[4] = run<0, 16>(out, blocks, iters); r[5] = run<1, 16>(out, blocks, iters);
      r[6] = run<2, 16>(out, blocks, iters); r[7] = run<3, 16>(out, blocks, iters);
    }
    printf("{\"ctas_per_sm\": %d, \"warps_per_sm\": %d, \"ffma_reg_8acc\": %.2f, \"ffma_ur_8acc\": %.2f, \"ffma2_reg_8acc\": %.2f, "
           "\"ffma2_ur_8acc\": %.2f, \"ffma_reg_16acc\": %.2f, \"ffma_ur_16acc\": %.2f, \"ffma2_reg_16acc\": %.2f, "
           "\"ffma2_ur_16acc\": %.2f, \"unit\": \"TFMA/s\"}\n", occ, occ * 8, r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7]);
  }
  return 0;
}
