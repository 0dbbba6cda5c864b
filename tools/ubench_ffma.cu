// Microbenchmark: FP32 FMA issue forms on sm_100a (B200).
// Purpose: decide how the separable-blur inner loop should feed its weights
// (register / immediate / constant bank / uniform register / shared memory / FFMA2).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_ffma ubench_ffma.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float cw[64];

#define NACC 8
#define UNR 16

template <int V>
__global__ void __launch_bounds__(256) kff(float* out, int iters, float s0, float s1) {
  __shared__ float sw[64];
  if (threadIdx.x < 64) sw[threadIdx.x] = 0.5f + threadIdx.x * 1e-3f;
  __syncthreads();
  float x[NACC], acc[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) { x[k] = s0 + (threadIdx.x + k) * 1e-6f; acc[k] = 0.f; }
  float wreg = s1 * (1.0f + threadIdx.x * 1e-9f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      float w;
      if (V == 0) w = wreg + u * 1e-7f;              // register weight (3-reg FFMA)
      else if (V == 1) w = 0.37f + u * 0.01f;        // immediate
      else if (V == 2) w = cw[u];                    // constant bank, compile-time address
      else if (V == 3) w = cw[(it * UNR + u) & 63];  // constant, runtime-uniform address
      else if (V == 4) w = sw[(it * UNR + u) & 63];  // shared-memory broadcast
      if (V <= 4) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) acc[k] = fmaf(x[k], w, acc[k]);
      } else {
        float wv = (V == 5) ? (wreg + u * 1e-7f) : (V == 6 ? cw[u] : 0.37f + u * 0.01f);
        float2 w2 = make_float2(wv, wv);
#pragma unroll
        for (int k = 0; k < NACC; k += 2) {
          float2 a2 = make_float2(acc[k], acc[k + 1]);
          float2 x2 = make_float2(x[k], x[k + 1]);
          a2 = __ffma2_rn(x2, w2, a2);
          acc[k] = a2.x; acc[k + 1] = a2.y;
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NACC; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
double run(float* out, int blocks, int iters) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  kff<V><<<blocks, 256>>>(out, 2, 1.f, 0.5f);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  kff<V><<<blocks, 256>>>(out, iters, 1.f, 0.5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fmas = (double)blocks * 256 * iters * UNR * NACC;
  return fmas / (ms * 1e-3) / 1e12;
}

int main() {
  float h[64]; for (int i = 0; i < 64; ++i) h[i] = 0.25f + i * 1e-3f;
  cudaMemcpyToSymbol(cw, h, sizeof(h));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int blocks = sms * 8;
  float* out; cudaMalloc(&out, blocks * 256 * sizeof(float));
  int iters = 20000;
  const char* names[] = {"ffma_reg3", "ffma_imm", "ffma_cbank", "ffma_cbank_runtime_idx", "ffma_smem_bcast",
                         "ffma2_reg", "ffma2_cbank", "ffma2_imm"};
  double r[8];
  for (int rep = 0; rep < 2; ++rep) {
    r[0] = run<0>(out, blocks, iters); r[1] = run<1>(out, blocks, iters);
    r[2] = run<2>(out, blocks, iters); r[3] = run<3>(out, blocks, iters);
    r[4] = run<4>(out, blocks, iters); r[5] = run<5>(out, blocks, iters);
    r[6] = run<6>(out, blocks, iters); r[7] = run<7>(out, blocks, iters);
  }
  printf("{\"sms\": %d, \"clock_khz_attr\": %d", sms, clk);
  for (int v = 0; v < 8; ++v) printf(", \"%s_tfma_s\": %.3f", names[v], r[v]);
  printf("}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
