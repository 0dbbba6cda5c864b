// tc_timeline.cu — clock64 timeline of k_tc on CTA 0 (issuer and epilogue thread 0) for
// the bench configuration (4096^2 u8, sigma 1-10, n 10), to locate tensor-pipe bubbles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2108_12050_b200/csrc tools/tc_timeline.cu -o tools/tc_timeline -lcuda
#include <cstdio>
#include <vector>
#include <cmath>
#include <cudaTypedefs.h>
#include "k_tc.cuh"
using namespace mhfd;

int main(int argc, char** argv) {
  const int W = 4096, H = 4096, B = 2, nlev = 11;
  int R[nlev]; double t[nlev];
  std::vector<std::vector<double>> w(nlev);
  for (int i = 0; i < nlev; ++i) {
    t[i] = 1.0 + 0.9 * i; R[i] = (int)std::ceil(5.0 * t[i]);
    double sum = 0; for (int d = -R[i]; d <= R[i]; ++d) sum += std::exp(-d * d / (2 * t[i] * t[i]));
    for (int d = -R[i]; d <= R[i]; ++d) w[i].push_back(std::exp(-d * d / (2 * t[i] * t[i])) / sum);
  }
  TcPlan P; tc_plan_build(P, nlev, R, t);
  std::vector<uint8_t> tab(P.tab_bytes); tc_fill_tables(P, w, tab.data());
  uint8_t *dimg, *dtab, *didx; float* dv; ImgPar* dpar; unsigned long long* dtr;
  cudaMalloc(&dimg, (size_t)W * H * B); cudaMalloc(&dtab, P.tab_bytes);
  cudaMalloc(&dv, (size_t)W * H * B * 4); cudaMalloc(&didx, (size_t)W * H * B);
  cudaMalloc(&dpar, sizeof(ImgPar) * B); cudaMalloc(&dtr, 64 * 16 * 8);
  std::vector<uint8_t> img((size_t)W * H * B);
  for (size_t i = 0; i < img.size(); ++i) img[i] = (uint8_t)((i * 2654435761u) >> 24);
  cudaMemcpy(dimg, img.data(), img.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dtab, tab.data(), tab.size(), cudaMemcpyHostToDevice);
  ImgPar ip[B]; for (int b = 0; b < B; ++b) { ip[b].lo = 0; ip[b].hi = 255; ip[b].inv = 1.f / 255; ip[b].degen = 0; }
  cudaMemcpy(dpar, ip, sizeof(ip), cudaMemcpyHostToDevice);
  cudaMemset(dtr, 0, 64 * 16 * 8);
  // TMA descriptor
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm; const cuuint64_t gd[2] = {(cuuint64_t)W, (cuuint64_t)H * B}; const cuuint64_t gs[1] = {(cuuint64_t)W};
  const cuuint32_t box[2] = {(cuuint32_t)tc_lw(P), (cuuint32_t)P.S}; const cuuint32_t es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dimg, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = tc_smem(P);
  cudaFuncSetAttribute(k_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  Shape s{W, H, (int64_t)W, 1};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_tc<false><<<148, kTcThreads + 32, smem>>>(dimg, s, dpar, P, dtab, tm, 1, dv, didx, nullptr, B, 0, H, 0, nullptr, nullptr, rep == 2 ? dtr : nullptr);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("rep %d: %.3f ms (%.3f ms/image)\n", rep, ms, ms / B);
  }
  unsigned long long tr[64 * 16]; cudaMemcpy(tr, dtr, sizeof(tr), cudaMemcpyDeviceToHost);
  const unsigned long long t0 = tr[0];
  printf("slots: I0 top, I1 table ok, I2 row issued, I3-6 split grp ok, I7 col issued | E8 top, E9 colDone(g-1), E10 consumed, E11 rowDone, E12-15 split grp arrived\n");
  printf("  g lev   K |   I0     I1     I2     I3     I4     I5     I6     I7  |   E8     E9    E10    E11    E12    E13    E14    E15\n");
  for (int g = 0; g < 40; ++g) {
    printf("%3d %3d %3d |", g, g % nlev, P.lev[g % nlev].K);
    for (int k = 0; k < 16; ++k) {
      if (k == 8) printf(" |");
      printf(" %6lld", tr[g * 16 + k] ? (long long)(tr[g * 16 + k] - t0) : -1LL);
    }
    printf("\n");
  }
  return 0;
}
