// tc_plan_check.cpp — host-side check of the k_tc operand tables (tc_plan.h), no GPU.
// For each sigma grid: every level's window fits the staged tile, covers every tap of
// every output, and the pair table read through the kernel's descriptor addressing
// (K-step j: pair q = E1 - 2j + a for row group a, half = chunk-in-step, 8x8 core
// matrix row-major) equals T[m][k] = w[k - m - s - R] split into fp16 hi + lo.
// Prints "OK" or the first failure; exit status 0/1.
#include <cmath>
#include <cstdio>
#include <vector>

#include "../../paper_2108_12050_b200/csrc/tc_plan.h"

using namespace mhfd;

static int check(double tmin, double tmax, int n) {
  const int nlev = n + 1;
  std::vector<int> R(nlev);
  std::vector<double> t(nlev);
  std::vector<std::vector<double>> w(nlev);
  for (int i = 0; i < nlev; ++i) {
    t[i] = tmin + i * (tmax - tmin) / n;
    R[i] = (int)std::ceil(5.0 * t[i]);
    double sum = 0;
    for (int d = -R[i]; d <= R[i]; ++d) sum += std::exp(-d * d / (2 * t[i] * t[i]));
    for (int d = -R[i]; d <= R[i]; ++d) w[i].push_back(std::exp(-d * d / (2 * t[i] * t[i])) / sum);
  }
  TcPlan P;
  if (!tc_plan_build(P, nlev, R.data(), t.data())) {
    std::printf("plan rejected for sigma %.2f-%.2f n %d (expected only when 128 + 2 Rmax > %d)\n", tmin, tmax, n,
                kTcMaxS);
    return (128 + 2 * R[nlev - 1] + 15) / 16 * 16 > kTcMaxS ? 0 : 1;
  }
  std::vector<uint8_t> tab(P.tab_bytes);
  tc_fill_tables(P, w, tab.data());
  for (int i = 0; i < nlev; ++i) {
    const TcLevel& L = P.lev[i];
    if (L.c0 % 8 || L.K % 16 || L.c0 + L.K > P.S || L.s < 0 || L.c0 + L.s + L.R != P.H0) {
      std::printf("level %d geometry: c0 %d s %d K %d S %d H0 %d\n", i, L.c0, L.s, L.K, P.S, P.H0);
      return 1;
    }
    if (L.s + 127 + 2 * L.R >= L.K) { std::printf("level %d: window misses taps\n", i); return 1; }
    const uint16_t* hi = reinterpret_cast<const uint16_t*>(tab.data() + L.tab_off);
    const uint16_t* lo = hi + L.npairs * 128;
    const int E1 = L.K / 8 - 2;
    for (int m = 0; m < 128; ++m)
      for (int k = 0; k < L.K; ++k) {
        const int j = k / 16, a = m / 8, half = (k % 16) / 8;
        const int q = E1 - 2 * j + a;                       // descriptor start pair + a * SBO/256
        if (q < 0 || q >= L.npairs) { std::printf("level %d: pair %d out of range\n", i, q); return 1; }
        const int idx = q * 128 + half * 64 + (m % 8) * 8 + (k % 8);   // LBO = 128 B = 64 halves
        const int d = k - m - L.s - L.R;
        const double wt = (d >= -L.R && d <= L.R) ? w[i][d + L.R] * kTcWScale : 0.0;
        const double got = (double)tc_h2f(hi[idx]) + (double)tc_h2f(lo[idx]);
        // hi + lo represents the scaled tap to within half an ulp of lo (2^-24 once lo is
        // an fp16 subnormal, i.e. for taps below ~2^-3 of the scale 2^12 w)
        const double tol = std::fabs(wt) * std::ldexp(1.0, -20) + std::ldexp(1.0, -25);
        if (std::fabs(got - wt) > tol) {
          std::printf("level %d m %d k %d: table %.9g vs tap %.9g\n", i, m, k, got, wt);
          return 1;
        }
      }
  }
  return 0;
}

int main() {
  int bad = 0;
  bad |= check(1.0, 10.0, 10);   // C2-C4
  bad |= check(1.0, 5.0, 5);     // C1
  bad |= check(0.8, 4.0, 7);
  bad |= check(2.0, 11.0, 3);    // R_max = 55: the largest window that fits
  bad |= check(1.0, 30.0, 20);   // C5: rejected (generic schedule)
  std::printf(bad ? "FAIL\n" : "OK\n");
  return bad;
}
