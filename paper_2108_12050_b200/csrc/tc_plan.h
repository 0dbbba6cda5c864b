// tc_plan.h — host-side geometry and banded-Toeplitz operand tables of the tensor-core
// blur (k_tc).  Plain C++ (no CUDA types) so the layout probe can share it.
//
// The separable Gaussian blur of one level (periodic boundary,
// sampled taps w_i[d], |d| <= R_i, renormalised in f64) on a 128 x 128 output tile is
// two banded matrix products:
//   row pass     Rx[c][n] = sum_k T_i[c][k] X[c0+n][c0+k]      (c = output column)
//   column pass  L [c][m] = sum_k Rx[c][k] T_i[m][k]            (m = output row)
// with the same Toeplitz matrix T_i[m][k] = w_i[k - m - s_i - R_i] (zero outside the
// band), where X is the staged S x S tile whose origin is H0 pixels above/left of the
// output tile, c0_i = the 8-aligned start of level i's window and s_i its residual
// shift (H0 - R_i = c0_i + s_i).  K_i = window length (multiple of 16).
//
// T_i is block-Toeplitz in 8 x 8 core matrices: block (a, b) (a = m/8, b = k/8) depends
// only on e = b - a.  One MMA (K = 16) reads blocks (a, 2j) and (a, 2j+1) for a = 0..15,
// so the table stores PAIRS P_e = [D_e | D_{e+1}] (2 x 128 B) in DESCENDING e: pair q
// holds e = E1 - q, E1 = K/8 - 2.  The descriptor of K-step j then starts at pair
// q = E1 - 2j with SBO = 256 (next row group -> e - 1) and LBO = 128 (-> D_{e+1}).
// Weights are stored as fp16 hi/lo splits of w * 2^12 (hi = fp16(w'), lo = fp16(w' - hi)).
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace mhfd {

constexpr int kTcTile = 128;            // output tile edge (MMA M)
constexpr int kTcMaxS = 240;            // staged tile edge limit (smem budget)
constexpr float kTcWScale = 4096.f;     // weights scaled by 2^12 before the fp16 split
constexpr int kTcMaxLev = 64;

struct TcLevel {
  int32_t R, c0, s, K;      // radius, window start (multiple of 8), shift, window length
  int32_t npairs;           // K/8 + 14
  int32_t tab_off;          // byte offset of this level's [hi pairs | lo pairs] block
  float tdog;               // t_i (Eq. 2 factor of DoG plane i)
  int32_t pad;
};

struct TcPlan {
  int32_t S, H0, nlev, rmax;
  int32_t reflect;          // blur boundary: 0 periodic (R7), 1 half-sample symmetric (R25)
  int32_t tab_bytes;        // total bytes of all levels' tables
  int32_t max_level_bytes;  // largest single-level block (smem buffer size)
  TcLevel lev[kTcMaxLev];
};

// IEEE binary16 round-to-nearest-even of a float (host side, no CUDA headers)
inline uint16_t tc_f2h(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  x &= 0x7FFFFFFFu;
  if (x >= 0x47800000u) return (uint16_t)(sign | 0x7C00u);          // overflow -> inf (never here)
  if (x < 0x33000000u) return (uint16_t)sign;                         // < 2^-25 -> 0
  const int e = (int)(x >> 23) - 127;
  uint32_t mant = (x & 0x7FFFFFu) | 0x800000u;
  if (e < -14) {                                                       // subnormal half
    const int shift = 13 + (-14 - e);
    const uint32_t q = mant >> shift, rem = mant & ((1u << shift) - 1), half = 1u << (shift - 1);
    uint32_t r = q + ((rem > half || (rem == half && (q & 1))) ? 1u : 0u);
    return (uint16_t)(sign | r);
  }
  const uint32_t q = mant >> 13, rem = mant & 0x1FFFu;
  uint32_t r = ((uint32_t)(e + 15) << 10) | (q & 0x3FFu);
  if (rem > 0x1000u || (rem == 0x1000u && (r & 1))) ++r;
  return (uint16_t)(sign | r);
}
inline float tc_h2f(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const int e = (h >> 10) & 0x1F;
  const uint32_t m = h & 0x3FFu;
  float f;
  if (e == 0) f = std::ldexp((float)m, -24);
  else f = std::ldexp((float)(m | 0x400u), e - 25);
  uint32_t x;
  std::memcpy(&x, &f, 4);
  x |= sign;
  std::memcpy(&f, &x, 4);
  return f;
}

// Geometry for levels with radii R[0..nlev) (ceil(5 t_i)); false if it does not fit.
inline bool tc_plan_build(TcPlan& P, int nlev, const int* R, const double* t) {
  std::memset(&P, 0, sizeof(P));
  if (nlev > kTcMaxLev) return false;
  int rmax = 0;
  for (int i = 0; i < nlev; ++i) rmax = R[i] > rmax ? R[i] : rmax;
  const int S = ((kTcTile + 2 * rmax + 15) / 16) * 16;
  if (S > kTcMaxS) return false;
  P.S = S;
  P.H0 = (S - kTcTile) / 2;
  P.nlev = nlev;
  P.rmax = rmax;
  int off = 0, maxb = 0;
  for (int i = 0; i < nlev; ++i) {
    TcLevel& L = P.lev[i];
    L.R = R[i];
    int c0 = ((P.H0 - R[i]) / 8) * 8;
    for (;;) {
      const int s = P.H0 - R[i] - c0;
      const int K = ((s + kTcTile + 2 * R[i] + 15) / 16) * 16;
      if (c0 + K <= S) { L.c0 = c0; L.s = s; L.K = K; break; }
      c0 -= 8;
      if (c0 < 0) return false;
    }
    L.npairs = L.K / 8 + 14;
    L.tab_off = off;
    L.tdog = (float)t[i];
    const int bytes = 2 * L.npairs * 256;
    off += bytes;
    maxb = bytes > maxb ? bytes : maxb;
  }
  P.tab_bytes = off;
  P.max_level_bytes = maxb;
  return true;
}

// Fill the pair tables of every level; taps w[i] = the 2R_i+1 renormalised f64 taps.
inline void tc_fill_tables(const TcPlan& P, const std::vector<std::vector<double>>& w, uint8_t* out) {
  std::memset(out, 0, (size_t)P.tab_bytes);
  for (int i = 0; i < P.nlev; ++i) {
    const TcLevel& L = P.lev[i];
    const int E1 = L.K / 8 - 2;
    uint16_t* hi = reinterpret_cast<uint16_t*>(out + L.tab_off);
    uint16_t* lo = hi + L.npairs * 128;   // 128 halves per pair
    for (int q = 0; q < L.npairs; ++q) {
      for (int half = 0; half < 2; ++half) {
        const int e = E1 - q + half;
        for (int jr = 0; jr < 8; ++jr)
          for (int l = 0; l < 8; ++l) {
            const int d = 8 * e + l - jr - L.s - L.R;   // tap index relative to the centre
            float wf = 0.f;
            if (d >= -L.R && d <= L.R) wf = (float)(w[i][d + L.R] * (double)kTcWScale);
            const uint16_t h = tc_f2h(wf);
            const uint16_t g = tc_f2h(wf - tc_h2f(h));
            const int idx = q * 128 + half * 64 + jr * 8 + l;
            hi[idx] = h;
            lo[idx] = g;
          }
      }
    }
  }
}

}  // namespace mhfd
