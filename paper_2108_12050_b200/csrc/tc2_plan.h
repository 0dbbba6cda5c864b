// tc2_plan.h — host-side geometry and Toeplitz operand tables of the two-pass
// tensor-core schedule k_tc2 (u16 / f32 images and radii beyond k_tc's staged tile;
// SURVEY.md §8(f) f1 "main target: C5").  Plain C++ (no CUDA types).
//
// Same mathematics as every other schedule: the sampled renormalised Gaussian blur of
// each level (periodic), DoG = t_i (L_{i+1} - L_i) (Eq. 2,
// PAPER.md:171), first argmax over scales.  The separable blur runs
// as two banded Toeplitz products through an HBM intermediate instead of k_tc's single
// staged tile (which cannot hold a (128 + 2 R)^2 window once R > 56 or the input needs
// two fp16 planes):
//
//   k_tc2_prep  x = 1024 (clamp((p - lo) inv, 0, 1) - 1/2) -> fp16 hi + lo planes,
//               in a tiled layout whose per-tile windows are contiguous runs
//   k_tc2_rows  Rx_i[c][n] = sum_k T_i[c][k] x[n][k]     M = 128 output columns c,
//               N = NR rows n of a tile, K = the level's window; three fp16 products
//               (T_hi x_hi + T_lo x_hi + T_hi x_lo), f32 in TMEM; the epilogue splits
//               2^-12 Rx into fp16 hi + lo and stores it TRANSPOSED (column-major) in
//               4 KB slabs (16 rows x 128 columns, canonical K-major order)
//   k_tc2_cols  L_i[c][m] = sum_k Rx_i[k][c] T_i[m][k]    M = 128 columns c,
//               N = 224 rows m, K = the level's row window, streamed slab by slab;
//               three products again; epilogue: DoG, running max, first argmax
//
// T_i[m][k] = w_i[k - m - s - R] (zero outside the band) is block-Toeplitz in 8 x 8
// core matrices, stored as PAIRS [D_e | D_{e+1}] in descending e (tc_plan.h); a
// product with rg row groups (M or N / 8) reads pairs E1 - 2j + a for a < rg, so a
// table holds K/8 + rg - 2 pairs.  Weights are the hi/lo fp16 split of 2^12 w.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "tc_plan.h"

namespace mhfd {

constexpr int kT2Cols = 128;        // output columns per tile (TMEM lanes, MMA M) in both passes
constexpr int kT2ColRows = 224;     // output rows per k_tc2_cols tile (MMA N; 56 per epilogue thread)
constexpr int kT2SlabRows = 16;     // rows per Rx slab (one K-step of k_tc2_cols)
constexpr int kT2SlabBytes = kT2SlabRows * kT2Cols * 2;   // 4 KB per plane
constexpr float kT2XScale = 1024.f; // normalised pixels scaled before the fp16 split
constexpr int kT2Stages = 10;       // Rx slab ring depth of k_tc2_cols (x 8 KB)
constexpr int kT2MaxLev = 64;
constexpr size_t kT2SmemLimit = 227 * 1024;

struct Tc2Level {
  int32_t R;
  int32_t c0, s, K, npairs, tab_off;      // k_tc2_rows: window columns [c0, c0 + K) of the staged X
  int32_t s2, K2, npairs2, tab_off2;      // k_tc2_cols: window rows y0 - R - s2 + [0, K2)
  float tdog;                             // Eq. 2 factor t_i (signed by polarity)
  int32_t pad;
};

struct Tc2Plan {
  int32_t S;          // staged window width of k_tc2_rows (columns) = roundup16(128 + 2 rmax)
  int32_t H0;         // window origin left of the tile (multiple of 8)
  int32_t NR;         // rows per k_tc2_rows tile (MMA N, multiple of 16)
  int32_t nlev, rmax;
  int32_t tab_bytes;
  int32_t max_lev_bytes1, max_lev_bytes2;
  int32_t max_K2;
  Tc2Level lev[kT2MaxLev];
};

inline size_t tc2_rows_smem(const Tc2Plan& P) {   // X window (2 planes) + 2 table buffers + barriers
  return (size_t)P.NR * P.S * 4 + 2 * (size_t)P.max_lev_bytes1 + 256;
}
inline size_t tc2_cols_smem(const Tc2Plan& P) {   // slab ring + 2 table buffers + barriers
  return (size_t)kT2Stages * 2 * kT2SlabBytes + 2 * (size_t)P.max_lev_bytes2 + 512;
}

// Geometry for levels with radii R[0..nlev) (ceil(5 t_i)).  False if it does not fit.
inline bool tc2_plan_build(Tc2Plan& P, int nlev, const int* R, const double* t) {
  std::memset(&P, 0, sizeof(P));
  if (nlev > kT2MaxLev) return false;
  int rmax = 0;
  for (int i = 0; i < nlev; ++i) rmax = R[i] > rmax ? R[i] : rmax;
  P.S = ((kT2Cols + 2 * rmax + 15) / 16) * 16;
  P.H0 = (P.S - kT2Cols) / 2;
  P.nlev = nlev;
  P.rmax = rmax;
  int off = 0, mb1 = 0, mb2 = 0, mk2 = 0;
  for (int i = 0; i < nlev; ++i) {
    Tc2Level& L = P.lev[i];
    L.R = R[i];
    int c0 = ((P.H0 - R[i]) / 8) * 8;
    for (;;) {
      const int s = P.H0 - R[i] - c0;
      const int K = ((s + kT2Cols + 2 * R[i] + 15) / 16) * 16;
      if (c0 + K <= P.S) { L.c0 = c0; L.s = s; L.K = K; break; }
      c0 -= 8;
      if (c0 < 0) return false;
    }
    L.npairs = L.K / 8 + kT2Cols / 8 - 2;
    L.tab_off = off;
    off += 2 * L.npairs * 256;
    mb1 = 2 * L.npairs * 256 > mb1 ? 2 * L.npairs * 256 : mb1;
    L.s2 = (kT2SlabRows - R[i] % kT2SlabRows) % kT2SlabRows;   // y0 - R - s2 is slab-aligned
    L.K2 = ((L.s2 + kT2ColRows + 2 * R[i] + 15) / 16) * 16;
    L.npairs2 = L.K2 / 8 + kT2ColRows / 8 - 2;
    L.tab_off2 = off;
    off += 2 * L.npairs2 * 256;
    mb2 = 2 * L.npairs2 * 256 > mb2 ? 2 * L.npairs2 * 256 : mb2;
    mk2 = L.K2 > mk2 ? L.K2 : mk2;
    L.tdog = (float)t[i];
  }
  P.tab_bytes = off;
  P.max_lev_bytes1 = mb1;
  P.max_lev_bytes2 = mb2;
  P.max_K2 = mk2;
  // rows per k_tc2_rows tile: the largest multiple of 16 (<= 256) whose window fits
  // beside the table double buffer; MMAs with N >= 128 keep the operand reads within the
  // shared-memory bandwidth (A 4 KB + B N*32 B per N/2 cycles)
  P.NR = 0;
  for (int nr = 256; nr >= 64; nr -= 16) {
    P.NR = nr;
    if (tc2_rows_smem(P) <= kT2SmemLimit) break;
    P.NR = 0;
  }
  return P.NR > 0 && tc2_cols_smem(P) <= kT2SmemLimit;
}

// Pair tables of one product orientation: rg row groups (16 for k_tc2_rows' A operand,
// kT2ColRows / 8 for k_tc2_cols' B operand), window K, shift s, radius R.
inline void tc2_fill_pairs(uint16_t* hi, uint16_t* lo, int npairs, int K, int s, int R,
                           const std::vector<double>& w) {
  const int E1 = K / 8 - 2;
  for (int q = 0; q < npairs; ++q)
    for (int half = 0; half < 2; ++half) {
      const int e = E1 - q + half;
      for (int jr = 0; jr < 8; ++jr)
        for (int l = 0; l < 8; ++l) {
          const int d = 8 * e + l - jr - s - R;   // tap index relative to the centre
          float wf = 0.f;
          if (d >= -R && d <= R) wf = (float)(w[d + R] * (double)kTcWScale);
          const uint16_t h = tc_f2h(wf);
          const uint16_t g = tc_f2h(wf - tc_h2f(h));
          const int idx = q * 128 + half * 64 + jr * 8 + l;
          hi[idx] = h;
          lo[idx] = g;
        }
    }
}

// Row-pass taps wr[i] and column-pass taps wc[i] of every level (the Gaussian levels of
// Eq. 2 use the same taps in both passes; the LoG sub-levels do not, see k_tc2.cuh)
inline void tc2_fill_tables(const Tc2Plan& P, const std::vector<std::vector<double>>& wr,
                            const std::vector<std::vector<double>>& wc, uint8_t* out) {
  std::memset(out, 0, (size_t)P.tab_bytes);
  for (int i = 0; i < P.nlev; ++i) {
    const Tc2Level& L = P.lev[i];
    uint16_t* h1 = reinterpret_cast<uint16_t*>(out + L.tab_off);
    tc2_fill_pairs(h1, h1 + L.npairs * 128, L.npairs, L.K, L.s, L.R, wr[i]);
    uint16_t* h2 = reinterpret_cast<uint16_t*>(out + L.tab_off2);
    tc2_fill_pairs(h2, h2 + L.npairs2 * 128, L.npairs2, L.K2, L.s2, L.R, wc[i]);
  }
}
inline void tc2_fill_tables(const Tc2Plan& P, const std::vector<std::vector<double>>& w, uint8_t* out) {
  tc2_fill_tables(P, w, w, out);
}

}  // namespace mhfd
