// k_band.cuh — the hot kernel for u8 images (hot-path rows a2-a6), "band" schedule.
//
// Same mathematics as k_scale_space (PAPER.md:136-141 blur, :171 Eq. 2 DoG, :240-244
// inner argmax, :257 stretch), laid out for one CTA per SM:
//
//   CTA = one image x one strip of 32 columns x one band of BH = 256 rows, 512 threads.
//   prologue : the raw u8 band with its halo ((256+2Rmax+3) x (32+2*ceil16(Rmax+3)) bytes,
//              ~60 KB at sigma <= 10) comes from HBM ONCE, by TMA (image-edge CTAs: plain
//              loads with periodic wrap).  Each byte is then saturated to [lo, hi] (VIMNMX on
//              u16 pairs) into a copy with a conflict-free row pitch; the row pass
//              re-centres it, x = p' - mid, in its exact u8 -> f32 conversion.  The stretch I' - 1/2 = (x + mid - lo) inv - 1/2 is
//              affine in x and the blur kernels sum to one, so every level is blurred on x
//              and the DoG is t_i inv (L'_{i+1} - L'_i)  (exact for unit-sum kernels).
//   per level: row pass — lane = row, 16 consecutive output columns per thread, input
//              bytes converted in registers (PRMT into 2^23 + u, one FADD2 per pair: exact),
//              tap-pair FFMA2 (even outputs: weights (w[2k], w[2k+1]); odd outputs:
//              (w[2k-1], w[2k]) from a shifted copy) -> hbuf (256+2R+p rows x 32 columns).
//              column pass — 8 rows x 2 columns per thread, column-pair FFMA2 with a
//              broadcast weight; DoG, running max and first argmax in registers.
//   epilogue : v (f32) and argmax (u8) of the 256 x 32 block to HBM.
//
// Why this shape: on B200 the FP32 pipe (128 FMA/clk/SM) and the shared-memory crossbar
// (128 B/clk/SM) have the same width, so each loaded byte must feed many FMAs: one 4-byte
// raw load feeds 64 FMAs in the row pass, one 8-byte hbuf load feeds 16 in the column
// pass, weights are warp-broadcast loads, and no per-level conversion phase or per-chunk
// barrier interrupts the FMA stream.
#pragma once
#include "common.cuh"
#include "k_scale_space.cuh"

namespace mhfd {

constexpr int kBandThreads = 512;
constexpr int kBandBH = 256;
constexpr int kBandHP = 36;         // hbuf pitch (floats): 4 x odd -> conflict-free STS.128 by rows
constexpr int kBandBoxRows = 128;   // TMA box height for the raw band

__host__ __device__ inline int band_rm(int rmax) { return (rmax + 3 + 15) & ~15; }   // margin, 16-B aligned
__host__ __device__ inline int band_raw_w(int rmax) { return kStripW + 2 * band_rm(rmax); }
__host__ __device__ inline int band_raw_rows(int rmax) { return kBandBH + 2 * rmax + 3; }
__host__ __device__ inline int band_land_rows(int rmax) {
  return (band_raw_rows(rmax) + kBandBoxRows - 1) / kBandBoxRows * kBandBoxRows;
}
// saturated copy: row pitch 4 x odd bytes (conflict-free 4-byte loads with lane = row),
// wide enough for the row-pass window overrun
__host__ __device__ inline int band_rwp(int rmax) {
  int q = (band_raw_w(rmax) + 16 + 3) / 4;
  if ((q & 1) == 0) ++q;
  return 4 * q;
}
__host__ __device__ inline int band_hrows(int rmax) { return kBandBH + 2 * rmax + 19; }
__host__ __device__ inline size_t band_land_bytes(int rmax) { return (size_t)band_land_rows(rmax) * band_raw_w(rmax); }
__host__ __device__ inline size_t band_rawp_bytes(int rmax) {
  return (((size_t)band_raw_rows(rmax) + 1) * band_rwp(rmax) + 127) & ~(size_t)127;
}
__host__ __device__ inline size_t band_smem(int rmax, int ntaps_total) {
  return band_land_bytes(rmax) + band_rawp_bytes(rmax) +
         sizeof(float) * ((size_t)band_hrows(rmax) * kBandHP + 3 * (size_t)wtab_floats(ntaps_total)) + 16;
}
__host__ __device__ inline bool band_ok(int W, int H, int rmax, int ntaps_total) {
  return band_smem(rmax, ntaps_total) <= 224 * 1024 && W >= band_raw_w(rmax) && H >= band_raw_rows(rmax);
}

// Exact floats x = p' - mid for two bytes p' of w (PRMT builds 2^23 + p', one FADD2
// subtracts nc = 2^23 + mid; every value is an integer below 2^24, so nothing rounds).
__device__ __forceinline__ float2 byte_pair(uint32_t w, uint32_t sel_lo, uint32_t sel_hi, float2 nc) {
  const uint32_t a = __byte_perm(w, 0x4B000000u, sel_lo);
  const uint32_t b = __byte_perm(w, 0x4B000000u, sel_hi);
  return __fadd2_rn(make_float2(__uint_as_float(a), __uint_as_float(b)), nc);
}
// one 4-byte word -> pairs (x0, x1), (x2, x3)
__device__ __forceinline__ void word_pairs(uint32_t w, float2& p0, float2& p1, float2 nc) {
  p0 = byte_pair(w, 0x7540u, 0x7541u, nc);
  p1 = byte_pair(w, 0x7542u, 0x7543u, nc);
}
// saturate the 4 bytes of w to [lo, hi] (two VIMNMX.U16x2 per half-word pair); lo4/hi4 =
// the bounds replicated in both 16-bit halves
__device__ __forceinline__ uint32_t clamp_bytes(uint32_t w, uint32_t lo2, uint32_t hi2) {
  const uint32_t e = __vminu2(__vmaxu2(__byte_perm(w, 0u, 0x4240u), lo2), hi2);   // bytes 0, 2
  const uint32_t o = __vminu2(__vmaxu2(__byte_perm(w, 0u, 0x4341u), lo2), hi2);   // bytes 1, 3
  return __byte_perm(e, o, 0x6240u);
}

// Row pass over 8 taps for NQ output pairs (2*NQ consecutive outputs): the input pairs
// k0 .. k0+NQ+3 sit in NB = NQ/4+1 rotating 4-pair blocks starting at block u0.
template <int NQ, int NB>
__device__ __forceinline__ void row_group(float2 (&acc)[2 * NQ], const float2 (&Q)[NB][4], int u0,
                                          const float* __restrict__ wa, const float* __restrict__ wb) {
  const float4 A0 = reinterpret_cast<const float4*>(wa)[0], A1 = reinterpret_cast<const float4*>(wa)[1];
  const float4 B0 = reinterpret_cast<const float4*>(wb)[0], B1 = reinterpret_cast<const float4*>(wb)[1];
  const float2 WA[4] = {lo2(A0), hi2(A0), lo2(A1), hi2(A1)};
  const float2 WB[4] = {lo2(B0), hi2(B0), lo2(B1), hi2(B1)};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq) {
      const int m = qq + kk;
      const float2 q = Q[(u0 + m / 4) % NB][m % 4];
      acc[2 * qq] = __ffma2_rn(q, WA[kk], acc[2 * qq]);
      acc[2 * qq + 1] = __ffma2_rn(q, WB[kk], acc[2 * qq + 1]);
    }
  }
}

template <int NB>
__device__ __forceinline__ void load_block(float2 (&Q)[NB][4], int blk, const uint32_t* __restrict__ src, int word,
                                           float2 nc) {
  word_pairs(src[word], Q[blk][0], Q[blk][1], nc);
  word_pairs(src[word + 1], Q[blk][2], Q[blk][3], nc);
}

// One row-pass item: 2*NQ consecutive outputs of one row (src = its first input word),
// written to hdst (2*NQ floats, 16-byte aligned).
template <int NQ>
__device__ __forceinline__ void row_item(const uint32_t* __restrict__ src, const float* __restrict__ wa,
                                         const float* __restrict__ wb, int ntap, float* __restrict__ hdst,
                                         bool store, float2 nc) {
  constexpr int NB = NQ / 4 + 1;
  float2 acc[2 * NQ];
#pragma unroll
  for (int o = 0; o < 2 * NQ; ++o) acc[o] = make_float2(0.f, 0.f);
  float2 Q[NB][4];
#pragma unroll
  for (int bb = 0; bb + 1 < NB; ++bb) load_block(Q, bb, src, 2 * bb, nc);
  const int ng = ntap >> 3;   // groups of 8 taps; group gi uses blocks gi .. gi+NB-1 (mod NB)
  int gi = 0;
  for (; gi + NB <= ng; gi += NB) {
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      load_block(Q, (u + NB - 1) % NB, src, 2 * (gi + u + NB - 1), nc);
      row_group<NQ, NB>(acc, Q, u, wa + 8 * (gi + u), wb + 8 * (gi + u));
    }
  }
  const int rem = ng - gi;
#pragma unroll
  for (int u = 0; u < NB - 1; ++u) {
    if (u < rem) {
      load_block(Q, (u + NB - 1) % NB, src, 2 * (gi + u + NB - 1), nc);
      row_group<NQ, NB>(acc, Q, u, wa + 8 * (gi + u), wb + 8 * (gi + u));
    }
  }
  // odd outputs: tap pair (ntap-1, ntap) on input pairs ntap/2 + qq (window now starts at
  // block rem, whose first NB-1 blocks hold them)
  {
    const float2 wl = reinterpret_cast<const float2*>(wb)[ntap >> 1];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      if (u == rem) {
#pragma unroll
        for (int qq = 0; qq < NQ; ++qq) acc[2 * qq + 1] = __ffma2_rn(Q[(u + qq / 4) % NB][qq % 4], wl, acc[2 * qq + 1]);
      }
    }
  }
  if (!store) return;
#pragma unroll
  for (int v4 = 0; v4 < NQ / 2; ++v4)
    reinterpret_cast<float4*>(hdst)[v4] =
        make_float4(acc[4 * v4].x + acc[4 * v4].y, acc[4 * v4 + 1].x + acc[4 * v4 + 1].y,
                    acc[4 * v4 + 2].x + acc[4 * v4 + 2].y, acc[4 * v4 + 3].x + acc[4 * v4 + 3].y);
}

// Column pass + DoG + running max/argmax for the 8 rows x 2 columns a thread owns:
// src = hbuf row (8 rg + p) column 2 cp (the first real tap row), L' = sum_{t<n} wc[t]
// src[o + t] with n = 2R+1 unpadded taps (wc = the level's taps without the row-pass
// prefix); DoG of the previous level = tinv (L' - lprev) (tinv = t_{lev-1} inv, Eq. 2 on
// the re-centred input).
template <int HP>
__device__ __forceinline__ void col_pass(const float* __restrict__ src, const float* __restrict__ wc, int n,
                                         int lev, float tinv, float (&lprev)[16], float (&vbest)[16],
                                         uint32_t (&ibest)[4]) {
  float2 acc[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.f, 0.f);
  float2 Xa[8], Xb[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) Xa[k] = *reinterpret_cast<const float2*>(src + k * HP);
  auto group = [&](const float2 (&Xl)[8], const float2 (&Xh)[8], int jj, int cnt) {
    const float4 W0 = reinterpret_cast<const float4*>(wc + jj)[0];
    const float4 W1 = reinterpret_cast<const float4*>(wc + jj)[1];
    const float w8[8] = {W0.x, W0.y, W0.z, W0.w, W1.x, W1.y, W1.z, W1.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (t < cnt) {
        const float2 wt = make_float2(w8[t], w8[t]);
#pragma unroll
        for (int o = 0; o < 8; ++o) {
          const int m = o + t;
          acc[o] = __ffma2_rn(m < 8 ? Xl[m] : Xh[m - 8], wt, acc[o]);
        }
      }
    }
  };
  int j = 0;
  for (; j + 16 <= n; j += 16) {
#pragma unroll
    for (int k = 0; k < 8; ++k) Xb[k] = *reinterpret_cast<const float2*>(src + (j + 8 + k) * HP);
    group(Xa, Xb, j, 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) Xa[k] = *reinterpret_cast<const float2*>(src + (j + 16 + k) * HP);
    group(Xb, Xa, j + 8, 8);
  }
  if (j < n) {   // 1 .. 15 remaining taps
#pragma unroll
    for (int k = 0; k < 8; ++k) Xb[k] = *reinterpret_cast<const float2*>(src + (j + 8 + k) * HP);
    group(Xa, Xb, j, min(8, n - j));
    if (j + 8 < n) {
#pragma unroll
      for (int k = 0; k < 8; ++k) Xa[k] = *reinterpret_cast<const float2*>(src + (j + 16 + k) * HP);
      group(Xb, Xa, j + 8, n - j - 8);
    }
  }
#pragma unroll
  for (int o = 0; o < 8; ++o) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int k = 2 * o + c;
      const float L = c ? acc[o].y : acc[o].x;
      if (lev > 0) {
        const float D = tinv * (L - lprev[k]);
        if (D > vbest[k]) {
          vbest[k] = D;
          const int sh = (k & 3) * 8;
          ibest[k >> 2] = (ibest[k >> 2] & ~(0xffu << sh)) | ((uint32_t)(lev - 1) << sh);
        }
      }
      lprev[k] = L;
    }
  }
}

struct BandTile {
  int b, x0, Y0;
};
__device__ __forceinline__ BandTile band_tile(int t, int strips, int bands) {
  BandTile bt;
  bt.x0 = (t % strips) * kStripW;
  t /= strips;
  bt.Y0 = (t % bands) * kBandBH;
  bt.b = t / bands;
  return bt;
}

// Issue the copy of tile bt's raw band into the landing zone.  Returns the mode:
// 2 = TMA boxes, 1 = per-row bulk copies (both complete on `bar`), 0 = plain loads (done).
__device__ __forceinline__ int band_fetch(const BandTile& bt, uint8_t* land, uint64_t* bar, const uint8_t* images,
                                          const Shape& s, const CUtensorMap* tmap, int use_tmap, int rmax) {
  const int RM = band_rm(rmax), RW = band_raw_w(rmax), NRB = band_raw_rows(rmax);
  const int yr = bt.Y0 - rmax - 3, xr = bt.x0 - RM;
  const int tid = threadIdx.x;
  const bool tma = use_tmap && xr >= 0 && xr + RW <= s.W && yr >= 0 && yr + NRB <= s.H;
  const bool bulk = !tma && (s.W % 16) == 0 && (s.pitch % 16) == 0;
  if (tma) {
    if (tid == 0) {
      const int nbox = band_land_rows(rmax) / kBandBoxRows;
      mbar_arrive_expect_tx(bar, (uint32_t)(nbox * kBandBoxRows * RW));
      for (int k = 0; k < nbox; ++k)
        tma_2d_g2s(land + (size_t)k * kBandBoxRows * RW, tmap, xr, bt.b * s.H + yr + k * kBandBoxRows, bar);
    }
    return 2;
  }
  const uint8_t* img = images + (int64_t)bt.b * s.H * s.pitch;
  if (bulk) {   // image-edge tile: one 1-D bulk copy per row (two where the row wraps)
    if (tid == 0) mbar_arrive_expect_tx(bar, (uint32_t)(NRB * RW));
    __syncthreads();   // expect_tx registered before any copy completes
    for (int r = tid; r < NRB; r += kBandThreads) {
      const uint8_t* row = img + (int64_t)wrap_idx(yr + r, s.H) * s.pitch;
      uint8_t* dst = land + (size_t)r * RW;
      if (xr < 0) {
        bulk_g2s(dst, row + (s.W + xr), (uint32_t)(-xr), bar);
        bulk_g2s(dst - xr, row, (uint32_t)(RW + xr), bar);
      } else if (xr + RW > s.W) {
        bulk_g2s(dst, row + xr, (uint32_t)(s.W - xr), bar);
        bulk_g2s(dst + (s.W - xr), row, (uint32_t)(xr + RW - s.W), bar);
      } else {
        bulk_g2s(dst, row + xr, (uint32_t)RW, bar);
      }
    }
    return 1;
  }
  const int warp = tid >> 5, lane = tid & 31;   // generic widths: plain loads with wrap
  for (int r = warp; r < NRB; r += kBandThreads / 32) {
    const uint8_t* row = img + (int64_t)wrap_idx(yr + r, s.H) * s.pitch;
    for (int c = lane; c < RW; c += 32) land[(size_t)r * RW + c] = row[wrap_idx(xr + c, s.W)];
  }
  return 0;
}

// Persistent: grid = one CTA per SM, each CTA walks tiles t = blockIdx.x + k * gridDim.x;
// the raw band of the next tile is fetched (TMA / bulk copies) while the current one is
// processed, so the HBM latency and the v/argmax stores overlap the FMA work.
__global__ void __launch_bounds__(kBandThreads, 1)
k_band(const uint8_t* __restrict__ images, Shape s, const ImgPar* __restrict__ par,
       const __grid_constant__ LevelTable tab, const __grid_constant__ CUtensorMap tmap, int use_tmap,
       float* __restrict__ v_out, uint8_t* __restrict__ idx_out, int batch) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int rmax = tab.rmax;
  const int RM = band_rm(rmax);
  const int RW = band_raw_w(rmax);
  const int NRB = band_raw_rows(rmax);
  const int RWP = band_rwp(rmax);
  uint8_t* land = smem_raw;                                   // TMA landing: land_rows x RW
  uint8_t* rawp = land + band_land_bytes(rmax);               // (NRB+1) x RWP, saturated bytes p'
  float* hbuf = reinterpret_cast<float*>(rawp + band_rawp_bytes(rmax));   // hrows x 36
  float* wA = hbuf + band_hrows(rmax) * kBandHP;
  float* wB = wA + wtab_floats(tab.ntaps_total);
  float* wC = wB + wtab_floats(tab.ntaps_total);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wC + wtab_floats(tab.ntaps_total));

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t plane = (int64_t)s.H * s.W;
  const int strips = (s.W + kStripW - 1) / kStripW;
  const int bands = (s.H + kBandBH - 1) / kBandBH;
  const int ntiles = strips * bands * batch;
  int t = blockIdx.x;
  if (t >= ntiles) return;

  // ---- once per CTA: tap tables, zero padding rows of hbuf, barrier
  for (int i = kBandBH * kBandHP + tid; i < band_hrows(rmax) * kBandHP; i += kBandThreads) hbuf[i] = 0.f;
  for (int i = tid; i < tab.ntaps_total; i += kBandThreads) wA[i] = tab.w[i];
  for (int l = 0; l < tab.nlev; ++l)
    for (int i = tid; i < tab.ntap[l] + 8; i += kBandThreads) {
      wB[tab.woff[l] + i] = i ? tab.w[tab.woff[l] + i - 1] : 0.f;
      wC[tab.woff[l] + i] = i < 2 * tab.R[l] + 1 ? tab.w[tab.woff[l] + tab.pre[l] + i] : 0.f;
    }
  for (int i = tid; i < RWP / 4; i += kBandThreads)   // row past the band: x = 0 (meets zero taps)
    reinterpret_cast<uint32_t*>(rawp + (size_t)NRB * RWP)[i] = 0u;
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  BandTile bt = band_tile(t, strips, bands);
  int mode = band_fetch(bt, land, bar, images, s, &tmap, use_tmap, rmax);

  // column-pass ownership: 8 rows x 2 columns; row-pass ownership: row lane + 32*(warp/2)
  const int cp = lane & 15;
  const int rg = 2 * warp + (lane >> 4);
  const int prow = lane + 32 * (warp >> 1);
  const int g = warp & 1;

  for (;;) {
    // ---- the fetched band: wait, then saturate into rawp (p' = clamp(p, lo, hi))
    if (mode) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    }
    __syncthreads();
    const ImgPar ip = par[bt.b];
    const int lo = ip.lo, hi = ip.hi;
    const int mid = lo + (hi - lo + 1) / 2;   // x = p' - mid in [-128, 127] since hi - lo <= 255
    const uint32_t lo2 = (uint32_t)lo * 0x10001u, hi2 = (uint32_t)hi * 0x10001u;
    const float2 nc = make_float2(-(8388608.f + (float)mid), -(8388608.f + (float)mid));
    {
      const int nw = RW / 4;
      for (int r = warp; r < NRB; r += 16) {
        const uint32_t* srow = reinterpret_cast<const uint32_t*>(land + (size_t)r * RW);
        uint32_t* drow = reinterpret_cast<uint32_t*>(rawp + (size_t)r * RWP);
        for (int c4 = lane; c4 < RWP / 4; c4 += 32) {
          drow[c4] = c4 < nw ? clamp_bytes(srow[c4], lo2, hi2) : 0u;   // past the band: meets zero taps
        }
      }
    }
    __syncthreads();   // rawp ready, landing zone free
    // ---- prefetch the next tile's band while this one is processed
    const int tn = t + gridDim.x;
    BandTile bn;
    int mode_n = 0;
    if (tn < ntiles) {
      bn = band_tile(tn, strips, bands);
      mode_n = band_fetch(bn, land, bar, images, s, &tmap, use_tmap, rmax);
    }

    const int b = bt.b, x0 = bt.x0, Y0 = bt.Y0;
    if (ip.degen) {  // hi == lo: I' == 0, every DoG plane is exactly 0
      for (int i = tid; i < kBandBH * kStripW; i += kBandThreads) {
        const int y = Y0 + i / kStripW, x = x0 + i % kStripW;
        if (x < s.W && y < s.H) {
          v_out[(int64_t)b * plane + (int64_t)y * s.W + x] = 0.f;
          idx_out[(int64_t)b * plane + (int64_t)y * s.W + x] = 0;
        }
      }
    } else {
      const float inv = ip.inv;
      float lprev[16], vbest[16];
      uint32_t ibest[4];
#pragma unroll
      for (int k = 0; k < 16; ++k) { lprev[k] = 0.f; vbest[k] = -INFINITY; }
#pragma unroll
      for (int k = 0; k < 4; ++k) ibest[k] = 0u;

      for (int lev = 0; lev < tab.nlev; ++lev) {
        const int R = tab.R[lev], p = tab.pre[lev], ntap = tab.ntap[lev];
        const float* wa = wA + tab.woff[lev];
        const float* wb = wB + tab.woff[lev];
        const int nrow = kBandBH + 2 * R + p;            // hbuf rows: band rows -R-p .. BH+R-1
        const int cs = RM - R - p;                       // rawp column of the first staged column (x4)
        const int rs = rmax + 3 - R - p;                 // rawp row of hbuf row 0
        // ---------------- row pass ----------------
#ifndef MHFD_EXP_SKIP_ROW
        // rows 0..255: one 32-row x 16-column item per warp; the 2R+p remaining rows are cut
        // into 32-row x 8-column items spread over all 16 warps (no warp does two full items)
        {
          const uint8_t* rbase = rawp + (size_t)(rs + prow) * RWP + cs;
          row_item<8>(reinterpret_cast<const uint32_t*>(rbase + 16 * g), wa, wb, ntap,
                      hbuf + prow * kBandHP + 16 * g, true, nc);
          const int n2 = nrow - 256;                       // 13 .. 2*rmax+3 rows
          const int items = ((n2 + 31) >> 5) * 4;          // 32 rows x 8 columns each
          for (int it = warp; it < items; it += 16) {
            const int r2 = 256 + 32 * (it >> 2) + lane;    // hbuf row
            const int c2 = 8 * (it & 3);
            row_item<4>(reinterpret_cast<const uint32_t*>(rawp + (size_t)(rs + r2) * RWP + cs + c2), wa, wb, ntap,
                        hbuf + r2 * kBandHP + c2, r2 < nrow, nc);
          }
        }
#endif
        __syncthreads();  // hbuf complete

        // ---------------- column pass + DoG + running argmax ----------------
#ifndef MHFD_EXP_SKIP_COL
        col_pass<kBandHP>(hbuf + (8 * rg + p) * kBandHP + 2 * cp, wC + tab.woff[lev], 2 * R + 1, lev,
                          lev > 0 ? tab.tdog[lev - 1] * inv : 0.f, lprev, vbest, ibest);
#endif
        __syncthreads();  // hbuf is rewritten by the next level
      }
      // ---- epilogue: v and argmax of the 256 x 32 block
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        const int y = Y0 + 8 * rg + o;
        const int x = x0 + 2 * cp;
        if (y < s.H) {
          const int64_t pidx = (int64_t)b * plane + (int64_t)y * s.W + x;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (x + c < s.W) {
              const int k = 2 * o + c;
              v_out[pidx + c] = vbest[k];
              idx_out[pidx + c] = (uint8_t)((ibest[k >> 2] >> ((k & 3) * 8)) & 0xffu);
            }
          }
        }
      }
    }
    if (tn >= ntiles) break;
    t = tn;
    bt = bn;
    mode = mode_n;
    __syncthreads();   // hbuf / rawp reuse by the next tile
  }
}

}  // namespace mhfd
