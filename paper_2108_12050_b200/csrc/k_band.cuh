// k_band.cuh — the hot kernel for u8 images (hot-path rows a2-a6), "band" schedule.
//
// Same arithmetic as k_scale_space (PAPER.md:136-141 blur, :171 Eq. 2 DoG, :240-244
// inner argmax, :257 stretch), laid out for one CTA per SM:
//
//   CTA = one image x one strip of 32 columns x one band of BH = 256 rows, 512 threads.
//   prologue   : the raw u8 band with its halo ((256+2Rmax+3) x (32+2Rmax+8) bytes, ~52
//                KB at sigma <= 10) is read from HBM ONCE into shared memory; every level
//                then re-reads it from shared memory (6.5 B/px of L2 traffic instead of
//                ~150 B/px for restaging an f32 image per level).
//   per level  : for each chunk of 128 rows: stretch+centre the needed raw bytes into an
//                f32 chunk buffer (same f32 arithmetic as k_normalize), then
//                the row pass: lane = row, 8 consecutive output columns per thread, tap-pair
//                FFMA2 (weights wA = w, wB = w shifted by one) -> hbuf.  Then the column
//                pass: 8 rows x 2 columns per thread, column-pair FFMA2 with a broadcast
//                weight, DoG / running max / first argmax kept in registers.
//   epilogue   : v (f32) and argmax (u8) of the 256 x 32 block to HBM.
//
// Shared-memory traffic per FMA is what bounds this loop on B200 (128 B/clk/SM against
// 128 FMA/clk/SM): both passes are register-blocked so one 16-byte (row pass) or 8-byte
// (column pass) load feeds 16 FMAs, and weight loads are warp-broadcast (1 wavefront).
#pragma once
#include "common.cuh"
#include "k_scale_space.cuh"

namespace mhfd {

constexpr int kBandThreads = 512;
constexpr int kBandBH = 256;
constexpr int kBandChunk = 128;   // row-pass rows per chunk (4 warps x 32 lanes)
constexpr int kBandHP = 36;       // hbuf pitch: 4 x odd -> conflict-free STS.128 by rows

__host__ __device__ inline int band_rmax4(int rmax) { return (rmax + 3 + 15) & ~15; }  // >= rmax+3, 16-byte aligned TMA box start
__host__ __device__ inline int band_raw_w(int rmax) { return (kStripW + 2 * band_rmax4(rmax) + 15) & ~15; }
__host__ __device__ inline int band_raw_rows(int rmax) { return kBandBH + 2 * rmax + 3; }
constexpr int kBandBoxRows = 128;   // TMA box height for the raw band
__host__ __device__ inline int band_raw_alloc_rows(int rmax) {
  return (band_raw_rows(rmax) + kBandBoxRows - 1) / kBandBoxRows * kBandBoxRows;
}
__host__ __device__ inline int band_fp(int rmax) {   // f32 chunk pitch: 4 x odd, >= the row-pass window reach
  int q = (2 * rmax + 3 + 8 + 32 + 3) / 4;
  if ((q & 1) == 0) ++q;
  return 4 * q;
}
__host__ __device__ inline int band_hrows(int rmax) { return kBandBH + 2 * rmax + 19; }
__host__ __device__ inline size_t band_smem(int rmax, int ntaps_total) {
  const size_t raw = ((size_t)band_raw_alloc_rows(rmax) * band_raw_w(rmax) + 127) & ~(size_t)127;
  return raw + sizeof(float) * ((size_t)kBandChunk * band_fp(rmax) + (size_t)band_hrows(rmax) * kBandHP +
                                2 * (size_t)wtab_floats(ntaps_total)) + 16;
}
// the band schedule needs the raw band to fit (sigma_max <= ~12) and one wrap at most
__host__ __device__ inline bool band_ok(int W, int H, int rmax, int ntaps_total) {
  return band_smem(rmax, ntaps_total) <= 220 * 1024 && W >= band_raw_w(rmax) && H >= band_raw_rows(rmax);
}

__global__ void __launch_bounds__(kBandThreads, 1)
k_band(const uint8_t* __restrict__ images, Shape s, const ImgPar* __restrict__ par,
       const __grid_constant__ LevelTable tab, const __grid_constant__ CUtensorMap tmap, int use_tmap,
       float* __restrict__ v_out, uint8_t* __restrict__ idx_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int rmax = tab.rmax;
  const int RM4 = band_rmax4(rmax);
  const int RW = band_raw_w(rmax);
  const int NRB = band_raw_rows(rmax);
  const int FP = band_fp(rmax);
  uint8_t* raw = smem_raw;                                                            // NRB x RW bytes
  float* fb = reinterpret_cast<float*>(smem_raw + (((size_t)band_raw_alloc_rows(rmax) * RW + 127) & ~(size_t)127));
  float* hbuf = fb + kBandChunk * FP;                                                 // hrows x 36
  float* wA = hbuf + band_hrows(rmax) * kBandHP;
  float* wB = wA + wtab_floats(tab.ntaps_total);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wB + wtab_floats(tab.ntaps_total));

  const int b = blockIdx.z;
  const int x0 = blockIdx.x * kStripW;
  const int Y0 = blockIdx.y * kBandBH;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t plane = (int64_t)s.H * s.W;
  const ImgPar ip = par[b];

  if (ip.degen) {  // hi == lo: I' == 0, every DoG plane is exactly 0
    for (int i = tid; i < kBandBH * kStripW; i += kBandThreads) {
      const int y = Y0 + i / kStripW, x = x0 + i % kStripW;
      if (x < s.W && y < s.H) {
        v_out[(int64_t)b * plane + (int64_t)y * s.W + x] = 0.f;
        idx_out[(int64_t)b * plane + (int64_t)y * s.W + x] = 0;
      }
    }
    return;
  }

  // ---- prologue: raw band (rows Y0-rmax-3 .., cols x0-RM4 ..) -> shared memory, once
  {
    const int yr = Y0 - rmax - 3, xr = x0 - RM4;
    const bool interior = use_tmap && xr >= 0 && xr + RW <= s.W && yr >= 0 && yr + NRB <= s.H;
    if (interior) {   // TMA: ceil(NRB/128) boxes of 128 rows x RW bytes
      if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int nbox = band_raw_alloc_rows(rmax) / kBandBoxRows;
        mbar_arrive_expect_tx(bar, (uint32_t)(nbox * kBandBoxRows * RW));
        for (int k = 0; k < nbox; ++k)
          tma_2d_g2s(raw + (size_t)k * kBandBoxRows * RW, &tmap, xr, b * s.H + yr + k * kBandBoxRows, bar);
      }
    } else {          // image edge: plain loads with periodic wrap
      const uint8_t* img = images + (int64_t)b * s.H * s.pitch;
      const int nw = RW / 4;   // 32-bit words per raw row
      const bool xin = xr >= 0 && xr + RW <= s.W;
      for (int i = tid; i < NRB * nw; i += kBandThreads) {
        const int r = i / nw, c4 = i - r * nw;
        const uint8_t* row = img + (int64_t)wrap_idx(yr + r, s.H) * s.pitch;
        uint32_t wd;
        if (xin) {
          wd = __ldg(reinterpret_cast<const uint32_t*>(row + xr) + c4);
        } else {
          wd = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) wd |= (uint32_t)row[wrap_idx(xr + 4 * c4 + k, s.W)] << (8 * k);
        }
        reinterpret_cast<uint32_t*>(raw)[i] = wd;
      }
    }
  }
  for (int i = tid; i < kBandChunk * FP + band_hrows(rmax) * kBandHP; i += kBandThreads) fb[i] = 0.f;
  for (int i = tid; i < tab.ntaps_total; i += kBandThreads) wA[i] = tab.w[i];
  for (int l = 0; l < tab.nlev; ++l)
    for (int i = tid; i < tab.ntap[l] + 8; i += kBandThreads) wB[tab.woff[l] + i] = i ? tab.w[tab.woff[l] + i - 1] : 0.f;

  // wait for the band, then saturate every byte to [lo, hi] once so the
  // per-level conversion is one I2F + one FFMA per element
  {
    const int yr = Y0 - rmax - 3, xr = x0 - RM4;
    if (use_tmap && xr >= 0 && xr + RW <= s.W && yr >= 0 && yr + NRB <= s.H) {
      __syncthreads();   // barrier init visible before anyone waits
      mbar_wait(bar, 0);
    }
  }
  __syncthreads();
  {
    const uint32_t l = (uint32_t)ip.lo, h = (uint32_t)ip.hi;
    uint32_t* rw = reinterpret_cast<uint32_t*>(raw);
    for (int i = tid; i < NRB * (RW / 4); i += kBandThreads) {
      const uint32_t wd = rw[i];
      uint32_t o = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) o |= min(max((wd >> (8 * k)) & 255u, l), h) << (8 * k);
      rw[i] = o;
    }
  }
  const float inv = ip.inv;
  const float c0 = -(float)ip.lo * inv - 0.5f;   // f = p' * inv + c0, p' = clamp(p, lo, hi)

  // column-pass ownership: 8 rows x 2 columns
  const int cp = lane & 15;                    // column pair
  const int rg = 2 * warp + (lane >> 4);       // row group 0..31
  float lprev[16], vbest[16];
  uint32_t ibest[4];
#pragma unroll
  for (int k = 0; k < 16; ++k) { lprev[k] = 0.f; vbest[k] = -INFINITY; }
#pragma unroll
  for (int k = 0; k < 4; ++k) ibest[k] = 0u;

  // row-pass ownership: row lane + 32*(warp/4) of the chunk, columns 8g .. 8g+7
  const int prow = lane + 32 * (warp >> 2);
  const int g = warp & 3;

  for (int lev = 0; lev < tab.nlev; ++lev) {
    const int R = tab.R[lev], p = tab.pre[lev], ntap = tab.ntap[lev];
    const float* wa = wA + tab.woff[lev];
    const float* wb = wB + tab.woff[lev];
    const int nrow = kBandBH + 2 * R + p;            // hbuf rows: band rows -R-p .. BH+R-1
    const int ngrp = (kStripW + 2 * R + p + 3) >> 2; // 4-column groups to convert per row
    const int cs = RM4 - R - p;                      // raw column of f32 column 0 (multiple of 4)
    const int rs = rmax + 3 - R - p;                 // raw row of hbuf row 0
    const uint32_t magic = 0xffffffffu / (uint32_t)ngrp + 1u;   // i / ngrp for small i

    for (int r0 = 0; r0 < nrow; r0 += kBandChunk) {
      const int nr = min(kBandChunk, nrow - r0);
      __syncthreads();  // fb free (previous chunk's row pass done)
      // stretch + centre raw -> f32
      for (int i = tid; i < nr * ngrp; i += kBandThreads) {
        const int r = (int)__umulhi((uint32_t)i, magic);
        const int q = i - r * ngrp;
        const uint32_t wd = *reinterpret_cast<const uint32_t*>(raw + (size_t)(rs + r0 + r) * RW + cs + 4 * q);
        float4 f;
        f.x = fmaf((float)(wd & 255u), inv, c0);
        f.y = fmaf((float)((wd >> 8) & 255u), inv, c0);
        f.z = fmaf((float)((wd >> 16) & 255u), inv, c0);
        f.w = fmaf((float)(wd >> 24), inv, c0);
        *reinterpret_cast<float4*>(fb + r * FP + 4 * q) = f;
      }
      __syncthreads();
      if (32 * (warp >> 2) < nr) {   // warp-uniform: skip warps past the last row
        // row pass: 8 outputs per thread, tap pairs (wA for even, wB for odd outputs)
        const float4* s4 = reinterpret_cast<const float4*>(fb + prow * FP + 8 * g);
        float2 acc[8];
#pragma unroll
        for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.f, 0.f);
        float4 x0v = s4[0], x1v = s4[1];
        for (int j = 0; j < ntap; j += 8) {
          const int q4 = j >> 2;
          const float4 x2v = s4[q4 + 2], x3v = s4[q4 + 3];
          const float2 P[8] = {lo2(x0v), hi2(x0v), lo2(x1v), hi2(x1v), lo2(x2v), hi2(x2v), lo2(x3v), hi2(x3v)};
          const float4 A0 = reinterpret_cast<const float4*>(wa)[q4], A1 = reinterpret_cast<const float4*>(wa)[q4 + 1];
          const float4 B0 = reinterpret_cast<const float4*>(wb)[q4], B1 = reinterpret_cast<const float4*>(wb)[q4 + 1];
          const float2 WA[4] = {lo2(A0), hi2(A0), lo2(A1), hi2(A1)};
          const float2 WB[4] = {lo2(B0), hi2(B0), lo2(B1), hi2(B1)};
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              acc[2 * qq] = __ffma2_rn(P[qq + kk], WA[kk], acc[2 * qq]);
              acc[2 * qq + 1] = __ffma2_rn(P[qq + kk], WB[kk], acc[2 * qq + 1]);
            }
          }
          x0v = x2v;
          x1v = x3v;
        }
        {  // odd outputs: tap pair (ntap-1, ntap) on input pairs ntap/2 + qq
          const float2 wl = reinterpret_cast<const float2*>(wb)[ntap >> 1];
          const float2 P[4] = {lo2(x0v), hi2(x0v), lo2(x1v), hi2(x1v)};
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) acc[2 * qq + 1] = __ffma2_rn(P[qq], wl, acc[2 * qq + 1]);
        }
        if (prow < nr) {
          float4* h = reinterpret_cast<float4*>(hbuf + (r0 + prow) * kBandHP + 8 * g);
          h[0] = make_float4(acc[0].x + acc[0].y, acc[1].x + acc[1].y, acc[2].x + acc[2].y, acc[3].x + acc[3].y);
          h[1] = make_float4(acc[4].x + acc[4].y, acc[5].x + acc[5].y, acc[6].x + acc[6].y, acc[7].x + acc[7].y);
        }
      }
    }
    __syncthreads();  // hbuf complete

    // column pass: rows 8rg .. 8rg+7, columns 2cp, 2cp+1; hbuf row (8rg + o + t) at tap t
    {
      const float* src = hbuf + (8 * rg) * kBandHP + 2 * cp;
      float2 acc[8];
#pragma unroll
      for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.f, 0.f);
      float2 Xa[8], Xb[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) Xa[k] = *reinterpret_cast<const float2*>(src + k * kBandHP);
      int j = 0;
      auto group = [&](const float2 (&Xl)[8], const float2 (&Xh)[8], int jj) {
        const float4 W0 = reinterpret_cast<const float4*>(wa + jj)[0];
        const float4 W1 = reinterpret_cast<const float4*>(wa + jj)[1];
        const float w8[8] = {W0.x, W0.y, W0.z, W0.w, W1.x, W1.y, W1.z, W1.w};
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float2 wt = make_float2(w8[t], w8[t]);
#pragma unroll
          for (int o = 0; o < 8; ++o) {
            const int m = o + t;
            acc[o] = __ffma2_rn(m < 8 ? Xl[m] : Xh[m - 8], wt, acc[o]);
          }
        }
      };
      for (; j + 16 <= ntap; j += 16) {
#pragma unroll
        for (int k = 0; k < 8; ++k) Xb[k] = *reinterpret_cast<const float2*>(src + (j + 8 + k) * kBandHP);
        group(Xa, Xb, j);
#pragma unroll
        for (int k = 0; k < 8; ++k) Xa[k] = *reinterpret_cast<const float2*>(src + (j + 16 + k) * kBandHP);
        group(Xb, Xa, j + 8);
      }
      if (j < ntap) {
#pragma unroll
        for (int k = 0; k < 8; ++k) Xb[k] = *reinterpret_cast<const float2*>(src + (j + 8 + k) * kBandHP);
        group(Xa, Xb, j);
      }
      const float tprev = lev > 0 ? tab.tdog[lev - 1] : 0.f;
#pragma unroll
      for (int o = 0; o < 8; ++o) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int k = 2 * o + c;
          const float L = c ? acc[o].y : acc[o].x;
          if (lev > 0) {
            const float D = tprev * (L - lprev[k]);
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

}  // namespace mhfd
