// k_band2.cuh — hot kernel for u8 images, two CTAs per SM ("band2" schedule).
//
// Same mathematics and the same register-blocked passes as k_band (row pass: lane = row,
// 16 outputs per thread, tap-pair FFMA2 on bytes converted in registers; column pass:
// 8 rows x 2 columns per thread, column-pair FFMA2), but a CTA is 256 threads on a
// 128-row band and needs ~84 KB of shared memory, so two CTAs share an SM and one CTA's
// staging, barriers and DoG updates overlap the other's FMA stream.  The raw band is
// staged by plain 4-byte loads straight into the saturated layout (p' = clamp(p, lo, hi),
// PAPER.md:257; the row pass re-centres x = p' - mid while converting), no landing buffer.  The taller-halo cost
// (row pass on 128 + 2R + p rows per 128) is the price of the second CTA.
#pragma once
#include "common.cuh"
#include "k_band.cuh"

namespace mhfd {

constexpr int kBand2Threads = 256;
constexpr int kBand2BH = 128;

__host__ __device__ inline int band2_raw_rows(int rmax) { return kBand2BH + 2 * rmax + 3; }
__host__ __device__ inline int band2_hrows(int rmax) { return kBand2BH + 2 * rmax + 19; }
__host__ __device__ inline size_t band2_rawp_bytes(int rmax) {
  return (((size_t)band2_raw_rows(rmax) + 1) * band_rwp(rmax) + 127) & ~(size_t)127;
}
__host__ __device__ inline size_t band2_smem(int rmax, int ntaps_total) {
  return band2_rawp_bytes(rmax) +
         sizeof(float) * ((size_t)band2_hrows(rmax) * kBandHP + 3 * (size_t)wtab_floats(ntaps_total));
}
__host__ __device__ inline bool band2_ok(int W, int H, int rmax, int ntaps_total) {
  return band2_smem(rmax, ntaps_total) <= 110 * 1024 && W >= band_raw_w(rmax) && H >= band2_raw_rows(rmax) &&
         2 * rmax + 3 <= 4 * 32;   // the second row-pass pass fits in 4 row groups
}

__global__ void __launch_bounds__(kBand2Threads, 2)
k_band2(const uint8_t* __restrict__ images, Shape s, const ImgPar* __restrict__ par,
        const __grid_constant__ LevelTable tab, float* __restrict__ v_out, uint8_t* __restrict__ idx_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int rmax = tab.rmax;
  const int RM = band_rm(rmax);
  const int RW = band_raw_w(rmax);
  const int NRB = band2_raw_rows(rmax);
  const int RWP = band_rwp(rmax);
  uint8_t* rawp = smem_raw;                                                  // (NRB+1) x RWP
  float* hbuf = reinterpret_cast<float*>(rawp + band2_rawp_bytes(rmax));     // hrows x 36
  float* wA = hbuf + band2_hrows(rmax) * kBandHP;
  float* wB = wA + wtab_floats(tab.ntaps_total);
  float* wC = wB + wtab_floats(tab.ntaps_total);

  const int b = blockIdx.z;
  const int x0 = blockIdx.x * kStripW;
  const int Y0 = blockIdx.y * kBand2BH;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t plane = (int64_t)s.H * s.W;
  const ImgPar ip = par[b];

  if (ip.degen) {  // hi == lo: I' == 0, every DoG plane is exactly 0
    for (int i = tid; i < kBand2BH * kStripW; i += kBand2Threads) {
      const int y = Y0 + i / kStripW, x = x0 + i % kStripW;
      if (x < s.W && y < s.H) {
        v_out[(int64_t)b * plane + (int64_t)y * s.W + x] = 0.f;
        idx_out[(int64_t)b * plane + (int64_t)y * s.W + x] = 0;
      }
    }
    return;
  }

  // ---- stage the band (rows Y0-rmax-3 .., columns x0-RM ..), saturated
  {
    const uint8_t* img = images + (int64_t)b * s.H * s.pitch;
    const int yr = Y0 - rmax - 3, xr = x0 - RM;
    const bool xin = xr >= 0 && xr + RW <= s.W;
    const uint32_t lo2 = (uint32_t)ip.lo * 0x10001u, hi2 = (uint32_t)ip.hi * 0x10001u;
    const int nw = RW / 4, nwp = RWP / 4;
#pragma unroll 4
    for (int r = warp; r <= NRB; r += 8) {
      uint32_t* drow = reinterpret_cast<uint32_t*>(rawp + (size_t)r * RWP);
      if (r == NRB) {   // padding row (meets zero taps only)
        for (int c4 = lane; c4 < nwp; c4 += 32) drow[c4] = 0u;
        continue;
      }
      const uint8_t* row = img + (int64_t)wrap_idx(yr + r, s.H) * s.pitch;
      for (int c4 = lane; c4 < nwp; c4 += 32) {
        uint32_t o = 0u;
        if (c4 < nw) {
          uint32_t wd;
          if (xin) {
            wd = __ldg(reinterpret_cast<const uint32_t*>(row + xr) + c4);
          } else {
            wd = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) wd |= (uint32_t)row[wrap_idx(xr + 4 * c4 + k, s.W)] << (8 * k);
          }
          o = clamp_bytes(wd, lo2, hi2);
        }
        drow[c4] = o;
      }
    }
  }
  for (int i = kBand2BH * kBandHP + tid; i < band2_hrows(rmax) * kBandHP; i += kBand2Threads) hbuf[i] = 0.f;
  for (int i = tid; i < tab.ntaps_total; i += kBand2Threads) wA[i] = tab.w[i];
  for (int l = 0; l < tab.nlev; ++l)
    for (int i = tid; i < tab.ntap[l] + 8; i += kBand2Threads) {
      wB[tab.woff[l] + i] = i ? tab.w[tab.woff[l] + i - 1] : 0.f;
      wC[tab.woff[l] + i] = i < 2 * tab.R[l] + 1 ? tab.w[tab.woff[l] + tab.pre[l] + i] : 0.f;
    }
  __syncthreads();

  const float inv = ip.inv;
  const int mid = ip.lo + (ip.hi - ip.lo + 1) / 2;   // x = p' - mid in [-128, 127]
  const float2 nc = make_float2(-(8388608.f + (float)mid), -(8388608.f + (float)mid));
  const int cp = lane & 15;                    // column pair
  const int rg = 2 * warp + (lane >> 4);       // row group 0..15 (8 rows each)
  const int prow = lane + 32 * (warp >> 1);    // row-pass row in a 128-row pass
  const int g = warp & 1;                      // row-pass column half
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
    const int nrow = kBand2BH + 2 * R + p;           // hbuf rows: band rows -R-p .. BH+R-1
    const int cs = RM - R - p;
    const int rs = rmax + 3 - R - p;
    // ---- row pass: rows 0..127 one 32x16 item per warp; the 2R+p remaining rows as
    //      32x16 items on warps 0 .. 2*ceil((2R+p)/32)-1
    row_item<8>(reinterpret_cast<const uint32_t*>(rawp + (size_t)(rs + prow) * RWP + cs + 16 * g), wa, wb, ntap,
                hbuf + prow * kBandHP + 16 * g, true, nc);
    {
      const int items = ((nrow - kBand2BH + 31) >> 5) * 2;
      if (warp < items) {
        const int r2 = kBand2BH + 32 * (warp >> 1) + lane;
        row_item<8>(reinterpret_cast<const uint32_t*>(rawp + (size_t)(rs + r2) * RWP + cs + 16 * g), wa, wb, ntap,
                    hbuf + r2 * kBandHP + 16 * g, r2 < nrow, nc);
      }
    }
    __syncthreads();  // hbuf complete
    col_pass<kBandHP>(hbuf + (8 * rg + p) * kBandHP + 2 * cp, wC + tab.woff[lev], 2 * R + 1, lev,
                      lev > 0 ? tab.tdog[lev - 1] * inv : 0.f, lprev, vbest, ibest);
    __syncthreads();  // hbuf is rewritten by the next level
  }

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
