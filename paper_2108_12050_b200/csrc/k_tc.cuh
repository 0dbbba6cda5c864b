// k_tc.cuh — the hot kernel for u8 images on the 5th-generation tensor cores
// (hot-path rows a2-a6, "banded-GEMM formulation of the blur").
//
// Same mathematics as k_band / k_scale_space: stretch, sampled
// renormalised Gaussian blur at every level with periodic wrap (PAPER.md:134-141,
// :166-168), DoG = t_i (L_{i+1} - L_i) (Eq. 2), first argmax over the
// scales.  Per 128 x 128 output tile and level i the separable blur
// is two banded products on tcgen05 (tc_plan.h gives the geometry and tables):
//
//   row pass    D1[c][n] = sum_k T_i[c][k] X[c0+n][c0+k]        SS MMA, M=128, N=K_i
//               (A = Toeplitz pairs in smem, B = the staged tile X, fp16 exact
//               integers x = p' - mid; T = hi + lo fp16 split of 2^12 w)
//   split       D1 -> (hi, lo) fp16 in place in TMEM (A operand of the next pass)
//   column pass D2[c][m] = sum_k A2[c][k] T_i[m][k]             TS MMA, M=128, N=128
//               (A2_hi T_hi + A2_hi T_lo + A2_lo T_hi)
//   epilogue    DoG, running max and first argmax in registers (lane = column c,
//               32 rows per thread), overlapped with the next level's row pass.
//
// Persistent: one 512-thread CTA per SM walks tiles; the next tile's raw u8 window
// ((S+off) x S bytes, periodic) is fetched by TMA / bulk copies while the current
// tile computes; each level's Toeplitz table (<= 22.5 KB) is bulk-copied from the
// context's device table two levels ahead into a double buffer.
// Accuracy (tools/umma_probe.cu): D1 and D2 within ~1e-6 relative of f64 sums.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "k_band.cuh"
#include "k_scale_space.cuh"
#include "tc_plan.h"
#include "umma.cuh"

namespace mhfd {

constexpr int kTcThreads = 512;

__host__ __device__ inline int tc_off(const TcPlan& P) { return (16 - P.H0 % 16) % 16; }   // landing column offset
__host__ __device__ inline int tc_lw(const TcPlan& P) { return (P.S + tc_off(P) + 15) / 16 * 16; }
__host__ __device__ inline size_t tc_b1_bytes(const TcPlan& P) { return (size_t)P.S * P.S * 2; }
__host__ __device__ inline size_t tc_land_bytes(const TcPlan& P) { return (size_t)tc_lw(P) * P.S; }
__host__ __device__ inline size_t tc_smem(const TcPlan& P) {
  return tc_b1_bytes(P) + tc_land_bytes(P) + 2 * (size_t)P.max_level_bytes + 64;
}
inline bool tc_ok(const TcPlan& P, int W, int H) {
  return P.S > 0 && tc_lw(P) <= 256 && tc_smem(P) <= 227 * 1024 && W >= tc_lw(P) && H >= P.S;
}

struct TcTile {
  int b, x0, y0;
};
__device__ __forceinline__ TcTile tc_tile(int t, int tx, int ty) {
  TcTile r;
  r.x0 = (t % tx) * kTcTile;
  t /= tx;
  r.y0 = (t % ty) * kTcTile;
  r.b = t / ty;
  return r;
}

// Fetch the raw window of tile tt into `land` (LW x S bytes, row pitch LW): columns
// x0 - H0 - off .. +LW, rows y0 - H0 .. +S, periodic.  Mode as band_fetch: 2 = TMA box,
// 1 = bulk copies per row, 0 = plain loads (complete on return).
__device__ __forceinline__ int tc_fetch(const TcTile& tt, uint8_t* land, uint64_t* bar, const uint8_t* images,
                                        const Shape& s, const CUtensorMap* tmap, int use_tmap, const TcPlan& P) {
  const int LW = tc_lw(P), S = P.S;
  const int xr = tt.x0 - P.H0 - tc_off(P), yr = tt.y0 - P.H0;
  const int tid = threadIdx.x;
  const bool tma = use_tmap && xr >= 0 && xr + LW <= s.W && yr >= 0 && yr + S <= s.H;
  const bool bulk = !tma && (s.W % 16) == 0 && (s.pitch % 16) == 0;
  if (tma) {
    if (tid == 0) {
      mbar_arrive_expect_tx(bar, (uint32_t)(LW * S));
      tma_2d_g2s(land, tmap, xr, tt.b * s.H + yr, bar);
    }
    return 2;
  }
  const uint8_t* img = images + (int64_t)tt.b * s.H * s.pitch;
  if (bulk) {
    if (tid == 0) mbar_arrive_expect_tx(bar, (uint32_t)(S * LW));
    __syncthreads();   // expect_tx registered before any copy completes
    const int xw = wrap_idx(xr, s.W);
    for (int r = tid; r < S; r += kTcThreads) {
      const uint8_t* row = img + (int64_t)wrap_idx(yr + r, s.H) * s.pitch;
      uint8_t* dst = land + (size_t)r * LW;
      if (xw + LW > s.W) {
        bulk_g2s(dst, row + xw, (uint32_t)(s.W - xw), bar);
        bulk_g2s(dst + (s.W - xw), row, (uint32_t)(xw + LW - s.W), bar);
      } else {
        bulk_g2s(dst, row + xw, (uint32_t)LW, bar);
      }
    }
    return 1;
  }
  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < S; r += kTcThreads / 32) {
    const uint8_t* row = img + (int64_t)wrap_idx(yr + r, s.H) * s.pitch;
    for (int c = lane; c < LW; c += 32) land[(size_t)r * LW + c] = row[wrap_idx(xr + c, s.W)];
  }
  return 0;
}

__global__ void __launch_bounds__(kTcThreads, 1)
k_tc(const uint8_t* __restrict__ images, Shape s, const ImgPar* __restrict__ par, const __grid_constant__ TcPlan P,
     const uint8_t* __restrict__ tabs, const __grid_constant__ CUtensorMap tmap, int use_tmap,
     float* __restrict__ v_out, uint8_t* __restrict__ idx_out, int batch) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int S = P.S, LW = tc_lw(P), OFF = tc_off(P);
  uint8_t* B1 = smem_raw;                                          // S x S fp16, canonical K-major
  uint8_t* land = B1 + tc_b1_bytes(P);                             // LW x S raw bytes
  uint8_t* tbuf = land + tc_land_bytes(P);                         // 2 x max_level_bytes
  uint64_t* bars = reinterpret_cast<uint64_t*>(tbuf + 2 * (size_t)P.max_level_bytes);   // land, mma, tab0, tab1
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  uint64_t* bar_land = bars;
  uint64_t* bar_mma = bars + 1;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, wg = warp >> 2;   // TMEM lane quarter, row group
  const int tx = (s.W + kTcTile - 1) / kTcTile, ty = (s.H + kTcTile - 1) / kTcTile;
  const int ntiles = tx * ty * batch;
  int t = blockIdx.x;
  if (t >= ntiles) return;
  const int my_tiles = (ntiles - 1 - t) / gridDim.x + 1;
  const int G = my_tiles * P.nlev;   // levels this CTA processes
  const int SBO1 = (S / 8) * 128;
  const int64_t plane = (int64_t)s.H * s.W;

  if (tid == 0) {
    for (int k = 0; k < 4; ++k) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc(tslot, 512);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;            // D1 / A2: columns [0, 256); D2: [256, 384)
  const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);

  auto issue_table = [&](int g) {          // thread 0: level table of global level g
    const int lev = g % P.nlev;
    const int bytes = 2 * P.lev[lev].npairs * 256;
    uint64_t* tb = &bars[2 + (g & 1)];
    mbar_arrive_expect_tx(tb, (uint32_t)bytes);
    bulk_g2s(tbuf + (size_t)(g & 1) * P.max_level_bytes, tabs + P.lev[lev].tab_off, (uint32_t)bytes, tb);
  };
  if (tid == 0) {
    issue_table(0);
    if (G > 1) issue_table(1);
  }
  TcTile tt = tc_tile(t, tx, ty);
  int mode = tc_fetch(tt, land, bar_land, images, s, &tmap, use_tmap, P);
  uint32_t land_phase = 0, mma_phase = 0;
  int g = 0;

  for (int it = 0;; ++it) {
    // ---- staged raw window -> B1 (saturate, centre, fp16 exact)
    if (mode) {
      mbar_wait(bar_land, land_phase);
      land_phase ^= 1u;
    }
    __syncthreads();
    const ImgPar ip = par[tt.b];
    const int lo = ip.lo, hi = ip.hi;
    const int mid = lo + (hi - lo + 1) / 2;
    {
      const uint32_t lo2 = (uint32_t)lo * 0x10001u, hi2 = (uint32_t)hi * 0x10001u;
      const __half2 cm = __floats2half2_rn(1024.f + (float)mid, 1024.f + (float)mid);
      const int nchunk = S * S / 8;
      for (int gch = tid; gch < nchunk; gch += kTcThreads) {
        const int cm8 = gch >> 3;
        const int r = (cm8 / (S / 8)) * 8 + (gch & 7), kc = cm8 % (S / 8);
        const uint2 raw = *reinterpret_cast<const uint2*>(land + (size_t)r * LW + OFF + 8 * kc);
        const uint32_t a = clamp_bytes(raw.x, lo2, hi2), bb = clamp_bytes(raw.y, lo2, hi2);
        uint4 o;
        const uint32_t p0 = __byte_perm(a, 0x64646464u, 0x4140u), p1 = __byte_perm(a, 0x64646464u, 0x4342u);
        const uint32_t p2 = __byte_perm(bb, 0x64646464u, 0x4140u), p3 = __byte_perm(bb, 0x64646464u, 0x4342u);
        __half2 x0 = __hsub2(*reinterpret_cast<const __half2*>(&p0), cm);
        __half2 x1 = __hsub2(*reinterpret_cast<const __half2*>(&p1), cm);
        __half2 x2 = __hsub2(*reinterpret_cast<const __half2*>(&p2), cm);
        __half2 x3 = __hsub2(*reinterpret_cast<const __half2*>(&p3), cm);
        o.x = *reinterpret_cast<uint32_t*>(&x0);
        o.y = *reinterpret_cast<uint32_t*>(&x1);
        o.z = *reinterpret_cast<uint32_t*>(&x2);
        o.w = *reinterpret_cast<uint32_t*>(&x3);
        *reinterpret_cast<uint4*>(B1 + (size_t)gch * 16) = o;
      }
    }
    umma::fence_async_smem();
    __syncthreads();   // B1 ready (async proxy), landing free
    const int tn = t + gridDim.x;
    TcTile tn_t;
    int mode_n = 0;
    if (tn < ntiles) {
      tn_t = tc_tile(tn, tx, ty);
      mode_n = tc_fetch(tn_t, land, bar_land, images, s, &tmap, use_tmap, P);
    }

    const float inv = ip.inv * (1.f / kTcWScale);
    float lprev[32], vbest[32];
    uint32_t ibest[8];
#pragma unroll
    for (int u = 0; u < 32; ++u) { lprev[u] = 0.f; vbest[u] = -INFINITY; }
#pragma unroll
    for (int u = 0; u < 8; ++u) ibest[u] = 0u;

    // DoG epilogue of level `lev` (D2 holds L_lev): rows 32 wg .. +32 of column c = 32 q + lane
    auto consume = [&](int lev) {
      uint32_t r0[16], r1[16];
      umma::ld16(tq + 256 + 32 * wg, r0);
      umma::ld16(tq + 256 + 32 * wg + 16, r1);
      umma::wait_ld();
      const float tf = lev > 0 ? P.lev[lev - 1].tdog * inv : 0.f;
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const float L = __uint_as_float(u < 16 ? r0[u] : r1[u - 16]);
        if (lev > 0) {
          const float D = tf * (L - lprev[u]);
          if (D > vbest[u]) {
            vbest[u] = D;
            const int sh = (u & 3) * 8;
            ibest[u >> 2] = (ibest[u >> 2] & ~(0xffu << sh)) | ((uint32_t)(lev - 1) << sh);
          }
        }
        lprev[u] = L;
      }
    };

    for (int lev = 0; lev < P.nlev; ++lev, ++g) {
      const TcLevel& L = P.lev[lev];
      const int K = L.K;
      const int npairs = L.npairs, E1 = K / 8 - 2;
      const uint32_t thi = umma::smem_addr(tbuf + (size_t)(g & 1) * P.max_level_bytes);
      const uint32_t tlo = thi + npairs * 256;
      // ---- row pass (thread 0 issues)
      if (tid == 0) {
        mbar_wait(&bars[2 + (g & 1)], (uint32_t)((g >> 1) & 1));
        umma::fence_after();
        const uint32_t b1 = umma::smem_addr(B1) + (L.c0 / 8) * SBO1 + (L.c0 / 8) * 128;
        const uint32_t id = umma::idesc_f16(128, K);
        for (int j = 0; j < K / 16; ++j) {
          const uint64_t bd = umma::desc_kmajor(b1 + 256 * j, 128, SBO1);
          umma::mma_ss(tmem, umma::desc_kmajor(thi + (E1 - 2 * j) * 256, 128, 256), bd, id, j > 0);
          umma::mma_ss(tmem, umma::desc_kmajor(tlo + (E1 - 2 * j) * 256, 128, 256), bd, id, 1);
        }
        umma::commit(bar_mma);
      }
      // ---- previous level's DoG epilogue overlaps the row pass
      if (lev > 0) consume(lev - 1);
      mbar_wait(bar_mma, mma_phase);
      mma_phase ^= 1u;
      umma::fence_after();
      // ---- split D1 -> (hi, lo) fp16 in place: chunk j = 16 columns -> hi at 16j, lo at 16j+8
      for (int j = wg; j < K / 16; j += 4) {
        uint32_t r[16];
        umma::ld16(tq + 16 * j, r);
        umma::wait_ld();
        uint32_t h8[8], l8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float y0 = __uint_as_float(r[2 * u]) * (1.f / kTcWScale);
          const float y1 = __uint_as_float(r[2 * u + 1]) * (1.f / kTcWScale);
          const __half2 hh = __floats2half2_rn(y0, y1);
          const float2 hf = __half22float2(hh);
          const __half2 ll = __floats2half2_rn(y0 - hf.x, y1 - hf.y);
          h8[u] = *reinterpret_cast<const uint32_t*>(&hh);
          l8[u] = *reinterpret_cast<const uint32_t*>(&ll);
        }
        umma::st8(tq + 16 * j, h8);
        umma::st8(tq + 16 * j + 8, l8);
      }
      umma::wait_st();
      umma::fence_before();
      __syncthreads();
      // ---- column pass (thread 0 issues)
      if (tid == 0) {
        umma::fence_after();
        const uint32_t id = umma::idesc_f16(128, 128);
        for (int j = 0; j < K / 16; ++j) {
          const uint64_t bh = umma::desc_kmajor(thi + (E1 - 2 * j) * 256, 128, 256);
          const uint64_t bl = umma::desc_kmajor(tlo + (E1 - 2 * j) * 256, 128, 256);
          umma::mma_ts(tmem + 256, tmem + 16 * j, bh, id, j > 0);
          umma::mma_ts(tmem + 256, tmem + 16 * j, bl, id, 1);
          umma::mma_ts(tmem + 256, tmem + 16 * j + 8, bh, id, 1);
        }
        umma::commit(bar_mma);
      }
      mbar_wait(bar_mma, mma_phase);
      mma_phase ^= 1u;
      umma::fence_after();
      // table buffer (g & 1) is free: prefetch level g + 2
      if (tid == 0 && g + 2 < G) issue_table(g + 2);
    }
    consume(P.nlev - 1);
    umma::fence_before();   // TMEM reads done before the next tile's MMAs (after the barrier below)

    // ---- v and argmax of column c, rows 32 wg .. +32
    {
      const int x = tt.x0 + 32 * q + lane;
      const bool degen = ip.degen != 0;
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int y = tt.y0 + 32 * wg + u;
        if (x < s.W && y < s.H) {
          const int64_t pidx = (int64_t)tt.b * plane + (int64_t)y * s.W + x;
          v_out[pidx] = degen ? 0.f : vbest[u];
          idx_out[pidx] = degen ? (uint8_t)0 : (uint8_t)((ibest[u >> 2] >> ((u & 3) * 8)) & 0xffu);
        }
      }
    }
    if (tn >= ntiles) break;
    t = tn;
    tt = tn_t;
    mode = mode_n;
    __syncthreads();
    umma::fence_after();
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 512);
}

}  // namespace mhfd
