// k_tc2.cuh — the two-pass tensor-core schedule (hot-path rows a2-a6 for u16 / f32
// images and radii beyond k_tc's staged tile).  Geometry and
// operand tables: tc2_plan.h.  Mathematics as every other schedule: stretch
// (PAPER.md:257), sampled renormalised Gaussian at every level with periodic wrap
// (PAPER.md:134-141, 166-168), DoG = t_i (L_{i+1} - L_i) (Eq. 2), first
// argmax over the scales.
//
//   k_tc2_prep  stretch + centre + x1024 -> fp16 hi/lo planes, tiled so that the staged
//               window of every k_tc2_rows tile is one contiguous run per plane
//   k_tc2_rows  persistent; warp 16 issues tcgen05.mma (SS, M=128 columns, N=NR rows,
//               3 fp16 products), warp 17 bulk-copies the tile's X window and each
//               level's Toeplitz pairs; 16 epilogue warps drain D1 (double-buffered in
//               TMEM), split 2^-12 Rx into fp16 hi/lo and store 16-byte pieces of the
//               transposed slabs (a warp writes 512 contiguous bytes)
//   k_tc2_cols  persistent; warp 17 streams each level's Rx slabs (two 4 KB bulk copies
//               per K-step) through a 10-stage ring, warp 16 issues the SS MMAs (M=128
//               columns, N=224 rows, 3 products), 16 epilogue warps form the DoG from
//               the two TMEM accumulators (L_i, L_{i-1}), keep the running max / first
//               argmax in registers and write v / argmax (or the DoG planes)
//
// Precision: x = 1024 (clamp((p-lo) inv, 0, 1) - 1/2) split hi + lo (~22 bits), weights
// 4096 w split hi + lo, the row sums 2^-12 Rx split again; the dropped lo x lo terms are
// ~2^-22 relative.  Accumulation in f32 (TMEM).
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "k_scale_space.cuh"
#include "tc2_plan.h"
#include "umma.cuh"

namespace mhfd {

constexpr int kT2Epi = 512;                // 16 epilogue warps
constexpr int kT2Threads = kT2Epi + 64;    // + MMA issuer warp + copy producer warp

__device__ __forceinline__ void t2_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void t2_epi_sync() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

// 8 f32 -> 4 packed half2 hi and 4 packed half2 lo (value = hi + lo to ~2^-22 relative)
__device__ __forceinline__ void t2_split8(const float (&f)[8], uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const __half2 hh = __floats2half2_rn(f[2 * u], f[2 * u + 1]);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(f[2 * u] - hf.x, f[2 * u + 1] - hf.y);
    h[u] = *reinterpret_cast<const uint32_t*>(&hh);
    l[u] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Byte offsets of the tiled buffers.
//  X  (k_tc2_prep -> k_tc2_rows): [b][plane][rt][cg = W/8][NR rows][8 cols] fp16
//  Rx (k_tc2_rows -> k_tc2_cols): [b][lev][plane][xt = W/128][rc = H/16][kg 2][c 128][8 rows] fp16
__host__ __device__ inline size_t t2_x_plane_bytes(int W, int nrt, int NR) { return (size_t)nrt * NR * W * 2; }
__host__ __device__ inline size_t t2_rx_plane_bytes(int W, int H) { return (size_t)W * H * 2; }

// ---------------------------------------------------------------------------------
// k_tc2_prep: one thread per (image, row, 8-column group); consecutive threads take
// consecutive rows of one column group, so the 16-byte output pieces are contiguous.
// Reflect (pg, pr > 0): the staged image has pg mirrored column groups of 8 on either
// side and pr mirrored rows above and below (staged row r = image row r - pr, half-sample
// symmetric, reading R25); periodic: pg = pr = 0.
template <int BPP>
__global__ void __launch_bounds__(256) k_tc2_prep(const uint8_t* __restrict__ images, Shape s,
                                                  const ImgPar* __restrict__ par, uint8_t* __restrict__ xt, int NR,
                                                  int nrt, int batch, int pg = 0, int pr = 0) {
  const int G = s.W / 8 + 2 * pg;
  const int hx = s.H + 2 * pr;
  const int64_t rows_pad = (int64_t)nrt * NR;
  const int64_t per_img = rows_pad * G;
  const int64_t total = per_img * batch;
  const size_t pb = t2_x_plane_bytes(8 * G, nrt, NR);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / per_img);
    const int64_t r = i - (int64_t)b * per_img;
    const int rt = (int)(r / ((int64_t)NR * G));
    const int64_t r2 = r - (int64_t)rt * NR * G;
    const int cg = (int)(r2 / NR), n = (int)(r2 - (int64_t)cg * NR);
    const int ye = rt * NR + n;
    float f[8];
    const int xe = 8 * (cg - pg);   // first image column of this group (reflect: may be outside)
    if (ye < hx && pr + pg > 0 && (xe < 0 || xe + 8 > s.W || ye < pr || ye >= s.H + pr)) {
      // mirrored margins, pixel by pixel (the same stretch as below)
      const ImgPar ip = par[b];
      const int y = ye - pr < 0 ? pr - ye - 1 : (ye - pr >= s.H ? 2 * s.H - 1 - (ye - pr) : ye - pr);
      const uint8_t* row = images + ((int64_t)b * s.H + y) * s.pitch;
      const float lo = BPP == 4 ? __int_as_float(ip.lo) : (float)ip.lo, inv = ip.inv;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int x0 = xe + k, x = x0 < 0 ? -x0 - 1 : (x0 >= s.W ? 2 * s.W - 1 - x0 : x0);
        float q;
        if (BPP == 4) q = __ldg(reinterpret_cast<const float*>(row) + x);
        else if (BPP == 2) q = (float)__ldg(reinterpret_cast<const uint16_t*>(row) + x);
        else q = (float)__ldg(row + x);
        f[k] = kT2XScale * (fminf(fmaxf((q - lo) * inv, 0.f), 1.f) - 0.5f);
      }
    } else if (ye < hx) {
      const int y = ye - pr;
      const ImgPar ip = par[b];
      const uint8_t* row = images + ((int64_t)b * s.H + y) * s.pitch;
      const int cgi = cg - pg;   // the group's index in the image row
      if (BPP == 4) {
        const float lo = __int_as_float(ip.lo), inv = ip.inv;
        const float4 a = __ldg(reinterpret_cast<const float4*>(row) + 2 * cgi);
        const float4 c = __ldg(reinterpret_cast<const float4*>(row) + 2 * cgi + 1);
        const float q[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = kT2XScale * (fminf(fmaxf((q[k] - lo) * inv, 0.f), 1.f) - 0.5f);
      } else {
        const float lo = (float)ip.lo, inv = ip.inv;
        uint32_t p[8];
        if (BPP == 2) {
          const uint4 q = __ldg(reinterpret_cast<const uint4*>(row) + cgi);
          const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int k = 0; k < 8; ++k) p[k] = (w4[k >> 1] >> (16 * (k & 1))) & 0xffffu;
        } else {
          const uint2 q = __ldg(reinterpret_cast<const uint2*>(row) + cgi);
          const uint32_t w2[2] = {q.x, q.y};
#pragma unroll
          for (int k = 0; k < 8; ++k) p[k] = (w2[k >> 2] >> (8 * (k & 3))) & 0xffu;
        }
        // the CUDA-core schedules' stretch (k_normalize), scaled by 2^10 (exact)
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = kT2XScale * (fminf(fmaxf(((float)p[k] - lo) * inv, 0.f), 1.f) - 0.5f);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = 0.f;
    }
    uint4 hi, lo;
    t2_split8(f, hi, lo);
    const size_t off = ((size_t)rt * G + cg) * NR * 16 + (size_t)n * 16;
    uint8_t* base = xt + (size_t)b * 2 * pb;
    *reinterpret_cast<uint4*>(base + off) = hi;
    *reinterpret_cast<uint4*>(base + pb + off) = lo;
  }
}

// ---------------------------------------------------------------------------------
// k_tc2_rows.  Barriers: 0/1 d1 full (commit), 2/3 d1 empty (16 warps), 4/5 table full
// (tx), 6/7 table free (commit), 8 X full (tx), 9 X free (commit).
__global__ void __launch_bounds__(kT2Threads, 1)
k_tc2_rows(const uint8_t* __restrict__ xt, const __grid_constant__ Tc2Plan P, const uint8_t* __restrict__ tabs,
           uint8_t* __restrict__ rx, int W, int H, int batch, int nrt, int rt_first, int rt_count, int pg = 0) {
  // H: rows of Rx (reflect: the image's plus the mirrored margins); pg: the staged X's
  // mirrored margin groups on either side (reflect), so windows never wrap
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int NR = P.NR, S = P.S, nlev = P.nlev;
  const size_t xplane = (size_t)(S / 8) * NR * 16;
  uint8_t* xs = smem_raw;                       // 2 planes of the staged window [cg][row][8]
  uint8_t* tbuf = xs + 2 * xplane;              // 2 x max_lev_bytes1
  uint64_t* bars = reinterpret_cast<uint64_t*>(tbuf + 2 * (size_t)P.max_lev_bytes1);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 10);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;   // warp-uniform roles
  const int ntx = W / kT2Cols;
  const int ntiles = ntx * rt_count * batch;   // row tiles [rt_first, rt_first + rt_count) (band mode: a subset)
  const int t0 = blockIdx.x;
  if (t0 >= ntiles) return;
  const int my_tiles = (ntiles - 1 - t0) / gridDim.x + 1;
  const int G = my_tiles * nlev;

  if (tid == kT2Epi) {
    for (int k = 0; k < 10; ++k) mbar_init(&bars[k], (k == 2 || k == 3) ? 16 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc(tslot, 512);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;
  auto tile_of = [&](int k, int& b, int& x0, int& rt) {   // k-th tile of this CTA
    int t = t0 + k * (int)gridDim.x;
    const int xti = t % ntx;
    t /= ntx;
    rt = rt_first + t % rt_count;
    b = t / rt_count;
    x0 = xti * kT2Cols;
  };

  if (warp == kT2Epi / 32) {
    // ================= MMA issuer (whole warp, elected lane issues; umma::*_w) =================
    {
      const uint32_t idesc = umma::idesc_f16(128, NR);
      for (int g = 0; g < G; ++g) {
        const int lev = g % nlev;
        const Tc2Level& L = P.lev[lev];
        if (lev == 0) mbar_wait(&bars[8], (uint32_t)((g / nlev) & 1));
        mbar_wait(&bars[4 + (g & 1)], (uint32_t)((g >> 1) & 1));
        if (g >= 2) mbar_wait(&bars[2 + (g & 1)], (uint32_t)(((g >> 1) - 1) & 1));
        umma::fence_after();
        const int E1 = L.K / 8 - 2;
        const uint32_t thi = umma::smem_addr(tbuf + (size_t)(g & 1) * P.max_lev_bytes1);
        const uint32_t tlo = thi + L.npairs * 256;
        const uint64_t dH = umma::desc_kmajor(thi + E1 * 256, 128, 256);
        const uint64_t dL = umma::desc_kmajor(tlo + E1 * 256, 128, 256);
        const uint32_t xb = umma::smem_addr(xs) + (uint32_t)(L.c0 / 8) * NR * 16;
        const uint64_t dXh = umma::desc_kmajor(xb, NR * 16, 128);
        const uint64_t dXl = umma::desc_kmajor(xb + (uint32_t)xplane, NR * 16, 128);
        const uint32_t d1 = tmem + (uint32_t)((g & 1) * NR);
        const uint32_t stepx = 2u * NR;   // two column groups per K-step, in 16-byte units
        for (int j = 0; j < L.K / 16; ++j) {
          umma::mma_ss_w(d1, dH - 32u * j, dXh + stepx * j, idesc, j > 0);
          umma::mma_ss_w(d1, dL - 32u * j, dXh + stepx * j, idesc, 1);
          umma::mma_ss_w(d1, dH - 32u * j, dXl + stepx * j, idesc, 1);
        }
        umma::commit_w(&bars[g & 1]);
        umma::commit_w(&bars[6 + (g & 1)]);
        if (lev == nlev - 1) umma::commit_w(&bars[9]);
      }
    }
    __syncwarp();
  } else if (warp == kT2Epi / 32 + 1) {
    // ================= copy producer =================
    if (lane == 0) {
      for (int g = 0; g < G; ++g) {
        const int lev = g % nlev;
        if (g >= 2) mbar_wait(&bars[6 + (g & 1)], (uint32_t)(((g >> 1) - 1) & 1));
        const uint32_t tb = 2u * P.lev[lev].npairs * 256;
        mbar_arrive_expect_tx(&bars[4 + (g & 1)], tb);
        bulk_g2s(tbuf + (size_t)(g & 1) * P.max_lev_bytes1, tabs + P.lev[lev].tab_off, tb, &bars[4 + (g & 1)]);
        if (lev == 0) {
          int b, x0, rt;
          tile_of(g / nlev, b, x0, rt);
          if (g > 0) mbar_wait(&bars[9], (uint32_t)(((g / nlev) - 1) & 1));
          mbar_arrive_expect_tx(&bars[8], (uint32_t)(2 * xplane));
          const int Gc = W / 8 + 2 * pg, SG = S / 8;
          int g0 = (x0 - P.H0) / 8 + pg;
          if (g0 < 0) g0 += Gc;
          const size_t pb = t2_x_plane_bytes(8 * Gc, nrt, NR);
          for (int p = 0; p < 2; ++p) {
            const uint8_t* src = xt + ((size_t)b * 2 + p) * pb + (size_t)rt * Gc * NR * 16;
            uint8_t* dst = xs + (size_t)p * xplane;
            const int n1 = g0 + SG <= Gc ? SG : Gc - g0;
            bulk_g2s(dst, src + (size_t)g0 * NR * 16, (uint32_t)(n1 * NR * 16), &bars[8]);
            if (n1 < SG) bulk_g2s(dst + (size_t)n1 * NR * 16, src, (uint32_t)((SG - n1) * NR * 16), &bars[8]);
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue: D1 -> fp16 hi/lo transposed slabs =================
    const int q = warp & 3, rg = warp >> 2;
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
    const int c = 32 * q + lane;
    const size_t rxp = t2_rx_plane_bytes(W, H);
    for (int g = 0; g < G; ++g) {
      const int lev = g % nlev;
      int b, x0, rt;
      tile_of(g / nlev, b, x0, rt);
      mbar_wait(&bars[g & 1], (uint32_t)((g >> 1) & 1));
      umma::fence_after();
      const uint32_t d1 = tq + (uint32_t)((g & 1) * NR);
      uint8_t* base = rx + ((size_t)b * nlev + lev) * 2 * rxp + (size_t)(x0 / kT2Cols) * (H / 16) * kT2SlabBytes +
                      (size_t)c * 16;
      for (int k = rg; k < NR / 8; k += 4) {
        const int y = rt * NR + 8 * k;
        if (y >= H) break;   // warp-uniform (NR and H are multiples of 16)
        uint32_t r[8];
        umma::ld8(d1 + 8 * k, r);
        umma::wait_ld();
        float f[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(r[u]) * (1.f / kTcWScale);
        uint4 hi, lo;
        t2_split8(f, hi, lo);
        const size_t off = (size_t)(y / 16) * kT2SlabBytes + (size_t)((y / 8) & 1) * (kT2SlabBytes / 2);
        *reinterpret_cast<uint4*>(base + off) = hi;
        *reinterpret_cast<uint4*>(base + rxp + off) = lo;
      }
      umma::fence_before();
      __syncwarp();
      if (lane == 0) t2_arrive(&bars[2 + (g & 1)]);
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------------
// k_tc2_cols.  Barriers: 0/1 d2 full (commit), 2/3 d2 empty (16 warps), 4/5 table full
// (tx), 6/7 table free (commit), 8.. stage full (tx), 8+kT2Stages.. stage empty (commit).
// 18 warps: at most 5 per SM sub-partition, so 96 registers; each epilogue thread keeps
// 56 running maxima and 56 packed argmax bytes (N = 224 rows; 256 would spill)
//
// LOG (reading R23, response = t_j^2 (d_xx + d_yy) L(., t_j)): the plan's levels are 2n
// sub-levels, 2j with row taps w_j and column taps t_j^2 w2_j, 2j+1 with row taps
// t_j^2 w2_j and column taps w_j, so  t_j^2 (w2 (x) w + w (x) w2) x  is the sum of the two
// sub-levels' column products: both accumulate into one TMEM accumulator (j), and the
// epilogue takes the response from it directly (scaled and signed by lev[2j].tdog).
// The row pass and the slab / table producer are the DoG ones, level for sub-level.
template <bool DOG, bool LOG = false, bool REFL = false>
__global__ void __launch_bounds__(kT2Threads, 1)
k_tc2_cols(const uint8_t* __restrict__ rx, const ImgPar* __restrict__ par, const __grid_constant__ Tc2Plan P,
           const uint8_t* __restrict__ tabs, float* __restrict__ v_out, uint8_t* __restrict__ idx_out,
           float* __restrict__ dog_out, int W, int H, int batch, int yt_first, int yt_count, int hx, int pr) {
  // REFL (reflect, reading R25): Rx has hx rows, image row 0 at Rx row pr (mirrored
  // margins), and windows never wrap; periodic instantiations ignore hx / pr (a separate
  // instantiation keeps their code as it was)
  if (!REFL) hx = H, pr = 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int nlev = P.nlev;
  uint8_t* ring = smem_raw;                                        // kT2Stages x (hi 4 KB | lo 4 KB)
  uint8_t* tbuf = ring + (size_t)kT2Stages * 2 * kT2SlabBytes;     // 2 x max_lev_bytes2
  uint64_t* bars = reinterpret_cast<uint64_t*>(tbuf + 2 * (size_t)P.max_lev_bytes2);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * kT2Stages);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;   // warp-uniform roles
  const int ntx = W / kT2Cols, nty = yt_count;   // output row tiles [yt_first, yt_first + yt_count)
  const int ntiles = ntx * nty * batch;
  const int t0 = blockIdx.x;
  if (t0 >= ntiles) return;
  const int my_tiles = (ntiles - 1 - t0) / gridDim.x + 1;
  const int G = my_tiles * nlev;
  const size_t rxp = t2_rx_plane_bytes(W, hx);

  if (tid == kT2Epi) {
    for (int k = 0; k < 8 + 2 * kT2Stages; ++k) mbar_init(&bars[k], (k == 2 || k == 3) ? 16 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc(tslot, 512);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;
  auto tile_of = [&](int k, int& b, int& x0, int& y0) {
    int t = t0 + k * (int)gridDim.x;
    const int xti = t % ntx;
    t /= ntx;
    y0 = (yt_first + t % nty) * kT2ColRows;
    b = t / nty;
    x0 = xti * kT2Cols;
  };

  if (warp == kT2Epi / 32) {
    // ================= MMA issuer (whole warp, elected lane issues; umma::*_w) =================
    {
      const uint32_t idesc = umma::idesc_f16(128, kT2ColRows);
      const uint32_t ring0 = umma::smem_addr(ring);
      uint32_t cnt = 0;
      for (int g = 0; g < G; ++g) {
        const int lev = g % nlev;
        const int K2 = P.lev[lev].K2, np2 = P.lev[lev].npairs2;
        const int ga = LOG ? (g >> 1) : g;            // accumulator index (LOG: two sub-levels each)
        const bool first = !LOG || (lev & 1) == 0;    // first product into this accumulator
        mbar_wait(&bars[4 + (g & 1)], (uint32_t)((g >> 1) & 1));
        if (first && ga >= 2) mbar_wait(&bars[2 + (ga & 1)], (uint32_t)(((ga >> 1) - 1) & 1));
        umma::fence_after();
        const int E1 = K2 / 8 - 2;
        const uint32_t thi = umma::smem_addr(tbuf + (size_t)(g & 1) * P.max_lev_bytes2);
        const uint64_t dH = umma::desc_kmajor(thi + E1 * 256, 128, 256);
        const uint64_t dL = umma::desc_kmajor(thi + np2 * 256 + E1 * 256, 128, 256);
        const uint32_t d2 = tmem + (uint32_t)(kT2ColRows * (ga & 1));
        for (int j = 0; j < K2 / 16; ++j, ++cnt) {
          const uint32_t st = cnt % kT2Stages;
          mbar_wait(&bars[8 + st], (cnt / kT2Stages) & 1u);
          umma::fence_after();
          const uint64_t aH = umma::desc_kmajor(ring0 + st * 2 * kT2SlabBytes, kT2SlabBytes / 2, 128);
          const uint64_t aL = umma::desc_kmajor(ring0 + st * 2 * kT2SlabBytes + kT2SlabBytes, kT2SlabBytes / 2, 128);
          umma::mma_ss_w(d2, aH, dH - 32u * j, idesc, j > 0 || !first);
          umma::mma_ss_w(d2, aH, dL - 32u * j, idesc, 1);
          umma::mma_ss_w(d2, aL, dH - 32u * j, idesc, 1);
          umma::commit_w(&bars[8 + kT2Stages + st]);
        }
        if (!first || !LOG) umma::commit_w(&bars[ga & 1]);
        umma::commit_w(&bars[6 + (g & 1)]);
      }
    }
    __syncwarp();
  } else if (warp == kT2Epi / 32 + 1) {
    // ================= slab / table producer =================
    if (lane == 0) {
      uint32_t cnt = 0;
      for (int g = 0; g < G; ++g) {
        const int lev = g % nlev;
        const Tc2Level& L = P.lev[lev];
        if (g >= 2) mbar_wait(&bars[6 + (g & 1)], (uint32_t)(((g >> 1) - 1) & 1));
        const uint32_t tb = 2u * L.npairs2 * 256;
        mbar_arrive_expect_tx(&bars[4 + (g & 1)], tb);
        bulk_g2s(tbuf + (size_t)(g & 1) * P.max_lev_bytes2, tabs + L.tab_off2, tb, &bars[4 + (g & 1)]);
        int b, x0, y0;
        tile_of(g / nlev, b, x0, y0);
        const uint8_t* src = rx + ((size_t)b * nlev + lev) * 2 * rxp + (size_t)(x0 / kT2Cols) * (hx / 16) * kT2SlabBytes;
        int ws = y0 - L.R - L.s2 + pr;   // slab-aligned first window row (periodic: wraps)
        while (ws < 0) ws += hx;
        for (int j = 0; j < L.K2 / 16; ++j, ++cnt) {
          const uint32_t st = cnt % kT2Stages;
          if (cnt >= (uint32_t)kT2Stages) mbar_wait(&bars[8 + kT2Stages + st], ((cnt / kT2Stages) - 1) & 1u);
          int row = ws + 16 * j;
          if (REFL) row = min(row, hx - 16);   // rows past the margin feed only outputs y >= H
          while (row >= hx) row -= hx;
          const uint8_t* s0 = src + (size_t)(row / 16) * kT2SlabBytes;
          uint8_t* dst = ring + (size_t)st * 2 * kT2SlabBytes;
          mbar_arrive_expect_tx(&bars[8 + st], 2 * kT2SlabBytes);
          bulk_g2s(dst, s0, kT2SlabBytes, &bars[8 + st]);
          bulk_g2s(dst + kT2SlabBytes, s0 + rxp, kT2SlabBytes, &bars[8 + st]);
        }
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue: DoG, running max, first argmax =================
    constexpr int RPW = kT2ColRows / 4;       // rows per epilogue thread
    const int q = warp & 3, wg = warp >> 2;   // lanes 32q.., rows RPW wg ..
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
    const int c = 32 * q + lane;
    const int64_t plane = (int64_t)H * W;
    float vbest[RPW];
    uint32_t ibest[RPW / 4];
    int odeg = 0;
    if (LOG) {   // one accumulator per plane j: the response itself
      const int n = nlev / 2;
      for (int ga = 0; ga < G / 2; ++ga) {
        const int jp = ga % n;
        int b, x0, y0;
        tile_of(ga / n, b, x0, y0);
        mbar_wait(&bars[ga & 1], (uint32_t)((ga >> 1) & 1));
        umma::fence_after();
        if (jp == 0) {
          odeg = par[b].degen;
#pragma unroll
          for (int u = 0; u < RPW; ++u) vbest[u] = -INFINITY;
#pragma unroll
          for (int u = 0; u < RPW / 4; ++u) ibest[u] = 0u;
        }
        const float tf = P.lev[2 * jp].tdog * (1.f / (kTcWScale * kT2XScale));
        const uint32_t cur = tq + kT2ColRows * (ga & 1) + RPW * wg;
#pragma unroll
        for (int qq = 0; qq < RPW / 8; ++qq) {
          uint32_t a8[8];
          umma::ld8(cur + 8 * qq, a8);
          umma::wait_ld();
#pragma unroll
          for (int uu = 0; uu < 8; ++uu) {
            const int u = 8 * qq + uu;
            const float D = tf * __uint_as_float(a8[uu]);
            if (DOG) {
              const int y = y0 + RPW * wg + u;
              if (y < H) dog_out[((int64_t)b * n + jp) * plane + (int64_t)y * W + x0 + c] = odeg ? 0.f : D;
            }
            if (D > vbest[u]) {
              vbest[u] = D;
              const int sh = (u & 3) * 8;
              ibest[u >> 2] = (ibest[u >> 2] & ~(0xffu << sh)) | ((uint32_t)jp << sh);
            }
          }
        }
        umma::fence_before();
        __syncwarp();
        if (lane == 0) t2_arrive(&bars[2 + (ga & 1)]);
        if (jp == n - 1 && v_out) {
#pragma unroll
          for (int u = 0; u < RPW; ++u) {
            const int y = y0 + RPW * wg + u;
            if (y < H) {
              const int64_t pidx = (int64_t)b * plane + (int64_t)y * W + x0 + c;
              v_out[pidx] = odeg ? 0.f : vbest[u];
              idx_out[pidx] = odeg ? (uint8_t)0 : (uint8_t)((ibest[u >> 2] >> ((u & 3) * 8)) & 0xffu);
            }
          }
        }
      }
    }
    for (int g = 0; g < (LOG ? 0 : G); ++g) {
      const int lev = g % nlev;
      int b, x0, y0;
      tile_of(g / nlev, b, x0, y0);
      mbar_wait(&bars[g & 1], (uint32_t)((g >> 1) & 1));
      umma::fence_after();
      if (lev == 0) {
        odeg = par[b].degen;
#pragma unroll
        for (int u = 0; u < RPW; ++u) vbest[u] = -INFINITY;
#pragma unroll
        for (int u = 0; u < RPW / 4; ++u) ibest[u] = 0u;
      } else {
        // D_{lev-1} = t_{lev-1} (L_lev - L_{lev-1}); both accumulators carry 2^22 L
        const float tf = P.lev[lev - 1].tdog * (1.f / (kTcWScale * kT2XScale));
        const uint32_t cur = tq + kT2ColRows * (g & 1) + RPW * wg, prv = tq + kT2ColRows * ((g - 1) & 1) + RPW * wg;
#pragma unroll
        for (int qq = 0; qq < RPW / 4; ++qq) {   // 4 rows at a time (register budget)
          uint32_t a[4], bb[4];
          umma::ld4(cur + 4 * qq, a);
          umma::ld4(prv + 4 * qq, bb);
          umma::wait_ld();
#pragma unroll
          for (int uu = 0; uu < 4; ++uu) {
            const int u = 4 * qq + uu;
            const float D = tf * (__uint_as_float(a[uu]) - __uint_as_float(bb[uu]));
            if (DOG) {
              const int y = y0 + RPW * wg + u;
              if (y < H)
                dog_out[((int64_t)b * (nlev - 1) + (lev - 1)) * plane + (int64_t)y * W + x0 + c] = odeg ? 0.f : D;
            }
            if (D > vbest[u]) {
              vbest[u] = D;
              const int sh = (u & 3) * 8;
              ibest[u >> 2] = (ibest[u >> 2] & ~(0xffu << sh)) | ((uint32_t)(lev - 1) << sh);
            }
          }
        }
        umma::fence_before();
        __syncwarp();
        if (lane == 0) t2_arrive(&bars[2 + ((g - 1) & 1)]);   // L_{lev-1} no longer needed
      }
      if (lev == nlev - 1) {
        if (v_out) {
#pragma unroll
          for (int u = 0; u < RPW; ++u) {
            const int y = y0 + RPW * wg + u;
            if (y < H) {
              const int64_t pidx = (int64_t)b * plane + (int64_t)y * W + x0 + c;
              v_out[pidx] = odeg ? 0.f : vbest[u];
              idx_out[pidx] = odeg ? (uint8_t)0 : (uint8_t)((ibest[u >> 2] >> ((u & 3) * 8)) & 0xffu);
            }
          }
        }
        umma::fence_before();
        __syncwarp();
        if (lane == 0) t2_arrive(&bars[2 + (g & 1)]);
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 512);
}

}  // namespace mhfd
