// k_twopass.cuh — large-radius schedule (hot-path rows a2-a6) for the generic path:
// the separable blur of each level as two kernels with an HBM intermediate, so neither
// pass recomputes a halo (the fused band kernel recomputes (BH + 2R)/BH row-pass rows per
// output: 1.8x at R = 150 even with 384-row bands).  Same mathematics and the same f32
// tap-pair FFMA2 sums as k_scale_space (PAPER.md:134-141 blur, :171 Eq. 2, :240-244
// argmax; periodic boundary), so results match it bit for bit.
//
//   k_rows2 (level i): Rx_i = row blur of the centred image; CTA = 32 rows x 256 output
//            columns, the 32 x (256 + 2R + p) input window staged by bulk copies (wrap at
//            the image edge), conv4_row with lane = row, 16-byte stores per lane (no
//            transpose buffer: three CTAs per SM).
//   k_cols_all (all levels): CTA = 32 columns x 256 rows; per level the (256 + 2R + p)
//            x 32 window of Rx_i in shared memory, conv8_col with lane = column, DoG
//            against L_{i-1} and the running max / first argmax in registers across the
//            levels (one write of v / argmax per pixel at the end).
// HBM per level and pixel: 4 (Rx write) + ~4-9 (Rx window reads, halo through L2) bytes.
#pragma once
#include "common.cuh"
#include "k_scale_space.cuh"
#include "k_band.cuh"

namespace mhfd {

constexpr int kR2Cols = 256;   // k_rows2 output columns per CTA
constexpr int kC2Rows = 256;   // k_cols_all output rows per CTA

__host__ __device__ inline int rows2_pitch(int R, int p) {   // 4 x odd floats, >= window + overrun
  int q = (kR2Cols + 2 * R + p + 16 + 3) / 4;
  if ((q & 1) == 0) ++q;
  return 4 * q;
}
__host__ __device__ inline size_t rows2_smem(int rmax) {
  return sizeof(float) * ((size_t)32 * rows2_pitch(rmax, 3)) + 16;
}
__host__ __device__ inline int cols2_rows(int R, int p) { return kC2Rows + 2 * R + p + 19; }
__host__ __device__ inline size_t cols2_smem(int rmax) {
  return sizeof(float) * (size_t)cols2_rows(rmax, 3) * kHP + 16;
}

__global__ void __launch_bounds__(256) k_rows2(const float* __restrict__ fimg, int W, int H,
                                               const __grid_constant__ LevelTable tab, int lev,
                                               float* __restrict__ rx) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int R = tab.R[lev], p = tab.pre[lev], ntap = tab.ntap[lev];
  const int SP = rows2_pitch(R, p);
  float* in = reinterpret_cast<float*>(smem_raw);              // 32 x SP
  uint64_t* bar = reinterpret_cast<uint64_t*>(in + 32 * SP);
  const int b = blockIdx.z, y0 = blockIdx.y * 32, x0 = blockIdx.x * kR2Cols;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float* img = fimg + (int64_t)b * H * W;
  const int xs = x0 - R - p;                                   // first staged column (multiple of 4)
  const int ncol = (kR2Cols + 2 * R + p + 3) & ~3;
  const int nrow = min(32, H - y0);
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {   // one bulk copy per row (two where it wraps), completing on bar
    if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(nrow * ncol * 4));
    __syncwarp();
    if (lane < nrow) {
      const float* row = img + (int64_t)(y0 + lane) * W;
      float* dst = in + lane * SP;
      const int xw = wrap_idx(xs, W);
      if (xw + ncol > W) {
        bulk_g2s(dst, row + xw, (uint32_t)((W - xw) * 4), bar);
        bulk_g2s(dst + (W - xw), row, (uint32_t)((xw + ncol - W) * 4), bar);
      } else {
        bulk_g2s(dst, row + xw, (uint32_t)(ncol * 4), bar);
      }
    }
  }
  // the window overrun past ncol meets zero taps; keep it finite
  for (int i = tid; i < 32 * (SP - ncol); i += 256) in[(i / (SP - ncol)) * SP + ncol + i % (SP - ncol)] = 0.f;
  const float* wA = tab.w + tab.woff[lev];
  __shared__ __align__(16) float wsA[kMaxTaps / 4], wsB[kMaxTaps / 4];   // this level's taps (<= 4 x 256 + pad)
  for (int i = tid; i < ntap + 8; i += 256) {
    wsA[i] = wA[i];
    wsB[i] = i ? wA[i - 1] : 0.f;
  }
  mbar_wait(bar, 0);
  __syncthreads();
  // lane = row; warp w covers output columns 32 k + 4 w .. +4 for k = 0..7 (16-byte stores)
  float* orow = rx + ((int64_t)b * H + y0 + lane) * W + x0;
  for (int k = 0; k < kR2Cols / 32; ++k) {
    const int c = 32 * k + 4 * warp;
    float acc[4];
    conv4_row(acc, in + lane * SP + c, wsA, wsB, ntap);
    if (lane < nrow) *reinterpret_cast<float4*>(orow + c) = make_float4(acc[0], acc[1], acc[2], acc[3]);
  }
}

// Column pass over ALL levels of one 32-column x 256-row tile (instead of per-level column
// launches): Rx of every level is in HBM (rx_all, level-major), each level's window is
// staged into shared memory, L_{i-1}, the running max and the first argmax stay in
// registers for the whole tile, so the only per-level HBM traffic is the Rx window.
__global__ void __launch_bounds__(256, 2) k_cols_all(const float* __restrict__ rx_all, int W, int H, int B,
                                                     const __grid_constant__ LevelTable tab,
                                                     float* __restrict__ v, uint8_t* __restrict__ idx,
                                                     float* __restrict__ dog, const ImgPar* __restrict__ par) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* hb = reinterpret_cast<float*>(smem_raw);              // cols2_rows(rmax) x kHP
  __shared__ __align__(16) float wsA[kMaxTaps / 4], wsB[kMaxTaps / 4];
  const int b = blockIdx.z, Y0 = blockIdx.y * kC2Rows, x0 = blockIdx.x * kStripW;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t plane = (int64_t)H * W;
  const int x = x0 + lane;
  const bool inx = x < W;
  const bool degen = par[b].degen != 0;
  float lprev[32], vbest[32];
  uint32_t ibest[8];
#pragma unroll
  for (int u = 0; u < 32; ++u) { lprev[u] = 0.f; vbest[u] = -INFINITY; }
#pragma unroll
  for (int u = 0; u < 8; ++u) ibest[u] = 0u;
  for (int lev = 0; lev < tab.nlev; ++lev) {
    const int R = tab.R[lev], p = tab.pre[lev], ntap = tab.ntap[lev];
    const float* src = rx_all + ((int64_t)lev * B + b) * plane;
    const int nr = kC2Rows + 2 * R + p + 16;
    __syncthreads();   // the previous level's hb / taps are no longer read
    {
      int y = wrap_idx(Y0 - R - p + warp, H);
      for (int r = warp; r < cols2_rows(R, p); r += 8) {
        hb[r * kHP + lane] = (r < nr && inx) ? __ldg(src + (int64_t)y * W + x) : 0.f;
        y += 8;
        if (y >= H) y -= H;
      }
    }
    const float* wA = tab.w + tab.woff[lev];
    for (int i = tid; i < ntap + 8; i += 256) {
      wsA[i] = wA[i];
      wsB[i] = i ? wA[i - 1] : 0.f;
    }
    __syncthreads();
    const float tdog = lev > 0 ? tab.tdog[lev - 1] : 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int rb = warp * 32 + q * 8;
      float acc[8];
      conv8_col(acc, hb + rb * kHP + lane, kHP, wsA, wsB, ntap);
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        const int u = q * 8 + o;
        const float L = acc[o];
        if (lev > 0) {
          const float D = degen ? 0.f : tdog * (L - lprev[u]);
          if (dog) {
            const int y = Y0 + rb + o;
            if (inx && y < H) dog[((int64_t)b * (tab.nlev - 1) + (lev - 1)) * plane + (int64_t)y * W + x] = D;
          }
          if (D > vbest[u]) {
            vbest[u] = D;
            const int sh = (u & 3) * 8;
            ibest[u >> 2] = (ibest[u >> 2] & ~(0xffu << sh)) | ((uint32_t)(lev - 1) << sh);
          }
        }
        lprev[u] = L;
      }
    }
  }
  if (v) {
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int y = Y0 + warp * 32 + u;
      if (inx && y < H) {
        const int64_t pi = (int64_t)b * plane + (int64_t)y * W + x;
        v[pi] = degen ? 0.f : vbest[u];
        idx[pi] = degen ? (uint8_t)0 : (uint8_t)((ibest[u >> 2] >> ((u & 3) * 8)) & 0xffu);
      }
    }
  }
}

// Column pass over all levels, paper mode (no DoG planes): the same tile and the same
// register-resident L_{i-1} / max / first argmax as k_cols_all, but the conv is the u8
// band kernel's col_pass (8 rows x 2 columns per thread, float2 loads, column-pair FFMA2
// with a broadcast tap: 4 FFMA2 per shared load where conv8_col issues 2, which left
// conv8_col load-issue bound at ~31 % FMA activity), and the next level's Rx window is
// prefetched with cp.async into a second buffer while the current level convolves.
// Same taps, f32, summed in tap order d = -R..R in one accumulator per pixel (conv8_col
// sums two interleaved partial sums), so results agree with k_cols_all to rounding, not
// bit for bit; the DoG-dump path keeps k_cols_all.
constexpr int kC3Threads = 512;
__host__ __device__ inline int c3_taps(int R) { return ((2 * R + 1 + 15) & ~15) + 16; }   // zero-padded
__host__ __device__ inline int c3_rows(int R) { return kC2Rows + ((2 * R + 1 + 15) & ~15) + 24; }
__host__ __device__ inline int c3_buf_floats(int rmax) { return c3_rows(rmax) * kBandHP + c3_taps(rmax); }
__host__ __device__ inline size_t c3_smem(int rmax) { return sizeof(float) * 2 * (size_t)c3_buf_floats(rmax) + 16; }

// blur boundary index: periodic (reading R7) or half-sample symmetric reflection (R25);
// |a| < 2m (one reflection: R_max < W, H)
__device__ __forceinline__ int bidx(int a, int m, int reflect) {
  if (reflect) return a < 0 ? -a - 1 : (a >= m ? 2 * m - 1 - a : a);
  a %= m;
  return a < 0 ? a + m : a;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

// LOG (reading R23): tab holds 2n sub-levels, Rx of sub-level 2i = w_i along x and of
// 2i + 1 = w2_i along x; the column taps of sub-level s are the row taps of s ^ 1, so
// sub-level 2i gives d_yy L_i and 2i + 1 gives d_xx L_i, and plane i's response is
// tdog[2i] (= +-t_i^2) x their sum; optional `dog` receives the n planes.
template <bool LOG>
__global__ void __launch_bounds__(kC3Threads, 1) k_cols_pair(const float* __restrict__ rx_all, int W, int H, int B,
                                                             const __grid_constant__ LevelTable tab,
                                                             float* __restrict__ v, uint8_t* __restrict__ idx,
                                                             float* __restrict__ dog,
                                                             const ImgPar* __restrict__ par, int reflect,
                                                             int ty0, int need_lo, int need_hi) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* buf0 = reinterpret_cast<float*>(smem_raw);
  const int bufsz = c3_buf_floats(tab.rmax);
  // ty0: first 256-row output tile (single-image bands compute a sub-range of tiles)
  const int b = blockIdx.z, Y0 = (blockIdx.y + ty0) * kC2Rows, x0 = blockIdx.x * kStripW;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t plane = (int64_t)H * W;
  // stage level `lev` into buffer `k`: rows Y0 - R .. (c3_rows), wrapped; taps 0..2R
  auto stage = [&](int lev, int k) {
    float* hb = buf0 + k * bufsz;
    float* wc = hb + c3_rows(tab.rmax) * kBandHP;
    const int R = tab.R[lev];
    const float* src = rx_all + ((int64_t)lev * B + b) * plane + x0;
    const int nr = c3_rows(R);
    for (int i = tid; i < nr * 8; i += kC3Threads) {
      const int r = i >> 3, c = i & 7;
      const int y = bidx(Y0 - R + r, H, reflect);
      cp_async16(hb + r * kBandHP + 4 * c, src + (int64_t)y * W + 4 * c);
    }
    const int cl = LOG ? (lev ^ 1) : lev;   // the level whose taps run along y
    const float* w = tab.w + tab.woff[cl] + tab.pre[cl];
    for (int i = tid; i < c3_taps(R); i += kC3Threads) wc[i] = i < 2 * R + 1 ? w[i] : 0.f;
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int cp = lane & 15;
  const int rg = 2 * warp + (lane >> 4);
  float lprev[16], vbest[16], part[16];
  uint32_t ibest[4];
#pragma unroll
  for (int k = 0; k < 16; ++k) { lprev[k] = 0.f; vbest[k] = -INFINITY; part[k] = 0.f; }
#pragma unroll
  for (int k = 0; k < 4; ++k) ibest[k] = 0u;
  const bool degen = par[b].degen != 0;
  // single-image bands: rows outside [need_lo, need_hi) need no response (whole 8-row
  // groups skip the column convolution)
  const bool active = Y0 + 8 * rg < need_hi && Y0 + 8 * rg + 8 > need_lo;
  stage(0, 0);
  for (int lev = 0; lev < tab.nlev; ++lev) {
    if (lev + 1 < tab.nlev) {
      stage(lev + 1, (lev + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();   // level lev's window and taps are in
    const float* hb = buf0 + (lev & 1) * bufsz;
    const float* wc = hb + c3_rows(tab.rmax) * kBandHP;
    // threads whose 8 rows are outside [need_lo, need_hi) only stage and take the barriers
    // (both __syncthreads stay outside the branch: the groups of one warp can differ)
    if (active) {
    // lev = 0: col_pass only returns the 16 column sums (in Lc)
    float Lc[16];
    col_pass<kBandHP>(hb + 8 * rg * kBandHP + 2 * cp, wc, 2 * tab.R[lev] + 1, 0, 0.f, Lc, vbest, ibest);
    // plane i gets its response now: DoG plane lev - 1 = tdog (L_lev - L_{lev-1}) (Eq. 2),
    // LoG plane lev / 2 = tdog (d_yy + d_xx) at odd sub-levels (reading R23)
    const bool emit = LOG ? (lev & 1) != 0 : lev > 0;
    if (emit) {
      const int i = LOG ? lev >> 1 : lev - 1;
      const float tf = LOG ? tab.tdog[lev] : tab.tdog[lev - 1];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float D = degen ? 0.f : (LOG ? tf * (part[k] + Lc[k]) : tf * (Lc[k] - part[k]));
        if (D > vbest[k]) {
          vbest[k] = D;
          const int sh = (k & 3) * 8;
          ibest[k >> 2] = (ibest[k >> 2] & ~(0xffu << sh)) | ((uint32_t)i << sh);
        }
        lprev[k] = D;
      }
      if (dog) {
        const int nplanes = LOG ? tab.nlev / 2 : tab.nlev - 1;
#pragma unroll
        for (int o = 0; o < 8; ++o) {
          const int y = Y0 + 8 * rg + o;
          if (y < H)
            *reinterpret_cast<float2*>(dog + ((int64_t)b * nplanes + i) * plane + (int64_t)y * W + x0 + 2 * cp) =
                make_float2(lprev[2 * o], lprev[2 * o + 1]);
        }
      }
    }
    // DoG: the next level's difference needs L_lev; LoG: d_yy of the next plane
    if (!LOG || (lev & 1) == 0) {
#pragma unroll
      for (int k = 0; k < 16; ++k) part[k] = Lc[k];
    }
    }   // active
    __syncthreads();   // buffer lev & 1 is free for level lev + 2
  }
  if (!v || !active) return;
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    const int y = Y0 + 8 * rg + o;
    if (y < H) {
      const int64_t pi = (int64_t)b * plane + (int64_t)y * W + x0 + 2 * cp;
      const int k = 2 * o;
      *reinterpret_cast<float2*>(v + pi) = degen ? make_float2(0.f, 0.f) : make_float2(vbest[k], vbest[k + 1]);
      const uint32_t i0 = (ibest[k >> 2] >> ((k & 3) * 8)) & 0xffu, i1 = (ibest[(k + 1) >> 2] >> (((k + 1) & 3) * 8)) & 0xffu;
      *reinterpret_cast<uchar2*>(idx + pi) = degen ? make_uchar2(0, 0) : make_uchar2((uint8_t)i0, (uint8_t)i1);
    }
  }
}

// Row pass over ALL levels of one 32-row x 256-column tile, paper mode (pairs with
// k_cols_pair): the centred image window (32 rows x 256 + 2 R_max + pad columns) is staged
// ONCE, transposed (column-major, pitch kBandHP), and every level's row blur is col_pass
// run along x on that buffer (8 outputs along x x 2 rows per thread, row-pair FFMA2 with a
// broadcast tap), written to Rx_i.  Against k_rows2 (one launch per level, the window
// re-staged per level, conv4_row at ~40 % FMA activity) the staging is amortised over the
// levels and the FFMA2 : shared-load ratio is 4 : 1.  Tap-order f32 sums.
constexpr int kR3Cols = 256;
__host__ __device__ inline int r3_pre(int rmax) { return (4 - rmax % 4) % 4; }
__host__ __device__ inline int r3_nx(int rmax) { return (2 * rmax + r3_pre(rmax) + 288 + 7) & ~7; }
__host__ __device__ inline int r3_taps_total(const LevelTable& t) {
  int n = 0;
  for (int l = 0; l < t.nlev; ++l) n += c3_taps(t.R[l]);
  return n;
}
__host__ __device__ inline size_t r3_smem(int rmax, int taps_total) {
  return sizeof(float) * ((size_t)r3_nx(rmax) * kBandHP + taps_total) + 16;
}

__global__ void __launch_bounds__(kC3Threads, 1) k_rows_pair(const float* __restrict__ fimg, int W, int H,
                                                             const __grid_constant__ LevelTable tab,
                                                             float* __restrict__ rx_all, int B, int reflect,
                                                             int ry0) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* T = reinterpret_cast<float*>(smem_raw);                 // r3_nx x kBandHP, T[xi][row]
  const int NX = r3_nx(tab.rmax);
  float* wc_all = T + NX * kBandHP;
  // ry0: first 32-row tile (single-image bands compute the Rx rows their columns need)
  const int b = blockIdx.z, y0 = (blockIdx.y + ry0) * 32, x0 = blockIdx.x * kR3Cols;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t plane = (int64_t)H * W;
  const int pm = r3_pre(tab.rmax);
  const int xs = x0 - tab.rmax - pm;                             // multiple of 4
  {
    // lane = row (conflict-free transposed stores), 32 contiguous bytes of that row per chunk
    const float* row = fimg + (int64_t)b * plane + (int64_t)min(y0 + lane, H - 1) * W;
    for (int q = warp; q < NX / 8; q += kC3Threads / 32) {
      const int xq = xs + 8 * q;
      float4 a, c;
      if (!reflect || (xq >= 0 && xq + 8 <= W)) {   // periodic (4-aligned, never straddles) or interior
        const int xa = bidx(xq, W, 0), xb = bidx(xq + 4, W, 0);
        a = __ldg(reinterpret_cast<const float4*>(row + xa));
        c = __ldg(reinterpret_cast<const float4*>(row + xb));
      } else {   // mirrored edge pieces, pixel by pixel
        a = make_float4(row[bidx(xq, W, 1)], row[bidx(xq + 1, W, 1)], row[bidx(xq + 2, W, 1)], row[bidx(xq + 3, W, 1)]);
        c = make_float4(row[bidx(xq + 4, W, 1)], row[bidx(xq + 5, W, 1)], row[bidx(xq + 6, W, 1)],
                        row[bidx(xq + 7, W, 1)]);
      }
      float* d = T + (8 * q) * kBandHP + lane;
      d[0 * kBandHP] = a.x; d[1 * kBandHP] = a.y; d[2 * kBandHP] = a.z; d[3 * kBandHP] = a.w;
      d[4 * kBandHP] = c.x; d[5 * kBandHP] = c.y; d[6 * kBandHP] = c.z; d[7 * kBandHP] = c.w;
    }
    int off = 0;
    for (int l = 0; l < tab.nlev; ++l) {
      const int R = tab.R[l], n = c3_taps(R);
      const float* w = tab.w + tab.woff[l] + tab.pre[l];
      for (int i = tid; i < n; i += kC3Threads) wc_all[off + i] = i < 2 * R + 1 ? w[i] : 0.f;
      off += n;
    }
  }
  __syncthreads();
  const int cp = lane & 15;                  // row pair 2cp, 2cp + 1
  const int rg = 2 * warp + (lane >> 4);     // output columns 8 rg .. 8 rg + 7
  float L[16], vd[16];
  uint32_t id[4];
  int off = 0;
  for (int lev = 0; lev < tab.nlev; ++lev) {
    const int R = tab.R[lev];
    col_pass<kBandHP>(T + (tab.rmax + pm - R + 8 * rg) * kBandHP + 2 * cp, wc_all + off, 2 * R + 1, 0, 0.f, L, vd,
                      id);
    off += c3_taps(R);
    float* out = rx_all + ((int64_t)lev * B + b) * plane + x0 + 8 * rg;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int y = y0 + 2 * cp + c;
      if (y < H) {
        float4* o4 = reinterpret_cast<float4*>(out + (int64_t)y * W);
        o4[0] = make_float4(L[0 + c], L[2 + c], L[4 + c], L[6 + c]);
        o4[1] = make_float4(L[8 + c], L[10 + c], L[12 + c], L[14 + c]);
      }
    }
  }
}

}  // namespace mhfd
