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

}  // namespace mhfd
