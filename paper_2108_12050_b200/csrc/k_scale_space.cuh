// k_scale_space.cuh — stretch-on-load prepass and the hot kernel: separable Gaussian
// blur at all n+1 scales, Eq. 2 DoG and the Eq. 3 inner argmax over scale, fused (hot-
// path rows a2-a6).  The response stack never touches HBM: per pixel only v = max_i DoG
// (f32) and its first argmax (u8) are written (or, in 26-NMS / dump mode, the n planes).
//
//  PAPER.md:257        I' = clamp((I-lo)/(hi-lo), 0, 1)   (centred by -1/2; the DoG is
//                      unchanged because every level's taps sum to 1)      [k_normalize]
//  PAPER.md:136-141    L(.,.,t_i) = G(t_i) * I', sigma = t_i, periodic boundary
//                      (readings R1, R7); taps sampled, renormalised, |d| <= ceil(5 t_i)
//                      (reading R6)
//  PAPER.md:171        DoG_i = t_i (L_{i+1} - L_i)
//  PAPER.md:240-244    v = max_i DoG_i, i^ = first argmax (reading R10)
//
// Layout: one CTA = one image x one strip of 32 columns x one band of
// BH = 8*RPT rows; 256 threads, 2 CTAs per SM.  Levels are processed one after another.
//   row pass   : chunks of 32 rows x (32+2R+pad) columns of the normalised f32 image are
//                brought into shared memory by TMA (one 2-D cp.async.bulk.tensor box per
//                chunk; chunks that wrap around the image edge use one 1-D cp.async.bulk
//                per row, split at the edge), in a 3-stage mbarrier pipeline so the copies
//                of chunks k+1, k+2 overlap the FMAs of chunk k.  Lane =
//                row; each thread convolves 4 consecutive columns with 128-bit LDS (row
//                pitch = 4 x odd words -> conflict-free), writing (BH+2R+p) x 32 filtered
//                rows to `hbuf`.
//   column pass: lane = column, each thread convolves RPT consecutive rows (8 at a time)
//                from `hbuf`, then updates DoG / running max / argmax held in registers.
// Taps are prefixed with p = (-R) mod 4 zeros so every window starts 16-byte aligned; the
// same prefixed table serves both passes (hbuf row 0 = band row -R-p).  The tap table is
// copied from the kernel parameters into shared memory once per CTA and read with
// broadcast 128-bit loads (4 weights per instruction).
#pragma once
#include "common.cuh"

namespace mhfd {

constexpr int kChunkRows = 32;
constexpr int kStages = 3;         // stage buffers in the copy pipeline
constexpr int kHP = kStripW + 1;   // hbuf pitch (odd: conflict-free row-pass stores)

// stage pitch: 4*q floats with q odd (conflict-free LDS.128 with lane = row), holding
// 32 + 2R + p columns plus the window overrun of the padded tap loop
__host__ __device__ inline int stage_pitch(int rmax) {
  int q = (2 * rmax + 47 + 3) / 4;   // >= 32+2R+p+3 staged columns and the 2R+p+43 window reach
  if ((q & 1) == 0) ++q;
  return 4 * q;
}
__host__ __device__ inline int hbuf_rows(int rmax, int BH) { return BH + 2 * rmax + 3 + 16; }
// hbuf floats, rounded to 32 so the tap table and mbarriers after it stay 128-byte aligned
__host__ __device__ inline int hbuf_floats(int rmax, int BH) { return (hbuf_rows(rmax, BH) * kHP + 31) & ~31; }
__host__ __device__ inline int wtab_floats(int ntaps_total) { return (ntaps_total + 31) & ~31; }
// layout: [stage: stages x 32 x SP][hbuf][weights wA][weights wB][mbarriers]
__host__ __device__ inline size_t scale_space_smem(int rmax, int BH, int ntaps_total, int stages = kStages) {
  return sizeof(float) * ((size_t)stages * kChunkRows * stage_pitch(rmax) + 64 + (size_t)hbuf_floats(rmax, BH) +
                          2 * wtab_floats(ntaps_total)) +
         8 * stages;
}
// 2-D TMA boxes hold SP <= 256 columns
__host__ __device__ inline bool tma_boxes(int rmax) { return stage_pitch(rmax) <= 256; }
// the bulk-copy staging path needs every row segment to wrap at most once, at a
// 16-byte boundary
__host__ __device__ inline bool fast_staging(int W, int rmax) { return (W % 4) == 0 && W >= kStripW + 2 * rmax + 16; }

__device__ __forceinline__ int wrap_idx(int a, int n) {
  while (a < 0) a += n;
  while (a >= n) a -= n;
  return a;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tma_2d_g2s(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------------
// k_normalize: u8/u16 -> centred f32 I' - 1/2, row-major W floats per row (a2).
template <int BPP>
__global__ void __launch_bounds__(256) k_normalize(const uint8_t* __restrict__ images, Shape s,
                                                   const ImgPar* __restrict__ par, float* __restrict__ out) {
  const int b = blockIdx.y;
  const ImgPar ip = par[b];
  const float lo = (float)ip.lo, inv = ip.inv;
  const uint8_t* img = images + (int64_t)b * s.H * s.pitch;
  float* o = out + (int64_t)b * s.H * s.W;
  const int64_t total = (int64_t)s.H * s.W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / s.W), x = (int)(i - (int64_t)y * s.W);
    const float p = (float)load_px(img, s.pitch, BPP, y, x);
    o[i] = fminf(fmaxf((p - lo) * inv, 0.f), 1.f) - 0.5f;
  }
}

// f32 input (reading R24): lo/hi are float32 bit patterns in ImgPar; 4 pixels per
// 16-byte load when W % 4 == 0
__global__ void __launch_bounds__(256) k_normalize_f32(const uint8_t* __restrict__ images, Shape s,
                                                       const ImgPar* __restrict__ par, float* __restrict__ out) {
  const int b = blockIdx.y;
  const ImgPar ip = par[b];
  const float lo = __int_as_float(ip.lo), inv = ip.inv;
  const uint8_t* img = images + (int64_t)b * s.H * s.pitch;
  float* o = out + (int64_t)b * s.H * s.W;
  if (s.W % 4 == 0) {
    const int vpr = s.W / 4;
    const int64_t total = (int64_t)s.H * vpr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      const int y = (int)(i / vpr), v = (int)(i - (int64_t)y * vpr);
      const float4 q = __ldg(reinterpret_cast<const float4*>(img + (int64_t)y * s.pitch) + v);
      float4 r;
      r.x = fminf(fmaxf((q.x - lo) * inv, 0.f), 1.f) - 0.5f;
      r.y = fminf(fmaxf((q.y - lo) * inv, 0.f), 1.f) - 0.5f;
      r.z = fminf(fmaxf((q.z - lo) * inv, 0.f), 1.f) - 0.5f;
      r.w = fminf(fmaxf((q.w - lo) * inv, 0.f), 1.f) - 0.5f;
      reinterpret_cast<float4*>(o)[i] = r;
    }
  } else {
    const int64_t total = (int64_t)s.H * s.W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      const int y = (int)(i / s.W), x = (int)(i - (int64_t)y * s.W);
      const float p = reinterpret_cast<const float*>(img + (int64_t)y * s.pitch)[x];
      o[i] = fminf(fmaxf((p - lo) * inv, 0.f), 1.f) - 0.5f;
    }
  }
}

// vectorised variant: 16 input bytes per thread-iteration; needs W % 16 == 0 (u8) or
// W % 8 == 0 (u16)
template <int BPP>
__global__ void __launch_bounds__(256) k_normalize_vec(const uint8_t* __restrict__ images, Shape s,
                                                       const ImgPar* __restrict__ par, float* __restrict__ out) {
  constexpr int PX = 16 / BPP;   // pixels per 16-byte vector
  const int b = blockIdx.y;
  const ImgPar ip = par[b];
  const float lo = (float)ip.lo, inv = ip.inv;
  const uint8_t* img = images + (int64_t)b * s.H * s.pitch;
  float* o = out + (int64_t)b * s.H * s.W;
  const int vpr = s.W / PX;  // vectors per row
  const int64_t total = (int64_t)s.H * vpr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / vpr), v = (int)(i - (int64_t)y * vpr);
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(img + (int64_t)y * s.pitch) + v);
    const uint32_t wds[4] = {q.x, q.y, q.z, q.w};
    float f[PX];
#pragma unroll
    for (int k = 0; k < PX; ++k) {
      const uint32_t p = BPP == 1 ? (wds[k >> 2] >> (8 * (k & 3))) & 0xffu : (wds[k >> 1] >> (16 * (k & 1))) & 0xffffu;
      f[k] = fminf(fmaxf(((float)p - lo) * inv, 0.f), 1.f) - 0.5f;
    }
    float4* dst = reinterpret_cast<float4*>(o + (int64_t)y * s.W + (int64_t)v * PX);
#pragma unroll
    for (int k = 0; k < PX / 4; ++k) dst[k] = make_float4(f[4 * k], f[4 * k + 1], f[4 * k + 2], f[4 * k + 3]);
  }
}

// ---------------------------------------------------------------------------------
// Packed FFMA2 convolutions.  A 1-D convolution out[o] = sum_t w[t] x[o+t] is computed
// with tap pairs: FFMA2 multiplies an input pair (x[2m], x[2m+1]) by a weight pair and
// accumulates into (acc.x, acc.y), out[o] = acc.x + acc.y.  Even outputs use the pairs
// (w[2k], w[2k+1]) (table wA = w), odd outputs the pairs (w[2k-1], w[2k]) (table wB[i] =
// w[i-1]); both then meet 2-aligned input pairs, so every operand is an aligned register
// pair and no shuffling is needed.  Odd outputs need one extra pair k = ntap/2 whose
// second weight w[ntap] is the zero padding after each level's taps.
__device__ __forceinline__ float2 lo2(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4& v) { return make_float2(v.z, v.w); }

// row pass: out[o] = sum_{t<ntap} w[t] src[o+t], o = 0..3; src 16-byte aligned, ntap % 8 == 0
__device__ __forceinline__ void conv4_row(float (&out)[4], const float* __restrict__ src, const float* __restrict__ wA,
                                          const float* __restrict__ wB, int ntap) {
  float2 acc[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) acc[o] = make_float2(0.f, 0.f);
  const float4* s4 = reinterpret_cast<const float4*>(src);
  const float4* a4 = reinterpret_cast<const float4*>(wA);
  const float4* b4 = reinterpret_cast<const float4*>(wB);
  float4 xa = s4[0];
  for (int j = 0; j < ntap; j += 8) {
    const int q = j >> 2;
    const float4 xb = s4[q + 1], xc = s4[q + 2];
    const float4 A0 = a4[q], A1 = a4[q + 1], B0 = b4[q], B1 = b4[q + 1];
    const float2 P[5] = {lo2(xa), hi2(xa), lo2(xb), hi2(xb), lo2(xc)};
    const float2 WA[4] = {lo2(A0), hi2(A0), lo2(A1), hi2(A1)};
    const float2 WB[4] = {lo2(B0), hi2(B0), lo2(B1), hi2(B1)};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      acc[0] = __ffma2_rn(P[kk], WA[kk], acc[0]);
      acc[1] = __ffma2_rn(P[kk], WB[kk], acc[1]);
      acc[2] = __ffma2_rn(P[kk + 1], WA[kk], acc[2]);
      acc[3] = __ffma2_rn(P[kk + 1], WB[kk], acc[3]);
    }
    xa = xc;
  }
  {  // odd outputs: tap pair (ntap-1, ntap)
    const float2 wb = reinterpret_cast<const float2*>(wB)[ntap >> 1];
    acc[1] = __ffma2_rn(lo2(xa), wb, acc[1]);
    acc[3] = __ffma2_rn(hi2(xa), wb, acc[3]);
  }
#pragma unroll
  for (int o = 0; o < 4; ++o) out[o] = acc[o].x + acc[o].y;
}

// acc[2q], acc[2q+1] += pair (q + kk) x (wA, wB) pair kk, for the 8 outputs of the column pass
__device__ __forceinline__ void col_group(float2 (&acc)[8], const float2 (&Pa)[4], const float2 (&Pb)[4],
                                          const float* __restrict__ wA, const float* __restrict__ wB) {
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const float2 wa = reinterpret_cast<const float2*>(wA)[kk];
    const float2 wb = reinterpret_cast<const float2*>(wB)[kk];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int m = q + kk;
      const float2 x = m < 4 ? Pa[m] : Pb[m - 4];
      acc[2 * q] = __ffma2_rn(x, wa, acc[2 * q]);
      acc[2 * q + 1] = __ffma2_rn(x, wb, acc[2 * q + 1]);
    }
  }
}

__device__ __forceinline__ void load_pairs(float2 (&P)[4], const float* __restrict__ src, int stride, int m0) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    P[k] = make_float2(src[(2 * (m0 + k)) * stride], src[(2 * (m0 + k) + 1) * stride]);
}

// column pass: out[o] = sum_{t<ntap} w[t] src[(o+t)*stride], o = 0..7, ntap % 8 == 0
__device__ __forceinline__ void conv8_col(float (&out)[8], const float* __restrict__ src, int stride,
                                          const float* __restrict__ wA, const float* __restrict__ wB, int ntap) {
  float2 acc[8];
#pragma unroll
  for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.f, 0.f);
  float2 Pa[4], Pb[4];
  load_pairs(Pa, src, stride, 0);
  int j = 0;
  for (; j + 16 <= ntap; j += 16) {
    load_pairs(Pb, src, stride, (j >> 1) + 4);
    col_group(acc, Pa, Pb, wA + j, wB + j);
    load_pairs(Pa, src, stride, (j >> 1) + 8);
    col_group(acc, Pb, Pa, wA + j + 8, wB + j + 8);
  }
  if (j < ntap) {  // ntap % 16 == 8
    load_pairs(Pb, src, stride, (j >> 1) + 4);
    col_group(acc, Pa, Pb, wA + j, wB + j);
#pragma unroll
    for (int k = 0; k < 4; ++k) Pa[k] = Pb[k];
  }
  {  // odd outputs: tap pair (ntap-1, ntap), input pairs ntap/2 + q (now in Pa)
    const float2 wb = reinterpret_cast<const float2*>(wB)[ntap >> 1];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[2 * q + 1] = __ffma2_rn(Pa[q], wb, acc[2 * q + 1]);
  }
#pragma unroll
  for (int o = 0; o < 8; ++o) out[o] = acc[o].x + acc[o].y;
}

// Stage rows [r0, r0 + nrow) of a level's row-pass input (image rows Y0-R-p+r, columns
// x0-R-p .. x0+32+R+3) into `dst0` (kChunkRows x SP floats).  FAST: warp 0 issues one
// bulk copy per row (two where the row wraps at the image edge) completing on `bar`;
// otherwise every thread copies with plain loads (caller synchronises).
template <bool FAST>
__device__ __forceinline__ void stage_rows(float* dst0, uint64_t* bar, const float* __restrict__ img,
                                           const void* tmap, int b, int W, int H, int x0, int Y0, int R, int p,
                                           int r0, int nrow, int SP, int warp, int lane) {
  const int xs = x0 - R - p;                  // first staged column (multiple of 4)
  const int ncol = (kStripW + 2 * R + p + 3) & ~3;
  const int yf = Y0 - R - p + r0;             // first image row of the chunk
  if (FAST && tmap != nullptr && xs >= 0 && xs + ncol <= W && yf >= 0 && yf + nrow <= H) {
    // interior chunk: one 2-D box of 32 rows x SP columns (rows/columns past the needed
    // ones are harmless: they meet zero taps or are not stored)
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(bar, (uint32_t)(kChunkRows * SP * 4));
      tma_2d_g2s(dst0, tmap, xs, b * H + yf, bar);
    }
  } else if (FAST) {
    if (warp == 0) {
      if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(nrow * ncol * 4));
      __syncwarp();
      if (lane < nrow) {
        const int y = wrap_idx(Y0 - R - p + r0 + lane, H);
        const float* row = img + (int64_t)y * W;
        float* dst = dst0 + lane * SP;
        if (xs < 0) {
          bulk_g2s(dst, row + (W + xs), (uint32_t)(-xs * 4), bar);
          bulk_g2s(dst - xs, row, (uint32_t)((ncol + xs) * 4), bar);
        } else if (xs + ncol > W) {
          bulk_g2s(dst, row + xs, (uint32_t)((W - xs) * 4), bar);
          bulk_g2s(dst + (W - xs), row, (uint32_t)((xs + ncol - W) * 4), bar);
        } else {
          bulk_g2s(dst, row + xs, (uint32_t)(ncol * 4), bar);
        }
      }
    }
  } else {
    for (int k = warp; k < nrow; k += 8) {
      const int y = wrap_idx(Y0 - R - p + r0 + k, H);
      const float* row = img + (int64_t)y * W;
      for (int cc = lane; cc < ncol; cc += 32) dst0[k * SP + cc] = row[wrap_idx(xs + cc, W)];
    }
  }
}

// RPT rows per thread (band height BH = 8 RPT), NST copy stages.  The 384-row band
// (RPT = 48, two stages, one CTA per SM) is for large radii, where the row pass
// recomputes (BH + 2R) / BH rows per output (3.3x at R = 150 with 128-row bands).
template <int RPT, bool WRITE_V, bool WRITE_DOG, bool FAST, int NST = kStages>
__global__ void __launch_bounds__(kThreads, RPT > 32 ? 1 : 2)
k_scale_space(const float* __restrict__ fimg, Shape s, const ImgPar* __restrict__ par,
              const __grid_constant__ LevelTable tab, const __grid_constant__ CUtensorMap tmap, int use_tmap,
              float* __restrict__ v_out,
              uint8_t* __restrict__ idx_out, float* __restrict__ dog_out) {
  constexpr int BH = 8 * RPT;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* smem = reinterpret_cast<float*>(smem_raw);
  const int rmax = tab.rmax;
  const int SP = stage_pitch(rmax);
  float* stage = smem;                                         // NST x kChunkRows x SP
  float* hbuf = smem + NST * kChunkRows * SP + 64;             // hbuf_rows x kHP
  float* wsm = hbuf + hbuf_floats(rmax, BH);                   // tap table
  float* wsmB = wsm + wtab_floats(tab.ntaps_total);            // shifted tap table w[i-1]
  uint64_t* bars = reinterpret_cast<uint64_t*>(wsmB + wtab_floats(tab.ntaps_total));

  const int b = blockIdx.z;
  const int x0 = blockIdx.x * kStripW;
  const int Y0 = blockIdx.y * BH;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const float* img = fimg + (int64_t)b * s.H * s.W;
  const int64_t plane = (int64_t)s.H * s.W;

  if (par[b].degen) {  // hi == lo: I' == 0, every DoG plane is exactly 0
    const int x = x0 + lane;
    for (int r = 0; r < RPT; ++r) {
      const int y = Y0 + warp * RPT + r;
      if (x < s.W && y < s.H) {
        const int64_t p = (int64_t)y * s.W + x;
        if (WRITE_V) { v_out[(int64_t)b * plane + p] = 0.f; idx_out[(int64_t)b * plane + p] = 0; }
        if (WRITE_DOG)
          for (int i = 0; i + 1 < tab.nlev; ++i) dog_out[((int64_t)b * (tab.nlev - 1) + i) * plane + p] = 0.f;
      }
    }
    return;
  }

  // zero stage and hbuf once: entries past a level's valid columns / rows are read only
  // against zero (padding) taps and must stay finite
  const int nzero = NST * kChunkRows * SP + 64 + hbuf_floats(rmax, BH);
  for (int i = threadIdx.x; i < nzero; i += kThreads) smem[i] = 0.f;
  for (int i = threadIdx.x; i < tab.ntaps_total; i += kThreads) wsm[i] = tab.w[i];
  for (int l = 0; l < tab.nlev; ++l)  // wB = each level's taps shifted right by one (zero in front)
    for (int i = threadIdx.x; i < tab.ntap[l] + 8; i += kThreads)
      wsmB[tab.woff[l] + i] = i ? tab.w[tab.woff[l] + i - 1] : 0.f;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const void* tm = use_tmap ? (const void*)&tmap : nullptr;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  float lprev[RPT], vbest[RPT];
  uint32_t ibest[RPT / 4];
#pragma unroll
  for (int r = 0; r < RPT; ++r) { lprev[r] = 0.f; vbest[r] = -INFINITY; }
#pragma unroll
  for (int r = 0; r < RPT / 4; ++r) ibest[r] = 0u;

  const int nlev = tab.nlev;
  uint32_t phases = 0u;   // bit k: parity of mbarrier k
  // copy cursor: the (level, first row) of the next item to stage; items rotate through
  // the NST buffers, NST-1 of them in flight ahead of the one being convolved
  auto rows_of = [BH](int R, int p) { return BH + 2 * R + p; };
  int cl = 0, cq = 0;
  auto stage_next = [&](int dst) {
    if (cl >= nlev) return;
    const int R = tab.R[cl], p = tab.pre[cl];
    stage_rows<FAST>(stage + dst * kChunkRows * SP, &bars[dst], img, tm, b, s.W, s.H, x0, Y0, R, p, cq,
                     min(kChunkRows, rows_of(R, p) - cq), SP, warp, lane);
    cq += kChunkRows;
    if (cq >= rows_of(R, p)) { ++cl; cq = 0; }
  };
  for (int k = 0; k + 1 < NST; ++k) stage_next(k);   // prologue
  int buf = 0;

  for (int lev = 0; lev < nlev; ++lev) {
    const int ntap = tab.ntap[lev];
    const float* w = wsm + tab.woff[lev];
    const float* wB = wsmB + tab.woff[lev];
    const int nrow = rows_of(tab.R[lev], tab.pre[lev]);   // hbuf rows: band rows -R-p .. BH+R-1

    // ---------------- row pass (chunks of 32 rows) ----------------
    for (int r0 = 0; r0 < nrow; r0 += kChunkRows) {
      stage_next((buf + NST - 1) % NST);   // into the buffer the previous item freed
      if (FAST) {
        mbar_wait(&bars[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
      } else {
        __syncthreads();
      }
      const float* src = stage + buf * kChunkRows * SP + lane * SP + 4 * warp;
      float acc[4];
      conv4_row(acc, src, w, wB, ntap);
      if (r0 + lane < nrow) {
        float* h = hbuf + (r0 + lane) * kHP + 4 * warp;
#pragma unroll
        for (int o = 0; o < 4; ++o) h[o] = acc[o];
      }
      buf = (buf + 1) % NST;
      __syncthreads();   // this stage buffer is free for the copy issued in the next iteration
    }

    // ---------------- column pass + DoG + running argmax ----------------
    const float tprev = lev > 0 ? tab.tdog[lev - 1] : 0.f;
#pragma unroll
    for (int q = 0; q < RPT / 8; ++q) {
      const int rb = warp * RPT + q * 8;      // first band row of this group
      float acc[8];
      conv8_col(acc, hbuf + rb * kHP + lane, kHP, w, wB, ntap);
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        const int r = q * 8 + o;
        const float L = acc[o];
        if (lev > 0) {
          const float D = tprev * (L - lprev[r]);
          if (D > vbest[r]) {
            vbest[r] = D;
            const int sh = (r & 3) * 8;
            ibest[r >> 2] = (ibest[r >> 2] & ~(0xffu << sh)) | ((uint32_t)(lev - 1) << sh);
          }
          if (WRITE_DOG) {
            const int x = x0 + lane, y = Y0 + rb + o;
            if (x < s.W && y < s.H)
              dog_out[((int64_t)b * (tab.nlev - 1) + (lev - 1)) * plane + (int64_t)y * s.W + x] = D;
          }
        }
        lprev[r] = L;
      }
    }
    __syncthreads();  // hbuf is rewritten by the next level
  }

  if (WRITE_V) {
    const int x = x0 + lane;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int y = Y0 + warp * RPT + r;
      if (x < s.W && y < s.H) {
        const int64_t p = (int64_t)b * plane + (int64_t)y * s.W + x;
        v_out[p] = vbest[r];
        idx_out[p] = (uint8_t)((ibest[r >> 2] >> ((r & 3) * 8)) & 0xffu);
      }
    }
  }
}

}  // namespace mhfd
