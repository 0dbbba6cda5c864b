// k_downsample.cuh — bilinear downsampling pre-step (PAPER.md:401,
// SPEC.md:48-56; semantics in include/mhfd.h and DESIGN.md reading R22).
//
// For an integer factor f the half-pixel sample position of output X is
// x = X f + (f - 1)/2: twice it, 2 X f + f - 1, is an integer whose parity gives the
// fractional part (0 or 1/2).  With weights counted in halves, the exact bilinear value
// times 4 is an integer S, and the output is (S + 2) >> 2 (round half up): integer
// arithmetic only.  Both neighbour indices are clamped to the last row/column (the last of
// ceil(W/f) samples may lie past it).  HBM-bound: each thread produces 4 consecutive outputs of one row;
// loads of a warp cover 128 f contiguous input bytes per sampled row.
#pragma once
#include <cstdint>

namespace mhfd {

template <typename T>
__global__ void __launch_bounds__(256) k_downsample(const uint8_t* __restrict__ in, int W, int H, int64_t in_pitch,
                                                    int f, uint8_t* __restrict__ out, int OW, int OH,
                                                    int64_t out_pitch, int batch) {
  const int qw = (OW + 3) / 4;                       // 4-output groups per row
  const int64_t total = (int64_t)batch * OH * qw;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(i % qw);
    const int64_t r = i / qw;
    const int Y = (int)(r % OH), b = (int)(r / OH);
    const int y2 = 2 * Y * f + f - 1;                 // twice the sample row
    const int ay = y2 & 1, y0 = min(y2 >> 1, H - 1), y1 = min((y2 >> 1) + 1, H - 1);
    const T* r0 = reinterpret_cast<const T*>(in + ((int64_t)b * H + y0) * in_pitch);
    const T* r1 = reinterpret_cast<const T*>(in + ((int64_t)b * H + y1) * in_pitch);
    T* o = reinterpret_cast<T*>(out + ((int64_t)b * OH + Y) * out_pitch);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int X = 4 * g + k;
      if (X >= OW) break;
      const int x2 = 2 * X * f + f - 1;
      const int ax = x2 & 1, x0 = min(x2 >> 1, W - 1), x1 = min((x2 >> 1) + 1, W - 1);
      // weights in halves: (2 - a) at index 0, a at index 1
      uint32_t s = (uint32_t)(2 - ax) * (2 - ay) * r0[x0];
      if (ax) s += (uint32_t)(2 - ay) * r0[x1];
      if (ay) s += (uint32_t)(2 - ax) * r1[x0];
      if (ax && ay) s += (uint32_t)r1[x1];
      o[X] = (T)((s + 2u) >> 2);
    }
  }
}

// Factor-2 fast path (rows and row pitches multiples of 16 bytes, even W): every output
// is the rounded-half-up mean of a 2 x 2 block (rows 2Y, min(2Y + 1, H - 1)); a thread
// reads 16 bytes of each row with one 128-bit load and writes 8 bytes (u8: 8 outputs,
// u16: 4 outputs).  Same integer formula as k_downsample.
template <typename T>
__global__ void __launch_bounds__(256) k_downsample2(const uint8_t* __restrict__ in, int W, int H, int64_t in_pitch,
                                                     uint8_t* __restrict__ out, int OH, int64_t out_pitch,
                                                     int batch) {
  constexpr int NPX = 16 / sizeof(T);                 // input pixels per 16-byte chunk
  const int nc = W / NPX;                             // chunks per row
  const int64_t total = (int64_t)batch * OH * nc;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % nc);
    const int64_t r = i / nc;
    const int Y = (int)(r % OH), b = (int)(r / OH);
    const int y0 = 2 * Y, y1 = min(2 * Y + 1, H - 1);
    const uint4 p = __ldg(reinterpret_cast<const uint4*>(in + ((int64_t)b * H + y0) * in_pitch) + c);
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(in + ((int64_t)b * H + y1) * in_pitch) + c);
    const T* a = reinterpret_cast<const T*>(&p);
    const T* d = reinterpret_cast<const T*>(&q);
    T o[NPX / 2];
#pragma unroll
    for (int k = 0; k < NPX / 2; ++k)
      o[k] = (T)(((uint32_t)a[2 * k] + a[2 * k + 1] + d[2 * k] + d[2 * k + 1] + 2u) >> 2);
    *reinterpret_cast<uint2*>(out + ((int64_t)b * OH + Y) * out_pitch + (int64_t)c * 8) =
        *reinterpret_cast<const uint2*>(o);
  }
}

}  // namespace mhfd
