// common.cuh — shared device-side definitions of the MHFD CUDA path (sm_100a).
// Product code: none of this is shared with oracle/ (DESIGN.md §2).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/mhfd.h"

namespace mhfd {

constexpr int kMaxLevels = 64;   // n+1 <= 63 Gaussian levels
constexpr int kMaxTaps = 7168;   // sum over levels of padded 2R+1 taps (28 KB of kernel params)
constexpr int kMaxRadius = 160;  // R = ceil(5 t) <= 160
constexpr int kTapUnroll = 8;    // tap loop unroll; every level's tap run is padded to this
constexpr int kStripW = 32;      // columns per CTA strip (one lane per column in the column pass)
constexpr int kThreads = 256;    // 8 warps per CTA in the scale-space kernel

// Per-image stretch parameters written by the percentile kernels.
struct ImgPar {
  int32_t lo, hi;   // nearest-rank percentile values
  float inv;        // 1/(hi-lo) in f32 (0 if degenerate)
  int32_t degen;    // hi == lo -> the image maps to all zeros
};

// Scale grid and f32 taps, passed by value as a kernel parameter (constant bank 0):
// the tap loop reads weights through uniform registers (LDCU), which keeps the
// FFMA at its full issue rate (profiles/r01_ubench_ffma.json).
struct LevelTable {
  int32_t nlev;                 // n + 1
  int32_t rmax;                 // max_i R_i
  int32_t ntaps_total;          // sum of ntap (floats of w[] in use)
  int32_t R[kMaxLevels];        // truncation radius of level i (ceil(5 t_i))
  int32_t pre[kMaxLevels];      // p = (-R) mod 4 zero taps in front (16-byte aligned windows)
  int32_t ntap[kMaxLevels];     // p+2R+1 rounded up to kTapUnroll
  int32_t woff[kMaxLevels];     // offset of level i's taps in w[]
  float tdog[kMaxLevels];       // t_i, the Eq. 2 factor of DoG plane i
  float w[kMaxTaps];            // p zeros, taps w_i[d] for d = -R..R, zero padding
};

// Integer-rank targets of the percentile selection (computed on the host in f64).
struct RankPar {
  int64_t npx;       // H*W
  int64_t rank_lo;   // floor(sat_low * N)
  int64_t rank_hi;   // N - 1 - floor(sat_high * N)
};

struct Shape {
  int32_t W, H;
  int64_t pitch;     // bytes per row
  int32_t bpp;       // 1 (u8) or 2 (u16)
};

__device__ __forceinline__ uint32_t load_px(const uint8_t* img, int64_t pitch, int bpp, int y, int x) {
  const uint8_t* row = img + (int64_t)y * pitch;
  return bpp == 1 ? (uint32_t)row[x] : (uint32_t)reinterpret_cast<const uint16_t*>(row)[x];
}

}  // namespace mhfd
