// k_percentile.cuh — histogram + nearest-rank percentile selection (hot-path row a1).
//
// PAPER.md:255-259 (§3): "saturating .175% of the darkest pixels, saturating .175%
// of the lightest pixels, and mapping the entire range to [0,1] ... parallelized
// using GPU primitives".  Nearest rank (reading R13): lo is the pixel value of
// rank floor(sat_low*N), hi the value of rank N-1-floor(sat_high*N) in the sorted
// image.  Exact integer radix select: pass 1 histograms the top byte (the whole
// value for u8); for u16 pass 2 histograms the low byte of the pixels in the two
// selected top-byte bins.  HBM-bound: the image is read once per pass with
// 128-bit loads; histograms are privatised per warp in shared memory.
#pragma once
#include "common.cuh"

namespace mhfd {

struct SelState {      // per image, between the two passes
  int32_t bin_lo, bin_hi;   // selected top-byte bins
  int64_t rem_lo, rem_hi;   // ranks inside those bins
};

__device__ __forceinline__ void finish(ImgPar* p, int lo, int hi) {
  p->lo = lo;
  p->hi = hi;
  p->degen = (hi == lo) ? 1 : 0;
  p->inv = (hi == lo) ? 0.0f : 1.0f / (float)(hi - lo);
}

// Smallest bin whose cumulative count exceeds `rank` (returns the rank left inside it),
// warp-cooperative: lane l holds bins 8l .. 8l + 7 (two 16-byte loads), a warp
// scan of the lane sums finds the lane whose range holds `rank`, that lane walks its 8
// bins (a serial 256-bin walk is 256 dependent loads: ~14 us for one image).
__device__ __forceinline__ int select_bin_warp(const uint32_t* h, int64_t rank, int64_t* rem) {
  const int lane = threadIdx.x & 31;
  const uint4 a = reinterpret_cast<const uint4*>(h)[2 * lane], c = reinterpret_cast<const uint4*>(h)[2 * lane + 1];
  const uint32_t v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
  int64_t sum = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) sum += v[i];
  int64_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int64_t excl = incl - sum;
  const uint32_t m = __ballot_sync(0xffffffffu, incl > rank);   // lanes past the rank
  int bin = 255;
  int64_t r = 0;
  if (m) {
    const int src = __ffs(m) - 1;
    if (lane == src) {
      int64_t cum = excl;
      bin = 8 * lane + 7;
      for (int i = 0; i < 8; ++i) {
        if (cum + v[i] > rank) { bin = 8 * lane + i; break; }
        cum += v[i];
      }
      r = rank - cum;
    }
    bin = __shfl_sync(0xffffffffu, bin, src);
    r = __shfl_sync(0xffffffffu, r, src);
  }
  *rem = r;
  return bin;
}

// Pass 1: 256-bin histogram of (u8 value) or (u16 value >> 8).
// Pass 2 (u16 only, second=true): low-byte histograms of the two selected bins.
// SELECT: the image's last CTA to flush (a per-image ticket after the histograms, zeroed
// with them) selects the two ranks itself: u8 percentiles take one launch, u16 two (pass 1
// leaves the high bytes and remaining ranks in sel, pass 2 finishes).
template <int BPP, bool SECOND, bool SELECT = false>
__global__ void __launch_bounds__(256) k_hist(const uint8_t* __restrict__ images, Shape s, int rows_per_cta,
                                              uint32_t* __restrict__ hist, SelState* __restrict__ sel,
                                              RankPar rk = RankPar{}, ImgPar* __restrict__ par = nullptr,
                                              uint32_t* __restrict__ ticket = nullptr) {
  constexpr int NH = SECOND ? 2 : 1;
  __shared__ uint32_t sh[8][NH * 256];
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * NH * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  int sel_lo = -1, sel_hi = -1;
  if (SECOND) { sel_lo = sel[b].bin_lo; sel_hi = sel[b].bin_hi; }
  const uint32_t sel_lo2 = (uint32_t)(sel_lo & 0xff) * 0x10001u, sel_hi2 = (uint32_t)(sel_hi & 0xff) * 0x10001u;
  __syncthreads();
  const uint8_t* img = images + (int64_t)b * s.H * s.pitch;
  const int y0 = blockIdx.x * rows_per_cta;
  const int y1 = min(s.H, y0 + rows_per_cta);
  const int row_bytes = s.W * BPP;
  const int nvec = (row_bytes + 15) >> 4;
  if ((row_bytes & 15) == 0) {
    // whole-vector rows (any width), both radix passes: the CTA's (row, vector) items are
    // walked four at a time per thread, so four loads are in flight before their atomics
    // instead of a chain of dependent load latencies (u8 8 x 4096^2: 0.10 ms; one 4096^2
    // u16 tile's two passes 0.055 -> 0.041 ms)
    uint32_t* hw = sh[warp];
    auto acc = [&](const uint4& q) {
      const uint32_t wds[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (BPP == 1) {
#pragma unroll
          for (int j = 0; j < 4; ++j) atomicAdd(hw + ((wds[k] >> (8 * j)) & 255u), 1u);
        } else if (!SECOND) {
          atomicAdd(hw + ((wds[k] >> 8) & 255u), 1u);
          atomicAdd(hw + (wds[k] >> 24), 1u);
        } else {
          // both 16-bit values' high bytes against the two selected bins at once (SIMD
          // compare): almost every word matches neither and costs four instructions
          const uint32_t hb = (wds[k] >> 8) & 0x00ff00ffu;
          if (__vcmpeq2(hb, sel_lo2) | __vcmpeq2(hb, sel_hi2)) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint32_t val = (wds[k] >> (16 * j)) & 0xffffu, top = val >> 8;
              if ((int)top == sel_lo) atomicAdd(hw + (val & 255u), 1u);
              if ((int)top == sel_hi) atomicAdd(hw + 256 + (val & 255u), 1u);
            }
          }
        }
      }
    };
    const int nvt = (nvec + blockDim.x - 1) / blockDim.x;   // vectors per thread and row
    const int nit = (y1 - y0) * nvt;
    for (int it = 0; it < nit; it += 4) {
      uint4 q[4];
      bool ok[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = it + r, yy = y0 + i / nvt, v = threadIdx.x + (i % nvt) * blockDim.x;
        ok[r] = i < nit && v < nvec;
        q[r] = ok[r] ? __ldg(reinterpret_cast<const uint4*>(img + (int64_t)yy * s.pitch) + v) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (ok[r]) acc(q[r]);
    }
  } else
  for (int y = y0; y < y1; ++y) {
    const uint4* row = reinterpret_cast<const uint4*>(img + (int64_t)y * s.pitch);
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
      uint4 q = __ldg(row + v);
      uint32_t wds[4] = {q.x, q.y, q.z, q.w};
      const int base = v * 16;
      if (!SECOND && base + 16 <= row_bytes) {   // whole vector inside the row: no per-pixel test
        uint32_t* hw = sh[warp];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (BPP == 1) {
#pragma unroll
            for (int j = 0; j < 4; ++j) atomicAdd(hw + ((wds[k] >> (8 * j)) & 255u), 1u);
          } else {
            atomicAdd(hw + ((wds[k] >> 8) & 255u), 1u);
            atomicAdd(hw + (wds[k] >> 24), 1u);
          }
        }
        continue;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (BPP == 1) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (base + 4 * k + j < row_bytes) atomicAdd(&sh[warp][(wds[k] >> (8 * j)) & 255u], 1u);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (base + 4 * k + 2 * j < row_bytes) {
              uint32_t val = (wds[k] >> (16 * j)) & 0xffffu;
              uint32_t top = val >> 8;
              if (!SECOND) {
                atomicAdd(&sh[warp][top], 1u);
              } else {
                if ((int)top == sel_lo) atomicAdd(&sh[warp][val & 255u], 1u);
                if ((int)top == sel_hi) atomicAdd(&sh[warp][256 + (val & 255u)], 1u);
              }
            }
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NH * 256; i += blockDim.x) {
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += sh[w][i];
    if (c) atomicAdd(&hist[(int64_t)b * (NH * 256) + i], c);
  }
  if (SELECT) {
    __shared__ int last;
    __threadfence();   // this CTA's bins are in L2 before its ticket
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&ticket[b], 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x < 32) {
      __threadfence();
      const uint32_t* h = hist + (int64_t)b * (NH * 256);   // every CTA's atomics have landed (L2; not in this L1)
      if (SECOND) {   // u16 pass 2: low bytes under the selected high bytes (k_select2's work)
        int64_t dummy;
        const int lo = (sel[b].bin_lo << 8) | select_bin_warp(h, sel[b].rem_lo, &dummy);
        const int hi = (sel[b].bin_hi << 8) | select_bin_warp(h + 256, sel[b].rem_hi, &dummy);
        if (threadIdx.x == 0) finish(&par[b], lo, hi);
      } else {
        int64_t rl, rh;
        const int bl = select_bin_warp(h, rk.rank_lo, &rl);
        const int bh = select_bin_warp(h, rk.rank_hi, &rh);
        if (threadIdx.x == 0) {
          if (BPP == 1) {
            finish(&par[b], bl, bh);
          } else {   // u16 pass 1: the high bytes and the ranks left inside them (k_select1's work)
            sel[b].bin_lo = bl; sel[b].bin_hi = bh; sel[b].rem_lo = rl; sel[b].rem_hi = rh;
          }
        }
      }
    }
  }
}

// One warp per image: select the two ranks in the 256-bin histogram(s).
template <int BPP>
__global__ void k_select1(const uint32_t* __restrict__ hist1, RankPar r, SelState* __restrict__ sel,
                          ImgPar* __restrict__ par, int batch) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= batch) return;
  const uint32_t* h = hist1 + (int64_t)b * 256;
  int64_t rl, rh;
  const int bl = select_bin_warp(h, r.rank_lo, &rl);
  const int bh = select_bin_warp(h, r.rank_hi, &rh);
  if ((threadIdx.x & 31) != 0) return;
  if (BPP == 1) {
    finish(&par[b], bl, bh);
  } else {
    sel[b].bin_lo = bl; sel[b].bin_hi = bh; sel[b].rem_lo = rl; sel[b].rem_hi = rh;
  }
}

__global__ void k_select2(const uint32_t* __restrict__ hist2, const SelState* __restrict__ sel,
                          ImgPar* __restrict__ par, int batch) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= batch) return;
  const uint32_t* h = hist2 + (int64_t)b * 512;
  int64_t dummy;
  const int lo = (sel[b].bin_lo << 8) | select_bin_warp(h, sel[b].rem_lo, &dummy);
  const int hi = (sel[b].bin_hi << 8) | select_bin_warp(h + 256, sel[b].rem_hi, &dummy);
  if ((threadIdx.x & 31) == 0) finish(&par[b], lo, hi);
}

// ---------------------------------------------------------------------------------
// f32 input (reading R24): the same nearest ranks on real values by a
// radix select over order-preserving 32-bit keys (sign flipped for positives, all bits
// inverted for negatives), 8 bits per pass, 4 passes.  Pass 0 histograms the top byte
// of every key (one histogram serves both ranks); pass p >= 1 histograms byte 3 - p of
// the keys whose higher bytes equal the prefix selected so far for lo (bins 0..255) and
// for hi (256..511).  The select kernel zeroes the histogram it consumed for the next
// pass.  HBM-bound: 4 B/px read per pass.
__device__ __forceinline__ uint32_t f32_key(uint32_t u) { return (u & 0x80000000u) ? ~u : (u | 0x80000000u); }
__device__ __forceinline__ uint32_t f32_unkey(uint32_t k) { return (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k; }

template <int PASS>
__global__ void __launch_bounds__(256) k_hist_f32(const uint8_t* __restrict__ images, Shape s, int rows_per_cta,
                                                  uint32_t* __restrict__ hist, const SelState* __restrict__ sel) {
  constexpr int NH = PASS == 0 ? 1 : 2;
  constexpr int SH = 24 - 8 * PASS;
  __shared__ uint32_t sh[8][NH * 256];
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * NH * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  uint32_t pl = 0, ph = 0;
  if (PASS > 0) { pl = (uint32_t)sel[b].bin_lo; ph = (uint32_t)sel[b].bin_hi; }
  __syncthreads();
  const uint8_t* img = images + (int64_t)b * s.H * s.pitch;
  const int y0 = blockIdx.x * rows_per_cta;
  const int y1 = min(s.H, y0 + rows_per_cta);
  const int nvec = (s.W + 3) >> 2;
  for (int y = y0; y < y1; ++y) {
    const uint4* row = reinterpret_cast<const uint4*>(img + (int64_t)y * s.pitch);
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
      const uint4 q = __ldg(row + v);
      const uint32_t wds[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (4 * v + k < s.W) {
          const uint32_t key = f32_key(wds[k]);
          const uint32_t bin = (key >> SH) & 255u;
          if (PASS == 0) {
            atomicAdd(&sh[warp][bin], 1u);
          } else {
            const uint32_t pre = key >> ((SH + 8) & 31);   // PASS >= 1: SH + 8 <= 24
            if (pre == pl) atomicAdd(&sh[warp][bin], 1u);
            if (pre == ph) atomicAdd(&sh[warp][256 + bin], 1u);
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NH * 256; i += blockDim.x) {
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += sh[w][i];
    if (c) atomicAdd(&hist[(int64_t)b * 512 + i], c);
  }
}

// one warp per image: extend the lo / hi prefixes by one byte; the last pass writes ImgPar
// (lo/hi as float32 bit patterns, inv = 1/(hi - lo) in f32)
template <int PASS>
__global__ void k_select_f32(uint32_t* __restrict__ hist, RankPar r, SelState* __restrict__ sel,
                             ImgPar* __restrict__ par, int batch) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= batch) return;
  const int lane = threadIdx.x & 31;
  uint32_t* h = hist + (int64_t)b * 512;
  int64_t rl, rh;
  int bl, bh;
  if (PASS == 0) {
    bl = select_bin_warp(h, r.rank_lo, &rl);
    bh = select_bin_warp(h, r.rank_hi, &rh);
  } else {
    bl = select_bin_warp(h, sel[b].rem_lo, &rl);
    bh = select_bin_warp(h + 256, sel[b].rem_hi, &rh);
  }
  __syncwarp();
  for (int i = lane; i < 512; i += 32) h[i] = 0u;   // clean for the next pass / call
  if (lane != 0) return;
  const uint32_t pl = PASS == 0 ? (uint32_t)bl : (((uint32_t)sel[b].bin_lo << 8) | (uint32_t)bl);
  const uint32_t ph = PASS == 0 ? (uint32_t)bh : (((uint32_t)sel[b].bin_hi << 8) | (uint32_t)bh);
  if (PASS < 3) {
    sel[b].bin_lo = (int32_t)pl; sel[b].bin_hi = (int32_t)ph; sel[b].rem_lo = rl; sel[b].rem_hi = rh;
  } else {
    const uint32_t ulo = f32_unkey(pl), uhi = f32_unkey(ph);
    const float lo = __uint_as_float(ulo), hi = __uint_as_float(uhi);
    par[b].lo = (int32_t)ulo;
    par[b].hi = (int32_t)uhi;
    par[b].degen = (hi == lo) ? 1 : 0;
    par[b].inv = (hi == lo) ? 0.0f : 1.0f / (hi - lo);
  }
}

}  // namespace mhfd
