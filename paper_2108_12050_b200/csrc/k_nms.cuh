// k_nms.cuh — scale-space NMS + threshold + ordered stream compaction (rows a7, a8).
//
// PAPER mode (Eq. 3): p is a candidate iff v(p) >= v(q) for every
//   in-image q in its 3x3 neighbourhood (the "comparison against maxpool_2d(3,3)",
//   -inf padding: reading R8; strict: v(p) > v(q), reading R9) and v(p) > tau (R11).
// 26 mode: (p, i) is a candidate iff D_i(p) >= D_j(q) for every existing
//   (q, j) of the 3x3x3 box other than itself (scale window truncated at the first and
//   last plane: reading R16) and D_i(p) > tau.
//
// Compaction: a "segment" is 1024 consecutive pixels in raster order, one per warp.
// k_nms_count writes per-segment candidate counts, k_seg_scan turns them into exclusive
// offsets per image, k_nms_write re-evaluates the predicate and writes records at
// segment offset + warp-ballot prefix.  The list is therefore in (y, x, scale) order
// without a sort and is identical run to run (no atomics decide positions).
#pragma once
#include "common.cuh"

namespace mhfd {

constexpr int kSeg = 1024;

struct NmsArgs {
  int W, H, n;
  float tau;
  int strict;
  const float* v;        // PAPER: B x H x W
  const uint8_t* idx;    // PAPER: B x H x W
  const float* dog;      // 26:    B x n x H x W
};

__device__ __forceinline__ bool dominates(float c, float q, int strict) { return strict ? (c > q) : (c >= q); }

__device__ __forceinline__ bool paper_cand(const float* __restrict__ v, int W, int H, int y, int x, float tau,
                                           int strict, float* val) {
  const float c = __ldg(v + (int64_t)y * W + x);
  *val = c;
  if (!(c > tau)) return false;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
    const int yy = y + dy;
    if (yy < 0 || yy >= H) continue;
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      if (dy == 0 && dx == 0) continue;
      const int xx = x + dx;
      if (xx < 0 || xx >= W) continue;
      // a NaN neighbour is skipped, as the count passes' fmaxf column-max chain skips it,
      // so the count and the write/re-evaluation predicates agree for every input (v is
      // NaN-free anyway: the stretch clamps, and a NaN centre fails c > tau in both)
      const float q = __ldg(v + (int64_t)yy * W + xx);
      if (q == q && !dominates(c, q, strict)) return false;
    }
  }
  return true;
}

__device__ __forceinline__ bool cand26(const float* __restrict__ dog, int W, int H, int n, int64_t plane, int i,
                                       int y, int x, float tau, int strict, float* val) {
  const float c = __ldg(dog + (int64_t)i * plane + (int64_t)y * W + x);
  *val = c;
  if (!(c > tau)) return false;
  for (int di = -1; di <= 1; ++di) {
    const int j = i + di;
    if (j < 0 || j >= n) continue;
    const float* P = dog + (int64_t)j * plane;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int yy = y + dy;
      if (yy < 0 || yy >= H) continue;
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        if (di == 0 && dy == 0 && dx == 0) continue;
        const int xx = x + dx;
        if (xx < 0 || xx >= W) continue;
        const float q = __ldg(P + (int64_t)yy * W + xx);   // NaN skipped, as in paper_cand
        if (q == q && !dominates(c, q, strict)) return false;
      }
    }
  }
  return true;
}

// Number of candidates at pixel p (0/1 in PAPER mode, 0..n in 26 mode); optionally
// writes them (in scale order) to out[].
template <int MODE>
__device__ __forceinline__ int pixel_cands(const NmsArgs& a, int b, int64_t p, mhfd_blob* out, int64_t base,
                                           int64_t cap) {
  const int64_t plane = (int64_t)a.H * a.W;
  const int y = (int)(p / a.W), x = (int)(p - (int64_t)y * a.W);
  int c = 0;
  if (MODE == MHFD_NMS_PAPER) {
    float val;
    if (paper_cand(a.v + (int64_t)b * plane, a.W, a.H, y, x, a.tau, a.strict, &val)) {
      if (out && base < cap) {
        mhfd_blob r;
        r.x = x; r.y = y; r.scale = a.idx[(int64_t)b * plane + p]; r.response = val;
        out[base] = r;
      }
      c = 1;
    }
  } else {
    const float* dog = a.dog + (int64_t)b * a.n * plane;
    for (int i = 0; i < a.n; ++i) {
      float val;
      if (cand26(dog, a.W, a.H, a.n, plane, i, y, x, a.tau, a.strict, &val)) {
        if (out && base + c < cap) {
          mhfd_blob r;
          r.x = x; r.y = y; r.scale = i; r.response = val;
          out[base + c] = r;
        }
        ++c;
      }
    }
  }
  return c;
}

// grid (ceil(nseg/8), B), 256 threads: warp w of CTA t owns segment 8t + w.
template <int MODE>
__global__ void __launch_bounds__(256) k_nms_count(NmsArgs a, int nseg, int32_t* __restrict__ segcnt) {
  const int b = blockIdx.y;
  const int seg = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (seg >= nseg) return;
  const int64_t plane = (int64_t)a.H * a.W;
  const int64_t p0 = (int64_t)seg * kSeg;
  int cnt = 0;
  for (int k = 0; k < kSeg; k += 32) {
    const int64_t p = p0 + k + lane;
    int c = (p < plane) ? pixel_cands<MODE>(a, b, p, nullptr, 0, 0) : 0;
    cnt += c;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  if (lane == 0) segcnt[(int64_t)b * nseg + seg] = cnt;
}

// One CTA (1024 threads) per image: exclusive scan of the segment counts.  Warp w owns a
// contiguous block of ceil(nseg / 1024) x 32 counts and walks it 32 at a time (coalesced
// loads, a warp scan per step, a running carry), the 32 warp totals are scanned once,
// and the block's offsets are written in a second coalesced walk.  (Round 1's 1024-wide
// loop with four barriers per step took 17 us for the 16384 segments of a 4096^2 tile;
// per-thread contiguous runs were uncoalesced and no faster.)
__global__ void __launch_bounds__(1024) k_seg_scan(const int32_t* __restrict__ segcnt, int nseg,
                                                   int32_t* __restrict__ segoff, int32_t* __restrict__ ncand) {
  __shared__ int32_t wsum[32];
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = ((nseg + 1023) / 1024) * 32;   // counts per warp (multiple of 32)
  const int i0 = min(nseg, warp * per), i1 = min(nseg, i0 + per);
  const int32_t* sc = segcnt + (int64_t)b * nseg;
  int32_t* so = segoff + (int64_t)b * nseg;
  int tot = 0;
#pragma unroll 4
  for (int i = i0 + lane; i - lane < i1; i += 32) tot += i < i1 ? __ldg(sc + i) : 0;
#pragma unroll
  for (int off = 16; off; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
  if (lane == 0) wsum[warp] = tot;
  __syncthreads();
  if (warp == 0) {
    const int v = wsum[lane];
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    wsum[lane] = x - v;   // exclusive
    if (lane == 31) ncand[b] = x;
  }
  __syncthreads();
  int carry = wsum[warp];
  for (int i = i0 + lane; i - lane < i1; i += 32) {
    const int v = i < i1 ? __ldg(sc + i) : 0;
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (i < i1) so[i] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_nms_write(NmsArgs a, int nseg, const int32_t* __restrict__ segoff,
                                                   mhfd_blob* __restrict__ cand, int64_t cap) {
  const int b = blockIdx.y;
  const int seg = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (seg >= nseg) return;
  const int64_t plane = (int64_t)a.H * a.W;
  const int64_t p0 = (int64_t)seg * kSeg;
  int64_t off = segoff[(int64_t)b * nseg + seg];
  mhfd_blob* out = cand + (int64_t)b * cap;
  for (int k = 0; k < kSeg; k += 32) {
    const int64_t p = p0 + k + lane;
    if (MODE == MHFD_NMS_PAPER) {
      float val = 0.f;
      bool c = false;
      int y = 0, x = 0;
      if (p < plane) {
        y = (int)(p / a.W); x = (int)(p - (int64_t)y * a.W);
        c = paper_cand(a.v + (int64_t)b * plane, a.W, a.H, y, x, a.tau, a.strict, &val);
      }
      const uint32_t m = __ballot_sync(0xffffffffu, c);
      if (c) {
        const int64_t pos = off + __popc(m & ((1u << lane) - 1u));
        if (pos < cap) {
          mhfd_blob r;
          r.x = x; r.y = y; r.scale = a.idx[(int64_t)b * plane + p]; r.response = val;
          out[pos] = r;
        }
      }
      off += __popc(m);
    } else {
      const int c = (p < plane) ? pixel_cands<MODE>(a, b, p, nullptr, 0, 0) : 0;
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (c) pixel_cands<MODE>(a, b, p, out, off + x - c, cap);
      off += __shfl_sync(0xffffffffu, x, 31);
    }
  }
}

}  // namespace mhfd

namespace mhfd {

// Row-segment fast path of the Eq. 3 NMS (PAPER mode) for W % kSeg == 0: a warp owns
// kNmsRows vertically adjacent 1024-pixel segments and walks them in 4 steps of 256 pixels; lane l holds
// pixels 8l .. 8l+7 of the step for the row and its two neighbours (two 128-bit loads
// each), gets the outer neighbours from lanes l-1 / l+1 by shuffles, and the candidates
// of a step come out lane-major, i.e. in raster order.  Same predicate and same
// segment bookkeeping as k_nms_count / k_nms_write.
constexpr int kNmsRows = 2;   // output rows per warp in k_nms_rows (4: 2.98 ms, 2: 2.77 ms per 64 images)

constexpr int kSlab = 64;    // records a segment parks in its slab during the count pass (32 -> 64: a sharp
                             // 4096^2 tile had enough overflowing segments to make the gather's re-evaluation 60 us)

template <bool WRITE>
__global__ void __launch_bounds__(256, 4) k_nms_rows(NmsArgs a, int nseg, int32_t* __restrict__ segcnt,
                                                  const int32_t* __restrict__ segoff, mhfd_blob* __restrict__ cand,
                                                  int64_t cap, int row0, int row1,
                                                  mhfd_blob* __restrict__ slab = nullptr) {
  // a warp owns kNmsRows vertically adjacent 1024-pixel segments (rows y0.., piece xs):
  // kNmsRows + 2 rows are loaded per step, so each v row leaves L2 1.5 times, not 3
  constexpr int NR = kNmsRows;
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int W = a.W, H = a.H;
  const int spr = W / kSeg;                                   // segments per row
  // output rows [row0, row1) (the image, or one band of it; neighbours come from v
  // rows row0-1 and row1, which the caller has computed); segments are numbered from row0
  const int grp = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int ngrp = ((row1 - row0 + NR - 1) / NR) * spr;
  if (grp >= ngrp) return;
  const int y0 = row0 + NR * (grp / spr);
  const int xseg = (grp % spr) * kSeg;
  const float* vb = a.v + (int64_t)b * H * W;
  const float* rows[NR + 2];
#pragma unroll
  for (int k = 0; k < NR + 2; ++k) {
    const int y = y0 - 1 + k;
    rows[k] = (y >= 0 && y < H) ? vb + (int64_t)y * W : nullptr;
  }
  const float NEG = -INFINITY;
  const int seg0 = ((y0 - row0) * W + xseg) / kSeg;
  int64_t off[NR];
  int total[NR], parked[NR];
#pragma unroll
  for (int o = 0; o < NR; ++o) {
    off[o] = (WRITE && y0 + o < row1) ? (int64_t)segoff[(int64_t)b * nseg + seg0 + o * spr] : 0;
    total[o] = 0;
    parked[o] = 0;
  }
  mhfd_blob* out = WRITE ? cand + (int64_t)b * cap : nullptr;
  const uint8_t* ib = a.idx + (int64_t)b * H * W;
  for (int step = 0; step < kSeg / 256; ++step) {
    const int x = xseg + step * 256 + 8 * lane;
    float R[NR + 2][10];
#pragma unroll
    for (int k = 0; k < NR + 2; ++k) {
      if (rows[k]) {
        const float4 p0 = __ldg(reinterpret_cast<const float4*>(rows[k] + x));
        const float4 p1 = __ldg(reinterpret_cast<const float4*>(rows[k] + x + 4));
        R[k][1] = p0.x; R[k][2] = p0.y; R[k][3] = p0.z; R[k][4] = p0.w;
        R[k][5] = p1.x; R[k][6] = p1.y; R[k][7] = p1.z; R[k][8] = p1.w;
      } else {
#pragma unroll
        for (int j = 1; j < 9; ++j) R[k][j] = NEG;
      }
    }
#pragma unroll
    for (int k = 0; k < NR + 2; ++k) {
      R[k][0] = __shfl_up_sync(0xffffffffu, R[k][8], 1);
      R[k][9] = __shfl_down_sync(0xffffffffu, R[k][1], 1);
    }
    if (lane == 0) {
      const bool in = x > 0;
#pragma unroll
      for (int k = 0; k < NR + 2; ++k) R[k][0] = (in && rows[k]) ? __ldg(rows[k] + x - 1) : NEG;
    }
    if (lane == 31) {
      const bool in = x + 8 < W;
#pragma unroll
      for (int k = 0; k < NR + 2; ++k) R[k][9] = (in && rows[k]) ? __ldg(rows[k] + x + 8) : NEG;
    }
#pragma unroll
    for (int o = 0; o < NR; ++o) {
      const float* u = R[o];
      const float* c = R[o + 1];
      const float* d = R[o + 2];
      uint32_t bb = 0;
#pragma unroll
      for (int k = 1; k < 9; ++k) {
        const float m = fmaxf(fmaxf(fmaxf(u[k - 1], u[k]), fmaxf(u[k + 1], c[k - 1])),
                              fmaxf(fmaxf(c[k + 1], d[k - 1]), fmaxf(d[k], d[k + 1])));
        const bool ok = (c[k] > a.tau) && (a.strict ? (c[k] > m) : (c[k] >= m));
        bb |= (uint32_t)ok << (k - 1);
      }
      if (y0 + o >= row1) bb = 0u;
      const int n = __popc(bb);
      if (!WRITE && slab) {   // park this step's records in the segment's slab (raster order)
        int incl = n;
#pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, sh);
          if (lane >= sh) incl += t;
        }
        int pos = parked[o] + incl - n;   // segment-wide running position
        parked[o] += __shfl_sync(0xffffffffu, incl, 31);
        const int y = y0 + o;
        const uint8_t* irow = ib + (int64_t)y * W;
        mhfd_blob* sl = slab + ((int64_t)b * nseg + seg0 + o * spr) * kSlab;
        uint32_t m = bb;
        while (m) {
          const int k = __ffs(m) - 1;
          m &= m - 1;
          if (pos < kSlab) {
            mhfd_blob r;
            r.x = x + k; r.y = y; r.scale = irow[x + k]; r.response = __ldg(rows[o + 1] + x + k);
            sl[pos] = r;
          }
          ++pos;
        }
      }
      if (WRITE) {
        int incl = n;
#pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, sh);
          if (lane >= sh) incl += t;
        }
        int64_t pos = off[o] + incl - n;
        const int y = y0 + o;
        const uint8_t* irow = ib + (int64_t)y * W;
        while (bb) {
          const int k = __ffs(bb) - 1;
          bb &= bb - 1;
          if (pos < cap) {
            mhfd_blob r;
            r.x = x + k; r.y = y; r.scale = irow[x + k]; r.response = __ldg(rows[o + 1] + x + k);
            out[pos] = r;
          }
          ++pos;
        }
        off[o] += __shfl_sync(0xffffffffu, incl, 31);
      } else {
        total[o] += n;
      }
    }
  }
  if (!WRITE) {
#pragma unroll
    for (int o = 0; o < NR; ++o) {
      int t = total[o];
#pragma unroll
      for (int sh = 16; sh; sh >>= 1) t += __shfl_xor_sync(0xffffffffu, t, sh);
      if (lane == 0 && y0 + o < row1) segcnt[(int64_t)b * nseg + seg0 + o * spr] = t;
    }
  }
}

// Rolling-window variant of k_nms_rows (count + park pass only): a warp owns NR
// vertically adjacent 1024-pixel segments and, per 256-pixel step, walks down its NR
// rows holding three v rows (with their shuffled halos) plus the next row in flight, so
// NR + 2 rows are loaded for NR output rows (1.25x at NR = 8, against 2x at kNmsRows = 2)
// with four rows live instead of NR + 2.  Same predicate, same slabs and counts, so
// k_seg_scan / k_nms_gather are unchanged.
struct NmsRow {
  float v[10];
};

__device__ __forceinline__ NmsRow nms_load_row(const float* __restrict__ row, int x, int W, int lane) {
  NmsRow r;
  if (row) {
    const float4 p0 = __ldg(reinterpret_cast<const float4*>(row + x));
    const float4 p1 = __ldg(reinterpret_cast<const float4*>(row + x + 4));
    r.v[1] = p0.x; r.v[2] = p0.y; r.v[3] = p0.z; r.v[4] = p0.w;
    r.v[5] = p1.x; r.v[6] = p1.y; r.v[7] = p1.z; r.v[8] = p1.w;
    r.v[0] = (lane == 0) ? (x > 0 ? __ldg(row + x - 1) : -INFINITY) : 0.f;
    r.v[9] = (lane == 31) ? (x + 8 < W ? __ldg(row + x + 8) : -INFINITY) : 0.f;
  } else {
#pragma unroll
    for (int j = 0; j < 10; ++j) r.v[j] = -INFINITY;
  }
  return r;
}

__device__ __forceinline__ void nms_halo(NmsRow& r, int lane) {
  const float up = __shfl_up_sync(0xffffffffu, r.v[8], 1);
  const float dn = __shfl_down_sync(0xffffffffu, r.v[1], 1);
  if (lane != 0) r.v[0] = up;
  if (lane != 31) r.v[9] = dn;
}

// Interior warps of k_nms_roll (all NR + 2 rows inside the image, NR output rows): no
// per-row validity tests, a pointer walk down the rows, and a fully unrolled row loop
// without early exits, so the three live rows rotate by renaming instead of ~60
// register moves per row (ncu: the generic loop issued ~250 instructions per 8-pixel
// row step, a quarter of them IMAD.MOV).
#ifndef NMS_FAST
#define NMS_FAST 1
#endif
template <int NR>
__device__ __forceinline__ void nms_roll_fast(const NmsArgs& a, const float* __restrict__ vb,
                                              const uint8_t* __restrict__ ib, int y0, int xseg, int lane,
                                              mhfd_blob* __restrict__ sl0, int spr, int& parked) {
  const int W = a.W;
  const float tau = a.tau;
  const bool strict = a.strict != 0;
  auto load = [&](const float* q, bool lft, bool rgt, float (&r)[10]) {
    const float4 p0 = __ldg(reinterpret_cast<const float4*>(q));
    const float4 p1 = __ldg(reinterpret_cast<const float4*>(q + 4));
    r[1] = p0.x; r[2] = p0.y; r[3] = p0.z; r[4] = p0.w;
    r[5] = p1.x; r[6] = p1.y; r[7] = p1.z; r[8] = p1.w;
    r[0] = lft ? __ldg(q - 1) : -INFINITY;   // lane 0 only (others take the shuffle)
    r[9] = rgt ? __ldg(q + 8) : -INFINITY;   // lane 31 only
  };
  auto halo = [&](float (&r)[10]) {
    const float up = __shfl_up_sync(0xffffffffu, r[8], 1);
    const float dn = __shfl_down_sync(0xffffffffu, r[1], 1);
    if (lane != 0) r[0] = up;
    if (lane != 31) r[9] = dn;
  };
#pragma unroll 1
  for (int step = 0; step < kSeg / 256; ++step) {
    const int x = xseg + step * 256 + 8 * lane;
    const bool lft = lane == 0 && x > 0, rgt = lane == 31 && x + 8 < W;
    const float* q = vb + (int64_t)(y0 - 1) * W + x;
    float u[10], c[10], d[10];
    load(q, lft, rgt, u);
    load(q + W, lft, rgt, c);
    load(q + 2 * W, lft, rgt, d);
    halo(u);
    halo(c);
#pragma unroll
    for (int o = 0; o < NR; ++o) {
      float nx[10];
      if (o + 1 < NR) load(q + (int64_t)(o + 3) * W, lft, rgt, nx);
      halo(d);
      float V[10];
#pragma unroll
      for (int j = 0; j < 10; ++j) V[j] = fmaxf(u[j], d[j]);
      uint32_t bb = 0;
#pragma unroll
      for (int k = 1; k < 9; ++k) {
        const float m = fmaxf(fmaxf(V[k - 1], V[k]), fmaxf(V[k + 1], fmaxf(c[k - 1], c[k + 1])));
        const bool ok = (c[k] > tau) && (strict ? (c[k] > m) : (c[k] >= m));
        bb |= (uint32_t)ok << (k - 1);
      }
      const int n = __popc(bb);
      int incl = n;
#pragma unroll
      for (int sh = 1; sh < 32; sh <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, sh);
        if (lane >= sh) incl += t;
      }
      int pos = __shfl_sync(0xffffffffu, parked, o) + incl - n;
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == o) parked += tot;
      if (bb) {
        const int y = y0 + o;
        const uint8_t* irow = ib + (int64_t)y * W;
        mhfd_blob* sl = sl0 + (int64_t)o * spr * kSlab;
        uint32_t m = bb;
        while (m) {
          const int k = __ffs(m) - 1;
          m &= m - 1;
          if (pos < kSlab) {
            mhfd_blob r;
            r.x = x + k; r.y = y; r.scale = irow[x + k]; r.response = c[1 + k];
            sl[pos] = r;
          }
          ++pos;
        }
      }
#pragma unroll
      for (int j = 0; j < 10; ++j) {
        u[j] = c[j];
        c[j] = d[j];
        if (o + 1 < NR) d[j] = nx[j];
      }
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(256, NR <= 2 ? 4 : 3) k_nms_roll(NmsArgs a, int nseg, int32_t* __restrict__ segcnt, int row0,
                                                    int row1, mhfd_blob* __restrict__ slab) {
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int W = a.W, H = a.H;
  const int spr = W / kSeg;
  const int grp = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int ngrp = ((row1 - row0 + NR - 1) / NR) * spr;
  if (grp >= ngrp) return;
  const int y0 = row0 + NR * (grp / spr);
  const int xseg = (grp % spr) * kSeg;
  const float* vb = a.v + (int64_t)b * H * W;
  const uint8_t* ib = a.idx + (int64_t)b * H * W;
  const int seg0 = ((y0 - row0) * W + xseg) / kSeg;
  const int nrow = min(NR, row1 - y0);   // output rows of this warp (ragged last group)
  auto rowp = [&](int y) -> const float* { return (y >= 0 && y < H) ? vb + (int64_t)y * W : nullptr; };
  int parked = 0;   // lane o holds the running count of segment o (NR <= 32)
  if (NMS_FAST && nrow == NR && y0 >= 1 && y0 + NR < H) {   // warp-uniform
    nms_roll_fast<NR>(a, vb, ib, y0, xseg, lane, slab + ((int64_t)b * nseg + seg0) * kSlab, spr, parked);
    if (lane < nrow) segcnt[(int64_t)b * nseg + seg0 + lane * spr] = parked;
    return;
  }
  for (int step = 0; step < kSeg / 256; ++step) {
    const int x = xseg + step * 256 + 8 * lane;
    NmsRow u = nms_load_row(rowp(y0 - 1), x, W, lane);
    NmsRow c = nms_load_row(rowp(y0), x, W, lane);
    NmsRow d = nms_load_row(rowp(y0 + 1), x, W, lane);
    nms_halo(u, lane);
    nms_halo(c, lane);
#pragma unroll
    for (int o = 0; o < NR; ++o) {
      if (o >= nrow) break;
      NmsRow nx;
      if (o + 1 < nrow) nx = nms_load_row(rowp(y0 + o + 2), x, W, lane);   // in flight during this row
      nms_halo(d, lane);
      // the 8-neighbour max through the column max V = max(u, d): 10 + 4 per pixel
      // fmax instead of 7 per pixel (max is exact, so the predicate is unchanged)
      float V[10];
#pragma unroll
      for (int j = 0; j < 10; ++j) V[j] = fmaxf(u.v[j], d.v[j]);
      uint32_t bb = 0;
#pragma unroll
      for (int k = 1; k < 9; ++k) {
        const float m = fmaxf(fmaxf(V[k - 1], V[k]), fmaxf(V[k + 1], fmaxf(c.v[k - 1], c.v[k + 1])));
        const bool ok = (c.v[k] > a.tau) && (a.strict ? (c.v[k] > m) : (c.v[k] >= m));
        bb |= (uint32_t)ok << (k - 1);
      }
      const int n = __popc(bb);
      int incl = n;
#pragma unroll
      for (int sh = 1; sh < 32; sh <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, sh);
        if (lane >= sh) incl += t;
      }
      int pos = __shfl_sync(0xffffffffu, parked, o) + incl - n;
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == o) parked += tot;
      if (bb) {
        const int y = y0 + o;
        const uint8_t* irow = ib + (int64_t)y * W;
        mhfd_blob* sl = slab + ((int64_t)b * nseg + seg0 + o * spr) * kSlab;
        uint32_t m = bb;
        while (m) {
          const int k = __ffs(m) - 1;
          m &= m - 1;
          if (pos < kSlab) {
            mhfd_blob r;
            r.x = x + k; r.y = y; r.scale = irow[x + k]; r.response = __ldg(vb + (int64_t)y * W + x + k);
            sl[pos] = r;
          }
          ++pos;
        }
      }
      u = c;
      c = d;
      d = nx;
    }
  }
  if (lane < nrow) segcnt[(int64_t)b * nseg + seg0 + lane * spr] = parked;
}

// 26-neighbour mode (readings R8, R16), count + park pass for widths that
// are whole 1024-pixel segments: one warp per (row y, segment), 8 pixels per lane per
// 256-pixel step.  The scale loop keeps, per pixel, D_i, the max of its 8 spatial
// neighbours in plane i (M8_i) and the 3 x 3 max of plane i-1 (M9_{i-1}); plane i+1's
// three rows are loaded while plane i is decided: (p, i) is a candidate iff D_i > tau and
// D_i >= max(M8_i, M9_{i-1}, M9_{i+1}) (> when strict), with -inf outside the image and
// no plane beyond the first / last — cand26's rule (the maxima skip NaN, as cand26 does).
// Each plane's rows are read once per output row (3 row loads per plane, the neighbouring
// rows from L1/L2) instead of 27 scattered loads per (pixel, plane) in both passes of the
// generic kernels.  Records go to the segment's slab in (x, scale) order; k_seg_scan and
// k_nms_gather4<MHFD_NMS_26> (overflowing segments re-evaluated with cand26) follow.
// 4 CTAs per SM (64-register cap, a few bytes of spills): the kernel is latency-bound
// (35 % warps active at 78 registers); 0.342 -> 0.327 ms per 4096^2 image batched
__global__ void __launch_bounds__(256, 4) k_nms26_roll(NmsArgs a, int nseg, int32_t* __restrict__ segcnt, int row0,
                                                    int row1, mhfd_blob* __restrict__ slab) {
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int W = a.W, H = a.H, n = a.n;
  const int spr = W / kSeg;
  const int grp = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (grp >= (row1 - row0) * spr) return;
  const int y = row0 + grp / spr;
  const int xseg = (grp % spr) * kSeg;
  const int seg = ((y - row0) * W + xseg) / kSeg;
  const int64_t plane = (int64_t)H * W;
  const float* dog = a.dog + (int64_t)b * n * plane;
  const float tau = a.tau;
  const bool strict = a.strict != 0;
  const bool up = y >= 1, dn = y + 1 < H;
  mhfd_blob* sl = slab + ((int64_t)b * nseg + seg) * kSlab;
  int parked = 0;
  for (int step = 0; step < kSeg / 256; ++step) {
    const int x = xseg + step * 256 + 8 * lane;
    const bool lft = lane == 0 && x > 0, rgt = lane == 31 && x + 8 < W;
    // plane j's centre row (8 values) and the max of its 8 spatial neighbours (M8)
    auto load_plane = [&](int j, float (&c)[8], float (&m8)[8]) {
      const float* q = dog + (int64_t)j * plane + (int64_t)y * W + x;
      float u[10], cc[10], d[10];
      auto ld = [&](const float* r, bool ok, float (&o)[10]) {
        if (ok) {
          const float4 p0 = __ldg(reinterpret_cast<const float4*>(r));
          const float4 p1 = __ldg(reinterpret_cast<const float4*>(r + 4));
          o[1] = p0.x; o[2] = p0.y; o[3] = p0.z; o[4] = p0.w;
          o[5] = p1.x; o[6] = p1.y; o[7] = p1.z; o[8] = p1.w;
          o[0] = lft ? __ldg(r - 1) : -INFINITY;
          o[9] = rgt ? __ldg(r + 8) : -INFINITY;
        } else {
#pragma unroll
          for (int k = 0; k < 10; ++k) o[k] = -INFINITY;
        }
        const float hu = __shfl_up_sync(0xffffffffu, o[8], 1);
        const float hd = __shfl_down_sync(0xffffffffu, o[1], 1);
        if (lane != 0) o[0] = hu;
        if (lane != 31) o[9] = hd;
      };
      ld(q - W, up, u);
      ld(q, true, cc);
      ld(q + W, dn, d);
      float V[10];
#pragma unroll
      for (int k = 0; k < 10; ++k) V[k] = fmaxf(u[k], d[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        c[k] = cc[k + 1];
        m8[k] = fmaxf(fmaxf(V[k], V[k + 1]), fmaxf(V[k + 2], fmaxf(cc[k], cc[k + 2])));
      }
    };
    float c0[8], m80[8], m9p[8];
    uint32_t bits[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      m9p[k] = -INFINITY;
      bits[k] = 0u;
    }
    load_plane(0, c0, m80);
    for (int i = 0; i < n; ++i) {
      float c1[8], m81[8];
      if (i + 1 < n) {
        load_plane(i + 1, c1, m81);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) c1[k] = m81[k] = -INFINITY;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float m = fmaxf(m80[k], fmaxf(m9p[k], fmaxf(m81[k], c1[k])));   // 26 neighbours
        const bool ok = (c0[k] > tau) && (strict ? (c0[k] > m) : (c0[k] >= m));
        bits[k] |= (uint32_t)ok << i;
        m9p[k] = fmaxf(m80[k], c0[k]);
        c0[k] = c1[k];
        m80[k] = m81[k];
      }
    }
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) cnt += __popc(bits[k]);
    int incl = cnt;
#pragma unroll
    for (int sh = 1; sh < 32; sh <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, sh);
      if (lane >= sh) incl += t;
    }
    int pos = parked + incl - cnt;
    parked += __shfl_sync(0xffffffffu, incl, 31);
    if (cnt) {
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        uint32_t m = bits[k];
        while (m) {
          const int i = __ffs(m) - 1;
          m &= m - 1;
          if (pos < kSlab) {
            mhfd_blob r;
            r.x = x + k; r.y = y; r.scale = i;
            r.response = __ldg(dog + (int64_t)i * plane + (int64_t)y * W + x + k);
            sl[pos] = r;
          }
          ++pos;
        }
      }
    }
  }
  if (lane == 0) segcnt[(int64_t)b * nseg + seg] = parked;
}

// Gather after the scan: one warp per segment copies its parked records to its final
// offset; a segment with more than kSlab candidates (its slab overflowed) re-evaluates
// its 1024 pixels with the full predicate instead (same records, same order).
__global__ void __launch_bounds__(256) k_nms_gather(NmsArgs a, int nseg, const int32_t* __restrict__ segcnt,
                                                    const int32_t* __restrict__ segoff,
                                                    const mhfd_blob* __restrict__ slab, mhfd_blob* __restrict__ cand,
                                                    int64_t cap, int row0) {
  const int b = blockIdx.y;
  const int seg = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (seg >= nseg) return;
  const int cnt = segcnt[(int64_t)b * nseg + seg];
  int64_t off = segoff[(int64_t)b * nseg + seg];
  mhfd_blob* out = cand + (int64_t)b * cap;
  if (cnt <= kSlab) {
    for (int r = lane; r < cnt; r += 32)
      if (off + r < cap) out[off + r] = slab[((int64_t)b * nseg + seg) * kSlab + r];
    return;
  }
  const int64_t plane = (int64_t)a.H * a.W;
  const int64_t p0 = (int64_t)row0 * a.W + (int64_t)seg * kSeg;
  for (int k = 0; k < kSeg; k += 32) {
    const int64_t p = p0 + k + lane;
    const int y = (int)(p / a.W), x = (int)(p - (int64_t)y * a.W);
    float val = 0.f;
    const bool c = paper_cand(a.v + (int64_t)b * plane, a.W, a.H, y, x, a.tau, a.strict, &val);
    const uint32_t m = __ballot_sync(0xffffffffu, c);
    if (c) {
      const int64_t pos = off + __popc(m & ((1u << lane) - 1u));
      if (pos < cap) {
        mhfd_blob r;
        r.x = x; r.y = y; r.scale = a.idx[(int64_t)b * plane + p]; r.response = val;
        out[pos] = r;
      }
    }
    off += __popc(m);
  }
}

// The same gather with four segments per warp (eight lanes per segment; a segment parks
// ~5 records on the C4 tiles, so a warp per segment left most lanes idle): parked
// records are copied by the segment's eight lanes; each overflowing segment is then
// re-evaluated by the whole warp as in k_nms_gather.
template <int MODE = MHFD_NMS_PAPER>
__global__ void __launch_bounds__(256) k_nms_gather4(NmsArgs a, int nseg, const int32_t* __restrict__ segcnt,
                                                     const int32_t* __restrict__ segoff,
                                                     const mhfd_blob* __restrict__ slab, mhfd_blob* __restrict__ cand,
                                                     int64_t cap, int row0) {
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int seg_base = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 4;
  if (seg_base >= nseg) return;
  const int seg = seg_base + (lane >> 3), j = lane & 7;
  const bool in = seg < nseg;
  const int cnt = in ? segcnt[(int64_t)b * nseg + seg] : 0;
  const int64_t off0 = in ? segoff[(int64_t)b * nseg + seg] : 0;
  mhfd_blob* out = cand + (int64_t)b * cap;
  if (cnt <= kSlab) {
    const mhfd_blob* sl = slab + ((int64_t)b * nseg + seg) * kSlab;
    for (int r = j; r < cnt; r += 8)
      if (off0 + r < cap) out[off0 + r] = sl[r];
  }
  uint32_t over = __ballot_sync(0xffffffffu, in && j == 0 && cnt > kSlab);
  const int64_t plane = (int64_t)a.H * a.W;
  while (over) {
    const int src = __ffs(over) - 1;
    over &= over - 1;
    const int s2 = seg_base + (src >> 3);
    int64_t off = __shfl_sync(0xffffffffu, off0, src);
    const int64_t p0 = (int64_t)row0 * a.W + (int64_t)s2 * kSeg;
    if (MODE == MHFD_NMS_26) {   // 0..n candidates per pixel, written in (x, scale) order
      for (int k = 0; k < kSeg; k += 32) {
        const int64_t p = p0 + k + lane;
        const int cnt = pixel_cands<MHFD_NMS_26>(a, b, p, nullptr, 0, 0);
        int incl = cnt;
#pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, sh);
          if (lane >= sh) incl += t;
        }
        if (cnt) pixel_cands<MHFD_NMS_26>(a, b, p, out, off + incl - cnt, cap);
        off += __shfl_sync(0xffffffffu, incl, 31);
      }
    } else {
      for (int k = 0; k < kSeg; k += 32) {
        const int64_t p = p0 + k + lane;
        const int y = (int)(p / a.W), x = (int)(p - (int64_t)y * a.W);
        float val = 0.f;
        const bool c = paper_cand(a.v + (int64_t)b * plane, a.W, a.H, y, x, a.tau, a.strict, &val);
        const uint32_t m = __ballot_sync(0xffffffffu, c);
        if (c) {
          const int64_t pos = off + __popc(m & ((1u << lane) - 1u));
          if (pos < cap) {
            mhfd_blob r;
            r.x = x; r.y = y; r.scale = a.idx[(int64_t)b * plane + p]; r.response = val;
            out[pos] = r;
          }
        }
        off += __popc(m);
      }
    }
  }
}

}  // namespace mhfd
