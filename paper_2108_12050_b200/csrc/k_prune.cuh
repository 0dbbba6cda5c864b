// k_prune.cuh — blob-overlap pruning, focus score and ordered output (rows a9, a10).
//
// Not in the paper: the north star's "blob-overlap pruning" (reading R12).  A blob of
// DoG plane s has radius r_s = sqrt(2) t_s; the overlap fraction of two blobs is the
// lens area of their disks over the area of the smaller disk.  Semantics = greedy in
// priority order (scale descending, then raster ascending): a blob is kept iff no kept,
// higher-priority blob overlaps it by more than `overlap`.
//
// Parallel equivalent (exact, not an approximation): every blob starts UNDECIDED; in a
// round, an undecided blob becomes REMOVED if some higher-priority overlapping blob is
// KEPT, KEPT if all of them are REMOVED, and stays UNDECIDED otherwise.  Each decision
// is final and equals the sequential one (induction on priority), and the highest-
// priority undecided blob always decides, so the rounds terminate (<= 10
// rounds on EM tiles).  One cooperative launch runs all rounds for the whole batch,
// separated by grid-wide barriers; candidates are looked up through a per-row index
// of the raster-sorted candidate list.
//
// Score: DOF = |C| after pruning.  The kept list is emitted in
// (y, x, scale) order by a chunked scan (no atomics decide positions).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace mhfd {

namespace cg = cooperative_groups;

constexpr uint8_t kUndecided = 0, kKept = 1, kRemoved = 2;
constexpr int kChunk = 256;

struct PruneArgs {
  int B, W, H;
  int64_t cap;              // candidate capacity per image
  const mhfd_blob* cand;    // B x cap, raster order
  const int32_t* ncand;     // exact candidate counts
  double overlap;
  int prune;                // overlap < 1
  double radmax;
  double rad[kMaxLevels];   // sqrt(2) * t_s
  int32_t dmax[kMaxLevels]; // search radius of a plane-s blob: ceil(sqrt(max_{s'>=s} thr_hi(s, s')))
  const float2* thr;        // n x n squared-distance band (lo, hi) of frac > overlap (host bisection)
  int n;                    // DoG planes
  uint8_t* st;              // B x cap
  int32_t* rowstart;        // B x (H + 1): first candidate of each row
  int32_t* rbi;             // B x H x (nbx + 1): first candidate of row y with x >= 32 k
  int nbx;                  // ceil(W / 32)
  int64_t* img_off;         // B + 1: prefix of effective candidate counts
  int64_t* chunk_off;       // B + 1: prefix of chunk counts
  int32_t* chunk_cnt;       // kept per chunk
  int32_t* chunk_pos;       // exclusive kept offsets per chunk (within the image)
  int32_t* counters;        // 8 ints: undecided counters (3), round count, worklist length
  int4* wl;                 // worklist of blobs undecided after round 0: 2 int4 per record
                            // {k_global, cnt, q0, q1}, {q2, q3, q4, q5}; cnt = kNbMax + 1: list overflow
  int64_t wl_cap;           // records
  mhfd_blob* blobs;         // nullable: B x blob_cap output
  int32_t blob_cap;
  int32_t* counts;          // nullable
  double* scores;           // nullable
  int32_t* flags;           // nullable
};

__device__ __forceinline__ double lens_fraction(double d, double r1, double r2) {
  const double rmin = fmin(r1, r2);
  if (d >= r1 + r2) return 0.0;
  if (d <= fabs(r1 - r2)) return 1.0;
  double a1 = (d * d + r1 * r1 - r2 * r2) / (2.0 * d * r1);
  double a2 = (d * d + r2 * r2 - r1 * r1) / (2.0 * d * r2);
  a1 = fmin(1.0, fmax(-1.0, a1));
  a2 = fmin(1.0, fmax(-1.0, a2));
  double k = (-d + r1 + r2) * (d + r1 - r2) * (d - r1 + r2) * (d + r1 + r2);
  k = fmax(k, 0.0);
  const double area = r1 * r1 * acos(a1) + r2 * r2 * acos(a2) - 0.5 * sqrt(k);
  return area / (3.14159265358979323846 * rmin * rmin);
}

__device__ __forceinline__ int image_of(const int64_t* off, int B, int64_t g) {
  int lo = 0, hi = B;  // largest b with off[b] <= g
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

constexpr int kNbMax = 6;   // neighbour indices kept per worklist record

// Scan the candidates around blob k for higher-priority blobs that overlap it by more
// than `overlap`; rows ylo + r0, ylo + r0 + rstep, ...  Returns true as soon as one of
// them is KEPT (k is then REMOVED); otherwise sets *blocked if one is UNDECIDED and
// passes every overlapping one to rec(q).
template <class Rec>
__device__ __forceinline__ bool scan_rows(const PruneArgs& a, int b, int64_t k, int r0, int rstep, bool* blocked,
                                          Rec rec) {
  const mhfd_blob* C = a.cand + (int64_t)b * a.cap;
  const uint8_t* st = a.st + (int64_t)b * a.cap;
  const mhfd_blob me = C[k];
  const double r = a.rad[me.scale];
  const int Dm = a.dmax[me.scale];
  const float2* th = a.thr + me.scale * a.n;
  const int ylo = max(0, me.y - Dm), yhi = min(a.H - 1, me.y + Dm);
  const int kb0 = max(0, me.x - Dm) >> 5, kb1 = min(a.nbx, ((me.x + Dm) >> 5) + 1);
  const int32_t* ri = a.rbi + (int64_t)b * a.H * (a.nbx + 1);
  for (int yy = ylo + r0; yy <= yhi; yy += rstep) {
    const int32_t* rrow = ri + (int64_t)yy * (a.nbx + 1);
    const int lo = __ldcg(rrow + kb0), hi = __ldcg(rrow + kb1);
    for (int q = lo; q < hi; ++q) {
      const mhfd_blob o = C[q];
      if (o.x > me.x + Dm) break;
      if (o.x < me.x - Dm) continue;
      if (q == k) continue;
      const bool higher = o.scale > me.scale ||
                          (o.scale == me.scale && (o.y < me.y || (o.y == me.y && o.x < me.x)));
      if (!higher) continue;
      // frac(d) > overlap, frac decreasing in d: d^2 < lo -> yes, d^2 >= hi -> no, else
      // evaluate the lens formula (the band is 1e-6 relative around the bisected root)
      const int dx = o.x - me.x, dy = o.y - me.y;
      const float d2 = (float)(dx * dx + dy * dy);
      const float2 t2 = __ldg(th + o.scale);
      const bool over = d2 < t2.x ? true
                        : d2 >= t2.y ? false
                                     : lens_fraction(sqrt((double)(dx * dx + dy * dy)), r, a.rad[o.scale]) > a.overlap;
      if (over) {
        const uint8_t s = __ldcg(st + q);
        if (s == kKept) return true;
        if (s == kUndecided) *blocked = true;
        rec(q);
      }
    }
  }
  return false;
}

__device__ uint8_t decide(const PruneArgs& a, int b, int64_t k) {
  bool blocked = false;
  if (scan_rows(a, b, k, 0, 1, &blocked, [](int) {})) return kRemoved;
  return blocked ? kUndecided : kKept;
}

// round-0 decision of blob k that also records its overlapping higher-priority
// neighbours (all of them: a blob that stays UNDECIDED scanned every row)
__device__ uint8_t decide_collect(const PruneArgs& a, int b, int64_t k, int* nq, int (&qs)[kNbMax]) {
  bool blocked = false;
  int n = 0;
  if (scan_rows(a, b, k, 0, 1, &blocked, [&](int q) {
        if (n < kNbMax) qs[n] = q;
        ++n;
      }))
    return kRemoved;
  *nq = n;
  return blocked ? kUndecided : kKept;
}

// later rounds: the recorded neighbours decide (no geometric search)
__device__ uint8_t decide_list(const PruneArgs& a, int b, const int4& r0, const int4& r1) {
  const uint8_t* st = a.st + (int64_t)b * a.cap;
  const int q[kNbMax] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
  bool blocked = false;
#pragma unroll
  for (int i = 0; i < kNbMax; ++i) {
    if (i < r0.y) {
      const uint8_t s = __ldcg(st + q[i]);
      if (s == kKept) return kRemoved;
      if (s == kUndecided) blocked = true;
    }
  }
  return blocked ? kUndecided : kKept;
}

__global__ void __launch_bounds__(256, 4) k_prune(PruneArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
  __shared__ int32_t red[8];
  __shared__ int32_t wpre[8];

  // phase 0: per-image prefixes (one thread; B is small)
  if (gtid == 0) {
    int64_t o = 0, c = 0;
    for (int b = 0; b < a.B; ++b) {
      a.img_off[b] = o;
      a.chunk_off[b] = c;
      const int64_t n = min((int64_t)a.ncand[b], a.cap);
      o += n;
      c += (n + kChunk - 1) / kChunk;
    }
    a.img_off[a.B] = o;
    a.chunk_off[a.B] = c;
    a.counters[0] = a.counters[1] = a.counters[2] = 0;
    a.counters[3] = 0;
    a.counters[4] = 0;
  }
  grid.sync();
  const int64_t total = a.img_off[a.B];
  const int64_t nchunks = a.chunk_off[a.B];

  // phase 1: row index rowstart[b][y] (first candidate of row >= y) and row-block index
  // rbi[b][y][k] (first candidate of row y with x >= 32 k; k = nbx -> row end), both by
  // scatter from the raster-sorted list: candidate k (and a sentinel k = n at row H)
  // owns the entries between its predecessor and itself, so each entry is written once.
  for (int64_t g = gtid; g < total + a.B; g += gsize) {
    // g enumerates, per image, candidates 0..n (n = sentinel): image b holds entries
    // [img_off[b] + b, img_off[b+1] + b + 1)
    int lo = 0, hi = a.B;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (a.img_off[mid] + mid <= g) lo = mid; else hi = mid;
    }
    const int b = lo;
    const int64_t k = g - a.img_off[b] - b;
    const int64_t n = a.img_off[b + 1] - a.img_off[b];
    const mhfd_blob* C = a.cand + (int64_t)b * a.cap;
    int y, x, yp, xp;
    if (k < n) { const mhfd_blob m = C[k]; y = m.y; x = m.x; } else { y = a.H; x = 0; }
    if (k > 0) { const mhfd_blob m = C[k - 1]; yp = m.y; xp = m.x; } else { yp = -1; xp = 0; }
    int32_t* rs = a.rowstart + (int64_t)b * (a.H + 1);
    for (int yy = yp + 1; yy <= y; ++yy) rs[yy] = (int32_t)k;
    if (k < n) a.st[(int64_t)b * a.cap + k] = a.prune ? kUndecided : kKept;
    if (!a.prune) continue;
    int32_t* ri = a.rbi + (int64_t)b * a.H * (a.nbx + 1);
    if (yp >= 0 && yp < y) {   // predecessor ends its row: its trailing blocks point past it
      for (int kb = (xp >> 5) + 1; kb <= a.nbx; ++kb) ri[(int64_t)yp * (a.nbx + 1) + kb] = (int32_t)k;
    }
    for (int yy = yp + 1; yy < y && yy < a.H; ++yy)   // empty rows in between
      for (int kb = 0; kb <= a.nbx; ++kb) ri[(int64_t)yy * (a.nbx + 1) + kb] = (int32_t)k;
    if (k < n) {   // blocks of row y whose first candidate is k
      const int kb0 = (yp == y) ? (xp >> 5) + 1 : 0;
      for (int kb = kb0; kb <= (x >> 5); ++kb) ri[(int64_t)y * (a.nbx + 1) + kb] = (int32_t)k;
    }
  }
  grid.sync();

  // phase 2: decision rounds.  Round 0 visits every blob; a blob it leaves UNDECIDED is
  // appended to the worklist with its overlapping higher-priority neighbours, and later
  // rounds visit only the worklist, deciding from those lists (a list that overflowed
  // kNbMax, or a full worklist, falls back to the geometric search).  Small inputs (one
  // tile) run round 0 one warp per blob, the rows of its search window split over the
  // lanes: the serial chain of dependent row-index loads, not throughput, bounds them.
  if (a.prune) {
    const int64_t gw = gtid >> 5, nwarps = gsize >> 5;
    const int lane0 = threadIdx.x & 31;
    int undecided = 0;
    if (gtid == 0) a.counters[1] = 0;
    auto append = [&](int64_t g, int nq, const int (&qs)[kNbMax]) -> bool {
      const int pos = atomicAdd(&a.counters[4], 1);
      if (pos >= a.wl_cap) return false;
      a.wl[2 * pos] = make_int4((int)g, nq > kNbMax ? kNbMax + 1 : nq, qs[0], qs[1]);
      a.wl[2 * pos + 1] = make_int4(qs[2], qs[3], qs[4], qs[5]);
      return true;
    };
    if (total * 32 <= gsize * 4) {   // warp per blob
      __shared__ int wq[8][kNbMax + 1];
      const int wib = threadIdx.x >> 5;
      for (int64_t g = gw; g < total; g += nwarps) {
        const int b = image_of(a.img_off, a.B, g);
        const int64_t k = g - a.img_off[b];
        if (lane0 == 0) wq[wib][kNbMax] = 0;
        __syncwarp();
        bool blocked = false;
        const bool rem = scan_rows(a, b, k, lane0, 32, &blocked, [&](int q) {
          const int pos = atomicAdd(&wq[wib][kNbMax], 1);
          if (pos < kNbMax) wq[wib][pos] = q;
        });
        const bool any_rem = __any_sync(0xffffffffu, rem);
        const bool any_blk = __any_sync(0xffffffffu, blocked);
        __syncwarp();
        if (lane0 == 0) {
          uint8_t d = any_rem ? kRemoved : any_blk ? kUndecided : kKept;
          if (d == kUndecided) {
            int qs[kNbMax];
            for (int i = 0; i < kNbMax; ++i) qs[i] = wq[wib][i];
            ++undecided;
            append(g, wq[wib][kNbMax], qs);
          }
          if (d != kUndecided) __stcg(a.st + (int64_t)b * a.cap + k, d);
        }
        __syncwarp();
      }
    } else {
      for (int64_t g = gtid; g < total; g += gsize) {
        const int b = image_of(a.img_off, a.B, g);
        const int64_t k = g - a.img_off[b];
        int nq = 0, qs[kNbMax] = {0, 0, 0, 0, 0, 0};
        const uint8_t d = decide_collect(a, b, k, &nq, qs);
        if (d != kUndecided) {
          __stcg(a.st + (int64_t)b * a.cap + k, d);
        } else {
          ++undecided;
          append(g, nq, qs);
        }
      }
    }
    if (undecided) atomicAdd(&a.counters[0], undecided);
    grid.sync();
    int left = *((volatile int32_t*)&a.counters[0]);
    const int64_t nwl = *((volatile int32_t*)&a.counters[4]);
    const bool full = nwl > a.wl_cap;   // some undecided blob is not on the list
    if (gtid == 0) a.counters[3] = 1;
    for (int round = 1; left > 0; ++round) {
      if (gtid == 0) a.counters[(round + 1) % 3] = 0;
      undecided = 0;
      if (!full) {
        for (int64_t i = gtid; i < nwl; i += gsize) {
          const int4 r0 = a.wl[2 * i];
          const int64_t g = r0.x;
          const int b = image_of(a.img_off, a.B, g);
          const int64_t k = g - a.img_off[b];
          uint8_t* sp = a.st + (int64_t)b * a.cap + k;
          if (__ldcg(sp) != kUndecided) continue;
          const uint8_t d = r0.y <= kNbMax ? decide_list(a, b, r0, a.wl[2 * i + 1]) : decide(a, b, k);
          if (d != kUndecided) __stcg(sp, d); else ++undecided;
        }
      } else {
        for (int64_t g = gtid; g < total; g += gsize) {
          const int b = image_of(a.img_off, a.B, g);
          const int64_t k = g - a.img_off[b];
          uint8_t* sp = a.st + (int64_t)b * a.cap + k;
          if (__ldcg(sp) != kUndecided) continue;
          const uint8_t d = decide(a, b, k);
          if (d != kUndecided) __stcg(sp, d); else ++undecided;
        }
      }
      if (undecided) atomicAdd(&a.counters[round % 3], undecided);
      grid.sync();
      left = *((volatile int32_t*)&a.counters[round % 3]);
      if (gtid == 0) a.counters[3] = round + 1;
    }
  }
  grid.sync();

  // phase 3: kept count per chunk of 256 candidates
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int b = image_of(a.chunk_off, a.B, c);
    const int64_t k = (c - a.chunk_off[b]) * kChunk + threadIdx.x;
    const int64_t n = a.img_off[b + 1] - a.img_off[b];
    const bool kept = k < n && __ldcg(a.st + (int64_t)b * a.cap + k) == kKept;
    const int cnt = __popc(__ballot_sync(0xffffffffu, kept));
    if (lane == 0) red[warp] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int w = 0; w < 8; ++w) s += red[w];
      a.chunk_cnt[c] = s;
    }
    __syncthreads();
  }
  grid.sync();

  // phase 4: per-image exclusive scan over chunks (one warp per image)
  {
    const int64_t gw = gtid >> 5, nw = gsize >> 5;
    for (int64_t b = gw; b < a.B; b += nw) {
      int64_t run = 0;
      for (int64_t c0 = a.chunk_off[b]; c0 < a.chunk_off[b + 1]; c0 += 32) {
        const int64_t c = c0 + lane;
        const int v = c < a.chunk_off[b + 1] ? __ldcg(a.chunk_cnt + c) : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (c < a.chunk_off[b + 1]) a.chunk_pos[c] = (int32_t)(run + x - v);
        run += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) {
        const int32_t nc = a.ncand[b];
        const int64_t count = a.prune ? run : (int64_t)nc;   // overlap = 1: every candidate kept
        int32_t f = (nc > a.cap) ? 1 : 0;
        if (a.blobs && count > a.blob_cap) f |= 2;
        if (a.counts) a.counts[b] = (int32_t)count;
        if (a.scores) a.scores[b] = (double)count;
        if (a.flags) a.flags[b] = f;
      }
    }
  }
  if (!a.blobs) return;
  grid.sync();

  // phase 5: write kept blobs in (y, x, scale) order
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int b = image_of(a.chunk_off, a.B, c);
    const int64_t k = (c - a.chunk_off[b]) * kChunk + threadIdx.x;
    const int64_t n = a.img_off[b + 1] - a.img_off[b];
    const bool kept = k < n && __ldcg(a.st + (int64_t)b * a.cap + k) == kKept;
    const uint32_t m = __ballot_sync(0xffffffffu, kept);
    if (lane == 0) red[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int w = 0; w < 8; ++w) { wpre[w] = s; s += red[w]; }
    }
    __syncthreads();
    if (kept) {
      const int64_t pos = (int64_t)__ldcg(a.chunk_pos + c) + wpre[warp] + __popc(m & ((1u << lane) - 1u));
      if (pos < a.blob_cap) a.blobs[(int64_t)b * a.blob_cap + pos] = a.cand[(int64_t)b * a.cap + k];
    }
    __syncthreads();
  }
}

}  // namespace mhfd
