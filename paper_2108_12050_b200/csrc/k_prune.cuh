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
// separated by grid-wide barriers.  Neighbours are found through a cell index: the
// image is cut into bands of cs rows (cs = a power of two >= every search radius) and
// each band's candidates (a contiguous range of the raster-sorted list) are counting-
// sorted by their cs-wide column cell into `crec`; the 3 x 3 cells around a blob are then
// three contiguous record ranges (cells cx-1..cx+1 of bands yb-1..yb+1), found with six
// independent index loads instead of a chain of ~2 Dm dependent per-row lookups.
//
// Score: DOF = |C| after pruning.  The kept list is emitted in
// (y, x, scale) order by a chunked scan (no atomics decide positions).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace mhfd {

namespace cg = cooperative_groups;

#ifndef PRUNE_STAMPS
#define PRUNE_STAMPS 0   // performance experiments: globaltimer after each grid barrier -> counters[16..],
#endif                   // records scanned -> counters[8]

constexpr uint8_t kUndecided = 0, kKept = 1, kRemoved = 2;

// State byte: decision in bits 0-1, and in synchronous mode (PruneArgs::sync) the round
// that decided it in bits 2-7 (saturating at 63).  Synchronous rounds (Jacobi instead of
// the default Gauss-Seidel, where a blob may use a decision made earlier in the same
// round) make a round-t decision a function of the candidates within (t + 1) dmax of the
// blob only: the certificate of the sharded pruning (mhfd_prune_band) rests on that.
__device__ __forceinline__ uint8_t st_vis(uint8_t s, int round, int sync) {
  const uint8_t d = s & 3u;
  return (sync && d != kUndecided && (int)(s >> 2) >= round) ? kUndecided : d;
}
__device__ __forceinline__ uint8_t st_enc(uint8_t d, int round, int sync) {
  return sync ? (uint8_t)(d | (min(round, 63) << 2)) : d;
}
constexpr int kChunk = 256;
constexpr int kPruneSmemB = 128;   // batches whose prefixes every k_prune CTA computes itself

struct PruneArgs {
  int B, W, H;
  int64_t cap;              // candidate capacity per image
  const mhfd_blob* cand;    // B x cap, raster order
  const int32_t* ncand;     // exact candidate counts
  double overlap;
  int prune;                // overlap < 1
  int sync;                 // synchronous rounds (f2 sharded pruning): see st_vis
  double radmax;
  double rad[kMaxLevels];   // sqrt(2) * t_s
  int32_t dmax[kMaxLevels]; // search radius of a plane-s blob: ceil(sqrt(max_{s'>=s} thr_hi(s, s')))
  const float2* thr;        // n x n squared-distance band (lo, hi) of frac > overlap (host bisection)
  int n;                    // DoG planes
  uint8_t* st;              // B x cap
  int32_t* rowstart;        // B x (H + 1): first candidate of each row
  const int32_t* segoff;    // nullable: NMS segment offsets (whole-row 1024-pixel segments) = row starts
  int nseg, spr;            // segments per image, per row
  int cs_shift;             // cell edge cs = 1 << cs_shift (>= every dmax)
  int ncx, nbands;          // ceil(W / cs) cells per band, ceil(H / cs) bands
  int nsk;                  // scale keys per cell: n (records of a cell sorted by scale, descending,
                            // which enables scan_cells' reach test) or 1 (unsorted; too many keys)
  int32_t* cellstart;       // B x nbands x cst_stride: first crec index of cell (band, cx); k_prune<false>:
                            // two classes per band, scale >= 1 (cells 0..ncx) then scale 0 (ncx+1 ..)
  int cst_stride;           // ncx + 1 (k_prune<true>) or 2 (ncx + 1) (k_prune<false>)
  int4* crec;               // B x cap: {x, y, scale, k} per candidate, band-major, cell-sorted
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

constexpr int kMaxCells = 2048;   // ncx + 1 per band
constexpr int kMaxKeys = 6144;    // (cell, scale) keys of the shared-memory counting sort per band

// Scan the candidates around blob k for higher-priority blobs that overlap it by more
// than `overlap`: the records of cells cx-1..cx+1 in bands yb-1..yb+1 (three contiguous
// ranges), entries i0, i0 + istep, ... of each.  Returns true as soon as one of them is
// KEPT (k is then REMOVED); otherwise sets *blocked if one is UNDECIDED and passes every
// overlapping one to rec(q).
// R: the image's cell-ordered records, or a shared-memory copy of a band window offset so
// that R[i] is record i (k_prune round 0)
template <bool SORTED, class Rec>
__device__ __forceinline__ bool scan_cells(const PruneArgs& a, int b, const int4 me4, const int4* R0p, const int4* R1p,
                                           const int4* R2p, int i0, int istep, bool* blocked, Rec rec, int round) {
  const uint8_t* st = a.st + (int64_t)b * a.cap;
  struct { int x, y, scale; } me = {me4.x, me4.y, me4.z};
  const int64_t k = me4.w;
  const double r = a.rad[me.scale];
  const int Dm = a.dmax[me.scale];
  const float2* th = a.thr + me.scale * a.n;
  const int yb = me.y >> a.cs_shift, cx = me.x >> a.cs_shift;
  const int b0 = max(0, yb - 1), b1 = min(a.nbands - 1, yb + 1);
  const int c0 = max(0, cx - 1), c1 = min(a.ncx, cx + 2);
  const int32_t* cst = a.cellstart + (int64_t)b * a.nbands * a.cst_stride;
  // the test of one record o: true = k is REMOVED (o is a kept, higher-priority blob
  // overlapping it by more than `overlap`)
  auto test = [&](const int4& o, const float2 t2) -> bool {
    const int dx = o.x - me.x, dy = o.y - me.y;
    if (dx > Dm || dx < -Dm || dy > Dm || dy < -Dm) return false;
    if (o.w == k) return false;
    const bool higher = o.z > me.scale || (o.z == me.scale && (o.y < me.y || (o.y == me.y && o.x < me.x)));
    if (!higher) return false;
    // frac(d) > overlap, frac decreasing in d: d^2 < lo -> yes, d^2 >= hi -> no, else
    // evaluate the lens formula (the band is 1e-6 relative around the bisected root)
    const float d2 = (float)(dx * dx + dy * dy);
    const bool over = d2 < t2.x ? true
                      : d2 >= t2.y ? false
                                   : lens_fraction(sqrt((double)(dx * dx + dy * dy)), r, a.rad[o.z]) > a.overlap;
    if (over) {
      const uint8_t s = st_vis(__ldcg(st + o.w), round, a.sync);
      if (s == kKept) return true;
      if (s == kUndecided) *blocked = true;
      rec(o.w);
    }
    return false;
  };
  // cst and R were written in phase 1b of this launch and are read-only since: plain
  // (L1-cached) loads are coherent here (no SM cached these lines before the barrier,
  // and L1 starts empty at launch), and neighbouring blobs share most of their windows
  if (!SORTED) {
    // Two classes per band.  Records of scales >= 1: cells c0 .. c1-1 of a band are one
    // contiguous range, scanned over the 3 x 3 cell window (the largest reach).  Records
    // of scale 0 (most blobs at small scales, e.g. 87 % on the C3 tiles): lower priority
    // than any blob of scale >= 1, so only a scale-0 blob scans them, and only the cells
    // within its reach of a scale-0 neighbour (sqrt thr_hi(0, 0), about a pixel).
    int lo[3], hi[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {   // six independent loads
      const int bb = min(b0 + j, b1);
      lo[j] = cst[(int64_t)bb * a.cst_stride + c0];
      hi[j] = b0 + j <= b1 ? cst[(int64_t)bb * a.cst_stride + c1] : lo[j];
    }
#pragma unroll 1
    for (int j = 0; j < 3; ++j) {
      const int4* R = j == 0 ? R0p : j == 1 ? R1p : R2p;   // records of band b0 + j
      if (PRUNE_STAMPS && hi[j] > lo[j] + i0) atomicAdd(&a.counters[8], (hi[j] - lo[j] - i0 + istep - 1) / istep);
#pragma unroll 4
      for (int i = lo[j] + i0; i < hi[j]; i += istep) {
        const int4 o = R[i];   // {x, y, scale, k}
        if (test(o, __ldg(th + o.z))) return true;
      }
    }
    if (me.scale == 0) {
      const int rr = (int)ceilf(sqrtf(__ldg(th).y));   // reach to a scale-0 neighbour (>= 0)
      const int ya = max(0, (me.y - rr) >> a.cs_shift), yz = min(a.nbands - 1, (me.y + rr) >> a.cs_shift);
      const int xa = max(0, (me.x - rr) >> a.cs_shift), xz = min(a.ncx - 1, (me.x + rr) >> a.cs_shift);
#pragma unroll 1
      for (int bb = ya; bb <= yz; ++bb) {
        const int j = bb - b0;   // within the 3 x 3 window: rr <= dmax <= cs
        const int4* R = j == 0 ? R0p : j == 1 ? R1p : R2p;
        const int32_t* cs0 = cst + (int64_t)bb * a.cst_stride + (a.ncx + 1);
        const int s_lo = cs0[xa], s_hi = cs0[xz + 1];
#pragma unroll 2
        for (int i = s_lo + i0; i < s_hi; i += istep) {
          const int4 o = R[i];
          if (test(o, __ldg(th))) return true;
        }
      }
    }
    return false;
  }
  // Scale-sorted cells (descending; large radii, where a cell is much larger than most
  // blobs' reach): every later record of a cell has a scale <= o.z, so a lower-priority
  // scale, or an overlap distance band thr_hi(s, s') (non-decreasing in s' >= s: the lens
  // grows with the larger disk) that cannot reach the cell's nearest pixel, ends the cell
  const int cs = 1 << a.cs_shift;
#pragma unroll 1
  for (int j = 0; j < 3; ++j) {
    if (b0 + j > b1) break;
    const int4* R = j == 0 ? R0p : j == 1 ? R1p : R2p;   // records of band b0 + j
    const int32_t* cb = cst + (int64_t)(b0 + j) * a.cst_stride;
    const int by0 = (b0 + j) * cs, ddy = me.y < by0 ? by0 - me.y : (me.y >= by0 + cs ? me.y - (by0 + cs - 1) : 0);
#pragma unroll 1
    for (int q = 0; q < c1 - c0; ++q) {
      const int i_lo = cb[c0 + q], i_hi = cb[c0 + q + 1];   // the cell's records
      const int cx0 = (c0 + q) * cs;
      const int ddx = me.x < cx0 ? cx0 - me.x : (me.x >= cx0 + cs ? me.x - (cx0 + cs - 1) : 0);
      const float dc2 = (float)(ddx * ddx + ddy * ddy);   // to the cell's nearest pixel
      if (PRUNE_STAMPS && i_hi > i_lo + i0) atomicAdd(&a.counters[8], (i_hi - i_lo - i0 + istep - 1) / istep);
#pragma unroll 1
      for (int i = i_lo + i0; i < i_hi; i += istep) {
        const int4 o = R[i];
        const float2 t2 = __ldg(th + o.z);
        if (o.z < me.scale || dc2 >= t2.y) break;
        if (test(o, t2)) return true;
      }
    }
  }
  return false;
}

template <bool SORTED, class Rec>
__device__ __forceinline__ bool scan_rows(const PruneArgs& a, int b, int64_t k, int i0, int istep, bool* blocked,
                                          Rec rec, int round) {
  const mhfd_blob m = a.cand[(int64_t)b * a.cap + k];
  const int4* R = a.crec + (int64_t)b * a.cap;
  return scan_cells<SORTED>(a, b, make_int4(m.x, m.y, m.scale, (int)k), R, R, R, i0, istep, blocked, rec, round);
}

template <bool SORTED>
__device__ uint8_t decide(const PruneArgs& a, int b, int64_t k, int round) {
  bool blocked = false;
  if (scan_rows<SORTED>(a, b, k, 0, 1, &blocked, [](int) {}, round)) return kRemoved;
  return blocked ? kUndecided : kKept;
}

// round-0 decision of blob k that also records its overlapping higher-priority
// neighbours (all of them: a blob that stays UNDECIDED scanned every row)
template <bool SORTED>
__device__ uint8_t decide_collect(const PruneArgs& a, int b, int64_t k, int* nq, int (&qs)[kNbMax]) {
  bool blocked = false;
  int n = 0;
  if (scan_rows<SORTED>(
          a, b, k, 0, 1, &blocked,
          [&](int q) {
            if (n < kNbMax) qs[n] = q;
            ++n;
          },
          0))
    return kRemoved;
  *nq = n;
  return blocked ? kUndecided : kKept;
}

// later rounds: the recorded neighbours decide (no geometric search)
__device__ uint8_t decide_list(const PruneArgs& a, int b, const int4& r0, const int4& r1, int round) {
  const uint8_t* st = a.st + (int64_t)b * a.cap;
  const int q[kNbMax] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
  bool blocked = false;
#pragma unroll
  for (int i = 0; i < kNbMax; ++i) {
    if (i < r0.y) {
      const uint8_t s = st_vis(__ldcg(st + q[i]), round, a.sync);
      if (s == kKept) return kRemoved;
      if (s == kUndecided) blocked = true;
    }
  }
  return blocked ? kUndecided : kKept;
}

template <bool SORTED>
__global__ void __launch_bounds__(256, 4) k_prune(PruneArgs a) {
  cg::grid_group grid = cg::this_grid();
  int pst_ = 0;
  auto PSTAMP = [&]() {
    if (PRUNE_STAMPS && blockIdx.x == 0 && threadIdx.x == 0 && pst_ < 24) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      reinterpret_cast<unsigned long long*>(a.counters + 16)[pst_] = t_;
    }
    ++pst_;
  };
  PSTAMP();
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
  __shared__ int32_t red[8];
  __shared__ int32_t wpre[8];

  // phase 0: per-image prefixes of the candidate and chunk counts.  For batches up to
  // kPruneSmemB every CTA computes them itself into shared memory (no grid barrier: one
  // of the ~8 that bound a single tile's latency); larger batches use one thread and
  // the global copy.  The counters are reset here; their first use is two barriers on.
  __shared__ int64_t s_off[2][kPruneSmemB + 1];
  const bool local_off = a.B <= kPruneSmemB;
  if (gtid == 0 || (local_off && threadIdx.x == 0)) {
    int64_t o = 0, c = 0;
    for (int b = 0; b < a.B; ++b) {
      if (gtid == 0) {
        a.img_off[b] = o;
        a.chunk_off[b] = c;
      }
      if (local_off) {
        s_off[0][b] = o;
        s_off[1][b] = c;
      }
      const int64_t n = min((int64_t)a.ncand[b], a.cap);
      o += n;
      c += (n + kChunk - 1) / kChunk;
    }
    if (gtid == 0) {
      a.img_off[a.B] = o;
      a.chunk_off[a.B] = c;
      a.counters[0] = a.counters[1] = a.counters[2] = 0;
      a.counters[3] = 0;
      a.counters[4] = 0;
      a.counters[5] = 0;
      if (PRUNE_STAMPS) a.counters[8] = 0;
    }
    if (local_off) {
      s_off[0][a.B] = o;
      s_off[1][a.B] = c;
    }
  }
  if (local_off) __syncthreads();
  else grid.sync();
  PSTAMP();
  const int64_t* img_off = local_off ? s_off[0] : a.img_off;
  const int64_t* chunk_off = local_off ? s_off[1] : a.chunk_off;
  const int64_t total = img_off[a.B];
  const int64_t nchunks = chunk_off[a.B];

  // phase 1: row index rowstart[b][y] (first candidate of row >= y), by scatter from the
  // raster-sorted list: candidate k (and a sentinel k = n at row H) owns the entries
  // between its predecessor's row and its own, so each entry is written once.
  // With the NMS's segment offsets (whole-row segments: row y starts at segoff[y spr])
  // the row index is already there: phase 1 and its barrier are skipped and phase 1b
  // initialises the states.
  const bool seg_rows = a.segoff != nullptr && a.prune;
  for (int64_t g = seg_rows ? total + a.B : gtid; g < total + a.B; g += gsize) {
    // g enumerates, per image, candidates 0..n (n = sentinel): image b holds entries
    // [img_off[b] + b, img_off[b+1] + b + 1)
    int lo = 0, hi = a.B;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (img_off[mid] + mid <= g) lo = mid; else hi = mid;
    }
    const int b = lo;
    const int64_t k = g - img_off[b] - b;
    const int64_t n = img_off[b + 1] - img_off[b];
    const mhfd_blob* C = a.cand + (int64_t)b * a.cap;
    const int y = k < n ? C[k].y : a.H, yp = k > 0 ? C[k - 1].y : -1;
    int32_t* rs = a.rowstart + (int64_t)b * (a.H + 1);
    for (int yy = yp + 1; yy <= y; ++yy) rs[yy] = (int32_t)k;
    if (k < n) a.st[(int64_t)b * a.cap + k] = a.prune ? kUndecided : kKept;
  }
  if (!seg_rows) grid.sync();
  PSTAMP();

  // phase 1b: cell index.  Band (b, j) = rows [j cs, (j+1) cs) = the contiguous range
  // [rowstart[j cs], rowstart[(j+1) cs]) of the raster list; one CTA counting-sorts it by
  // column cell in shared memory (order inside a cell is irrelevant: decisions do not
  // depend on it) and writes the cell starts and the cell-ordered records.
  if (a.prune) {
    __shared__ int32_t cell[kMaxKeys];
    const int cs = 1 << a.cs_shift;
    // keys: k_prune<true> (cell cx, scale s) -> cx nsk + (nsk - 1 - s), + the end;
    // k_prune<false> two classes: scale >= 1 -> cx, scale 0 -> ncx + 1 + cx (each with an end key)
    const int nk = SORTED ? a.ncx * a.nsk + 1 : 2 * (a.ncx + 1);
    auto key_of = [&](int x, int sc) {
      return SORTED ? (x >> a.cs_shift) * a.nsk + (a.nsk > 1 ? a.nsk - 1 - sc : 0)
                    : (sc == 0 ? a.ncx + 1 : 0) + (x >> a.cs_shift);
    };
    for (int64_t item = blockIdx.x; item < (int64_t)a.B * a.nbands; item += gridDim.x) {
      const int b = (int)(item / a.nbands), j = (int)(item % a.nbands);
      const int64_t nb_ = img_off[b + 1] - img_off[b];
      auto row_start = [&](int y) -> int {
        if (!seg_rows) return a.rowstart[(int64_t)b * (a.H + 1) + y];
        return y >= a.H ? (int)nb_ : (int)min((int64_t)a.segoff[(int64_t)b * a.nseg + (int64_t)y * a.spr], nb_);
      };
      const int k0 = row_start(j * cs), k1 = row_start(min(a.H, (j + 1) * cs));
      const mhfd_blob* C = a.cand + (int64_t)b * a.cap;
      if (seg_rows)
        for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) a.st[(int64_t)b * a.cap + k] = kUndecided;
      for (int c = threadIdx.x; c < nk; c += blockDim.x) cell[c] = 0;
      __syncthreads();
      for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) atomicAdd(&cell[key_of(C[k].x, C[k].scale)], 1);
      __syncthreads();
      if (threadIdx.x < 32) {   // exclusive scan of the key counts by one warp
        int carry = 0;
        for (int c0 = 0; c0 < nk; c0 += 32) {
          const int c = c0 + threadIdx.x;
          const int v = c < nk ? cell[c] : 0;
          int x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x, o);
            if ((int)threadIdx.x >= o) x += t;
          }
          if (c < nk) cell[c] = k0 + carry + x - v;
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
      }
      __syncthreads();
      int32_t* cst = a.cellstart + ((int64_t)b * a.nbands + j) * a.cst_stride;
      if (SORTED)
        for (int c = threadIdx.x; c <= a.ncx; c += blockDim.x) cst[c] = cell[c * a.nsk];   // first key of each cell
      else
        for (int c = threadIdx.x; c < nk; c += blockDim.x) cst[c] = cell[c];
      __syncthreads();
      int4* R = a.crec + (int64_t)b * a.cap;
      for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const mhfd_blob m = C[k];
        const int pos = atomicAdd(&cell[key_of(m.x, m.scale)], 1);
        R[pos] = make_int4(m.x, m.y, m.scale, k);
      }
      __syncthreads();
    }
    grid.sync();
    PSTAMP();
  }

  // phase 2: decision rounds.  Round 0 visits every blob; a blob it leaves UNDECIDED is
  // appended to the worklist with its overlapping higher-priority neighbours, and later
  // rounds visit only the worklist, deciding from those lists (a list that overflowed
  // kNbMax, or a full worklist, falls back to the geometric search).  Small inputs (one
  // tile) run round 0 one warp per blob, the rows of its search window split over the
  // lanes: the serial chain of dependent row-index loads, not throughput, bounds them.
  if (a.prune) {
    const int lane0 = threadIdx.x & 31;
    int undecided = 0;
    if (gtid == 0) a.counters[1] = 0;
    // Round 0.  Lanes per blob: enough groups of G lanes to give every thread about one
    // blob-share (1 for batches: many blobs per thread average the per-blob cost out; a
    // single tile has ~1 blob per thread, and the round lasts as long as the slowest
    // thread's window scan).  Measured alternative that lost: each CTA copying a band
    // piece's window into shared memory and scanning it there.
    int G = 1;
    // G doubles while total * G < 2 x threads, up to 16 (measured after the two-class cell
    // index: one 4096^2 tile takes G = 2, 0.066 -> 0.064 ms; one 1024^2 tile G = 16, 0.032
    // -> 0.030 ms; batches G = 1)
    while (G < 16 && total * G < gsize * 2) G <<= 1;
    if (G > 1) {   // a group of G lanes per blob, striding over its window's records
      __shared__ int wq[8][32][kNbMax + 1];
      const int wib = threadIdx.x >> 5, grp = lane0 / G, gl = lane0 & (G - 1);
      const uint32_t gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (grp * G);
      for (int64_t gb = (gtid - lane0) / G; gb < total; gb += gsize / G) {
        const int64_t g = gb + grp;
        const bool in = g < total;
        int b = 0;
        int64_t k = 0;
        if (gl == 0) wq[wib][grp][kNbMax] = 0;
        __syncwarp();
        bool blocked = false, rem = false;
        if (in) {
          b = image_of(img_off, a.B, g);
          k = g - img_off[b];
          rem = scan_rows<SORTED>(
              a, b, k, gl, G, &blocked,
              [&](int q) {
                const int pos = atomicAdd(&wq[wib][grp][kNbMax], 1);
                if (pos < kNbMax) wq[wib][grp][pos] = q;
              },
              0);
        }
        const bool any_rem = (__ballot_sync(0xffffffffu, rem) & gmask) != 0;
        const bool any_blk = (__ballot_sync(0xffffffffu, blocked) & gmask) != 0;
        __syncwarp();
        const bool lead = in && gl == 0;
        const uint8_t d = any_rem ? kRemoved : any_blk ? kUndecided : kKept;
        if (lead && d != kUndecided) __stcg(a.st + (int64_t)b * a.cap + k, st_enc(d, 0, a.sync));
        const uint32_t m = __ballot_sync(0xffffffffu, lead && d == kUndecided);
        if (m) {   // one worklist atomic per warp
          int base = 0;
          if (lane0 == __ffs(m) - 1) base = atomicAdd(&a.counters[4], __popc(m));
          base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
          if (lead && d == kUndecided) {
            ++undecided;
            const int pos = base + __popc(m & ((1u << lane0) - 1u));
            const int* w = wq[wib][grp];
            if (pos < a.wl_cap) {
              a.wl[2 * pos] = make_int4((int)g, w[kNbMax] > kNbMax ? kNbMax + 1 : w[kNbMax], w[0], w[1]);
              a.wl[2 * pos + 1] = make_int4(w[2], w[3], w[4], w[5]);
            }
          }
        }
        __syncwarp();
      }
    } else {
      // every lane of a warp runs the same number of iterations (gsize is a multiple of
      // 32), so the worklist slots are claimed with one atomic per warp and iteration: a
      // per-blob atomic on the one counter serialised ~10^5 appends
      for (int64_t g0 = gtid - lane0; g0 < total; g0 += gsize) {
        const int64_t g = g0 + lane0;
        const bool in = g < total;
        int b = 0;
        int64_t k = 0;
        int nq = 0, qs[kNbMax] = {0, 0, 0, 0, 0, 0};
        uint8_t d = kKept;
        if (in) {
          b = image_of(img_off, a.B, g);
          k = g - img_off[b];
          d = decide_collect<SORTED>(a, b, k, &nq, qs);
          if (d != kUndecided) __stcg(a.st + (int64_t)b * a.cap + k, st_enc(d, 0, a.sync));
        }
        const bool und = in && d == kUndecided;
        const uint32_t m = __ballot_sync(0xffffffffu, und);
        if (m) {
          int base = 0;
          if (lane0 == __ffs(m) - 1) base = atomicAdd(&a.counters[4], __popc(m));
          base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
          if (und) {
            ++undecided;
            const int pos = base + __popc(m & ((1u << lane0) - 1u));
            if (pos < a.wl_cap) {
              a.wl[2 * pos] = make_int4((int)g, nq > kNbMax ? kNbMax + 1 : nq, qs[0], qs[1]);
              a.wl[2 * pos + 1] = make_int4(qs[2], qs[3], qs[4], qs[5]);
            }
          }
        }
      }
    }
    if (undecided) atomicAdd(&a.counters[0], undecided);
    if (PRUNE_STAMPS) {   // per-CTA end of round-0 work (globaltimer, low 32 bits) -> the worklist's tail
      __syncthreads();
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      if (threadIdx.x == 0) reinterpret_cast<int32_t*>(a.wl + 2 * (a.wl_cap - 1024))[blockIdx.x] = (int32_t)(uint32_t)t_;
    }
    grid.sync();
    PSTAMP();
    int left = *((volatile int32_t*)&a.counters[0]);
    const int64_t nwl = *((volatile int32_t*)&a.counters[4]);
    const bool full = nwl > a.wl_cap;   // some undecided blob is not on the list
    if (gtid == 0) a.counters[3] = 1;
    // Default (Gauss-Seidel) mode with every undecided blob on the worklist: no rounds.
    // Each thread re-visits its own worklist blobs until they have decided, reading its
    // neighbours' states as other threads write them.  The decisions are the greedy ones
    // whatever the order (a blob decides only from decided higher-priority neighbours),
    // and it terminates because the grid is co-resident (cooperative launch) and the
    // highest-priority undecided blob always decides on its owner's next visit.  One grid
    // barrier instead of one per round (~3 us each; a 4096^2 tile needs 4-6 rounds).
    const bool async_rounds = !a.sync && !full && left > 0;
    if (async_rounds) {
      for (bool more = true; more;) {
        more = false;
        for (int64_t i = gtid; i < nwl; i += gsize) {
          const int4 r0 = a.wl[2 * i];
          const int64_t g = r0.x;
          const int b = image_of(img_off, a.B, g);
          const int64_t k = g - img_off[b];
          uint8_t* sp = a.st + (int64_t)b * a.cap + k;
          if ((__ldcg(sp) & 3u) != kUndecided) continue;
          const uint8_t d = r0.y <= kNbMax ? decide_list(a, b, r0, a.wl[2 * i + 1], 1) : decide<SORTED>(a, b, k, 1);
          if (d != kUndecided) __stcg(sp, d); else more = true;
        }
        if (more) {
          __nanosleep(32);
          asm volatile("" ::: "memory");   // re-read the states on the next pass
        }
      }
      left = 0;
    }
    for (int round = 1; left > 0; ++round) {
      if (gtid == 0) a.counters[(round + 1) % 3] = 0;
      undecided = 0;
      if (!full) {
        for (int64_t i = gtid; i < nwl; i += gsize) {
          const int4 r0 = a.wl[2 * i];
          const int64_t g = r0.x;
          const int b = image_of(img_off, a.B, g);
          const int64_t k = g - img_off[b];
          uint8_t* sp = a.st + (int64_t)b * a.cap + k;
          if ((__ldcg(sp) & 3u) != kUndecided) continue;
          const uint8_t d = r0.y <= kNbMax ? decide_list(a, b, r0, a.wl[2 * i + 1], round) : decide<SORTED>(a, b, k, round);
          if (d != kUndecided) __stcg(sp, st_enc(d, round, a.sync)); else ++undecided;
        }
      } else {
        for (int64_t g = gtid; g < total; g += gsize) {
          const int b = image_of(img_off, a.B, g);
          const int64_t k = g - img_off[b];
          uint8_t* sp = a.st + (int64_t)b * a.cap + k;
          if ((__ldcg(sp) & 3u) != kUndecided) continue;
          const uint8_t d = decide<SORTED>(a, b, k, round);
          if (d != kUndecided) __stcg(sp, st_enc(d, round, a.sync)); else ++undecided;
        }
      }
      if (undecided) atomicAdd(&a.counters[round % 3], undecided);
      grid.sync();
      PSTAMP();
      left = *((volatile int32_t*)&a.counters[round % 3]);
      if (gtid == 0) a.counters[3] = round + 1;
    }
    if (async_rounds) grid.sync();   // (the last round's barrier already separates phase 3)
  } else {
    grid.sync();
  }
  PSTAMP();

  // phase 3: kept count per chunk of 256 candidates
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int b = image_of(chunk_off, a.B, c);
    const int64_t k = (c - chunk_off[b]) * kChunk + threadIdx.x;
    const int64_t n = img_off[b + 1] - img_off[b];
    const bool kept = k < n && (__ldcg(a.st + (int64_t)b * a.cap + k) & 3u) == kKept;
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
  // Without an output list (focus scores) phase 4 runs in the CTA that finishes phase 3
  // last (a ticket instead of a grid barrier); with one, every warp of the grid scans.
  int64_t gw = gtid >> 5, nw = gsize >> 5;
  if (a.blobs) {
    grid.sync();
  } else {
    __shared__ int last_cta;
    __threadfence();   // this CTA's chunk counts are visible before its ticket
    __syncthreads();
    if (threadIdx.x == 0) last_cta = atomicAdd(&a.counters[5], 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last_cta) return;
    __threadfence();
    gw = warp;
    nw = blockDim.x >> 5;
  }
  PSTAMP();

  // phase 4: per-image exclusive scan over chunks (one warp per image)
  {
    for (int64_t b = gw; b < a.B; b += nw) {
      int64_t run = 0;
      for (int64_t c0 = chunk_off[b]; c0 < chunk_off[b + 1]; c0 += 32) {
        const int64_t c = c0 + lane;
        const int v = c < chunk_off[b + 1] ? __ldcg(a.chunk_cnt + c) : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (c < chunk_off[b + 1]) a.chunk_pos[c] = (int32_t)(run + x - v);
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
  PSTAMP();

  // phase 5: write kept blobs in (y, x, scale) order
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int b = image_of(chunk_off, a.B, c);
    const int64_t k = (c - chunk_off[b]) * kChunk + threadIdx.x;
    const int64_t n = img_off[b + 1] - img_off[b];
    const bool kept = k < n && (__ldcg(a.st + (int64_t)b * a.cap + k) & 3u) == kKept;
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
