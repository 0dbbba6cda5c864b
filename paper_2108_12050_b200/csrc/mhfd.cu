// mhfd.cu — C-ABI (include/mhfd.h) and host orchestration of the MHFD CUDA path.
//
// Host side: validate arguments, build the scale grid and f32 tap tables from f64
// (PAPER.md:134-137, 166-168), carve the caller's workspace, and enqueue the launch
// sequence on the caller's stream without any host synchronisation:
//
//   k_hist / k_select (u8: 1 pass, u16: 2 passes)   percentiles, row a1
//   k_tc (u8, tensor cores) | k_band (u8, CUDA cores) | k_scale_space (generic)
//                                                   stretch+blur+DoG+argmax, rows a2-a6
//   k_nms_count -> k_seg_scan -> k_nms_write        NMS+threshold+compaction, rows a7-a8
//   k_prune (cooperative, one launch)               pruning + score + ordered list, a9-a10
#include <algorithm>
#include <cstddef>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "k_nms.cuh"
#include "k_percentile.cuh"
#include "k_prune.cuh"
#include "k_scale_space.cuh"
#include "k_band.cuh"
#include "k_tc.cuh"
#include "k_tc2.cuh"
#include "k_twopass.cuh"
#include "k_downsample.cuh"

using namespace mhfd;

constexpr int kStageSlots = 3;   // host path: staging slots of `chunk` images each

struct mhfd_ctx {
  mhfd_params p;
  LevelTable* tab;   // host copy, passed by value to k_scale_space
  LevelTable* ltab;  // LoG response (reading R23): 2n sub-levels {w_i, w2_i} (k_rows_pair / k_cols_pair<true>)
  int n;             // DoG planes
  double dt;
  double t[kMaxLevels];
  double rad[kMaxLevels];
  double radmax;
  int64_t cap;       // candidates per image
  int prune_grid;    // cooperative grid size for k_prune
  int sms;
  int band_enabled;  // MHFD_NO_BAND=1 in the environment forces the generic schedule
  int band_kind;     // 3 = k_tc (default), 1 = k_band (params.schedule, else MHFD_SCHEDULE=tc|band|generic)
  int twopass;       // generic path for large radii: k_rows2 / k_cols_all (MHFD_NO_TWOPASS=1 disables)
  TcPlan* tc;        // tensor-core geometry (host copy, passed by value to k_tc)
  uint8_t* d_tctab;  // device copy of the Toeplitz pair tables (context-owned, immutable)
  Tc2Plan* tc2;      // two-pass tensor-core geometry (u16 / f32 / large radii), host copy
  uint8_t* d_tc2tab; // its device pair tables (context-owned, immutable)
  float2* d_thr;     // pruning: n x n squared-distance bands (context-owned, immutable)
  int32_t dmax[kMaxLevels];
  int cs_shift, ncx, nbands;   // pruning cell index: cell edge 1 << cs_shift >= every dmax
  // bench instrumentation (mhfd_timing_*): 5 events per recorded call
  cudaEvent_t* tev;
  int tmax, tcount;
  // e2e host path (mhfd_focus_score_host): copy stream + double-buffer events
  cudaStream_t copy_stream;
  cudaEvent_t ev_ready[kStageSlots], ev_free[kStageSlots], ev_done;   // host path (e2e)
  uint32_t stage_next;         // next staging slot (continues across calls)
  const void* stage_ptr;       // staging buffer / chunk of the previous host-path call
  int stage_chunk;
};

namespace {

constexpr size_t kSmemLimit = 227 * 1024;   // opt-in dynamic shared memory per CTA on sm_100
constexpr int kRxBatch = 8;                   // images per two-pass chunk (Rx workspace)

thread_local std::string g_err;
thread_local int32_t g_launches = 0;

mhfd_status fail(mhfd_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

mhfd_status cuda_fail(cudaError_t e, const char* where) {
  return fail(MHFD_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t par, sel, hist1, hist2, fimg, v, idx, v2, idx2, dog, segcnt, segoff, ncand, cand, st, rowstart, cellstart, crec, imgoff, chunkoff,
      chunkcnt, chunkpos, counters, scores, counts, rx, xtc, slab, wl, total;
};

// k_tc2 (two-pass tensor-core schedule) applies: Eq. 2 DoG or LoG, periodic, plan built, widths
// in whole 128-column tiles, heights in whole 16-row slabs, one periodic wrap of the
// staged row window
bool tc2_fit(const mhfd_ctx* c) {   // (a LoG context's plan holds its 2n sub-levels; reflect: tc2_geom)
  return c->tc2 && c->d_tc2tab && c->band_enabled && c->p.width % kT2Cols == 0 &&
         c->p.height % kT2SlabRows == 0 && c->p.width >= c->tc2->S;
}
// Reflect (reading R25) on k_tc2: the stretched image is staged with mirrored margins,
// pg column groups of 8 left and right and pr rows above and below, so neither pass
// wraps: Rx is computed for hx = H + 2 pr rows (slab row r = image row r - pr) and each
// window is one contiguous run.  Periodic: pg = pr = 0, hx = H (the passes wrap).
struct Tc2Geom {
  int pg, pr, hx, xw;   // margin groups, margin rows, Rx rows, staged X width (pixels)
};
Tc2Geom tc2_geom(const mhfd_ctx* c) {
  Tc2Geom g{0, 0, c->p.height, c->p.width};
  if (c->p.boundary == MHFD_BOUNDARY_REFLECT) {
    g.pg = c->tc2->H0 / 8;
    g.pr = (c->tc2->rmax + 16 + 15) / 16 * 16;
    g.hx = c->p.height + 2 * g.pr;
    g.xw = c->p.width + 16 * g.pg;
  }
  return g;
}
int tc2_nrt(const mhfd_ctx* c) { return (tc2_geom(c).hx + c->tc2->NR - 1) / c->tc2->NR; }

// k_tc splits each tile's levels over two CTAs when the call has at most half as many
// tiles as SMs (one 1024^2 tile: 64 tiles on 148 SMs), whole images only
bool tc_parts(const mhfd_ctx* c, int B) {
  if (!c->tc) return false;
  const int64_t tiles = (int64_t)((c->p.width + kTcTile - 1) / kTcTile) * ((c->p.height + kTcTile - 1) / kTcTile) * B;
  return c->tc->nlev >= 3 && tiles * 2 <= c->sms;
}
// the level both parts compute: balances sum_i (K_i^2/16 + 12 K_i) (row + column pass
// MMA cycles) between [0, m] and [m, nlev)
int tc_lsplit(const TcPlan& P) {
  std::vector<double> cost(P.nlev);
  for (int i = 0; i < P.nlev; ++i) cost[i] = P.lev[i].K * (double)P.lev[i].K / 16.0 + 12.0 * P.lev[i].K;
  int best = 1;
  double bmax = 1e300;
  for (int m = 1; m + 1 < P.nlev; ++m) {
    double a = 0, b = 0;
    for (int i = 0; i <= m; ++i) a += cost[i];
    for (int i = m; i < P.nlev; ++i) b += cost[i];
    if (std::max(a, b) < bmax) { bmax = std::max(a, b); best = m; }
  }
  return best;
}

int nseg_of(const mhfd_ctx* c) {
  const int64_t plane = (int64_t)c->p.width * c->p.height;
  return (int)((plane + kSeg - 1) / kSeg);
}

// pruning worklist capacity (records of blobs left undecided by round 0; overflow falls
// back to the geometric search, so this is a size/speed trade, not a correctness bound)
int64_t wl_cap_of(const mhfd_ctx* c, int B) {
  const int64_t all = c->cap * (int64_t)B;
  return std::min(all, ((int64_t)1 << 20) + all / 64);
}

// paper-mode two-pass kernels (k_rows_pair / k_cols_pair) fit; MHFD_NO_COLS_PAIR=1 selects
// k_rows2 / k_cols_all instead
bool pair_fit(const mhfd_ctx* c) {
  const LevelTable& T = *c->tab;
  return c->band_enabled && c->p.width % kR3Cols == 0 && c3_smem(T.rmax) <= kSmemLimit &&
         r3_smem(T.rmax, r3_taps_total(T)) <= kSmemLimit && getenv("MHFD_NO_COLS_PAIR") == nullptr;
}
bool pair_ok(const mhfd_ctx* c) {
  return (c->p.nms == MHFD_NMS_PAPER || c->p.boundary == MHFD_BOUNDARY_REFLECT) && pair_fit(c);
}

Layout layout(const mhfd_ctx* c, int B) {
  Layout L{};
  const int64_t plane = (int64_t)c->p.width * c->p.height;
  const int64_t nseg = nseg_of(c);
  const int64_t nchunk = (c->cap + kChunk - 1) / kChunk;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o += align256(bytes); return at; };
  L.par = take(sizeof(ImgPar) * B);
  L.sel = take(sizeof(SelState) * B);
  L.hist1 = take(sizeof(uint32_t) * 257 * B);   // 256 bins per image, then per-image tickets (u8 select)
  L.hist2 = take(sizeof(uint32_t) * 513 * B);   // 2 x 256 bins per image, then per-image tickets (u16 pass 2)
  L.fimg = take(sizeof(float) * plane * B);
  const bool paper = c->p.nms == MHFD_NMS_PAPER;
  L.v = take(paper ? sizeof(float) * plane * B : 0);
  L.idx = take(paper ? plane * B : 0);
  // k_tc's level parts (calls with fewer than half as many tiles as SMs): part 1's v / argmax
  const bool parts = paper && tc_parts(c, B);
  L.v2 = take(parts ? sizeof(float) * plane * B : 0);
  L.idx2 = take(parts ? plane * B : 0);
  L.dog = take(paper ? 0 : sizeof(float) * plane * c->n * B);
  L.segcnt = take(sizeof(int32_t) * nseg * B);
  L.segoff = take(sizeof(int32_t) * nseg * B);
  L.ncand = take(sizeof(int32_t) * B);
  L.cand = take(sizeof(mhfd_blob) * c->cap * B);
  L.st = take(c->cap * B);
  L.rowstart = take(sizeof(int32_t) * (c->p.height + 1) * (size_t)B);
  L.cellstart = take(sizeof(int32_t) * (size_t)c->nbands * 2 * (c->ncx + 1) * (size_t)B);   // pruning cell index
  L.crec = take(sizeof(int4) * c->cap * (size_t)B);
  L.imgoff = take(sizeof(int64_t) * (B + 1));
  L.chunkoff = take(sizeof(int64_t) * (B + 1));
  L.chunkcnt = take(sizeof(int32_t) * nchunk * B);
  L.chunkpos = take(sizeof(int32_t) * nchunk * B);
  L.counters = take(sizeof(int32_t) * 64);   // k_prune: [0, 9); mhfd_prune_band's tally: 12, 13; [16, 64): PRUNE_STAMPS
  L.scores = take(sizeof(double) * B);
  L.counts = take(sizeof(int32_t) * B);
  // two-pass schedules: Rx of every level (LoG: of each of the 2n sub-levels) for up to
  // kRxBatch images (run_front chunks larger batches)
  const int64_t rxb = std::min(B, kRxBatch);
  const bool any2 = c->ltab || c->twopass || pair_fit(c);
  const int64_t rx_rows = tc2_fit(c) ? std::max<int64_t>(c->p.height, tc2_geom(c).hx) : c->p.height;
  L.rx = take(any2 || tc2_fit(c) ? sizeof(float) * (int64_t)c->p.width * rx_rows * rxb * (c->ltab ? 2 * c->n : c->n + 1)
                                 : 0);
  // k_tc2: the stretched image as tiled fp16 hi/lo planes (rows padded to whole NR tiles)
  L.xtc = take(tc2_fit(c) ? 2 * t2_x_plane_bytes(tc2_geom(c).xw, tc2_nrt(c), c->tc2->NR) * rxb : 0);
  // NMS fast path (W % kSeg == 0): every segment parks up to kSlab records during the count
  L.slab = take(c->p.width % kSeg == 0 ? sizeof(mhfd_blob) * kSlab * (size_t)nseg * B : 0);   // both NMS modes
  L.wl = take(sizeof(int32_t) * 8 * (size_t)wl_cap_of(c, B));   // pruning worklist (k_prune.cuh)
  L.total = o;
  return L;
}

mhfd_status check_call(const mhfd_ctx* c, const void* d_images, int32_t dtype, int32_t batch, int64_t pitch,
                       const void* ws, size_t ws_bytes) {
  if (!c) return fail(MHFD_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (!d_images) return fail(MHFD_ERR_INVALID_ARGUMENT, "d_images is NULL");
  if (dtype != MHFD_U8 && dtype != MHFD_U16 && dtype != MHFD_F32)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "dtype %d", dtype);
  if (batch < 1) return fail(MHFD_ERR_SHAPE, "batch %d < 1", batch);
  const int bpp = dtype == MHFD_U8 ? 1 : dtype == MHFD_U16 ? 2 : 4;
  if (pitch < (int64_t)c->p.width * bpp || pitch % 16 != 0)
    return fail(MHFD_ERR_SHAPE, "pitch_bytes %lld: need >= width*bpp and a multiple of 16", (long long)pitch);
  if (((uintptr_t)d_images) % 16 != 0) return fail(MHFD_ERR_SHAPE, "d_images not 16-byte aligned");
  if (!ws) return fail(MHFD_ERR_WORKSPACE, "workspace is NULL");
  if (((uintptr_t)ws) % 256 != 0) return fail(MHFD_ERR_WORKSPACE, "workspace not 256-byte aligned");
  const size_t need = layout(c, batch).total;
  if (ws_bytes < need) return fail(MHFD_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != c->p.device)
    return fail(MHFD_ERR_DEVICE, "current device %d != context device %d", dev, c->p.device);
  return MHFD_OK;
}

#define LAUNCH_CHECK(where)                                  \
  do {                                                       \
    cudaError_t e_ = cudaGetLastError();                     \
    if (e_ != cudaSuccess) return cuda_fail(e_, where);      \
    ++launches;                                              \
  } while (0)

// Everything up to the candidate list.  dog_dump (nullable) receives the DoG planes.
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
bool encode_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t cols, uint64_t rows,
               uint64_t row_bytes, uint32_t box_cols, uint32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)row_bytes};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(m, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaEvent_t* next_timing(mhfd_ctx* c) {
  if (!c->tev || c->tcount >= c->tmax) return nullptr;
  return c->tev + 5 * (c->tcount++);
}

#define MARK(k)                                                     \
  do {                                                              \
    if (ev) {                                                       \
      cudaError_t em_ = cudaEventRecord(ev[k], st);                 \
      if (em_ != cudaSuccess) return cuda_fail(em_, "event record"); \
    }                                                               \
  } while (0)

mhfd_status run_nms(mhfd_ctx* c, int W, int H, int B, char* ws, const Layout& L, float* v, uint8_t* idx,
                    float* dog, cudaStream_t st, int& launches, cudaEvent_t* ev, int band_lo = 0, int band_hi = 0) {
  const bool paper = c->p.nms == MHFD_NMS_PAPER;
  // ---- a7-a8: NMS + threshold + ordered compaction
  NmsArgs na{W, H, c->n, c->p.threshold, c->p.strict, v, idx, dog};
  const bool band = band_lo < band_hi;
  const int row0 = band ? band_lo : 0, row1 = band ? band_hi : H;
  const int nseg = band ? (int)((int64_t)(row1 - row0) * W / kSeg) : nseg_of(c);   // band: W % kSeg == 0
  int32_t* segcnt = reinterpret_cast<int32_t*>(ws + L.segcnt);
  int32_t* segoff = reinterpret_cast<int32_t*>(ws + L.segoff);
  int32_t* ncand = reinterpret_cast<int32_t*>(ws + L.ncand);
  mhfd_blob* cand = reinterpret_cast<mhfd_blob*>(ws + L.cand);
  mhfd_blob* slab = reinterpret_cast<mhfd_blob*>(ws + L.slab);
  dim3 gn((nseg + 7) / 8, B);
  const bool rows_fast = paper && (W % kSeg) == 0;   // segments are whole-row pieces
  static const bool nms26_generic = getenv("MHFD_NMS26_GENERIC") != nullptr;   // A/B knob
  const bool rows26 = !paper && (W % kSeg) == 0 && !nms26_generic;
  const dim3 gr((((row1 - row0 + kNmsRows - 1) / kNmsRows) * (W / kSeg) + 7) / 8, B);   // kNmsRows segments per warp
  // k_nms_roll<8> is the default count pass (NMS stage 1.695 -> 1.551 ms per 64 tiles
  // against k_nms_rows; <4> 1.603); MHFD_NMS_ROLL=0/4/8 selects for A/B runs
  static const int roll = [] { const char* e = getenv("MHFD_NMS_ROLL"); return e ? atoi(e) : 8; }();
  if (rows_fast && (roll == 8 || roll == 4 || roll == 2 || roll == 1)) {
    // rows per warp: 8 when there is work for two waves of warp slots (3 CTAs x 8 warps per SM),
    // fewer for small calls, where the warps' serial row walks set the latency (one
    // 4096^2 tile: 256 CTAs of 8-row warps; one 1024^2 tile: 16)
    int nr = roll;
    while (nr > 1 && (int64_t)((row1 - row0 + nr - 1) / nr) * (W / kSeg) * B < (int64_t)c->sms * 48) nr >>= 1;
    const dim3 g8((((row1 - row0 + nr - 1) / nr) * (W / kSeg) + 7) / 8, B);
    if (nr == 8) k_nms_roll<8><<<g8, 256, 0, st>>>(na, nseg, segcnt, row0, row1, slab);
    else if (nr == 4) k_nms_roll<4><<<g8, 256, 0, st>>>(na, nseg, segcnt, row0, row1, slab);
    else if (nr == 2) k_nms_roll<2><<<g8, 256, 0, st>>>(na, nseg, segcnt, row0, row1, slab);
    else k_nms_roll<1><<<g8, 256, 0, st>>>(na, nseg, segcnt, row0, row1, slab);
  } else if (rows_fast) {
    k_nms_rows<false><<<gr, 256, 0, st>>>(na, nseg, segcnt, nullptr, nullptr, 0, row0, row1, slab);
  } else if (rows26) {
    k_nms26_roll<<<dim3((unsigned)(((int64_t)(row1 - row0) * (W / kSeg) + 7) / 8), B), 256, 0, st>>>(
        na, nseg, segcnt, row0, row1, slab);
  } else if (paper) {
    k_nms_count<MHFD_NMS_PAPER><<<gn, 256, 0, st>>>(na, nseg, segcnt);
  } else {
    k_nms_count<MHFD_NMS_26><<<gn, 256, 0, st>>>(na, nseg, segcnt);
  }
  LAUNCH_CHECK("k_nms_count");
  k_seg_scan<<<B, 1024, 0, st>>>(segcnt, nseg, segoff, ncand);
  LAUNCH_CHECK("k_seg_scan");
  if (rows_fast) {   // parked records to their offsets (overflowing segments re-evaluated)
    static const bool g1 = getenv("MHFD_NMS_GATHER1") != nullptr;   // A/B knob: one warp per segment
    if (g1) k_nms_gather<<<gn, 256, 0, st>>>(na, nseg, segcnt, segoff, slab, cand, c->cap, row0);
    else k_nms_gather4<<<dim3((nseg + 31) / 32, B), 256, 0, st>>>(na, nseg, segcnt, segoff, slab, cand, c->cap, row0);
  } else if (rows26) {
    k_nms_gather4<MHFD_NMS_26><<<dim3((nseg + 31) / 32, B), 256, 0, st>>>(na, nseg, segcnt, segoff, slab, cand,
                                                                          c->cap, row0);
  } else if (paper) {
    k_nms_write<MHFD_NMS_PAPER><<<gn, 256, 0, st>>>(na, nseg, segoff, cand, c->cap);
  } else {
    k_nms_write<MHFD_NMS_26><<<gn, 256, 0, st>>>(na, nseg, segoff, cand, c->cap);
  }
  LAUNCH_CHECK("k_nms_write");
  MARK(3);
  return MHFD_OK;
}

// band_lo < band_hi: single-image band mode (mhfd_detect_band): blur/DoG/argmax for rows
// [band_lo - 1, band_hi + 1) of the image, Eq. 3 NMS + compaction for rows [band_lo, band_hi)
mhfd_status run_front(mhfd_ctx* c, const void* d_images, int32_t dtype, int32_t B, int64_t pitch, char* ws,
                      const Layout& L, float* dog_dump, cudaStream_t st, int& launches, cudaEvent_t* ev,
                      int band_lo = 0, int band_hi = 0) {
  MARK(0);
  const int W = c->p.width, H = c->p.height;
  const int bpp = dtype == MHFD_U8 ? 1 : dtype == MHFD_U16 ? 2 : 4;
  const Shape s{W, H, pitch, bpp};
  const uint8_t* img = static_cast<const uint8_t*>(d_images);
  ImgPar* par = reinterpret_cast<ImgPar*>(ws + L.par);
  SelState* sel = reinterpret_cast<SelState*>(ws + L.sel);
  uint32_t* h1 = reinterpret_cast<uint32_t*>(ws + L.hist1);
  uint32_t* h2 = reinterpret_cast<uint32_t*>(ws + L.hist2);

  // ---- a1: percentiles
  const int64_t N = (int64_t)W * H;
  RankPar rp;
  rp.npx = N;
  rp.rank_lo = std::min<int64_t>((int64_t)std::floor((double)c->p.sat_low * (double)N), N - 1);
  rp.rank_hi = N - 1 - std::min<int64_t>((int64_t)std::floor((double)c->p.sat_high * (double)N), N - 1);
  cudaError_t e = bpp == 4 ? cudaSuccess : cudaMemsetAsync(ws + L.hist1, 0, sizeof(uint32_t) * 257 * B, st);
  if (e == cudaSuccess && bpp >= 2) e = cudaMemsetAsync(ws + L.hist2, 0, sizeof(uint32_t) * 513 * B, st);
  if (e != cudaSuccess) return cuda_fail(e, "memset hist");
  // ~2 CTAs per SM of rows (fewer, fuller CTAs: each flushes 256 global atomics)
  int rows_per_cta = std::max(1, (int)(((int64_t)H * B + 2 * c->sms - 1) / (2 * c->sms)));
  rows_per_cta = std::min(rows_per_cta, 64);
  dim3 hg((H + rows_per_cta - 1) / rows_per_cta, B);
  if (bpp == 4) {   // f32 (reading R24): 4 radix-select passes of 8 key bits
    k_hist_f32<0><<<hg, 256, 0, st>>>(img, s, rows_per_cta, h2, sel);
    k_select_f32<0><<<(B + 3) / 4, 128, 0, st>>>(h2, rp, sel, par, B);
    k_hist_f32<1><<<hg, 256, 0, st>>>(img, s, rows_per_cta, h2, sel);
    k_select_f32<1><<<(B + 3) / 4, 128, 0, st>>>(h2, rp, sel, par, B);
    k_hist_f32<2><<<hg, 256, 0, st>>>(img, s, rows_per_cta, h2, sel);
    k_select_f32<2><<<(B + 3) / 4, 128, 0, st>>>(h2, rp, sel, par, B);
    k_hist_f32<3><<<hg, 256, 0, st>>>(img, s, rows_per_cta, h2, sel);
    k_select_f32<3><<<(B + 3) / 4, 128, 0, st>>>(h2, rp, sel, par, B);
    LAUNCH_CHECK("k_hist_f32 / k_select_f32");
    launches += 7;
  } else if (bpp == 1) {   // histogram + select in one launch (the image's last CTA selects)
    k_hist<1, false, true><<<hg, 256, 0, st>>>(img, s, rows_per_cta, h1, sel, rp, par, h1 + 256 * B);
    LAUNCH_CHECK("k_hist");
  } else {
    // two radix passes, each selecting in its last CTA per image (no k_select1 / k_select2)
    k_hist<2, false, true><<<hg, 256, 0, st>>>(img, s, rows_per_cta, h1, sel, rp, par, h1 + 256 * B);
    LAUNCH_CHECK("k_hist");
    k_hist<2, true, true><<<hg, 256, 0, st>>>(img, s, rows_per_cta, h2, sel, rp, par, h2 + 512 * B);
    LAUNCH_CHECK("k_hist2");
  }

  MARK(1);
  const bool paper = c->p.nms == MHFD_NMS_PAPER;
  float* v = reinterpret_cast<float*>(ws + L.v);
  uint8_t* idx = reinterpret_cast<uint8_t*>(ws + L.idx);
  // ---- a2-a6 on u8 images on the tensor cores (banded-Toeplitz blur)
  const bool band = band_lo < band_hi;
  // k_tc also writes the DoG planes: for the 26-neighbour NMS and for debug dumps
  float* tc_dog = dog_dump ? dog_dump : (paper ? nullptr : reinterpret_cast<float*>(ws + L.dog));
  const bool dogr = c->p.response == MHFD_RESPONSE_DOG;
  const int reflect = c->p.boundary == MHFD_BOUNDARY_REFLECT ? 1 : 0;   // reading R25: k_tc (u8) or two-pass
  const bool fused_ok = dogr && !reflect;   // k_band: periodic only; k_tc mirrors its windows (P.reflect)
  if (dogr && bpp == 1 && c->band_enabled && c->band_kind == 3 && c->d_tctab && tc_ok(*c->tc, W, H) &&
      (!band || (paper && dog_dump == nullptr))) {
    const TcPlan& P = *c->tc;
    const size_t smem = tc_smem(P);
    const int nparts = (!band && paper && tc_parts(c, B)) ? 2 : 1;
    auto kern = reflect ? (tc_dog ? (nparts > 1 ? k_tc<true, 2, true> : k_tc<true, 1, true>)
                                  : (nparts > 1 ? k_tc<false, 2, true> : k_tc<false, 1, true>))
                        : (tc_dog ? (nparts > 1 ? k_tc<true, 2> : k_tc<true, 1>)
                                  : (nparts > 1 ? k_tc<false, 2> : k_tc<false, 1>));
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea != cudaSuccess) return cuda_fail(ea, "k_tc attribute");
    // band mode: rows [band_lo - 1, band_hi + 1) on the whole image's 128-row tile grid, so
    // every pixel sees the same K-step grouping (and rounding) as in the whole-image run
    const int r_lo = band ? std::max(0, band_lo - 1) / kTcTile * kTcTile : 0;
    const int r_hi = band ? std::min(H, (std::min(H, band_hi + 1) + kTcTile - 1) / kTcTile * kTcTile) : H;
    const int lsplit = nparts > 1 ? tc_lsplit(P) : 0;
    const int64_t ntiles = (int64_t)((W + kTcTile - 1) / kTcTile) * ((r_hi - r_lo + kTcTile - 1) / kTcTile) * B * nparts;
    int64_t grid = std::min<int64_t>(ntiles, c->sms);   // persistent: one CTA per SM
    if (nparts > 1) grid &= ~(int64_t)1;                 // even: a CTA's units share a part
    dim3 gb((unsigned)grid);
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    const int use_tm = (pitch % 16 == 0) && encode_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, img, (uint64_t)W,
                                                      (uint64_t)H * B, (uint64_t)pitch, (uint32_t)tc_lw(P),
                                                      (uint32_t)P.S);
    float* v2 = reinterpret_cast<float*>(ws + L.v2);
    uint8_t* idx2 = reinterpret_cast<uint8_t*>(ws + L.idx2);
    kern<<<gb, kTcThreads + 32, smem, st>>>(img, s, par, P, c->d_tctab, tm, use_tm, paper ? v : nullptr,
                                            paper ? idx : nullptr, tc_dog, B, r_lo, r_hi, lsplit, v2, idx2,
                                            nullptr);
    LAUNCH_CHECK("k_tc");
    if (nparts > 1) {
      const int64_t n4 = (int64_t)W * H * B / 4;
      k_merge_parts<<<(unsigned)std::min<int64_t>((n4 + 255) / 256, c->sms * 8), 256, 0, st>>>(v, idx, v2, idx2, n4);
      LAUNCH_CHECK("k_merge_parts");
    }
    MARK(2);
    return run_nms(c, W, H, B, ws, L, v, idx, paper ? nullptr : tc_dog, st, launches, ev, band_lo, band_hi);
  }
  // ---- a2-a6 on the two-pass tensor-core schedule (u16 / f32 images, u8 beyond k_tc's tile)
  if (tc2_fit(c) && c->band_kind == 3 && (!band || (paper && dog_dump == nullptr && !reflect))) {
    const Tc2Plan& P = *c->tc2;
    const int nrt = tc2_nrt(c);
    const Tc2Geom gm = tc2_geom(c);   // reflect: mirrored margins, no wrap
    // row tiles of k_tc2_rows and output row tiles of k_tc2_cols: everything, or in band
    // mode (f2) only the 256-row output tiles that cover [band_lo - 1, band_hi + 1) on the
    // whole image's grid and the NR-row tiles holding the Rx rows their windows read (at
    // most two ranges: the periodic wrap), so every response equals the whole-image run's
    int yt0 = 0, nyt = (H + kT2ColRows - 1) / kT2ColRows;
    int rr[2][2] = {{0, nrt}, {0, 0}};
    if (band) {
      const int o_lo = std::max(0, band_lo - 1), o_hi = std::min(H, band_hi + 1);
      yt0 = o_lo / kT2ColRows;
      nyt = (o_hi + kT2ColRows - 1) / kT2ColRows - yt0;
      const int lo = yt0 * kT2ColRows - P.rmax - kT2SlabRows, hi = (yt0 + nyt) * kT2ColRows + P.rmax + kT2SlabRows;
      if (hi - lo < H) {
        auto tiles = [&](int a, int z, int (&r)[2]) { r[0] = a / P.NR; r[1] = (z + P.NR - 1) / P.NR; };
        tiles(std::max(0, lo), std::min(H, hi), rr[0]);
        rr[1][0] = rr[1][1] = 0;
        if (lo < 0) tiles(H + lo, H, rr[1]);
        if (hi > H) tiles(0, hi - H, rr[1]);
      }
    }
    const size_t sm1 = tc2_rows_smem(P), sm2 = tc2_cols_smem(P);
    auto kc = reflect ? (dogr ? (tc_dog ? k_tc2_cols<true, false, true> : k_tc2_cols<false, false, true>)
                              : (tc_dog ? k_tc2_cols<true, true, true> : k_tc2_cols<false, true, true>))
                      : (dogr ? (tc_dog ? k_tc2_cols<true> : k_tc2_cols<false>)
                              : (tc_dog ? k_tc2_cols<true, true> : k_tc2_cols<false, true>));
    cudaError_t ea = cudaFuncSetAttribute(k_tc2_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    if (ea == cudaSuccess) ea = cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    if (ea != cudaSuccess) return cuda_fail(ea, "k_tc2 attributes");
    uint8_t* xt = reinterpret_cast<uint8_t*>(ws + L.xtc);
    uint8_t* rx = reinterpret_cast<uint8_t*>(ws + L.rx);
    const int64_t plane = (int64_t)W * H;
    for (int b0 = 0; b0 < B; b0 += kRxBatch) {
      const int Bc = std::min(kRxBatch, B - b0);
      const uint8_t* ic = img + (int64_t)b0 * H * pitch;
      const ImgPar* pc = par + b0;
      const int64_t work = (int64_t)Bc * nrt * P.NR * (gm.xw / 8);
      const dim3 gp((unsigned)std::min<int64_t>((work + 255) / 256, (int64_t)c->sms * 16));
      if (bpp == 1) k_tc2_prep<1><<<gp, 256, 0, st>>>(ic, s, pc, xt, P.NR, nrt, Bc, gm.pg, gm.pr);
      else if (bpp == 2) k_tc2_prep<2><<<gp, 256, 0, st>>>(ic, s, pc, xt, P.NR, nrt, Bc, gm.pg, gm.pr);
      else k_tc2_prep<4><<<gp, 256, 0, st>>>(ic, s, pc, xt, P.NR, nrt, Bc, gm.pg, gm.pr);
      LAUNCH_CHECK("k_tc2_prep");
      for (int k = 0; k < 2; ++k) {
        if (rr[k][1] <= rr[k][0]) continue;
        const int64_t t1 = (int64_t)(W / kT2Cols) * (rr[k][1] - rr[k][0]) * Bc;
        k_tc2_rows<<<(unsigned)std::min<int64_t>(t1, c->sms), kT2Threads, sm1, st>>>(
            xt, P, c->d_tc2tab, rx, W, gm.hx, Bc, nrt, rr[k][0], rr[k][1] - rr[k][0], gm.pg);
        LAUNCH_CHECK("k_tc2_rows");
      }
      const int64_t t2 = (int64_t)(W / kT2Cols) * nyt * Bc;
      kc<<<(unsigned)std::min<int64_t>(t2, c->sms), kT2Threads, sm2, st>>>(
          rx, pc, P, c->d_tc2tab, paper ? v + (int64_t)b0 * plane : nullptr, paper ? idx + (int64_t)b0 * plane : nullptr,
          tc_dog ? tc_dog + (int64_t)b0 * c->n * plane : nullptr, W, H, Bc, yt0, nyt, gm.hx, gm.pr);
      LAUNCH_CHECK("k_tc2_cols");
    }
    MARK(2);
    return run_nms(c, W, H, B, ws, L, v, idx, paper ? nullptr : tc_dog, st, launches, ev, band_lo, band_hi);
  }
  if (band && !(c->p.response == MHFD_RESPONSE_DOG && paper && dog_dump == nullptr && pair_fit(c)))
    return fail(MHFD_ERR_INVALID_ARGUMENT, "band mode needs the k_tc or the two-pass pair schedule (Eq. 3 NMS)");
  // ---- a2-a6 on u8 images: band schedule (raw band staged once per CTA, no f32 prepass)
  if (fused_ok && bpp == 1 && paper && dog_dump == nullptr && c->band_enabled &&
      band_ok(W, H, c->tab->rmax, c->tab->ntaps_total)) {
    const size_t smem = band_smem(c->tab->rmax, c->tab->ntaps_total);
    cudaError_t ea = cudaFuncSetAttribute(k_band, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea != cudaSuccess) return cuda_fail(ea, "k_band attribute");
    const int64_t ntiles = (int64_t)((W + kStripW - 1) / kStripW) * ((H + kBandBH - 1) / kBandBH) * B;
    dim3 gb((unsigned)std::min<int64_t>(ntiles, c->sms));   // persistent: one CTA per SM
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    const int use_tm = (pitch % 16 == 0) &&
                       encode_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, img, (uint64_t)W, (uint64_t)H * B, (uint64_t)pitch,
                                 (uint32_t)band_raw_w(c->tab->rmax), (uint32_t)kBandBoxRows);
    k_band<<<gb, kBandThreads, smem, st>>>(img, s, par, *c->tab, tm, use_tm, v, idx, B);
    LAUNCH_CHECK("k_band");
    MARK(2);
    return run_nms(c, W, H, B, ws, L, v, idx, nullptr, st, launches, ev);
  }
  // ---- a2: stretch on load -> centred f32 image
  float* fimg = reinterpret_cast<float*>(ws + L.fimg);
  // single-image bands (pair schedule): only the rows the band's Rx ranges read, by
  // offsetting the image and the output (B = 1)
  int nr[2][2] = {{0, H}, {0, 0}};
  if (band) {
    const LevelTable& T = *c->tab;
    const int o_lo = std::max(0, band_lo - 1), o_hi = std::min(H, band_hi + 1);
    const int lo = o_lo / 8 * 8 - T.rmax, hi = std::min(H, (o_hi + 7) / 8 * 8) + T.rmax;
    if (hi - lo < H) {
      nr[0][0] = std::max(0, lo);
      nr[0][1] = std::min(H, hi);
      if (lo < 0) { nr[1][0] = H + lo; nr[1][1] = H; }
      if (hi > H) { nr[1][0] = 0; nr[1][1] = hi - H; }
      for (int k = 0; k < 2; ++k)   // whole 32-row tiles of the row pass
        if (nr[k][1] > nr[k][0]) { nr[k][0] = nr[k][0] / 32 * 32; nr[k][1] = std::min(H, (nr[k][1] + 31) / 32 * 32); }
    }
  }
  for (int k = 0; k < 2; ++k) {
    if (nr[k][1] <= nr[k][0]) continue;
    const int Hk = nr[k][1] - nr[k][0];
    const Shape sk{W, Hk, pitch, bpp};
    const uint8_t* ik = img + (int64_t)nr[k][0] * pitch;
    float* fk = fimg + (int64_t)nr[k][0] * W;
    const int64_t plane = (int64_t)W * Hk;
    const bool vec = (bpp == 1) ? (W % 16 == 0) : (bpp == 2) ? (W % 8 == 0) : (W % 4 == 0);
    const int64_t work = vec ? plane / (16 / bpp) : plane;
    dim3 gn((unsigned)std::min<int64_t>((work + 255) / 256, (int64_t)c->sms * 8), B);
    if (bpp == 4) {
      k_normalize_f32<<<gn, 256, 0, st>>>(ik, sk, par, fk);
    } else if (vec) {
      if (bpp == 1) k_normalize_vec<1><<<gn, 256, 0, st>>>(ik, sk, par, fk);
      else k_normalize_vec<2><<<gn, 256, 0, st>>>(ik, sk, par, fk);
    } else {
      if (bpp == 1) k_normalize<1><<<gn, 256, 0, st>>>(ik, sk, par, fk);
      else k_normalize<2><<<gn, 256, 0, st>>>(ik, sk, par, fk);
    }
    LAUNCH_CHECK("k_normalize");
  }
  // ---- a3-a6: fused blur + DoG + argmax
  float* dog = dog_dump ? dog_dump : reinterpret_cast<float*>(ws + L.dog);
  const bool write_dog = dog_dump != nullptr || !paper;
  // ---- two passes through an HBM row-blur intermediate (k_twopass.cuh): the LoG response
  // (always), the paper-mode DoG pair kernels (any radius: 1.5x the fused generic kernel
  // on u16 at sigma 1-10), and large radii with DoG planes
  // (k_rows2 / k_cols_all).  Rx holds at most kRxBatch images: larger batches run in chunks.
  const bool pair = dogr && pair_fit(c) && (reflect || (paper && !write_dog));
  const bool big = dogr && !pair && !reflect && c->twopass && W % kR2Cols == 0;
  if (reflect && dogr && !pair)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "reflect boundary needs the two-pass schedule (MHFD_SCHEDULE/NO_COLS_PAIR)");
  if (!dogr || pair || big) {
    const LevelTable& T = dogr ? *c->tab : *c->ltab;
    float* rx = reinterpret_cast<float*>(ws + L.rx);
    const int64_t plane = (int64_t)W * H;
    const bool rows_pair = !big;
    const size_t sm_p = rows_pair ? r3_smem(T.rmax, r3_taps_total(T)) : rows2_smem(T.rmax);
    const size_t sm_c = rows_pair ? c3_smem(T.rmax) : cols2_smem(T.rmax);
    cudaError_t ea = rows_pair ? cudaFuncSetAttribute(k_rows_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_p)
                               : cudaFuncSetAttribute(k_rows2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_p);
    if (ea == cudaSuccess)
      ea = !dogr ? cudaFuncSetAttribute(k_cols_pair<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_c)
           : pair ? cudaFuncSetAttribute(k_cols_pair<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_c)
                  : cudaFuncSetAttribute(k_cols_all, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_c);
    if (ea != cudaSuccess) return cuda_fail(ea, "two-pass attributes");
    const int nplanes = c->n;   // DoG / LoG planes written for the 26 mode and dumps
    // single-image band (f2): output tiles covering rows [band_lo - 1, band_hi + 1) on the
    // whole image's 256-row grid (same sums as the whole-image run), and only the Rx rows
    // their windows read, as at most two row ranges (the periodic wrap)
    int ct0 = 0, nct = (H + kC2Rows - 1) / kC2Rows, need_lo = 0, need_hi = H;
    int rr[2][2] = {{0, H}, {0, 0}};   // Rx row ranges [start, end)
    if (band) {
      const int o_lo = std::max(0, band_lo - 1), o_hi = std::min(H, band_hi + 1);
      ct0 = o_lo / kC2Rows;
      nct = (o_hi + kC2Rows - 1) / kC2Rows - ct0;
      need_lo = o_lo;   // k_cols_pair skips 8-row groups outside [o_lo, o_hi)
      need_hi = o_hi;
      const int lo = o_lo / 8 * 8 - T.rmax, hi = std::min(H, (o_hi + 7) / 8 * 8) + T.rmax;
      if (hi - lo < H) {
        rr[0][0] = std::max(0, lo);
        rr[0][1] = std::min(H, hi);
        if (lo < 0) { rr[1][0] = H + lo; rr[1][1] = H; }
        if (hi > H) { rr[1][0] = 0; rr[1][1] = hi - H; }
      }
    }
    for (int b0 = 0; b0 < B; b0 += kRxBatch) {
      const int Bc = std::min(kRxBatch, B - b0);
      const float* fi = fimg + (int64_t)b0 * plane;
      const ImgPar* pc = par + b0;
      float* vc = paper ? v + (int64_t)b0 * plane : nullptr;
      uint8_t* ic = paper ? idx + (int64_t)b0 * plane : nullptr;
      float* dc = write_dog ? dog + (int64_t)b0 * nplanes * plane : nullptr;
      const dim3 gc((W + kStripW - 1) / kStripW, nct, Bc);
      if (rows_pair) {   // every level's row blur in one launch (per Rx row range)
        for (int k = 0; k < 2; ++k) {
          if (rr[k][1] <= rr[k][0]) continue;
          const int t0 = rr[k][0] / 32, t1 = (rr[k][1] + 31) / 32;
          k_rows_pair<<<dim3(W / kR3Cols, t1 - t0, Bc), kC3Threads, sm_p, st>>>(fi, W, H, T, rx, Bc, reflect, t0);
          LAUNCH_CHECK("k_rows_pair");
        }
      } else {
        for (int lev = 0; lev < T.nlev; ++lev) {
          k_rows2<<<dim3(W / kR2Cols, (H + 31) / 32, Bc), 256, sm_p, st>>>(fi, W, H, T, lev,
                                                                           rx + (int64_t)lev * Bc * plane);
          LAUNCH_CHECK("k_rows2");
        }
      }
      if (!dogr) {
        k_cols_pair<true><<<gc, kC3Threads, sm_c, st>>>(rx, W, H, Bc, T, vc, ic, dc, pc, reflect, ct0, need_lo,
                                                         need_hi);
      } else if (pair) {
        k_cols_pair<false><<<gc, kC3Threads, sm_c, st>>>(rx, W, H, Bc, T, vc, ic, dc, pc, reflect, ct0, need_lo,
                                                          need_hi);
      } else {
        k_cols_all<<<gc, 256, sm_c, st>>>(rx, W, H, Bc, T, vc, ic, dc, pc);
      }
      LAUNCH_CHECK("k_cols");
    }
    MARK(2);
    return run_nms(c, W, H, B, ws, L, v, idx, dog, st, launches, ev, band_lo, band_hi);
  }
  const int strips = (W + kStripW - 1) / kStripW;
  // band height: 256 rows when that still gives >= 4 waves of 2 CTAs/SM, else 128
  const int64_t ctas256 = (int64_t)strips * ((H + 255) / 256) * B;
  const bool fits256 = scale_space_smem(c->tab->rmax, 256, c->tab->ntaps_total) <= kSmemLimit;
  int RPT = (fits256 && ctas256 >= (int64_t)c->sms * 2 * 4) ? 32 : 16;
  int NST = kStages;
  // large radii: 384-row bands with two copy stages (one CTA per SM) when the 256-row
  // band does not fit, if that still gives >= 2 waves: the row pass recomputes
  // (BH + 2R) / BH rows per output
  {
    const int64_t ctas384 = (int64_t)strips * ((H + 383) / 384) * B;
    if (!fits256 && scale_space_smem(c->tab->rmax, 384, c->tab->ntaps_total, 2) <= kSmemLimit &&
        ctas384 >= (int64_t)c->sms * 2 && getenv("MHFD_NO_BH384") == nullptr) {
      RPT = 48;
      NST = 2;
    }
  }
  const int BH = 8 * RPT;
  const size_t smem = scale_space_smem(c->tab->rmax, BH, c->tab->ntaps_total, NST);
  const bool fast = fast_staging(W, c->tab->rmax);
  // 2-D TMA descriptor of the normalised batch viewed as a (B*H) x W f32 matrix
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  int use_tmap = 0;
  if (fast && tma_boxes(c->tab->rmax))
    use_tmap = encode_2d(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, fimg, (uint64_t)W, (uint64_t)H * B, (uint64_t)W * 4,
                         (uint32_t)stage_pitch(c->tab->rmax), (uint32_t)kChunkRows) ? 1 : 0;
  dim3 g3(strips, (H + BH - 1) / BH, B);
  const Shape sf{W, H, (int64_t)W * 4, 4};
  auto launch_ss = [&](auto kern) -> cudaError_t {
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea != cudaSuccess) return ea;
    kern<<<g3, kThreads, smem, st>>>(fimg, sf, par, *c->tab, tmap, use_tmap, v, idx, dog);
    return cudaGetLastError();
  };
#define SS_VARIANTS(RPTV, FASTV)                                                              \
  (paper && write_dog) ? launch_ss(k_scale_space<RPTV, true, true, FASTV>)                    \
  : paper              ? launch_ss(k_scale_space<RPTV, true, false, FASTV>)                   \
                       : launch_ss(k_scale_space<RPTV, false, true, FASTV>)
#define SS_VARIANTS2(RPTV, FASTV)                                                             \
  (paper && write_dog) ? launch_ss(k_scale_space<RPTV, true, true, FASTV, 2>)                 \
  : paper              ? launch_ss(k_scale_space<RPTV, true, false, FASTV, 2>)                \
                       : launch_ss(k_scale_space<RPTV, false, true, FASTV, 2>)
  cudaError_t es;
  if (RPT == 48) es = fast ? (SS_VARIANTS2(48, true)) : (SS_VARIANTS2(48, false));
  else if (RPT == 32) es = fast ? (SS_VARIANTS(32, true)) : (SS_VARIANTS(32, false));
  else es = fast ? (SS_VARIANTS(16, true)) : (SS_VARIANTS(16, false));
#undef SS_VARIANTS
#undef SS_VARIANTS2
  if (es != cudaSuccess) return cuda_fail(es, "k_scale_space");
  ++launches;
  MARK(2);

  return run_nms(c, W, H, B, ws, L, v, idx, dog, st, launches, ev);
}

mhfd_status run_prune(mhfd_ctx* c, int32_t B, char* ws, const Layout& L, mhfd_blob* blobs, int32_t blob_cap,
                      int32_t* counts, double* scores, int32_t* flags, cudaStream_t st, int& launches,
                      cudaEvent_t* ev, const mhfd_blob* ext_cand = nullptr, int sync = 0, bool seg_rows = false) {
  PruneArgs pa;
  memset(&pa, 0, sizeof(pa));
  pa.B = B;
  pa.W = c->p.width;
  pa.H = c->p.height;
  pa.cap = c->cap;
  pa.cand = ext_cand ? ext_cand : reinterpret_cast<const mhfd_blob*>(ws + L.cand);
  pa.ncand = reinterpret_cast<const int32_t*>(ws + L.ncand);
  pa.overlap = c->p.overlap;
  pa.prune = c->p.overlap < 1.0f ? 1 : 0;
  pa.sync = sync;
  pa.radmax = c->radmax;
  for (int s = 0; s < c->n; ++s) pa.rad[s] = c->rad[s];
  for (int s = 0; s < c->n; ++s) pa.dmax[s] = c->dmax[s];
  pa.thr = c->d_thr;
  pa.n = c->n;
  pa.st = reinterpret_cast<uint8_t*>(ws + L.st);
  pa.rowstart = reinterpret_cast<int32_t*>(ws + L.rowstart);
  // the NMS fast path's segment offsets are row starts when segments are whole-row pieces
  pa.segoff = (seg_rows && !ext_cand && c->p.nms == MHFD_NMS_PAPER && c->p.width % kSeg == 0)
                  ? reinterpret_cast<const int32_t*>(ws + L.segoff) : nullptr;
  pa.nseg = nseg_of(c);
  pa.spr = c->p.width / kSeg;
  pa.cs_shift = c->cs_shift;
  pa.ncx = c->ncx;
  pa.nbands = c->nbands;
  // scale-sorted cells with the reach test for large cells (cs >= 64: radii where most of a
  // 3 x 3 cell window is out of most blobs' reach; C5 pruning 0.32 -> 0.21 ms), plain
  // cell ranges for small ones (the per-cell loop cost more than it skipped at sigma 1-10)
  const bool sorted = c->cs_shift >= 6 && (int64_t)c->ncx * c->n + 1 <= kMaxKeys;
  pa.nsk = sorted ? c->n : 1;
  pa.cst_stride = sorted ? c->ncx + 1 : 2 * (c->ncx + 1);
  pa.cellstart = reinterpret_cast<int32_t*>(ws + L.cellstart);
  pa.crec = reinterpret_cast<int4*>(ws + L.crec);
  pa.img_off = reinterpret_cast<int64_t*>(ws + L.imgoff);
  pa.chunk_off = reinterpret_cast<int64_t*>(ws + L.chunkoff);
  pa.chunk_cnt = reinterpret_cast<int32_t*>(ws + L.chunkcnt);
  pa.chunk_pos = reinterpret_cast<int32_t*>(ws + L.chunkpos);
  pa.counters = reinterpret_cast<int32_t*>(ws + L.counters);
  pa.wl = reinterpret_cast<int4*>(ws + L.wl);
  pa.wl_cap = wl_cap_of(c, B);
  pa.blobs = blobs;
  pa.blob_cap = blob_cap;
  pa.counts = counts;
  pa.scores = scores;
  pa.flags = flags;
  void* args[] = {&pa};
  cudaError_t e = cudaLaunchCooperativeKernel(sorted ? (void*)k_prune<true> : (void*)k_prune<false>,
                                              dim3(c->prune_grid), dim3(256), args, 0, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_prune (cooperative)");
  ++launches;
  if (getenv("MHFD_PRUNE_TRACE")) {   // debug: decision rounds of this call (synchronises)
    int32_t r = -1;
    int64_t tot = -1;
    cudaMemcpyAsync(&r, pa.counters + 3, sizeof(r), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&tot, pa.img_off + B, sizeof(tot), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "mhfd prune: %lld candidates, %d rounds\n", (long long)tot, r);
    unsigned long long ts[24] = {0};
    cudaMemcpyAsync(ts, pa.counters + 16, sizeof(ts), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (ts[0]) {
      int32_t nrec = 0;
      cudaMemcpy(&nrec, pa.counters + 8, sizeof(nrec), cudaMemcpyDeviceToHost);
      fprintf(stderr, "mhfd prune: %d records scanned in all rounds\n", nrec);
      std::vector<uint32_t> ce(c->prune_grid);
      cudaMemcpy(ce.data(), pa.wl + 2 * (pa.wl_cap - 1024), 4 * ce.size(), cudaMemcpyDeviceToHost);
      std::vector<double> us;
      for (uint32_t v : ce) us.push_back((double)(uint32_t)(v - (uint32_t)ts[0]) / 1000.0);
      std::sort(us.begin(), us.end());
      fprintf(stderr, "mhfd prune: round-0 work end per CTA (us): min %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f\n", us[0],
              us[us.size() / 10], us[us.size() / 2], us[us.size() * 9 / 10], us.back());
      fprintf(stderr, "mhfd prune phase stamps (us from start):");
      for (int i = 1; i < 12 && ts[i] >= ts[0] && ts[i] - ts[0] < 100000000ull; ++i)
        fprintf(stderr, " %.1f", (ts[i] - ts[0]) / 1000.0);
      fprintf(stderr, "\n");
    }
  }
  MARK(4);
  return MHFD_OK;
}

// band mode helpers: copy min(n, cap) candidate records; set one device int
__global__ void k_copy_cands(const mhfd_blob* __restrict__ src, const int32_t* __restrict__ n, int64_t cap,
                             mhfd_blob* __restrict__ dst) {
  const int64_t m = min((int64_t)*n, cap);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void k_set_i32(int32_t* p, int32_t v) { *p = v; }

// mhfd_prune_band's tally: kept blobs of rows [y0, y1) and the certificate (out[1] starts
// at 1 and is cleared if some band blob's decision round t has (t + 1) D above its
// distance to a truncated edge of the extended band [e0, e1))
__global__ void k_band_tally(const mhfd_blob* __restrict__ cand, const uint8_t* __restrict__ st, int32_t n, int y0,
                             int y1, int e0, int e1, int H, int D, int32_t* __restrict__ out) {
  int kept = 0, nb = 0;
  bool bad = false;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int y = cand[k].y;
    if (y < y0 || y >= y1) continue;
    ++nb;
    const uint8_t s = st[k];
    kept += (s & 3u) == kKept;
    const int t = s >> 2;
    const int margin = min(e0 > 0 ? y - e0 : INT_MAX, e1 < H ? e1 - 1 - y : INT_MAX);
    if ((s & 3u) == kUndecided || t >= 63 || (int64_t)(t + 1) * D > margin) bad = true;
  }
  for (int o = 16; o; o >>= 1) {
    kept += __shfl_xor_sync(0xffffffffu, kept, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
  }
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (kept) atomicAdd(&out[0], kept);
    if (nb) atomicAdd(&out[2], nb);
    if (bad) atomicExch(&out[1], 0);
  }
}
__global__ void k_tally_init(int32_t* out) { out[0] = 0; out[1] = 1; out[2] = 0; }

__global__ void k_copy_lohi(const ImgPar* par, int32_t* lohi, int B) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) { lohi[2 * b] = par[b].lo; lohi[2 * b + 1] = par[b].hi; }
}

// e2e chunk sizes.  Round 1 ramped them up geometrically (2, 3, 4, 6, 8, 12, 16, ...:
// the compute, ~0.43 ms per image, outran the ~0.31 ms copy, so growing chunks kept the
// copies hidden).  Now a chunk of n images computes in ~0.31 n + 0.24 ms (the per-call
// latency of the percentiles, NMS and pruning), about as fast as its copy: a chunk
// larger than its predecessor by more than about one image makes the compute wait for
// the copy.  So the sizes grow by one image per chunk from 1 up to the caller's size
// (1, 2, ..., chunk, chunk, ...): only the first image's copy is exposed, and the chunk
// count (each costing its ~0.24 ms) stays small.  64 x 4096^2 u8: 24.9 ms (geometric, 16)
// -> 23.7 (uniform 8) -> see DESIGN.md §8 for this ramp.
std::vector<int> e2e_chunks(int batch, int chunk, bool ramp) {
  std::vector<int> out;
  for (int left = batch, n = ramp ? 1 : chunk; left > 0; n = std::min(chunk, n + 1)) {
    out.push_back(std::min(n, left));
    left -= out.back();
  }
  return out;
}

}  // namespace

extern "C" {

int32_t mhfd_abi_version(void) { return MHFD_ABI_VERSION; }
int32_t mhfd_last_launch_count(void) { return g_launches; }
const char* mhfd_last_error(void) { return g_err.c_str(); }

const char* mhfd_status_string(mhfd_status s) {
  switch (s) {
    case MHFD_OK: return "MHFD_OK";
    case MHFD_ERR_INVALID_ARGUMENT: return "MHFD_ERR_INVALID_ARGUMENT";
    case MHFD_ERR_SHAPE: return "MHFD_ERR_SHAPE";
    case MHFD_ERR_CAPACITY: return "MHFD_ERR_CAPACITY";
    case MHFD_ERR_WORKSPACE: return "MHFD_ERR_WORKSPACE";
    case MHFD_ERR_CUDA: return "MHFD_ERR_CUDA";
    case MHFD_ERR_DEVICE: return "MHFD_ERR_DEVICE";
  }
  return "MHFD_ERR_UNKNOWN";
}

void mhfd_params_default(mhfd_params* p) {
  if (!p) return;
  memset(p, 0, sizeof(*p));
  p->struct_size = sizeof(mhfd_params);
  p->min_sigma = 1.0f;
  p->max_sigma = 10.0f;
  p->num_scales = 10;
  p->threshold = 0.09f;  // 0.1 * dt for the paper-like grid (reading R11)
  p->overlap = 0.5f;
  p->sat_low = 0.00175f;
  p->sat_high = 0.00175f;
  p->nms = MHFD_NMS_PAPER;
  p->strict = 0;
  p->device = 0;
  p->max_candidates = 0;
  p->polarity = MHFD_DARK;
  p->schedule = MHFD_SCHEDULE_AUTO;
}

mhfd_status mhfd_create(const mhfd_params* p, mhfd_ctx** out) {
  g_err.clear();
  if (!p || !out) return fail(MHFD_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  // ABI 1 callers pass the struct without `polarity` (it then reads as MHFD_DARK)
  const size_t v1_size = offsetof(mhfd_params, polarity);
  if (p->struct_size < v1_size) return fail(MHFD_ERR_INVALID_ARGUMENT, "struct_size %u", p->struct_size);
  mhfd_params pp;
  memset(&pp, 0, sizeof(pp));
  memcpy(&pp, p, std::min<size_t>(p->struct_size, sizeof(mhfd_params)));
  pp.struct_size = sizeof(mhfd_params);
  p = &pp;
  if (p->polarity != MHFD_DARK && p->polarity != MHFD_BRIGHT)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "polarity %d", p->polarity);
  if (p->response != MHFD_RESPONSE_DOG && p->response != MHFD_RESPONSE_LOG)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "response %d", p->response);
  if (p->response == MHFD_RESPONSE_LOG && 2 * p->num_scales > kMaxLevels - 2)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "LoG response: 2 num_scales = %d > %d", 2 * p->num_scales, kMaxLevels - 2);
  if (p->response == MHFD_RESPONSE_LOG && p->width % kR3Cols != 0)
    return fail(MHFD_ERR_SHAPE, "LoG response: width %d is not a multiple of %d", p->width, kR3Cols);
  if (p->boundary != MHFD_BOUNDARY_PERIODIC && p->boundary != MHFD_BOUNDARY_REFLECT)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "boundary %d", p->boundary);
  if (p->boundary == MHFD_BOUNDARY_REFLECT && p->width % kR3Cols != 0)
    return fail(MHFD_ERR_SHAPE, "reflect boundary: width %d is not a multiple of %d", p->width, kR3Cols);
  if (!(std::isfinite(p->min_sigma) && p->min_sigma > 0.f))
    return fail(MHFD_ERR_INVALID_ARGUMENT, "min_sigma must be > 0 (NonPositiveScale)");
  if (!(std::isfinite(p->max_sigma) && p->max_sigma > p->min_sigma))
    return fail(MHFD_ERR_INVALID_ARGUMENT, "max_sigma must be > min_sigma");
  if (p->num_scales < 1 || p->num_scales > kMaxLevels - 2)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "num_scales %d not in [1, %d] (InsufficientLevels)", p->num_scales,
                kMaxLevels - 2);
  if (!(std::isfinite(p->threshold) && p->threshold >= 0.f))
    return fail(MHFD_ERR_INVALID_ARGUMENT, "threshold must be finite and >= 0");
  if (!(p->overlap >= 0.f && p->overlap <= 1.f)) return fail(MHFD_ERR_INVALID_ARGUMENT, "overlap not in [0,1]");
  if (!(p->sat_low >= 0.f && p->sat_low < 0.5f && p->sat_high >= 0.f && p->sat_high < 0.5f))
    return fail(MHFD_ERR_INVALID_ARGUMENT, "sat_low/sat_high not in [0, 0.5)");
  if (p->nms != MHFD_NMS_PAPER && p->nms != MHFD_NMS_26) return fail(MHFD_ERR_INVALID_ARGUMENT, "nms %d", p->nms);
  if (p->strict != 0 && p->strict != 1) return fail(MHFD_ERR_INVALID_ARGUMENT, "strict %d", p->strict);
  if (p->max_candidates < 0) return fail(MHFD_ERR_INVALID_ARGUMENT, "max_candidates < 0");
  if (p->schedule < MHFD_SCHEDULE_AUTO || p->schedule > MHFD_SCHEDULE_GENERIC)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "schedule %d", p->schedule);
  const int n = p->num_scales;
  // scale grid in f64
  double t[kMaxLevels];
  const double dt = ((double)p->max_sigma - (double)p->min_sigma) / n;
  int R[kMaxLevels];
  int rmax = 0;
  for (int i = 0; i <= n; ++i) {
    t[i] = (double)p->min_sigma + i * dt;
    R[i] = (int)std::ceil(5.0 * t[i]);
    rmax = std::max(rmax, R[i]);
  }
  if (rmax > kMaxRadius) return fail(MHFD_ERR_INVALID_ARGUMENT, "ceil(5*max_sigma) = %d > %d", rmax, kMaxRadius);
  if (p->width < 2 * rmax + 1 || p->height < 2 * rmax + 1 || p->width > 65535 || p->height > 65535)
    return fail(MHFD_ERR_SHAPE, "width/height %dx%d: need 2*ceil(5*max_sigma)+1 = %d <= W,H <= 65535", p->width,
                p->height, 2 * rmax + 1);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(MHFD_ERR_DEVICE, "no CUDA device");
  }
  if (p->device < 0 || p->device >= ndev) return fail(MHFD_ERR_DEVICE, "device %d of %d", p->device, ndev);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, p->device) != cudaSuccess) return fail(MHFD_ERR_DEVICE, "device properties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(MHFD_ERR_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a (B200)", p->device,
                prop.major, prop.minor);

  mhfd_ctx* c = new (std::nothrow) mhfd_ctx;
  if (!c) return fail(MHFD_ERR_INVALID_ARGUMENT, "out of host memory");
  memset(c, 0, sizeof(*c));
  c->tab = new (std::nothrow) LevelTable;
  if (!c->tab) { delete c; return fail(MHFD_ERR_INVALID_ARGUMENT, "out of host memory"); }
  memset(c->tab, 0, sizeof(LevelTable));
  c->p = *p;
  c->p.struct_size = sizeof(mhfd_params);
  c->n = n;
  c->dt = dt;
  c->sms = prop.multiProcessorCount;
  {
    // schedule: the params field (ABI 4) wins; MHFD_SCHEDULE / MHFD_NO_BAND remain
    // process-wide overrides for the measurement tools when the field is 0 (auto)
    const char* nb = getenv("MHFD_NO_BAND");
    c->band_enabled = !(nb && nb[0] == '1');
    const char* sch = getenv("MHFD_SCHEDULE");
    int choice = p->schedule;
    if (choice == MHFD_SCHEDULE_AUTO && sch) {
      if (strcmp(sch, "tc") == 0) choice = MHFD_SCHEDULE_TC;
      if (strcmp(sch, "band") == 0) choice = MHFD_SCHEDULE_BAND;
      if (strcmp(sch, "generic") == 0) choice = MHFD_SCHEDULE_GENERIC;
    }
    c->band_kind = choice == MHFD_SCHEDULE_BAND ? 1 : 3;
    if (choice == MHFD_SCHEDULE_GENERIC) c->band_enabled = 0;
  }
  LevelTable& T = *c->tab;
  T.nlev = n + 1;
  T.rmax = rmax;
  int off = 0;
  for (int i = 0; i <= n; ++i) {
    const int pre = (4 - R[i] % 4) % 4;
    const int ntap = ((pre + 2 * R[i] + 1) + kTapUnroll - 1) / kTapUnroll * kTapUnroll;
    if (off + ntap + 8 > kMaxTaps) {
      mhfd_destroy(c);
      return fail(MHFD_ERR_INVALID_ARGUMENT, "tap table exceeds %d floats", kMaxTaps);
    }
    // sampled Gaussian exp(-d^2/2t^2) (sigma = t), renormalised in f64, rounded once
    double sum = 0.0;
    for (int d = -R[i]; d <= R[i]; ++d) sum += std::exp(-(double)d * d / (2.0 * t[i] * t[i]));
    for (int d = -R[i]; d <= R[i]; ++d)
      T.w[off + pre + d + R[i]] = (float)(std::exp(-(double)d * d / (2.0 * t[i] * t[i])) / sum);
    T.R[i] = R[i];
    T.pre[i] = pre;
    T.ntap[i] = ntap;
    T.woff[i] = off;
    T.tdog[i] = (float)(p->polarity == MHFD_BRIGHT ? -t[i] : t[i]);   // Eq. 2 factor, signed by polarity
    off += ntap + 8;   // >= 1 zero after the taps (the FFMA2 odd-output pair reads w[ntap])
    c->t[i] = t[i];
  }
  T.ntaps_total = off;
  if (p->response == MHFD_RESPONSE_LOG) {   // reading R23: sub-levels 2i = w_i, 2i+1 = w2_i (row taps)
    c->ltab = new (std::nothrow) LevelTable;
    if (!c->ltab) {
      mhfd_destroy(c);
      return fail(MHFD_ERR_INVALID_ARGUMENT, "out of host memory");
    }
    LevelTable& LT = *c->ltab;
    memset(&LT, 0, sizeof(LT));
    LT.nlev = 2 * n;
    LT.rmax = 0;
    int lo = 0;
    for (int i = 0; i < n; ++i) {
      const int Ri = R[i];
      const int pre = (4 - Ri % 4) % 4;
      const int ntap = ((pre + 2 * Ri + 1) + kTapUnroll - 1) / kTapUnroll * kTapUnroll;
      std::vector<double> w(2 * Ri + 1), w2(2 * Ri + 1);
      double sum = 0.0, m2 = 0.0;
      for (int d = -Ri; d <= Ri; ++d) sum += std::exp(-(double)d * d / (2.0 * t[i] * t[i]));
      for (int d = -Ri; d <= Ri; ++d) {
        w[d + Ri] = std::exp(-(double)d * d / (2.0 * t[i] * t[i])) / sum;
        m2 += w[d + Ri] * (double)d * d;
      }
      const double t4 = t[i] * t[i] * t[i] * t[i];
      for (int d = -Ri; d <= Ri; ++d) w2[d + Ri] = w[d + Ri] * ((double)d * d - m2) / t4;
      for (int k = 0; k < 2; ++k) {
        const int sl = 2 * i + k;
        if (lo + ntap + 8 > kMaxTaps) {
          mhfd_destroy(c);
          return fail(MHFD_ERR_INVALID_ARGUMENT, "LoG tap table exceeds %d floats", kMaxTaps);
        }
        for (int d = -Ri; d <= Ri; ++d) LT.w[lo + pre + d + Ri] = (float)(k ? w2[d + Ri] : w[d + Ri]);
        LT.R[sl] = Ri;
        LT.pre[sl] = pre;
        LT.ntap[sl] = ntap;
        LT.woff[sl] = lo;
        LT.tdog[sl] = (float)((p->polarity == MHFD_BRIGHT ? -1.0 : 1.0) * t[i] * t[i]);   // t_i^2, signed
        lo += ntap + 8;
      }
      LT.rmax = std::max(LT.rmax, Ri);
    }
    LT.ntaps_total = lo;
    if (c3_smem(LT.rmax) > kSmemLimit || r3_smem(LT.rmax, r3_taps_total(LT)) > kSmemLimit) {
      mhfd_destroy(c);
      return fail(MHFD_ERR_INVALID_ARGUMENT, "LoG response: radius %d too large for the two-pass kernels", LT.rmax);
    }
  }
  // tensor-core plan and its Toeplitz tables (device copy owned by the context)
  c->tc = new (std::nothrow) TcPlan;
  if (c->tc && tc_plan_build(*c->tc, n + 1, R, t)) {
    c->tc->reflect = p->boundary == MHFD_BOUNDARY_REFLECT ? 1 : 0;
    if (p->polarity == MHFD_BRIGHT)
      for (int i = 0; i <= n; ++i) c->tc->lev[i].tdog = -c->tc->lev[i].tdog;
    std::vector<std::vector<double>> wv(n + 1);
    for (int i = 0; i <= n; ++i) {
      double sum = 0.0;
      for (int d = -R[i]; d <= R[i]; ++d) sum += std::exp(-(double)d * d / (2.0 * t[i] * t[i]));
      for (int d = -R[i]; d <= R[i]; ++d) wv[i].push_back(std::exp(-(double)d * d / (2.0 * t[i] * t[i])) / sum);
    }
    std::vector<uint8_t> tabh((size_t)c->tc->tab_bytes);
    tc_fill_tables(*c->tc, wv, tabh.data());
    int prev = 0;
    cudaGetDevice(&prev);
    const bool ok = cudaSetDevice(p->device) == cudaSuccess &&
                    cudaMalloc(&c->d_tctab, tabh.size()) == cudaSuccess &&
                    cudaMemcpy(c->d_tctab, tabh.data(), tabh.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    cudaSetDevice(prev);
    if (!ok) {   // fail loudly: no silent fallback to a slower schedule
      cudaGetLastError();
      mhfd_destroy(c);
      return fail(MHFD_ERR_CUDA, "Toeplitz table upload for k_tc failed");
    }
  }
  // two-pass tensor-core plan (k_tc2) and its tables
  // Eq. 2: the n + 1 Gaussian levels.  LoG (reading R23): 2n sub-levels, 2j = (rows w_j,
  // columns t_j^2 w2_j) and 2j+1 = (rows t_j^2 w2_j, columns w_j), whose column products
  // k_tc2_cols<., true> sums into t_j^2 (d_xx + d_yy) L(., t_j); w2 as the pair path's
  // (zero-sum sampled second derivative), with t_j^2 folded in (tdog = the sign only)
  const bool log_resp = p->response == MHFD_RESPONSE_LOG;
  std::vector<int> R2;
  std::vector<double> t2;
  for (int i = 0; i < (log_resp ? n : n + 1); ++i)
    for (int k = 0; k < (log_resp ? 2 : 1); ++k) {
      R2.push_back(R[i]);
      t2.push_back(t[i]);
    }
  c->tc2 = new (std::nothrow) Tc2Plan;
  if (c->tc2 && tc2_plan_build(*c->tc2, (int)R2.size(), R2.data(), t2.data())) {
    const int nl2 = (int)R2.size();
    std::vector<std::vector<double>> wr(nl2), wc(nl2);
    for (int i = 0; i < (log_resp ? n : n + 1); ++i) {
      std::vector<double> w, w2s;
      double sum = 0.0, m2 = 0.0;
      for (int d = -R[i]; d <= R[i]; ++d) sum += std::exp(-(double)d * d / (2.0 * t[i] * t[i]));
      for (int d = -R[i]; d <= R[i]; ++d) {
        w.push_back(std::exp(-(double)d * d / (2.0 * t[i] * t[i])) / sum);
        m2 += w.back() * (double)d * d;
      }
      if (!log_resp) {
        wr[i] = wc[i] = w;
        continue;
      }
      for (int d = -R[i]; d <= R[i]; ++d) w2s.push_back(w[d + R[i]] * ((double)d * d - m2) / (t[i] * t[i]));
      wr[2 * i] = wc[2 * i + 1] = w;
      wc[2 * i] = wr[2 * i + 1] = w2s;
      c->tc2->lev[2 * i].tdog = c->tc2->lev[2 * i + 1].tdog = 1.f;
    }
    if (p->polarity == MHFD_BRIGHT)
      for (int i = 0; i < nl2; ++i) c->tc2->lev[i].tdog = -c->tc2->lev[i].tdog;
    std::vector<uint8_t> tabh((size_t)c->tc2->tab_bytes);
    tc2_fill_tables(*c->tc2, wr, wc, tabh.data());
    int prev = 0;
    cudaGetDevice(&prev);
    const bool ok = cudaSetDevice(p->device) == cudaSuccess &&
                    cudaMalloc(&c->d_tc2tab, tabh.size()) == cudaSuccess &&
                    cudaMemcpy(c->d_tc2tab, tabh.data(), tabh.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    cudaSetDevice(prev);
    if (!ok) {
      cudaGetLastError();
      mhfd_destroy(c);
      return fail(MHFD_ERR_CUDA, "Toeplitz table upload for k_tc2 failed");
    }
  } else {
    delete c->tc2;
    c->tc2 = nullptr;
  }
  c->radmax = 0.0;
  for (int s = 0; s < n; ++s) {
    c->rad[s] = std::sqrt(2.0) * t[s];
    c->radmax = std::max(c->radmax, c->rad[s]);
  }
  // pruning thresholds: frac(d; r1, r2) (lens area / smaller disk) decreases in d, so
  // frac > overlap <=> d < d*(r1, r2); bisect d* in f64 and keep a 1e-6 band around d*^2
  // inside which the kernel evaluates the formula itself
  {
    std::vector<float2> thr((size_t)n * n);
    auto frac = [](double d, double r1, double r2) {
      const double rmin = std::min(r1, r2);
      if (d >= r1 + r2) return 0.0;
      if (d <= std::fabs(r1 - r2)) return 1.0;
      double a1 = (d * d + r1 * r1 - r2 * r2) / (2.0 * d * r1), a2 = (d * d + r2 * r2 - r1 * r1) / (2.0 * d * r2);
      a1 = std::min(1.0, std::max(-1.0, a1));
      a2 = std::min(1.0, std::max(-1.0, a2));
      double k = (-d + r1 + r2) * (d + r1 - r2) * (d - r1 + r2) * (d + r1 + r2);
      k = std::max(k, 0.0);
      return (r1 * r1 * std::acos(a1) + r2 * r2 * std::acos(a2) - 0.5 * std::sqrt(k)) / (M_PI * rmin * rmin);
    };
    for (int s1 = 0; s1 < n; ++s1) {
      double hmax = 0.0;
      for (int s2 = 0; s2 < n; ++s2) {
        const double r1 = c->rad[s1], r2 = c->rad[s2];
        double lo2 = -1.0, hi2 = -1.0;   // overlap >= 1: frac > overlap never holds
        if (p->overlap < 1.0f) {
          double a = 0.0, b = r1 + r2;   // frac(a) > overlap (>= 1 > overlap at containment), frac(b) = 0
          if (!(frac(a, r1, r2) > (double)p->overlap)) b = 0.0;
          for (int it = 0; it < 200 && b > 0.0; ++it) {
            const double m = 0.5 * (a + b);
            if (frac(m, r1, r2) > (double)p->overlap) a = m; else b = m;
          }
          lo2 = b * b * (1.0 - 1e-6) - 1e-6;
          hi2 = b * b * (1.0 + 1e-6) + 1e-6;
        }
        thr[(size_t)s1 * n + s2] = make_float2((float)lo2, (float)hi2);
        if (s2 >= s1) hmax = std::max(hmax, hi2);
      }
      c->dmax[s1] = hmax > 0.0 ? (int)std::ceil(std::sqrt(hmax)) + 1 : 0;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(p->device) != cudaSuccess || cudaMalloc(&c->d_thr, sizeof(float2) * thr.size()) != cudaSuccess ||
        cudaMemcpy(c->d_thr, thr.data(), sizeof(float2) * thr.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      cudaSetDevice(prev);
      mhfd_destroy(c);
      return fail(MHFD_ERR_CUDA, "pruning threshold table upload failed");
    }
    cudaSetDevice(prev);
  }
  {   // cell edge: a power of two >= every search radius, and few enough cells per band
    int dm = 8;
    for (int s = 0; s < n; ++s) dm = std::max(dm, (int)c->dmax[s]);
    int sh = 3;
    while ((1 << sh) < dm || (p->width + (1 << sh) - 1) / (1 << sh) + 1 > kMaxCells) ++sh;
    c->cs_shift = sh;
    c->ncx = (p->width + (1 << sh) - 1) >> sh;
    c->nbands = (p->height + (1 << sh) - 1) >> sh;
  }
  const int64_t half = (int64_t)((p->width + 1) / 2) * ((p->height + 1) / 2);
  c->cap = p->max_candidates > 0 ? p->max_candidates : (p->nms == MHFD_NMS_PAPER ? half : half * n);
  int bps = 0, bps2 = 0;   // both k_prune variants (cooperative grid = co-resident blocks)
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_prune<false>, 256, 0) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps2, k_prune<true>, 256, 0) != cudaSuccess ||
      std::min(bps, bps2) < 1) {
    mhfd_destroy(c);
    return fail(MHFD_ERR_CUDA, "occupancy query for k_prune failed");
  }
  c->prune_grid = std::min(bps, bps2) * c->sms;
  {   // large radii: the two-pass generic schedule (no halo recompute) when the fused
      // band kernel would recompute more than ~1.5x of its row pass
    const char* nt = getenv("MHFD_NO_TWOPASS");
    c->twopass = (rmax >= 96 && p->width % kR2Cols == 0 && !(nt && nt[0] == '1') &&
                  rows2_smem(rmax) <= kSmemLimit && cols2_smem(rmax) <= kSmemLimit) ? 1 : 0;
  }
  {
    const char* pg = getenv("MHFD_PRUNE_CTAS_PER_SM");   // tuning knob (<= the occupancy limit)
    if (pg && atoi(pg) > 0) c->prune_grid = std::min(bps, atoi(pg)) * c->sms;
  }
  if (scale_space_smem(rmax, 128, T.ntaps_total) > kSmemLimit) {
    mhfd_destroy(c);
    return fail(MHFD_ERR_INVALID_ARGUMENT, "ceil(5*max_sigma) = %d: the generic schedule's shared memory exceeds the "
                "sm_100 limit", rmax);
  }
  *out = c;
  return MHFD_OK;
}

mhfd_status mhfd_timing_enable(mhfd_ctx* c, int32_t max_calls) {
  if (!c || max_calls < 0) return fail(MHFD_ERR_INVALID_ARGUMENT, "bad argument");
  if (c->tev) {
    for (int i = 0; i < 5 * c->tmax; ++i) cudaEventDestroy(c->tev[i]);
    delete[] c->tev;
    c->tev = nullptr;
  }
  c->tmax = c->tcount = 0;
  if (max_calls == 0) return MHFD_OK;
  c->tev = new (std::nothrow) cudaEvent_t[5 * (size_t)max_calls];
  if (!c->tev) return fail(MHFD_ERR_INVALID_ARGUMENT, "out of host memory");
  for (int i = 0; i < 5 * max_calls; ++i) {
    cudaError_t e = cudaEventCreate(&c->tev[i]);
    if (e != cudaSuccess) {
      for (int j = 0; j < i; ++j) cudaEventDestroy(c->tev[j]);
      delete[] c->tev;
      c->tev = nullptr;
      return cuda_fail(e, "cudaEventCreate");
    }
  }
  c->tmax = max_calls;
  return MHFD_OK;
}

mhfd_status mhfd_timing_read(mhfd_ctx* c, float* ms, int32_t* ncalls) {
  if (!c || !ms || !ncalls) return fail(MHFD_ERR_INVALID_ARGUMENT, "NULL argument");
  *ncalls = 0;
  for (int k = 0; k < c->tcount; ++k) {
    cudaEvent_t* ev = c->tev + 5 * k;
    cudaError_t e = cudaEventSynchronize(ev[4]);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
    for (int st = 0; st < 4; ++st) {
      e = cudaEventElapsedTime(&ms[4 * k + st], ev[st], ev[st + 1]);
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
    }
  }
  *ncalls = c->tcount;
  return MHFD_OK;
}

void mhfd_destroy(mhfd_ctx* c) {
  if (!c) return;
  if (c->tev) {
    for (int i = 0; i < 5 * c->tmax; ++i) cudaEventDestroy(c->tev[i]);
    delete[] c->tev;
  }
  if (c->copy_stream) {
    cudaStreamDestroy(c->copy_stream);
    for (int i = 0; i < kStageSlots; ++i) { cudaEventDestroy(c->ev_ready[i]); cudaEventDestroy(c->ev_free[i]); }
    cudaEventDestroy(c->ev_done);
  }
  if (c->d_tctab) cudaFree(c->d_tctab);
  if (c->d_tc2tab) cudaFree(c->d_tc2tab);
  if (c->d_thr) cudaFree(c->d_thr);
  delete c->tc;
  delete c->tc2;
  delete c->tab;
  delete c->ltab;
  delete c;
}

mhfd_status mhfd_focus_score_host(mhfd_ctx* c, const void* h_images, int32_t dtype, int32_t batch,
                                  int64_t pitch_bytes, void* d_staging, size_t staging_bytes, void* d_workspace,
                                  size_t workspace_bytes, double* h_scores, int32_t* h_counts, void* stream) {
  g_err.clear();
  if (!c) return fail(MHFD_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (!h_images || !h_scores || !d_staging) return fail(MHFD_ERR_INVALID_ARGUMENT, "NULL argument");
  if (batch < 1) return fail(MHFD_ERR_SHAPE, "batch %d < 1", batch);
  const size_t img_bytes = (size_t)c->p.height * (size_t)pitch_bytes;
  const int chunk = (int)std::min<size_t>(staging_bytes / (kStageSlots * img_bytes), (size_t)batch);
  if (chunk < 1) return fail(MHFD_ERR_WORKSPACE, "staging holds < 1 image per slot (%d slots)", kStageSlots);
  if (((uintptr_t)d_staging) % 256 != 0) return fail(MHFD_ERR_WORKSPACE, "staging not 256-byte aligned");
  mhfd_status s = check_call(c, d_staging, dtype, chunk, pitch_bytes, d_workspace, workspace_bytes);
  if (s != MHFD_OK) return s;
  cudaError_t e = cudaSuccess;
  bool fresh = false;
  if (!c->copy_stream) {
    e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
    for (int i = 0; i < kStageSlots && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&c->ev_ready[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "host-path stream/events");
    fresh = true;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  const Layout L = layout(c, chunk);
  double* d_sc = reinterpret_cast<double*>(ws + L.scores);
  int32_t* d_ct = reinterpret_cast<int32_t*>(ws + L.counts);
  // Consecutive calls pipeline: chunk k's copy waits only for the compute that last used
  // its staging slot (ev_free), so the next call's first copies overlap this call's last
  // chunks.  A first call, or a different staging buffer / slot size, instead orders the
  // copies after everything already on the caller's stream (which may still read staging).
  if (fresh || c->stage_ptr != d_staging || c->stage_chunk != chunk) {
    for (int i = 0; i < kStageSlots && e == cudaSuccess; ++i) e = cudaEventRecord(c->ev_free[i], st);
    if (e != cudaSuccess) return cuda_fail(e, "event record");
    c->stage_ptr = d_staging;
    c->stage_chunk = chunk;
    c->stage_next = 0;
  }
  // Chunk plan: with the previous call still in flight its tail hides this call's first
  // copy, so every chunk is `chunk` images (fewest per-call overheads); on an idle device
  // the chunks ramp up 1, 2, 3, ... so that compute starts after one image's copy
  const bool in_flight = !fresh && cudaEventQuery(c->ev_done) == cudaErrorNotReady;
  cudaGetLastError();   // (cudaEventQuery's not-ready status is not an error)
  int launches = 0;
  const std::vector<int> sizes = e2e_chunks(batch, chunk, !in_flight);
  for (int b0 = 0, k = 0, nb = 0; k < (int)sizes.size(); b0 += nb, ++k) {
    nb = sizes[k];
    const int h = (int)(c->stage_next++ % kStageSlots);
    char* dst = static_cast<char*>(d_staging) + (size_t)h * chunk * img_bytes;
    e = cudaStreamWaitEvent(c->copy_stream, c->ev_free[h], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dst, static_cast<const char*>(h_images) + (size_t)b0 * img_bytes, (size_t)nb * img_bytes,
                          cudaMemcpyHostToDevice, c->copy_stream);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_ready[h], c->copy_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, c->ev_ready[h], 0);
    if (e != cudaSuccess) return cuda_fail(e, "host-path copy");
    cudaEvent_t* ev = next_timing(c);
    s = run_front(c, dst, dtype, nb, pitch_bytes, ws, L, nullptr, st, launches, ev);
    if (s != MHFD_OK) return s;
    s = run_prune(c, nb, ws, L, nullptr, 0, d_ct, d_sc, nullptr, st, launches, ev, nullptr, 0, true);
    if (s != MHFD_OK) return s;
    e = cudaEventRecord(c->ev_free[h], st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h_scores + b0, d_sc, sizeof(double) * nb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && h_counts)
      e = cudaMemcpyAsync(h_counts + b0, d_ct, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "host-path readback");
  }
  e = cudaEventRecord(c->ev_done, st);
  if (e != cudaSuccess) return cuda_fail(e, "event record");
  g_launches = launches;
  return MHFD_OK;
}

const char* mhfd_schedule_name(const mhfd_ctx* c, int32_t dtype) {
  if (!c) return "none";
  const int W = c->p.width, H = c->p.height;
  const bool paper = c->p.nms == MHFD_NMS_PAPER;
  if (c->p.response == MHFD_RESPONSE_LOG)
    return c->band_kind == 3 && tc2_fit(c) ? "k_tc2" : "k_rows_pair+k_cols_pair<log>";
  if (dtype == MHFD_U8 && c->band_enabled && c->band_kind == 3 && c->d_tctab && tc_ok(*c->tc, W, H)) return "k_tc";
  if (c->band_kind == 3 && tc2_fit(c)) return "k_tc2";
  if (c->p.boundary == MHFD_BOUNDARY_REFLECT) return pair_fit(c) ? "k_rows_pair+k_cols_pair" : "none";
  if (dtype == MHFD_U8 && paper && c->band_enabled && band_ok(W, H, c->tab->rmax, c->tab->ntaps_total))
    return "k_band";
  if (pair_ok(c)) return "k_rows_pair+k_cols_pair";
  if (c->twopass && W % kR2Cols == 0) return "k_rows2+k_cols_all";
  return "k_scale_space";
}

double mhfd_schedule_flops_per_pixel(const mhfd_ctx* c, int32_t dtype) {
  if (!c) return 0.0;
  const char* name = mhfd_schedule_name(c, dtype);
  if (strcmp(name, "k_tc") == 0) {   // banded products per 128 x 128 tile: 2 row splits, 3 column splits
    const TcPlan& P = *c->tc;
    double macs = 0.0;
    for (int i = 0; i < P.nlev; ++i) {
      const double K = P.lev[i].K;
      macs += 2.0 * kTcTile * K * K + 3.0 * kTcTile * kTcTile * K;
    }
    return 2.0 * macs / ((double)kTcTile * kTcTile);
  }
  if (strcmp(name, "k_tc2") == 0) {   // per pixel: 3 products x K_i (row pass) + 3 x K2_i (column pass)
    const Tc2Plan& P = *c->tc2;
    double macs = 0.0;
    for (int i = 0; i < P.nlev; ++i) macs += 3.0 * P.lev[i].K + 3.0 * P.lev[i].K2;
    return 2.0 * macs;
  }
  double f = 0.0;   // direct separable blur at R_i: 2 passes x (2R_i+1) FMA per level, + DoG/max
  if (c->ltab) {    // LoG: per plane 2 row convs (w, w2) + 2 column convs, + sum/scale/max
    for (int i = 0; i < c->n; ++i) f += 2.0 * 4.0 * (2.0 * c->tab->R[i] + 1.0);
    return f + 4.0 * c->n;
  }
  for (int i = 0; i <= c->n; ++i) f += 2.0 * 2.0 * (2.0 * c->tab->R[i] + 1.0);
  return f + 3.0 * c->n;
}

mhfd_status mhfd_detect_band(mhfd_ctx* c, const void* d_image, int32_t dtype, int64_t pitch_bytes, int32_t y0,
                             int32_t y1, void* d_workspace, size_t workspace_bytes, mhfd_blob* d_cands,
                             int32_t cand_capacity, int32_t* d_ncand, void* stream) {
  g_err.clear();
  mhfd_status s = check_call(c, d_image, dtype, 1, pitch_bytes, d_workspace, workspace_bytes);
  if (s != MHFD_OK) return s;
  const int W = c->p.width, H = c->p.height;
  if (!(0 <= y0 && y0 < y1 && y1 <= H)) return fail(MHFD_ERR_SHAPE, "band rows [%d, %d) not inside [0, %d)", y0, y1, H);
  if (W % kSeg != 0) return fail(MHFD_ERR_SHAPE, "band mode needs width %% %d == 0", kSeg);
  const char* sch = mhfd_schedule_name(c, dtype);
  if (strcmp(sch, "k_tc") != 0 && strcmp(sch, "k_tc2") != 0 && strcmp(sch, "k_rows_pair+k_cols_pair") != 0)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "band mode needs the k_tc, k_tc2 or two-pass pair schedule (Eq. 3 NMS)");
  if (!d_ncand || (!d_cands && cand_capacity > 0) || cand_capacity < 0)
    return fail(MHFD_ERR_INVALID_ARGUMENT, "d_ncand / d_cands / cand_capacity");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  const Layout L = layout(c, 1);
  int launches = 0;
  s = run_front(c, d_image, dtype, 1, pitch_bytes, ws, L, nullptr, st, launches, nullptr, y0, y1);
  if (s != MHFD_OK) return s;
  const int32_t* nc = reinterpret_cast<const int32_t*>(ws + L.ncand);
  if (cand_capacity > 0) {   // the workspace list holds at most c->cap records
    k_copy_cands<<<c->sms * 4, 256, 0, st>>>(reinterpret_cast<const mhfd_blob*>(ws + L.cand), nc,
                                              std::min<int64_t>(cand_capacity, c->cap), d_cands);
    ++launches;
  }
  cudaError_t e = cudaMemcpyAsync(d_ncand, nc, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "band outputs");
  g_launches = launches;
  return MHFD_OK;
}

mhfd_status mhfd_prune_candidates(mhfd_ctx* c, const mhfd_blob* d_cands, int32_t ncand, void* d_workspace,
                                  size_t workspace_bytes, mhfd_blob* d_blobs, int32_t blob_capacity,
                                  int32_t* d_count, double* d_score, int32_t* d_flags, void* stream) {
  g_err.clear();
  if (!c) return fail(MHFD_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (ncand < 0 || ncand > c->cap) return fail(MHFD_ERR_CAPACITY, "ncand %d not in [0, %lld]", ncand, (long long)c->cap);
  if (ncand > 0 && !d_cands) return fail(MHFD_ERR_INVALID_ARGUMENT, "d_cands is NULL");
  if (!d_count) return fail(MHFD_ERR_INVALID_ARGUMENT, "d_count is NULL");
  if (blob_capacity < 0 || (blob_capacity > 0 && !d_blobs)) return fail(MHFD_ERR_INVALID_ARGUMENT, "blobs");
  if (!d_workspace || ((uintptr_t)d_workspace) % 256 != 0) return fail(MHFD_ERR_WORKSPACE, "workspace");
  const Layout L = layout(c, 1);
  if (workspace_bytes < L.total) return fail(MHFD_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, L.total);
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != c->p.device)
    return fail(MHFD_ERR_DEVICE, "current device %d != context device %d", dev, c->p.device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  k_set_i32<<<1, 1, 0, st>>>(reinterpret_cast<int32_t*>(ws + L.ncand), ncand);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_set_i32");
  int launches = 1;
  mhfd_status s = run_prune(c, 1, ws, L, blob_capacity > 0 ? d_blobs : nullptr, blob_capacity, d_count, d_score,
                            d_flags, st, launches, nullptr, ncand > 0 ? d_cands : reinterpret_cast<const mhfd_blob*>(ws + L.cand));
  if (s != MHFD_OK) return s;
  g_launches = launches;
  return MHFD_OK;
}

int32_t mhfd_interaction_radius(const mhfd_ctx* c) {
  if (!c) return -1;
  int d = 0;
  for (int s = 0; s < c->n; ++s) d = std::max(d, (int)c->dmax[s]);
  return d;
}

mhfd_status mhfd_prune_band(mhfd_ctx* c, const mhfd_blob* d_cands, int32_t ncand, int32_t e0, int32_t e1, int32_t y0,
                            int32_t y1, void* d_workspace, size_t workspace_bytes, int32_t* d_count, int32_t* d_cert,
                            int32_t* d_nband, void* stream) {
  g_err.clear();
  if (!c) return fail(MHFD_ERR_INVALID_ARGUMENT, "ctx is NULL");
  const int H = c->p.height;
  if (!(0 <= e0 && e0 <= y0 && y0 < y1 && y1 <= e1 && e1 <= H))
    return fail(MHFD_ERR_SHAPE, "need 0 <= e0 <= y0 < y1 <= e1 <= height (%d %d %d %d, %d)", e0, y0, y1, e1, H);
  if (ncand < 0 || ncand > c->cap) return fail(MHFD_ERR_CAPACITY, "ncand %d not in [0, %lld]", ncand, (long long)c->cap);
  if (ncand > 0 && !d_cands) return fail(MHFD_ERR_INVALID_ARGUMENT, "d_cands is NULL");
  if (!d_count || !d_cert) return fail(MHFD_ERR_INVALID_ARGUMENT, "d_count / d_cert is NULL");
  if (!d_workspace || ((uintptr_t)d_workspace) % 256 != 0) return fail(MHFD_ERR_WORKSPACE, "workspace");
  const Layout L = layout(c, 1);
  if (workspace_bytes < L.total) return fail(MHFD_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, L.total);
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != c->p.device)
    return fail(MHFD_ERR_DEVICE, "current device %d != context device %d", dev, c->p.device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  k_set_i32<<<1, 1, 0, st>>>(reinterpret_cast<int32_t*>(ws + L.ncand), ncand);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_set_i32");
  int launches = 1;
  const mhfd_blob* cand = ncand > 0 ? d_cands : reinterpret_cast<const mhfd_blob*>(ws + L.cand);
  int32_t* scratch = reinterpret_cast<int32_t*>(ws + L.counts);   // 1 int (the full-list count, unused)
  mhfd_status s = run_prune(c, 1, ws, L, nullptr, 0, scratch, nullptr, nullptr, st, launches, nullptr, cand, 1);
  if (s != MHFD_OK) return s;
  int32_t* tally = reinterpret_cast<int32_t*>(ws + L.counters) + 12;   // {count, cert, nband}; k_prune: 0-8, 16-63
  k_tally_init<<<1, 1, 0, st>>>(tally);
  k_band_tally<<<std::max(1, std::min(c->sms * 4, (ncand + 255) / 256)), 256, 0, st>>>(
      cand, reinterpret_cast<const uint8_t*>(ws + L.st), ncand, y0, y1, e0, e1, H, mhfd_interaction_radius(c), tally);
  launches += 2;
  e = cudaMemcpyAsync(d_count, tally, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_cert, tally + 1, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && d_nband) e = cudaMemcpyAsync(d_nband, tally + 2, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "band tally");
  g_launches = launches;
  return MHFD_OK;
}

mhfd_status mhfd_downsample(const void* d_in, int32_t dtype, int32_t width, int32_t height, int64_t in_pitch,
                            int32_t factor, void* d_out, int64_t out_pitch, int32_t batch, void* stream) {
  g_launches = 0;
  if (!d_in || !d_out) return fail(MHFD_ERR_INVALID_ARGUMENT, "downsample: null image pointer");
  if (dtype != MHFD_U8 && dtype != MHFD_U16) return fail(MHFD_ERR_INVALID_ARGUMENT, "downsample: dtype %d", dtype);
  if (batch < 0) return fail(MHFD_ERR_INVALID_ARGUMENT, "downsample: batch < 0");
  if (width < 1 || height < 1 || width > 65535 || height > 65535)
    return fail(MHFD_ERR_SHAPE, "downsample: %dx%d", width, height);
  if (factor < 1 || factor > std::min(width, height))
    return fail(MHFD_ERR_INVALID_ARGUMENT, "downsample: factor %d not in [1, min(W, H) = %d]", factor,
                std::min(width, height));
  const int bpp = dtype == MHFD_U16 ? 2 : 1;
  const int OW = (width + factor - 1) / factor, OH = (height + factor - 1) / factor;
  if (in_pitch < (int64_t)width * bpp || out_pitch < (int64_t)OW * bpp || in_pitch % bpp || out_pitch % bpp)
    return fail(MHFD_ERR_SHAPE, "downsample: pitch smaller than a row or not a multiple of the pixel size");
  if (batch == 0) return MHFD_OK;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t work = (int64_t)batch * OH * ((OW + 3) / 4);
  const int grid = (int)std::min<int64_t>((work + 255) / 256, (int64_t)sms * 8);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint8_t* in = static_cast<const uint8_t*>(d_in);
  uint8_t* out = static_cast<uint8_t*>(d_out);
  int launches = 0;
  const bool fast2 = factor == 2 && ((int64_t)width * bpp) % 16 == 0 && in_pitch % 16 == 0 && out_pitch % 8 == 0 &&
                     reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 8 == 0;
  if (fast2) {
    const int64_t work2 = (int64_t)batch * OH * ((int64_t)width * bpp / 16);
    const int grid2 = (int)std::min<int64_t>((work2 + 255) / 256, (int64_t)sms * 16);
    if (bpp == 1) k_downsample2<uint8_t><<<grid2, 256, 0, st>>>(in, width, height, in_pitch, out, OH, out_pitch, batch);
    else k_downsample2<uint16_t><<<grid2, 256, 0, st>>>(in, width, height, in_pitch, out, OH, out_pitch, batch);
  } else if (bpp == 1) {
    k_downsample<uint8_t><<<grid, 256, 0, st>>>(in, width, height, in_pitch, factor, out, OW, OH, out_pitch, batch);
  } else {
    k_downsample<uint16_t><<<grid, 256, 0, st>>>(in, width, height, in_pitch, factor, out, OW, OH, out_pitch, batch);
  }
  LAUNCH_CHECK("k_downsample");
  g_launches = launches;
  return MHFD_OK;
}

mhfd_status mhfd_get_params(const mhfd_ctx* c, mhfd_params* out) {
  if (!c || !out) return fail(MHFD_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = c->p;
  out->max_candidates = (int32_t)c->cap;
  return MHFD_OK;
}

mhfd_status mhfd_workspace_bytes(const mhfd_ctx* c, int32_t batch, size_t* bytes) {
  if (!c || !bytes) return fail(MHFD_ERR_INVALID_ARGUMENT, "NULL argument");
  if (batch < 1) return fail(MHFD_ERR_SHAPE, "batch %d < 1", batch);
  *bytes = layout(c, batch).total;
  return MHFD_OK;
}

mhfd_status mhfd_detect_batch(mhfd_ctx* c, const void* d_images, int32_t dtype, int32_t batch, int64_t pitch_bytes,
                              void* d_workspace, size_t workspace_bytes, mhfd_blob* d_blobs, int32_t blob_capacity,
                              int32_t* d_counts, int32_t* d_flags, void* stream) {
  g_err.clear();
  mhfd_status s = check_call(c, d_images, dtype, batch, pitch_bytes, d_workspace, workspace_bytes);
  if (s != MHFD_OK) return s;
  if (blob_capacity < 0) return fail(MHFD_ERR_CAPACITY, "blob_capacity < 0");
  if (!d_counts) return fail(MHFD_ERR_INVALID_ARGUMENT, "d_counts is NULL");
  if (!d_blobs && blob_capacity > 0) return fail(MHFD_ERR_INVALID_ARGUMENT, "d_blobs is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  const Layout L = layout(c, batch);
  int launches = 0;
  cudaEvent_t* ev = next_timing(c);
  s = run_front(c, d_images, dtype, batch, pitch_bytes, ws, L, nullptr, st, launches, ev);
  if (s != MHFD_OK) return s;
  s = run_prune(c, batch, ws, L, d_blobs ? d_blobs : nullptr, blob_capacity, d_counts, nullptr, d_flags, st,
                launches, ev, nullptr, 0, true);
  if (s != MHFD_OK) return s;
  g_launches = launches;
  return MHFD_OK;
}

mhfd_status mhfd_focus_score(mhfd_ctx* c, const void* d_images, int32_t dtype, int32_t batch, int64_t pitch_bytes,
                             void* d_workspace, size_t workspace_bytes, double* d_scores, int32_t* d_counts,
                             void* stream) {
  g_err.clear();
  mhfd_status s = check_call(c, d_images, dtype, batch, pitch_bytes, d_workspace, workspace_bytes);
  if (s != MHFD_OK) return s;
  if (!d_scores) return fail(MHFD_ERR_INVALID_ARGUMENT, "d_scores is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  const Layout L = layout(c, batch);
  int launches = 0;
  cudaEvent_t* ev = next_timing(c);
  s = run_front(c, d_images, dtype, batch, pitch_bytes, ws, L, nullptr, st, launches, ev);
  if (s != MHFD_OK) return s;
  s = run_prune(c, batch, ws, L, nullptr, 0, d_counts, d_scores, nullptr, st, launches, ev, nullptr, 0, true);
  if (s != MHFD_OK) return s;
  g_launches = launches;
  return MHFD_OK;
}

mhfd_status mhfd_debug_dump(mhfd_ctx* c, const void* d_images, int32_t dtype, int32_t batch, int64_t pitch_bytes,
                            void* d_workspace, size_t workspace_bytes, int32_t* d_lohi, float* d_dog, float* d_v,
                            uint8_t* d_idx, mhfd_blob* d_cands, int32_t* d_ncand, void* stream) {
  g_err.clear();
  mhfd_status s = check_call(c, d_images, dtype, batch, pitch_bytes, d_workspace, workspace_bytes);
  if (s != MHFD_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(d_workspace);
  const Layout L = layout(c, batch);
  int launches = 0;
  s = run_front(c, d_images, dtype, batch, pitch_bytes, ws, L, d_dog, st, launches, nullptr);
  if (s != MHFD_OK) return s;
  const int64_t plane = (int64_t)c->p.width * c->p.height;
  cudaError_t e = cudaSuccess;
  if (d_lohi) {
    k_copy_lohi<<<(batch + 127) / 128, 128, 0, st>>>(reinterpret_cast<const ImgPar*>(ws + L.par), d_lohi, batch);
    e = cudaGetLastError();
    ++launches;
  }
  const bool paper = c->p.nms == MHFD_NMS_PAPER;
  if (e == cudaSuccess && d_v && paper)
    e = cudaMemcpyAsync(d_v, ws + L.v, sizeof(float) * plane * batch, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && d_idx && paper)
    e = cudaMemcpyAsync(d_idx, ws + L.idx, plane * batch, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && d_cands)
    e = cudaMemcpyAsync(d_cands, ws + L.cand, sizeof(mhfd_blob) * c->cap * batch, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && d_ncand)
    e = cudaMemcpyAsync(d_ncand, ws + L.ncand, sizeof(int32_t) * batch, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "debug copies");
  g_launches = launches;
  return MHFD_OK;
}

}  // extern "C"
