// k_tc.cuh — the hot kernel for u8 images on the 5th-generation tensor cores
// (hot-path rows a2-a6, "banded-GEMM formulation of the blur").
//
// Same mathematics as k_band / k_scale_space: stretch, sampled
// renormalised Gaussian blur at every level with periodic wrap (PAPER.md:134-141,
// :166-168), DoG = t_i (L_{i+1} - L_i) (Eq. 2), first argmax over the
// scales.  Per 128 x 128 output tile and level i the separable blur
// is two banded products on tcgen05 (tc_plan.h gives the geometry and tables):
//
//   row pass    D1[c][n] = sum_k T_i[c][k] X[c0+n][c0+k]        SS MMA, M=128, N=K_i
//               (A = Toeplitz pairs in smem, B = the staged tile X, fp16 exact
//               integers x = p' - mid; T = hi + lo fp16 split of 2^12 w)
//   split       D1 -> (hi, lo) fp16 in place in TMEM (A operand of the next pass)
//   column pass D2[c][m] = sum_k A2[c][k] T_i[m][k]             TS MMA, M=128, N=128
//               (A2_hi T_hi + A2_hi T_lo + A2_lo T_hi)
//   epilogue    DoG, running max and first argmax in registers (lane = column c,
//               32 rows per thread), overlapped with the next level's row pass.
//
// Persistent: one 512-thread CTA per SM walks tiles; the next tile's raw u8 window
// ((S+off) x S bytes, periodic) is fetched by TMA / bulk copies while the current
// tile computes; each level's Toeplitz table (<= 22.5 KB) is bulk-copied from the
// context's device table two levels ahead into a double buffer.
// Accuracy (tools/umma_probe.cu): D1 and D2 within ~1e-6 relative of f64 sums.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "k_band.cuh"
#include "k_scale_space.cuh"
#include "tc_plan.h"
#include "umma.cuh"

namespace mhfd {

#ifndef TC_EXP
#define TC_EXP 0   // performance experiments only (tools/tc_exp.py): 1 no DoG reads, 2 one DoG read, 3 no split, 4 = 1 + 3,
                   // 5 no output writes, 6 no staging conversion, 7 / 8 column pass without the
                   // A2_hi T_lo / A2_lo T_hi product (numerics: tools/precision_probe.py)
#endif

constexpr int kTcThreads = 512;

__host__ __device__ inline int tc_off(const TcPlan& P) { return (16 - P.H0 % 16) % 16; }   // landing column offset
__host__ __device__ inline int tc_lw(const TcPlan& P) { return (P.S + tc_off(P) + 15) / 16 * 16; }
__host__ __device__ inline size_t tc_b1_bytes(const TcPlan& P) { return (size_t)P.S * P.S * 2; }
__host__ __device__ inline size_t tc_land_bytes(const TcPlan& P) { return (size_t)tc_lw(P) * P.S; }
__host__ __device__ inline size_t tc_smem(const TcPlan& P) {
  return tc_b1_bytes(P) + tc_land_bytes(P) + 2 * (size_t)P.max_level_bytes + 128;
}
inline bool tc_ok(const TcPlan& P, int W, int H) {
  return P.S > 0 && tc_lw(P) <= 256 && tc_smem(P) <= 227 * 1024 && W >= tc_lw(P) && H >= P.S;
}

struct TcTile {
  int b, x0, y0;
};
__device__ __forceinline__ TcTile tc_tile(int t, int tx, int ty, int row_lo) {
  TcTile r;
  r.x0 = (t % tx) * kTcTile;
  t /= tx;
  r.y0 = row_lo + (t % ty) * kTcTile;
  r.b = t / ty;
  return r;
}

// Blur boundary index (P.reflect): periodic (reading R7) or half-sample symmetric
// ... c b a | a b c ... (R25; one reflection: R_max < W, H)
__device__ __forceinline__ int tc_bidx(int a, int m, int reflect) {
  if (reflect) return a < 0 ? -a - 1 : (a >= m ? 2 * m - 1 - a : a);
  return wrap_idx(a, m);
}

// Fetch the raw window of tile tt into `land` (LW x S bytes, row pitch LW): columns
// x0 - H0 - off .. +LW, rows y0 - H0 .. +S, periodic or mirrored.  Mode as band_fetch:
// 2 = TMA box, 1 = bulk copies per row, 0 = plain loads (complete on return), 3 = bulk
// copies of the in-image columns of mirrored rows (reflect), whose out-of-image columns
// tc_reflect_cols fills inside `land` once the copies have landed.
__device__ __forceinline__ void epi_sync();
template <bool REFLECT>
__device__ __forceinline__ int tc_fetch_epi(const TcTile& tt, uint8_t* land, uint64_t* bar, const uint8_t* images,
                                        const Shape& s, const CUtensorMap* tmap, int use_tmap, const TcPlan& P) {
  const int LW = tc_lw(P), S = P.S;
  const int xr = tt.x0 - P.H0 - tc_off(P), yr = tt.y0 - P.H0;
  const int tid = threadIdx.x;
  const bool tma = use_tmap && xr >= 0 && xr + LW <= s.W && yr >= 0 && yr + S <= s.H;
  const bool bulk = !tma && (s.W % 16) == 0 && (s.pitch % 16) == 0;
  if (tma) {
    if (tid == 0) {
      mbar_arrive_expect_tx(bar, (uint32_t)(LW * S));
      tma_2d_g2s(land, tmap, xr, tt.b * s.H + yr, bar);
    }
    return 2;
  }
  const uint8_t* img = images + (int64_t)tt.b * s.H * s.pitch;
  if (REFLECT && bulk) {
    const int cl = max(xr, 0), ch = min(xr + LW, s.W);
    if (tid == 0) mbar_arrive_expect_tx(bar, (uint32_t)(S * (ch - cl)));
    epi_sync();   // expect_tx registered before any copy completes
    for (int r = tid; r < S; r += kTcThreads)
      bulk_g2s(land + (size_t)r * LW + (cl - xr), img + (int64_t)tc_bidx(yr + r, s.H, 1) * s.pitch + cl,
               (uint32_t)(ch - cl), bar);
    return 3;
  }
  if (bulk) {
    if (tid == 0) mbar_arrive_expect_tx(bar, (uint32_t)(S * LW));
    epi_sync();   // expect_tx registered before any copy completes
    const int xw = wrap_idx(xr, s.W);
    for (int r = tid; r < S; r += kTcThreads) {
      const uint8_t* row = img + (int64_t)wrap_idx(yr + r, s.H) * s.pitch;
      uint8_t* dst = land + (size_t)r * LW;
      if (xw + LW > s.W) {
        bulk_g2s(dst, row + xw, (uint32_t)(s.W - xw), bar);
        bulk_g2s(dst + (s.W - xw), row, (uint32_t)(xw + LW - s.W), bar);
      } else {
        bulk_g2s(dst, row + xw, (uint32_t)LW, bar);
      }
    }
    return 1;
  }
  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < S; r += kTcThreads / 32) {
    const uint8_t* row = img + (int64_t)tc_bidx(yr + r, s.H, REFLECT) * s.pitch;
    for (int c = lane; c < LW; c += 32) land[(size_t)r * LW + c] = row[tc_bidx(xr + c, s.W, REFLECT)];
  }
  return 0;
}

// Mode 3 windows: out-of-image columns from their mirror images inside the window
__device__ __noinline__ void tc_reflect_cols(uint8_t* land, const TcPlan& P, int xr, int W) {
  const int LW = tc_lw(P), S = P.S;
  if (xr >= 0 && xr + LW <= W) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < S; r += kTcThreads / 32)
    for (int c = lane; c < LW; c += 32) {
      const int x = xr + c;
      if (x < 0 || x >= W) land[(size_t)r * LW + c] = land[(size_t)r * LW + (tc_bidx(x, W, 1) - xr)];
    }
}

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// raw window (land) -> B1: saturate to [lo, hi], centre on mid, exact fp16; chunk (r, kc)
// of 8 pixels lands at B1 + ((r/8 * S/8 + kc) * 8 + r%8) * 16 (canonical K-major: row
// group, column chunk, row).  Called by the 16 epilogue warps.  Each warp converts blocks
// of 8 rows x 16 chunks; lane -> (r8 = lane & 7, kc = lane/8 + 4 ((r8 + i) & 3)) in its
// i-th step, so the 8-byte loads hit 16 distinct bank pairs although every land row starts
// at the same bank (LW = 256), and the 16-byte stores of the 8 rows fall in 8 distinct bank
// groups: 2 and 4 wavefronts per instruction, the minimum (the raster mapping was 8-way
// conflicted on the loads).
__device__ __forceinline__ void tc_stage_b1(const uint8_t* land, uint8_t* B1, int S, int LW, int OFF, int lo, int hi,
                                            int mid) {
  const uint32_t lo2 = (uint32_t)lo * 0x10001u, hi2 = (uint32_t)hi * 0x10001u;
  const __half2 cm = __floats2half2_rn(1024.f + (float)mid, 1024.f + (float)mid);
  const int kcs = S / 8, nkb = (kcs + 15) / 16, nblk = (S / 8) * nkb;
  const int lane = threadIdx.x & 31, r8 = lane & 7;
  if (TC_EXP == 6) return;
  for (int blk = threadIdx.x >> 5; blk < nblk; blk += kTcThreads / 32) {
    const int rg = blk / nkb, kb = blk - rg * nkb;
    const int r = rg * 8 + r8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kc = kb * 16 + (lane >> 3) + 4 * ((r8 + i) & 3);
      if (kc >= kcs) continue;
      const uint2 raw = *reinterpret_cast<const uint2*>(land + (size_t)r * LW + OFF + 8 * kc);
      const uint32_t a = clamp_bytes(raw.x, lo2, hi2), bb = clamp_bytes(raw.y, lo2, hi2);
      // 0x64pp = fp16 1024 + p exactly; subtracting 1024 + mid leaves the integer p - mid
      const uint32_t p0 = __byte_perm(a, 0x64646464u, 0x4140u), p1 = __byte_perm(a, 0x64646464u, 0x4342u);
      const uint32_t p2 = __byte_perm(bb, 0x64646464u, 0x4140u), p3 = __byte_perm(bb, 0x64646464u, 0x4342u);
      __half2 x0 = __hsub2(*reinterpret_cast<const __half2*>(&p0), cm);
      __half2 x1 = __hsub2(*reinterpret_cast<const __half2*>(&p1), cm);
      __half2 x2 = __hsub2(*reinterpret_cast<const __half2*>(&p2), cm);
      __half2 x3 = __hsub2(*reinterpret_cast<const __half2*>(&p3), cm);
      uint4 o;
      o.x = *reinterpret_cast<uint32_t*>(&x0);
      o.y = *reinterpret_cast<uint32_t*>(&x1);
      o.z = *reinterpret_cast<uint32_t*>(&x2);
      o.w = *reinterpret_cast<uint32_t*>(&x3);
      *reinterpret_cast<uint4*>(B1 + ((size_t)(rg * kcs + kc) * 8 + r8) * 16) = o;
    }
  }
}

// D1 chunk j (16 f32 columns of this thread's lane) -> hi fp16 at 16j, lo fp16 at 16j+8,
// in two 8-column halves (fewer live registers).  In-place order: columns 16j..+7 are
// read, their hi goes to 16j..+3 (already read); their lo waits until columns 16j+8..+15
// have been read too, then lo(0-7) -> 16j+8..+11, hi(8-15) -> 16j+4..+7, lo(8-15) ->
// 16j+12..+15.
__device__ __forceinline__ void split_half(const uint32_t (&r)[8], uint32_t (&h4)[4], uint32_t (&l4)[4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float y0 = __uint_as_float(r[2 * u]) * (1.f / kTcWScale);
    const float y1 = __uint_as_float(r[2 * u + 1]) * (1.f / kTcWScale);
    const __half2 hh = __floats2half2_rn(y0, y1);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(y0 - hf.x, y1 - hf.y);
    h4[u] = *reinterpret_cast<const uint32_t*>(&hh);
    l4[u] = *reinterpret_cast<const uint32_t*>(&ll);
  }
}
__device__ __forceinline__ void tc_split_chunk(uint32_t tq, int j) {
  if (TC_EXP == 3 || TC_EXP == 4) return;
  const uint32_t base = tq + 16 * j;
  uint32_t r[8], h4[4], l4a[4], l4b[4];
  umma::ld8(base, r);
  umma::wait_ld();
  split_half(r, h4, l4a);
  umma::st4(base, h4);            // hi(0-7) over columns 0-3: read already
  umma::ld8(base + 8, r);
  umma::wait_ld();
  split_half(r, h4, l4b);
  umma::st4(base + 4, h4);        // hi(8-15)
  umma::st4(base + 8, l4a);       // lo(0-7): columns 8-11 have been read
  umma::st4(base + 12, l4b);      // lo(8-15)
}

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 512;" ::: "memory"); }   // epilogue warps only


// Roles: warps 0-15 = epilogue (TMEM lane quarter q = warp & 3, row group wg = warp >> 2):
// staging, split, DoG; warp 16 = MMA issuer (one lane).
// TMEM: D1 / A2 columns [0, 256); D2 double buffer [256, 384) and [384, 512) (level
// parity), so the previous level's L stays in TMEM for the DoG.
// Barriers (bars[]): 0 land (tx), 1 rowDone, 2 colDone (tcgen05.commit), 3-6 split groups
// (16 warp arrivals), 7 staged (16), 8/9 table buffers (tx).  Barriers 1-2 complete once
// per global level g (parity g & 1); 7 once per tile; split group k only on levels with
// more than 4k chunks (its phase is tracked explicitly).
//
// Per level g:
//   issuer : [tile start: wait staged] wait table g -> row pass (N = K_i, one MMA per
//            split and K-step) -> commit rowDone; wait colDone(g-1) -> table g+1 prefetch;
//            for each group of 4 chunks: wait split(grp) -> column K-steps of grp; commit colDone
//   epilogue: [tile start: stage B1] wait colDone(g-1) -> DoG of level g-1 (D2 buffers);
//            wait rowDone(g) -> per group: split own chunk -> arrive split(grp)
// Hazards: row(g) writes D1 after col(g-1) read A2 (in-order tcgen05.mma); col(g) writes
// D2[g&1] (= L_{g-2}) after every warp's DoG of g-1 (it precedes their split arrivals);
// B1 is restaged after rowDone of the tile's last level (waited before its split).
// DOG: also write every DoG plane to dog_out (26-neighbour NMS, dumps).  NP: level parts
// per tile (1, or 2 for calls with few tiles; a template so the batch path pays nothing)
// REFLECT (reading R25, P.reflect): mirrored windows at the image edges (mode 3 fetches
// and tc_reflect_cols); a separate instantiation, so the periodic kernels keep their
// register allocation
template <bool DOG, int NP = 1, bool REFLECT = false>
__global__ void __launch_bounds__(kTcThreads + 32, 1)
k_tc(const uint8_t* __restrict__ images, Shape s, const ImgPar* __restrict__ par, const __grid_constant__ TcPlan P,
     const uint8_t* __restrict__ tabs, const __grid_constant__ CUtensorMap tmap, int use_tmap,
     float* __restrict__ v_out, uint8_t* __restrict__ idx_out, float* __restrict__ dog_out, int batch,
     int row_lo, int row_hi, int lsplit, float* __restrict__ v_out2, uint8_t* __restrict__ idx_out2,
     unsigned long long* __restrict__ trace) {
  constexpr int nparts = NP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int S = P.S, LW = tc_lw(P), OFF = tc_off(P);
  uint8_t* B1 = smem_raw;                                          // S x S fp16, canonical K-major
  uint8_t* land = B1 + tc_b1_bytes(P);                             // LW x S raw bytes
  uint8_t* tbuf = land + tc_land_bytes(P);                         // 2 x max_level_bytes
  uint64_t* bars = reinterpret_cast<uint64_t*>(tbuf + 2 * (size_t)P.max_level_bytes);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 10);
  // timeline probe (tools/tc_timeline.cu): CTA 0, first 64 levels, 16 stamps per level
  unsigned long long* tr = (trace && blockIdx.x == 0) ? trace : nullptr;
#define TC_STAMP(g, slot) \
  do { if (tr && (g) < 64) tr[(g) * 16 + (slot)] = clock64(); } while (0)

  // warp index through a shuffle: the compiler can then prove the role branches below
  // warp-uniform and keep the issuer's descriptors in uniform registers
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  // rows [row_lo, row_hi) of every image (the whole image, or one band: mhfd_detect_band)
  const int tx = (s.W + kTcTile - 1) / kTcTile, ty = (row_hi - row_lo + kTcTile - 1) / kTcTile;
  // Work units: a tile (nparts = 1), or for calls with fewer tiles than SMs a tile's levels
  // in two parts (nparts = 2): part 0 levels [0, lsplit], part 1 [lsplit, nlev) (level
  // lsplit twice: part 1's first DoG plane needs it), DoG planes [0, lsplit) and
  // [lsplit, n), v / argmax of part 1 to v_out2 / idx_out2 (merged by k_merge_parts).
  // The grid is even, so a CTA's units all have the part t0 & 1.
  const int ntiles = tx * ty * batch * nparts;   // units
  const int t0 = blockIdx.x;
  if (t0 >= ntiles) return;
  const int part = nparts > 1 ? (t0 & 1) : 0;
  const int lev_lo = part ? lsplit : 0;
  const int nl2 = part ? P.nlev - lsplit : lsplit + 1;
#define nl (NP > 1 ? nl2 : P.nlev)   // levels per unit (NP = 1: read from the parameter bank, no register)
  const int my_tiles = (ntiles - 1 - t0) / gridDim.x + 1;
  const int G = my_tiles * nl;   // levels this CTA processes

  const int SBO1 = (S / 8) * 128;

  if (tid == kTcThreads) {
    for (int k = 0; k < 10; ++k) mbar_init(&bars[k], (k >= 3 && k <= 7) ? 16 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc(tslot, 512);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;

  if (warp == kTcThreads / 32) {
    // ================= MMA issuer =================
    // The whole warp runs this loop (warp-uniform branch: `warp` comes through
    // __shfl_sync), one elected lane issues each tcgen05 instruction (umma::*_w), so the
    // descriptors live in uniform registers.
    if (lane != 0) tr = nullptr;
    auto issue_table = [&](int gg) {
      if (lane == 0) {
        const int lev = lev_lo + gg % nl;
        const int bytes = 2 * P.lev[lev].npairs * 256;
        uint64_t* tb = &bars[8 + (gg & 1)];
        mbar_arrive_expect_tx(tb, (uint32_t)bytes);
        bulk_g2s(tbuf + (size_t)(gg & 1) * P.max_level_bytes, tabs + P.lev[lev].tab_off, (uint32_t)bytes, tb);
      }
      __syncwarp();
    };
    issue_table(0);
    if (G > 1) issue_table(1);
    int tile_i = 0;
    uint32_t sph = 0;   // phase bits of the split barriers (group 3 is not used on every level)
    for (int g = 0; g < G; ++g) {
      const int lev = lev_lo + g % nl;
      TC_STAMP(g, 0);
      if (lev == lev_lo) mbar_wait(&bars[7], (uint32_t)(tile_i++ & 1));
      mbar_wait(&bars[8 + (g & 1)], (uint32_t)((g >> 1) & 1));
      umma::fence_after();
      TC_STAMP(g, 1);
      const TcLevel& L = P.lev[lev];
      const int K = L.K, E1 = K / 8 - 2, nj = K / 16;
      const uint32_t thi = umma::smem_addr(tbuf + (size_t)(g & 1) * P.max_level_bytes);
      const uint32_t tlo = thi + L.npairs * 256;
      const uint32_t b1 = umma::smem_addr(B1) + (L.c0 / 8) * SBO1 + (L.c0 / 8) * 128;
      const uint32_t idr = umma::idesc_f16(128, K), idc = umma::idesc_f16(128, 128);
      // K-step j: B1 window +256 B (start field +16), Toeplitz pairs -512 B (field -32)
      const uint64_t dB = umma::desc_kmajor(b1, 128, SBO1);
      const uint64_t dH = umma::desc_kmajor(thi + E1 * 256, 128, 256);
      const uint64_t dL = umma::desc_kmajor(tlo + E1 * 256, 128, 256);
      // row pass of level g.  No wait for the previous column pass: tcgen05.mma from one
      // thread execute in issue order, so these writes of D1 follow its reads of A2.
      for (int j = 0; j < nj; ++j) {
        umma::mma_ss_w(tmem, dH - 32u * j, dB + 16u * j, idr, j > 0);
        umma::mma_ss_w(tmem, dL - 32u * j, dB + 16u * j, idr, 1);
      }
      umma::commit_w(&bars[1]);
      TC_STAMP(g, 2);
      if (g > 0) {
        mbar_wait(&bars[2], (uint32_t)((g - 1) & 1));   // column pass g-1 done: table buffer free
        if (g + 1 < G) issue_table(g + 1);
      }
      const uint32_t d2 = tmem + 256 + 128 * (g & 1);
      for (int grp = 0; 4 * grp < nj; ++grp) {
        mbar_wait(&bars[3 + grp], (sph >> grp) & 1u);
        sph ^= 1u << grp;
        umma::fence_after();
        TC_STAMP(g, 3 + grp);
        for (int j = 4 * grp; j < nj && j < 4 * grp + 4; ++j) {
          umma::mma_ts_w(d2, tmem + 16 * j, dH - 32u * j, idc, j > 0);
          if (TC_EXP != 7) umma::mma_ts_w(d2, tmem + 16 * j, dL - 32u * j, idc, 1);
          if (TC_EXP != 8) umma::mma_ts_w(d2, tmem + 16 * j + 8, dH - 32u * j, idc, 1);
        }
      }
      umma::commit_w(&bars[2]);
      TC_STAMP(g, 7);
    }
    __syncwarp();
  } else {
    // ================= epilogue warps =================
    const int q = warp & 3, wg = warp >> 2;
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
    const int64_t plane = (int64_t)s.H * s.W;
    // tiles are kept as unit indices (t: staged next, ou: current, wu: output pending) and
    // expanded with tc_tile where needed: three ints instead of three TcTiles of state
    auto tile_of = [&](int u) { return tc_tile(u / nparts, tx, ty, row_lo); };
    int t = t0, ou = t0;
    int mode = tc_fetch_epi<REFLECT>(tile_of(t), land, &bars[0], images, s, &tmap, use_tmap, P);
    uint32_t land_phase = 0;
    float oinv = 0.f;
    int odeg = 0;
    float vbest[32];
    uint32_t ibest[8];

    auto consume = [&](int gg) {   // DoG plane lev-1 from L_lev (D2[gg&1]) and L_{lev-1} (D2[(gg-1)&1])
      const int lev = lev_lo + gg % nl;
      if (lev == lev_lo) return;   // a unit's first level has no DoG of its own
      const float tf = P.lev[lev - 1].tdog * oinv;
      const TcTile ot = tile_of(ou);   // (the DOG variant's plane writes only)
      const uint32_t cur = tq + 256 + 128 * (gg & 1) + 32 * wg, prv = tq + 256 + 128 * ((gg - 1) & 1) + 32 * wg;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {   // 8 rows at a time: fewer live registers (96 with 17 warps)
        uint32_t a[8], b[8];
        if (TC_EXP == 1 || TC_EXP == 4) {
#pragma unroll
          for (int uu = 0; uu < 8; ++uu) a[uu] = b[uu] = __float_as_uint((float)uu);
        } else if (TC_EXP == 2) {
          umma::ld8(cur + 8 * qq, a);
          umma::wait_ld();
#pragma unroll
          for (int uu = 0; uu < 8; ++uu) b[uu] = a[(uu + 1) & 7];
        } else {
          umma::ld8(cur + 8 * qq, a);
          umma::ld8(prv + 8 * qq, b);
          umma::wait_ld();
        }
#pragma unroll
        for (int uu = 0; uu < 8; ++uu) {
          const int u = 8 * qq + uu;
          const float D = tf * (__uint_as_float(a[uu]) - __uint_as_float(b[uu]));
          if (DOG) {   // the DoG planes themselves (26-neighbour NMS, debug dumps)
            const int x = ot.x0 + 32 * q + lane, y = ot.y0 + 32 * wg + u;
            if (x < s.W && y < row_hi)
              dog_out[((int64_t)ot.b * (P.nlev - 1) + (lev - 1)) * plane + (int64_t)y * s.W + x] = D;
          }
          if (D > vbest[u]) {
            vbest[u] = D;
            const int sh = (u & 3) * 8;
            ibest[u >> 2] = (ibest[u >> 2] & ~(0xffu << sh)) | ((uint32_t)(lev - 1) << sh);
          }
        }
      }
    };
    auto write_out = [&](int wu, int wdeg) {   // v and argmax of column 32 q + lane, rows 32 wg .. +32
      if ((DOG && !v_out) || TC_EXP == 5) return;
      const TcTile wt = tile_of(wu);
      const int x = wt.x0 + 32 * q + lane, y0 = wt.y0 + 32 * wg;
      const int64_t p0 = (int64_t)wt.b * plane + (int64_t)y0 * s.W + x;
      float* vo = ((NP > 1 && part) ? v_out2 : v_out) + p0;      // level part 1 -> its own planes
      uint8_t* io = ((NP > 1 && part) ? idx_out2 : idx_out) + p0;
      if (x < s.W && y0 + 32 <= row_hi) {   // whole column piece inside: pointer walk, no checks
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          *vo = wdeg ? 0.f : vbest[u];
          *io = wdeg ? (uint8_t)0 : (uint8_t)((ibest[u >> 2] >> ((u & 3) * 8)) & 0xffu);
          vo += s.W;
          io += s.W;
        }
      } else if (x < s.W) {
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          if (y0 + u < row_hi) {
            vo[(int64_t)u * s.W] = wdeg ? 0.f : vbest[u];
            io[(int64_t)u * s.W] = wdeg ? (uint8_t)0 : (uint8_t)((ibest[u >> 2] >> ((u & 3) * 8)) & 0xffu);
          }
        }
      }
    };
    int wu = t0;   // unit whose output is pending (written after the split of the next unit's first level)
    int wdeg = 0;
    bool pending = false;

    if (tid != 0) tr = nullptr;
    // g == G is a tail step: the last level's DoG and the last tile's output only (one
    // call site each for consume and the output, which keeps the kernel's code small)
    for (int g = 0; g <= G; ++g) {
      const bool last = g == G;
      const int lev = last ? lev_lo : lev_lo + g % nl;
      const bool first = lev == lev_lo;   // a unit's first level (tile boundary) or the tail step
      const uint32_t par_g = (uint32_t)(g & 1);
      TC_STAMP(g, 8);
      ImgPar ip{};
      int tn = 0;
      if (first && !last) {
        // ---- stage tile tt (rowDone of the previous tile's last level was waited below)
        if (mode) {
          mbar_wait(&bars[0], land_phase);
          land_phase ^= 1u;
        }
        if (REFLECT && mode == 3) {   // mirrored columns (rows were mirrored by the copies)
          tc_reflect_cols(land, P, tile_of(t).x0 - P.H0 - tc_off(P), s.W);
          epi_sync();
        }
        epi_sync();
        ip = par[tile_of(t).b];
        tc_stage_b1(land, B1, S, LW, OFF, ip.lo, ip.hi, ip.lo + (ip.hi - ip.lo + 1) / 2);
        umma::fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive1(&bars[7]);
        epi_sync();   // landing zone free
        tn = t + gridDim.x;
        if (tn < ntiles) mode = tc_fetch_epi<REFLECT>(tile_of(tn), land, &bars[0], images, s, &tmap, use_tmap, P);
      }
      // ---- DoG of level g-1.  At level 0 that is the previous tile's last level; it runs
      // before this level's column pass overwrites D2[g & 1] (= its L_{n-1}), and the
      // tile's output is written after the split below, off the tensor pipe's critical
      // path (level 0 has no DoG, so v / argmax stay put until iteration g + 2)
      if (g > 0) {
        mbar_wait(&bars[2], (uint32_t)((g - 1) & 1));
        umma::fence_after();
        TC_STAMP(g, 9);
        consume(g - 1);
      }
      if (first) {
        if (g > 0) {
          wu = ou;
          wdeg = odeg;
          pending = true;
        }
        if (!last) {
          ou = t;
          oinv = ip.inv * (1.f / kTcWScale);
          odeg = ip.degen;
          if (tn < ntiles) t = tn;
        }
      }
      TC_STAMP(g, 10);
      if (!last) {
        // ---- split D1 -> A2 group by group (chunk 4 grp + wg of this warp's lane quarter)
        const int nj = P.lev[lev].K / 16;
        mbar_wait(&bars[1], par_g);
        umma::fence_after();
        TC_STAMP(g, 11);
        for (int grp = 0; 4 * grp < nj; ++grp) {
          const int j = 4 * grp + wg;
          if (j < nj) tc_split_chunk(tq, j);
          umma::wait_st();
          umma::fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive1(&bars[3 + grp]);
          TC_STAMP(g, 12 + grp);
        }
      }
      if (first) {
        if (pending) write_out(wu, wdeg);
        pending = false;
#pragma unroll
        for (int u = 0; u < 32; ++u) vbest[u] = -INFINITY;
#pragma unroll
        for (int u = 0; u < 8; ++u) ibest[u] = 0u;
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 512);
#undef TC_STAMP
#undef nl
}

// v / argmax of the two level parts (k_tc with nparts = 2): part 0 holds DoG planes
// [0, lsplit), part 1 [lsplit, n); the first argmax over all planes is part 1's only where
// its maximum is strictly larger.  4 pixels per thread (16-byte and 4-byte accesses).
__global__ void __launch_bounds__(256) k_merge_parts(float* __restrict__ v, uint8_t* __restrict__ idx,
                                                     const float* __restrict__ v2, const uint8_t* __restrict__ idx2,
                                                     int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<const float4*>(v)[i];
    const float4 b = __ldg(reinterpret_cast<const float4*>(v2) + i);
    uchar4 ia = reinterpret_cast<const uchar4*>(idx)[i];
    const uchar4 ib = __ldg(reinterpret_cast<const uchar4*>(idx2) + i);
    if (b.x > a.x) { a.x = b.x; ia.x = ib.x; }
    if (b.y > a.y) { a.y = b.y; ia.y = ib.y; }
    if (b.z > a.z) { a.z = b.z; ia.z = ib.z; }
    if (b.w > a.w) { a.w = b.w; ia.w = ib.w; }
    reinterpret_cast<float4*>(v)[i] = a;
    reinterpret_cast<uchar4*>(idx)[i] = ia;
  }
}

}  // namespace mhfd
