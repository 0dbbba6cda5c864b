/*
 * mhfd.h — C ABI of the B200-native MHFD hot path.
 *
 * Multi-scale Histologic Feature Detection (Levental et al., arXiv 2108.12050,
 * "Ultrafast Focus Detection for Automated Microscopy").  Per image the library
 * computes Algorithm 1 with a separable spatial blur in place
 * of the FFT, plus the threshold and blob-overlap pruning that the north star adds:
 *
 *   u8/u16 image I
 *   -> histogram stretch I' (saturate sat_low / sat_high of the darkest /
 *      lightest pixels, map to [0,1])
 *   -> L(x,y,t_i) = G(.,.,t_i) * I', t_i = min_t + (i-1) dt,
 *      dt = (max_t - min_t)/n, i = 1..n+1 (periodic)
 *   -> DoG(x,y,i) = t_i (L(x,y,t_{i+1}) - L(x,y,t_i))       Eq. 2
 *   -> C = argmaxlocal_{x,y} argmax_i DoG  (Eq. 3) or the
 *      conventional 3x3x3 scale-space maxima; response > threshold
 *   -> blob-overlap pruning (north star) -> DOF = |C|
 *
 * Every reading the paper leaves open (sigma = t, n+1 levels, periodic blur,
 * -inf NMS padding, first argmax on ties, nearest-rank percentiles, the pruning
 * rule ...) is listed in DESIGN.md §3 ("reading Rk").
 *
 * Conventions (apply to every entry point):
 *  - Pure C99; no torch or CUDA types.  `stream` is a cudaStream_t passed as
 *    void* (NULL = the legacy default stream).
 *  - Device pointers ("d_") must be device-accessible CUDA allocations on the
 *    context's device; the CALLER owns every buffer (images, workspace and
 *    outputs).  The library never allocates device memory inside
 *    mhfd_detect_batch / mhfd_focus_score; the context owns only its immutable
 *    parameters and tap tables (host memory).
 *  - Asynchrony: argument validation happens synchronously and, on failure,
 *    enqueues nothing and returns an error.  On MHFD_OK all work has been
 *    enqueued on `stream`; outputs are valid once the caller synchronises it.
 *    Launch failures return MHFD_ERR_CUDA; asynchronous faults surface at the
 *    caller's synchronisation.
 *  - CUDA graphs: mhfd_detect_batch, mhfd_focus_score and mhfd_debug_dump enqueue only
 *    kernels, memsets and device-to-device copies and never synchronise the host, so a
 *    call can be captured into a CUDA graph and replayed (on new contents of the same
 *    buffers); make one call outside the capture first (it sets kernel attributes).
 *    (tests/test_gpu_parity.py::test_focus_score_cuda_graph_capture)
 *  - Thread safety: a context is immutable after mhfd_create; concurrent calls
 *    with distinct workspaces (and outputs) on distinct streams are safe.
 *  - Determinism: results are bitwise reproducible run to run and independent
 *    of the batch composition and of how a batch is split across GPUs.
 *  - Image layout: batch images back to back, image b at
 *    d_images + b * height * pitch_bytes; row-major, rows pitch_bytes apart;
 *    pixel (x = column, y = row).  pitch_bytes % 16 == 0 and
 *    pitch_bytes >= width * bytes_per_pixel; d_images 16-byte aligned.
 *  - Coordinates in outputs are 0-based; `scale` is the 0-based DoG plane
 *    index s = i^ - 1, i.e. sigma = min_sigma + s * dt.
 *
 * Deliberate deviations from the boundary sketched in SURVEY.md §8(b):
 *  - mhfd_workspace_bytes takes no blob_capacity: the workspace never holds the
 *    caller's output list, and the internal candidate capacity is the context's
 *    max_candidates (fixed at mhfd_create), so the size depends on the batch only.
 *  - mhfd_last_error takes no context: the detail is thread-local (the failing call
 *    may not have a context, e.g. mhfd_create or mhfd_downsample).
 *  - A blob list longer than blob_capacity is not an error: the call returns MHFD_OK,
 *    the counts stay exact and d_flags bit 1 marks the truncated images (bit 0 marks
 *    candidate-capacity overflow).  An error status would force callers that only want
 *    the leading blobs of a dense image to treat a complete, correct result as a
 *    failure; MHFD_ERR_CAPACITY is kept for an invalid capacity argument.
 *  - Defaults differ from SPEC.md's CPU program on purpose (readings R9, R11):
 *    non-strict maxima (v == maxpool(v), the paper's primitive) and
 *    threshold 0.1*dt instead of SPEC.md:254,278's strict dominance and min_response 0.
 *    strict = 1 with threshold 0 selects SPEC.md's rule; counts then differ from the
 *    defaults' on plateaus and near-zero responses.
 */
#ifndef MHFD_H
#define MHFD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MHFD_ABI_VERSION 4

typedef struct mhfd_ctx mhfd_ctx; /* opaque, immutable after mhfd_create */

typedef enum {
  MHFD_OK = 0,
  MHFD_ERR_INVALID_ARGUMENT = 1, /* bad parameter value, NULL pointer, bad enum */
  MHFD_ERR_SHAPE = 2,            /* width/height/pitch/batch not supported */
  MHFD_ERR_CAPACITY = 3,         /* blob_capacity < 0 or too large */
  MHFD_ERR_WORKSPACE = 4,        /* workspace NULL or smaller than mhfd_workspace_bytes */
  MHFD_ERR_CUDA = 5,             /* CUDA runtime / launch error (text: mhfd_last_error) */
  MHFD_ERR_DEVICE = 6            /* no CUDA device, or device is not sm_100 (B200) */
} mhfd_status;

/* Pixel types.  MHFD_F32 (ABI 3): float32 images with the same nearest-rank percentiles
 * on real values (radix select over order-preserving keys; finite values required,
 * reading R24); they run the CUDA-core schedules (k_tc is u8 only). */
typedef enum { MHFD_U8 = 1, MHFD_U16 = 2, MHFD_F32 = 3 } mhfd_dtype;

/* Feature polarity (reading R5).  MHFD_DARK: Eq. 2 as written,
 * DoG_i = t_i (L_{i+1} - L_i), dark blobs on a bright background respond positively
 * (the paper's EM sections).  MHFD_BRIGHT: DoG_i = -t_i (L_{i+1} - L_i), bright blobs
 * on a dark background; equivalent to MHFD_DARK on the inverted image 255 - I
 * (65535 - I for u16) up to rounding. */
typedef enum { MHFD_DARK = 0, MHFD_BRIGHT = 1 } mhfd_polarity;

/* Response whose scale argmax / NMS / pruning follow (ABI 3).  MHFD_RESPONSE_DOG: Eq. 2
 * (PAPER.md:169-173), the paper's detector (default).  MHFD_RESPONSE_LOG: the
 * scale-normalised Laplacian it approximates, LoG_i = t_i^2 (d_xx + d_yy) L(., t_i) at the
 * n scales t_1..t_n (Eq. 1; reading R23):
 * d_xx by zero-sum sampled second-derivative taps w2(d) = w(d)(d^2 - m2)/t^4,
 * m2 = sum_d w(d) d^2, over the same support ceil(5 t) as the blur; same sign and
 * polarity conventions as Eq. 2, responses on the LoG scale (about 1/dt times Eq. 2's).
 * width % 256 == 0 and 2n <= 62 required.  LOG runs on "k_tc2" where it fits (height %
 * 16 == 0, width >= its staged window; either boundary), else on the two-pass CUDA-core
 * schedule "k_rows_pair+k_cols_pair<log>". */
typedef enum { MHFD_RESPONSE_DOG = 0, MHFD_RESPONSE_LOG = 1 } mhfd_response;

/* Image boundary of the blur (ABI 3).  MHFD_BOUNDARY_PERIODIC: what the paper's FFT
 * computes (reading R7; default).  MHFD_BOUNDARY_REFLECT: half-sample
 * symmetric extension (scipy.ndimage 'reflect', reading R25), run on
 * k_tc for u8 DoG where it fits (mirrored tile windows), on k_tc2 for u16 / f32 / LoG
 * where it fits (the stretched image staged with mirrored margins), else on the two-pass
 * CUDA-core schedule: width % 256 == 0 required.  The NMS window keeps its -inf padding
 * either way. */
typedef enum { MHFD_BOUNDARY_PERIODIC = 0, MHFD_BOUNDARY_REFLECT = 1 } mhfd_boundary;

/* Schedule selection (ABI 4): which kernels compute rows a2-a6.  AUTO picks the fastest
 * applicable one (mhfd_schedule_name reports it); TC / BAND / GENERIC force the tcgen05
 * schedules, the u8 CUDA-core band kernel or the generic CUDA-core kernels where they
 * apply (measurement and A/B use; every choice gives results within the parity
 * tolerances of the oracle).  With AUTO the process-wide environment variable
 * MHFD_SCHEDULE=tc|band|generic, read once in mhfd_create, is honoured (tools only). */
typedef enum {
  MHFD_SCHEDULE_AUTO = 0,
  MHFD_SCHEDULE_TC = 1,
  MHFD_SCHEDULE_BAND = 2,
  MHFD_SCHEDULE_GENERIC = 3
} mhfd_schedule;

typedef enum {
  MHFD_NMS_PAPER = 0, /* Eq. 3: global argmax over scale, 3x3 local max in space (default) */
  MHFD_NMS_26 = 1     /* conventional 3x3x3 scale-space maxima, 26 neighbours */
} mhfd_nms;

/* Parameters of Algorithm 1's "Require I, n, min_t, max_t" plus
 * the north star's threshold and overlap.  Fill with mhfd_params_default()
 * and override. */
typedef struct {
  uint32_t struct_size;   /* = sizeof(mhfd_params) (forward-compatible ABI) */
  int32_t width, height;  /* image shape, fixed per context; 2*R_max+1 <= W,H <= 65535,
                             R_max = ceil(5*max_sigma) (GPU truncation radius) */
  float min_sigma;        /* min_t = t_1 > 0 (sigma = t)           */
  float max_sigma;        /* max_t = t_{n+1} > min_t, ceil(5*max_sigma) <= 160       */
  int32_t num_scales;     /* n >= 1: n+1 Gaussian levels, n DoG planes; n <= 62      */
  float threshold;        /* keep response > threshold; finite, >= 0                 */
  float overlap;          /* in [0,1]: drop a blob whose disk overlaps a kept,
                             higher-priority blob by a fraction > overlap; 1 = off  */
  float sat_low;          /* fraction of darkest pixels saturated (paper: 0.00175)   */
  float sat_high;         /* fraction of lightest pixels saturated (paper: 0.00175)  */
  int32_t nms;            /* mhfd_nms                                                */
  int32_t strict;         /* 0: v == maxpool(v) (paper); 1: strictly
                             greater than every neighbour                            */
  int32_t device;         /* CUDA device ordinal the context is bound to             */
  int32_t max_candidates; /* per-image candidate capacity before pruning;
                             0 = default ceil(W/2)*ceil(H/2) (PAPER mode) or
                             n*ceil(W/2)*ceil(H/2) (26 mode)                         */
  int32_t polarity;       /* mhfd_polarity (ABI 2; a struct_size without this field
                             reads as MHFD_DARK)                                     */
  int32_t response;       /* mhfd_response (ABI 3; a struct_size without this field
                             reads as MHFD_RESPONSE_DOG)                             */
  int32_t boundary;       /* mhfd_boundary (ABI 3; absent -> MHFD_BOUNDARY_PERIODIC)  */
  int32_t schedule;       /* mhfd_schedule (ABI 4; absent -> MHFD_SCHEDULE_AUTO)      */
} mhfd_params;

/* One detected feature (x^_j, y^_j, i^_j) of Eq. 3 and its DoG
 * response. 16 bytes. */
typedef struct {
  int32_t x, y, scale;
  float response;
} mhfd_blob;

/* Paper defaults: sigma 1..10, n = 10, threshold 0.1*dt, overlap 0.5, 0.175% per
 * tail, Eq. 3 NMS, non-strict.  width/height are set to 0 (caller must set). */
void mhfd_params_default(mhfd_params* p);

/* Validate parameters and build the context (scale grid, f32 tap tables).
 * Errors: INVALID_ARGUMENT (p/out NULL, struct_size too small, sigma <= 0,
 * max <= min, n < 1 or n > 62, threshold < 0 or not finite, overlap not in
 * [0,1], sat fractions not in [0,0.5), nms/strict out of range,
 * ceil(5*max_sigma) > 160), SHAPE (width/height out of range),
 * DEVICE (device ordinal invalid or not compute capability 10.0). */
mhfd_status mhfd_create(const mhfd_params* p, mhfd_ctx** out);

/* Bytes of device workspace one call with `batch` images needs (batch >= 1).
 * Linear in batch; for 4096^2 PAPER mode about 5.5 B/px + 3*max_candidates*16 B
 * per image. */
mhfd_status mhfd_workspace_bytes(const mhfd_ctx* c, int32_t batch, size_t* bytes);

/* Detect blobs in `batch` images.
 *  d_images     : batch x height rows of pitch_bytes (u8 or u16 per `dtype`)
 *  d_workspace  : >= mhfd_workspace_bytes(c, batch) bytes, 256-byte aligned
 *  d_blobs      : batch x blob_capacity records; image b's kept blobs are at
 *                 d_blobs + b*blob_capacity, sorted by (y, x, scale); only the
 *                 first min(count, blob_capacity) are written
 *  d_counts     : batch int32, the exact number of kept blobs per image (the
 *                 focus score |C|), also when it exceeds blob_capacity
 *  d_flags      : nullable; batch int32, bit0 = candidate capacity exceeded
 *                 (pruning saw only the first max_candidates candidates in
 *                 raster order), bit1 = list truncated to blob_capacity
 * Errors: INVALID_ARGUMENT, SHAPE, CAPACITY (blob_capacity < 0), WORKSPACE, CUDA. */
mhfd_status mhfd_detect_batch(mhfd_ctx* c, const void* d_images, int32_t dtype, int32_t batch,
                              int64_t pitch_bytes, void* d_workspace, size_t workspace_bytes,
                              mhfd_blob* d_blobs, int32_t blob_capacity, int32_t* d_counts,
                              int32_t* d_flags, void* stream);

/* Focus score only: d_scores[b] = (double)|C_b|; d_counts
 * (nullable) receives the int32 counts.  Same work as mhfd_detect_batch minus
 * writing the blob list. */
mhfd_status mhfd_focus_score(mhfd_ctx* c, const void* d_images, int32_t dtype, int32_t batch,
                             int64_t pitch_bytes, void* d_workspace, size_t workspace_bytes,
                             double* d_scores, int32_t* d_counts, void* stream);

/* End-to-end call with HOST buffers (the e2e path): h_images is batch x height
 * rows of pitch_bytes in host memory (pinned for overlap; pageable works but
 * serialises).  The batch is processed in chunks of at most
 *   chunk = staging_bytes / (3 * height * pitch_bytes)   images (>= 1 required):
 * d_staging holds three slots of `chunk` images, used round-robin; the next chunks
 * are copied host->device into free slots on a context-owned copy stream while
 * earlier ones are processed on `stream`, and each chunk's scores are copied
 * device->host into h_scores (batch doubles) and, if non-NULL, h_counts.
 * Back-to-back calls with the same staging buffer pipeline: a call's copies wait only
 * for the compute that last used their slot, so they overlap the previous call's last
 * chunks, and such a call uses whole chunks throughout; a call that finds the device
 * idle ramps its chunks up (1, 2, 3, ... images) so compute starts after one image's
 * copy.  The staging buffer therefore stays in use until `stream` is synchronised.
 * d_workspace must hold mhfd_workspace_bytes(c, chunk).  Outputs are valid after
 * the caller synchronises `stream` (h_scores / h_counts of a call are written by its
 * own chunks only).  Uses context-owned streams/events: do not call concurrently on
 * the same context.
 * Errors: as mhfd_focus_score; WORKSPACE if the staging holds < 1 image per slot. */
mhfd_status mhfd_focus_score_host(mhfd_ctx* c, const void* h_images, int32_t dtype, int32_t batch,
                                  int64_t pitch_bytes, void* d_staging, size_t staging_bytes,
                                  void* d_workspace, size_t workspace_bytes, double* h_scores,
                                  int32_t* h_counts, void* stream);

/* Per-stage device timing (bench instrumentation; not thread-safe).
 * mhfd_timing_enable(c, k) arms k records (k = 0 disables); each subsequent
 * mhfd_detect_batch / mhfd_focus_score call records CUDA events on its stream
 * around its 4 stages: [0] percentiles (a1), [1] the fused blur kernel (a2-a6,
 * the one mhfd_schedule_name names),
 * [2] NMS + compaction (a7-a8), [3] pruning + score (a9-a10).
 * mhfd_timing_read waits for the recorded events and writes ms[call*4 + stage]
 * for *ncalls (<= k) calls. */
mhfd_status mhfd_timing_enable(mhfd_ctx* c, int32_t max_calls);
mhfd_status mhfd_timing_read(mhfd_ctx* c, float* ms, int32_t* ncalls);

/* Introspection for parity tests (same kernels as the two calls above):
 *  d_lohi  : nullable, batch x 2 int32 (percentile values lo, hi)
 *  d_dog   : nullable, batch x n x height x width f32 DoG planes (Eq. 2)
 *  d_v     : nullable, batch x height x width f32 max_i DoG (Eq. 3 inner argmax)
 *  d_idx   : nullable, batch x height x width u8 first argmax (0-based)
 *  d_cands : nullable, batch x max_candidates blobs before pruning (raster order)
 *  d_ncand : nullable, batch int32 exact candidate counts before pruning */
mhfd_status mhfd_debug_dump(mhfd_ctx* c, const void* d_images, int32_t dtype, int32_t batch,
                            int64_t pitch_bytes, void* d_workspace, size_t workspace_bytes,
                            int32_t* d_lohi, float* d_dog, float* d_v, uint8_t* d_idx,
                            mhfd_blob* d_cands, int32_t* d_ncand, void* stream);

/* Single-image multi-GPU spatial sharding.  The image is split into
 * row bands, one per GPU; every GPU holds the whole image (the caller broadcasts it),
 * so a band needs no halo exchange: its blur windows and its Eq. 3 NMS neighbours
 * (rows y0-1 and y1) are evaluated locally, and the percentiles are those of the whole
 * image.  The bands' candidate lists, concatenated in band order (NCCL all-gather), are
 * the whole image's candidate list in raster order, bit-identical to the one
 * mhfd_detect_batch prunes; mhfd_prune_candidates then prunes it and scores the image
 * (the only step that needs every band: overlaps cross band edges).
 *
 * mhfd_detect_band: candidates of rows [y0, y1) of ONE image.
 *  d_image        : height x pitch_bytes bytes (the "k_tc" schedule for u8, or the
 *                   "k_rows_pair+k_cols_pair" schedule for u16/f32; Eq. 3 NMS)
 *  0 <= y0 < y1 <= height; width % 1024 == 0
 *  d_workspace    : >= mhfd_workspace_bytes(c, 1)
 *  d_cands        : cand_capacity records; the band's candidates in (y, x) order,
 *                   truncated to cand_capacity (the count is exact)
 *  d_ncand        : 1 int32, the band's exact candidate count
 * Errors: as mhfd_detect_batch; SHAPE for the band/width; INVALID_ARGUMENT when the
 * context's schedule for dtype is neither of those two. */
mhfd_status mhfd_detect_band(mhfd_ctx* c, const void* d_image, int32_t dtype, int64_t pitch_bytes, int32_t y0,
                             int32_t y1, void* d_workspace, size_t workspace_bytes, mhfd_blob* d_cands,
                             int32_t cand_capacity, int32_t* d_ncand, void* stream);

/* mhfd_prune_candidates: pruning + focus score of one image from its full candidate
 * list (ncand records at d_cands, raster (y, x) order, ncand <= the context's
 * max_candidates).  d_blobs (nullable if blob_capacity == 0): kept blobs in (y, x,
 * scale) order; d_count, d_score (nullable), d_flags (nullable): as mhfd_detect_batch /
 * mhfd_focus_score for one image.  d_workspace as mhfd_detect_band. */
mhfd_status mhfd_prune_candidates(mhfd_ctx* c, const mhfd_blob* d_cands, int32_t ncand, void* d_workspace,
                                  size_t workspace_bytes, mhfd_blob* d_blobs, int32_t blob_capacity,
                                  int32_t* d_count, double* d_score, int32_t* d_flags, void* stream);

/* Sharded pruning of one image ("border-blob exchange for pruning";
 * the paper's gather bottleneck): instead of every rank pruning the
 * gathered full list, rank r prunes only its band [y0, y1) from the candidates of an
 * extended band [e0, e1) (mhfd_detect_band on the extended rows) and the ranks sum their
 * counts (one all-reduce of 8 bytes).
 *
 * mhfd_prune_band: the pruning rule of mhfd_prune_candidates applied to the ncand
 * raster-ordered candidates of rows [e0, e1) (0 <= e0 <= y0 < y1 <= e1 <= height), in
 * synchronous rounds (a round's decisions read only the previous rounds' states, so a
 * blob decided in round t depends only on the candidates within (t + 1) D of it, D =
 * mhfd_interaction_radius).  d_count (1 int32) = kept blobs with y0 <= y < y1.  d_cert
 * (1 int32) = 1 when every such blob was decided in a round t with (t + 1) D <= its
 * distance to a truncated edge of [e0, e1) (e0 > 0 or e1 < height), i.e. when d_count is
 * provably the whole image's count of kept blobs in [y0, y1); else 0, and the caller
 * falls back to mhfd_prune_candidates on the gathered full list.  Errors: as
 * mhfd_prune_candidates; SHAPE for the row ranges.  d_nband (nullable, 1 int32) = the
 * candidates with y0 <= y < y1 (their sum over the bands is the image's candidate count,
 * which the caller compares with max_candidates: mhfd_detect_batch truncates the list).
 *
 * mhfd_interaction_radius: D in pixels, the largest pruning search radius (a blob's
 * decision can only involve candidates closer than D in one round); -1 if c is NULL. */
mhfd_status mhfd_prune_band(mhfd_ctx* c, const mhfd_blob* d_cands, int32_t ncand, int32_t e0, int32_t e1, int32_t y0,
                            int32_t y1, void* d_workspace, size_t workspace_bytes, int32_t* d_count, int32_t* d_cert,
                            int32_t* d_nband, void* stream);
int32_t mhfd_interaction_radius(const mhfd_ctx* c);

/* mhfd_downsample: the bilinear downsampling pre-step (PAPER.md:401
 * "preprocessing by downsampling, by bilinear interpolation, in order to satisfy GPU RAM
 * constraints"; SPEC.md:48-56 fixes the output shape ceil(W/f) x ceil(H/f) and factor 1 =
 * identity).  Context-free.  Output pixel (X, Y) samples the input at the pixel-centre
 * coordinates x = (X + 1/2) f - 1/2, y = (Y + 1/2) f - 1/2 (half-pixel convention), with
 * bilinear weights and both neighbour indices clamped to the last row/column; for an integer
 * factor the fractional parts are 0 (odd f: the sample is one pixel) or 1/2 (even f: the
 * mean of a 2 x 2, 2 x 1 or 1 x 1 block), so the exact value is a multiple of 1/4 and is
 * rounded half up to the input's integer type (reading R22).
 *  d_in      : batch images, height x in_pitch bytes each (u8 or u16, row-major)
 *  d_out     : batch images, ceil(height/f) x out_pitch bytes each, same dtype
 *  factor    : 1 <= factor <= min(width, height)
 * Errors: INVALID_ARGUMENT (null pointer, bad dtype, factor, batch < 0); SHAPE (width or
 * height < 1 or > 65535, a pitch smaller than its row or not a multiple of the pixel
 * size); CUDA (launch).  Enqueued on
 * `stream`; nothing is enqueued on a validation error. */
mhfd_status mhfd_downsample(const void* d_in, int32_t dtype, int32_t width, int32_t height, int64_t in_pitch,
                            int32_t factor, void* d_out, int64_t out_pitch, int32_t batch, void* stream);

/* Read back the parameters a context was built with (derived fields filled). */
mhfd_status mhfd_get_params(const mhfd_ctx* c, mhfd_params* out);

/* Name of the kernel that computes rows a2-a6 (stretch, blur, DoG, scale argmax)
 * for images of `dtype` in mhfd_detect_batch / mhfd_focus_score on this context:
 * "k_tc" (u8, Eq. 3 NMS, tensor-core banded blur; default when the staged tile
 * fits), "k_band" (u8, CUDA-core band schedule), "k_scale_space"
 * (generic: widths that are not multiples of 256, MHFD_SCHEDULE=generic, and DoG-plane
 * calls below R_max 96), or the two-pass schedule through an HBM row-blur intermediate:
 * "k_rows_pair+k_cols_pair" (Eq. 3 NMS, width % 256 == 0, any radius; also the
 * MHFD_RESPONSE_LOG contexts k_tc2 does not fit, named "k_rows_pair+k_cols_pair<log>"),
 * "k_rows2+k_cols_all"
 * (DoG planes at R_max >= 96: 3x3x3 mode, dumps, MHFD_NO_COLS_PAIR=1).  params.schedule
 * (or, with MHFD_SCHEDULE_AUTO, the environment variable MHFD_SCHEDULE=tc|band|generic
 * read at mhfd_create) selects among the applicable ones.  Static string; "none" for a
 * NULL context. */
const char* mhfd_schedule_name(const mhfd_ctx* c, int32_t dtype);

/* Floating-point operations per output pixel that the kernel named by
 * mhfd_schedule_name executes by construction (bench roofline): for "k_tc" the
 * tensor-core MMA flops of the banded formulation (sum over levels of
 * 2 x 2*128*K_i^2 + 3 x 2*128*128*K_i per 128 x 128 tile, K_i = the level's
 * window); otherwise the direct separable blur, 2 x 2(2R_i+1) FMA
 * per level plus 3 per DoG plane.  0 for a NULL context. */
double mhfd_schedule_flops_per_pixel(const mhfd_ctx* c, int32_t dtype);

/* Number of kernel launches the last successful call on this thread enqueued. */
int32_t mhfd_last_launch_count(void);

/* NULL-safe. */
void mhfd_destroy(mhfd_ctx* c);

/* Static string for a status code. */
const char* mhfd_status_string(mhfd_status s);

/* Thread-local detail of the last failing call on this thread ("" if none). */
const char* mhfd_last_error(void);

/* MHFD_ABI_VERSION of the built library. */
int32_t mhfd_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MHFD_H */
