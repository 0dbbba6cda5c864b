/*
 * mhfd_oracle.c — CPU ORACLE for the MHFD hot path (arXiv 2108.12050).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link,
 * load or execute this file: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it.  It shares no
 * code, header, table or constant with paper_2108_12050_b200/ (the CUDA
 * path), and it does not include any header from include/.
 *
 * What it computes, in the paper's order and notation ("PAPER.md:N" is line
 * N of the paper's LaTeX; readings R1..R21 are listed in DESIGN.md §3):
 *
 *   1. percentiles  lo, hi            PAPER.md:255-259 (§3 histogram stretch),
 *                                      nearest rank per SPEC.md:112 (reading R13)
 *   2. stretch      I' = clamp((I-lo)/(hi-lo), 0, 1)
 *   3. scale grid   dt = (max_t-min_t)/n, t_i = min_t+(i-1)dt
 *   4. Gaussian     G(x,y,t) = exp(-(x^2+y^2)/2t^2)/(2 pi t^2)
 *                   sampled at integer offsets, renormalised to unit sum,
 *                   truncated at R = ceil(6 t)            (reading R6)
 *   5. scale space  L(.,.,t_i) = G(.,.,t_i) * I'  periodic (reading R7:
 *                   the paper's Fourier-domain product, PAPER.md:248-253,
 *                   is a circular convolution)
 *   6. DoG (Eq. 2)  DoG(x,y,i) = t_i (L(x,y,t_{i+1}) - L(x,y,t_i)), i=1..n
 *                                                         PAPER.md:169-173
 *   7a. Eq. 3 NMS   v = max_i DoG, i^ = first argmax;
 *                   keep p iff v(p) == maxpool_3x3(v)(p)
 *                   and v(p) > tau (threshold: north_star, reading R11)
 *   7b. 26-NMS      conventional 3x3x3 scale-space maxima
 *   8. pruning      greedy blob-overlap pruning (north_star; reading R12)
 *   9. score        DOF = |C|
 *
 * Arithmetic is IEEE double throughout.  Convolution is direct (no FFT),
 * NMS is brute force over the neighbourhood, pruning is O(n^2).  The only
 * parallelism is an OpenMP "parallel for" over independent output rows,
 * which does not change any result.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_PI 3.14159265358979323846

/* A detected feature (x^_j, y^_j, i^_j) of Eq. 3 plus its response
 * (PAPER.md:233).  x = column, y = row, scale = i^ - 1 (0-based). */
typedef struct {
  int32_t x, y, scale, pad;
  double response;
} oracle_blob;

int oracle_abi_version(void) { return 1; }

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ */
/* 1. Percentiles — PAPER.md:257 ".175% of the darkest ... .175% of the
 * lightest"; nearest rank on the sorted pixel list:
 * k_lo = floor(sat_low*N), lo = sorted[k_lo]; k_hi = floor(sat_high*N),
 * hi = sorted[N-1-k_hi].                                               */
static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

static uint32_t pixel_at(const void* img, int bytes_per_px, int64_t i) {
  if (bytes_per_px == 1) return ((const uint8_t*)img)[i];
  return ((const uint16_t*)img)[i];
}

int oracle_percentiles(const void* img, int bytes_per_px, int64_t npx,
                       double sat_low, double sat_high, int64_t* lo, int64_t* hi) {
  if (npx <= 0 || (bytes_per_px != 1 && bytes_per_px != 2)) return -1;
  uint32_t* s = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)npx);
  if (!s) return -2;
  for (int64_t i = 0; i < npx; ++i) s[i] = pixel_at(img, bytes_per_px, i);
  qsort(s, (size_t)npx, sizeof(uint32_t), cmp_u32);
  int64_t klo = (int64_t)floor(sat_low * (double)npx);
  int64_t khi = (int64_t)floor(sat_high * (double)npx);
  if (klo > npx - 1) klo = npx - 1;
  if (khi > npx - 1) khi = npx - 1;
  *lo = s[klo];
  *hi = s[npx - 1 - khi];
  free(s);
  return 0;
}

/* 2. Stretch — PAPER.md:257 "mapping the entire range to [0,1]";
 * hi == lo gives the all-zero image (reading R14).        */
void oracle_stretch(const void* img, int bytes_per_px, int64_t npx,
                    int64_t lo, int64_t hi, double* out) {
  for (int64_t i = 0; i < npx; ++i) {
    if (hi == lo) { out[i] = 0.0; continue; }
    double v = ((double)pixel_at(img, bytes_per_px, i) - (double)lo) / (double)(hi - lo);
    out[i] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  }
}

/* f32 input (SURVEY 8(f) f3 "f32 input dtype with a float-quantile select"; reading R24):
 * the same nearest-rank percentiles on the real values (finite inputs; -0.0 and +0.0
 * are equal values) and the same stretch, in f64.  lo/hi are returned as doubles. */
static int cmp_f64(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

int oracle_percentiles_f32(const float* img, int64_t npx, double sat_low, double sat_high, double* lo, double* hi) {
  if (npx <= 0) return -1;
  double* s = (double*)malloc(sizeof(double) * (size_t)npx);
  if (!s) return -2;
  for (int64_t i = 0; i < npx; ++i) s[i] = (double)img[i];
  qsort(s, (size_t)npx, sizeof(double), cmp_f64);
  int64_t klo = (int64_t)floor(sat_low * (double)npx);
  int64_t khi = (int64_t)floor(sat_high * (double)npx);
  if (klo > npx - 1) klo = npx - 1;
  if (khi > npx - 1) khi = npx - 1;
  *lo = s[klo];
  *hi = s[npx - 1 - khi];
  free(s);
  return 0;
}

void oracle_stretch_f32(const float* img, int64_t npx, double lo, double hi, double* out) {
  for (int64_t i = 0; i < npx; ++i) {
    if (hi == lo) { out[i] = 0.0; continue; }
    double v = ((double)img[i] - lo) / (hi - lo);
    out[i] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  }
}

/* 3. Scale grid — PAPER.md:167: dt = (max_t - min_t)/n,
 * t_i = min_t + (i-1) dt, i = 1..n+1 (n+1 levels, reading R2).          */
void oracle_scale_grid(double min_t, double max_t, int n, double* t) {
  double dt = (max_t - min_t) / (double)n;
  for (int i = 1; i <= n + 1; ++i) t[i - 1] = min_t + (double)(i - 1) * dt;
}

/* 4. Gaussian filter — PAPER.md:136 G(x,y,sigma) = exp(-(x^2+y^2)/2 sigma^2)
 * / (2 pi sigma^2) with sigma = t (reading R1).
 * The 2-D kernel sampled on |x|,|y| <= R and renormalised to unit sum is
 * exactly the outer product of the renormalised 1-D samples below, so the
 * 2-D convolution is evaluated as a row pass followed by a column pass.  */
int oracle_radius(double t) { return (int)ceil(6.0 * t); }

double oracle_gaussian_2d(double x, double y, double sigma) {
  return exp(-(x * x + y * y) / (2.0 * sigma * sigma)) / (2.0 * ORACLE_PI * sigma * sigma);
}

void oracle_gaussian_taps(double t, int R, double* w /* 2R+1 */) {
  double s = 0.0;
  for (int d = -R; d <= R; ++d) {
    w[d + R] = exp(-(double)(d * d) / (2.0 * t * t));
    s += w[d + R];
  }
  for (int d = -R; d <= R; ++d) w[d + R] /= s;
}

/* Image boundary of the blur: periodic (reading R7, the default) or half-sample
 * symmetric reflection (SURVEY 8(f) f3 "reflect boundary", reading R25: ... c b a | a b c
 * ... x y z | z y x ..., scipy.ndimage mode 'reflect').  A process-wide setting of this
 * test oracle (oracle_set_boundary; the Python wrapper sets and restores it per call). */
static int g_boundary = 0;
void oracle_set_boundary(int b) { g_boundary = b ? 1 : 0; }
int oracle_get_boundary(void) { return g_boundary; }

static int64_t wrap(int64_t a, int64_t m) {
  if (g_boundary) {
    while (a < 0 || a >= m) a = a < 0 ? -a - 1 : 2 * m - 1 - a;
    return a;
  }
  int64_t r = a % m;
  return r < 0 ? r + m : r;
}

/* 5. Scale space — PAPER.md:140 L(x,y,t) = G(x,y,t) * I(x,y), periodic
 * boundary (reading R7).  Computes output rows [y0, y1) of L.          */
void oracle_blur_rows(const double* f, int H, int W, double t, int y0, int y1, double* L /* (y1-y0) x W */) {
  int R = oracle_radius(t);
  double* w = (double*)malloc(sizeof(double) * (size_t)(2 * R + 1));
  oracle_gaussian_taps(t, R, w);
  int nrow = (y1 - y0) + 2 * R;            /* input rows y0-R .. y1+R-1 */
  double* tmp = (double*)malloc(sizeof(double) * (size_t)nrow * (size_t)W);
  /* row pass: tmp(r, x) = sum_b w[b] f(r, x+b) */
#pragma omp parallel for schedule(static)
  for (int r = 0; r < nrow; ++r) {
    const double* src = f + wrap((int64_t)(y0 - R + r), H) * W;
    for (int x = 0; x < W; ++x) {
      double acc = 0.0;
      for (int b = -R; b <= R; ++b) acc += w[b + R] * src[wrap((int64_t)x + b, W)];
      tmp[(int64_t)r * W + x] = acc;
    }
  }
  /* column pass: L(y, x) = sum_a w[a] tmp(y+a, x) */
#pragma omp parallel for schedule(static)
  for (int y = y0; y < y1; ++y) {
    double* dst = L + (int64_t)(y - y0) * W;
    for (int x = 0; x < W; ++x) dst[x] = 0.0;
    for (int a = -R; a <= R; ++a) {
      const double* src = tmp + (int64_t)(y - y0 + R + a) * W;
      double wa = w[a + R];
      for (int x = 0; x < W; ++x) dst[x] += wa * src[x];
    }
  }
  free(tmp);
  free(w);
}

void oracle_blur(const double* f, int H, int W, double t, double* L) {
  oracle_blur_rows(f, H, W, t, 0, H, L);
}

/* 6. DoG stack, Eq. 2: D_i = t_i (L_{i+1} - L_i), i = 1..n,
 * for output rows [y0, y1).  D is n planes of (y1-y0) x W.              */
void oracle_dog_stack_rows(const double* f, int H, int W, double min_t, double max_t, int n,
                           int y0, int y1, double* D) {
  double* t = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  oracle_scale_grid(min_t, max_t, n, t);
  int64_t plane = (int64_t)(y1 - y0) * W;
  double* Lprev = (double*)malloc(sizeof(double) * (size_t)plane);
  double* Lcur = (double*)malloc(sizeof(double) * (size_t)plane);
  oracle_blur_rows(f, H, W, t[0], y0, y1, Lprev);
  for (int i = 1; i <= n; ++i) {
    oracle_blur_rows(f, H, W, t[i], y0, y1, Lcur);
    double* Di = D + (int64_t)(i - 1) * plane;
    for (int64_t p = 0; p < plane; ++p) Di[p] = t[i - 1] * (Lcur[p] - Lprev[p]);
    double* s = Lprev; Lprev = Lcur; Lcur = s;
  }
  free(Lprev); free(Lcur); free(t);
}

void oracle_dog_stack(const double* f, int H, int W, double min_t, double max_t, int n, double* D) {
  oracle_dog_stack_rows(f, H, W, min_t, max_t, n, 0, H, D);
}

/* Scale-normalised Laplacian response (SURVEY 8(f) f3 "true sigma^2 lap L"
 * Eq. 1 and :163 "t^2 lap^2 L"; reading R23): LoG_i = t_i^2 (d_xx + d_yy) L(., t_i) for the
 * n scales t_1..t_n of Eq. 2's planes.  Discrete second derivative of the sampled,
 * renormalised Gaussian (taps w, support R): w2(d) = w(d) (d^2 - m2) / t^4 with
 * m2 = sum_d w(d) d^2, so sum_d w2 = 0 (a constant image responds 0) and
 * sum_d w2(d) d^2 / 2 = (sum w d^4 - m2^2) / (2 t^4) ~ 1; the 2-D operator is the sum
 * of the two separable products w2 (x) w + w (x) w2, periodic boundary. */
void oracle_log_taps(double t, int R, double* w /* 2R+1 */, double* w2 /* 2R+1 */) {
  oracle_gaussian_taps(t, R, w);
  double m2 = 0.0;
  for (int d = -R; d <= R; ++d) m2 += w[d + R] * (double)d * d;
  const double t4 = t * t * t * t;
  for (int d = -R; d <= R; ++d) w2[d + R] = w[d + R] * ((double)d * d - m2) / t4;
}

void oracle_log_stack_rows(const double* f, int H, int W, double min_t, double max_t, int n,
                           int y0, int y1, double* D) {
  double* t = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  oracle_scale_grid(min_t, max_t, n, t);
  const int64_t plane = (int64_t)(y1 - y0) * W;
  for (int i = 0; i < n; ++i) {
    const int R = oracle_radius(t[i]);
    double* w = (double*)malloc(sizeof(double) * (size_t)(2 * R + 1));
    double* w2 = (double*)malloc(sizeof(double) * (size_t)(2 * R + 1));
    oracle_log_taps(t[i], R, w, w2);
    const int nrow = (y1 - y0) + 2 * R;   /* input rows y0-R .. y1+R-1 */
    double* A = (double*)malloc(sizeof(double) * (size_t)nrow * (size_t)W);    /* w  along x */
    double* Bx = (double*)malloc(sizeof(double) * (size_t)nrow * (size_t)W);   /* w2 along x */
#pragma omp parallel for schedule(static)
    for (int r = 0; r < nrow; ++r) {
      const double* src = f + wrap((int64_t)(y0 - R + r), H) * W;
      for (int x = 0; x < W; ++x) {
        double a = 0.0, bb = 0.0;
        for (int b = -R; b <= R; ++b) {
          const double v = src[wrap((int64_t)x + b, W)];
          a += w[b + R] * v;
          bb += w2[b + R] * v;
        }
        A[(int64_t)r * W + x] = a;
        Bx[(int64_t)r * W + x] = bb;
      }
    }
    double* Di = D + (int64_t)i * plane;
    const double t2 = t[i] * t[i];
#pragma omp parallel for schedule(static)
    for (int y = y0; y < y1; ++y) {
      for (int x = 0; x < W; ++x) {
        double yy = 0.0, xx = 0.0;   /* d_yy L: w2 along y of A;  d_xx L: w along y of Bx */
        for (int a = -R; a <= R; ++a) {
          const int64_t r = (int64_t)(y - y0 + R + a) * W + x;
          yy += w2[a + R] * A[r];
          xx += w[a + R] * Bx[r];
        }
        Di[(int64_t)(y - y0) * W + x] = t2 * (xx + yy);
      }
    }
    free(A); free(Bx); free(w); free(w2);
  }
  free(t);
}

/* DoG at one pixel, evaluated straight from the 2-D definition
 * (sum over the (2R+1)^2 window of G * I', periodic) — used to check
 * sampled outputs of full-size images.  Dvec receives n values.          */
void oracle_dog_at(const double* f, int H, int W, double min_t, double max_t, int n,
                   int y, int x, double* Dvec) {
  double* t = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  oracle_scale_grid(min_t, max_t, n, t);
  double Lprev = 0.0;
  for (int i = 0; i <= n; ++i) {
    int R = oracle_radius(t[i]);
    double* w = (double*)malloc(sizeof(double) * (size_t)(2 * R + 1));
    oracle_gaussian_taps(t[i], R, w);
    double L = 0.0;
    for (int a = -R; a <= R; ++a) {
      const double* row = f + wrap((int64_t)y + a, H) * W;
      for (int b = -R; b <= R; ++b) L += w[a + R] * w[b + R] * row[wrap((int64_t)x + b, W)];
    }
    free(w);
    if (i > 0) Dvec[i - 1] = t[i - 1] * (L - Lprev);
    Lprev = L;
  }
  free(t);
}

/* ------------------------------------------------------------------ */
/* 7a. Eq. 3: inner argmax over ALL scales (first
 * maximum on ties, PAPER.md:244 / reading R10), outer local argmax over
 * space by comparison with maxpool_2d(3,3) with -inf padding
 * (reading R8); threshold v > tau (reading R11).  strict=1 requires v to
 * exceed every neighbour (reading R9).                     */
void oracle_scale_argmax(const double* D, int n, int64_t plane, double* v, int32_t* idx) {
  for (int64_t p = 0; p < plane; ++p) {
    double best = D[p];
    int bi = 0;
    for (int i = 1; i < n; ++i) {
      double d = D[(int64_t)i * plane + p];
      if (d > best) { best = d; bi = i; }
    }
    v[p] = best;
    idx[p] = bi;
  }
}

int64_t oracle_nms_paper_v(const double* v, const int32_t* idx, int H, int W, double tau, int strict,
                           oracle_blob* out, int64_t cap) {
  int64_t cnt = 0;
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      double c = v[(int64_t)y * W + x];
      if (!(c > tau)) continue;
      int ok = 1;
      for (int dy = -1; dy <= 1 && ok; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (dy == 0 && dx == 0) continue;
          int yy = y + dy, xx = x + dx;
          if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue; /* -inf padding */
          double q = v[(int64_t)yy * W + xx];
          if (strict ? !(c > q) : !(c >= q)) { ok = 0; break; }
        }
      if (!ok) continue;
      if (cnt < cap) {
        out[cnt].x = x; out[cnt].y = y; out[cnt].scale = idx[(int64_t)y * W + x];
        out[cnt].pad = 0; out[cnt].response = c;
      }
      ++cnt;
    }
  return cnt;
}

int64_t oracle_nms_paper(const double* D, int n, int H, int W, double tau, int strict,
                         oracle_blob* out, int64_t cap) {
  int64_t plane = (int64_t)H * W;
  double* v = (double*)malloc(sizeof(double) * (size_t)plane);
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)plane);
  oracle_scale_argmax(D, n, plane, v, idx);
  int64_t c = oracle_nms_paper_v(v, idx, H, W, tau, strict, out, cap);
  free(v); free(idx);
  return c;
}

/* 7b. Conventional scale-space maxima: (p, i) is kept iff
 * D_i(p) >= D_j(q) for every existing (q, j) of the 3x3x3 box around
 * (p, i) other than itself (-inf padding in space, scale window truncated
 * at 1 and n: reading R16), and D_i(p) > tau.  Output order: raster, then
 * scale ascending (reading R18).                                         */
int64_t oracle_nms_26(const double* D, int n, int H, int W, double tau, int strict,
                      oracle_blob* out, int64_t cap) {
  int64_t plane = (int64_t)H * W, cnt = 0;
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x)
      for (int i = 0; i < n; ++i) {
        double c = D[(int64_t)i * plane + (int64_t)y * W + x];
        if (!(c > tau)) continue;
        int ok = 1;
        for (int di = -1; di <= 1 && ok; ++di) {
          int j = i + di;
          if (j < 0 || j >= n) continue;
          for (int dy = -1; dy <= 1 && ok; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              if (di == 0 && dy == 0 && dx == 0) continue;
              int yy = y + dy, xx = x + dx;
              if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
              double q = D[(int64_t)j * plane + (int64_t)yy * W + xx];
              if (strict ? !(c > q) : !(c >= q)) { ok = 0; break; }
            }
        }
        if (!ok) continue;
        if (cnt < cap) {
          out[cnt].x = x; out[cnt].y = y; out[cnt].scale = i; out[cnt].pad = 0; out[cnt].response = c;
        }
        ++cnt;
      }
  return cnt;
}

/* ------------------------------------------------------------------ */
/* 8. Blob-overlap pruning (north_star "blob-overlap pruning"; not in the
 * paper — reading R12).  A blob of scale index s has radius
 * r = sqrt(2) * t_{s+1} (t of its DoG plane).  The overlap fraction of two
 * blobs is the lens (intersection) area of their disks divided by the
 * area of the smaller disk: 0 if d >= r1 + r2, 1 if d <= |r1 - r2|.
 * Blobs are visited in priority order (scale descending, then raster
 * ascending); a blob is kept iff no already-kept blob overlaps it by a
 * fraction > overlap.  overlap >= 1 keeps every blob.                   */
double oracle_lens_fraction(double d, double r1, double r2) {
  double rmin = r1 < r2 ? r1 : r2;
  if (d >= r1 + r2) return 0.0;
  if (d <= fabs(r1 - r2)) return 1.0;
  double a1 = (d * d + r1 * r1 - r2 * r2) / (2.0 * d * r1);
  double a2 = (d * d + r2 * r2 - r1 * r1) / (2.0 * d * r2);
  if (a1 > 1.0) a1 = 1.0; if (a1 < -1.0) a1 = -1.0;
  if (a2 > 1.0) a2 = 1.0; if (a2 < -1.0) a2 = -1.0;
  double k = (-d + r1 + r2) * (d + r1 - r2) * (d - r1 + r2) * (d + r1 + r2);
  if (k < 0.0) k = 0.0;
  double area = r1 * r1 * acos(a1) + r2 * r2 * acos(a2) - 0.5 * sqrt(k);
  return area / (ORACLE_PI * rmin * rmin);
}

static const oracle_blob* g_sort_blobs;
static int cmp_priority(const void* a, const void* b) {
  const oracle_blob* p = &g_sort_blobs[*(const int64_t*)a];
  const oracle_blob* q = &g_sort_blobs[*(const int64_t*)b];
  if (p->scale != q->scale) return p->scale > q->scale ? -1 : 1;
  if (p->y != q->y) return p->y < q->y ? -1 : 1;
  if (p->x != q->x) return p->x < q->x ? -1 : 1;
  return 0;
}

int64_t oracle_prune(const oracle_blob* c, int64_t nc, double min_t, double max_t, int n,
                     double overlap, uint8_t* keep) {
  if (overlap >= 1.0) {
    for (int64_t k = 0; k < nc; ++k) keep[k] = 1;
    return nc;
  }
  double* t = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  oracle_scale_grid(min_t, max_t, n, t);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
  int64_t* kept = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
  for (int64_t k = 0; k < nc; ++k) { order[k] = k; keep[k] = 0; }
  g_sort_blobs = c;
  qsort(order, (size_t)nc, sizeof(int64_t), cmp_priority);
  int64_t nk = 0;
  for (int64_t o = 0; o < nc; ++o) {
    const oracle_blob* b = &c[order[o]];
    double rb = sqrt(2.0) * t[b->scale];
    int ok = 1;
    for (int64_t m = 0; m < nk; ++m) {
      const oracle_blob* q = &c[kept[m]];
      double rq = sqrt(2.0) * t[q->scale];
      double dx = (double)(b->x - q->x), dy = (double)(b->y - q->y);
      if (oracle_lens_fraction(sqrt(dx * dx + dy * dy), rb, rq) > overlap) { ok = 0; break; }
    }
    if (ok) { keep[order[o]] = 1; kept[nk++] = order[o]; }
  }
  free(order); free(kept); free(t);
  return nk;
}

/* 8b. The same greedy rule with an exact early-out for large lists (round 2; reading
 * R12 unchanged).  A pair at distance d >= r_b + r_q has lens fraction 0, which never
 * exceeds overlap >= 0, so only kept blobs closer than r_b + r_q <= 2 r_max can drop
 * b.  Kept blobs are filed in square cells of edge >= 2 r_max; b is tested against the
 * kept blobs of its own and the 8 adjacent cells with the same oracle_lens_fraction and
 * the same "> overlap" comparison, in the same priority order, so every decision equals
 * oracle_prune's (pinned: tests/test_oracle_pins.py compares the two on clustered random
 * lists).  Used for lists of 10^5 blobs (4096^2 tiles), where the O(n^2) scan takes
 * minutes.                                                                           */
int64_t oracle_prune_grid(const oracle_blob* c, int64_t nc, double min_t, double max_t, int n,
                          double overlap, uint8_t* keep) {
  if (overlap >= 1.0 || nc == 0) {
    for (int64_t k = 0; k < nc; ++k) keep[k] = 1;
    return nc;
  }
  double* t = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  oracle_scale_grid(min_t, max_t, n, t);
  double rmax = 0.0;
  for (int i = 0; i <= n; ++i) if (sqrt(2.0) * t[i] > rmax) rmax = sqrt(2.0) * t[i];
  int32_t xmin = c[0].x, xmax = c[0].x, ymin = c[0].y, ymax = c[0].y;
  for (int64_t k = 1; k < nc; ++k) {
    if (c[k].x < xmin) xmin = c[k].x;
    if (c[k].x > xmax) xmax = c[k].x;
    if (c[k].y < ymin) ymin = c[k].y;
    if (c[k].y > ymax) ymax = c[k].y;
  }
  const int64_t cell = (int64_t)ceil(2.0 * rmax) + 1;
  const int64_t gx = (xmax - xmin) / cell + 1, gy = (ymax - ymin) / cell + 1;
  int64_t* head = (int64_t*)malloc(sizeof(int64_t) * (size_t)(gx * gy));   /* kept blobs per cell */
  int64_t* next = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
  for (int64_t k = 0; k < gx * gy; ++k) head[k] = -1;
  for (int64_t k = 0; k < nc; ++k) { order[k] = k; keep[k] = 0; }
  g_sort_blobs = c;
  qsort(order, (size_t)nc, sizeof(int64_t), cmp_priority);
  int64_t nk = 0;
  for (int64_t o = 0; o < nc; ++o) {
    const int64_t bi = order[o];
    const oracle_blob* b = &c[bi];
    const double rb = sqrt(2.0) * t[b->scale];
    const int64_t cx = (b->x - xmin) / cell, cy = (b->y - ymin) / cell;
    int ok = 1;
    for (int64_t yy = cy - 1; yy <= cy + 1 && ok; ++yy) {
      if (yy < 0 || yy >= gy) continue;
      for (int64_t xx = cx - 1; xx <= cx + 1 && ok; ++xx) {
        if (xx < 0 || xx >= gx) continue;
        for (int64_t m = head[yy * gx + xx]; m >= 0; m = next[m]) {
          const oracle_blob* q = &c[m];
          const double rq = sqrt(2.0) * t[q->scale];
          const double dx = (double)(b->x - q->x), dy = (double)(b->y - q->y);
          if (oracle_lens_fraction(sqrt(dx * dx + dy * dy), rb, rq) > overlap) { ok = 0; break; }
        }
      }
    }
    if (ok) {
      keep[bi] = 1;
      ++nk;
      next[bi] = head[cy * gx + cx];
      head[cy * gx + cx] = bi;
    }
  }
  free(head); free(next); free(order); free(t);
  return nk;
}

/* Pruning used by oracle_detect*: 0 = oracle_prune (O(n^2), default), 1 = oracle_prune_grid
 * (identical decisions; set by the Python wrapper for full-size images only). */
static int g_prune_grid = 0;
void oracle_set_prune_grid(int on) { g_prune_grid = on ? 1 : 0; }

/* ------------------------------------------------------------------ */
/* 9. End to end, Algorithm 1 with the threshold and the
 * pruning of north_star.  nms: 0 = Eq. 3 (paper), 1 = 26-neighbour.
 * Returns the number of kept blobs (the focus score DOF = |C|,
 * PAPER.md:236); `out` receives up to `cap` kept blobs in (y, x, scale)
 * order; *n_cand receives the candidate count before pruning; D_dump
 * (nullable) receives the n DoG planes; v_dump/idx_dump (nullable) the
 * Eq. 3 inner argmax.  Returns -1 on allocation failure.                 */
int64_t oracle_detect_resp(const void* img, int bytes_per_px, int H, int W,
                           double min_t, double max_t, int n, double tau, double overlap,
                           double sat_low, double sat_high, int nms, int strict, int polarity, int response,
                           oracle_blob* out, int64_t cap, int64_t* n_cand,
                           double* D_dump, double* v_dump, int32_t* idx_dump,
                           int64_t* lo_out, int64_t* hi_out) {
  int64_t plane = (int64_t)H * W;
  double* f = (double*)malloc(sizeof(double) * (size_t)plane);
  if (!f) return -1;
  if (bytes_per_px == 4) {   /* f32 input (reading R24); lo/hi reported as their float32 bit patterns */
    double flo, fhi;
    if (oracle_percentiles_f32((const float*)img, plane, sat_low, sat_high, &flo, &fhi) != 0) { free(f); return -1; }
    float l32 = (float)flo, h32 = (float)fhi;
    uint32_t lb, hb;
    memcpy(&lb, &l32, 4);
    memcpy(&hb, &h32, 4);
    if (lo_out) *lo_out = (int64_t)lb;
    if (hi_out) *hi_out = (int64_t)hb;
    oracle_stretch_f32((const float*)img, plane, flo, fhi, f);
  } else {
    int64_t lo, hi;
    if (oracle_percentiles(img, bytes_per_px, plane, sat_low, sat_high, &lo, &hi) != 0) { free(f); return -1; }
    if (lo_out) *lo_out = lo;
    if (hi_out) *hi_out = hi;
    oracle_stretch(img, bytes_per_px, plane, lo, hi, f);
  }
  double* D = D_dump ? D_dump : (double*)malloc(sizeof(double) * (size_t)plane * (size_t)n);
  if (!D) { free(f); return -1; }
  if (response == 1) oracle_log_stack_rows(f, H, W, min_t, max_t, n, 0, H, D);   /* reading R23 */
  else oracle_dog_stack(f, H, W, min_t, max_t, n, D);
  /* polarity (not in the paper): bright features use the negated
   * Eq. 2 response D_i = -t_i (L_{i+1} - L_i) */
  if (polarity)
    for (int64_t i = 0; i < plane * n; ++i) D[i] = -D[i];
  int64_t ccap = nms == 0 ? plane : plane * n;
  oracle_blob* cand = (oracle_blob*)malloc(sizeof(oracle_blob) * (size_t)ccap);
  int64_t nc;
  if (nms == 0) {
    double* v = v_dump ? v_dump : (double*)malloc(sizeof(double) * (size_t)plane);
    int32_t* idx = idx_dump ? idx_dump : (int32_t*)malloc(sizeof(int32_t) * (size_t)plane);
    oracle_scale_argmax(D, n, plane, v, idx);
    nc = oracle_nms_paper_v(v, idx, H, W, tau, strict, cand, ccap);
    if (!v_dump) free(v);
    if (!idx_dump) free(idx);
  } else {
    nc = oracle_nms_26(D, n, H, W, tau, strict, cand, ccap);
  }
  if (n_cand) *n_cand = nc;
  uint8_t* keep = (uint8_t*)malloc((size_t)(nc > 0 ? nc : 1));
  int64_t nk = g_prune_grid ? oracle_prune_grid(cand, nc, min_t, max_t, n, overlap, keep)
                            : oracle_prune(cand, nc, min_t, max_t, n, overlap, keep);
  int64_t w = 0;
  for (int64_t k = 0; k < nc; ++k)
    if (keep[k]) { if (w < cap) out[w] = cand[k]; ++w; }
  free(keep); free(cand); free(f);
  if (!D_dump) free(D);
  return nk;
}

int64_t oracle_detect_pol(const void* img, int bytes_per_px, int H, int W,
                          double min_t, double max_t, int n, double tau, double overlap,
                          double sat_low, double sat_high, int nms, int strict, int polarity,
                          oracle_blob* out, int64_t cap, int64_t* n_cand,
                          double* D_dump, double* v_dump, int32_t* idx_dump,
                          int64_t* lo_out, int64_t* hi_out) {
  return oracle_detect_resp(img, bytes_per_px, H, W, min_t, max_t, n, tau, overlap, sat_low, sat_high, nms, strict,
                            polarity, 0, out, cap, n_cand, D_dump, v_dump, idx_dump, lo_out, hi_out);
}

/* Algorithm 1 as written (dark features, Eq. 2). */
int64_t oracle_detect(const void* img, int bytes_per_px, int H, int W,
                      double min_t, double max_t, int n, double tau, double overlap,
                      double sat_low, double sat_high, int nms, int strict,
                      oracle_blob* out, int64_t cap, int64_t* n_cand,
                      double* D_dump, double* v_dump, int32_t* idx_dump,
                      int64_t* lo_out, int64_t* hi_out) {
  return oracle_detect_pol(img, bytes_per_px, H, W, min_t, max_t, n, tau, overlap, sat_low, sat_high, nms, strict, 0,
                           out, cap, n_cand, D_dump, v_dump, idx_dump, lo_out, hi_out);
}

/* Bilinear downsampling pre-step.  PAPER.md:401: "preprocessing by
 * downsampling, by bilinear interpolation"; output ceil(W/f) x ceil(H/f),
 * factor 1 = identity, values by a scalar bilinear formula at sample centres.  Textbook
 * bilinear interpolation in f64: output (X, Y) samples the input at x = (X + 1/2) f - 1/2,
 * y = (Y + 1/2) f - 1/2; x0 = floor(x), fx = x - x0, both neighbours x0, x0 + 1 clamped
 * to W - 1 (the last of ceil(W/f) samples may lie past the last column; same for y); value = (1-fy)((1-fx) p(y0,x0) + fx p(y0,x1)) + fy((1-fx) p(y1,x0) + fx p(y1,x1)),
 * rounded half up to the input's integer type (reading R22).  Returns 0, or -1 on bad
 * arguments. */
int oracle_downsample(const void* img, int bytes_per_px, int H, int W, int f, void* out) {
  if (f < 1 || f > H || f > W || (bytes_per_px != 1 && bytes_per_px != 2)) return -1;
  const int OH = (H + f - 1) / f, OW = (W + f - 1) / f;
  for (int Y = 0; Y < OH; ++Y) {
    const double y = (Y + 0.5) * f - 0.5;
    const int y0f = (int)floor(y);
    const double fy = y - y0f;
    const int y0 = y0f < H ? y0f : H - 1;   /* ceil(H/f) rows: the last sample may lie past row H-1 */
    const int y1 = y0f + 1 < H ? y0f + 1 : H - 1;
    for (int X = 0; X < OW; ++X) {
      const double x = (X + 0.5) * f - 0.5;
      const int x0f = (int)floor(x);
      const double fx = x - x0f;
      const int x0 = x0f < W ? x0f : W - 1;
      const int x1 = x0f + 1 < W ? x0f + 1 : W - 1;
      double p00, p01, p10, p11;
      if (bytes_per_px == 1) {
        const uint8_t* a = (const uint8_t*)img;
        p00 = a[(int64_t)y0 * W + x0]; p01 = a[(int64_t)y0 * W + x1];
        p10 = a[(int64_t)y1 * W + x0]; p11 = a[(int64_t)y1 * W + x1];
      } else {
        const uint16_t* a = (const uint16_t*)img;
        p00 = a[(int64_t)y0 * W + x0]; p01 = a[(int64_t)y0 * W + x1];
        p10 = a[(int64_t)y1 * W + x0]; p11 = a[(int64_t)y1 * W + x1];
      }
      const double v = (1.0 - fy) * ((1.0 - fx) * p00 + fx * p01) + fy * ((1.0 - fx) * p10 + fx * p11);
      const double r = floor(v + 0.5);
      if (bytes_per_px == 1) ((uint8_t*)out)[(int64_t)Y * OW + X] = (uint8_t)r;
      else ((uint16_t*)out)[(int64_t)Y * OW + X] = (uint16_t)r;
    }
  }
  return 0;
}
