/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 * See oracle.h for the contract; every function cites the reference
 * (wavecgh 0.1.0, /root/reference/proj) file:line it restates. */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* haar.cpp:12-30 — one averaging 2x2 analysis level. */
static void analyze_level(const double* in, int n, double* a, double* h, double* v, double* d) {
  const int m = n / 2;
  for (int y = 0; y < m; ++y) {
    for (int x = 0; x < m; ++x) {
      const double c00 = in[(size_t)(2 * y) * n + 2 * x];
      const double c01 = in[(size_t)(2 * y) * n + 2 * x + 1];
      const double c10 = in[(size_t)(2 * y + 1) * n + 2 * x];
      const double c11 = in[(size_t)(2 * y + 1) * n + 2 * x + 1];
      const size_t o = (size_t)y * m + x;
      a[o] = (c00 + c01 + c10 + c11) * 0.25;
      h[o] = (c00 - c01 + c10 - c11) * 0.25;
      v[o] = (c00 + c01 - c10 - c11) * 0.25;
      d[o] = (c00 - c01 - c10 + c11) * 0.25;
    }
  }
}

/* haar.cpp:52-74 */
int orc_haar_analyze(const double* image, int n, int levels, double* pyramid) {
  if (levels < 1 || n % (1 << levels) != 0) return 1;
  double* cur = malloc(sizeof(double) * (size_t)n * n);
  memcpy(cur, image, sizeof(double) * (size_t)n * n);
  const int ma = n >> levels;
  double* out = pyramid + (size_t)ma * ma;
  int side = n;
  for (int l = 0; l < levels; ++l) {
    const int m = side / 2;
    const size_t mm = (size_t)m * m;
    double* a = malloc(sizeof(double) * mm);
    analyze_level(cur, side, a, out, out + mm, out + 2 * mm);
    out += 3 * mm;
    free(cur);
    cur = a;
    side = m;
  }
  memcpy(pyramid, cur, sizeof(double) * (size_t)ma * ma);
  free(cur);
  return 0;
}

/* haar.cpp:32-48 with a == 0 (expand_residual, haar.cpp:88-96). */
void orc_expand_residual(const double* h, const double* v, const double* d, int m, double* out) {
  const int n = 2 * m;
  for (int y = 0; y < m; ++y) {
    for (int x = 0; x < m; ++x) {
      const size_t o = (size_t)y * m + x;
      const double av = 0.0, hh = h[o], vv = v[o], dd = d[o];
      out[(size_t)(2 * y) * n + 2 * x] = av + hh + vv + dd;
      out[(size_t)(2 * y) * n + 2 * x + 1] = av - hh + vv - dd;
      out[(size_t)(2 * y + 1) * n + 2 * x] = av + hh - vv - dd;
      out[(size_t)(2 * y + 1) * n + 2 * x + 1] = av - hh - vv + dd;
    }
  }
}

/* haar.cpp:98-109 */
void orc_upsample_replicate(const double* coarse, int m, int factor, double* out) {
  const int n = m * factor;
  for (int y = 0; y < n; ++y)
    for (int x = 0; x < n; ++x) out[(size_t)y * n + x] = coarse[(size_t)(y / factor) * m + x / factor];
}

/* saliency.cpp:12-26 */
static void block_max(const double* full, int n, int f, double* out) {
  const int m = n / f;
  for (int y = 0; y < m; ++y) {
    for (int x = 0; x < m; ++x) {
      double best = 0.0;
      for (int by = 0; by < f; ++by)
        for (int bx = 0; bx < f; ++bx) {
          const double s = full[(size_t)(y * f + by) * n + (size_t)x * f + bx];
          best = s > best ? s : best; /* std::max(best, s) */
        }
      out[(size_t)y * m + x] = best;
    }
  }
}

/* saliency.cpp:41-61 */
int orc_quantize_saliency(const double* sal, int n, double* sal_pyr) {
  if (n % 8 != 0) return 1;
  for (size_t i = 0; i < (size_t)n * n; ++i)
    if (!(sal[i] >= 0.0 && sal[i] <= 1.0)) return 1;
  const size_t q2 = (size_t)(n / 2) * (n / 2), q4 = (size_t)(n / 4) * (n / 4);
  block_max(sal, n, 2, sal_pyr);
  block_max(sal, n, 4, sal_pyr + q2);
  block_max(sal, n, 8, sal_pyr + q2 + q4);
  return 0;
}

/* Gate loop (synthesis.cpp:107-119): strict '>' against the threshold. */
static uint64_t gate(const double* level, int m, double t, int enabled, uint8_t* mask) {
  uint64_t count = 0;
  for (size_t i = 0; i < (size_t)m * m; ++i) {
    const uint8_t on = (uint8_t)(enabled && level[i] > t);
    mask[i] = on;
    count += on;
  }
  return count;
}

int orc_analysis(const double* object, const double* saliency, int n, const double* thresholds,
                 const int* enables, double* pyramid, double* sal_pyr, uint8_t* masks,
                 double* a_eff, uint64_t* ops) {
  /* RefinementPlan::validate (synthesis.cpp:127-131) */
  if (!(0.0 <= thresholds[0] && thresholds[0] <= thresholds[1] &&
        thresholds[1] <= thresholds[2] && thresholds[2] <= 1.0))
    return 1;
  if (n < 8 || n % 8 != 0) return 1;
  for (size_t i = 0; i < (size_t)n * n; ++i)
    if (!isfinite(object[i])) return 1; /* require_finite (field.cpp:55-61) */

  const size_t n2 = (size_t)n * n, h2 = n2 / 4, q2 = n2 / 16, e2 = n2 / 64;
  double* pyr = malloc(sizeof(double) * (e2 + 3 * (h2 + q2 + e2)));
  double* sp = malloc(sizeof(double) * (h2 + q2 + e2));
  uint8_t* mk = malloc(q2 + h2 + n2);
  if (orc_quantize_saliency(saliency, n, sp)) {
    free(pyr), free(sp), free(mk);
    return 1;
  }
  orc_haar_analyze(object, n, 3, pyr);

  /* stage order: LL uses details[2] + by_factor(4), L uses details[1] +
   * by_factor(2), full uses details[0] + the full map (synthesis.cpp:246-250) */
  const double* lll = pyr;
  const double* det0 = pyr + e2;            /* h,v,d at n/2 */
  const double* det1 = det0 + 3 * h2;       /* at n/4 */
  const double* det2 = det1 + 3 * q2;       /* at n/8 */
  uint64_t c_ll = gate(sp + h2, n / 4, thresholds[0], enables[0], mk);
  uint64_t c_l = gate(sp, n / 2, thresholds[1], enables[1], mk + q2);
  uint64_t c_full = gate(saliency, n, thresholds[2], enables[2], mk + q2 + h2);

  if (a_eff) {
    double* r_ll = malloc(sizeof(double) * q2);
    double* r_l = malloc(sizeof(double) * h2);
    double* r_f = malloc(sizeof(double) * n2);
    orc_expand_residual(det2, det2 + e2, det2 + 2 * e2, n / 8, r_ll);
    orc_expand_residual(det1, det1 + q2, det1 + 2 * q2, n / 4, r_l);
    orc_expand_residual(det0, det0 + h2, det0 + 2 * h2, n / 2, r_f);
    for (int y = 0; y < n; ++y) {
      for (int x = 0; x < n; ++x) {
        double a = lll[(size_t)(y / 8) * (n / 8) + x / 8];
        const size_t i4 = (size_t)(y / 4) * (n / 4) + x / 4;
        const size_t i2 = (size_t)(y / 2) * (n / 2) + x / 2;
        const size_t i1 = (size_t)y * n + x;
        if (mk[i4]) a += r_ll[i4];
        if (mk[q2 + i2]) a += r_l[i2];
        if (mk[q2 + h2 + i1]) a += r_f[i1];
        a_eff[i1] = a;
      }
    }
    free(r_ll), free(r_l), free(r_f);
  }
  if (pyramid) memcpy(pyramid, pyr, sizeof(double) * (e2 + 3 * (h2 + q2 + e2)));
  if (sal_pyr) memcpy(sal_pyr, sp, sizeof(double) * (h2 + q2 + e2));
  if (masks) memcpy(masks, mk, q2 + h2 + n2);
  if (ops) {
    ops[0] = e2; /* base covers every LLL cell (synthesis.cpp:77-88) */
    ops[1] = c_ll;
    ops[2] = c_l;
    ops[3] = c_full;
    ops[4] = 0;
  }
  free(pyr), free(sp), free(mk);
  return 0;
}

int64_t orc_compact(const double* a_eff, int n, int off, int32_t* xs, int32_t* ys, double* amps) {
  int64_t k = 0;
  for (int y = 0; y < n; ++y)
    for (int x = 0; x < n; ++x) {
      const double a = a_eff[(size_t)y * n + x];
      if (a == 0.0) continue; /* oracles.cpp:25 skips zero amplitudes */
      if (xs) xs[k] = x + off;
      if (ys) ys[k] = y + off;
      if (amps) amps[k] = a;
      ++k;
    }
  return k;
}

/* fringe_lut.cpp:27-32 */
void orc_point_fringe(double wavelength, double pitch, double z, int dx, int dy, double* out2) {
  const double px = dx * pitch, py = dy * pitch;
  const double r = sqrt(px * px + py * py + z * z);
  const double k = 2.0 * M_PI / wavelength; /* field.cpp:82 */
  out2[0] = (1.0 / r) * cos(k * r);
  out2[1] = (1.0 / r) * sin(k * r);
}

/* tests/support/oracles.cpp:12-36 over a point list. */
void orc_direct_pixels(const int32_t* xs, const int32_t* ys, const double* amps,
                       const int32_t* layer, int64_t n_points, const double* wavelength,
                       const double* pitch, const double* z, const int32_t* px,
                       const int32_t* py, int64_t n_pix, double* out) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < n_pix; ++i) {
    double sr = 0.0, si = 0.0;
    for (int64_t j = 0; j < n_points; ++j) {
      const int l = layer ? layer[j] : 0;
      const double k = 2.0 * M_PI / wavelength[l];
      const double dx = (double)(px[i] - xs[j]) * pitch[l];
      const double dy = (double)(py[i] - ys[j]) * pitch[l];
      const double r = sqrt(dx * dx + dy * dy + z[l] * z[l]);
      const double m = amps[j] * (1.0 / r);
      sr += m * cos(k * r);
      si += m * sin(k * r);
    }
    out[2 * i] = sr;
    out[2 * i + 1] = si;
  }
}

/* fringe_lut.cpp:53-93 */
int orc_build_block_lut(double wavelength, double pitch, double z, int n, int block, double* out) {
  if (!(block == 1 || block == 2 || block == 4 || block == 8) || block > n) return 1;
  const int span = 2 * n - 1, ext = span + block - 1, lo = -(n - 1) - (block - 1);
  double* base = malloc(sizeof(double) * 2 * (size_t)ext * ext);
#pragma omp parallel for
  for (int row = 0; row < ext; ++row)
    for (int col = 0; col < ext; ++col)
      orc_point_fringe(wavelength, pitch, z, lo + col, lo + row, base + 2 * ((size_t)row * ext + col));
#pragma omp parallel for
  for (int row = 0; row < span; ++row) {
    for (int col = 0; col < span; ++col) {
      double sr = 0.0, si = 0.0;
      for (int pv = 0; pv < block; ++pv) {
        const double* src = base + 2 * (size_t)(row - pv + block - 1) * ext;
        for (int pu = 0; pu < block; ++pu) {
          sr += src[2 * (col - pu + block - 1)];
          si += src[2 * (col - pu + block - 1) + 1];
        }
      }
      out[2 * ((size_t)row * span + col)] = sr;
      out[2 * ((size_t)row * span + col) + 1] = si;
    }
  }
  free(base);
  return 0;
}

/* synthesis.cpp:18-42 */
void orc_apply_block(double* plane, int n, const double* support, int ax, int ay, double w_re,
                     double w_im) {
  if (w_re == 0.0 && w_im == 0.0) return;
  const int sw = 2 * n - 1;
  for (int y = 0; y < n; ++y) {
    const double* s = support + 2 * ((size_t)(y - ay + n - 1) * sw + (size_t)(n - 1 - ax));
    double* p = plane + 2 * (size_t)y * n;
    for (int x = 0; x < n; ++x) {
      const double sr = s[2 * x], si = s[2 * x + 1];
      p[2 * x] += w_re * sr - w_im * si;
      p[2 * x + 1] += w_re * si + w_im * sr;
    }
  }
}

/* apply_cells (synthesis.cpp:55-69) without the chunked scratch planes:
 * sequential in cell order (the reference's result is bitwise independent of
 * workers; this restatement is within rounding of it). */
static void apply_cells(double* plane, int n, const double* lut, int b, int m, const uint8_t* on,
                        const double* w) {
  for (int cy = 0; cy < m; ++cy)
    for (int cx = 0; cx < m; ++cx)
      if (!on || on[(size_t)cy * m + cx]) orc_apply_block(plane, n, lut, cx * b, cy * b, w[(size_t)cy * m + cx], 0.0);
}

/* synthesis.cpp:180-253 (real amplitudes). */
int orc_synthesize_progressive(const double* object, const double* saliency, int n,
                               const double* thresholds, const int* enables,
                               const double* const* luts, double* planes, double* after_full,
                               uint8_t* masks, uint64_t* ops) {
  const size_t n2 = (size_t)n * n, h2 = n2 / 4, q2 = n2 / 16, e2 = n2 / 64;
  double* pyr = malloc(sizeof(double) * (e2 + 3 * (h2 + q2 + e2)));
  uint8_t* mk = malloc(q2 + h2 + n2);
  uint64_t lops[5];
  if (orc_analysis(object, saliency, n, thresholds, enables, pyr, NULL, mk, NULL, lops)) {
    free(pyr), free(mk);
    return 1;
  }
  double* plane = calloc(2 * n2, sizeof(double));
  double* res = malloc(sizeof(double) * n2);
  const double* det0 = pyr + e2;
  const double* det1 = det0 + 3 * h2;
  const double* det2 = det1 + 3 * q2;
  apply_cells(plane, n, luts[3], 8, n / 8, NULL, pyr); /* base_stage */
  if (planes) memcpy(planes, plane, sizeof(double) * 2 * n2);
  orc_expand_residual(det2, det2 + e2, det2 + 2 * e2, n / 8, res);
  apply_cells(plane, n, luts[2], 4, n / 4, mk, res);
  if (planes) memcpy(planes + 2 * n2, plane, sizeof(double) * 2 * n2);
  orc_expand_residual(det1, det1 + q2, det1 + 2 * q2, n / 4, res);
  apply_cells(plane, n, luts[1], 2, n / 2, mk + q2, res);
  if (planes) memcpy(planes + 4 * n2, plane, sizeof(double) * 2 * n2);
  orc_expand_residual(det0, det0 + h2, det0 + 2 * h2, n / 2, res);
  apply_cells(plane, n, luts[0], 1, n, mk + q2 + h2, res);
  if (planes) memcpy(planes + 6 * n2, plane, sizeof(double) * 2 * n2);
  if (after_full) memcpy(after_full, plane, sizeof(double) * 2 * n2);
  if (masks) memcpy(masks, mk, q2 + h2 + n2);
  if (ops) memcpy(ops, lops, sizeof(lops));
  free(pyr), free(mk), free(plane), free(res);
  return 0;
}

/* metrics.cpp:18-46 */
static double* integral_table(const double* a, const double* b, int w, int h, int which) {
  double* t = calloc((size_t)(w + 1) * (h + 1), sizeof(double));
  for (int y = 0; y < h; ++y) {
    double* cur = t + (size_t)(y + 1) * (w + 1);
    const double* prev = t + (size_t)y * (w + 1);
    for (int x = 0; x < w; ++x) {
      const double ra = a[(size_t)y * w + x], rb = b[(size_t)y * w + x];
      double v = 0.0;
      switch (which) {
        case 0: v = ra; break;
        case 1: v = rb; break;
        case 2: v = ra * ra; break;
        case 3: v = rb * rb; break;
        default: v = ra * rb; break;
      }
      cur[x + 1] = v + cur[x] + prev[x + 1] - prev[x];
    }
  }
  return t;
}

static double window_sum(const double* t, int stride, int x, int y, int win) {
  return t[(size_t)(y + win) * stride + x + win] - t[(size_t)(y + win) * stride + x] -
         t[(size_t)y * stride + x + win] + t[(size_t)y * stride + x];
}

/* metrics.cpp:50-85 */
double orc_ssim(const double* a, const double* b, int w, int h, int window, double k1, double k2,
                double dynamic_range) {
  double* t[5];
  for (int i = 0; i < 5; ++i) t[i] = integral_table(a, b, w, h, i);
  const int stride = w + 1;
  const double c1 = (k1 * dynamic_range) * (k1 * dynamic_range);
  const double c2 = (k2 * dynamic_range) * (k2 * dynamic_range);
  const double inv_n = 1.0 / ((double)window * (double)window);
  double total = 0.0;
  size_t count = 0;
  for (int y = 0; y + window <= h; ++y)
    for (int x = 0; x + window <= w; ++x) {
      const double mu_a = window_sum(t[0], stride, x, y, window) * inv_n;
      const double mu_b = window_sum(t[1], stride, x, y, window) * inv_n;
      const double var_a = window_sum(t[2], stride, x, y, window) * inv_n - mu_a * mu_a;
      const double var_b = window_sum(t[3], stride, x, y, window) * inv_n - mu_b * mu_b;
      const double cov = window_sum(t[4], stride, x, y, window) * inv_n - mu_a * mu_b;
      total += ((2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2)) /
               ((mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2));
      ++count;
    }
  for (int i = 0; i < 5; ++i) free(t[i]);
  return total / (double)count;
}
