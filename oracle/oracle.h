/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference (wavecgh 0.1.0) hot path, in fp64,
 * used by tests/ and bench.py's cpu_baseline leg to check the CUDA path.
 * Each function cites the reference file:line it restates (paths relative
 * to /root/reference/proj). The restatement is pinned against the reference
 * itself (oracle/_ref, compiled from the unmodified sources) and against the
 * committed golden vectors in tests/golden/.
 *
 * Layout conventions (all row-major, square):
 *   pyramid  : approx (n>>L)^2, then for l = 0..L-1 (finest first) h, v, d
 *              each (n>>(l+1))^2                      (haar.hpp:20-34)
 *   sal_pyr  : half (n/2)^2, quarter (n/4)^2, eighth (n/8)^2 (saliency.hpp:64-76)
 *   masks    : mask_ll (n/4)^2, mask_l (n/2)^2, mask_full n^2 (synthesis.hpp:43-54)
 *   complex  : interleaved (re, im) doubles
 */
#ifndef WCGH_ORACLE_H
#define WCGH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* haar.cpp:12-30 + 52-74. Returns 0, or 1 on a dimension error. */
int orc_haar_analyze(const double* image, int n, int levels, double* pyramid);
/* haar.cpp:32-48 + 88-96: synthesis with a zero approximation. */
void orc_expand_residual(const double* h, const double* v, const double* d, int m, double* out);
/* haar.cpp:98-109 */
void orc_upsample_replicate(const double* coarse, int m, int factor, double* out);
/* saliency.cpp:12-26 + 41-61. Returns 1 on a validation error. */
int orc_quantize_saliency(const double* sal, int n, double* sal_pyr);

/* The analysis half of synthesize_progressive (synthesis.cpp:216-251):
 * pyramid, saliency pyramid, strict-'>' gates (synthesis.cpp:107-119),
 * operator counts (synthesis.cpp:68: base counts every LLL cell) and the
 * effective amplitude A_eff = up8(LLL) + sum_stage mask_s (.) up_B(residual_s),
 * whose point-wise hologram equals after_full (SURVEY.md §0 finding 1).
 * thresholds = {t_ll, t_l, t_full}; enables = {ll, l, full}.
 * Any output pointer may be NULL. ops[5] follows OpLevel (field.hpp:114-120).
 * Returns 0, or 1 on a validation error. */
int orc_analysis(const double* object, const double* saliency, int n, const double* thresholds,
                 const int* enables, double* pyramid, double* sal_pyr, uint8_t* masks,
                 double* a_eff, uint64_t* ops);

/* Order-preserving compaction of nonzero A_eff samples (row-major
 * ascending, the order pointwise_sum visits them, tests/support/oracles.cpp:
 * 18-26). Writes (x + off, y + off) hologram coordinates and amplitudes.
 * Returns the count. Any output may be NULL (count only). */
int64_t orc_compact(const double* a_eff, int n, int off, int32_t* xs, int32_t* ys, double* amps);

/* point_fringe (fringe_lut.cpp:27-32). */
void orc_point_fringe(double wavelength, double pitch, double z, int dx, int dy, double* out2);

/* Direct Eq.(1) over a compacted point list, restating pointwise_sum
 * (tests/support/oracles.cpp:12-36) with per-point layers (z per layer; a
 * multi-depth scene is the per-layer sum). Evaluates the
 * n_pix hologram pixels (px[i], py[i]) into out (complex). OpenMP over pixels. */
void orc_direct_pixels(const int32_t* xs, const int32_t* ys, const double* amps,
                       const int32_t* layer, int64_t n_points, const double* wavelength,
                       const double* pitch, const double* z, const int32_t* px,
                       const int32_t* py, int64_t n_pix, double* out);

/* build_block_lut (fringe_lut.cpp:53-93): (2n-1)^2 complex support. */
int orc_build_block_lut(double wavelength, double pitch, double z, int n, int block, double* out);

/* apply_block_unchecked (synthesis.cpp:18-42) on an n x n plane. */
void orc_apply_block(double* plane, int n, const double* support, int ax, int ay, double w_re,
                     double w_im);

/* synthesize_progressive (synthesis.cpp:180-253), LUT method, real
 * amplitudes, object == plane size, with LUTs luts[0..3] for B = 1,2,4,8.
 * planes: 4 x n^2 complex (base, after_ll, after_l, after_full) or NULL for
 * after_full only in `after_full`. Returns 0 or 1 (validation). */
int orc_synthesize_progressive(const double* object, const double* saliency, int n,
                               const double* thresholds, const int* enables,
                               const double* const* luts, double* planes, double* after_full,
                               uint8_t* masks, uint64_t* ops);

/* metrics.cpp:18-85 (summed-area-table SSIM). */
double orc_ssim(const double* a, const double* b, int w, int h, int window, double k1, double k2,
                double dynamic_range);

#ifdef __cplusplus
}
#endif

#endif
