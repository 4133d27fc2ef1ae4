/* wcgh.h — C ABI of the B200-native Fresnel hot path (sm_100a CUDA kernels).
 *
 * Drop-in boundary for the reference wavecgh 0.1.0 hot path
 * (/root/reference/proj). The reference has no C ABI, plugin registry or FFI;
 * its "operator API" is the set of C++ free functions listed beside each
 * entry point below. Those functions keep their names, argument meaning and
 * error behaviour in the host mirrors above this ABI (Python:
 * paper_2211_09938_b200/stages.py, hologram.py; C++: integration/wavecgh_gpu.cpp) and call
 * these entry points, which launch the kernels. There is no CPU fallback: a
 * missing device or a CUDA failure returns WCGH_ERUNTIME.
 *
 * Conventions
 *  - Every call returns WCGH_OK (0), WCGH_EVALIDATION (1, the reference's
 *    ValidationError, errors.hpp:10-13, CLI exit 1) or WCGH_ERUNTIME (2, the
 *    IoError class, errors.hpp:17-20, CLI exit 2). No C++ exception crosses
 *    the ABI; the message is in wcgh_last_error().
 *  - Buffers are caller-owned. Unless a name ends in _dev, pointers are HOST
 *    pointers (pinned or pageable) and calls are synchronous: results are
 *    complete on return. Device memory is owned by the context / job.
 *  - All images are square and row-major. Complex outputs are interleaved
 *    float32 (re, im) = complex64, the CGHL/CGH1 payload layout
 *    (fringe_lut.cpp:107-113, image_io.cpp:220-242).
 *  - One context per GPU and host thread (one process per GPU). `workers`
 *    arguments of the reference have no counterpart: results are bitwise
 *    independent of the launch configuration and of the row-band split, the
 *    GPU analogue of accumulate_deterministic (parallel.hpp:163-171).
 */
#ifndef WCGH_H
#define WCGH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WCGH_ABI_VERSION 1

enum { WCGH_OK = 0, WCGH_EVALIDATION = 1, WCGH_ERUNTIME = 2 };

/* Input sample types. U8 objects are amplitudes v * obj_scale; U8 saliency is
 * v * (1/255), the reference loader's scale_to_unit (image_io.cpp:177-190).
 * C128 (job objects only) is an interleaved complex<double> amplitude, the
 * random-initial-phase object of synthesize_progressive(..., seed)
 * (synthesis.cpp:205-219; make it with wcgh_random_phase_field). */
enum { WCGH_U8 = 0, WCGH_F32 = 1, WCGH_F64 = 2, WCGH_C128 = 3 };

/* Synthesis method. DIRECT evaluates Eq.(1) per (point, pixel) on the SFU
 * (tests/support/oracles.cpp:12-36 applied to the effective amplitude);
 * LUT is the reference's production block-LUT superposition
 * (synthesis.cpp:18-42, 55-69) for block sizes 8/4/2/1. */
enum { WCGH_METHOD_DIRECT = 0, WCGH_METHOD_LUT = 1, WCGH_METHOD_FFT = 2 };
/* FFT: the same hologram as a circular correlation of A_eff with the point
 * fringe on a 2Nh x 2Nh grid (hand-written FFTs, no cuFFT), O(Nh^2 log Nh);
 * SURVEY.md §8(f) row 4. */

/* Phase evaluation for DIRECT. FIXED: exact 0.64 fixed-point quadratic phase
 * frac(s * p^2/(2 lambda z)) + fp32 higher-order correction; FP64: r and
 * k*r in double, then fp32 sin/cos of the reduced phase. */
enum { WCGH_PHASE_FIXED = 0, WCGH_PHASE_FP64 = 1 };

/* Operator levels, OpLevel (field.hpp:114-120). */
enum { WCGH_OP_BASE_LLL = 0, WCGH_OP_REFINE_LL, WCGH_OP_REFINE_L, WCGH_OP_REFINE_FULL,
       WCGH_OP_POINTWISE_ORACLE, WCGH_OP_LEVELS };

/* One depth layer: SceneParams (field.hpp:91-108) minus plane_size. */
typedef struct {
  double wavelength; /* m */
  double pitch;      /* m per pixel (object and hologram share the grid) */
  double z;          /* m, object layer to hologram distance */
} wcgh_layer;

/* RefinementPlan (synthesis.hpp:18-29). */
typedef struct {
  double t_ll, t_l, t_full;
  int enable_ll, enable_l, enable_full;
} wcgh_plan;

/* Compacted effective-amplitude point: hologram-grid coordinates (object
 * offset applied), amplitude, depth layer. 16 bytes, the record the
 * accumulation kernel stages through shared memory. */
typedef struct {
  int32_t x, y;
  float a;
  int32_t layer;
} wcgh_point;

/* A hologram job: n_layers objects of object_size^2 samples centred on a
 * plane_size^2 hologram (offset (plane_size - object_size)/2, a multiple of
 * 8 so Haar cells align with the reference's zero-padded run), of which this
 * context computes rows [row0, row0 + rows). */
typedef struct {
  int object_size;  /* No: multiple of 8 */
  int plane_size;   /* Nh: power of two >= No */
  int n_layers;     /* 1..16 */
  const wcgh_layer* layers;
  wcgh_plan plan;
  int method;       /* WCGH_METHOD_* */
  int phase_mode;   /* WCGH_PHASE_* */
  int row0, rows;   /* row band; rows = plane_size for a whole hologram */
  int obj_dtype;    /* WCGH_U8 / WCGH_F32 / WCGH_F64 */
  double obj_scale; /* amplitude = sample * obj_scale */
  int sal_dtype;    /* WCGH_U8 / WCGH_F32 / WCGH_F64 */
} wcgh_desc;

/* Statistics of the last wcgh_job_run. */
typedef struct {
  uint64_t ops[WCGH_OP_LEVELS]; /* summed over layers */
  int64_t n_points;             /* direct: compacted nonzero A_eff points;
                                   LUT: nonzero-weight gated cells, all stages */
  double updates;               /* algorithmic updates of the synthesis kernel */
  float ms_analysis;            /* device time: DWT + gate + compaction */
  float ms_synthesis;           /* device time: accumulation kernel(s) */
  float ms_reduce;              /* device time: chunk reduction */
  float ms_total;               /* device time of the whole run */
  int synth_launches;           /* kernel launches of the synthesis step */
  int total_launches;           /* all kernel launches of the run */
} wcgh_stats;

typedef struct wcgh_ctx wcgh_ctx;
typedef struct wcgh_job wcgh_job;

/* ---- context ----------------------------------------------------------- */
int wcgh_abi_version(void);
/* Creates a context on CUDA device `device`. */
int wcgh_create(int device, wcgh_ctx** out);
void wcgh_destroy(wcgh_ctx* ctx);
/* Last error message of this thread (ctx may be NULL). */
const char* wcgh_last_error(const wcgh_ctx* ctx);
/* Runs all work of this context on `stream` (a cudaStream_t; NULL = the
 * context's own stream). */
int wcgh_set_stream(wcgh_ctx* ctx, void* stream);
/* Number of SMs and the device name, for reporting. */
int wcgh_device_info(wcgh_ctx* ctx, int* sm_count, char* name, int name_len);

/* ---- stage entry points (host buffers; parity tests, C++/Python mirrors) --
 *
 * Replaces haar_analyze (haar.hpp:36, haar.cpp:52-74). pyramid layout: approx
 * (n>>levels)^2, then per level l = 0..levels-1 (finest first) h, v, d each
 * (n>>(l+1))^2, as doubles. Arithmetic is fp64 in the reference's order, so
 * the bands are bit-identical to the reference for any input. */
int wcgh_haar_analyze(wcgh_ctx* ctx, const void* image, int dtype, double scale, int n,
                      int levels, double* pyramid);

/* Replaces expand_residual (haar.hpp:46-47, haar.cpp:88-96): m x m -> (2m)^2. */
int wcgh_expand_residual(wcgh_ctx* ctx, const double* h, const double* v, const double* d,
                         int m, double* out);

/* Replaces quantize_saliency (saliency.hpp:78, saliency.cpp:41-61): half,
 * quarter, eighth block-max maps (doubles); validates [0,1] and n % 8. */
int wcgh_quantize_saliency(wcgh_ctx* ctx, const void* saliency, int dtype, int n,
                           double* sal_pyr);

/* Analysis half of synthesize_progressive (synthesis.cpp:216-251) for one
 * layer of n x n: gates (strict '>', synthesis.cpp:107-119), operator counts
 * (synthesis.cpp:68), gated cell lists (row-major ascending y*m+x), the
 * effective amplitude A_eff and its order-preserving compaction. Every output
 * may be NULL. cells: concatenated ll, l, full lists (capacity (n/4)^2 +
 * (n/2)^2 + n^2); cell_counts[3]. points: capacity n^2, coordinates offset by
 * `offset`. */
typedef struct {
  double* pyramid;      /* 3-level layout of wcgh_haar_analyze */
  double* sal_pyr;      /* half, quarter, eighth */
  uint8_t* masks;       /* mask_ll (n/4)^2, mask_l (n/2)^2, mask_full n^2 */
  float* a_eff;         /* n^2 */
  uint32_t* cells;      /* gated cells per stage */
  int64_t cell_counts[3];
  wcgh_point* points;   /* compacted A_eff */
  int64_t n_points;
  uint64_t ops[WCGH_OP_LEVELS];
} wcgh_analysis;
int wcgh_analyze(wcgh_ctx* ctx, const void* object, int obj_dtype, double obj_scale,
                 const void* saliency, int sal_dtype, int n, const wcgh_plan* plan,
                 int offset, int layer, wcgh_analysis* out);

/* Direct Eq.(1) accumulation of a host point list over hologram rows
 * [row0, row0+rows) of an nh-wide plane: out = rows x nh complex64.
 * Points must be sorted by layer. The exact sum the reference's
 * pointwise_sum forms (tests/support/oracles.cpp:12-36), per layer z. */
int wcgh_synth_points(wcgh_ctx* ctx, const wcgh_point* points, int64_t n_points,
                      const wcgh_layer* layers, int n_layers, int nh, int row0, int rows,
                      int phase_mode, float* out);

/* Replaces build_block_lut (fringe_lut.hpp:126, fringe_lut.cpp:53-93) on the
 * GPU: the (2n-1)^2 support of a B x B block, summed in fp64 and stored as
 * complex64 (the CGHL payload, fringe_lut.cpp:107-113). */
int wcgh_build_block_lut(wcgh_ctx* ctx, const wcgh_layer* scene, int n, int block, float* out);

/* Replaces apply_block (synthesis.hpp:68-69, synthesis.cpp:149-160) for a
 * batch: plane (n x n complex64, in/out) += sum_i w_i * crop(S_B at cell_i),
 * with S_B built on the device for `scene`. cells are y*m+x on the m = n/B
 * grid; zero weights add nothing but count (ops_out += n_cells). */
int wcgh_apply_blocks(wcgh_ctx* ctx, const wcgh_layer* scene, int n, int block,
                      const uint32_t* cells, const float* weights, int64_t n_cells,
                      float* plane, uint64_t* ops_out);

/* Replaces refine (synthesis.hpp:79-82, synthesis.cpp:90-123 + 171-178):
 * expands (h, v, d) (m x m each) into the 2m x 2m residual, gates it with
 * saliency_finer (2m x 2m, doubles) by the strict '>' against `threshold`,
 * and adds the block-B LUT contribution of every gated cell to `plane`
 * (n x n complex64, in/out), where B = n / (2m). mask_out (2m x 2m bytes)
 * may be NULL; ops_out += number of gated cells. */
int wcgh_refine(wcgh_ctx* ctx, const wcgh_layer* scene, int n, const double* h, const double* v,
                const double* d, int m, const double* saliency_finer, double threshold,
                float* plane, uint8_t* mask_out, uint64_t* ops_out);

/* The reference's small helpers, on the device (no host arithmetic in the
 * drop-in): haar_synthesize (haar.hpp:43, haar.cpp:76-86; the pyramid in
 * wcgh_haar_analyze's flat layout, out n x n, bit-identical),
 * upsample_replicate (haar.hpp:51, haar.cpp:98-109; out (w*f) x (h*f),
 * bit-identical) and point_fringe (fringe_lut.hpp:15, fringe_lut.cpp:27-32;
 * out2 = (re, im) in fp64, the device sin/cos within 2 ulp of the host's). */
int wcgh_haar_synthesize(wcgh_ctx* ctx, const double* pyramid, int n, int levels, double* out);
int wcgh_upsample_replicate(wcgh_ctx* ctx, const double* coarse, int width, int height, int factor,
                            double* out);
int wcgh_point_fringe(wcgh_ctx* ctx, const wcgh_layer* scene, int dx, int dy, double* out2);

/* ---- device-resident LUTs and planes (the caller's FringeLut / ComplexField)
 * The reference's apply_block / synthesize_base / refine read the CALLER's
 * FringeLut samples (lut.support(), synthesis.cpp:18-42,149-178), which may
 * come from the f32 CGHL cache (pipeline.cpp:174-177) or be built by the
 * caller. A wcgh_lut holds such a support on the device (uploaded once, in a
 * guarded allocation the superposition kernel reads without bounds checks);
 * a wcgh_plane is a device-resident n x n complex64 hologram that stage
 * calls accumulate into with no host round trip. */
typedef struct wcgh_lut wcgh_lut;
typedef struct wcgh_plane wcgh_plane;
/* FringeLut(scene, block, support) (fringe_lut.cpp:34-51) on the device:
 * `samples` = the (2n-1)^2 support, row-major, interleaved (re, im) as
 * complex64 (dtype WCGH_F32, the CGHL payload) or complex128 (WCGH_F64, the
 * reference's std::complex<double>; rounded once to complex64), or NULL to
 * build it on the device (build_block_lut, fringe_lut.cpp:53-93). Non-finite
 * samples are a ValidationError. */
int wcgh_lut_create(wcgh_ctx* ctx, const wcgh_layer* scene, int n, int block, const void* samples,
                    int dtype, wcgh_lut** out);
void wcgh_lut_destroy(wcgh_lut* lut);
/* D2H of the device support (complex64 (2n-1)^2). */
int wcgh_lut_download(wcgh_lut* lut, float* out);
/* An n x n complex64 plane on the context's device, zeroed. */
int wcgh_plane_create(wcgh_ctx* ctx, int n, wcgh_plane** out);
void wcgh_plane_destroy(wcgh_plane* plane);
int wcgh_plane_zero(wcgh_plane* plane);
/* H2D / D2H of the whole plane, complex64 (WCGH_F32) or complex128 (WCGH_F64). */
int wcgh_plane_upload(wcgh_plane* plane, const void* host, int dtype);
int wcgh_plane_download(wcgh_plane* plane, void* host, int dtype);
/* Device pointer of the plane (n*n complex64), e.g. for a zero-copy view. */
void* wcgh_plane_dev(wcgh_plane* plane);
/* apply_block (synthesis.cpp:149-160) batched, with the caller's LUT:
 * plane += sum_i (w_re[i] + i w_im[i]) * crop(S_B at cell_i); cells y*m+x
 * on the m = n/B grid (out of range: ValidationError); w_im may be NULL;
 * ops_out += n_cells (zero weights count, synthesis.cpp:20). */
int wcgh_lut_apply_blocks(wcgh_lut* lut, const uint32_t* cells, const float* w_re,
                          const float* w_im, int64_t n_cells, wcgh_plane* plane,
                          uint64_t* ops_out);
/* refine (synthesis.cpp:171-178 + 90-123) with the caller's LUT: residual of
 * (h, v, d) (m x m doubles), strict '>' gate against saliency_finer (2m x 2m
 * doubles), plane += the gated cells' superposition; B = n / (2m) must be
 * the LUT's block size. mask_out (2m x 2m) may be NULL. */
int wcgh_lut_refine(wcgh_lut* lut, const double* h, const double* v, const double* d, int m,
                    const double* saliency_finer, double threshold, wcgh_plane* plane,
                    uint8_t* mask_out, uint64_t* ops_out);

/* ---- jobs: resident inputs, device-side hologram ------------------------ */
int wcgh_job_create(wcgh_ctx* ctx, const wcgh_desc* desc, wcgh_job** out);
void wcgh_job_destroy(wcgh_job* job);
/* H2D of n_layers x No^2 object and saliency samples (layer-major). */
int wcgh_job_upload(wcgh_job* job, const void* object, const void* saliency);
/* Same from device pointers (device-to-device copy). */
int wcgh_job_upload_dev(wcgh_job* job, const void* object_dev, const void* saliency_dev);
/* Analysis + compaction + synthesis of the row band into the job's device
 * plane. Returns after the work is enqueued AND complete (synchronous). */
int wcgh_job_run(wcgh_job* job);
/* D2H of the row band: rows x Nh complex64. */
/* Front end only (K1/K2: DWT, saliency, gates, A_eff, compaction or run
 * lists): fills the stats' ops, n_points (compacted points, or nonzero gated
 * cells for the LUT method) and ms_analysis; no synthesis. */
int wcgh_job_analyze(wcgh_job* job);
int wcgh_job_download(wcgh_job* job, float* out);
/* Fused row-tile gather: register the full-plane buffers
 * (plane_size x plane_size complex64, device pointers valid in this process —
 * the other ranks' planes mapped over NVLink with CUDA IPC, and this rank's
 * own) that every later run also writes its band into, at rows
 * [row0, row0 + rows), from the kernel that produces the band's final values
 * (no collective call). n_planes = 0 clears the list; at most 16. */
int wcgh_job_set_peer_planes(wcgh_job* job, void* const* planes_dev, int n_planes);
/* CUDA-IPC helpers for those planes: allocate a zeroed full plane on
 * `device` and export its 64-byte IPC handle; map a peer's plane from its
 * handle (lazy NVLink peer access); unmap; free. */
int wcgh_ipc_alloc_plane(int device, int n, void** dev_ptr, unsigned char* handle64);
int wcgh_ipc_open_plane(int device, const unsigned char* handle64, void** dev_ptr);
int wcgh_ipc_close_plane(void* dev_ptr);
int wcgh_ipc_free_plane(void* dev_ptr);
/* A_eff of the last run or analyze (n_layers x No^2 fp32, row-major). */
int wcgh_job_download_a_eff(wcgh_job* job, float* out);
/* Compacted point list of the last direct-method run or analyze (row-major
 * ascending per layer): *n_out = count; copies it when out != NULL and
 * capacity >= count. */
int wcgh_job_download_points(wcgh_job* job, wcgh_point* out, int64_t capacity, int64_t* n_out);
/* Complex-object jobs (obj_dtype WCGH_C128): the imaginary parts matching
 * wcgh_job_download_a_eff / wcgh_job_download_points (whose values are the
 * real parts; a point is kept when either part is nonzero). */
int wcgh_job_download_a_eff_im(wcgh_job* job, float* out);
int wcgh_job_download_points_im(wcgh_job* job, float* out, int64_t capacity);
/* Stage snapshots of the last run: base_LLL, after_LL, after_L, after_full
 * (synthesis.hpp:43-54), each rows x Nh complex64. The LUT method keeps its
 * stage planes from the run; the direct and FFT methods synthesise the four
 * per-stage amplitude deltas on demand (first call after a run). */
int wcgh_job_download_stages(wcgh_job* job, float* out4);
/* Device pointer of the row band (rows x Nh complex64), valid until destroy. */
void* wcgh_job_plane_dev(wcgh_job* job);
int wcgh_job_stats(const wcgh_job* job, wcgh_stats* out);
/* Which K3 form the last direct-method run launched (tuning and the bench's
 * roofline; no reference counterpart): form 0 per-pixel, 1 recurrence,
 * 2 chirp-factored recurrence, 3 fp64 phase, -1 before the first run (or an
 * empty point list); hold = steps a run multiplier is held for (1, 2 or 4;
 * form 2 only). */
int wcgh_job_direct_form(const wcgh_job* job, int* form, int* hold);

/* Replaces random_phase_field (synthesis.hpp:101-104, synthesis.cpp:288-296):
 * out[i] = polar(amplitude[i], U[0, 2pi)) with std::mt19937_64(seed) drawn
 * in sample order — the reference's own sequential host RNG (libstdc++), so
 * the complex object is bit-identical. HOST function: no device work.
 * out: width x height interleaved complex128, the WCGH_C128 object layout. */
int wcgh_random_phase_field(const double* amplitude, int width, int height, uint64_t seed,
                            double* out);

/* ---- CGH1 hologram files (image_io.cpp:220-278) --------------
 * "CGH1", u16 version = 1, u32 N, f64 wavelength, f64 pitch, f64 z (little
 * endian, 34 bytes), then N^2 interleaved f32 (re, im), row-major — exactly
 * the device complex64 layout. Host I/O; no device needed. File errors return
 * WCGH_ERUNTIME (IoError); a bad scene or non-finite payload WCGH_EVALIDATION. */
int wcgh_write_cgh1(const char* path, const float* plane, int n, const wcgh_layer* scene);
/* Reads a CGH1 file: header into *n_out / *scene_out (either may be NULL),
 * payload into `plane` if it is non-NULL and capacity >= N^2 complex64. */
int wcgh_read_cgh1(const char* path, float* plane, int64_t capacity, int* n_out,
                   wcgh_layer* scene_out);
/* Writes the last run's full plane (stage < 0) or a stage snapshot
 * (0..3 = base_LLL, after_LL, after_L, after_full) of a whole-plane job
 * (row0 = 0, rows = plane_size) as CGH1, scene = layer 0. */
int wcgh_job_write_cgh1(wcgh_job* job, const char* path, int stage);

/* ---- Reconstruction and metrics -------------------
 * fp64 on the device like the reference; n must be a power of two. Complex
 * arrays are interleaved (re, im); `dtype` selects complex64 input
 * (WCGH_F32, e.g. a synthesised hologram) or complex128 (WCGH_F64). The
 * scene's z is ignored where an explicit z_signed is taken. */
/* fft_2d (fft.cpp:45-68): forward or inverse (scaled by 1/n^2) 2-D DFT. */
int wcgh_fft_2d(wcgh_ctx* ctx, const double* field, int n, int inverse, double* out);
/* build_kernel (angular_spectrum.cpp:11-33): transfer function, DC first,
 * evanescent samples zero; z_signed != 0. */
int wcgh_propagation_kernel(wcgh_ctx* ctx, const wcgh_layer* scene, int n, double z_signed,
                            double* out);
/* propagate (angular_spectrum.cpp:35-45): IDFT(DFT(field) * transfer). */
int wcgh_propagate(wcgh_ctx* ctx, const void* field, int dtype, int n, const wcgh_layer* scene,
                   double z_signed, double* out);
/* reconstruct (angular_spectrum.cpp:47-61): back-propagate by -scene.z and
 * return |.| (intensity = 0) or |.|^2, n x n doubles. */
int wcgh_reconstruct(wcgh_ctx* ctx, const void* hologram, int dtype, int n,
                     const wcgh_layer* scene, int intensity, double* out);
/* Same on the last run's plane of a whole-plane job, without a host copy. */
int wcgh_job_reconstruct(wcgh_job* job, const wcgh_layer* scene, int intensity, double* out);
/* ssim (metrics.cpp:49-85): mean box-window SSIM of two width x height
 * images; window in [1, min(width, height)], dynamic_range > 0. */
int wcgh_ssim(wcgh_ctx* ctx, const double* a, const double* b, int width, int height, int window,
              double k1, double k2, double dynamic_range, double* score);

/* ---- CGHL LUT cache files (fringe_lut.cpp:95-166, lut_cache_store/load) ---
 * "CGHL", u16 version = 1, u16 block size, u32 N, f64 wavelength, f64 pitch,
 * f64 z (native little endian, 36 bytes), then (2N-1)^2 interleaved f32
 * (re, im) — the layout wcgh_build_block_lut returns and the jobs keep on
 * the device. File errors return WCGH_ERUNTIME (IoError class). */
int wcgh_write_cghl(const char* path, const float* lut, int n, int block, const wcgh_layer* scene);
/* Header into *n_out / *block_out / *scene_out (any may be NULL); payload into
 * `lut` if non-NULL and capacity >= (2N-1)^2 complex64. Scene / block checks
 * against an expected LUT (StaleCacheError) are the caller's. */
int wcgh_read_cghl(const char* path, float* lut, int64_t capacity, int* n_out, int* block_out,
                   wcgh_layer* scene_out);
/* LUT-method job: replace the block-`block` LUT of `layer` (built at job
 * creation) with caller data, (2N-1)^2 complex64 — e.g. a reference CGHL
 * cache, so the job superposes exactly the reference's LUT samples. */
int wcgh_job_load_lut(wcgh_job* job, int layer, int block, const float* lut);
/* The same from a device LUT (wcgh_lut_create; device-to-device): the LUT
 * job of synthesize_progressive(..., const LutSet& luts, ...) superposes the
 * caller's LutSet (synthesis.cpp:180-253 reads luts.of(B)). The LUT's plane
 * size must equal the job's; its scene must equal the layer's (the
 * reference's "LUTs built for a different scene" check). */
int wcgh_job_use_lut(wcgh_job* job, int layer, const wcgh_lut* lut);

/* One-shot: job create + upload + run + download + destroy. The entry the
 * C++ synthesize_progressive mirror calls (synthesis.hpp:88-91). */
int wcgh_synthesize(wcgh_ctx* ctx, const wcgh_desc* desc, const void* object,
                    const void* saliency, float* out, wcgh_stats* stats);

/* Single-process multi-GPU one-shot: the whole plane
 * (desc->row0 = 0, rows = plane_size) split into contiguous row bands, one per
 * listed device (equal splits, remainder to the first; a device may repeat),
 * each band synthesised on its device by its own host thread and written
 * straight into its rows of `out` — the band results are bitwise those of a
 * single-device run. Processes that own one GPU each use the job API per band
 * and an NCCL all-gather instead (paper_2211_09938_b200/tiles.py). */
int wcgh_synthesize_multi(int n_devices, const int* devices, const wcgh_desc* desc,
                          const void* object, const void* saliency, float* out,
                          wcgh_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* WCGH_H */
