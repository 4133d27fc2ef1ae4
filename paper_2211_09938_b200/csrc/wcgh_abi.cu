// C ABI of the B200-native hot path (include/wcgh.h): contexts, jobs and the
// stage entry points the host mirrors call. Validation mirrors the
// reference's ValidationError sites; CUDA failures map to WCGH_ERUNTIME.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "wcgh_internal.cuh"

using namespace wcgh;

namespace {

thread_local std::string t_last_error;

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

size_t dtype_size(int dt) {
  switch (dt) {
    case WCGH_U8: return 1;
    case WCGH_F32: return 4;
    case WCGH_F64: return 8;
    default: throw ValidationError("dtype must be WCGH_U8, WCGH_F32 or WCGH_F64");
  }
}

void validate_plan(const wcgh_plan& p) {
  // RefinementPlan::validate (synthesis.cpp:127-131)
  require(0.0 <= p.t_ll && p.t_ll <= p.t_l && p.t_l <= p.t_full && p.t_full <= 1.0,
          "thresholds: need 0 <= t_ll <= t_l <= t_full <= 1");
}

void validate_layer(const wcgh_layer& L) {
  // SceneParams (field.cpp:71-80)
  require(L.wavelength > 0.0, "scene: wavelength must be positive");
  require(L.pitch > 0.0, "scene: pitch must be positive");
  require(L.z > 0.0, "scene: z must be positive");
}

}  // namespace

struct wcgh_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  std::string name;
  // scratch for the stage entry points
  DevBuf b_in, b_in2, b_out, b_out2, b_misc, b_pts, b_plane, b_lut, b_lut_scratch, lut_partial;
  DirectScratch direct;
  StageCells cells;
  ReconPlan recon;  // reconstruction / FFT entry points
  DevBuf b_ssim, b_scan;
  std::mutex mu;
};

struct wcgh_job {
  wcgh_ctx* ctx = nullptr;
  wcgh_desc desc{};
  std::vector<wcgh_layer> layers;
  int off = 0;
  size_t in_elems = 0;  // per layer No^2
  DevBuf obj, sal, a_eff, seg_counts, seg_offsets, scan_scratch, ops, err, points, plane;
  // LUT method
  DevBuf w_stage, stage_planes, lut_scratch, lut_partial;
  std::vector<std::unique_ptr<StageCells>> cells;  // [layer * 4 + stage]
  std::vector<std::unique_ptr<DevBuf>> luts;  // [layer * 4 + stage], guarded allocations
  std::vector<float2*> lut_base;              // support element (0, 0) in each
  DirectScratch direct;
  DirectTiming timing;
  FftPlan fft;  // FFT method
  // pinned host staging
  int64_t* h_offsets = nullptr;       // n_layers + 1
  unsigned long long* h_ops = nullptr;  // n_layers * 5
  int* h_err = nullptr;
  int* h_tot = nullptr;  // LUT: (runs, dense steps, nnz) per stage
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  wcgh_stats stats{};
  bool uploaded = false;
  bool ran = false;           // a run finished since the last upload
  bool stages_ready = false;  // stage_planes hold the per-stage planes of the last run
  DevBuf snap_img, snap_points;  // direct/FFT snapshots (computed on demand)
  PeerPlanes peers;              // fused row-tile gather targets (wcgh_job_set_peer_planes)
  ~wcgh_job() {
    if (h_tot) cudaFreeHost(h_tot);
    if (h_offsets) cudaFreeHost(h_offsets);
    if (h_ops) cudaFreeHost(h_ops);
    if (h_err) cudaFreeHost(h_err);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

template <typename F>
int guard(const wcgh_ctx* ctx, F&& f) {
  (void)ctx;
  try {
    f();
    return WCGH_OK;
  } catch (const ValidationError& e) {
    t_last_error = e.what();
    return WCGH_EVALIDATION;
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return WCGH_ERUNTIME;
  }
}

void use_device(wcgh_ctx* ctx) { WCGH_CUDA(cudaSetDevice(ctx->device)); }

void sync(cudaStream_t s) { WCGH_CUDA(cudaStreamSynchronize(s)); }

void check_analysis_flags(int flags) {
  if (flags & kErrObjectNonFinite) throw ValidationError("object: non-finite sample");
  if (flags & kErrSaliencyRange) throw ValidationError("quantize_saliency: values must lie in [0,1]");
}

void job_validate(const wcgh_desc& d) {
  require(d.n_layers >= 1 && d.n_layers <= kMaxLayers, "job: n_layers must be 1..16");
  require(d.layers != nullptr, "job: layers must not be NULL");
  for (int l = 0; l < d.n_layers; ++l) validate_layer(d.layers[l]);
  validate_plan(d.plan);
  require(d.object_size >= 8 && d.object_size % 8 == 0,
          "synthesize_progressive: object side must be a multiple of 8 and >= 8");
  require(is_pow2(d.plane_size), "scene: plane_size must be a power of two, got " +
                                     std::to_string(d.plane_size));
  require(d.plane_size <= 16384, "scene: plane_size above 16384 is not supported");
  require(d.object_size <= d.plane_size, "synthesize_progressive: object larger than the plane");
  // compaction offsets and run lists are int32
  require(size_t(d.n_layers) * size_t(d.object_size) * size_t(d.object_size) < (size_t(1) << 31),
          "job: n_layers x object_size^2 must stay below 2^31 samples");
  require((d.plane_size - d.object_size) % 16 == 0,
          "synthesize_progressive: (plane_size - object_size)/2 must be a multiple of 8");
  require(d.row0 >= 0 && d.rows >= 1 && d.row0 + d.rows <= d.plane_size,
          "job: row band outside the plane");
  require(d.method == WCGH_METHOD_DIRECT || d.method == WCGH_METHOD_LUT ||
              d.method == WCGH_METHOD_FFT,
          "job: unknown method");
  require(d.phase_mode == WCGH_PHASE_FIXED || d.phase_mode == WCGH_PHASE_FP64,
          "job: unknown phase mode");
  dtype_size(d.obj_dtype);
  dtype_size(d.sal_dtype);
  if (d.method == WCGH_METHOD_LUT) {
    for (int l = 1; l < d.n_layers; ++l)
      require(d.layers[l].wavelength == d.layers[0].wavelength && d.layers[l].pitch == d.layers[0].pitch,
              "job (LUT): layers must share wavelength and pitch");
  }
}

}  // namespace

extern "C" {

int wcgh_abi_version(void) { return WCGH_ABI_VERSION; }

const char* wcgh_last_error(const wcgh_ctx*) { return t_last_error.c_str(); }

int wcgh_create(int device, wcgh_ctx** out) {
  return guard(nullptr, [&] {
    require(out != nullptr, "wcgh_create: out must not be NULL");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      throw RuntimeError(std::string("wcgh_create: no CUDA device available (") +
                         cudaGetErrorString(e) + "); the hot path has no CPU fallback");
    require(device >= 0 && device < count, "wcgh_create: device index out of range");
    auto ctx = std::make_unique<wcgh_ctx>();
    ctx->device = device;
    WCGH_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    WCGH_CUDA(cudaGetDeviceProperties(&prop, device));
    ctx->sm_count = prop.multiProcessorCount;
    ctx->name = prop.name;
    WCGH_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    *out = ctx.release();
  });
}

void wcgh_destroy(wcgh_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->own_stream) {
    cudaStreamSynchronize(ctx->own_stream);
    cudaStreamDestroy(ctx->own_stream);
  }
  delete ctx;
}

int wcgh_set_stream(wcgh_ctx* ctx, void* stream) {
  return guard(ctx, [&] {
    require(ctx != nullptr, "wcgh_set_stream: NULL context");
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  });
}

int wcgh_device_info(wcgh_ctx* ctx, int* sm_count, char* name, int name_len) {
  return guard(ctx, [&] {
    require(ctx != nullptr, "wcgh_device_info: NULL context");
    if (sm_count) *sm_count = ctx->sm_count;
    if (name && name_len > 0) {
      std::strncpy(name, ctx->name.c_str(), size_t(name_len) - 1);
      name[name_len - 1] = 0;
    }
  });
}

// ---------------------------------------------------------------------------

int wcgh_haar_analyze(wcgh_ctx* ctx, const void* image, int dtype, double scale, int n,
                      int levels, double* pyramid) {
  return guard(ctx, [&] {
    require(ctx && image && pyramid, "haar_analyze: NULL argument");
    // haar.cpp:53-60
    require(levels >= 1, "haar_analyze: levels must be >= 1");
    require(levels <= 14 && n > 0 && n % (1 << levels) == 0,
            "haar_analyze: side " + std::to_string(n) + " not divisible by 2^" + std::to_string(levels));
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t n2 = size_t(n) * n;
    if (levels != 3) {
      // generic per-level path (the fused 3-level K1 serves the pipeline)
      size_t plen = 0, side = size_t(n);
      for (int l = 0; l < levels; ++l) { side /= 2; plen += 3 * side * side; }
      plen += side * side;
      char* in = static_cast<char*>(ctx->b_in.reserve(n2 * dtype_size(dtype)));
      WCGH_CUDA(cudaMemcpyAsync(in, image, n2 * dtype_size(dtype), cudaMemcpyHostToDevice, s));
      double* o = static_cast<double*>(ctx->b_out.reserve((plen + 2 * n2) * 8));
      int* err = static_cast<int*>(ctx->b_misc.reserve(64));
      WCGH_CUDA(cudaMemsetAsync(err, 0, 64, s));
      launch_haar_levels(in, dtype, scale, n, levels, o, o + plen, err, s);
      int flags = 0;
      WCGH_CUDA(cudaMemcpyAsync(pyramid, o, plen * 8, cudaMemcpyDeviceToHost, s));
      WCGH_CUDA(cudaMemcpyAsync(&flags, err, sizeof(int), cudaMemcpyDeviceToHost, s));
      sync(s);
      if (flags & kErrObjectNonFinite) throw ValidationError("haar_analyze: non-finite sample");
      return;
    }
    char* in = static_cast<char*>(ctx->b_in.reserve(n2 * dtype_size(dtype) + n2));
    uint8_t* zero_sal = reinterpret_cast<uint8_t*>(in + n2 * dtype_size(dtype));
    WCGH_CUDA(cudaMemcpyAsync(in, image, n2 * dtype_size(dtype), cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemsetAsync(zero_sal, 0, n2, s));
    char* o = static_cast<char*>(ctx->b_out.reserve(pyr_len(n) * 8 + n2 * 4 + 64));
    AnalysisOut ao;
    ao.pyramid = reinterpret_cast<double*>(o);
    ao.a_eff = reinterpret_cast<float*>(o + pyr_len(n) * 8);
    unsigned long long* ops = static_cast<unsigned long long*>(ctx->b_misc.reserve(64));
    ao.ops = ops;
    ao.err = reinterpret_cast<int*>(ops + WCGH_OP_LEVELS);
    WCGH_CUDA(cudaMemsetAsync(ops, 0, 64, s));
    wcgh_plan plan{0.5, 0.7, 0.9, 1, 1, 1};
    launch_analysis(in, dtype, scale, zero_sal, WCGH_U8, n, 1, plan, ao, s);
    int flags = 0;
    WCGH_CUDA(cudaMemcpyAsync(pyramid, ao.pyramid, pyr_len(n) * 8, cudaMemcpyDeviceToHost, s));
    WCGH_CUDA(cudaMemcpyAsync(&flags, ao.err, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync(s);
    if (flags & kErrObjectNonFinite) throw ValidationError("haar_analyze: non-finite sample");
  });
}

int wcgh_expand_residual(wcgh_ctx* ctx, const double* h, const double* v, const double* d, int m,
                         double* out) {
  return guard(ctx, [&] {
    require(ctx && h && v && d && out, "expand_residual: NULL argument");
    require(m >= 1, "expand_residual: detail subbands must be non-empty");
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t m2 = size_t(m) * m;
    double* in = static_cast<double*>(ctx->b_in.reserve(3 * m2 * 8));
    double* o = static_cast<double*>(ctx->b_out.reserve(4 * m2 * 8));
    WCGH_CUDA(cudaMemcpyAsync(in, h, m2 * 8, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(in + m2, v, m2 * 8, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(in + 2 * m2, d, m2 * 8, cudaMemcpyHostToDevice, s));
    launch_expand_residual(in, in + m2, in + 2 * m2, m, o, s);
    WCGH_CUDA(cudaMemcpyAsync(out, o, 4 * m2 * 8, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_quantize_saliency(wcgh_ctx* ctx, const void* saliency, int dtype, int n, double* sal_pyr) {
  return guard(ctx, [&] {
    require(ctx && saliency && sal_pyr, "quantize_saliency: NULL argument");
    // saliency.cpp:42-48
    require(n % 8 == 0 && n > 0,
            "quantize_saliency: side must be divisible by 8, got " + std::to_string(n));
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t n2 = size_t(n) * n;
    char* in = static_cast<char*>(ctx->b_in.reserve(n2 * dtype_size(dtype) + n2));
    uint8_t* zero_obj = reinterpret_cast<uint8_t*>(in + n2 * dtype_size(dtype));
    WCGH_CUDA(cudaMemcpyAsync(in, saliency, n2 * dtype_size(dtype), cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemsetAsync(zero_obj, 0, n2, s));
    char* o = static_cast<char*>(ctx->b_out.reserve(salpyr_len(n) * 8 + n2 * 4 + 64));
    AnalysisOut ao;
    ao.sal_pyr = reinterpret_cast<double*>(o);
    ao.a_eff = reinterpret_cast<float*>(o + salpyr_len(n) * 8);
    unsigned long long* ops = static_cast<unsigned long long*>(ctx->b_misc.reserve(64));
    ao.ops = ops;
    ao.err = reinterpret_cast<int*>(ops + WCGH_OP_LEVELS);
    WCGH_CUDA(cudaMemsetAsync(ops, 0, 64, s));
    wcgh_plan plan{0.5, 0.7, 0.9, 1, 1, 1};
    launch_analysis(zero_obj, WCGH_U8, 1.0, in, dtype, n, 1, plan, ao, s);
    int flags = 0;
    WCGH_CUDA(cudaMemcpyAsync(sal_pyr, ao.sal_pyr, salpyr_len(n) * 8, cudaMemcpyDeviceToHost, s));
    WCGH_CUDA(cudaMemcpyAsync(&flags, ao.err, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync(s);
    check_analysis_flags(flags & kErrSaliencyRange);
  });
}

int wcgh_analyze(wcgh_ctx* ctx, const void* object, int obj_dtype, double obj_scale,
                 const void* saliency, int sal_dtype, int n, const wcgh_plan* plan, int offset,
                 int layer, wcgh_analysis* out) {
  return guard(ctx, [&] {
    require(ctx && object && saliency && plan && out, "analyze: NULL argument");
    validate_plan(*plan);
    require(n >= 8 && n % 8 == 0, "analyze: side must be a positive multiple of 8");
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t n2 = size_t(n) * n;
    const size_t os = dtype_size(obj_dtype), ss = dtype_size(sal_dtype);
    char* in = static_cast<char*>(ctx->b_in.reserve(n2 * (os + ss)));
    WCGH_CUDA(cudaMemcpyAsync(in, object, n2 * os, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(in + n2 * os, saliency, n2 * ss, cudaMemcpyHostToDevice, s));
    const int segs = seg_per_row(n);
    const size_t nseg = size_t(n) * segs;
    // device outputs
    size_t bytes = pyr_len(n) * 8 + salpyr_len(n) * 8 + masks_len(n) + n2 * 4 + 2 * (nseg + 1) * 4 + 256;
    char* o = static_cast<char*>(ctx->b_out.reserve(bytes));
    AnalysisOut ao;
    char* cur = o;
    ao.pyramid = reinterpret_cast<double*>(cur); cur += pyr_len(n) * 8;
    ao.sal_pyr = reinterpret_cast<double*>(cur); cur += salpyr_len(n) * 8;
    ao.a_eff = reinterpret_cast<float*>(cur); cur += n2 * 4;
    ao.seg_counts = reinterpret_cast<int*>(cur); cur += (nseg + 1) * 4;
    int* seg_off = reinterpret_cast<int*>(cur); cur += (nseg + 1) * 4;
    ao.masks = reinterpret_cast<uint8_t*>(cur);
    unsigned long long* ops = static_cast<unsigned long long*>(ctx->b_misc.reserve(64));
    ao.ops = ops;
    ao.err = reinterpret_cast<int*>(ops + WCGH_OP_LEVELS);
    WCGH_CUDA(cudaMemsetAsync(ops, 0, 64, s));
    launch_analysis(in, obj_dtype, obj_scale, in + n2 * os, sal_dtype, n, 1, *plan, ao, s);
    launch_scan(ao.seg_counts, seg_off, int(nseg), s, &ctx->b_scan);
    unsigned long long h_ops[WCGH_OP_LEVELS];
    int flags = 0, total = 0;
    WCGH_CUDA(cudaMemcpyAsync(h_ops, ops, sizeof(h_ops), cudaMemcpyDeviceToHost, s));
    WCGH_CUDA(cudaMemcpyAsync(&flags, ao.err, sizeof(int), cudaMemcpyDeviceToHost, s));
    WCGH_CUDA(cudaMemcpyAsync(&total, seg_off + nseg, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync(s);
    check_analysis_flags(flags);
    for (int i = 0; i < WCGH_OP_LEVELS; ++i) out->ops[i] = h_ops[i];
    out->n_points = total;
    if (out->points) {
      wcgh_point* pts = static_cast<wcgh_point*>(ctx->b_pts.reserve(sizeof(wcgh_point) * (size_t(total) + 1)));
      launch_compact_points(ao.a_eff, seg_off, n, 1, offset, layer, pts, s);
      WCGH_CUDA(cudaMemcpyAsync(out->points, pts, sizeof(wcgh_point) * size_t(total), cudaMemcpyDeviceToHost, s));
    }
    if (out->pyramid) WCGH_CUDA(cudaMemcpyAsync(out->pyramid, ao.pyramid, pyr_len(n) * 8, cudaMemcpyDeviceToHost, s));
    if (out->sal_pyr) WCGH_CUDA(cudaMemcpyAsync(out->sal_pyr, ao.sal_pyr, salpyr_len(n) * 8, cudaMemcpyDeviceToHost, s));
    if (out->masks) WCGH_CUDA(cudaMemcpyAsync(out->masks, ao.masks, masks_len(n), cudaMemcpyDeviceToHost, s));
    if (out->a_eff) WCGH_CUDA(cudaMemcpyAsync(out->a_eff, ao.a_eff, n2 * 4, cudaMemcpyDeviceToHost, s));
    if (out->cells) {
      // gated cell lists of the three refinement stages (synthesis.cpp:111-117)
      const int ms[3] = {n / 4, n / 2, n};
      const size_t mofs[3] = {0, size_t(n / 4) * (n / 4), size_t(n / 4) * (n / 4) + size_t(n / 2) * (n / 2)};
      size_t cell_base = 0;
      for (int st = 0; st < 3; ++st) {
        const int m = ms[st];
        const size_t nsg = size_t(m) * seg_per_row(m);
        int* cnt = static_cast<int*>(ctx->b_misc.reserve(64 + 2 * (nsg + 1) * 4));
        cnt = reinterpret_cast<int*>(reinterpret_cast<char*>(cnt) + 64);
        int* ofs = cnt + nsg + 1;
        // b_misc was possibly reallocated: ops already copied out above
        launch_mask_counts(ao.masks + mofs[st], m, cnt, s);
        launch_scan(cnt, ofs, int(nsg), s, &ctx->b_scan);
        int c = 0;
        WCGH_CUDA(cudaMemcpyAsync(&c, ofs + nsg, sizeof(int), cudaMemcpyDeviceToHost, s));
        sync(s);
        out->cell_counts[st] = c;
        uint32_t* cells = static_cast<uint32_t*>(ctx->b_pts.reserve(std::max<size_t>(size_t(c) * 4, 16)));
        if (c) {
          launch_compact_mask(ao.masks + mofs[st], m, ofs, cells, s);
          WCGH_CUDA(cudaMemcpyAsync(out->cells + cell_base, cells, size_t(c) * 4, cudaMemcpyDeviceToHost, s));
        }
        sync(s);
        cell_base += size_t(c);
      }
    }
    sync(s);
  });
}

int wcgh_synth_points(wcgh_ctx* ctx, const wcgh_point* points, int64_t n_points,
                      const wcgh_layer* layers, int n_layers, int nh, int row0, int rows,
                      int phase_mode, float* out) {
  return guard(ctx, [&] {
    require(ctx && layers && out && (points || n_points == 0), "synth_points: NULL argument");
    require(n_layers >= 1 && n_layers <= kMaxLayers, "synth_points: 1..16 layers");
    for (int l = 0; l < n_layers; ++l) validate_layer(layers[l]);
    require(nh >= 1 && nh <= 16384, "synth_points: plane size must be 1..16384");
    require(row0 >= 0 && rows >= 1 && row0 + rows <= nh, "synth_points: row band outside the plane");
    std::vector<int64_t> lb(size_t(n_layers) + 1, 0);
    double max_dx = 0, max_dy = 0;
    int prev = 0;
    for (int64_t i = 0; i < n_points; ++i) {
      const wcgh_point& p = points[i];
      require(p.layer >= 0 && p.layer < n_layers && p.layer >= prev,
              "synth_points: points must be sorted by layer, layers in range");
      require(std::isfinite(p.a), "synth_points: non-finite amplitude");
      prev = p.layer;
      lb[size_t(p.layer) + 1]++;
      max_dx = std::max({max_dx, std::fabs(double(p.x)), std::fabs(double(nh - 1 - p.x))});
      max_dy = std::max({max_dy, std::fabs(double(p.y - row0)), std::fabs(double(row0 + rows - 1 - p.y))});
    }
    require(max_dx < 32768 && max_dy < 32768, "synth_points: offsets beyond 32767 pixels");
    for (int l = 0; l < n_layers; ++l) lb[size_t(l) + 1] += lb[size_t(l)];
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    wcgh_point* pts = static_cast<wcgh_point*>(ctx->b_pts.reserve(sizeof(wcgh_point) * size_t(std::max<int64_t>(n_points, 1))));
    if (n_points) WCGH_CUDA(cudaMemcpyAsync(pts, points, sizeof(wcgh_point) * size_t(n_points), cudaMemcpyHostToDevice, s));
    float2* plane = static_cast<float2*>(ctx->b_plane.reserve(sizeof(float2) * size_t(rows) * nh));
    launch_direct(pts, lb.data(), n_layers, layers, nh, row0, rows, phase_mode, max_dx, max_dy,
                  plane, ctx->direct, s, nullptr, nullptr);
    WCGH_CUDA(cudaMemcpyAsync(out, plane, sizeof(float2) * size_t(rows) * nh, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_build_block_lut(wcgh_ctx* ctx, const wcgh_layer* scene, int n, int block, float* out) {
  return guard(ctx, [&] {
    require(ctx && scene && out, "build_block_lut: NULL argument");
    validate_layer(*scene);
    require(is_pow2(n), "scene: plane_size must be a power of two, got " + std::to_string(n));
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t span = size_t(2 * n - 1);
    float2* lut = lut_in_alloc(ctx->b_lut, n, s);
    launch_build_lut(*scene, n, block, lut, ctx->b_lut_scratch, s);
    WCGH_CUDA(cudaMemcpyAsync(out, lut, sizeof(float2) * span * span, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_apply_blocks(wcgh_ctx* ctx, const wcgh_layer* scene, int n, int block,
                      const uint32_t* cells, const float* weights, int64_t n_cells, float* plane,
                      uint64_t* ops_out) {
  return guard(ctx, [&] {
    require(ctx && scene && plane && (n_cells == 0 || (cells && weights)), "apply_blocks: NULL argument");
    validate_layer(*scene);
    require(is_pow2(n), "scene: plane_size must be a power of two, got " + std::to_string(n));
    require(block == 1 || block == 2 || block == 4 || block == 8, "apply_block: unsupported block size");
    require(block <= n, "apply_block: block size exceeds plane size");
    const int m = n / block;
    // apply_block (synthesis.cpp:149-160): range check, then plane += w * crop(S_B)
    std::vector<float> dense(size_t(m) * m, 0.0f);
    for (int64_t i = 0; i < n_cells; ++i) {
      require(cells[i] < uint32_t(m) * uint32_t(m),
              "apply_block: cell " + std::to_string(cells[i]) + " out of range");
      dense[cells[i]] += weights[i];
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t n2 = size_t(n) * n;
    float2* lut = lut_in_alloc(ctx->b_lut, n, s);
    launch_build_lut(*scene, n, block, lut, ctx->b_lut_scratch, s);
    const size_t wbytes = ((dense.size() * 4 + 255) / 256) * 256;
    char* buf = static_cast<char*>(ctx->b_out.reserve(wbytes + 2 * n2 * 8));
    float* w = reinterpret_cast<float*>(buf);
    float2* contrib = reinterpret_cast<float2*>(buf + wbytes);
    WCGH_CUDA(cudaMemcpyAsync(w, dense.data(), dense.size() * 4, cudaMemcpyHostToDevice, s));
    launch_lut_dense(lut, n, block, w, m, 0, 0, n, contrib, ctx->cells, ctx->lut_partial, s, nullptr);
    std::vector<float> c(2 * n2);
    WCGH_CUDA(cudaMemcpyAsync(c.data(), contrib, 2 * n2 * 4, cudaMemcpyDeviceToHost, s));
    sync(s);
    for (size_t i = 0; i < 2 * n2; ++i) plane[i] += c[i];
    if (ops_out) *ops_out += uint64_t(n_cells);
  });
}

int wcgh_refine(wcgh_ctx* ctx, const wcgh_layer* scene, int n, const double* h, const double* v,
                const double* d, int m, const double* saliency_finer, double threshold,
                float* plane, uint8_t* mask_out, uint64_t* ops_out) {
  return guard(ctx, [&] {
    require(ctx && scene && h && v && d && saliency_finer && plane, "refine: NULL argument");
    validate_layer(*scene);
    require(is_pow2(n), "scene: plane_size must be a power of two, got " + std::to_string(n));
    require(m >= 1, "refine: residual must be square");
    // refine_stage (synthesis.cpp:94-105)
    require(n % (2 * m) == 0, "refine: LUT block size does not match the residual level");
    const int block = n / (2 * m);
    require(block == 1 || block == 2 || block == 4 || block == 8,
            "refine: LUT block size does not match the residual level");
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const int mr = 2 * m;
    const size_t m2 = size_t(m) * m, r2 = size_t(mr) * mr, n2 = size_t(n) * n;
    float2* lut = lut_in_alloc(ctx->b_lut, n, s);
    launch_build_lut(*scene, n, block, lut, ctx->b_lut_scratch, s);
    char* in = static_cast<char*>(ctx->b_in.reserve((3 * m2 + r2) * 8));
    double* bands = reinterpret_cast<double*>(in);
    double* sal = bands + 3 * m2;
    WCGH_CUDA(cudaMemcpyAsync(bands, h, m2 * 8, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(bands + m2, v, m2 * 8, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(bands + 2 * m2, d, m2 * 8, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(sal, saliency_finer, r2 * 8, cudaMemcpyHostToDevice, s));
    const size_t wbytes = ((r2 * 4 + 255) / 256) * 256, mbytes = ((r2 + 255) / 256) * 256;
    char* o = static_cast<char*>(ctx->b_out.reserve(wbytes + mbytes + 256 + n2 * 8));
    float* w = reinterpret_cast<float*>(o);
    uint8_t* mask = reinterpret_cast<uint8_t*>(o + wbytes);
    unsigned long long* count = reinterpret_cast<unsigned long long*>(o + wbytes + mbytes);
    float2* contrib = reinterpret_cast<float2*>(o + wbytes + mbytes + 256);
    WCGH_CUDA(cudaMemsetAsync(count, 0, 8, s));
    launch_refine_gate(bands, bands + m2, bands + 2 * m2, m, sal, threshold, w, mask, count, s);
    launch_lut_dense(lut, n, block, w, mr, 0, 0, n, contrib, ctx->cells, ctx->lut_partial, s, nullptr);
    std::vector<float> c(2 * n2);
    unsigned long long gated = 0;
    WCGH_CUDA(cudaMemcpyAsync(c.data(), contrib, 2 * n2 * 4, cudaMemcpyDeviceToHost, s));
    WCGH_CUDA(cudaMemcpyAsync(&gated, count, 8, cudaMemcpyDeviceToHost, s));
    if (mask_out) WCGH_CUDA(cudaMemcpyAsync(mask_out, mask, r2, cudaMemcpyDeviceToHost, s));
    sync(s);
    for (size_t i = 0; i < 2 * n2; ++i) plane[i] += c[i];
    if (ops_out) *ops_out += gated;
  });
}

// ---------------------------------------------------------------------------
// jobs

int wcgh_job_create(wcgh_ctx* ctx, const wcgh_desc* desc, wcgh_job** out) {
  return guard(ctx, [&] {
    require(ctx && desc && out, "job_create: NULL argument");
    job_validate(*desc);
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    auto j = std::make_unique<wcgh_job>();
    j->ctx = ctx;
    j->desc = *desc;
    j->layers.assign(desc->layers, desc->layers + desc->n_layers);
    j->desc.layers = j->layers.data();
    const wcgh_desc& d = j->desc;
    const int No = d.object_size, L = d.n_layers;
    j->off = (d.plane_size - No) / 2;
    j->in_elems = size_t(No) * No;
    j->obj.reserve(j->in_elems * L * dtype_size(d.obj_dtype));
    j->sal.reserve(j->in_elems * L * dtype_size(d.sal_dtype));
    j->a_eff.reserve(j->in_elems * L * 4);
    const size_t nseg = size_t(L) * No * seg_per_row(No);
    j->seg_counts.reserve((nseg + 1) * 4);
    j->seg_offsets.reserve((nseg + 1) * 4);
    j->ops.reserve(sizeof(unsigned long long) * WCGH_OP_LEVELS * L + 64);
    j->err.reserve(64);
    j->plane.reserve(sizeof(float2) * size_t(d.rows) * d.plane_size);
    WCGH_CUDA(cudaMallocHost(&j->h_offsets, sizeof(int64_t) * (L + 1)));
    WCGH_CUDA(cudaMallocHost(&j->h_ops, sizeof(unsigned long long) * WCGH_OP_LEVELS * L));
    WCGH_CUDA(cudaMallocHost(&j->h_err, sizeof(int) * 4));
    WCGH_CUDA(cudaMallocHost(&j->h_tot, sizeof(int) * 3 * 4 * kMaxLayers));
    for (auto& e : j->ev) WCGH_CUDA(cudaEventCreate(&e));
    if (d.method == WCGH_METHOD_DIRECT) {
      j->points.reserve(sizeof(wcgh_point) * (j->in_elems * L + 1));
    } else if (d.method == WCGH_METHOD_FFT) {
      // fringe spectra per layer on the 2Nh grid (precompute)
      fft_prepare(j->fft, d.layers, L, d.plane_size, ctx->stream);
      sync(ctx->stream);
    } else {
      // LUT method: precompute the four block LUTs per layer (reported
      // separately from synthesis, like the reference's lut_build).
      j->w_stage.reserve(sizeof(float) * wstage_len(No) * L);
      j->stage_planes.reserve(sizeof(float2) * size_t(d.rows) * d.plane_size * 4);
      const int blocks[4] = {8, 4, 2, 1};
      for (int l = 0; l < L; ++l) {
        for (int st = 0; st < 4; ++st) {
          auto b = std::make_unique<DevBuf>();
          float2* base = lut_in_alloc(*b, d.plane_size, ctx->stream);
          launch_build_lut(d.layers[l], d.plane_size, blocks[st], base, j->lut_scratch,
                           ctx->stream);
          j->luts.push_back(std::move(b));
          j->lut_base.push_back(base);
        }
      }
      sync(ctx->stream);
      j->lut_scratch.release();
    }
    *out = j.release();
  });
}

void wcgh_job_destroy(wcgh_job* job) {
  if (!job) return;
  cudaSetDevice(job->ctx->device);
  cudaStreamSynchronize(job->ctx->stream);
  delete job;
}

int wcgh_job_upload(wcgh_job* job, const void* object, const void* saliency) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && object && saliency, "job_upload: NULL argument");
    use_device(job->ctx);
    cudaStream_t s = job->ctx->stream;
    const size_t L = size_t(job->desc.n_layers);
    WCGH_CUDA(cudaMemcpyAsync(job->obj.p, object, job->in_elems * L * dtype_size(job->desc.obj_dtype), cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(job->sal.p, saliency, job->in_elems * L * dtype_size(job->desc.sal_dtype), cudaMemcpyHostToDevice, s));
    job->uploaded = true;
    job->ran = job->stages_ready = false;
  });
}

int wcgh_job_upload_dev(wcgh_job* job, const void* object, const void* saliency) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && object && saliency, "job_upload_dev: NULL argument");
    use_device(job->ctx);
    cudaStream_t s = job->ctx->stream;
    const size_t L = size_t(job->desc.n_layers);
    WCGH_CUDA(cudaMemcpyAsync(job->obj.p, object, job->in_elems * L * dtype_size(job->desc.obj_dtype), cudaMemcpyDeviceToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(job->sal.p, saliency, job->in_elems * L * dtype_size(job->desc.sal_dtype), cudaMemcpyDeviceToDevice, s));
    job->uploaded = true;
    job->ran = job->stages_ready = false;
  });
}

}  // extern "C"

namespace {

void run_analysis(wcgh_job* j, cudaStream_t s, bool lut) {
  const wcgh_desc& d = j->desc;
  const int No = d.object_size, L = d.n_layers;
  WCGH_CUDA(cudaMemsetAsync(j->ops.p, 0, sizeof(unsigned long long) * WCGH_OP_LEVELS * L + sizeof(int), s));
  AnalysisOut ao;
  ao.a_eff = j->a_eff.as<float>();
  ao.seg_counts = lut ? nullptr : j->seg_counts.as<int>();
  ao.w_stage = lut ? j->w_stage.as<float>() : nullptr;
  ao.ops = j->ops.as<unsigned long long>();
  ao.err = reinterpret_cast<int*>(ao.ops + WCGH_OP_LEVELS * L);
  launch_analysis(j->obj.p, d.obj_dtype, d.obj_scale, j->sal.p, d.sal_dtype, No, L, d.plan, ao, s);
  j->stats.total_launches += 1;
}

void finish_stats(wcgh_job* j, const unsigned long long* ops) {
  const int L = j->desc.n_layers;
  for (int k = 0; k < WCGH_OP_LEVELS; ++k) {
    uint64_t t = 0;
    for (int l = 0; l < L; ++l) t += ops[l * WCGH_OP_LEVELS + k];
    j->stats.ops[k] = t;
  }
}

void run_job_direct(wcgh_job* j, cudaStream_t s, bool synth) {
  const wcgh_desc& d = j->desc;
  const int No = d.object_size, L = d.n_layers;
  j->timing.reset();
  WCGH_CUDA(cudaEventRecord(j->ev[0], s));
  run_analysis(j, s, false);
  const size_t per_layer = size_t(No) * seg_per_row(No);
  const size_t nseg = per_layer * L;
  const bool fft = d.method == WCGH_METHOD_FFT;
  const int scan_launches = launch_scan(j->seg_counts.as<int>(), j->seg_offsets.as<int>(), int(nseg), s,
                                        &j->scan_scratch);
  if (!fft)
    launch_compact_points(j->a_eff.as<float>(), j->seg_offsets.as<int>(), No, L, j->off, 0,
                          j->points.as<wcgh_point>(), s);
  j->stats.total_launches += scan_launches + (fft ? 0 : 1);
  WCGH_CUDA(cudaEventRecord(j->ev[1], s));
  // layer boundaries of the compacted list, ops and validation flags
  for (int l = 0; l <= L; ++l) {
    WCGH_CUDA(cudaMemcpyAsync(reinterpret_cast<int*>(j->h_offsets) + l,
                              j->seg_offsets.as<int>() + per_layer * size_t(l), sizeof(int),
                              cudaMemcpyDeviceToHost, s));
  }
  WCGH_CUDA(cudaMemcpyAsync(j->h_ops, j->ops.p, sizeof(unsigned long long) * WCGH_OP_LEVELS * L, cudaMemcpyDeviceToHost, s));
  WCGH_CUDA(cudaMemcpyAsync(j->h_err, j->ops.as<unsigned long long>() + WCGH_OP_LEVELS * L, sizeof(int), cudaMemcpyDeviceToHost, s));
  sync(s);
  check_analysis_flags(*j->h_err);
  finish_stats(j, j->h_ops);
  int64_t lb[kMaxLayers + 1];
  const int* hoff = reinterpret_cast<const int*>(j->h_offsets);
  for (int l = 0; l <= L; ++l) lb[l] = hoff[l];
  j->stats.n_points = lb[L];
  if (!synth) {  // front end only (wcgh_job_analyze)
    WCGH_CUDA(cudaEventElapsedTime(&j->stats.ms_analysis, j->ev[0], j->ev[1]));
    j->stats.ms_total = j->stats.ms_analysis;
    return;
  }
  // geometry bound on |dx|, |dy| for the phase-series plan
  const double far = double(j->off + No - 1);
  const double max_dy = std::max(std::fabs(double(d.row0) - (j->off + No - 1)),
                                 std::fabs(double(d.row0 + d.rows - 1) - j->off));
  int launches = 0;
  if (fft) {
    // same hologram by FFT correlation; `updates` keeps the direct-sum count
    j->stats.updates = double(lb[L]) * double(d.rows) * double(d.plane_size);
    launches = launch_fft_synthesis(j->fft, j->a_eff.as<float>(), No, j->off, d.plane_size,
                                    d.row0, d.rows, j->plane.as<float2>(), s, &j->timing,
                                    &j->peers);
  } else {
    launches = launch_direct(j->points.as<wcgh_point>(), lb, L, d.layers, d.plane_size, d.row0,
                             d.rows, d.phase_mode, far, max_dy, j->plane.as<float2>(), j->direct,
                             s, &j->timing, &j->stats.updates, &j->peers);
  }
  j->stats.synth_launches = j->timing.launches();
  j->stats.total_launches += launches;
  WCGH_CUDA(cudaEventRecord(j->ev[3], s));
  sync(s);
  WCGH_CUDA(cudaEventElapsedTime(&j->stats.ms_analysis, j->ev[0], j->ev[1]));
  j->stats.ms_synthesis = j->timing.elapsed_ms();
  float synth_phase = 0.f;
  WCGH_CUDA(cudaEventElapsedTime(&synth_phase, j->ev[1], j->ev[3]));
  j->stats.ms_reduce = std::max(0.f, synth_phase - j->stats.ms_synthesis);
  WCGH_CUDA(cudaEventElapsedTime(&j->stats.ms_total, j->ev[0], j->ev[3]));
}

__global__ void k_sum_stages(const float2* __restrict__ planes, size_t count, int n_stages,
                             float2* __restrict__ out, PeerPlanes peers) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  float re = 0.f, im = 0.f;
  for (int st = 0; st < n_stages; ++st) {
    const float2 v = planes[size_t(st) * count + i];
    re += v.x;
    im += v.y;
  }
  out[i] = make_float2(re, im);
  store_peers(peers, i, make_float2(re, im));  // fused row-tile gather (job run only)
}

void run_job_lut(wcgh_job* j, cudaStream_t s, bool synth) {
  const wcgh_desc& d = j->desc;
  const int No = d.object_size, L = d.n_layers;
  j->timing.reset();
  WCGH_CUDA(cudaEventRecord(j->ev[0], s));
  run_analysis(j, s, true);
  const int blocks[4] = {8, 4, 2, 1};
  const int ms[4] = {No / 8, No / 4, No / 2, No};
  size_t wofs[4];
  wofs[0] = 0;
  for (int st = 1; st < 4; ++st) wofs[st] = wofs[st - 1] + size_t(ms[st - 1]) * ms[st - 1];
  // run lists of the nonzero gated cells per (layer, stage) (K2 for the LUT path)
  while (j->cells.size() < size_t(L) * 4) j->cells.push_back(std::make_unique<StageCells>());
  for (int l = 0; l < L; ++l)
    for (int st = 0; st < 4; ++st) {
      const float* w = j->w_stage.as<float>() + wstage_len(No) * l + wofs[st];
      StageCells& sc = *j->cells[size_t(l) * 4 + st];
      j->stats.total_launches += launch_stage_cells(w, ms[st], sc, s);
      stage_cells_totals_async(sc, j->h_tot + 3 * (l * 4 + st), s);
    }
  WCGH_CUDA(cudaMemcpyAsync(j->h_ops, j->ops.p, sizeof(unsigned long long) * WCGH_OP_LEVELS * L, cudaMemcpyDeviceToHost, s));
  WCGH_CUDA(cudaMemcpyAsync(j->h_err, j->ops.as<unsigned long long>() + WCGH_OP_LEVELS * L, sizeof(int), cudaMemcpyDeviceToHost, s));
  WCGH_CUDA(cudaEventRecord(j->ev[1], s));
  sync(s);
  check_analysis_flags(*j->h_err);
  finish_stats(j, j->h_ops);
  if (!synth) {  // front end only (wcgh_job_analyze): nonzero gated cells
    long long cells = 0;
    for (int k = 0; k < 4 * L; ++k) cells += j->h_tot[3 * k + 2];
    j->stats.n_points = cells;
    WCGH_CUDA(cudaEventElapsedTime(&j->stats.ms_analysis, j->ev[0], j->ev[1]));
    j->stats.ms_total = j->stats.ms_analysis;
    return;
  }
  const size_t band = size_t(d.rows) * d.plane_size;
  float2* sp = j->stage_planes.as<float2>();
  long long cells = 0;
  // stage planes accumulate over depth layers (multi-depth = per-layer sum)
  for (int st = 0; st < 4; ++st)
    for (int l = 0; l < L; ++l) {
      const int k = l * 4 + st;
      StageCells& sc = *j->cells[k];
      sc.n_runs = j->h_tot[3 * k];
      sc.n_dense = j->h_tot[3 * k + 1];
      sc.nnz = j->h_tot[3 * k + 2];
      j->stats.total_launches += launch_lut_stage(j->lut_base[k], d.plane_size, blocks[st], sc,
                                                  j->off, d.row0, d.rows, sp + band * st,
                                                  j->lut_partial, s, &j->timing, l > 0);
      cells += sc.nnz;
    }
  j->stats.synth_launches = j->timing.launches();
  WCGH_CUDA(cudaEventRecord(j->ev[2], s));
  k_sum_stages<<<unsigned((band + 255) / 256), 256, 0, s>>>(sp, band, 4, j->plane.as<float2>(),
                                                            j->peers);
  WCGH_CHECK_LAUNCH();
  j->stats.total_launches += 1;
  WCGH_CUDA(cudaEventRecord(j->ev[3], s));
  sync(s);
  // algorithmic updates: (nonzero gated cell, pixel) MACs
  j->stats.n_points = cells;
  j->stats.updates = double(cells) * double(d.rows) * double(d.plane_size);
  WCGH_CUDA(cudaEventElapsedTime(&j->stats.ms_analysis, j->ev[0], j->ev[1]));
  j->stats.ms_synthesis = j->timing.elapsed_ms();
  float synth_phase = 0.f;
  WCGH_CUDA(cudaEventElapsedTime(&synth_phase, j->ev[1], j->ev[3]));
  j->stats.ms_reduce = std::max(0.f, synth_phase - j->stats.ms_synthesis);
  WCGH_CUDA(cudaEventElapsedTime(&j->stats.ms_total, j->ev[0], j->ev[3]));
}

// Stage snapshots of a direct- or FFT-method job (synthesis.hpp:43-54):
// per-stage planes of the stage's amplitude contribution (base LLL, gated
// LL, L, full residuals), synthesised by the job's own method; their prefix
// sums are base_LLL, after_LL, after_L, after_full (linearity). Computed on
// demand, outside wcgh_job_run.
void compute_stage_planes(wcgh_job* j, cudaStream_t s) {
  const wcgh_desc& d = j->desc;
  const int No = d.object_size, L = d.n_layers;
  const wcgh_stats keep = j->stats;
  const size_t band = size_t(d.rows) * d.plane_size;
  j->w_stage.reserve(sizeof(float) * wstage_len(No) * L);
  float2* planes = static_cast<float2*>(j->stage_planes.reserve(sizeof(float2) * band * 4));
  run_analysis(j, s, true);
  float* img = static_cast<float*>(j->snap_img.reserve(sizeof(float) * j->in_elems * L));
  const size_t per_layer = size_t(No) * seg_per_row(No);
  const size_t nseg = per_layer * L;
  const double far = double(j->off + No - 1);
  const double max_dy = std::max(std::fabs(double(d.row0) - (j->off + No - 1)),
                                 std::fabs(double(d.row0 + d.rows - 1) - j->off));
  for (int st = 0; st < 4; ++st) {
    launch_stage_delta(j->w_stage.as<float>(), No, L, st, img, s);
    float2* out = planes + band * st;
    if (d.method == WCGH_METHOD_FFT) {
      launch_fft_synthesis(j->fft, img, No, j->off, d.plane_size, d.row0, d.rows, out, s, nullptr);
      continue;
    }
    launch_seg_counts_f32(img, No, L, j->seg_counts.as<int>(), s);
    launch_scan(j->seg_counts.as<int>(), j->seg_offsets.as<int>(), int(nseg), s, &j->scan_scratch);
    wcgh_point* pts = static_cast<wcgh_point*>(j->snap_points.reserve(sizeof(wcgh_point) * (j->in_elems * L + 1)));
    launch_compact_points(img, j->seg_offsets.as<int>(), No, L, j->off, 0, pts, s);
    for (int l = 0; l <= L; ++l)
      WCGH_CUDA(cudaMemcpyAsync(reinterpret_cast<int*>(j->h_offsets) + l,
                                j->seg_offsets.as<int>() + per_layer * size_t(l), sizeof(int),
                                cudaMemcpyDeviceToHost, s));
    sync(s);
    int64_t lb[kMaxLayers + 1];
    for (int l = 0; l <= L; ++l) lb[l] = reinterpret_cast<const int*>(j->h_offsets)[l];
    launch_direct(pts, lb, L, d.layers, d.plane_size, d.row0, d.rows, d.phase_mode, far, max_dy,
                  out, j->direct, s, nullptr, nullptr);
  }
  sync(s);
  j->stats = keep;
  j->stages_ready = true;
}

}  // namespace

extern "C" {

int wcgh_job_run(wcgh_job* job) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job != nullptr, "job_run: NULL job");
    require(job->uploaded, "job_run: inputs not uploaded");
    use_device(job->ctx);
    job->stats = wcgh_stats{};
    job->ran = job->stages_ready = false;
    if (job->desc.method == WCGH_METHOD_LUT)
      run_job_lut(job, job->ctx->stream, true);
    else  // direct and FFT share the analysis + compaction front end
      run_job_direct(job, job->ctx->stream, true);
    job->ran = true;
    job->stages_ready = job->desc.method == WCGH_METHOD_LUT;
  });
}

int wcgh_job_analyze(wcgh_job* job) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job != nullptr, "job_analyze: NULL job");
    require(job->uploaded, "job_analyze: inputs not uploaded");
    use_device(job->ctx);
    job->stats = wcgh_stats{};
    if (job->desc.method == WCGH_METHOD_LUT)
      run_job_lut(job, job->ctx->stream, false);
    else
      run_job_direct(job, job->ctx->stream, false);
  });
}

int wcgh_job_download(wcgh_job* job, float* out) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && out, "job_download: NULL argument");
    use_device(job->ctx);
    cudaStream_t s = job->ctx->stream;
    WCGH_CUDA(cudaMemcpyAsync(out, job->plane.p, sizeof(float2) * size_t(job->desc.rows) * job->desc.plane_size, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_job_set_peer_planes(wcgh_job* job, void* const* planes_dev, int n_planes) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job != nullptr, "job_set_peer_planes: NULL job");
    require(n_planes >= 0 && n_planes <= kMaxPeers, "job_set_peer_planes: 0..16 planes");
    require(n_planes == 0 || planes_dev != nullptr, "job_set_peer_planes: NULL plane list");
    PeerPlanes pp{};
    for (int k = 0; k < n_planes; ++k) {
      require(planes_dev[k] != nullptr, "job_set_peer_planes: NULL plane pointer");
      pp.p[k] = static_cast<float2*>(planes_dev[k]);
    }
    pp.n = n_planes;
    pp.offset = size_t(job->desc.row0) * size_t(job->desc.plane_size);
    job->peers = pp;
  });
}

// ---- CUDA IPC for the fused gather (one process per GPU) --------------------

int wcgh_ipc_alloc_plane(int device, int n, void** dev_ptr, unsigned char* handle64) {
  return guard(nullptr, [&] {
    require(dev_ptr && handle64, "ipc_alloc_plane: NULL argument");
    require(n >= 1 && n <= 65536, "ipc_alloc_plane: bad plane size");
    WCGH_CUDA(cudaSetDevice(device));
    void* p = nullptr;
    WCGH_CUDA(cudaMalloc(&p, sizeof(float2) * size_t(n) * size_t(n)));
    WCGH_CUDA(cudaMemset(p, 0, sizeof(float2) * size_t(n) * size_t(n)));
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      throw RuntimeError(std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    std::memcpy(handle64, &h, 64);
    *dev_ptr = p;
  });
}

int wcgh_ipc_open_plane(int device, const unsigned char* handle64, void** dev_ptr) {
  return guard(nullptr, [&] {
    require(dev_ptr && handle64, "ipc_open_plane: NULL argument");
    WCGH_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    WCGH_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int wcgh_ipc_close_plane(void* dev_ptr) {
  return guard(nullptr, [&] { WCGH_CUDA(cudaIpcCloseMemHandle(dev_ptr)); });
}

int wcgh_ipc_free_plane(void* dev_ptr) {
  return guard(nullptr, [&] { WCGH_CUDA(cudaFree(dev_ptr)); });
}

int wcgh_job_download_a_eff(wcgh_job* job, float* out) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && out, "job_download_a_eff: NULL argument");
    use_device(job->ctx);
    cudaStream_t s = job->ctx->stream;
    WCGH_CUDA(cudaMemcpyAsync(out, job->a_eff.p, sizeof(float) * job->in_elems * job->desc.n_layers,
                              cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_job_download_points(wcgh_job* job, wcgh_point* out, int64_t capacity, int64_t* n_out) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job != nullptr, "job_download_points: NULL job");
    require(job->desc.method != WCGH_METHOD_LUT && job->desc.method != WCGH_METHOD_FFT,
            "job_download_points: the compacted point list is built by the direct method");
    const int64_t n = int64_t(job->stats.n_points);
    if (n_out) *n_out = n;
    if (out == nullptr) return;
    require(capacity >= n, "job_download_points: capacity below the point count");
    use_device(job->ctx);
    cudaStream_t s = job->ctx->stream;
    WCGH_CUDA(cudaMemcpyAsync(out, job->points.p, sizeof(wcgh_point) * size_t(n), cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_job_download_stages(wcgh_job* job, float* out4) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && out4, "job_download_stages: NULL argument");
    require(job->ran, "job_download_stages: run the job first");
    use_device(job->ctx);
    cudaStream_t s = job->ctx->stream;
    if (!job->stages_ready) compute_stage_planes(job, s);
    const size_t band = size_t(job->desc.rows) * job->desc.plane_size;
    float2* tmp = static_cast<float2*>(job->lut_scratch.reserve(sizeof(float2) * band));
    for (int st = 0; st < 4; ++st) {
      // snapshot after stage st = sum of stage planes 0..st, in stage order
      k_sum_stages<<<unsigned((band + 255) / 256), 256, 0, s>>>(job->stage_planes.as<float2>(), band,
                                                                st + 1, tmp, PeerPlanes{});
      WCGH_CHECK_LAUNCH();
      WCGH_CUDA(cudaMemcpyAsync(out4 + 2 * band * st, tmp, sizeof(float2) * band, cudaMemcpyDeviceToHost, s));
      sync(s);
    }
  });
}

void* wcgh_job_plane_dev(wcgh_job* job) { return job ? job->plane.p : nullptr; }

int wcgh_job_stats(const wcgh_job* job, wcgh_stats* out) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && out, "job_stats: NULL argument");
    *out = job->stats;
  });
}

// ---- CGH1 files (image_io.cpp:220-278): 34-byte header + f32 payload ------

int wcgh_write_cgh1(const char* path, const float* plane, int n, const wcgh_layer* scene) {
  return guard(nullptr, [&] {
    require(path && plane && scene, "save_hologram: NULL argument");
    validate_layer(*scene);
    require(is_pow2(n), "save_hologram: field size does not match scene plane_size");
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw RuntimeError(std::string("hologram: cannot open ") + path + " for writing");
    const char magic[4] = {'C', 'G', 'H', '1'};
    const uint16_t version = 1;
    const uint32_t un = uint32_t(n);
    bool ok = std::fwrite(magic, 1, 4, f) == 4 && std::fwrite(&version, 2, 1, f) == 1 &&
              std::fwrite(&un, 4, 1, f) == 1 && std::fwrite(&scene->wavelength, 8, 1, f) == 1 &&
              std::fwrite(&scene->pitch, 8, 1, f) == 1 && std::fwrite(&scene->z, 8, 1, f) == 1;
    const size_t count = size_t(n) * n * 2;
    ok = ok && std::fwrite(plane, sizeof(float), count, f) == count;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw RuntimeError(std::string("hologram: write failed for ") + path);
  });
}

int wcgh_read_cgh1(const char* path, float* plane, int64_t capacity, int* n_out,
                   wcgh_layer* scene_out) {
  return guard(nullptr, [&] {
    require(path != nullptr, "load_hologram: NULL path");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw RuntimeError(std::string("hologram: cannot open ") + path);
    struct Closer {
      std::FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "CGH1", 4) != 0)
      throw RuntimeError(std::string("hologram: bad magic in ") + path);
    uint16_t version = 0;
    uint32_t un = 0;
    wcgh_layer sc{};
    if (std::fread(&version, 2, 1, f) != 1 || std::fread(&un, 4, 1, f) != 1 ||
        std::fread(&sc.wavelength, 8, 1, f) != 1 || std::fread(&sc.pitch, 8, 1, f) != 1 ||
        std::fread(&sc.z, 8, 1, f) != 1)
      throw RuntimeError("hologram: truncated or unreadable header");
    if (version != 1) throw RuntimeError("hologram: unsupported version " + std::to_string(version));
    validate_layer(sc);
    require(un > 0 && un <= 65536 && is_pow2(int(un)),
            "scene: plane_size must be a power of two, got " + std::to_string(un));
    if (n_out) *n_out = int(un);
    if (scene_out) *scene_out = sc;
    if (plane) {
      const size_t count = size_t(un) * un;
      require(capacity >= int64_t(count), "load_hologram: output buffer too small");
      if (std::fread(plane, sizeof(float) * 2, count, f) != count)
        throw RuntimeError("hologram: truncated payload");
      for (size_t i = 0; i < 2 * count; ++i)
        if (!std::isfinite(plane[i]))
          throw ValidationError(std::string("hologram ") + path + ": non-finite sample");
    }
  });
}

// ---- CGHL LUT cache files (fringe_lut.cpp:95-166): 36-byte header + f32 ----

int wcgh_write_cghl(const char* path, const float* lut, int n, int block, const wcgh_layer* scene) {
  return guard(nullptr, [&] {
    require(path && lut && scene, "lut cache: NULL argument");
    validate_layer(*scene);
    require(is_pow2(n), "scene: plane_size must be a power of two, got " + std::to_string(n));
    require(block == 1 || block == 2 || block == 4 || block == 8,
            "build_block_lut: unsupported block size " + std::to_string(block));
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw RuntimeError(std::string("lut cache: cannot open ") + path + " for writing");
    const char magic[4] = {'C', 'G', 'H', 'L'};
    const uint16_t version = 1, b = uint16_t(block);
    const uint32_t un = uint32_t(n);
    bool ok = std::fwrite(magic, 1, 4, f) == 4 && std::fwrite(&version, 2, 1, f) == 1 &&
              std::fwrite(&b, 2, 1, f) == 1 && std::fwrite(&un, 4, 1, f) == 1 &&
              std::fwrite(&scene->wavelength, 8, 1, f) == 1 &&
              std::fwrite(&scene->pitch, 8, 1, f) == 1 && std::fwrite(&scene->z, 8, 1, f) == 1;
    const size_t span = size_t(2 * n - 1);
    const size_t count = span * span * 2;
    ok = ok && std::fwrite(lut, sizeof(float), count, f) == count;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw RuntimeError(std::string("lut cache: write failed for ") + path);
  });
}

int wcgh_read_cghl(const char* path, float* lut, int64_t capacity, int* n_out, int* block_out,
                   wcgh_layer* scene_out) {
  return guard(nullptr, [&] {
    require(path != nullptr, "lut cache: NULL path");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw RuntimeError(std::string("lut cache: cannot open ") + path);
    struct Closer {
      std::FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "CGHL", 4) != 0)
      throw RuntimeError(std::string("lut cache: bad magic in ") + path);
    uint16_t version = 0, block = 0;
    uint32_t un = 0;
    wcgh_layer sc{};
    if (std::fread(&version, 2, 1, f) != 1 || std::fread(&block, 2, 1, f) != 1 ||
        std::fread(&un, 4, 1, f) != 1 || std::fread(&sc.wavelength, 8, 1, f) != 1 ||
        std::fread(&sc.pitch, 8, 1, f) != 1 || std::fread(&sc.z, 8, 1, f) != 1)
      throw RuntimeError("lut cache: truncated header");
    if (version != 1) throw RuntimeError("lut cache: unsupported version " + std::to_string(version));
    require(un > 0 && un <= 65536 && is_pow2(int(un)),
            "scene: plane_size must be a power of two, got " + std::to_string(un));
    if (n_out) *n_out = int(un);
    if (block_out) *block_out = int(block);
    if (scene_out) *scene_out = sc;
    if (lut) {
      const size_t span = size_t(2 * un - 1);
      const size_t count = span * span;
      require(capacity >= int64_t(count), "lut cache: output buffer too small");
      if (std::fread(lut, sizeof(float) * 2, count, f) != count)
        throw RuntimeError("lut cache: truncated payload");
      for (size_t i = 0; i < 2 * count; ++i)
        if (!std::isfinite(lut[i]))
          throw ValidationError(std::string("lut cache ") + path + ": non-finite sample");
    }
  });
}

int wcgh_job_load_lut(wcgh_job* job, int layer, int block, const float* lut) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && lut, "job_load_lut: NULL argument");
    require(job->desc.method == WCGH_METHOD_LUT, "job_load_lut: the job does not use the LUT method");
    require(layer >= 0 && layer < job->desc.n_layers, "job_load_lut: layer out of range");
    int st = -1;
    const int blocks[4] = {8, 4, 2, 1};
    for (int k = 0; k < 4; ++k)
      if (blocks[k] == block) st = k;
    require(st >= 0, "build_block_lut: unsupported block size " + std::to_string(block));
    for (int i = 0; i < 2 * (2 * job->desc.plane_size - 1) * (2 * job->desc.plane_size - 1); ++i)
      if (!std::isfinite(lut[i])) throw ValidationError("lut: non-finite sample");
    use_device(job->ctx);
    const size_t span = size_t(2 * job->desc.plane_size - 1);
    WCGH_CUDA(cudaMemcpyAsync(job->lut_base[size_t(layer) * 4 + st], lut, sizeof(float2) * span * span,
                              cudaMemcpyHostToDevice, job->ctx->stream));
    sync(job->ctx->stream);
  });
}

int wcgh_job_write_cgh1(wcgh_job* job, const char* path, int stage) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && path, "job_write_cgh1: NULL argument");
    const wcgh_desc& d = job->desc;
    require(d.row0 == 0 && d.rows == d.plane_size,
            "save_hologram: field size does not match scene plane_size (job holds a row band)");
    require(stage < 4, "job_write_cgh1: stage index out of range");
    const size_t count = size_t(d.plane_size) * d.plane_size;
    std::vector<float> host(2 * count);
    if (stage < 0) {
      use_device(job->ctx);
      WCGH_CUDA(cudaMemcpyAsync(host.data(), job->plane.p, sizeof(float2) * count, cudaMemcpyDeviceToHost,
                                job->ctx->stream));
      sync(job->ctx->stream);
    } else {
      std::vector<float> all(8 * count);
      const int rc = wcgh_job_download_stages(job, all.data());
      if (rc == WCGH_EVALIDATION) throw ValidationError(t_last_error);
      if (rc) throw RuntimeError(t_last_error);
      std::memcpy(host.data(), all.data() + 2 * count * size_t(stage), sizeof(float) * 2 * count);
    }
    const int rc = wcgh_write_cgh1(path, host.data(), d.plane_size, &job->layers[0]);
    if (rc == WCGH_EVALIDATION) throw ValidationError(t_last_error);
    if (rc) throw RuntimeError(t_last_error);
  });
}

// ---- reconstruction and metrics (angular_spectrum.cpp, fft.cpp, metrics.cpp)

namespace {
void require_fft_side(int n) {
  require(n >= 1 && is_pow2(n), "fft_2d: side must be a power of two");
}
void require_complex_dtype(int dtype) {
  require(dtype == WCGH_F32 || dtype == WCGH_F64,
          "field: dtype must be WCGH_F32 (complex64) or WCGH_F64 (complex128)");
}
void require_optics(const wcgh_layer* scene) {
  require(scene != nullptr, "scene: NULL");
  require(scene->wavelength > 0.0, "scene: wavelength must be positive");
  require(scene->pitch > 0.0, "scene: pitch must be positive");
}
}  // namespace

int wcgh_fft_2d(wcgh_ctx* ctx, const double* field, int n, int inverse, double* out) {
  return guard(ctx, [&] {
    require(ctx && field && out, "fft_2d: NULL argument");
    require_fft_side(n);
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t bytes = sizeof(double2) * size_t(n) * n;
    double2* f = recon_field(ctx->recon, n);
    WCGH_CUDA(cudaMemcpyAsync(f, field, bytes, cudaMemcpyHostToDevice, s));
    launch_fft2d(ctx->recon, n, inverse != 0, s);
    WCGH_CUDA(cudaMemcpyAsync(out, f, bytes, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_propagation_kernel(wcgh_ctx* ctx, const wcgh_layer* scene, int n, double z_signed,
                            double* out) {
  return guard(ctx, [&] {
    require(ctx && out, "build_kernel: NULL argument");
    require_optics(scene);
    require(z_signed != 0.0, "build_kernel: |z| must be positive");
    require_fft_side(n);
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    double2* f = recon_field(ctx->recon, n);
    launch_transfer(n, scene->wavelength, scene->pitch, z_signed, f, s);
    WCGH_CUDA(cudaMemcpyAsync(out, f, sizeof(double2) * size_t(n) * n, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_propagate(wcgh_ctx* ctx, const void* field, int dtype, int n, const wcgh_layer* scene,
                   double z_signed, double* out) {
  return guard(ctx, [&] {
    require(ctx && field && out, "propagate: NULL argument");
    require_optics(scene);
    require(z_signed != 0.0, "build_kernel: |z| must be positive");
    require_complex_dtype(dtype);
    require_fft_side(n);
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t nn = size_t(n) * n;
    const bool single = dtype == WCGH_F32;
    void* in = ctx->b_in.reserve((single ? sizeof(float2) : sizeof(double2)) * nn);
    WCGH_CUDA(cudaMemcpyAsync(in, field, (single ? sizeof(float2) : sizeof(double2)) * nn,
                              cudaMemcpyHostToDevice, s));
    load_field(ctx->recon, in, single, n, s);
    launch_propagate(ctx->recon, n, scene->wavelength, scene->pitch, z_signed, true, s);
    WCGH_CUDA(cudaMemcpyAsync(out, ctx->recon.field.p, sizeof(double2) * nn, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_reconstruct(wcgh_ctx* ctx, const void* hologram, int dtype, int n,
                     const wcgh_layer* scene, int intensity, double* out) {
  return guard(ctx, [&] {
    require(ctx && hologram && out, "reconstruct: NULL argument");
    require_optics(scene);
    require(scene->z != 0.0, "build_kernel: |z| must be positive");
    require_complex_dtype(dtype);
    require_fft_side(n);
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t nn = size_t(n) * n;
    const bool single = dtype == WCGH_F32;
    void* in = ctx->b_in.reserve((single ? sizeof(float2) : sizeof(double2)) * nn);
    WCGH_CUDA(cudaMemcpyAsync(in, hologram, (single ? sizeof(float2) : sizeof(double2)) * nn,
                              cudaMemcpyHostToDevice, s));
    load_field(ctx->recon, in, single, n, s);
    double* img = static_cast<double*>(ctx->b_out.reserve(sizeof(double) * nn));
    launch_reconstruct(ctx->recon, n, scene->wavelength, scene->pitch, scene->z, intensity != 0,
                       img, s);
    WCGH_CUDA(cudaMemcpyAsync(out, img, sizeof(double) * nn, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_job_reconstruct(wcgh_job* job, const wcgh_layer* scene, int intensity, double* out) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && out, "reconstruct: NULL argument");
    require_optics(scene);
    require(scene->z != 0.0, "build_kernel: |z| must be positive");
    const int n = job->desc.plane_size;
    require(job->desc.row0 == 0 && job->desc.rows == n,
            "reconstruct: the job must hold the whole plane (row0 = 0, rows = plane_size)");
    wcgh_ctx* ctx = job->ctx;
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t nn = size_t(n) * n;
    load_field(ctx->recon, job->plane.p, true, n, s);
    double* img = static_cast<double*>(ctx->b_out.reserve(sizeof(double) * nn));
    launch_reconstruct(ctx->recon, n, scene->wavelength, scene->pitch, scene->z, intensity != 0,
                       img, s);
    WCGH_CUDA(cudaMemcpyAsync(out, img, sizeof(double) * nn, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_ssim(wcgh_ctx* ctx, const double* a, const double* b, int width, int height, int window,
              double k1, double k2, double dynamic_range, double* score) {
  return guard(ctx, [&] {
    require(ctx && a && b && score, "ssim: NULL argument");
    require(width >= 1 && height >= 1, "ssim: image sizes differ");
    require(window > 0 && window <= std::min(width, height),
            "ssim: window must fit inside the images");
    require(dynamic_range > 0.0, "ssim: dynamic range must be positive");
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const size_t nn = size_t(width) * height;
    double* da = static_cast<double*>(ctx->b_in.reserve(sizeof(double) * nn));
    double* db = static_cast<double*>(ctx->b_in2.reserve(sizeof(double) * nn));
    double* dr = static_cast<double*>(ctx->b_misc.reserve(sizeof(double)));
    WCGH_CUDA(cudaMemcpyAsync(da, a, sizeof(double) * nn, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(db, b, sizeof(double) * nn, cudaMemcpyHostToDevice, s));
    launch_ssim(da, db, width, height, window, k1, k2, dynamic_range, ctx->b_ssim, dr, s);
    double total = 0.0;
    WCGH_CUDA(cudaMemcpyAsync(&total, dr, sizeof(double), cudaMemcpyDeviceToHost, s));
    sync(s);
    const double count = double(width - window + 1) * double(height - window + 1);
    *score = total / count;
  });
}

int wcgh_synthesize(wcgh_ctx* ctx, const wcgh_desc* desc, const void* object, const void* saliency,
                    float* out, wcgh_stats* stats) {
  wcgh_job* job = nullptr;
  int rc = wcgh_job_create(ctx, desc, &job);
  if (rc) return rc;
  rc = wcgh_job_upload(job, object, saliency);
  if (!rc) rc = wcgh_job_run(job);
  if (!rc) rc = wcgh_job_download(job, out);
  if (!rc && stats) rc = wcgh_job_stats(job, stats);
  wcgh_job_destroy(job);
  return rc;
}

}  // extern "C"

namespace {
// Row band `rank` of `world` (tiles.band: equal splits, remainder to the
// first) on `device`, written into its rows of the host plane `out`.
void synth_band(int rank, int world, int device, const wcgh_desc* desc, const void* object,
                const void* saliency, float* out, wcgh_stats* st, int* rc_out, std::string* err) {
  const int n = desc->plane_size;
  const int base = n / world, rem = n % world;
  wcgh_desc d = *desc;
  d.row0 = rank * base + std::min(rank, rem);
  d.rows = base + (rank < rem ? 1 : 0);
  wcgh_ctx* ctx = nullptr;
  int rc = wcgh_create(device, &ctx);
  if (rc == WCGH_OK) rc = wcgh_synthesize(ctx, &d, object, saliency, out + size_t(2) * d.row0 * n, st);
  if (rc != WCGH_OK) *err = t_last_error;
  *rc_out = rc;
  if (ctx) wcgh_destroy(ctx);
}
}  // namespace

extern "C" {

int wcgh_synthesize_multi(int n_devices, const int* devices, const wcgh_desc* desc,
                          const void* object, const void* saliency, float* out,
                          wcgh_stats* stats) {
  return guard(nullptr, [&] {
    require(n_devices >= 1 && n_devices <= 64, "synthesize_multi: 1..64 devices");
    require(devices && desc && object && saliency && out, "synthesize_multi: NULL argument");
    require(desc->row0 == 0 && desc->rows == desc->plane_size,
            "synthesize_multi: desc must describe the whole plane (row0 = 0, rows = plane_size)");
    require(n_devices <= desc->plane_size, "synthesize_multi: more devices than plane rows");
    std::vector<int> rcs(size_t(n_devices), WCGH_OK);
    std::vector<std::string> errs(static_cast<size_t>(n_devices));
    std::vector<wcgh_stats> st(static_cast<size_t>(n_devices));
    std::vector<std::thread> workers;
    for (int i = 0; i < n_devices; ++i)
      workers.emplace_back(synth_band, i, n_devices, devices[i], desc, object, saliency, out,
                           st.data() + i, rcs.data() + i, errs.data() + i);
    for (auto& w : workers) w.join();
    for (int i = 0; i < n_devices; ++i) {
      if (rcs[size_t(i)] == WCGH_EVALIDATION) throw ValidationError(errs[size_t(i)]);
      if (rcs[size_t(i)] != WCGH_OK)
        throw RuntimeError(errs[size_t(i)] + " (device " + std::to_string(devices[i]) + ")");
    }
    if (stats) {
      // ops / points come from the (identical, redundant) analysis of every
      // band; work adds up, times are the slowest band's
      wcgh_stats agg = st[0];
      for (int i = 1; i < n_devices; ++i) {
        const wcgh_stats& t = st[size_t(i)];
        agg.updates += t.updates;
        agg.ms_analysis = std::max(agg.ms_analysis, t.ms_analysis);
        agg.ms_synthesis = std::max(agg.ms_synthesis, t.ms_synthesis);
        agg.ms_reduce = std::max(agg.ms_reduce, t.ms_reduce);
        agg.ms_total = std::max(agg.ms_total, t.ms_total);
        agg.synth_launches += t.synth_launches;
        agg.total_launches += t.total_launches;
      }
      *stats = agg;
    }
  });
}

}  // extern "C"
