// C ABI of the B200-native hot path (include/wcgh.h): contexts, the stage
// entry points the host mirrors call, and the reconstruction / metrics
// entry points. Jobs and multi-GPU are in wcgh_job.cu, file I/O in
// wcgh_io.cu. Validation mirrors the reference's ValidationError sites; CUDA
// failures map to WCGH_ERUNTIME.
#include <complex>
#include <random>

#include "wcgh_state.cuh"

using namespace wcgh;
using namespace wcgh::abi;

thread_local std::string wcgh::abi::t_last_error;

#ifdef WCGH_CHECKED
namespace wcgh {
namespace chk {
void collect_wcgh_analysis();
void collect_wcgh_direct();
void collect_wcgh_lut();
void collect_wcgh_fft();
void collect_wcgh_recon();
void collect_wcgh_abi();
void collect_wcgh_job();
void collect_wcgh_io();
void collect_wcgh_lutobj();
void collect_wcgh_helpers();
void collect_wcgh_fftk();
void collect_all() {
  collect_wcgh_analysis();
  collect_wcgh_direct();
  collect_wcgh_lut();
  collect_wcgh_fft();
  collect_wcgh_recon();
  collect_wcgh_abi();
  collect_wcgh_job();
  collect_wcgh_io();
  collect_wcgh_lutobj();
  collect_wcgh_helpers();
  collect_wcgh_fftk();
}
}  // namespace chk
}  // namespace wcgh
#endif

extern "C" {

int wcgh_abi_version(void) { return WCGH_ABI_VERSION; }

// The reference's random initial phase, on the host with the same standard
// library engine and distribution, so the complex object is bit-identical.
int wcgh_random_phase_field(const double* amplitude, int width, int height, uint64_t seed,
                            double* out) {
  return guard(nullptr, [&] {
    require(amplitude && out, "random_phase_field: NULL argument");
    require(width >= 0 && height >= 0, "random_phase_field: negative size");
    std::mt19937_64 rng(seed);
    // 2 * std::numbers::pi (the same double)
    std::uniform_real_distribution<double> angle(0.0, 2.0 * 3.141592653589793238462643383279502884);
    const size_t count = size_t(width) * size_t(height);
    for (size_t i = 0; i < count; ++i) {
      const std::complex<double> v = std::polar(amplitude[i], angle(rng));
      out[2 * i] = v.real();
      out[2 * i + 1] = v.imag();
    }
  });
}

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
    require(obj_dtype != WCGH_C128 && sal_dtype != WCGH_C128,
            "analyze: real images only (complex objects go through a job)");
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
    const size_t rep_bytes = sizeof(unsigned long long) * WCGH_OP_LEVELS * kOpReplicas;
    ao.ops_rep = static_cast<unsigned long long*>(ctx->b_ops_rep.reserve(rep_bytes));
    WCGH_CUDA(cudaMemsetAsync(ao.ops_rep, 0, rep_bytes, s));
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
      // the series plan covers the whole plane, not just the band, so any row
      // band of it is bitwise the same rows of the full plane (fixed chunks)
      max_dy = std::max({max_dy, std::fabs(double(p.y)), std::fabs(double(nh - 1 - p.y))});
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

}  // extern "C"

WCGH_CHK_TU(wcgh_abi)
