// Device-resident LUTs and planes (include/wcgh.h "device-resident LUTs and
// planes"): the caller's FringeLut support uploaded once (fringe_lut.cpp:34-51,
// read by apply_block_unchecked, synthesis.cpp:18-42) and a hologram plane
// that apply_block / refine stage calls (synthesis.cpp:149-178) accumulate
// into on the device, without the per-call plane round trip of the
// scene-based wcgh_apply_blocks / wcgh_refine.
#include <cstring>

#include "wcgh_state.cuh"

using namespace wcgh;
using namespace wcgh::abi;

struct wcgh_lut {
  wcgh_ctx* ctx = nullptr;
  wcgh_layer scene{};
  int n = 0, block = 0;
  DevBuf buf;            // guarded allocation (lut_alloc_bytes)
  float2* base = nullptr;  // support element (0, 0)
};

struct wcgh_plane {
  wcgh_ctx* ctx = nullptr;
  int n = 0;
  DevBuf buf;  // n * n complex64
};

namespace {

// complex64/complex128 host samples -> complex64 device support, rounding
// once (the CGHL payload rounding, fringe_lut.cpp:107-113); a non-finite
// sample raises the error flag.
template <typename T>
__global__ void k_import_complex(const T* __restrict__ src, size_t count, float2* __restrict__ dst,
                                 int* __restrict__ err) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const T re = src[2 * i], im = src[2 * i + 1];
  if (!isfinite(re) || !isfinite(im)) atomicOr(err, 1);
  dst[i] = make_float2(float(re), float(im));
}

__global__ void k_widen_complex(const float2* __restrict__ src, size_t count, double2* __restrict__ dst) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) dst[i] = make_double2(double(src[i].x), double(src[i].y));
}

// Host samples of `count` complex values (dtype WCGH_F32 = complex64,
// WCGH_F64 = complex128) into a device complex64 array, validated.
void import_complex(wcgh_ctx* ctx, const void* host, int dtype, size_t count, float2* dst,
                    const char* what) {
  require(dtype == WCGH_F32 || dtype == WCGH_F64,
          std::string(what) + ": dtype must be WCGH_F32 (complex64) or WCGH_F64 (complex128)");
  cudaStream_t s = ctx->stream;
  const size_t bytes = count * 2 * (dtype == WCGH_F32 ? 4 : 8);
  const size_t err_at = (bytes + 255) / 256 * 256;
  char* stage = static_cast<char*>(ctx->b_in2.reserve(err_at + 256));
  int* err = reinterpret_cast<int*>(stage + err_at);
  WCGH_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
  WCGH_CUDA(cudaMemcpyAsync(stage, host, bytes, cudaMemcpyHostToDevice, s));
  const unsigned g = unsigned((count + 255) / 256);
  if (dtype == WCGH_F32)
    k_import_complex<float><<<g, 256, 0, s>>>(reinterpret_cast<const float*>(stage), count, dst, err);
  else
    k_import_complex<double><<<g, 256, 0, s>>>(reinterpret_cast<const double*>(stage), count, dst, err);
  WCGH_CHECK_LAUNCH();
  int h_err = 0;
  WCGH_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  sync(s);
  if (h_err) throw ValidationError(std::string(what) + ": non-finite sample");
}

bool same_scene(const wcgh_layer& a, const wcgh_layer& b) {
  return a.wavelength == b.wavelength && a.pitch == b.pitch && a.z == b.z;
}

}  // namespace

extern "C" {

int wcgh_lut_create(wcgh_ctx* ctx, const wcgh_layer* scene, int n, int block, const void* samples,
                    int dtype, wcgh_lut** out) {
  return guard(ctx, [&] {
    require(ctx && scene && out, "lut_create: NULL argument");
    validate_layer(*scene);
    require(is_pow2(n), "scene: plane_size must be a power of two, got " + std::to_string(n));
    require(block == 1 || block == 2 || block == 4 || block == 8,
            "FringeLut: unsupported block size " + std::to_string(block));
    require(block <= n, "FringeLut: block size exceeds plane size");
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    auto lut = std::make_unique<wcgh_lut>();
    lut->ctx = ctx;
    lut->scene = *scene;
    lut->n = n;
    lut->block = block;
    cudaStream_t s = ctx->stream;
    lut->base = lut_in_alloc(lut->buf, n, s);
    const size_t span = size_t(2 * n - 1);
    if (samples)
      import_complex(ctx, samples, dtype, span * span, lut->base, "FringeLut: support");
    else
      launch_build_lut(*scene, n, block, lut->base, ctx->b_lut_scratch, s);
    sync(s);
    *out = lut.release();
  });
}

void wcgh_lut_destroy(wcgh_lut* lut) {
  if (!lut) return;
  cudaSetDevice(lut->ctx->device);
  delete lut;
}

int wcgh_lut_download(wcgh_lut* lut, float* out) {
  return guard(lut ? lut->ctx : nullptr, [&] {
    require(lut && out, "lut_download: NULL argument");
    std::lock_guard<std::mutex> lk(lut->ctx->mu);
    use_device(lut->ctx);
    const size_t span = size_t(2 * lut->n - 1);
    WCGH_CUDA(cudaMemcpyAsync(out, lut->base, sizeof(float2) * span * span, cudaMemcpyDeviceToHost,
                              lut->ctx->stream));
    sync(lut->ctx->stream);
  });
}

int wcgh_plane_create(wcgh_ctx* ctx, int n, wcgh_plane** out) {
  return guard(ctx, [&] {
    require(ctx && out, "plane_create: NULL argument");
    require(n >= 1 && n <= 65536, "plane_create: side must be in [1, 65536]");
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    auto p = std::make_unique<wcgh_plane>();
    p->ctx = ctx;
    p->n = n;
    const size_t bytes = size_t(n) * n * sizeof(float2);
    p->buf.reserve(bytes);
    WCGH_CUDA(cudaMemsetAsync(p->buf.p, 0, bytes, ctx->stream));
    sync(ctx->stream);
    *out = p.release();
  });
}

void wcgh_plane_destroy(wcgh_plane* plane) {
  if (!plane) return;
  cudaSetDevice(plane->ctx->device);
  delete plane;
}

int wcgh_plane_zero(wcgh_plane* plane) {
  return guard(plane ? plane->ctx : nullptr, [&] {
    require(plane != nullptr, "plane_zero: NULL plane");
    std::lock_guard<std::mutex> lk(plane->ctx->mu);
    use_device(plane->ctx);
    WCGH_CUDA(cudaMemsetAsync(plane->buf.p, 0, size_t(plane->n) * plane->n * sizeof(float2),
                              plane->ctx->stream));
    sync(plane->ctx->stream);
  });
}

int wcgh_plane_upload(wcgh_plane* plane, const void* host, int dtype) {
  return guard(plane ? plane->ctx : nullptr, [&] {
    require(plane && host, "plane_upload: NULL argument");
    std::lock_guard<std::mutex> lk(plane->ctx->mu);
    use_device(plane->ctx);
    import_complex(plane->ctx, host, dtype, size_t(plane->n) * plane->n, plane->buf.as<float2>(),
                   "plane_upload");
  });
}

int wcgh_plane_download(wcgh_plane* plane, void* host, int dtype) {
  return guard(plane ? plane->ctx : nullptr, [&] {
    require(plane && host, "plane_download: NULL argument");
    require(dtype == WCGH_F32 || dtype == WCGH_F64,
            "plane_download: dtype must be WCGH_F32 (complex64) or WCGH_F64 (complex128)");
    std::lock_guard<std::mutex> lk(plane->ctx->mu);
    use_device(plane->ctx);
    cudaStream_t s = plane->ctx->stream;
    const size_t count = size_t(plane->n) * plane->n;
    if (dtype == WCGH_F32) {
      WCGH_CUDA(cudaMemcpyAsync(host, plane->buf.p, count * sizeof(float2), cudaMemcpyDeviceToHost, s));
    } else {
      double2* wide = static_cast<double2*>(plane->ctx->b_in2.reserve(count * sizeof(double2)));
      k_widen_complex<<<unsigned((count + 255) / 256), 256, 0, s>>>(plane->buf.as<float2>(), count, wide);
      WCGH_CHECK_LAUNCH();
      WCGH_CUDA(cudaMemcpyAsync(host, wide, count * sizeof(double2), cudaMemcpyDeviceToHost, s));
    }
    sync(s);
  });
}

void* wcgh_plane_dev(wcgh_plane* plane) { return plane ? plane->buf.p : nullptr; }

int wcgh_lut_apply_blocks(wcgh_lut* lut, const uint32_t* cells, const float* w_re,
                          const float* w_im, int64_t n_cells, wcgh_plane* plane,
                          uint64_t* ops_out) {
  return guard(lut ? lut->ctx : nullptr, [&] {
    require(lut && plane && (n_cells == 0 || (cells && w_re)), "apply_block: NULL argument");
    require(n_cells >= 0, "apply_block: negative cell count");
    require(plane->ctx == lut->ctx, "apply_block: plane and LUT belong to different contexts");
    require(plane->n == lut->n, "apply_block: plane size does not match the LUT scene");
    const int n = lut->n, m = n / lut->block;
    // apply_block's range check (synthesis.cpp:149-160), then dense weights
    std::vector<float> re(size_t(m) * m, 0.0f), im;
    bool any_im = false;
    if (w_im) im.assign(size_t(m) * m, 0.0f);
    for (int64_t i = 0; i < n_cells; ++i) {
      require(cells[i] < uint32_t(m) * uint32_t(m),
              "apply_block: cell " + std::to_string(cells[i]) + " out of range");
      re[cells[i]] += w_re[i];
      if (w_im && w_im[i] != 0.0f) {
        im[cells[i]] += w_im[i];
        any_im = true;
      }
    }
    wcgh_ctx* ctx = lut->ctx;
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    float* w = static_cast<float*>(ctx->b_out.reserve(re.size() * 4));
    float2* out = plane->buf.as<float2>();
    WCGH_CUDA(cudaMemcpyAsync(w, re.data(), re.size() * 4, cudaMemcpyHostToDevice, s));
    launch_lut_dense(lut->base, n, lut->block, w, m, 0, 0, n, out, ctx->cells, ctx->lut_partial, s,
                     nullptr, /*accumulate=*/true);
    if (any_im) {  // plane += i * sum w_im S (synthesis.cpp:37-41)
      WCGH_CUDA(cudaMemcpyAsync(w, im.data(), im.size() * 4, cudaMemcpyHostToDevice, s));
      launch_lut_dense(lut->base, n, lut->block, w, m, 0, 0, n, out, ctx->cells, ctx->lut_partial,
                       s, nullptr, true, /*rotate=*/true);
    }
    sync(s);
    if (ops_out) *ops_out += uint64_t(n_cells);
  });
}

int wcgh_lut_refine(wcgh_lut* lut, const double* h, const double* v, const double* d, int m,
                    const double* saliency_finer, double threshold, wcgh_plane* plane,
                    uint8_t* mask_out, uint64_t* ops_out) {
  return guard(lut ? lut->ctx : nullptr, [&] {
    require(lut && plane && h && v && d && saliency_finer, "refine: NULL argument");
    require(plane->ctx == lut->ctx, "refine: plane and LUT belong to different contexts");
    const int n = lut->n;
    require(plane->n == n, "refine: plane size does not match the LUT scene");
    require(m >= 1, "refine: residual must be square");
    require(2 * m * lut->block == n, "refine: LUT block size does not match the residual level");
    wcgh_ctx* ctx = lut->ctx;
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    const int mr = 2 * m;
    const size_t m2 = size_t(m) * m, r2 = size_t(mr) * mr;
    char* in = static_cast<char*>(ctx->b_in.reserve((3 * m2 + r2) * 8));
    double* bands = reinterpret_cast<double*>(in);
    double* sal = bands + 3 * m2;
    WCGH_CUDA(cudaMemcpyAsync(bands, h, m2 * 8, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(bands + m2, v, m2 * 8, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(bands + 2 * m2, d, m2 * 8, cudaMemcpyHostToDevice, s));
    WCGH_CUDA(cudaMemcpyAsync(sal, saliency_finer, r2 * 8, cudaMemcpyHostToDevice, s));
    const size_t wbytes = ((r2 * 4 + 255) / 256) * 256, mbytes = ((r2 + 255) / 256) * 256;
    char* o = static_cast<char*>(ctx->b_out.reserve(wbytes + mbytes + 256));
    float* w = reinterpret_cast<float*>(o);
    uint8_t* mask = reinterpret_cast<uint8_t*>(o + wbytes);
    unsigned long long* count = reinterpret_cast<unsigned long long*>(o + wbytes + mbytes);
    WCGH_CUDA(cudaMemsetAsync(count, 0, 8, s));
    launch_refine_gate(bands, bands + m2, bands + 2 * m2, m, sal, threshold, w, mask, count, s);
    launch_lut_dense(lut->base, n, lut->block, w, mr, 0, 0, n, plane->buf.as<float2>(), ctx->cells,
                     ctx->lut_partial, s, nullptr, /*accumulate=*/true);
    unsigned long long gated = 0;
    WCGH_CUDA(cudaMemcpyAsync(&gated, count, 8, cudaMemcpyDeviceToHost, s));
    if (mask_out) WCGH_CUDA(cudaMemcpyAsync(mask_out, mask, r2, cudaMemcpyDeviceToHost, s));
    sync(s);
    if (ops_out) *ops_out += gated;
  });
}

int wcgh_job_use_lut(wcgh_job* job, int layer, const wcgh_lut* lut) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && lut, "job_use_lut: NULL argument");
    require(job->desc.method == WCGH_METHOD_LUT, "job_use_lut: the job does not use the LUT method");
    require(layer >= 0 && layer < job->desc.n_layers, "job_use_lut: layer out of range");
    require(lut->n == job->desc.plane_size, "synthesize_progressive: LUTs built for a different scene");
    require(same_scene(lut->scene, job->layers[size_t(layer)]),
            "synthesize_progressive: LUTs built for a different scene");
    require(lut->ctx->device == job->ctx->device, "job_use_lut: LUT on another device");
    int st = -1;
    const int blocks[4] = {8, 4, 2, 1};
    for (int k = 0; k < 4; ++k)
      if (blocks[k] == lut->block) st = k;
    use_device(job->ctx);
    const size_t span = size_t(2 * job->desc.plane_size - 1);
    WCGH_CUDA(cudaMemcpyAsync(job->lut_base[size_t(layer) * 4 + st], lut->base, sizeof(float2) * span * span,
                              cudaMemcpyDeviceToDevice, job->ctx->stream));
    sync(job->ctx->stream);
  });
}

}  // extern "C"

WCGH_CHK_TU(wcgh_lutobj)
