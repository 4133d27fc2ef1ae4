// The reference's small validation helpers on the device, so the drop-in and
// the Python mirror run no hot-path-adjacent host arithmetic (north_star: no
// CPU fallback): haar_synthesize (haar.cpp:76-86 over synthesize_level,
// haar.cpp:32-48), upsample_replicate (haar.cpp:98-109), point_fringe
// (fringe_lut.cpp:27-32). fp64 in the reference's operation order with
// explicit round-to-nearest intrinsics (no contraction), so the first two are
// bit-identical and point_fringe differs only by the device sin/cos (<= 2 ulp).
#include "wcgh_state.cuh"

using namespace wcgh;
using namespace wcgh::abi;

namespace {

// synthesize_level: out(2x+sx, 2y+sy) from a(x,y) and the three details,
// evaluated left to right like the reference (av +- h +- v +- d).
__global__ void k_synthesize_level(const double* __restrict__ a, const double* __restrict__ h,
                                   const double* __restrict__ v, const double* __restrict__ d,
                                   int m, double* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= size_t(m) * m) return;
  const int x = int(i % m), y = int(i / m);
  const size_t n = size_t(2 * m);
  const double av = a[i], hv = h[i], vv = v[i], dv = d[i];
  out[size_t(2 * y) * n + 2 * x] = __dadd_rn(__dadd_rn(__dadd_rn(av, hv), vv), dv);
  out[size_t(2 * y) * n + 2 * x + 1] = __dsub_rn(__dadd_rn(__dsub_rn(av, hv), vv), dv);
  out[size_t(2 * y + 1) * n + 2 * x] = __dsub_rn(__dsub_rn(__dadd_rn(av, hv), vv), dv);
  out[size_t(2 * y + 1) * n + 2 * x + 1] = __dadd_rn(__dsub_rn(__dsub_rn(av, hv), vv), dv);
}

__global__ void k_upsample(const double* __restrict__ c, int w, int h, int f, double* __restrict__ out) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t W = size_t(w) * f;
  if (i >= W * size_t(h) * f) return;
  const size_t x = i % W, y = i / W;
  out[i] = c[(y / f) * w + x / f];
}

__global__ void k_point_fringe(double pitch, double z, double k, int dx, int dy, double* __restrict__ out) {
  const double px = __dmul_rn(double(dx), pitch);
  const double py = __dmul_rn(double(dy), pitch);
  const double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)), __dmul_rn(z, z)));
  const double rho = __ddiv_rn(1.0, r);
  double s, c;
  sincos(__dmul_rn(k, r), &s, &c);
  out[0] = __dmul_rn(rho, c);
  out[1] = __dmul_rn(rho, s);
}

}  // namespace

extern "C" {

int wcgh_haar_synthesize(wcgh_ctx* ctx, const double* pyramid, int n, int levels, double* out) {
  return guard(ctx, [&] {
    require(ctx && pyramid && out, "haar_synthesize: NULL argument");
    require(levels >= 1, "haar_synthesize: empty pyramid");
    require(n >= 1 && n % (1 << levels) == 0, "haar_synthesize: subband sizes inconsistent");
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    // layout of wcgh_haar_analyze: approx (n>>L)^2, then (h, v, d) per level, finest first
    size_t len = 0;
    for (int l = 0; l < levels; ++l) len += 3 * size_t(n >> (l + 1)) * size_t(n >> (l + 1));
    len += size_t(n >> levels) * size_t(n >> levels);
    const size_t n2 = size_t(n) * n;
    char* buf = static_cast<char*>(ctx->b_in.reserve(8 * (len + 2 * n2)));
    double* pyr = reinterpret_cast<double*>(buf);
    double* cur = pyr + len;
    double* nxt = cur + n2;
    WCGH_CUDA(cudaMemcpyAsync(pyr, pyramid, 8 * len, cudaMemcpyHostToDevice, s));
    const int ma = n >> levels;
    WCGH_CUDA(cudaMemcpyAsync(cur, pyr, 8 * size_t(ma) * ma, cudaMemcpyDeviceToDevice, s));
    // detail offsets, finest (level 0) first
    std::vector<size_t> off(levels);
    size_t o = size_t(ma) * ma;
    for (int l = 0; l < levels; ++l) {
      off[l] = o;
      o += 3 * size_t(n >> (l + 1)) * size_t(n >> (l + 1));
    }
    for (int l = levels - 1; l >= 0; --l) {  // coarsest detail first (details.rbegin())
      const int m = n >> (l + 1);
      const size_t mm = size_t(m) * m;
      const double* h = pyr + off[l];
      k_synthesize_level<<<unsigned((mm + 255) / 256), 256, 0, s>>>(cur, h, h + mm, h + 2 * mm, m, nxt);
      WCGH_CHECK_LAUNCH();
      std::swap(cur, nxt);
    }
    WCGH_CUDA(cudaMemcpyAsync(out, cur, 8 * n2, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_upsample_replicate(wcgh_ctx* ctx, const double* coarse, int width, int height, int factor,
                            double* out) {
  return guard(ctx, [&] {
    require(ctx && coarse && out, "upsample_replicate: NULL argument");
    require(factor >= 2 && is_pow2(factor), "upsample_replicate: factor must be a power of two >= 2");
    require(width >= 0 && height >= 0, "upsample_replicate: negative size");
    const size_t nc = size_t(width) * height, no = nc * size_t(factor) * factor;
    if (no == 0) return;
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    char* buf = static_cast<char*>(ctx->b_in.reserve(8 * (nc + no)));
    double* c = reinterpret_cast<double*>(buf);
    double* o = c + nc;
    WCGH_CUDA(cudaMemcpyAsync(c, coarse, 8 * nc, cudaMemcpyHostToDevice, s));
    k_upsample<<<unsigned((no + 255) / 256), 256, 0, s>>>(c, width, height, factor, o);
    WCGH_CHECK_LAUNCH();
    WCGH_CUDA(cudaMemcpyAsync(out, o, 8 * no, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_point_fringe(wcgh_ctx* ctx, const wcgh_layer* scene, int dx, int dy, double* out2) {
  return guard(ctx, [&] {
    require(ctx && scene && out2, "point_fringe: NULL argument");
    validate_layer(*scene);
    std::lock_guard<std::mutex> lk(ctx->mu);
    use_device(ctx);
    cudaStream_t s = ctx->stream;
    double* d = static_cast<double*>(ctx->b_misc.reserve(64));
    const double k = 2.0 * 3.141592653589793238462643383279502884 / scene->wavelength;
    k_point_fringe<<<1, 1, 0, s>>>(scene->pitch, scene->z, k, dx, dy, d);
    WCGH_CHECK_LAUNCH();
    WCGH_CUDA(cudaMemcpyAsync(out2, d, 16, cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

}  // extern "C"

WCGH_CHK_TU(wcgh_helpers)
