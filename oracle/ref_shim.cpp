// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference sources (wavecgh 0.1.0,
// /root/reference/proj), compiled by oracle/Makefile with
// -Dwavecgh=wavecgh_ref into oracle/_ref/libwavecgh_ref.so. It lets the
// pytest suite and bench.py's reference arm call the reference's own public
// functions through ctypes. Every entry returns 0 on success, 1 for
// ValidationError, 2 for IoError/other (the reference CLI's exit codes,
// tools/wavecgh_main.cpp:167-179) and leaves the message in ref_last_error().
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs may load this library.

#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "support/oracles.hpp"
#include "wavecgh/angular_spectrum.hpp"
#include "wavecgh/errors.hpp"
#include "wavecgh/fringe_lut.hpp"
#include "wavecgh/haar.hpp"
#include "wavecgh/metrics.hpp"
#include "wavecgh/parallel.hpp"
#include "wavecgh/saliency.hpp"
#include "wavecgh/synthesis.hpp"

using namespace wavecgh;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

RealImage real_in(const double* p, int n) {
  return RealImage(n, n, std::vector<double>(p, p + std::size_t(n) * n));
}

void complex_out(const ComplexField& f, double* out) {
  std::memcpy(out, f.data().data(), f.size() * sizeof(std::complex<double>));
}

void real_out(const RealImage& im, double* out) {
  std::memcpy(out, im.data().data(), im.size() * sizeof(double));
}

ComplexField support_in(const double* p, std::size_t span) {
  const int w = static_cast<int>(span);
  ComplexField f(w, w);
  std::memcpy(f.data().data(), p, span * span * sizeof(std::complex<double>));
  return f;
}

RefinementPlan plan_of(const double* t, const int* en) {
  RefinementPlan plan;
  plan.t_ll = t[0];
  plan.t_l = t[1];
  plan.t_full = t[2];
  plan.enable_ll = en[0] != 0;
  plan.enable_l = en[1] != 0;
  plan.enable_full = en[2] != 0;
  return plan;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_default_worker_count() { return default_worker_count(); }

// haar_analyze (haar.cpp:52-74). Output layout: approx (n>>L)^2 then, for
// level l = 0..L-1 (finest first), h, v, d each (n>>(l+1))^2.
int ref_haar_analyze(const double* image, int n, int levels, double* out) {
  return guard([&] {
    const HaarPyramid p = haar_analyze(real_in(image, n), levels);
    real_out(p.approx, out);
    out += p.approx.size();
    for (const auto& b : p.details) {
      real_out(b.h, out);
      out += b.h.size();
      real_out(b.v, out);
      out += b.v.size();
      real_out(b.d, out);
      out += b.d.size();
    }
  });
}

// expand_residual (haar.cpp:88-96): m x m bands -> (2m)^2.
int ref_expand_residual(const double* h, const double* v, const double* d, int m,
                        double* out) {
  return guard([&] { real_out(expand_residual(real_in(h, m), real_in(v, m), real_in(d, m)), out); });
}

// upsample_replicate (haar.cpp:98-109).
int ref_upsample_replicate(const double* coarse, int m, int factor, double* out) {
  return guard([&] { real_out(upsample_replicate(real_in(coarse, m), factor), out); });
}

// quantize_saliency (saliency.cpp:41-61): out = half, quarter, eighth maps.
int ref_quantize_saliency(const double* sal, int n, double* out) {
  return guard([&] {
    const SaliencyPyramid p = quantize_saliency(real_in(sal, n));
    for (int f : {2, 4, 8}) {
      real_out(p.by_factor(f), out);
      out += p.by_factor(f).size();
    }
  });
}

// point_fringe (fringe_lut.cpp:27-32).
int ref_point_fringe(double wl, double pitch, double z, int n, int dx, int dy, double* out2) {
  return guard([&] {
    const auto v = point_fringe(make_scene(wl, pitch, z, n), dx, dy);
    out2[0] = v.real();
    out2[1] = v.imag();
  });
}

// build_block_lut (fringe_lut.cpp:53-93): out = (2n-1)^2 complex<double>.
int ref_build_block_lut(double wl, double pitch, double z, int n, int block, int workers,
                        double* out) {
  return guard([&] {
    complex_out(build_block_lut(make_scene(wl, pitch, z, n), block, workers).support(), out);
  });
}

// lut_cache_store (fringe_lut.cpp:95-115): the reference's CGHL file of a
// freshly built LUT.
int ref_lut_cache_store(const char* path, double wl, double pitch, double z, int n, int block) {
  return guard([&] { lut_cache_store(build_block_lut(make_scene(wl, pitch, z, n), block, 0), path); });
}

// apply_block (synthesis.cpp:149-160) on a caller plane with a freshly built LUT.
int ref_apply_block(double wl, double pitch, double z, int n, int block, int cx, int cy,
                    double w_re, double w_im, double* plane, std::uint64_t* ops) {
  return guard([&] {
    const SceneParams scene = make_scene(wl, pitch, z, n);
    const FringeLut lut = build_block_lut(scene, block, 0);
    ComplexField p(n, n);
    std::memcpy(p.data().data(), plane, p.size() * sizeof(std::complex<double>));
    OpCounter counter;
    apply_block(p, lut, GridCell{cx, cy}, {w_re, w_im}, counter, OpLevel::kRefineFull);
    complex_out(p, plane);
    *ops = counter.get(OpLevel::kRefineFull);
  });
}

// apply_block with the CALLER's LUT samples: FringeLut(scene, block, support)
// (fringe_lut.cpp:34-51) from a (2n-1)^2 complex<double> array.
int ref_apply_block_lut(double wl, double pitch, double z, int n, int block,
                        const double* support, int cx, int cy, double w_re, double w_im,
                        double* plane, std::uint64_t* ops) {
  return guard([&] {
    const SceneParams scene = make_scene(wl, pitch, z, n);
    const std::size_t span = std::size_t(2 * n - 1);
    const FringeLut lut(scene, block, support_in(support, span));
    ComplexField p(n, n);
    std::memcpy(p.data().data(), plane, p.size() * sizeof(std::complex<double>));
    OpCounter counter;
    apply_block(p, lut, GridCell{cx, cy}, {w_re, w_im}, counter, OpLevel::kRefineFull);
    complex_out(p, plane);
    *ops = counter.get(OpLevel::kRefineFull);
  });
}

// synthesize_progressive with a CALLER LutSet: supports[k] = the (2n-1)^2
// complex<double> samples of block 1, 2, 4, 8 (k = 0..3).
int ref_synthesize_progressive_luts(const double* object, const double* saliency, int n,
                                    double wl, double pitch, double z, const double* thresholds,
                                    const int* enables, const double* const* supports,
                                    double* planes_out, std::uint64_t* ops_out) {
  return guard([&] {
    const SceneParams scene = make_scene(wl, pitch, z, n);
    const std::size_t span = std::size_t(2 * n - 1);
    LutSet luts;
    const int blocks[4] = {1, 2, 4, 8};
    for (int k = 0; k < 4; ++k) {
      luts.put(FringeLut(scene, blocks[k], support_in(supports[k], span)));
    }
    const ProgressiveResult r = synthesize_progressive(real_in(object, n), real_in(saliency, n), scene,
                                                       plan_of(thresholds, enables), luts, 0);
    for (int i = 0; i < 4; ++i) complex_out(r.stage(i), planes_out + 2 * std::size_t(i) * n * n);
    for (int i = 0; i < kOpLevelCount; ++i) ops_out[i] = r.ops.get(kAllOpLevels[i]);
  });
}

// synthesize_progressive (synthesis.cpp:180-253) with LutSet::build
// (fringe_lut.cpp:165-169). planes_out: 4 x n^2 complex<double> (base,
// after_ll, after_l, after_full) or NULL; masks_out: (n/4)^2 + (n/2)^2 + n^2
// bytes or NULL; ops_out[5] per OpLevel.
int ref_synthesize_progressive(const double* object, const double* saliency, int n, double wl,
                               double pitch, double z, const double* thresholds,
                               const int* enables, int workers, int use_seed,
                               std::uint64_t seed, double* planes_out,
                               std::uint8_t* masks_out, std::uint64_t* ops_out) {
  return guard([&] {
    const SceneParams scene = make_scene(wl, pitch, z, n);
    const LutSet luts = LutSet::build(scene, workers);
    std::optional<std::uint64_t> s;
    if (use_seed) s = seed;
    const ProgressiveResult r =
        synthesize_progressive(real_in(object, n), real_in(saliency, n), scene,
                               plan_of(thresholds, enables), luts, workers, s);
    if (planes_out) {
      for (int i = 0; i < 4; ++i) complex_out(r.stage(i), planes_out + 2 * std::size_t(i) * n * n);
    }
    if (masks_out) {
      for (const GateMask* m : {&r.mask_ll, &r.mask_l, &r.mask_full}) {
        std::memcpy(masks_out, m->on.data(), m->on.size());
        masks_out += m->on.size();
      }
    }
    for (int i = 0; i < kOpLevelCount; ++i) ops_out[i] = r.ops.get(kAllOpLevels[i]);
  });
}

// synthesize_pointwise_oracle (synthesis.cpp:255-286), optional random phase seed.
int ref_synthesize_pointwise_oracle(const double* object, int n, double wl, double pitch,
                                    double z, int workers, int use_seed, std::uint64_t seed,
                                    double* out, std::uint64_t* ops) {
  return guard([&] {
    const SceneParams scene = make_scene(wl, pitch, z, n);
    const FringeLut unit = build_block_lut(scene, 1, workers);
    OpCounter counter;
    std::optional<std::uint64_t> s;
    if (use_seed) s = seed;
    complex_out(synthesize_pointwise_oracle(real_in(object, n), scene, counter, unit, workers, s),
                out);
    *ops = counter.get(OpLevel::kPointwiseOracle);
  });
}

// Direct Eq.(1) double loop from the reference's own test oracle
// (tests/support/oracles.cpp:12-50). amp_im may be NULL (real amplitudes).
int ref_pointwise_hologram_reference(const double* amp_re, const double* amp_im, int n,
                                     double wl, double pitch, double z, double* out) {
  return guard([&] {
    const SceneParams scene = make_scene(wl, pitch, z, n);
    if (!amp_im) {
      complex_out(testing::pointwise_hologram_reference(real_in(amp_re, n), scene), out);
      return;
    }
    ComplexField a(n, n);
    for (std::size_t i = 0; i < a.size(); ++i) a.data()[i] = {amp_re[i], amp_im[i]};
    complex_out(testing::pointwise_hologram_reference(a, scene), out);
  });
}

// random_image (tests/support/oracles.cpp:139-145): mt19937_64 uniform [0,1).
int ref_random_image(int w, int h, std::uint64_t seed, double* out) {
  return guard([&] {
    const RealImage im = testing::random_image(w, h, seed);
    std::memcpy(out, im.data().data(), im.size() * sizeof(double));
  });
}

// random_phase_field (synthesis.cpp:288-296).
int ref_random_phase_field(const double* amp, int n, std::uint64_t seed, double* out) {
  return guard([&] { complex_out(random_phase_field(real_in(amp, n), seed), out); });
}

// reconstruct (angular_spectrum.cpp:46-61).
int ref_reconstruct(const double* holo, int n, double wl, double pitch, double z,
                    int intensity, double* out) {
  return guard([&] {
    ComplexField h(n, n);
    std::memcpy(h.data().data(), holo, h.size() * sizeof(std::complex<double>));
    real_out(reconstruct(h, make_scene(wl, pitch, z, n), intensity != 0), out);
  });
}

// ssim (metrics.cpp:50-85).
int ref_ssim(const double* a, const double* b, int n, int window, double k1, double k2,
             double dynamic_range, double* out) {
  return guard([&] { *out = ssim(real_in(a, n), real_in(b, n), window, k1, k2, dynamic_range); });
}

// ---------------------------------------------------------------------------
// Bounded timing sample for the CPU baseline (bench.py only).
//
// Runs the reference's own multi-threaded refine() (synthesis.cpp:171-178 ->
// refine_stage -> apply_cells -> accumulate_deterministic, parallel.cpp:49-98)
// with a LUT of block size `block` on `count` real cells whose weights are
// the given residual values, and returns the wall time in seconds. The
// residual bands are given as (h,v,d) of size m = n/block/2... callers pass
// the expanded residual directly via a saliency map that gates exactly the
// sampled cells, so the reference code path is unchanged.
struct RefLutCache {
  SceneParams scene;
  LutSet luts;
};

void* ref_lutset_build(double wl, double pitch, double z, int n, int workers) {
  RefLutCache* c = nullptr;
  const int rc = guard([&] {
    const SceneParams scene = make_scene(wl, pitch, z, n);
    c = new RefLutCache{scene, LutSet::build(scene, workers)};
  });
  return rc == 0 ? c : nullptr;
}

void ref_lutset_free(void* h) { delete static_cast<RefLutCache*>(h); }

// Times refine() on detail bands (h, v, d; m x m each, so the residual and
// gate grid are 2m x 2m with block size n / (2m)) gated by `gate_map`
// (2m x 2m saliency in [0,1]) at threshold t. Returns seconds in *secs and
// the operator count in *ops.
int ref_time_refine(void* h, const double* bh, const double* bv, const double* bd, int m,
                    const double* gate_map, double t, int workers, double* secs,
                    std::uint64_t* ops) {
  return guard([&] {
    auto* c = static_cast<RefLutCache*>(h);
    const int n = c->scene.plane_size();
    const int block = n / (2 * m);
    ComplexField plane(n, n);
    OpCounter counter;
    const auto t0 = std::chrono::steady_clock::now();
    refine(plane, real_in(bh, m), real_in(bv, m), real_in(bd, m), real_in(gate_map, 2 * m),
           c->luts.of(block), t, counter, OpLevel::kRefineFull, nullptr, workers);
    const auto t1 = std::chrono::steady_clock::now();
    *secs = std::chrono::duration<double>(t1 - t0).count();
    *ops = counter.get(OpLevel::kRefineFull);
  });
}

// Full synthesize_progressive timing with a prebuilt LutSet (bench.py only).
int ref_time_progressive(void* h, const double* object, const double* saliency,
                         const double* thresholds, const int* enables, int workers,
                         double* secs, double* after_full_out, std::uint64_t* ops_out) {
  return guard([&] {
    auto* c = static_cast<RefLutCache*>(h);
    const int n = c->scene.plane_size();
    const auto t0 = std::chrono::steady_clock::now();
    const ProgressiveResult r =
        synthesize_progressive(real_in(object, n), real_in(saliency, n), c->scene,
                               plan_of(thresholds, enables), c->luts, workers);
    const auto t1 = std::chrono::steady_clock::now();
    *secs = std::chrono::duration<double>(t1 - t0).count();
    if (after_full_out) complex_out(r.after_full, after_full_out);
    for (int i = 0; i < kOpLevelCount; ++i) ops_out[i] = r.ops.get(kAllOpLevels[i]);
  });
}

}  // extern "C"
