// Drop-in check: the reference's own C++ API (namespace wavecgh, reference
// headers and types) backed by integration/wavecgh_gpu.cpp + libwcgh.so,
// compared with the unmodified CPU reference (oracle/_ref, namespace
// wavecgh_ref, through its C shim). Exit code 0 = all checks passed.
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <vector>

#include "wavecgh/angular_spectrum.hpp"
#include "wavecgh/errors.hpp"
#include "wavecgh/fringe_lut.hpp"
#include "wavecgh/haar.hpp"
#include "wavecgh/saliency.hpp"
#include "wavecgh/synthesis.hpp"
#include "wavecgh_gpu.hpp"

extern "C" {
int ref_haar_analyze(const double* image, int n, int levels, double* out);
int ref_quantize_saliency(const double* sal, int n, double* out);
int ref_synthesize_progressive(const double* object, const double* saliency, int n, double wl,
                               double pitch, double z, const double* thresholds,
                               const int* enables, int workers, int use_seed, std::uint64_t seed,
                               double* planes_out, std::uint8_t* masks_out, std::uint64_t* ops_out);
int ref_synthesize_pointwise_oracle(const double* object, int n, double wl, double pitch, double z,
                                    int workers, int use_seed, std::uint64_t seed, double* out,
                                    std::uint64_t* ops);
int ref_random_phase_field(const double* amp, int n, std::uint64_t seed, double* out);
int ref_random_image(int w, int h, std::uint64_t seed, double* out);
int ref_build_block_lut(double wl, double pitch, double z, int n, int block, int workers, double* out);
int ref_reconstruct(const double* holo, int n, double wl, double pitch, double z, int intensity,
                    double* out);
int ref_apply_block(double wl, double pitch, double z, int n, int block, int cx, int cy,
                    double w_re, double w_im, double* plane, std::uint64_t* ops);
int ref_apply_block_lut(double wl, double pitch, double z, int n, int block, const double* support,
                        int cx, int cy, double w_re, double w_im, double* plane, std::uint64_t* ops);
int ref_synthesize_progressive_luts(const double* object, const double* saliency, int n, double wl,
                                    double pitch, double z, const double* thresholds,
                                    const int* enables, const double* const* supports,
                                    double* planes_out, std::uint64_t* ops_out);
}

using namespace wavecgh;

static int failures = 0;
#define EXPECT(cond, ...)                        \
  do {                                           \
    if (!(cond)) {                               \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);                  \
      std::printf("\n");                         \
      ++failures;                                \
    }                                            \
  } while (0)

static RealImage random_image(int n, std::uint64_t seed) {
  std::vector<double> v(std::size_t(n) * n);
  ref_random_image(n, n, seed, v.data());
  return RealImage(n, n, std::move(v));
}

static double rel_l2(const ComplexField& a, const double* ref) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const std::complex<double> r(ref[2 * i], ref[2 * i + 1]);
    num += std::norm(a.data()[i] - r);
    den += std::norm(r);
  }
  return std::sqrt(num / den);
}

int main() {
  const double wl = 532e-9, pitch = 8e-6, z = 0.1;
  for (int n : {16, 32, 64}) {
    const RealImage object = random_image(n, 900 + n);
    const RealImage saliency = random_image(n, 77 + n);
    // haar_analyze and quantize_saliency: bit-identical
    const HaarPyramid p = haar_analyze(object, 3);
    std::vector<double> ref(std::size_t(n) * n * 2);
    ref_haar_analyze(object.data().data(), n, 3, ref.data());
    bool same = std::memcmp(p.approx.data().data(), ref.data(), p.approx.size() * 8) == 0;
    std::size_t o = p.approx.size();
    for (const auto& b : p.details)
      for (const RealImage* im : {&b.h, &b.v, &b.d}) {
        same = same && std::memcmp(im->data().data(), ref.data() + o, im->size() * 8) == 0;
        o += im->size();
      }
    EXPECT(same, "haar_analyze n=%d not bit-identical", n);
    const SaliencyPyramid sp = quantize_saliency(saliency);
    ref_quantize_saliency(saliency.data().data(), n, ref.data());
    same = std::memcmp(sp.by_factor(2).data().data(), ref.data(), std::size_t(n) * n / 4 * 8) == 0 &&
           std::memcmp(sp.by_factor(4).data().data(), ref.data() + n * n / 4, std::size_t(n) * n / 16 * 8) == 0;
    EXPECT(same, "quantize_saliency n=%d not bit-identical", n);

    // synthesize_progressive: all four stages, masks, operator counts
    const SceneParams scene = make_scene(wl, pitch, z, n);
    const LutSet luts = LutSet::build(scene);
    const RefinementPlan plan;
    const ProgressiveResult r = synthesize_progressive(object, saliency, scene, plan, luts);
    std::vector<double> planes(std::size_t(8) * n * n);
    std::vector<std::uint8_t> masks(std::size_t(n) * n * 21 / 16);
    std::uint64_t ops[5];
    const double th[3] = {plan.t_ll, plan.t_l, plan.t_full};
    const int en[3] = {1, 1, 1};
    ref_synthesize_progressive(object.data().data(), saliency.data().data(), n, wl, pitch, z, th, en,
                               1, 0, 0, planes.data(), masks.data(), ops);
    for (int s = 0; s < 4; ++s) {
      const double e = rel_l2(r.stage(s), planes.data() + std::size_t(2) * n * n * s);
      EXPECT(e <= 1e-4, "synthesize_progressive n=%d stage %d rel L2 %.3e", n, s, e);
    }
    EXPECT(std::memcmp(r.mask_ll.on.data(), masks.data(), r.mask_ll.on.size()) == 0, "mask_ll n=%d", n);
    EXPECT(std::memcmp(r.mask_full.on.data(), masks.data() + n * n / 16 + n * n / 4, r.mask_full.on.size()) == 0,
           "mask_full n=%d", n);
    for (int i = 0; i < 5; ++i)
      EXPECT(r.ops.get(kAllOpLevels[i]) == ops[i], "ops[%d] n=%d: %llu vs %llu", i, n,
             (unsigned long long)r.ops.get(kAllOpLevels[i]), (unsigned long long)ops[i]);

    // point-wise oracle
    OpCounter pc;
    const ComplexField pw = synthesize_pointwise_oracle(object, scene, pc, luts.of(1));
    std::uint64_t pops = 0;
    ref_synthesize_pointwise_oracle(object.data().data(), n, wl, pitch, z, 1, 0, 0, planes.data(), &pops);
    EXPECT(rel_l2(pw, planes.data()) <= 1e-4, "pointwise oracle n=%d", n);
    EXPECT(pc.get(OpLevel::kPointwiseOracle) == pops, "pointwise ops n=%d", n);

    // random initial phase (synthesis.cpp:205-219, 269-284, 288-296)
    const std::uint64_t seed = 424242 + n;
    const ComplexField rot = random_phase_field(object, seed);
    std::vector<double> rref(std::size_t(2) * n * n);
    ref_random_phase_field(object.data().data(), n, seed, rref.data());
    EXPECT(std::memcmp(rot.data().data(), rref.data(), rref.size() * 8) == 0,
           "random_phase_field n=%d not bit-identical", n);
    const ProgressiveResult rp = synthesize_progressive(object, saliency, scene, plan, luts, 1, seed);
    ref_synthesize_progressive(object.data().data(), saliency.data().data(), n, wl, pitch, z, th, en,
                               1, 1, seed, planes.data(), masks.data(), ops);
    for (int s = 0; s < 4; ++s) {
      const double e = rel_l2(rp.stage(s), planes.data() + std::size_t(2) * n * n * s);
      EXPECT(e <= 1e-4, "random phase n=%d stage %d rel L2 %.3e", n, s, e);
    }
    for (int i = 0; i < 5; ++i) EXPECT(rp.ops.get(kAllOpLevels[i]) == ops[i], "random phase ops[%d] n=%d", i, n);
    OpCounter pc2;
    const ComplexField pw2 = synthesize_pointwise_oracle(object, scene, pc2, luts.of(1), 1, seed);
    ref_synthesize_pointwise_oracle(object.data().data(), n, wl, pitch, z, 1, 1, seed, planes.data(), &pops);
    EXPECT(rel_l2(pw2, planes.data()) <= 1e-4, "pointwise oracle (random phase) n=%d", n);
    EXPECT(pc2.get(OpLevel::kPointwiseOracle) == pops, "pointwise ops (random phase) n=%d", n);

    // apply_block with a complex weight (synthesis.cpp:37-41)
    ComplexField plane(n, n);
    OpCounter ac;
    apply_block(plane, luts.of(2), GridCell{1, 2}, {0.3, -0.7}, ac, OpLevel::kRefineL);
    std::vector<double> pl(std::size_t(2) * n * n, 0.0);
    std::uint64_t aops = 0;
    ref_apply_block(wl, pitch, z, n, 2, 1, 2, 0.3, -0.7, pl.data(), &aops);
    EXPECT(rel_l2(plane, pl.data()) <= 1e-5, "apply_block complex weight n=%d", n);
    EXPECT(ac.get(OpLevel::kRefineL) == 1, "apply_block count");

    // the CALLER's LUT samples are what the GPU superposes (synthesis.cpp:
    // 18-42 reads lut.support()): one perturbed sample of a caller-built
    // FringeLut moves exactly one pixel by w * delta, as in the reference
    {
      const int span = 2 * n - 1;
      ComplexField sup = luts.of(2).support();
      const int dx = 3, dy = -2, cx = 1, cy = 2;
      const std::complex<double> delta(0.37, -0.21), w(0.8, 0.25);
      sup.at(dx + n - 1, dy + n - 1) += delta;
      const FringeLut pert(scene, 2, sup);
      ComplexField p0(n, n), p1(n, n);
      OpCounter oc;
      apply_block(p0, luts.of(2), GridCell{cx, cy}, w, oc, OpLevel::kRefineL);
      apply_block(p1, pert, GridCell{cx, cy}, w, oc, OpLevel::kRefineL);
      std::vector<double> r1(std::size_t(2) * n * n, 0.0);
      std::uint64_t o1 = 0;
      ref_apply_block_lut(wl, pitch, z, n, 2, reinterpret_cast<const double*>(sup.data().data()), cx, cy,
                          w.real(), w.imag(), r1.data(), &o1);
      EXPECT(rel_l2(p1, r1.data()) <= 1e-5, "apply_block with a caller-modified LUT n=%d", n);
      int moved = 0;
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x)
          if (p1.at(x, y) != p0.at(x, y)) {
            ++moved;
            EXPECT(x == cx * 2 + dx && y == cy * 2 + dy, "perturbed LUT moved pixel (%d,%d)", x, y);
            // complex64 device samples: each plane rounded at the sample's magnitude
            EXPECT(std::abs(p1.at(x, y) - p0.at(x, y) - w * delta) <=
                       4e-7 * std::abs(w) * std::abs(sup.at(dx + n - 1, dy + n - 1)) + 1e-7,
                   "perturbed LUT delta n=%d", n);
          }
      EXPECT(moved == 1, "perturbed LUT sample must move exactly one pixel (moved %d)", moved);
      (void)span;
      // synthesize_progressive with a caller LutSet whose B=1 LUT is modified
      LutSet mod = luts;
      ComplexField s1 = luts.of(1).support();
      s1.at(n - 1, n - 1) += std::complex<double>(0.05, 0.02);
      mod.put(FringeLut(scene, 1, s1));
      const ProgressiveResult rm = synthesize_progressive(object, saliency, scene, plan, mod);
      std::vector<const double*> sp;
      for (int b : {1, 2, 4, 8}) sp.push_back(reinterpret_cast<const double*>(mod.of(b).support().data().data()));
      const double th[3] = {plan.t_ll, plan.t_l, plan.t_full};
      const int en[3] = {1, 1, 1};
      std::vector<double> rp(std::size_t(8) * n * n);
      std::uint64_t rops[5] = {};
      ref_synthesize_progressive_luts(object.data().data(), saliency.data().data(), n, wl, pitch, z, th, en,
                                      sp.data(), rp.data(), rops);
      for (int st = 0; st < 4; ++st)
        EXPECT(rel_l2(rm.stage(st), rp.data() + std::size_t(2) * st * n * n) <= 1e-5,
               "synthesize_progressive with a caller-modified LutSet stage %d n=%d", st, n);
    }
  }
  // fringe_lut.cpp on the device: build_block_lut vs the reference's fp64 LUT
  // (complex64 precision), CGHL round trip through the reference's format
  {
    const SceneParams scene = make_scene(wl, pitch, z, 32);
    for (int b : {1, 2, 4, 8}) {
      const FringeLut g = build_block_lut(scene, b);
      std::vector<double> ref(std::size_t(2) * 63 * 63);
      ref_build_block_lut(wl, pitch, z, 32, b, 1, ref.data());
      double md = 0, mr = 0;
      for (std::size_t i = 0; i < g.support().size(); ++i) {
        const std::complex<double> r(ref[2 * i], ref[2 * i + 1]);
        md = std::max(md, std::abs(g.support().data()[i] - r));
        mr = std::max(mr, std::abs(r));
      }
      EXPECT(md <= 2e-7 * mr, "build_block_lut b=%d max rel %.3e", b, md / mr);
      EXPECT(std::abs(g.at_offset(0, 0) - g.support().at(31, 31)) == 0.0, "at_offset");
    }
    const FringeLut l2 = build_block_lut(scene, 2);
    const std::string path = "/tmp/dropin_lut_b2.cghl";
    lut_cache_store(l2, path);
    const FringeLut back = lut_cache_load(path, scene, 2);
    bool same = true;
    for (std::size_t i = 0; i < l2.support().size(); ++i) same = same && back.support().data()[i] == l2.support().data()[i];
    EXPECT(same, "lut cache round trip");
    bool stale = false;
    try {
      lut_cache_load(path, scene, 4);
    } catch (const StaleCacheError&) {
      stale = true;
    }
    EXPECT(stale, "lut cache block mismatch must throw StaleCacheError");
    const LutSet set = LutSet::build(scene);
    EXPECT(set.has(1) && set.has(8) && set.of(4).block_size() == 4, "LutSet");
  }
  // explicit-method overload and the layered (multi-depth) entry (wavecgh_gpu.hpp)
  {
    const int n = 64;
    const double th[3] = {0.5, 0.7, 0.9};
    const int en[3] = {1, 1, 1};
    std::vector<double> planes(std::size_t(8) * n * n), sum(std::size_t(8) * n * n, 0.0);
    std::vector<std::uint8_t> masks(std::size_t(n) * n * 21 / 16);
    std::uint64_t ops[5], ops_sum[5] = {0, 0, 0, 0, 0};
    std::vector<RealImage> objs, sals;
    std::vector<SceneParams> scenes;
    for (int l = 0; l < 2; ++l) {
      const double zl = 0.05 + 0.03 * l;
      objs.push_back(random_image(n, 300 + l));
      sals.push_back(random_image(n, 400 + l));
      scenes.push_back(make_scene(wl, pitch, zl, n));
      ref_synthesize_progressive(objs[l].data().data(), sals[l].data().data(), n, wl, pitch, zl, th,
                                 en, 1, 0, 0, planes.data(), masks.data(), ops);
      for (std::size_t i = 0; i < planes.size(); ++i) sum[i] += planes[i];
      for (int i = 0; i < 5; ++i) ops_sum[i] += ops[i];
      if (l == 0) {
        for (SynthesisMethod m : {SynthesisMethod::kLut, SynthesisMethod::kDirect, SynthesisMethod::kFft}) {
          const ProgressiveResult r = synthesize_progressive(objs[0], sals[0], scenes[0], RefinementPlan{}, m);
          for (int st = 0; st < 4; ++st) {
            const double e = rel_l2(r.stage(st), planes.data() + std::size_t(2) * n * n * st);
            EXPECT(e <= 1e-4, "method %d stage %d rel L2 %.3e", int(m), st, e);
          }
          for (int i = 0; i < 5; ++i) EXPECT(r.ops.get(kAllOpLevels[i]) == ops[i], "method %d ops[%d]", int(m), i);
        }
      }
    }
    for (SynthesisMethod m : {SynthesisMethod::kLut, SynthesisMethod::kDirect, SynthesisMethod::kFft}) {
      const ProgressiveResult r = synthesize_progressive_layered(objs, sals, scenes, RefinementPlan{}, m);
      for (int st = 0; st < 4; ++st) {
        const double e = rel_l2(r.stage(st), sum.data() + std::size_t(2) * n * n * st);
        EXPECT(e <= 1e-4, "layered method %d stage %d rel L2 %.3e", int(m), st, e);
      }
      for (int i = 0; i < 5; ++i) EXPECT(r.ops.get(kAllOpLevels[i]) == ops_sum[i], "layered ops[%d]", i);
    }
  }
  // reconstruct of a synthesised hologram (angular_spectrum.cpp:47-61), fp64 on the device
  {
    const int n = 64;
    const SceneParams scene = make_scene(wl, pitch, z, n);
    const LutSet luts = LutSet::build(scene);
    const ProgressiveResult r =
        synthesize_progressive(random_image(n, 5), random_image(n, 6), scene, RefinementPlan{}, luts);
    for (bool inten : {false, true}) {
      const RealImage img = reconstruct(r.after_full, scene, inten);
      std::vector<double> ref(std::size_t(n) * n);
      ref_reconstruct(reinterpret_cast<const double*>(r.after_full.data().data()), n, wl, pitch, z,
                      inten ? 1 : 0, ref.data());
      double md = 0, mr = 0;
      for (std::size_t i = 0; i < ref.size(); ++i) {
        md = std::max(md, std::abs(img.data()[i] - ref[i]));
        mr = std::max(mr, std::abs(ref[i]));
      }
      EXPECT(md <= 1e-11 * mr, "reconstruct intensity=%d max rel %.3e", int(inten), md / mr);
    }
    const PropagationKernel k = build_kernel(scene, -z);
    const ComplexField back = propagate(propagate(r.after_full, build_kernel(scene, z)), k);
    double md = 0, mr = 0;
    for (std::size_t i = 0; i < back.size(); ++i) {
      md = std::max(md, std::abs(back.data()[i] - r.after_full.data()[i]));
      mr = std::max(mr, std::abs(r.after_full.data()[i]));
    }
    EXPECT(md <= 1e-10 * mr, "propagate round trip %.3e", md / mr);
    bool threw = false;
    try {
      build_kernel(scene, 0.0);
    } catch (const ValidationError&) {
      threw = true;
    }
    EXPECT(threw, "build_kernel(0) must throw ValidationError");
  }
  // validation behaviour (synthesis.cpp:184-202)
  {
    const SceneParams scene = make_scene(wl, pitch, z, 16);
    const LutSet luts = LutSet::build(scene);
    bool threw = false;
    try {
      synthesize_progressive(random_image(8, 1), uniform_saliency(8), scene, RefinementPlan{}, luts);
    } catch (const ValidationError&) {
      threw = true;
    }
    EXPECT(threw, "size mismatch must throw ValidationError");
    threw = false;
    RealImage bad(16, 16);
    bad.at(1, 1) = 1.5;
    try {
      quantize_saliency(bad);
    } catch (const ValidationError&) {
      threw = true;
    }
    EXPECT(threw, "saliency out of range must throw ValidationError");
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
