// Extensions of the reference API provided by the GPU drop-in
// (integration/wavecgh_gpu.cpp): the synthesis method as an
// explicit argument (one algorithm choice per call, not a backend dispatch)
// and a layered entry for multi-depth scenes. Everything else keeps the
// reference's own declarations (wavecgh/synthesis.hpp etc.).
#pragma once

#include <vector>

#include "wavecgh/synthesis.hpp"

namespace wavecgh {

enum class SynthesisMethod {
  kLut,     // the reference's block-LUT superposition (what its LutSet overload runs)
  kDirect,  // Eq.(1) per (effective-amplitude point, pixel)
  kFft,     // the same hologram by FFT correlation with the point fringe
};

// synthesize_progressive with an explicit method; all four stage snapshots,
// gate masks and operator counts as in the reference (synthesis.hpp:43-54).
ProgressiveResult synthesize_progressive(const RealImage& object, const RealImage& saliency,
                                         const SceneParams& scene, const RefinementPlan& plan,
                                         SynthesisMethod method, int workers = 1);

// Multi-depth scene: objects[l] / saliencies[l] at layers[l] (same wavelength,
// pitch and plane size; own z). Stage planes are the per-layer sums (the
// reference's linearity); operator counts add up over the
// layers; the gate masks are layer 0's.
ProgressiveResult synthesize_progressive_layered(const std::vector<RealImage>& objects,
                                                 const std::vector<RealImage>& saliencies,
                                                 const std::vector<SceneParams>& layers,
                                                 const RefinementPlan& plan,
                                                 SynthesisMethod method, int workers = 1);

}  // namespace wavecgh
