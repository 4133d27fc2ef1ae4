// Internal state shared by the C ABI translation units (wcgh_abi.cu:
// contexts, stage entry points, reconstruction; wcgh_job.cu: jobs and
// multi-GPU; wcgh_io.cu: CGH1/CGHL files): the opaque wcgh_ctx / wcgh_job
// types and the error-mapping guard.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "wcgh_internal.cuh"

struct wcgh_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  std::string name;
  // scratch for the stage entry points
  wcgh::DevBuf b_in, b_in2, b_out, b_out2, b_misc, b_pts, b_plane, b_lut, b_lut_scratch, lut_partial;
  wcgh::DirectScratch direct;
  wcgh::StageCells cells;
  wcgh::ReconPlan recon;  // reconstruction / FFT entry points
  wcgh::DevBuf b_ssim, b_scan, b_ops_rep;
  std::mutex mu;
};

struct wcgh_job {
  wcgh_ctx* ctx = nullptr;
  wcgh_desc desc{};
  std::vector<wcgh_layer> layers;
  int off = 0;
  size_t in_elems = 0;  // per layer No^2
  wcgh::DevBuf obj, sal, a_eff, seg_counts, seg_offsets, scan_scratch, ops, ops_rep, err, points, plane;
  // LUT method
  wcgh::DevBuf w_stage, stage_planes, lut_scratch, lut_partial;
  std::vector<std::unique_ptr<wcgh::StageCells>> cells;  // [layer * 4 + stage]
  std::vector<std::unique_ptr<wcgh::DevBuf>> luts;  // [layer * 4 + stage], guarded allocations
  std::vector<float2*> lut_base;              // support element (0, 0) in each
  wcgh::DirectScratch direct;
  wcgh::DirectTiming timing;
  wcgh::FftPlan fft;  // FFT method
  // pinned host staging
  int64_t* h_offsets = nullptr;       // n_layers + 1
  unsigned long long* h_ops = nullptr;  // n_layers * 5
  int* h_err = nullptr;
  int* h_tot = nullptr;  // LUT: (runs, dense steps, nnz) per stage (re, then im lists)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  wcgh_stats stats{};
  bool uploaded = false;
  bool ran = false;           // a run finished since the last upload
  bool stages_ready = false;  // stage_planes hold the per-stage planes of the last run
  wcgh::DevBuf snap_img, snap_points;  // direct/FFT snapshots (computed on demand)
  // complex objects (obj_dtype WCGH_C128): imaginary-part counterparts
  wcgh::DevBuf a_eff_im, w_stage_im, ops_im, points_im, snap_img_im, snap_points_im;
  std::vector<std::unique_ptr<wcgh::StageCells>> cells_im;
  bool complex_obj() const { return desc.obj_dtype == WCGH_C128; }
  wcgh::PeerPlanes peers;              // fused row-tile gather targets (wcgh_job_set_peer_planes)
  ~wcgh_job() {
    if (h_tot) cudaFreeHost(h_tot);
    if (h_offsets) cudaFreeHost(h_offsets);
    if (h_ops) cudaFreeHost(h_ops);
    if (h_err) cudaFreeHost(h_err);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
};

namespace wcgh {
namespace abi {

// message of the last failed call on this thread (wcgh_last_error)
extern thread_local std::string t_last_error;

inline bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

inline size_t dtype_size(int dt) {
  switch (dt) {
    case WCGH_U8: return 1;
    case WCGH_F32: return 4;
    case WCGH_F64: return 8;
    case WCGH_C128: return 16;
    default: throw ValidationError("dtype must be WCGH_U8, WCGH_F32, WCGH_F64 or WCGH_C128");
  }
}

inline void validate_plan(const wcgh_plan& p) {
  // RefinementPlan::validate (synthesis.cpp:127-131)
  require(0.0 <= p.t_ll && p.t_ll <= p.t_l && p.t_l <= p.t_full && p.t_full <= 1.0,
          "thresholds: need 0 <= t_ll <= t_l <= t_full <= 1");
}

inline void validate_layer(const wcgh_layer& L) {
  // SceneParams (field.cpp:71-80)
  require(L.wavelength > 0.0, "scene: wavelength must be positive");
  require(L.pitch > 0.0, "scene: pitch must be positive");
  require(L.z > 0.0, "scene: z must be positive");
}

template <typename F>
int guard(const wcgh_ctx* ctx, F&& f) {
  (void)ctx;
  try {
    f();
#ifdef WCGH_CHECKED
    chk::collect_all();
#endif
    return WCGH_OK;
  } catch (const ValidationError& e) {
    t_last_error = e.what();
    return WCGH_EVALIDATION;
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return WCGH_ERUNTIME;
  }
}

inline void use_device(wcgh_ctx* ctx) { WCGH_CUDA(cudaSetDevice(ctx->device)); }

inline void sync(cudaStream_t s) { WCGH_CUDA(cudaStreamSynchronize(s)); }

inline void check_analysis_flags(int flags) {
  if (flags & kErrObjectNonFinite) throw ValidationError("object: non-finite sample");
  if (flags & kErrSaliencyRange) throw ValidationError("quantize_saliency: values must lie in [0,1]");
}


// job descriptor checks (wcgh_job.cu)
void job_validate(const wcgh_desc& d);

}  // namespace abi
}  // namespace wcgh

