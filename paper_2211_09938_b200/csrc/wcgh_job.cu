// C ABI: hologram jobs (create / upload / run / downloads / stage snapshots
// / fused multi-GPU gather) and the one-shot entry points.
#include <thread>

#include <cstdlib>

#include "wcgh_state.cuh"

using namespace wcgh;
using namespace wcgh::abi;

#ifdef WCGH_CHECKED
__global__ void k_inject_one(int* c) { *c += 1; }  // checked-build negative control
#endif

void wcgh::abi::job_validate(const wcgh_desc& d) {
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
  require(d.sal_dtype != WCGH_C128, "saliency dtype must be WCGH_U8, WCGH_F32 or WCGH_F64");
  if (d.method == WCGH_METHOD_LUT) {
    for (int l = 1; l < d.n_layers; ++l)
      require(d.layers[l].wavelength == d.layers[0].wavelength && d.layers[l].pitch == d.layers[0].pitch,
              "job (LUT): layers must share wavelength and pitch");
  }
}

extern "C" {

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
    j->ops_rep.reserve(sizeof(unsigned long long) * WCGH_OP_LEVELS * L * kOpReplicas);
    WCGH_CUDA(cudaMemsetAsync(j->ops_rep.p, 0, sizeof(unsigned long long) * WCGH_OP_LEVELS * L * kOpReplicas,
                              ctx->stream));
    sync(ctx->stream);  // zeroed before any stream the job later runs on
    j->err.reserve(64);
    j->plane.reserve(sizeof(float2) * size_t(d.rows) * d.plane_size);
    WCGH_CUDA(cudaMallocHost(&j->h_offsets, sizeof(int64_t) * (L + 1)));
    WCGH_CUDA(cudaMallocHost(&j->h_ops, sizeof(unsigned long long) * WCGH_OP_LEVELS * L));
    WCGH_CUDA(cudaMallocHost(&j->h_err, sizeof(int) * 4));
    WCGH_CUDA(cudaMallocHost(&j->h_tot, sizeof(int) * 2 * 3 * 4 * kMaxLayers));
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

// K1 (+ the compaction counts of the direct/FFT methods). A complex object
// (random initial phase, synthesis.cpp:205-219) is analysed part by part,
// as the reference does (pyr_re, pyr_im): the gates depend on the saliency
// only, so the two passes gate identically and the operator counts are the
// first pass's.
void run_analysis(wcgh_job* j, cudaStream_t s, bool lut) {
  const wcgh_desc& d = j->desc;
  const int No = d.object_size, L = d.n_layers;
  const bool cplx = j->complex_obj();
  const size_t ops_bytes = sizeof(unsigned long long) * WCGH_OP_LEVELS * L;
  WCGH_CUDA(cudaMemsetAsync(j->ops.p, 0, ops_bytes + sizeof(int), s));
  AnalysisOut ao;
  ao.a_eff = j->a_eff.as<float>();
  ao.seg_counts = (lut || cplx) ? nullptr : j->seg_counts.as<int>();
  ao.w_stage = lut ? j->w_stage.as<float>() : nullptr;
  ao.ops = j->ops.as<unsigned long long>();
  ao.ops_rep = j->ops_rep.as<unsigned long long>();  // zeroed at creation, re-zeroed by the fold
  ao.err = reinterpret_cast<int*>(ao.ops + WCGH_OP_LEVELS * L);
  j->stats.total_launches +=
      launch_analysis(j->obj.p, d.obj_dtype, d.obj_scale, j->sal.p, d.sal_dtype, No, L, d.plan, ao, s);
  if (!cplx) return;
  AnalysisOut bo = ao;
  bo.a_eff = static_cast<float*>(j->a_eff_im.reserve(sizeof(float) * j->in_elems * L));
  bo.w_stage = lut ? static_cast<float*>(j->w_stage_im.reserve(sizeof(float) * wstage_len(No) * L))
                   : nullptr;
  bo.ops = static_cast<unsigned long long*>(j->ops_im.reserve(ops_bytes));
  WCGH_CUDA(cudaMemsetAsync(bo.ops, 0, ops_bytes, s));
  j->stats.total_launches +=
      launch_analysis(static_cast<const char*>(j->obj.p) + sizeof(double), d.obj_dtype, d.obj_scale,
                      j->sal.p, d.sal_dtype, No, L, d.plan, bo, s);
  if (!lut) {
    launch_seg_counts_f32(ao.a_eff, No, L, j->seg_counts.as<int>(), s, bo.a_eff);
    j->stats.total_launches += 1;
  }
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
#ifdef WCGH_CHECKED
  // negative control of the checked build: one extra count in the last
  // segment makes K2's record count disagree with K1's (caught by the
  // compaction check; all writes stay inside the point buffer)
  if (const char* e = std::getenv("WCGH_CHK_INJECT"); e && std::string(e) == "segcount") {
    k_inject_one<<<1, 1, 0, s>>>(j->seg_counts.as<int>() + nseg - 1);
    WCGH_CHECK_LAUNCH();
  }
#endif
  const int scan_launches = launch_scan(j->seg_counts.as<int>(), j->seg_offsets.as<int>(), int(nseg), s,
                                        &j->scan_scratch);
  const bool cplx = j->complex_obj();
  const float* a_im = cplx ? j->a_eff_im.as<float>() : nullptr;
  float* p_im = cplx && !fft ? static_cast<float*>(j->points_im.reserve(sizeof(float) * (j->in_elems * L + 1)))
                             : nullptr;
  if (!fft)
    launch_compact_points(j->a_eff.as<float>(), j->seg_offsets.as<int>(), No, L, j->off, 0,
                          j->points.as<wcgh_point>(), s, a_im, p_im);
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
  // geometry bound on |dx|, |dy| for the phase-series plan: the FULL plane's, never the
  // band's, so every rank picks the same series lengths, kernel form and hold as a
  // single-GPU run and its band stays bitwise equal to those rows of the whole plane
  const double far = double(j->off + No - 1);
  const double max_dy = std::max(far, double(d.plane_size - 1 - j->off));
  int launches = 0;
  if (fft) {
    // same hologram by FFT correlation; `updates` keeps the direct-sum count
    j->stats.updates = double(lb[L]) * double(d.rows) * double(d.plane_size);
    launches = launch_fft_synthesis(j->fft, j->a_eff.as<float>(), No, j->off, d.plane_size,
                                    d.row0, d.rows, j->plane.as<float2>(), s, &j->timing,
                                    &j->peers, a_im);
  } else {
    launches = launch_direct(j->points.as<wcgh_point>(), lb, L, d.layers, d.plane_size, d.row0,
                             d.rows, d.phase_mode, far, max_dy, j->plane.as<float2>(), j->direct,
                             s, &j->timing, &j->stats.updates, &j->peers, p_im);
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

// Two pixels per thread: float4 loads of the stage planes, float4 complex64
// stores of the plane and the peer planes (same per-pixel order, bitwise equal).
__global__ void k_sum_stages2(const float4* __restrict__ planes, size_t count2, int n_stages,
                              float4* __restrict__ out, PeerPlanes peers) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count2) return;
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int st = 0; st < n_stages; ++st) {
    const float4 v = planes[size_t(st) * count2 + i];
    r.x += v.x;
    r.y += v.y;
    r.z += v.z;
    r.w += v.w;
  }
  out[i] = r;
  store_peers2(peers, 2 * i, r);
}

void launch_sum_stages(const float2* planes, size_t band, int n_stages, float2* out,
                       const PeerPlanes& peers, cudaStream_t s) {
  if (band % 2 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(planes) % 16 == 0 && peers_aligned16(peers))
    k_sum_stages2<<<unsigned((band / 2 + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const float4*>(planes), band / 2, n_stages, reinterpret_cast<float4*>(out), peers);
  else
    k_sum_stages<<<unsigned((band + 255) / 256), 256, 0, s>>>(planes, band, n_stages, out, peers);
  WCGH_CHECK_LAUNCH();
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
  // run lists of the nonzero gated cells per (layer, stage) (K2 for the LUT
  // path); a complex object adds the lists of its imaginary weights
  const bool cplx = j->complex_obj();
  while (j->cells.size() < size_t(L) * 4) j->cells.push_back(std::make_unique<StageCells>());
  while (cplx && j->cells_im.size() < size_t(L) * 4) j->cells_im.push_back(std::make_unique<StageCells>());
  int* h_tot_im = j->h_tot + 3 * 4 * kMaxLayers;
  for (int l = 0; l < L; ++l)
    for (int st = 0; st < 4; ++st) {
      const float* w = j->w_stage.as<float>() + wstage_len(No) * l + wofs[st];
      StageCells& sc = *j->cells[size_t(l) * 4 + st];
      j->stats.total_launches += launch_stage_cells(w, ms[st], sc, s);
      stage_cells_totals_async(sc, j->h_tot + 3 * (l * 4 + st), s);
      if (cplx) {
        const float* wi = j->w_stage_im.as<float>() + wstage_len(No) * l + wofs[st];
        StageCells& si = *j->cells_im[size_t(l) * 4 + st];
        j->stats.total_launches += launch_stage_cells(wi, ms[st], si, s);
        stage_cells_totals_async(si, h_tot_im + 3 * (l * 4 + st), s);
      }
    }
  WCGH_CUDA(cudaMemcpyAsync(j->h_ops, j->ops.p, sizeof(unsigned long long) * WCGH_OP_LEVELS * L, cudaMemcpyDeviceToHost, s));
  WCGH_CUDA(cudaMemcpyAsync(j->h_err, j->ops.as<unsigned long long>() + WCGH_OP_LEVELS * L, sizeof(int), cudaMemcpyDeviceToHost, s));
  WCGH_CUDA(cudaEventRecord(j->ev[1], s));
  sync(s);
  check_analysis_flags(*j->h_err);
  finish_stats(j, j->h_ops);
  if (!synth) {  // front end only (wcgh_job_analyze): nonzero gated cells
    long long cells = 0;
    for (int k = 0; k < 4 * L; ++k) cells += j->h_tot[3 * k + 2] + (cplx ? h_tot_im[3 * k + 2] : 0);
    j->stats.n_points = cells;
    WCGH_CUDA(cudaEventElapsedTime(&j->stats.ms_analysis, j->ev[0], j->ev[1]));
    j->stats.ms_total = j->stats.ms_analysis;
    return;
  }
  // the K4 chunk kernel takes the run lists as parameter blocks: one copy of
  // every stage's list to the host while the stream is idle
  for (int k = 0; k < 4 * L; ++k) {
    StageCells& sc = *j->cells[k];
    sc.n_runs = j->h_tot[3 * k];
    sc.n_dense = j->h_tot[3 * k + 1];
    sc.nnz = j->h_tot[3 * k + 2];
    stage_cells_fetch(sc, s);
    if (cplx) {
      StageCells& si = *j->cells_im[k];
      si.n_runs = h_tot_im[3 * k];
      si.n_dense = h_tot_im[3 * k + 1];
      si.nnz = h_tot_im[3 * k + 2];
      stage_cells_fetch(si, s);
    }
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
      if (cplx) {  // + i * (imaginary weights' superposition), by linearity
        StageCells& si = *j->cells_im[k];
        si.n_runs = h_tot_im[3 * k];
        si.n_dense = h_tot_im[3 * k + 1];
        si.nnz = h_tot_im[3 * k + 2];
        j->stats.total_launches += launch_lut_stage(j->lut_base[k], d.plane_size, blocks[st], si,
                                                    j->off, d.row0, d.rows, sp + band * st,
                                                    j->lut_partial, s, &j->timing, true, true);
        cells += si.nnz;
      }
    }
  j->stats.synth_launches = j->timing.launches();
  WCGH_CUDA(cudaEventRecord(j->ev[2], s));
  launch_sum_stages(sp, band, 4, j->plane.as<float2>(), j->peers, s);
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
  const double max_dy = std::max(far, double(d.plane_size - 1 - j->off));  // full plane (see run)
  const bool cplx = j->complex_obj();
  float* img_im = cplx ? static_cast<float*>(j->snap_img_im.reserve(sizeof(float) * j->in_elems * L)) : nullptr;
  float* pim = cplx ? static_cast<float*>(j->snap_points_im.reserve(sizeof(float) * (j->in_elems * L + 1)))
                    : nullptr;
  for (int st = 0; st < 4; ++st) {
    launch_stage_delta(j->w_stage.as<float>(), No, L, st, img, s);
    if (cplx) launch_stage_delta(j->w_stage_im.as<float>(), No, L, st, img_im, s);
    float2* out = planes + band * st;
    if (d.method == WCGH_METHOD_FFT) {
      launch_fft_synthesis(j->fft, img, No, j->off, d.plane_size, d.row0, d.rows, out, s, nullptr,
                           nullptr, img_im);
      continue;
    }
    launch_seg_counts_f32(img, No, L, j->seg_counts.as<int>(), s, img_im);
    launch_scan(j->seg_counts.as<int>(), j->seg_offsets.as<int>(), int(nseg), s, &j->scan_scratch);
    wcgh_point* pts = static_cast<wcgh_point*>(j->snap_points.reserve(sizeof(wcgh_point) * (j->in_elems * L + 1)));
    launch_compact_points(img, j->seg_offsets.as<int>(), No, L, j->off, 0, pts, s, img_im, pim);
    for (int l = 0; l <= L; ++l)
      WCGH_CUDA(cudaMemcpyAsync(reinterpret_cast<int*>(j->h_offsets) + l,
                                j->seg_offsets.as<int>() + per_layer * size_t(l), sizeof(int),
                                cudaMemcpyDeviceToHost, s));
    sync(s);
    int64_t lb[kMaxLayers + 1];
    for (int l = 0; l <= L; ++l) lb[l] = reinterpret_cast<const int*>(j->h_offsets)[l];
    launch_direct(pts, lb, L, d.layers, d.plane_size, d.row0, d.rows, d.phase_mode, far, max_dy,
                  out, j->direct, s, nullptr, nullptr, nullptr, pim);
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
    pp.limit = size_t(job->desc.plane_size) * size_t(job->desc.plane_size);
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

int wcgh_job_download_a_eff_im(wcgh_job* job, float* out) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && out, "job_download_a_eff_im: NULL argument");
    require(job->complex_obj(), "job_download_a_eff_im: the job's object is real (not WCGH_C128)");
    require(job->a_eff_im.p != nullptr, "job_download_a_eff_im: run or analyze the job first");
    use_device(job->ctx);
    cudaStream_t s = job->ctx->stream;
    WCGH_CUDA(cudaMemcpyAsync(out, job->a_eff_im.p, sizeof(float) * job->in_elems * job->desc.n_layers,
                              cudaMemcpyDeviceToHost, s));
    sync(s);
  });
}

int wcgh_job_download_points_im(wcgh_job* job, float* out, int64_t capacity) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && out, "job_download_points_im: NULL argument");
    require(job->complex_obj(), "job_download_points_im: the job's object is real (not WCGH_C128)");
    require(job->desc.method == WCGH_METHOD_DIRECT,
            "job_download_points: the compacted point list is built by the direct method");
    require(job->points_im.p != nullptr, "job_download_points_im: run or analyze the job first");
    const int64_t n = int64_t(job->stats.n_points);
    require(capacity >= n, "job_download_points_im: capacity below the point count");
    use_device(job->ctx);
    cudaStream_t s = job->ctx->stream;
    WCGH_CUDA(cudaMemcpyAsync(out, job->points_im.p, sizeof(float) * size_t(n), cudaMemcpyDeviceToHost, s));
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
      launch_sum_stages(job->stage_planes.as<float2>(), band, st + 1, tmp, PeerPlanes{}, s);
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

int wcgh_job_direct_form(const wcgh_job* job, int* form, int* hold) {
  return guard(job ? job->ctx : nullptr, [&] {
    require(job && form && hold, "job_direct_form: NULL argument");
    require(job->desc.method == WCGH_METHOD_DIRECT, "job_direct_form: the job does not use the direct method");
    *form = job->timing.form;
    *hold = job->timing.hold;
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

WCGH_CHK_TU(wcgh_job)
