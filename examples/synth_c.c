/* Plain-C client of the C ABI (include/wcgh.h): what an FFI binding (cgo,
 * JNI, ctypes, N-API) does. Synthesises a small seeded hologram with the
 * direct, LUT and FFT methods, checks they agree, writes/reads it as CGH1,
 * reconstructs it and scores the reconstruction against itself with SSIM.
 *
 *   gcc -std=c99 -O2 -I include examples/synth_c.c \
 *       -L paper_2211_09938_b200 -l:libwcgh.so -Wl,-rpath,$PWD/paper_2211_09938_b200 -lm
 *
 * Exit code 0 = all checks passed; 2 = no GPU (the ABI fails loudly). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "wcgh.h"

#define CHECK(call)                                                              \
  do {                                                                           \
    int rc_ = (call);                                                            \
    if (rc_ != WCGH_OK) {                                                        \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, wcgh_last_error(NULL)); \
      return rc_ == WCGH_EVALIDATION ? 1 : 2;                                    \
    }                                                                            \
  } while (0)

static unsigned lcg(unsigned* s) { return *s = *s * 1664525u + 1013904223u; }

int main(int argc, char** argv) {
  const int no = 64, nh = 128;
  const char* path = argc > 1 ? argv[1] : "synth_c.cgh";
  unsigned seed = 12345u;
  uint8_t* obj = malloc((size_t)no * no);
  uint8_t* sal = malloc((size_t)no * no);
  for (int i = 0; i < no * no; ++i) {
    unsigned v = lcg(&seed) >> 24;
    obj[i] = (uint8_t)(v < 80 ? 0 : v);              /* ~70% nonzero amplitudes */
    sal[i] = (uint8_t)((lcg(&seed) >> 24) < 64 ? 255 : 0);  /* ~25% salient */
  }
  wcgh_ctx* ctx = NULL;
  CHECK(wcgh_create(0, &ctx));
  int sms = 0;
  char name[64];
  CHECK(wcgh_device_info(ctx, &sms, name, (int)sizeof name));
  printf("device %s, %d SMs, ABI %d\n", name, sms, wcgh_abi_version());

  wcgh_layer layer = {532e-9, 8e-6, 0.05};
  wcgh_desc d;
  memset(&d, 0, sizeof d);
  d.object_size = no;
  d.plane_size = nh;
  d.n_layers = 1;
  d.layers = &layer;
  d.plan.t_ll = 0.5;
  d.plan.t_l = 0.7;
  d.plan.t_full = 0.9;
  d.plan.enable_ll = d.plan.enable_l = d.plan.enable_full = 1;
  d.phase_mode = WCGH_PHASE_FIXED;
  d.row0 = 0;
  d.rows = nh;
  d.obj_dtype = WCGH_U8;
  d.obj_scale = 1.0;
  d.sal_dtype = WCGH_U8;

  const size_t n2 = (size_t)nh * nh;
  float* planes[3];
  wcgh_stats st[3];
  const int methods[3] = {WCGH_METHOD_DIRECT, WCGH_METHOD_LUT, WCGH_METHOD_FFT};
  for (int m = 0; m < 3; ++m) {
    planes[m] = malloc(sizeof(float) * 2 * n2);
    d.method = methods[m];
    CHECK(wcgh_synthesize(ctx, &d, obj, sal, planes[m], &st[m]));
    printf("method %d: %.3f ms, %lld points/cells, ops %llu/%llu/%llu/%llu\n", methods[m],
           st[m].ms_total, (long long)st[m].n_points, (unsigned long long)st[m].ops[0],
           (unsigned long long)st[m].ops[1], (unsigned long long)st[m].ops[2],
           (unsigned long long)st[m].ops[3]);
  }
  int fail = 0;
  for (int m = 1; m < 3; ++m) {
    double num = 0, den = 0;
    for (size_t i = 0; i < 2 * n2; ++i) {
      const double e = (double)planes[m][i] - planes[0][i];
      num += e * e;
      den += (double)planes[0][i] * planes[0][i];
    }
    const double rel = sqrt(num / den);
    printf("rel L2 method %d vs direct: %.3e\n", methods[m], rel);
    if (!(rel <= 1e-4)) fail = 1;
    for (int k = 0; k < 4; ++k)
      if (st[m].ops[k] != st[0].ops[k]) fail = 1;
  }
  /* CGH1 round trip (image_io.cpp:220-278) */
  CHECK(wcgh_write_cgh1(path, planes[0], nh, &layer));
  int n_read = 0;
  wcgh_layer back;
  float* rd = malloc(sizeof(float) * 2 * n2);
  CHECK(wcgh_read_cgh1(path, rd, (int64_t)n2, &n_read, &back));
  if (n_read != nh || memcmp(rd, planes[0], sizeof(float) * 2 * n2) != 0 || back.z != layer.z) fail = 1;
  /* reconstruction + SSIM (angular_spectrum.cpp:47-61, metrics.cpp:49-85) */
  double* rec = malloc(sizeof(double) * n2);
  CHECK(wcgh_reconstruct(ctx, planes[0], WCGH_F32, nh, &layer, 0, rec));
  double score = 0.0;
  CHECK(wcgh_ssim(ctx, rec, rec, nh, nh, 8, 0.01, 0.03, 1.0, &score));
  if (score != 1.0) fail = 1;
  /* validation errors map to WCGH_EVALIDATION */
  d.plane_size = 100;
  if (wcgh_synthesize(ctx, &d, obj, sal, planes[0], NULL) != WCGH_EVALIDATION) fail = 1;
  printf("%s\n", fail ? "FAILED" : "PASSED");
  wcgh_destroy(ctx);
  return fail;
}
