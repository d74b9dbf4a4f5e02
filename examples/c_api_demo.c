/* Plain-C use of the libfllf boundary (include/fllf.h), no CUDA headers:
 * host buffers in, host buffers out (fllf_filter_host; fllf_destroy
 * synchronises the device before the results are read).  Checks properties
 * that fix the output without an oracle (SURVEY 8(c) pins): m = 0 gives the
 * input back exactly, F(I + c) = F(I) + c, and the error paths.
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_2206_04681_b200/lib -lfllf \
 *       -Wl,-rpath,$PWD/paper_2206_04681_b200/lib -lm -o c_api_demo && ./c_api_demo   */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "fllf.h"

#define H 256
#define W 256

static int run(double m, const float* in, float* out) {
  fllf_plan p = NULL;
  fllf_status st = fllf_plan_create(H, W, 4, 4, 510.0, 30.0, m, &p);
  if (st != FLLF_OK) {
    fprintf(stderr, "plan_create: %s (%s)\n", fllf_status_string(st), fllf_last_error_message());
    return 1;
  }
  st = fllf_filter_host(p, in, out, NULL);
  if (st != FLLF_OK) {
    fprintf(stderr, "filter_host: %s (%s)\n", fllf_status_string(st), fllf_last_error_message());
    fllf_destroy(p);
    return 1;
  }
  return fllf_destroy(p) == FLLF_OK ? 0 : 1; /* synchronises the device */
}

int main(void) {
  float* img = malloc(sizeof(float) * H * W);
  float* img2 = malloc(sizeof(float) * H * W);
  float* o0 = malloc(sizeof(float) * H * W);
  float* o1 = malloc(sizeof(float) * H * W);
  float* o2 = malloc(sizeof(float) * H * W);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      /* a step edge, a ramp and texture in [0, 255] */
      const float v = 60.f + 0.3f * x + (x + y > 260 ? 90.f : 0.f) + 12.f * sinf(0.7f * x) * cosf(0.5f * y);
      img[y * W + x] = v;
      img2[y * W + x] = v + 10.f;
    }
  if (run(0.0, img, o0) || run(2.0, img, o1) || run(2.0, img2, o2)) return 1;
  double e_id = 0.0, e_shift = 0.0, detail = 0.0;
  for (int i = 0; i < H * W; ++i) {
    e_id = fmax(e_id, fabs((double)o0[i] - img[i]));
    e_shift = fmax(e_shift, fabs((double)o2[i] - o1[i] - 10.0));
    detail = fmax(detail, fabs((double)o1[i] - img[i]));
  }
  /* error paths: levels < 2, NULL plan */
  fllf_plan bad = NULL;
  const int e1 = fllf_plan_create(H, W, 1, 4, 510.0, 30.0, 1.0, &bad) == FLLF_ERR_INVALID_ARGUMENT;
  const int e2 = fllf_filter_host(NULL, img, o0, NULL) == FLLF_ERR_BAD_POINTER;
  printf("c_api_demo: m=0 identity err %.3g, shift err %.3g, max |F(I)-I| %.3g, errors %d %d\n", e_id, e_shift,
         detail, e1, e2);
  const int ok = e_id <= 1e-3 && e_shift <= 2e-3 && detail > 1.0 && e1 && e2;
  free(img); free(img2); free(o0); free(o1); free(o2);
  puts(ok ? "c_api_demo ok" : "c_api_demo FAILED");
  return ok ? 0 : 1;
}
