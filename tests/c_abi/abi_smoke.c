/*
 * Pure-C client of libtwofold_b200.so: proves the drop-in boundary needs no
 * Python, no torch and no CUDA headers — only include/twofold_b200.h.
 *
 *   abi_smoke cpu   argument validation only (no device needed)
 *   abi_smoke gpu   + known-answer tests through the host-plane entry points
 *                   (tf_elementwise_host, tf_reduce_host, tf_selftest)
 *
 * KATs from the reference's own tests: test_acceptance.py:333-352,
 * test_arith.py:89-95, test_kernels.py:143-155.
 */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "twofold_b200.h"

static int fails = 0;
#define CHECK(cond, msg)                                   \
  do {                                                     \
    if (!(cond)) {                                         \
      fprintf(stderr, "FAIL: %s (%s)\n", msg, tf_last_error()); \
      fails++;                                             \
    }                                                      \
  } while (0)

static int run4(int op, double x0, double x1, double y0, double y1, double* z0, double* z1) {
  const void* in[4] = {&x0, &x1, &y0, &y1};
  void* out[2] = {z0, z1};
  return tf_elementwise_host(op, TF_F64, 1, in, out, 0);
}

int main(int argc, char** argv) {
  const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
  CHECK(tf_abi_version() == TF_ABI_VERSION, "abi version");
  CHECK(tf_num_inputs(TF_VTADD2) == 4 && tf_num_inputs(TF_VTSQRT) == 1, "num_inputs");
  CHECK(tf_num_inputs(99) == TF_EINVAL, "unknown op rejected");
  double a = 1, b = 2;
  const void* in[4] = {&a, &a, &a, &a};
  void* out[2] = {&b, &b};
  CHECK(tf_elementwise(99, TF_F64, 1, in, out, NULL) == TF_EINVAL, "bad op");
  CHECK(tf_elementwise(TF_VTADD2, 7, 1, in, out, NULL) == TF_EINVAL, "bad dtype");
  CHECK(tf_elementwise(TF_VTADD2, TF_F64, -1, in, out, NULL) == TF_EINVAL, "negative n");
  CHECK(strstr(tf_last_error(), "negative") != NULL, "error text");
  CHECK(tf_elementwise(TF_VTADD2, TF_F64, 0, in, out, NULL) == TF_OK, "n == 0 is a no-op");
  int V, W, K;
  CHECK(tf_reduce_geometry(TF_F64, &V, &W, &K) == TF_OK && V * W * K == 65536, "geometry");
  if (gpu) {
    CHECK(tf_selftest(0) == TF_OK, "device self-test");
    const double eps = ldexp(1.0, -53);
    double z0, z1;
    CHECK(run4(TF_VTADD2, 1.0, -eps, eps, -eps * eps, &z0, &z1) == TF_OK && z0 == 1.0 && z1 == 0.0,
          "tadd((1,-e),(e,-e^2)) == (1,0)");
    CHECK(run4(TF_VTDIV2, 1.0, 0.0, 1.0 - eps, eps, &z0, &z1) == TF_OK && z0 == 1.0 + 2 * eps &&
              z1 == -2 * eps,
          "tdiv((1,0),(1-e,e)) == (1+2e,-2e)");
    const double t = 1.0 + ldexp(1.0, -27);
    CHECK(run4(TF_VTMUL2, t, 0.0, t, 0.0, &z0, &z1) == TF_OK && z0 == 1.0 + ldexp(1.0, -26) &&
              z1 == ldexp(1.0, -54),
          "tmul FMA residual 2^-54");
    double x1[3] = {1.0, 0.0, -1.0}, y1[3] = {0.0, 0.0, INFINITY}, v[3], e[3];
    const void* in2[2] = {x1, y1};
    void* out2[2] = {v, e};
    CHECK(tf_elementwise_host(TF_VTDIV, TF_F64, 3, in2, out2, 0) == TF_OK && v[0] == INFINITY &&
              isnan(e[0]) && isnan(v[1]) && v[2] == 0.0 && signbit(v[2]),
          "vtdiv specials");
    double xs[1000], r[2];
    for (int i = 0; i < 1000; i++) xs[i] = 0.1;
    CHECK(tf_reduce_host(TF_RSUM, TF_F64, 1000, xs, NULL, r, 0) == TF_OK &&
              fabs(r[0] + r[1] - 100.0) < 1e-13,
          "reduce_host sum");
  }
  if (fails) return 1;
  printf("abi_smoke %s ok\n", gpu ? "gpu" : "cpu");
  return 0;
}
