/*
 * pbs_oracle.c -- TEST INFRASTRUCTURE ONLY (see pbs_oracle.h).
 * CPU restatement of the reference hot path; instantiated for float and
 * double from pbs_oracle_impl.inc.  Built by oracle/Makefile into
 * oracle/_build/libpbs_oracle.so with -O2 -ffp-contract=off (no -march).
 */
#define _POSIX_C_SOURCE 200809L
#include "pbs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char pbso_err[512];

const char* pbso_last_error(void) { return pbso_err; }

static int pbso_fail(int code, const char* prefix, const char* msg) {
  snprintf(pbso_err, sizeof pbso_err, "%s: %s", prefix, msg);
  return code;
}

/* steady clock in microseconds (detail::StageClock, pipeline.hpp:87-99) */
static double pbso_now_us(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec * 1e6 + (double)ts.tv_nsec * 1e-3;
}

/* Permutation::inverse (permutation.hpp:51-55) */
void pbso_inverse(const int32_t* perm, size_t n, int32_t* inv) {
  for (size_t i = 0; i < n; ++i) inv[perm[i]] = (int32_t)i;
}

void pbso_expf(const float* x, float* y, size_t n) {
  for (size_t i = 0; i < n; ++i) y[i] = expf(x[i]);
}

#define REAL float
#define SFX f32
#include "pbs_oracle_impl.inc"
#undef REAL
#undef SFX

#define REAL double
#define SFX f64
#include "pbs_oracle_impl.inc"
#undef REAL
#undef SFX
