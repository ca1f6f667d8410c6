/* Plain-C restatement of sparsewire/_kernels.py:15-39 (eprop_accumulate_batch)
 * for the CPU baseline and large oracle checks.  TEST INFRASTRUCTURE ONLY.
 * Compiled with -O2 -ffp-contract=off: every float32 op is separately
 * rounded, grad accumulates float64(float32 product) in (b, i, s) order,
 * exactly the numba loop (per synapse; the rows of a replica run in parallel). */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Within one replica the rows are independent, so each replica's rows are
 * split over OpenMP threads; replicas stay in ascending order (one parallel
 * loop per replica), so every synapse's grad sees the same sequence of
 * float64 additions as the serial loop: bit-identical results. */
void oracle_eprop_accumulate_batch(const int32_t* targets, const int32_t* row_length,
                                   int64_t P, int64_t S, const float* restrict pre_trace,
                                   const float* psi, const float* lsig, int64_t B, int64_t H,
                                   float* restrict eps, float* restrict ebar, double* restrict grad, float beta,
                                   float rho, float alpha) {
#pragma omp parallel
  for (int64_t b = 0; b < B; ++b) {
#pragma omp for schedule(static)
    for (int64_t i = 0; i < P; ++i) {
      const float zb = pre_trace[b * P + i];
      const int32_t n = row_length[i];
      for (int64_t s = 0; s < n; ++s) {
        const int64_t q = (b * P + i) * S + s;
        const int32_t j = targets[i * S + s];
        const float e = psi[b * H + j] * (zb - beta * eps[q]);
        const float eb = alpha * ebar[q] + e;
        ebar[q] = eb;
        const float t = lsig[b * H + j] * eb;
        grad[i * S + s] += (double)t;
        eps[q] = rho * eps[q] + e;
      }
    }
  }
}

int oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* The learning signal lsig[b][h] = f32(sum_c d[b][c] * w[c][h]) as the
 * device computes it (classifier.py:223, the device's stated order): classes
 * ascending from +0.0, one correctly rounded fused multiply-add per class
 * (C99 fma). */
void oracle_lsig_fma(const double* d, const double* w, int64_t B, int64_t C, int64_t H, float* out) {
  for (int64_t b = 0; b < B; ++b)
    for (int64_t h = 0; h < H; ++h) {
      double ls = 0.0;
      for (int64_t c = 0; c < C; ++c) ls = fma(d[b * C + c], w[c * H + h], ls);
      out[b * H + h] = (float)ls;
    }
}
