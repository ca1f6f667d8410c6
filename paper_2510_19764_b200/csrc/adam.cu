// Adam over float64 planes (sparsewire/plasticity.py:198-227), exact op order:
//   m = m*b1 + (1-b1)*g ; v = v*b2 + ((1-b2)*g)*g
//   p = p - (lr*(m/c1)) / (sqrt(v/c2) + eps) ; g = 0
// c1 = 1 - b1**t, c2 = 1 - b2**t are host Python floats (as in the reference).
#include "common.cuh"

__global__ void k_adam_f64(double* __restrict__ p, double* __restrict__ g, double* __restrict__ m,
                           double* __restrict__ v, int64_t n, double b1, double omb1, double b2,
                           double omb2, double c1, double c2, double lr, double eps) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    const double mi = __dadd_rn(__dmul_rn(m[i], b1), __dmul_rn(omb1, gi));
    const double vi = __dadd_rn(__dmul_rn(v[i], b2), __dmul_rn(__dmul_rn(omb2, gi), gi));
    m[i] = mi;
    v[i] = vi;
    const double mh = __ddiv_rn(mi, c1);
    const double vh = __ddiv_rn(vi, c2);
    p[i] = __dsub_rn(p[i], __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps)));
    g[i] = 0.0;
  }
}

extern "C" int sw_adam_f64(double* p, double* g, double* m, double* v, int64_t n, double b1,
                           double one_minus_b1, double b2, double one_minus_b2, double c1, double c2,
                           double lr, double eps, void* stream) {
  if (n <= 0) return SW_OK;
  int64_t grid = (n + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  k_adam_f64<<<(int)grid, 256, 0, (cudaStream_t)stream>>>(p, g, m, v, n, b1, one_minus_b1, b2,
                                                           one_minus_b2, c1, c2, lr, eps); sw::count_launch();
  SW_CHECK_LAUNCH("sw_adam_f64");
  return SW_OK;
}
