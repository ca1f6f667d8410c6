// Neuron updates (sparsewire/neurons.py).
//  * ALIF (float32, neurons.py:60-73): exact NumPy-2 op order with the
//    Python-float constants rounded to float32 first (NEP 50).
//  * Conductance LIF with exponential Euler (float64, neurons.py:137-148);
//    exp() is the only non-IEEE-exact op (tolerance).
//  * Poisson source step (neurons.py:189-195): counter-exact uniform01 < p.
#include "common.cuh"

namespace {

__device__ __forceinline__ float alif_thr(float a, float beta, float v_thr) {
  return __fadd_rn(v_thr, __fmul_rn(beta, a));
}

__global__ void k_alif_step(float* v, float* a, float* z, const float* rec, const float* ext,
                            int64_t n, float alpha, float rho, float beta, float v_thr) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const float zo = z[x];
    float vv = __fmul_rn(alpha, __fsub_rn(v[x], __fmul_rn(zo, v_thr)));
    vv = __fadd_rn(__fadd_rn(vv, rec[x]), ext[x]);
    const float aa = __fadd_rn(__fmul_rn(rho, a[x]), zo);
    v[x] = vv;
    a[x] = aa;
    z[x] = (vv >= alif_thr(aa, beta, v_thr)) ? 1.0f : 0.0f;
  }
}

__global__ void k_alif_surrogate(const float* v, const float* a, float* psi, int64_t n, float beta,
                                 float v_thr) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const float c = __fdiv_rn(__fsub_rn(v[x], alif_thr(a[x], beta, v_thr)), v_thr);
    const float r = __fsub_rn(1.0f, fabsf(c));
    psi[x] = __fmul_rn(0.5f, (r > 0.0f || r != r) ? r : 0.0f);
  }
}

// g = (g + in) * decay_s; active = k > refractory_until; r = g / g_leak;
// v_inf = (V_rest + r*E) / (1 + r); V = v_inf + (V - v_inf) * exp(-h*(1+r)/tau_m)
// refractory -> V_reset; spike if V >= V_theta -> V_reset, until = k + ref_steps.
__global__ void k_lif_cond_step(double* V, double* g, int64_t* ref_until, const double* incoming,
                                int n, int64_t k, double decay_s, double g_leak, double v_rest,
                                double e_exc, double v_theta, double v_reset, double h,
                                double tau_m, int64_t ref_steps, uint32_t* spike_bits,
                                int32_t* spike_list, int32_t* spike_count) {
  const int lane = threadIdx.x & 31;
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const int x = base + threadIdx.x;
    bool spk = false;
    if (x < n) {
      const double gg = __dmul_rn(__dadd_rn(g[x], incoming[x]), decay_s);
      g[x] = gg;
      const bool active = k > ref_until[x];
      const double r = __ddiv_rn(gg, g_leak);
      const double vinf = __ddiv_rn(__dadd_rn(v_rest, __dmul_rn(r, e_exc)), __dadd_rn(1.0, r));
      const double arg = __ddiv_rn(__dmul_rn(-h, __dadd_rn(1.0, r)), tau_m);
      const double vn = __dadd_rn(vinf, __dmul_rn(__dsub_rn(V[x], vinf), exp(arg)));
      double vv = active ? vn : v_reset;
      spk = active && (vv >= v_theta);
      if (spk) {
        vv = v_reset;
        ref_until[x] = k + ref_steps;
      }
      V[x] = vv;
    }
    const unsigned b = __ballot_sync(SW_FULL_MASK, spk);
    if (spike_bits && lane == 0 && base + (threadIdx.x & ~31) < n)
      spike_bits[(base + (threadIdx.x & ~31)) >> 5] = b;
    if (spike_list && spk) {
      // unordered append; callers needing ascending order use spike_bits
      const int pos = atomicAdd(spike_count, 1);
      spike_list[pos] = x;
    }
  }
}

// Bernoulli(p[node]) with u = uniform01 draw #(step*n + node) (neurons.py:189-195)
__global__ void k_poisson_step(uint64_t key, int64_t counter0, const double* p, int n,
                               uint32_t* spike_bits) {
  const int lane = threadIdx.x & 31;
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const int x = base + threadIdx.x;
    bool spk = false;
    if (x < n) spk = sw::u01(sw::draw(key, (uint64_t)(counter0 + x))) < p[x];
    const unsigned b = __ballot_sync(SW_FULL_MASK, spk);
    if (lane == 0 && base + (threadIdx.x & ~31) < n) spike_bits[(base + (threadIdx.x & ~31)) >> 5] = b;
  }
}

int grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" int sw_alif_step(float* v, float* a, float* z, const float* rec, const float* ext,
                            int64_t n, float alpha, float rho, float beta, float v_thr, void* stream) {
  if (n <= 0) return SW_OK;
  k_alif_step<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(v, a, z, rec, ext, n, alpha, rho, beta, v_thr); sw::count_launch();
  SW_CHECK_LAUNCH("sw_alif_step");
  return SW_OK;
}

extern "C" int sw_alif_surrogate(const float* v, const float* a, float* psi, int64_t n, float beta,
                                 float v_thr, void* stream) {
  if (n <= 0) return SW_OK;
  k_alif_surrogate<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(v, a, psi, n, beta, v_thr); sw::count_launch();
  SW_CHECK_LAUNCH("sw_alif_surrogate");
  return SW_OK;
}

extern "C" int sw_lif_cond_step(double* V, double* g, int64_t* ref_until, const double* incoming,
                                int32_t n, int64_t step_index, double decay_s, double g_leak,
                                double v_rest, double e_exc, double v_theta, double v_reset,
                                double h, double tau_m, int64_t ref_steps, uint32_t* spike_bits,
                                void* stream) {
  if (n <= 0) return SW_OK;
  k_lif_cond_step<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(
      V, g, ref_until, incoming, n, step_index, decay_s, g_leak, v_rest, e_exc, v_theta, v_reset, h,
      tau_m, ref_steps, spike_bits, nullptr, nullptr); sw::count_launch();
  SW_CHECK_LAUNCH("sw_lif_cond_step");
  return SW_OK;
}

extern "C" int sw_poisson_step(uint64_t key, int64_t counter0, const double* p, int32_t n,
                               uint32_t* spike_bits, void* stream) {
  if (n <= 0) return SW_OK;
  k_poisson_step<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(key, counter0, p, n, spike_bits); sw::count_launch();
  SW_CHECK_LAUNCH("sw_poisson_step");
  return SW_OK;
}

// PoissonSource.set_correlated_rates + probabilities on the device
// (neurons.py:175-183, 189-193): rate = f_base + f_peak * sum_c exp(-d_c^2 /
// (2 sigma^2)), d_c the torus distance to centre c, p = 1 - exp(-rate*h*1e-3).
// CUDA exp/hypot: within a few ulp of numpy, a model option for
// large grids where the host loop over s^2 centres dominates.
__global__ void k_poisson_rates(int side, int n, const double* centers, int n_centers, double f_base,
                                double f_peak, double two_sigma2, double h, double* rates, double* p) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    const double gx = (double)(x % side), gy = (double)(x / side);
    double bump = 0.0;
    for (int c = 0; c < n_centers; ++c) {
      double dx = fabs(gx - centers[2 * c]), dy = fabs(gy - centers[2 * c + 1]);
      dx = fmin(dx, side - dx);
      dy = fmin(dy, side - dy);
      const double d = hypot(dx, dy);
      bump = __dadd_rn(bump, exp(-(d * d) / two_sigma2));
    }
    const double r = __dadd_rn(f_base, __dmul_rn(f_peak, bump));
    rates[x] = r;
    p[x] = 1.0 - exp(-r * h * 1e-3);
  }
}

extern "C" int sw_poisson_rates(int32_t side, const double* centers, int32_t n_centers, double f_base,
                                double f_peak, double sigma, double h, double* rates, double* p,
                                void* stream) {
  const int n = side * side;
  if (n <= 0) return SW_OK;
  k_poisson_rates<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(side, n, centers, n_centers, f_base, f_peak,
                                                              2.0 * sigma * sigma, h, rates, p); sw::count_launch();
  SW_CHECK_LAUNCH("sw_poisson_rates");
  return SW_OK;
}
