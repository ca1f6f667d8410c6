// One 0.1 ms step of the topographic-map model (topomap.py:419-452) as four
// launches with all step state on the device (graph-capturable):
//   k_tm_neurons  Poisson source spikes (neurons.py:189-195, counter =
//                 step*n + node) and the conductance-LIF target update
//                 (neurons.py:137-148) with last step's pending input;
//   k_tm_prop     ordered propagation of both projections through their
//                 transposes into pending (ff then lat, topomap.py:433-437),
//                 fused with the STDP trace decays (plasticity.py:64-66);
//   k_tm_pre      STDP depression of the spiking source rows (ff) and
//                 spiking target rows (lat), then x += 1 (plasticity.py:68-81);
//   k_tm_post     STDP potentiation through the transposes for the spiking
//                 targets, then y += 1 (plasticity.py:83-95); step += 1.
#include "common.cuh"

namespace {

__device__ __forceinline__ bool bit(const uint32_t* b, int i) { return (b[i >> 5] >> (i & 31)) & 1u; }

__global__ void k_tm_neurons(sw_topomap_step_t S) {
  const int lane = threadIdx.x & 31;
  const int64_t k = *S.step;
  const int n = S.n;
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const int x = base + threadIdx.x;
    bool src = false, tgt = false;
    // the owned range is word-aligned, so a warp is either owned or not
    const bool own = x >= S.post_lo && x < S.post_hi;
    if (x < n) src = sw::u01(sw::draw(S.poisson_key, (uint64_t)(k * n + x))) < S.p_src[x];
    if (x < n && own) {
      const double gg = __dmul_rn(__dadd_rn(S.g_tot[x], S.pending[x]), S.decay_s);
      S.g_tot[x] = gg;
      const bool active = k > S.ref_until[x];
      const double r = __ddiv_rn(gg, S.g_leak);
      const double vinf = __ddiv_rn(__dadd_rn(S.v_rest, __dmul_rn(r, S.e_exc)), __dadd_rn(1.0, r));
      const double arg = __ddiv_rn(__dmul_rn(-S.h, __dadd_rn(1.0, r)), S.tau_m);
      double vv = active ? __dadd_rn(vinf, __dmul_rn(__dsub_rn(S.V[x], vinf), exp(arg))) : S.v_reset;
      tgt = active && vv >= S.v_theta;
      if (tgt) {
        vv = S.v_reset;
        S.ref_until[x] = k + S.ref_steps;
      }
      S.V[x] = vv;
    }
    const unsigned bs = __ballot_sync(SW_FULL_MASK, src);
    const unsigned bt = __ballot_sync(SW_FULL_MASK, tgt);
    if (lane == 0 && base + (threadIdx.x & ~31) < n) {
      const int w = (base + (threadIdx.x & ~31)) >> 5;
      S.src_bits[w] = bs;
      if (own) S.tgt_bits[w] = bt;
    }
  }
}

__global__ void k_tm_prop(sw_topomap_step_t S) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < S.n; j += gridDim.x * blockDim.x) {
    // trace decays (x per pre, y per post; square model: n pres and n posts)
    S.ff_x[j] = __dmul_rn(S.ff_x[j], S.decay_x);
    S.ff_y[j] = __dmul_rn(S.ff_y[j], S.decay_y);
    S.lat_x[j] = __dmul_rn(S.lat_x[j], S.decay_x);
    S.lat_y[j] = __dmul_rn(S.lat_y[j], S.decay_y);
    if (j < S.post_lo || j >= S.post_hi) continue;
    double acc = 0.0;
    for (int q = S.ff_col_ptr[j]; q < S.ff_col_ptr[j + 1]; ++q) {
      const int i = S.ff_src_pre[q];
      if (bit(S.src_bits, i)) acc = __dadd_rn(acc, S.ff_g[(int64_t)i * S.ff_stride + S.ff_src_slot[q]]);
    }
    for (int q = S.lat_col_ptr[j]; q < S.lat_col_ptr[j + 1]; ++q) {
      const int i = S.lat_src_pre[q];
      if (bit(S.tgt_bits, i)) acc = __dadd_rn(acc, S.lat_g[(int64_t)i * S.lat_stride + S.lat_src_slot[q]]);
    }
    S.pending[j] = acc;
  }
}

__device__ __forceinline__ void depress_row(const int32_t* rl, const int32_t* tg, double* w, int stride,
                                            int i, const double* y, double a_minus, double w_min,
                                            double w_max, int lane) {
  const int len = rl[i];
  const int64_t off = (int64_t)i * stride;
  for (int s = lane; s < len; s += 32) {
    double v = __dsub_rn(w[off + s], __dmul_rn(a_minus, y[tg[off + s]]));
    v = fmax(v, w_min);
    w[off + s] = fmin(v, w_max);
  }
}

__global__ void k_tm_pre(sw_topomap_step_t S) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int groups = (S.n + 31) / 32;
  for (int g = blockIdx.x * wpb + (threadIdx.x >> 5); g < 2 * groups; g += gridDim.x * wpb) {
    const bool ff = g < groups;
    const int grp = ff ? g : g - groups;
    unsigned m = ff ? S.src_bits[grp] : S.tgt_bits[grp];
    while (m) {
      const int i = grp * 32 + __ffs(m) - 1;
      m &= m - 1;
      if (ff) depress_row(S.ff_row_length, S.ff_target, S.ff_g, S.ff_stride, i, S.ff_y, S.a_minus, S.w_min, S.w_max, lane);
      else depress_row(S.lat_row_length, S.lat_target, S.lat_g, S.lat_stride, i, S.lat_y, S.a_minus, S.w_min, S.w_max, lane);
      if (lane == 0) {
        if (ff) S.ff_x[i] = __dadd_rn(S.ff_x[i], 1.0);
        else S.lat_x[i] = __dadd_rn(S.lat_x[i], 1.0);
      }
    }
  }
}

__global__ void k_tm_post(sw_topomap_step_t S) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < S.n; j += gridDim.x * blockDim.x) {
    if (!bit(S.tgt_bits, j)) continue;
    for (int q = S.ff_col_ptr[j]; q < S.ff_col_ptr[j + 1]; ++q) {
      const int i = S.ff_src_pre[q];
      const int64_t o = (int64_t)i * S.ff_stride + S.ff_src_slot[q];
      double v = __dadd_rn(S.ff_g[o], __dmul_rn(S.a_plus, S.ff_x[i]));
      v = fmax(v, S.w_min);
      S.ff_g[o] = fmin(v, S.w_max);
    }
    S.ff_y[j] = __dadd_rn(S.ff_y[j], 1.0);
    for (int q = S.lat_col_ptr[j]; q < S.lat_col_ptr[j + 1]; ++q) {
      const int i = S.lat_src_pre[q];
      const int64_t o = (int64_t)i * S.lat_stride + S.lat_src_slot[q];
      double v = __dadd_rn(S.lat_g[o], __dmul_rn(S.a_plus, S.lat_x[i]));
      v = fmax(v, S.w_min);
      S.lat_g[o] = fmin(v, S.w_max);
    }
    S.lat_y[j] = __dadd_rn(S.lat_y[j], 1.0);
  }
}

__global__ void k_tm_tick(sw_topomap_step_t S, int64_t* spike_counts) {
  // step += 1 and per-step spike counters (source, target)
  __shared__ int cs, ct;
  if (threadIdx.x == 0) { cs = 0; ct = 0; }
  __syncthreads();
  const int words = (S.n + 31) / 32;
  int a = 0, b = 0;
  for (int w = threadIdx.x; w < words; w += blockDim.x) {
    a += __popc(S.src_bits[w]);
    b += __popc(S.tgt_bits[w]);
  }
  atomicAdd(&cs, a);
  atomicAdd(&ct, b);
  __syncthreads();
  if (threadIdx.x == 0) {
    *S.step += 1;
    if (spike_counts) {
      spike_counts[0] += cs;
      spike_counts[1] += ct;
    }
  }
}

int grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

static int check_step(const sw_topomap_step_t* s) {
  if (s->post_lo < 0 || s->post_hi > s->n || s->post_lo > s->post_hi || (s->post_lo & 31) ||
      ((s->post_hi & 31) && s->post_hi != s->n)) {
    sw::set_last_error("topomap step: post shard must be [lo, hi) on 32-post word boundaries");
    return SW_ERR_INVALID_ARG;
  }
  return SW_OK;
}

extern "C" int sw_topomap_neurons(const sw_topomap_step_t* s, void* stream) {
  if (int e = check_step(s)) return e;
  const int n = s->n;
  if (n <= 0) return SW_OK;
  k_tm_neurons<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(*s); sw::count_launch();
  SW_CHECK_LAUNCH("sw_topomap_neurons");
  return SW_OK;
}

extern "C" int sw_topomap_synapses(const sw_topomap_step_t* s, int64_t* spike_counts, void* stream) {
  if (int e = check_step(s)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const int n = s->n;
  if (n <= 0) return SW_OK;
  k_tm_prop<<<grid1(n), 256, 0, st>>>(*s); sw::count_launch();
  int groups = (n + 31) / 32;
  int blocks = (2 * groups + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_tm_pre<<<blocks, 256, 0, st>>>(*s); sw::count_launch();
  k_tm_post<<<grid1(n), 256, 0, st>>>(*s); sw::count_launch();
  k_tm_tick<<<1, 256, 0, st>>>(*s, spike_counts); sw::count_launch();
  SW_CHECK_LAUNCH("sw_topomap_synapses");
  return SW_OK;
}

extern "C" int sw_topomap_step(const sw_topomap_step_t* s, int64_t* spike_counts, void* stream) {
  if (int e = sw_topomap_neurons(s, stream)) return e;
  return sw_topomap_synapses(s, spike_counts, stream);
}
