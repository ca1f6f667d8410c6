// Spike propagation over ragged rows (connectivity.py:139-148,
// topomap.py:433-437) and trace STDP (plasticity.py:42-95).
//
// * sw_propagate_atomic: event-driven, warp per spiking row, 128-bit
//   coalesced loads of the row's targets / weights, float64 atomics into the
//   (L2-resident) output.  Fast; summation order is not deterministic.
// * sw_propagate_ordered: bit-exact with np.add.at in spike order: thread per
//   post gathers its incoming synapses through the transpose (CSR, ascending
//   pre) and adds the spiking ones, projection after projection (ff then
//   lat, topomap.py:435-436) — the reference's per-post sequential sum.
#include "common.cuh"

namespace {

__device__ __forceinline__ bool spk(const uint32_t* bits, int i) { return (bits[i >> 5] >> (i & 31)) & 1u; }

__global__ void k_prop_atomic(const int32_t* __restrict__ row_length, const int32_t* __restrict__ target,
                              const double* __restrict__ w, int stride, const int32_t* __restrict__ spikes,
                              const int32_t* n_spikes, double* out, int vec) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int n = *n_spikes;
  for (int q = blockIdx.x * wpb + (threadIdx.x >> 5); q < n; q += gridDim.x * wpb) {
    const int i = spikes[q];
    const int len = row_length[i];
    const int64_t off = (int64_t)i * stride;
    if (vec) {
      // 4 slots per lane per step: int4 targets, 2 x double2 weights
      const int4* t4 = reinterpret_cast<const int4*>(target + off);
      const double2* w2 = reinterpret_cast<const double2*>(w + off);
      for (int s = lane * 4; s < len; s += 128) {
        const int4 t = __ldg(t4 + (s >> 2));
        const double2 wa = __ldg(w2 + (s >> 1));
        const double2 wb = __ldg(w2 + (s >> 1) + 1);
        atomicAdd(out + t.x, wa.x);
        if (s + 1 < len) atomicAdd(out + t.y, wa.y);
        if (s + 2 < len) atomicAdd(out + t.z, wb.x);
        if (s + 3 < len) atomicAdd(out + t.w, wb.y);
      }
    } else {
      for (int s = lane; s < len; s += 32) atomicAdd(out + __ldg(target + off + s), __ldg(w + off + s));
    }
  }
}

struct Proj {
  const int32_t* col_ptr;
  const int32_t* src_pre;
  const int32_t* src_slot;
  const double* w;
  const uint32_t* bits;
  int stride;
};

__global__ void k_prop_ordered(Proj p0, Proj p1, int n_proj, int N, double* out, int accumulate) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
    double acc = accumulate ? out[j] : 0.0;
    for (int k = 0; k < n_proj; ++k) {
      const Proj& p = k ? p1 : p0;
      const int a = p.col_ptr[j], e = p.col_ptr[j + 1];
      for (int q = a; q < e; ++q) {
        const int i = p.src_pre[q];
        if (spk(p.bits, i)) acc = __dadd_rn(acc, p.w[(int64_t)i * p.stride + p.src_slot[q]]);
      }
    }
    out[j] = acc;
  }
}

// ---- STDP (plasticity.py:64-95) ---------------------------------------------------
__global__ void k_stdp_decay(double* x, int nx, double dx, double* y, int ny, double dy) {
  const int n = nx > ny ? nx : ny;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    if (k < nx) x[k] = __dmul_rn(x[k], dx);
    if (k < ny) y[k] = __dmul_rn(y[k], dy);
  }
}

// depression for every synapse of the spiking rows, then x[pre] += 1
__global__ void k_stdp_pre(const int32_t* __restrict__ row_length, const int32_t* __restrict__ target,
                           double* w, int stride, int P, const uint32_t* bits, const double* y, double* x,
                           double a_minus, double w_min, double w_max) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int grp = blockIdx.x * wpb + (threadIdx.x >> 5); grp * 32 < P; grp += gridDim.x * wpb) {
    unsigned m = bits[grp];
    while (m) {
      const int i = grp * 32 + __ffs(m) - 1;
      m &= m - 1;
      const int len = row_length[i];
      const int64_t off = (int64_t)i * stride;
      for (int s = lane; s < len; s += 32) {
        double v = __dsub_rn(w[off + s], __dmul_rn(a_minus, y[target[off + s]]));
        v = fmax(v, w_min);
        w[off + s] = fmin(v, w_max);
      }
      if (lane == 0) x[i] = __dadd_rn(x[i], 1.0);
    }
  }
}

// potentiation of the incoming synapses of spiking posts (transpose), then y[post] += 1
__global__ void k_stdp_post(const int32_t* col_ptr, const int32_t* src_pre, const int32_t* src_slot,
                            double* w, int stride, int N, const uint32_t* bits, const double* x,
                            double* y, double a_plus, double w_min, double w_max) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
    if (!spk(bits, j)) continue;
    const int a = col_ptr[j], e = col_ptr[j + 1];
    for (int q = a; q < e; ++q) {
      const int i = src_pre[q];
      const int64_t o = (int64_t)i * stride + src_slot[q];
      double v = __dadd_rn(w[o], __dmul_rn(a_plus, x[i]));
      v = fmax(v, w_min);
      w[o] = fmin(v, w_max);
    }
    y[j] = __dadd_rn(y[j], 1.0);
  }
}

// ascending spike list from a bitmask (for the event-driven kernels)
__global__ void k_bits_to_list(const uint32_t* bits, int n, int32_t* list, int32_t* count) {
  // single block, ascending order
  __shared__ int32_t base;
  __shared__ int32_t wsum[32];
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int words = (n + 31) / 32;
  for (int w0 = 0; w0 < words; w0 += blockDim.x) {
    const int wd = w0 + threadIdx.x;
    const uint32_t b = wd < words ? bits[wd] : 0u;
    int c = __popc(b);
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(SW_FULL_MASK, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int before = base;
    for (int k = 0; k < warp; ++k) before += wsum[k];
    int pos = before + inc - c;
    uint32_t m = b;
    while (m) {
      list[pos++] = wd * 32 + __ffs(m) - 1;
      m &= m - 1;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base = before + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

int grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" int sw_propagate_atomic(const int32_t* row_length, const int32_t* target, const double* w,
                                   int32_t stride, const int32_t* spikes, const int32_t* n_spikes,
                                   int32_t max_spikes, double* out, void* stream) {
  if (max_spikes <= 0) return SW_OK;
  const int vec = (stride % 4 == 0) && (((uintptr_t)target | (uintptr_t)w) % 16 == 0);
  int64_t blocks = ((int64_t)max_spikes + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_prop_atomic<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(row_length, target, w, stride, spikes,
                                                               n_spikes, out, vec); sw::count_launch();
  SW_CHECK_LAUNCH("sw_propagate_atomic");
  return SW_OK;
}

extern "C" int sw_propagate_ordered(const sw_prop_proj_t* projs, int32_t n_proj, int32_t num_post,
                                    double* out, int32_t accumulate, void* stream) {
  if (n_proj < 1 || n_proj > 2) { sw::set_last_error("propagate_ordered: 1 or 2 projections"); return SW_ERR_INVALID_ARG; }
  Proj p[2] = {};
  for (int k = 0; k < n_proj; ++k)
    p[k] = Proj{projs[k].col_ptr, projs[k].src_pre, projs[k].src_slot, projs[k].weights,
                projs[k].spike_bits, projs[k].stride};
  if (num_post <= 0) return SW_OK;
  k_prop_ordered<<<grid1(num_post), 256, 0, (cudaStream_t)stream>>>(p[0], p[1], n_proj, num_post, out,
                                                                    accumulate); sw::count_launch();
  SW_CHECK_LAUNCH("sw_propagate_ordered");
  return SW_OK;
}

extern "C" int sw_spike_bits_to_list(const uint32_t* bits, int32_t n, int32_t* list, int32_t* count,
                                     void* stream) {
  k_bits_to_list<<<1, 1024, 0, (cudaStream_t)stream>>>(bits, n, list, count); sw::count_launch();
  SW_CHECK_LAUNCH("sw_spike_bits_to_list");
  return SW_OK;
}

extern "C" int sw_stdp_decay(double* x, int32_t nx, double dx, double* y, int32_t ny, double dy,
                             void* stream) {
  const int n = nx > ny ? nx : ny;
  if (n <= 0) return SW_OK;
  k_stdp_decay<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(x, nx, dx, y, ny, dy); sw::count_launch();
  SW_CHECK_LAUNCH("sw_stdp_decay");
  return SW_OK;
}

extern "C" int sw_stdp_pre(const int32_t* row_length, const int32_t* target, double* w, int32_t stride,
                           int32_t num_pre, const uint32_t* pre_bits, const double* y, double* x,
                           double a_minus, double w_min, double w_max, void* stream) {
  if (num_pre <= 0) return SW_OK;
  const int groups = (num_pre + 31) / 32;
  int blocks = (groups + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_stdp_pre<<<blocks, 256, 0, (cudaStream_t)stream>>>(row_length, target, w, stride, num_pre, pre_bits,
                                                       y, x, a_minus, w_min, w_max); sw::count_launch();
  SW_CHECK_LAUNCH("sw_stdp_pre");
  return SW_OK;
}

extern "C" int sw_stdp_post(const int32_t* col_ptr, const int32_t* src_pre, const int32_t* src_slot,
                            double* w, int32_t stride, int32_t num_post, const uint32_t* post_bits,
                            const double* x, double* y, double a_plus, double w_min, double w_max,
                            void* stream) {
  if (num_post <= 0) return SW_OK;
  k_stdp_post<<<grid1(num_post), 256, 0, (cudaStream_t)stream>>>(col_ptr, src_pre, src_slot, w, stride,
                                                                 num_post, post_bits, x, y, a_plus,
                                                                 w_min, w_max); sw::count_launch();
  SW_CHECK_LAUNCH("sw_stdp_post");
  return SW_OK;
}
