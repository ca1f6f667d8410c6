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
#include "sm100_async.cuh"
#include <cstdlib>
#include <cstring>

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

// ---- shared-memory slab variant of the atomic mode --------------------------------
// float64 RED into L2 caps the warp-per-row kernel at ~0.16 G contributions
// per microsecond (measured), i.e. ~2 TB/s of row data.  Shared-memory
// float64 atomics sustain ~3x that per SM, so here the output lives in
// shared memory: CTA b owns post slab (b % 4) of 16384 float64 (128 KB) and
// scans the rows of its group (b / 4), accumulating only the targets in its
// slab.  The four CTAs of a group read the same rows at about the same time,
// so HBM delivers each row once and L2 serves the other three reads.  The
// per-group slabs are then written to a scratch plane and, after a grid-wide
// barrier (cooperative launch: one CTA per SM, all co-resident), every CTA
// sums a contiguous post range over the groups in ascending group order and
// adds it to `out` — one plain store per post instead of one RED per
// contribution.
constexpr int kSlabs = 4;        // post slabs (CTAs per group)
constexpr int kSlab = 16384;     // posts per slab
constexpr int kSW = 32;          // warps per CTA
constexpr int kPropSlabSmem = kSlab * 8;
constexpr int kPropSlabMinSpikes = 32768;  // below: warp-per-row kernel

__global__ void __launch_bounds__(kSW * 32, 1)
k_prop_slab(const int32_t* __restrict__ row_length, const int32_t* __restrict__ target,
            const double* __restrict__ w, int stride, const int32_t* __restrict__ spikes,
            const int32_t* n_spikes, double* out, int N, double* scratch, unsigned* arrive, int vec) {
  extern __shared__ __align__(16) double acc[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x % kSlabs;
  const int g = blockIdx.x / kSlabs;
  const int G = gridDim.x / kSlabs;
  const int slab0 = c * kSlab;
  for (int k = threadIdx.x; k < kSlab; k += blockDim.x) acc[k] = 0.0;
  __syncthreads();
  const int S = *n_spikes;
  for (int q = g * kSW + warp; q < S; q += G * kSW) {
    const int i = __ldg(spikes + q);
    const int n = __ldg(row_length + i);
    const int64_t off = (int64_t)i * stride;
    if (vec) {
      const int4* t4 = reinterpret_cast<const int4*>(target + off);
      const double2* w2 = reinterpret_cast<const double2*>(w + off);
#pragma unroll 2
      for (int s = lane * 4; s < n; s += 128) {
        const int4 t = __ldg(t4 + (s >> 2));
        const double2 wa = __ldg(w2 + (s >> 1));
        const double2 wb = __ldg(w2 + (s >> 1) + 1);
        const int r0 = t.x - slab0, r1 = t.y - slab0, r2 = t.z - slab0, r3 = t.w - slab0;
        if ((unsigned)r0 < (unsigned)kSlab) atomicAdd(acc + r0, wa.x);
        if (s + 1 < n && (unsigned)r1 < (unsigned)kSlab) atomicAdd(acc + r1, wa.y);
        if (s + 2 < n && (unsigned)r2 < (unsigned)kSlab) atomicAdd(acc + r2, wb.x);
        if (s + 3 < n && (unsigned)r3 < (unsigned)kSlab) atomicAdd(acc + r3, wb.y);
      }
    } else {
      for (int s = lane; s < n; s += 32) {
        const int r = __ldg(target + off + s) - slab0;
        if ((unsigned)r < (unsigned)kSlab) atomicAdd(acc + r, __ldg(w + off + s));
      }
    }
  }
  __syncthreads();
  // slab -> scratch[g][c*kSlab + k]
  double* mine = scratch + (int64_t)g * (kSlabs * kSlab) + slab0;
  for (int k = threadIdx.x; k < kSlab; k += blockDim.x) mine[k] = acc[k];
  // grid barrier (all CTAs co-resident: cooperative launch)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(arrive, 1u);
    while (atomicAdd(arrive, 0u) < gridDim.x) __nanosleep(64);
  }
  __syncthreads();
  __threadfence();
  // post range of this CTA, summed over the groups in ascending order
  const int per = (N + gridDim.x - 1) / gridDim.x;
  const int j0 = blockIdx.x * per, j1 = min(N, j0 + per);
  // partials loaded kGB groups at a time, added in ascending group order
  constexpr int kGB = 16;
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    double v = 0.0;
    for (int g0 = 0; g0 < G; g0 += kGB) {
      double p[kGB];
#pragma unroll
      for (int u = 0; u < kGB; ++u)
        p[u] = g0 + u < G ? __ldcg(scratch + (int64_t)(g0 + u) * (kSlabs * kSlab) + j) : 0.0;
#pragma unroll
      for (int u = 0; u < kGB; ++u)
        if (g0 + u < G) v = __dadd_rn(v, p[u]);
    }
    out[j] = __dadd_rn(out[j], v);
  }
}

struct Proj {
  const int32_t* col_ptr;
  const int32_t* col_len;
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
      const int a = p.col_ptr[j], e = a + p.col_len[j];
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
__global__ void k_stdp_post(const int32_t* col_ptr, const int32_t* col_len, const int32_t* src_pre, const int32_t* src_slot,
                            double* w, int stride, int N, const uint32_t* bits, const double* x,
                            double* y, double a_plus, double w_min, double w_max) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
    if (!spk(bits, j)) continue;
    const int a = col_ptr[j], e = a + col_len[j];
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

// propagation form override for measurements: SW_PROP_MODE=plain|slab
int prop_mode() {
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("SW_PROP_MODE");
    mode = -1;
    if (e) {
      if (!strcmp(e, "plain")) mode = 0;
      else if (!strcmp(e, "slab")) mode = 1;
    }
  }
  return mode;
}

// CTAs of the cooperative slab kernel on the current device (multiple of kSlabs)
int slab_ctas() {
  static int ctas = -1;
  if (ctas < 0) {
    cudaFuncSetAttribute((const void*)k_prop_slab, cudaFuncAttributeMaxDynamicSharedMemorySize, kPropSlabSmem);
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_prop_slab, kSW * 32,
                                                      kPropSlabSmem) != cudaSuccess) per_sm = 0;
    cudaGetLastError();
    ctas = (per_sm * sms / kSlabs) * kSlabs;
  }
  return ctas;
}

}  // namespace

extern "C" int64_t sw_propagate_workspace_bytes(void) {
  const int ctas = slab_ctas();
  return (int64_t)(ctas / kSlabs) * kSlabs * kSlab * 8 + 256;
}

extern "C" int sw_propagate_atomic(const int32_t* row_length, const int32_t* target, const double* w,
                                   int32_t num_pre, int32_t num_post, int32_t stride,
                                   const int32_t* spikes, const int32_t* n_spikes, int32_t max_spikes,
                                   double* out, void* workspace, int64_t workspace_bytes,
                                   void* stream) {
  if (max_spikes <= 0) return SW_OK;
  const int mode = prop_mode();
  const bool big = max_spikes >= kPropSlabMinSpikes && num_post > 0 && num_post <= kSlabs * kSlab;
  // many spiking rows and an output that fits the shared-memory slabs: the
  // slab kernel (cooperative launch, per-group slabs in the caller workspace)
  const int coop_ctas = (mode == -1 || mode == 1) ? slab_ctas() : 0;
  if (coop_ctas >= kSlabs && big && workspace != nullptr) {
    const int groups = coop_ctas / kSlabs;
    const int64_t need = (int64_t)groups * kSlabs * kSlab * 8 + 256;
    if (workspace_bytes >= need) {
      double* scratch = reinterpret_cast<double*>(workspace);
      unsigned* arrive = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(workspace) + need - 256);
      cudaStream_t st = (cudaStream_t)stream;
      cudaMemsetAsync(arrive, 0, sizeof(unsigned), st);
      const int vec = (stride % 4 == 0) && (((uintptr_t)target | (uintptr_t)w) % 16 == 0);
      int N = num_post;
      void* args[] = {(void*)&row_length, (void*)&target, (void*)&w, (void*)&stride, (void*)&spikes,
                      (void*)&n_spikes, (void*)&out, (void*)&N, (void*)&scratch, (void*)&arrive,
                      (void*)&vec};
      cudaLaunchCooperativeKernel((const void*)k_prop_slab, dim3(coop_ctas), dim3(kSW * 32), args,
                                  kPropSlabSmem, st);
      sw::count_launch();
      SW_CHECK_LAUNCH("sw_propagate_atomic(slab)");
      return SW_OK;
    }
  }
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
    p[k] = Proj{projs[k].col_ptr, projs[k].col_length, projs[k].src_pre, projs[k].src_slot, projs[k].weights,
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

extern "C" int sw_stdp_post(const int32_t* col_ptr, const int32_t* col_len, const int32_t* src_pre, const int32_t* src_slot,
                            double* w, int32_t stride, int32_t num_post, const uint32_t* post_bits,
                            const double* x, double* y, double a_plus, double w_min, double w_max,
                            void* stream) {
  if (num_post <= 0) return SW_OK;
  k_stdp_post<<<grid1(num_post), 256, 0, (cudaStream_t)stream>>>(col_ptr, col_len, src_pre, src_slot, w, stride,
                                                                 num_post, post_bits, x, y, a_plus,
                                                                 w_min, w_max); sw::count_launch();
  SW_CHECK_LAUNCH("sw_stdp_post");
  return SW_OK;
}
