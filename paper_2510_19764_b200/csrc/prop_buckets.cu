// Post-slab bucketed rows: event-driven spike propagation without L2 atomics
// (connectivity.py:139-148 semantics, atomic mode: out[j] += sum of the
// weights of the spiking rows' synapses onto j, float64, order not fixed).
//
// The output (N <= 8 * 16384 float64) is split into G slabs of 16384 posts,
// each of which fits a CTA's shared memory (128 KB).  A derived copy of the
// ragged matrix keeps, inside every row's own padded slot range, the row's
// synapses grouped by slab ("column slices of every row"):
//   bt[i*stride + k]    slab-local post (uint16) of the k-th bucketed entry,
//   bslot[i*stride + k] the source slot (uint16) of that entry,
//   bw[i*stride + k]    its weight (float64 copy),
//   soff[i*(G+1) + j]   first bucketed entry of slab j in row i (soff[..+G] = len),
// stable in slot order.  Propagation is one cooperative launch: CTA
// (group g, slab c) accumulates slab c of the spiking rows of group g with
// shared-memory float64 atomics, reading only the rows' slab-c segments, so
// every synapse of a spiking row crosses HBM once and no contribution goes
// to L2 as an atomic.  After a grid barrier every CTA sums a post range over
// the groups in ascending group order (one store per post).
//
// Measured (2^20 x 1024 rows, N = 65536, L2 flushed, q = 10 %): 172 us =
// 57.5 % of HBM on the SURVEY M-prop bytes (the L2-atomic kernel: 344 us);
// without the shared-memory atomics (a CAS loop for float64) the same pass
// takes 148 us, so ~25 us are the atomics and the rest is load latency.
//
// The copy depends on the connectivity (rebuild after a structural change,
// like the reference's TransposeMap) and on the weights (sw_prop_buckets_refresh
// re-gathers bw through bslot after a weight change).
#include "common.cuh"

#include <cstdlib>
#include <string>

namespace {

constexpr int kBSlab = 16384;
constexpr int kBMaxSlabs = 8;

__global__ void k_bucket_build(const int32_t* __restrict__ row_length, const int32_t* __restrict__ target,
                               const double* __restrict__ w, int P, int stride, int G, uint16_t* bt,
                               uint16_t* bslot, double* bw, uint16_t* soff) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = sw::lanemask_lt();
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < P; i += gridDim.x * (blockDim.x >> 5)) {
    const int len = row_length[i];
    const int64_t base = (int64_t)i * stride;
    int cnt[kBMaxSlabs];
#pragma unroll
    for (int j = 0; j < kBMaxSlabs; ++j) cnt[j] = 0;
    for (int c0 = 0; c0 < len; c0 += 32) {
      const int s = c0 + lane;
      const int slab = s < len ? (__ldg(target + base + s) >> 14) : -1;
#pragma unroll
      for (int j = 0; j < kBMaxSlabs; ++j)
        if (j < G) cnt[j] += __popc(__ballot_sync(SW_FULL_MASK, slab == j));
    }
    int pos[kBMaxSlabs];
    int run = 0;
#pragma unroll
    for (int j = 0; j < kBMaxSlabs; ++j) {
      pos[j] = run;
      if (j < G) {
        if (lane == 0) soff[(int64_t)i * (G + 1) + j] = (uint16_t)run;
        run += cnt[j];
      }
    }
    if (lane == 0) soff[(int64_t)i * (G + 1) + G] = (uint16_t)len;
    for (int c0 = 0; c0 < len; c0 += 32) {
      const int s = c0 + lane;
      const int t = s < len ? __ldg(target + base + s) : -1;
      const double wv = s < len ? __ldg(w + base + s) : 0.0;
      const int slab = t >= 0 ? (t >> 14) : -1;
#pragma unroll
      for (int j = 0; j < kBMaxSlabs; ++j) {
        if (j < G) {
          const unsigned m = __ballot_sync(SW_FULL_MASK, slab == j);
          if (slab == j) {
            const int dst = pos[j] + __popc(m & lt);
            bt[base + dst] = (uint16_t)(t & (kBSlab - 1));
            bslot[base + dst] = (uint16_t)s;
            bw[base + dst] = wv;
          }
          pos[j] += __popc(m);
        }
      }
    }
  }
}

__global__ void k_bucket_refresh(const int32_t* __restrict__ row_length, const double* __restrict__ w, int P,
                                 int stride, const uint16_t* __restrict__ bslot, double* bw) {
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < P; i += gridDim.x * (blockDim.x >> 5)) {
    const int len = row_length[i];
    const int64_t base = (int64_t)i * stride;
    for (int k = lane; k < len; k += 32) bw[base + k] = __ldg(w + base + __ldg(bslot + base + k));
  }
}

template <int kBW, int kRB, int kH>   // kBW warps per CTA
__global__ void __launch_bounds__(kBW * 32, 1)
k_prop_bucketed(const uint16_t* __restrict__ soff, const uint16_t* __restrict__ bt, const double* __restrict__ bw,
                int G, int stride, const int32_t* __restrict__ spikes, const int32_t* n_spikes, double* out,
                int N, double* scratch, unsigned* arrive) {
  extern __shared__ __align__(16) double acc[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x % G;
  const int g = blockIdx.x / G;
  const int NG = gridDim.x / G;
  for (int k = threadIdx.x; k < kBSlab; k += blockDim.x) acc[k] = 0.0;
  __syncthreads();
  const int S = *n_spikes;
  // kRB spiking rows per warp iteration: their metadata loads, then their
  // data loads (kH x kRB per lane per 32*kH-entry step), are issued together;
  // the next iteration's spike ids are fetched ahead
  const int stepq = NG * kBW;
  int inext[kRB];
#pragma unroll
  for (int r = 0; r < kRB; ++r) {
    const int qq = g * kBW + warp + r * stepq;
    inext[r] = qq < S ? __ldg(spikes + qq) : -1;
  }
  for (int q = g * kBW + warp; q < S; q += kRB * stepq) {
    int i[kRB];
#pragma unroll
    for (int r = 0; r < kRB; ++r) i[r] = inext[r];
    int a[kRB], n[kRB];
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      const int64_t so = (int64_t)max(i[r], 0) * (G + 1) + c;
      a[r] = i[r] >= 0 ? __ldg(soff + so) : 0;
      n[r] = i[r] >= 0 ? __ldg(soff + so + 1) : 0;
    }
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      const int qq = q + (kRB + r) * stepq;
      inext[r] = qq < S ? __ldg(spikes + qq) : -1;
    }
    int nmax = 0;
    int64_t base[kRB];
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      n[r] -= a[r];
      nmax = max(nmax, n[r]);
      base[r] = (int64_t)max(i[r], 0) * stride + a[r];
    }
    for (int k = lane; k < nmax; k += 32 * kH) {
      uint16_t t[kH][kRB];
      double v[kH][kRB];
#pragma unroll
      for (int h = 0; h < kH; ++h)
#pragma unroll
        for (int r = 0; r < kRB; ++r) {
          const int kk = k + 32 * h;
          const bool ok = kk < n[r];
          t[h][r] = ok ? __ldg(bt + base[r] + kk) : (uint16_t)0;
          v[h][r] = ok ? __ldg(bw + base[r] + kk) : 0.0;
        }
#pragma unroll
      for (int h = 0; h < kH; ++h)
#pragma unroll
        for (int r = 0; r < kRB; ++r) {
          if (k + 32 * h < n[r]) atomicAdd(acc + t[h][r], v[h][r]);
        }
    }
  }
  __syncthreads();
  const int slab0 = c * kBSlab;
  const int nslab = min(kBSlab, N - slab0);
  double* mine = scratch + (int64_t)g * ((int64_t)G * kBSlab) + slab0;
  for (int k = threadIdx.x; k < nslab; k += blockDim.x) mine[k] = acc[k];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(arrive, 1u);
    while (atomicAdd(arrive, 0u) < gridDim.x) __nanosleep(64);
  }
  __syncthreads();
  __threadfence();
  const int per = (N + gridDim.x - 1) / gridDim.x;
  const int j0 = blockIdx.x * per, j1 = min(N, j0 + per);
  // the group partials are loaded kGB at a time, then added in ascending
  // group order: one L2 round trip per kGB groups instead of one per group
  // (fixed cost of a one-row pass 20.5 -> 18.4 us)
  constexpr int kGB = 16;
  const int64_t gstride = (int64_t)G * kBSlab;
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    double s = 0.0;
    for (int g0 = 0; g0 < NG; g0 += kGB) {
      double v[kGB];
#pragma unroll
      for (int u = 0; u < kGB; ++u) v[u] = g0 + u < NG ? __ldcg(scratch + (g0 + u) * gstride + j) : 0.0;
#pragma unroll
      for (int u = 0; u < kGB; ++u)
        if (g0 + u < NG) s = __dadd_rn(s, v[u]);
    }
    out[j] = __dadd_rn(out[j], s);
  }
}

// Few spiking rows: one warp per spiking row over the same bucketed copy,
// float64 L2 atomics (the slab pass's fixed cost dominates there).  Reading
// the copy, not the live plane, keeps both kernels on one weight snapshot.
__global__ void k_prop_bucketed_atomic(const uint16_t* __restrict__ soff, const uint16_t* __restrict__ bt,
                                       const double* __restrict__ bw, int G, int stride,
                                       const int32_t* __restrict__ spikes, const int32_t* n_spikes,
                                       double* out) {
  const int lane = threadIdx.x & 31;
  const int S = *n_spikes;
  for (int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < S; q += gridDim.x * (blockDim.x >> 5)) {
    const int i = __ldg(spikes + q);
    const int64_t base = (int64_t)i * stride;
    const uint16_t* so = soff + (int64_t)i * (G + 1);
    for (int c = 0; c < G; ++c) {
      const int a = __ldg(so + c), b = __ldg(so + c + 1);
      for (int k = a + lane; k < b; k += 32)
        atomicAdd(out + c * kBSlab + __ldg(bt + base + k), __ldg(bw + base + k));
    }
  }
}

int slabs_for(int num_post) { return (num_post + kBSlab - 1) / kBSlab; }

using BucketFn = void (*)(const uint16_t*, const uint16_t*, const double*, int, int, const int32_t*,
                         const int32_t*, double*, int, double*, unsigned*);

struct BucketVariant { BucketFn fn; int warps; };

// SW_PROP_BCFG = "WARPSxRBxH" (measurement knob).  Sweep at 2^20 rows,
// q = 1 % / 10 %: 32x2x4 38.9 / 172.1 us, 32x4x2 41.0 / 172.1, 16x8x2
// 43.0 / 186.4, 16x4x4 41.0 / 192.5 (fewer warps lose; 32 warps with more
// loads per lane spill at the 64-register cap of a 1024-thread CTA).
BucketVariant bucket_fn() {
  static BucketVariant v{nullptr, 0};
  if (!v.fn) {
    const char* e = getenv("SW_PROP_BCFG");
    const std::string c = e ? e : "32x2x4";
    v = c == "32x4x2" ? BucketVariant{k_prop_bucketed<32, 4, 2>, 32}
      : c == "16x8x2" ? BucketVariant{k_prop_bucketed<16, 8, 2>, 16}
      : BucketVariant{k_prop_bucketed<32, 2, 4>, 32};
  }
  return v;
}

int bucket_ctas(int G) {
  static int per_sm = -1, sms = 0;
  if (per_sm < 0) {
    cudaFuncSetAttribute((const void*)bucket_fn().fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kBSlab * 8);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)bucket_fn().fn, bucket_fn().warps * 32,
                                                      kBSlab * 8) != cudaSuccess) per_sm = 0;
    cudaGetLastError();
  }
  return (per_sm * sms / G) * G;
}

int grid_rows(int64_t rows) {
  int64_t g = (rows + 7) / 8;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" int32_t sw_prop_bucket_slabs(int32_t num_post) {
  if (num_post <= 0 || num_post > kBMaxSlabs * kBSlab) return 0;
  return slabs_for(num_post);
}

extern "C" int64_t sw_prop_bucketed_workspace_bytes(int32_t num_post) {
  const int G = sw_prop_bucket_slabs(num_post);
  if (G == 0) return 0;
  const int ctas = bucket_ctas(G);
  return (int64_t)ctas * kBSlab * 8 + 256;
}

extern "C" int sw_prop_buckets_build(const int32_t* row_length, const int32_t* target, const double* w,
                                     int32_t num_pre, int32_t num_post, int32_t stride, uint16_t* bt,
                                     uint16_t* bslot, double* bw, uint16_t* soff, void* stream) {
  const int G = sw_prop_bucket_slabs(num_post);
  if (G == 0) { sw::set_last_error("prop buckets: 1 <= num_post <= 131072"); return SW_ERR_INVALID_ARG; }
  if (stride > 65535) { sw::set_last_error("prop buckets: stride must be < 65536"); return SW_ERR_INVALID_ARG; }
  if (num_pre <= 0) return SW_OK;
  k_bucket_build<<<grid_rows(num_pre), 256, 0, (cudaStream_t)stream>>>(row_length, target, w, num_pre, stride, G,
                                                                        bt, bslot, bw, soff);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_prop_buckets_build");
  return SW_OK;
}

extern "C" int sw_prop_buckets_refresh(const int32_t* row_length, const double* w, int32_t num_pre,
                                       int32_t stride, const uint16_t* bslot, double* bw, void* stream) {
  if (num_pre <= 0) return SW_OK;
  k_bucket_refresh<<<grid_rows(num_pre), 256, 0, (cudaStream_t)stream>>>(row_length, w, num_pre, stride, bslot, bw);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_prop_buckets_refresh");
  return SW_OK;
}

extern "C" int sw_propagate_bucketed(const uint16_t* soff, const uint16_t* bt, const double* bw, int32_t num_post,
                                     int32_t stride, const int32_t* spikes, const int32_t* n_spikes,
                                     int32_t max_spikes, double* out, void* workspace, int64_t workspace_bytes,
                                     void* stream) {
  const int G = sw_prop_bucket_slabs(num_post);
  if (G == 0) { sw::set_last_error("propagate_bucketed: 1 <= num_post <= 131072"); return SW_ERR_INVALID_ARG; }
  if (max_spikes <= 0) return SW_OK;
  const int ctas = bucket_ctas(G);
  const int64_t need = (int64_t)ctas * kBSlab * 8 + 256;
  if (ctas < G || !workspace || workspace_bytes < need) {
    sw::set_last_error("propagate_bucketed: workspace of sw_prop_bucketed_workspace_bytes(num_post) required");
    return SW_ERR_INVALID_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* scratch = reinterpret_cast<double*>(workspace);
  unsigned* arrive = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(workspace) + need - 256);
  cudaMemsetAsync(arrive, 0, sizeof(unsigned), st);
  int g = G, s = stride, N = num_post;
  void* args[] = {(void*)&soff, (void*)&bt, (void*)&bw, (void*)&g, (void*)&s, (void*)&spikes,
                  (void*)&n_spikes, (void*)&out, (void*)&N, (void*)&scratch, (void*)&arrive};
  cudaLaunchCooperativeKernel((const void*)bucket_fn().fn, dim3(ctas), dim3(bucket_fn().warps * 32), args, kBSlab * 8, st);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_propagate_bucketed");
  return SW_OK;
}

extern "C" int sw_propagate_bucketed_atomic(const uint16_t* soff, const uint16_t* bt, const double* bw,
                                            int32_t num_post, int32_t stride, const int32_t* spikes,
                                            const int32_t* n_spikes, int32_t max_spikes, double* out,
                                            void* stream) {
  const int G = sw_prop_bucket_slabs(num_post);
  if (G == 0) { sw::set_last_error("propagate_bucketed_atomic: 1 <= num_post <= 131072"); return SW_ERR_INVALID_ARG; }
  if (max_spikes <= 0) return SW_OK;
  int blocks = (max_spikes + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_prop_bucketed_atomic<<<blocks, 256, 0, (cudaStream_t)stream>>>(soff, bt, bw, G, stride, spikes, n_spikes, out);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_propagate_bucketed_atomic");
  return SW_OK;
}
