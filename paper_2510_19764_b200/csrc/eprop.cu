// e-prop eligibility recursion + gradient accumulation (sparsewire/_kernels.py:15-39).
//
// Per (replica b, synapse i->j):
//   e    = psi[b,j] * (zb - beta*eps)        (float32, separately rounded)
//   ebar = alpha*ebar + e
//   grad += (double)(lsig[b,j] * ebar)      (float64, replicas ascending)
//   eps  = rho*eps + e
//
// Two entry points:
//  * sw_eprop_accumulate_batch: the reference layout ([B,P,S] eps/ebar,
//    [P,S] grad), thread per synapse, replicas ascending — the drop-in.
//  * sw_eprop_fused_step: the hot path.  Synapses are stored compactly in a
//    per-batch "plan" order: bucketed by 32-post group, then by pre, then
//    slot (sw_eprop_plan_*), so a warp's 32 synapses touch one 128-byte line
//    of psi/lsig and one or two sectors of the pre trace per replica, and
//    eps/ebar[b, e] are perfectly coalesced.  A block owns 32 synapses and
//    all replicas: warps compute the float32 terms for disjoint replica
//    chunks into shared memory, warp 0 folds them into the float64 gradient
//    in ascending replica order (bit-identical to the reference's loop).
//    Extra blocks of the same launch reduce the readout gradients
//    g_w_out += d^T zbar, g_b_out += sum_b d (classifier.py:221-222).
#include "common.cuh"


namespace {

__global__ void k_eprop_ref(const int32_t* targets, const int32_t* row_length, int P, int S,
                            const float* pre_trace, const float* psi, const float* lsig, int B,
                            int H, float* eps, float* ebar, double* grad, float beta, float rho,
                            float alpha) {
  const int64_t total = (int64_t)P * S;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(x / S), s = (int)(x - (int64_t)i * S);
    if (s >= row_length[i]) continue;
    const int j = targets[x];
    double g = grad[x];
    for (int b = 0; b < B; ++b) {
      const int64_t q = (int64_t)b * total + x;
      const float zb = pre_trace[(int64_t)b * P + i];
      const float ep = eps[q];
      const float e = __fmul_rn(psi[(int64_t)b * H + j], __fsub_rn(zb, __fmul_rn(beta, ep)));
      const float eb = __fadd_rn(__fmul_rn(alpha, ebar[q]), e);
      ebar[q] = eb;
      g = __dadd_rn(g, (double)__fmul_rn(lsig[(int64_t)b * H + j], eb));
      eps[q] = __fadd_rn(__fmul_rn(rho, ep), e);
    }
    grad[x] = g;
  }
}

// ---- plan: bucket synapses by (target >> shift, pre, slot) ----------------------------
__global__ void k_bucket_count(const int32_t* row_length, const int32_t* target, int P, int S,
                               int shift, int32_t* counts /* [G*P] */) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    const int n = row_length[i];
    for (int s = 0; s < n; ++s) atomicAdd(&counts[(target[(int64_t)i * S + s] >> shift) * P + i], 1);
  }
}

// exclusive scan of the bucket counts in three launches: per-tile scan
// (kScanTile elements per 1024-thread block) with tile sums, a one-block scan
// of the tile sums (+ the total), then tile offsets added while the cursor
// copy is written
constexpr int kScanTile = 4096;
__device__ __forceinline__ int block_scan_1024(int v, int* warp_sums, int* block_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(SW_FULL_MASK, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(SW_FULL_MASK, w, o);
      if (lane >= o) w += t;
    }
    warp_sums[lane] = w;   // inclusive
  }
  __syncthreads();
  const int before = warp ? warp_sums[warp - 1] : 0;
  *block_total = warp_sums[31];
  __syncthreads();
  return before + inc - v;   // exclusive
}

__global__ void __launch_bounds__(1024) k_scan_tiles(int32_t* a, int n, int32_t* tile_sum) {
  __shared__ int warp_sums[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 4;
  int v[4], s = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) { v[u] = base + u < n ? a[base + u] : 0; s += v[u]; }
  int tot;
  int ex = block_scan_1024(s, warp_sums, &tot);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (base + u < n) a[base + u] = ex;
    ex += v[u];
  }
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_sums(int32_t* tile_sum, int nt, int32_t* total) {
  __shared__ int warp_sums[32];
  int carry = 0;
  for (int b0 = 0; b0 < nt; b0 += 1024) {
    const int x = b0 + threadIdx.x;
    const int v = x < nt ? tile_sum[x] : 0;
    int tot;
    const int ex = block_scan_1024(v, warp_sums, &tot);
    if (x < nt) tile_sum[x] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void k_scan_add(int32_t* a, int n, const int32_t* tile_sum, int32_t* copy) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int v = a[x] + tile_sum[x / kScanTile];
    a[x] = v;
    copy[x] = v;
  }
}

__global__ void k_bucket_fill(const int32_t* row_length, const int32_t* target, int P, int S,
                              int shift, int32_t* cursor /* [G*P], starts as offsets */,
                              int32_t* out_pre, int32_t* out_post, int32_t* out_off) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    const int n = row_length[i];
    for (int s = 0; s < n; ++s) {
      const int j = target[(int64_t)i * S + s];
      const int pos = atomicAdd(&cursor[(j >> shift) * P + i], 1);   // only this thread touches it
      out_pre[pos] = i;
      out_post[pos] = j;
      out_off[pos] = i * S + s;
    }
  }
}

__global__ void k_plan_pad(int32_t* pre, int32_t* post, int32_t* off, const int32_t* total, int e_pad) {
  const int e0 = *total;
  for (int e = e0 + blockIdx.x * blockDim.x + threadIdx.x; e < e_pad; e += gridDim.x * blockDim.x) {
    pre[e] = 0;
    post[e] = 0;
    off[e] = -1;
  }
}

__global__ void k_gather_f64(const double* plane, const int32_t* off, int n, double* out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    out[e] = off[e] >= 0 ? plane[off[e]] : 0.0;
}

__global__ void k_scatter_f64(double* plane, const int32_t* off, int n, const double* in) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    if (off[e] >= 0) plane[off[e]] = in[e];
}

int grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" int sw_eprop_accumulate_batch(const int32_t* targets, const int32_t* row_length,
                                         int32_t num_pre, int32_t stride, const float* pre_trace,
                                         const float* psi, const float* lsig, int32_t batch,
                                         int32_t num_post, float* eps, float* ebar, double* grad,
                                         float beta, float rho, float alpha, void* stream) {
  const int64_t total = (int64_t)num_pre * stride;
  if (total == 0) return SW_OK;
  k_eprop_ref<<<grid1(total), 256, 0, (cudaStream_t)stream>>>(targets, row_length, num_pre, stride,
                                                              pre_trace, psi, lsig, batch, num_post,
                                                              eps, ebar, grad, beta, rho, alpha); sw::count_launch();
  SW_CHECK_LAUNCH("sw_eprop_accumulate_batch");
  return SW_OK;
}

extern "C" int sw_eprop_plan(const int32_t* row_length, const int32_t* target, int32_t num_pre,
                             int32_t stride, int32_t num_post, int32_t shift, int32_t* scratch,
                             int32_t* out_pre, int32_t* out_post, int32_t* out_off,
                             int32_t e_pad, int32_t* total, void* stream) {
  // scratch: counts/offsets [n], cursor [n], scan tile sums [ceil(n/4096)]
  cudaStream_t st = (cudaStream_t)stream;
  const int G = ((num_post - 1) >> shift) + 1;
  const int n = G * num_pre;
  int32_t* counts = scratch;
  int32_t* cursor = scratch + n;
  cudaMemsetAsync(counts, 0, (size_t)n * 4, st);
  if (num_pre > 0) {
    k_bucket_count<<<grid1(num_pre), 256, 0, st>>>(row_length, target, num_pre, stride, shift, counts); sw::count_launch();
    const int nt = (n + kScanTile - 1) / kScanTile;
    int32_t* tile_sum = cursor + n;
    k_scan_tiles<<<nt, 1024, 0, st>>>(counts, n, tile_sum); sw::count_launch();
    k_scan_sums<<<1, 1024, 0, st>>>(tile_sum, nt, total); sw::count_launch();
    k_scan_add<<<grid1(n), 256, 0, st>>>(counts, n, tile_sum, cursor); sw::count_launch();
    k_bucket_fill<<<grid1(num_pre), 256, 0, st>>>(row_length, target, num_pre, stride, shift, cursor,
                                                  out_pre, out_post, out_off); sw::count_launch();
  } else {
    cudaMemsetAsync(total, 0, 4, st);
  }
  k_plan_pad<<<grid1(e_pad), 256, 0, st>>>(out_pre, out_post, out_off, total, e_pad); sw::count_launch();
  SW_CHECK_LAUNCH("sw_eprop_plan");
  return SW_OK;
}

extern "C" int sw_gather_f64(const double* plane, const int32_t* off, int32_t n, double* out, void* stream) {
  if (n <= 0) return SW_OK;
  k_gather_f64<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(plane, off, n, out); sw::count_launch();
  SW_CHECK_LAUNCH("sw_gather_f64");
  return SW_OK;
}

extern "C" int sw_scatter_f64(double* plane, const int32_t* off, int32_t n, const double* in, void* stream) {
  if (n <= 0) return SW_OK;
  k_scatter_f64<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(plane, off, n, in); sw::count_launch();
  SW_CHECK_LAUNCH("sw_scatter_f64");
  return SW_OK;
}

