#include "util.cuh"

namespace sw {

__global__ void k_scan_excl_i32(int32_t* a, int n, int32_t* total) {
  __shared__ int32_t warp_sums[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < n; base += blockDim.x) {
    const int x = base + threadIdx.x;
    const int v = x < n ? a[x] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(SW_FULL_MASK, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(SW_FULL_MASK, w, o);
        if (lane >= o) w += t;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int before = carry + (warp ? warp_sums[warp - 1] : 0);
    if (x < n) a[x] = before + inc - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void k_hist_draws(int64_t D, uint64_t key, uint64_t P, uint64_t rem, int32_t* act,
                             int64_t* rej) {
  const bool pow2 = (P & (P - 1)) == 0;
  int64_t r = 0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < D;
       c += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = draw(key, (uint64_t)c);
    if (draw_valid(h, rem)) atomicAdd(act + (pow2 ? (h & (P - 1)) : (h % P)), 1);
    else ++r;
  }
  if (r) atomicAdd((unsigned long long*)rej, (unsigned long long)r);
}

__global__ void k_hist_fix(int64_t D, uint64_t key, uint64_t P, uint64_t rem, int32_t* act,
                           const int64_t* rej) {
  int64_t need = *rej;
  uint64_t c = (uint64_t)D;
  while (need > 0) {
    const uint64_t h = draw(key, c++);
    if (draw_valid(h, rem)) { act[h % P] += 1; --need; }
  }
}

}  // namespace sw

namespace sw {

__global__ void k_hist_draws_dk(int64_t D, const uint64_t* key, uint64_t P, int32_t* act, int64_t* rej) {
  const uint64_t k = *key, rem = reject_rem(P);
  const bool pow2 = (P & (P - 1)) == 0;
  int64_t r = 0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < D;
       c += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = draw(k, (uint64_t)c);
    if (draw_valid(h, rem)) atomicAdd(act + (pow2 ? (h & (P - 1)) : (h % P)), 1);
    else ++r;
  }
  if (r) atomicAdd((unsigned long long*)rej, (unsigned long long)r);
}

__global__ void k_hist_fix_dk(int64_t D, const uint64_t* key, uint64_t P, int32_t* act, const int64_t* rej) {
  int64_t need = *rej;
  if (need == 0) return;
  const uint64_t k = *key, rem = reject_rem(P);
  uint64_t c = (uint64_t)D;
  while (need > 0) {
    const uint64_t h = draw(k, c++);
    if (draw_valid(h, rem)) { act[h % P] += 1; --need; }
  }
}

}  // namespace sw
