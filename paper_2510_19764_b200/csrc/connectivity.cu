// Pairwise-Bernoulli initialisation on the device (connectivity.py:212-245):
// row i draws uniform01 #(counter0 + i*num_post + j) for every column j and
// connects where u < p(i, j).  p is either a constant density (with optional
// diagonal exclusion, classifier.py:142-148) or a toroidal-offset LUT
// (topomap.py:376-388: p = formation_probability(toroidal_distance(i, j)),
// which depends only on the wrapped offset between the grid nodes).
#include "common.cuh"

namespace {

__device__ __forceinline__ double pair_prob(int mode, double density, const double* lut, int side,
                                            int64_t i, int j) {
  if (mode == 0) return density;
  if (mode == 1) return (j == (int)i) ? 0.0 : density;
  // mode 2: torus offset LUT indexed by ((xj-xi) mod L) + L*((yj-yi) mod L)
  const int xi = (int)(i % side), yi = (int)(i / side);
  const int xj = j % side, yj = j / side;
  const int dx = (xj - xi + side) % side, dy = (yj - yi + side) % side;
  return lut[dx + side * dy];
}

// pass 1: row lengths (warp per row); pass 2 (fill=true): ascending targets
template <bool FILL>
__global__ void k_bernoulli(int64_t num_pre, int num_post, uint64_t key, uint64_t c0, int mode,
                            double density, const double* lut, int side, int32_t* row_length,
                            int32_t* target, int stride, int32_t* max_len) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const unsigned lt = sw::lanemask_lt();
  for (int64_t i = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); i < num_pre;
       i += (int64_t)gridDim.x * wpb) {
    int n = 0;
    const uint64_t base = c0 + (uint64_t)i * (uint64_t)num_post;
    for (int j0 = 0; j0 < num_post; j0 += 32) {
      const int j = j0 + lane;
      bool hit = false;
      if (j < num_post) {
        const double u = sw::u01(sw::draw(key, base + (uint64_t)j));
        hit = u < pair_prob(mode, density, lut, side, i, j);
      }
      const unsigned b = __ballot_sync(SW_FULL_MASK, hit);
      if (FILL && hit) {
        const int s = n + __popc(b & lt);
        if (s < stride) target[i * (int64_t)stride + s] = j;
      }
      n += __popc(b);
    }
    if (lane == 0) {
      if (!FILL) {
        row_length[i] = n;
        atomicMax(max_len, n);
      } else {
        row_length[i] = n < stride ? n : stride;
      }
    }
  }
}

int grid_rows(int64_t rows) {
  int64_t g = (rows + 7) / 8;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" int sw_init_bernoulli_count(int64_t num_pre, int32_t num_post, uint64_t key,
                                       uint64_t counter0, int32_t mode, double density,
                                       const double* lut, int32_t side, int32_t* row_length,
                                       int32_t* max_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(max_len, 0, sizeof(int32_t), st);
  if (num_pre == 0 || num_post == 0) {
    if (num_pre) cudaMemsetAsync(row_length, 0, num_pre * sizeof(int32_t), st);
    return SW_OK;
  }
  k_bernoulli<false><<<grid_rows(num_pre), 256, 0, st>>>(num_pre, num_post, key, counter0, mode,
                                                         density, lut, side, row_length, nullptr,
                                                         1, max_len); sw::count_launch();
  SW_CHECK_LAUNCH("sw_init_bernoulli_count");
  return SW_OK;
}

extern "C" int sw_init_bernoulli_fill(int64_t num_pre, int32_t num_post, uint64_t key,
                                      uint64_t counter0, int32_t mode, double density,
                                      const double* lut, int32_t side, int32_t* row_length,
                                      int32_t* target, int32_t stride, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (num_pre == 0 || num_post == 0) return SW_OK;
  k_bernoulli<true><<<grid_rows(num_pre), 256, 0, st>>>(num_pre, num_post, key, counter0, mode,
                                                        density, lut, side, row_length, target,
                                                        stride, nullptr); sw::count_launch();
  SW_CHECK_LAUNCH("sw_init_bernoulli_fill");
  return SW_OK;
}
