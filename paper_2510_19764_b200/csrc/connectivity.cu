// Pairwise-Bernoulli initialisation on the device (connectivity.py:212-245):
// row i draws uniform01 #(counter0 + i*num_post + j) for every column j and
// connects where u < p(i, j).  p is either a constant density (with optional
// diagonal exclusion, classifier.py:142-148) or a toroidal-offset LUT
// (topomap.py:376-388: p = formation_probability(toroidal_distance(i, j)),
// which depends only on the wrapped offset between the grid nodes).
#include "common.cuh"
#include "ragged.cuh"

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

// ---- single-synapse edits (connectivity.py:91-136), one warp ---------------------------
namespace {

// add_synapse: RowFull, then (multapse-free) DuplicateEdge by a lane-parallel
// scan of the row, then append with every plane zeroed and the given values
// set.  status[0] = slot (>= 0) or -SW_ERR_*.
__global__ void k_add_synapse(sw_ragged_t m, int pre, int post, const double* vals,
                              const uint8_t* set_mask, int multapse_free, int32_t* status) {
  const int lane = threadIdx.x;
  const int n = m.row_length[pre];
  const int64_t off = (int64_t)pre * m.stride;
  if (n >= m.max_row_length) {
    if (lane == 0) status[0] = -SW_ERR_ROW_FULL;
    return;
  }
  bool dup = false;
  if (multapse_free)
    for (int s = lane; s < n; s += 32) dup |= m.target[off + s] == post;
  if (__any_sync(SW_FULL_MASK, dup)) {
    if (lane == 0) status[0] = -SW_ERR_DUPLICATE_EDGE;
    return;
  }
  if (lane == 0) {
    m.target[off + n] = post;
    sw::zero_slot(m, off, n);
    for (int p = 0; p < m.n_planes; ++p) {
      if (!(set_mask && set_mask[p])) continue;
      if (m.plane_bytes[p] == 8) ((double*)m.planes[p])[off + n] = vals[p];
      else ((float*)m.planes[p])[off + n] = (float)vals[p];
    }
    m.row_length[pre] = n + 1;
    status[0] = n;
  }
}

// remove_slots of one row: slots[0..k) in any order.  Distinct, in-range
// slots take the exact chained swap-with-last permutation (warp); anything
// else (duplicates) replays remove_synapse one slot at a time in descending
// order, as the reference loop does, stopping at the first out-of-range slot.
__global__ void k_remove_row_slots(sw_ragged_t m, int pre, const int32_t* slots, int k, int32_t* status) {
  extern __shared__ int lst[];
  const int lane = threadIdx.x;
  const int n = m.row_length[pre];
  const int64_t off = (int64_t)pre * m.stride;
  if (lane == 0) {
    for (int q = 0; q < k; ++q) lst[q] = slots[q];
    // insertion sort ascending
    for (int q = 1; q < k; ++q) {
      const int v = lst[q];
      int r = q - 1;
      while (r >= 0 && lst[r] > v) { lst[r + 1] = lst[r]; --r; }
      lst[r + 1] = v;
    }
    bool distinct = true;
    for (int q = 1; q < k; ++q) distinct &= lst[q] != lst[q - 1];
    status[1] = distinct && (k == 0 || (lst[0] >= 0 && lst[k - 1] < n));
  }
  __syncwarp();
  if (status[1]) {
    if (k > 0) {
      sw::warp_apply_removal(m, off, lst, n, k);
      if (lane == 0) m.row_length[pre] = n - k;
    }
    if (lane == 0) status[0] = 0;
    return;
  }
  if (lane == 0) {
    int len = n;
    status[0] = 0;
    for (int q = k - 1; q >= 0; --q) {
      const int slot = lst[q];
      if (slot < 0 || slot >= len) { status[0] = -SW_ERR_SLOT_OUT_OF_RANGE; break; }
      const int last = len - 1;
      if (slot != last) sw::move_slot(m, off, slot, last);
      len = last;
    }
    m.row_length[pre] = len;
  }
}

}  // namespace

extern "C" int sw_ragged_add_synapse(const sw_ragged_t* m, int32_t pre, int32_t post,
                                     const double* values, const uint8_t* set_mask,
                                     int32_t multapse_free, int32_t* status, void* stream) {
  if (pre < 0 || pre >= m->num_pre || post < 0 || post >= m->num_post) {
    sw::set_last_error("add_synapse: pre/post out of range");
    return SW_ERR_INVALID_ARG;
  }
  k_add_synapse<<<1, 32, 0, (cudaStream_t)stream>>>(*m, pre, post, values, set_mask, multapse_free,
                                                     status); sw::count_launch();
  SW_CHECK_LAUNCH("sw_ragged_add_synapse");
  return SW_OK;
}

extern "C" int sw_ragged_remove_row_slots(const sw_ragged_t* m, int32_t pre, const int32_t* slots,
                                          int32_t k, int32_t* status, void* stream) {
  if (pre < 0 || pre >= m->num_pre || k < 0 || k > m->stride) {
    sw::set_last_error("remove_slots: bad row or slot count");
    return SW_ERR_INVALID_ARG;
  }
  k_remove_row_slots<<<1, 32, (size_t)(k > 0 ? k : 1) * sizeof(int), (cudaStream_t)stream>>>(
      *m, pre, slots, k, status); sw::count_launch();
  SW_CHECK_LAUNCH("sw_ragged_remove_row_slots");
  return SW_OK;
}

// ---- column slice (SURVEY 8e M-prop: posts sharded) --------------------------
// dst row i = the synapses of src row i whose target lies in [lo, hi), in
// src slot order, target - lo, every plane copied.  Warp per row: ballot
// compaction keeps the slot order, so an ordered propagation over the
// slice sums each owned post's inputs in exactly the unsharded order.
namespace {
__global__ void k_column_slice(sw_ragged_t src, int lo, int hi, sw_ragged_t dst, int32_t* max_len) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const unsigned lt = sw::lanemask_lt();
  for (int64_t i = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); i < src.num_pre;
       i += (int64_t)gridDim.x * wpb) {
    const int len = src.row_length[i];
    const int64_t so = i * (int64_t)src.stride, dofs = i * (int64_t)dst.stride;
    int n = 0;
    for (int s0 = 0; s0 < len; s0 += 32) {
      const int s = s0 + lane;
      const int t = s < len ? src.target[so + s] : -1;
      const bool keep = t >= lo && t < hi;
      const unsigned b = __ballot_sync(SW_FULL_MASK, keep);
      const int d = n + __popc(b & lt);
      if (keep && d < dst.stride) {
        dst.target[dofs + d] = t - lo;
        for (int p = 0; p < src.n_planes; ++p) {
          if (src.plane_bytes[p] == 8)
            ((uint64_t*)dst.planes[p])[dofs + d] = ((const uint64_t*)src.planes[p])[so + s];
          else
            ((uint32_t*)dst.planes[p])[dofs + d] = ((const uint32_t*)src.planes[p])[so + s];
        }
      }
      n += __popc(b);
    }
    if (lane == 0) {
      dst.row_length[i] = n < dst.stride ? n : dst.stride;
      if (max_len) atomicMax(max_len, n);
    }
  }
}
}  // namespace

extern "C" int sw_ragged_column_slice(const sw_ragged_t* src, int32_t lo, int32_t hi, const sw_ragged_t* dst,
                                      int32_t* max_len, void* stream) {
  if (!src || !dst || lo < 0 || hi < lo || hi > src->num_post || dst->num_pre != src->num_pre ||
      dst->n_planes != src->n_planes || dst->num_post != hi - lo) {
    sw::set_last_error("sw_ragged_column_slice: bad slice or destination shape");
    return SW_ERR_INVALID_ARG;
  }
  for (int p = 0; p < src->n_planes; ++p)
    if (src->plane_bytes[p] != dst->plane_bytes[p]) {
      sw::set_last_error("sw_ragged_column_slice: plane types differ");
      return SW_ERR_INVALID_ARG;
    }
  if (src->num_pre == 0) return SW_OK;
  k_column_slice<<<grid_rows(src->num_pre), 256, 0, (cudaStream_t)stream>>>(*src, lo, hi, *dst, max_len);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_ragged_column_slice");
  return SW_OK;
}
