// TransposeMap.rebuild (connectivity.py:173-192) on the device, CSR layout
// with slack: for post j the (pre, slot) of its incoming synapses in
// [col_ptr[j], col_ptr[j] + col_length[j]), ordered by (pre, slot) — the
// reference's lexsort((slot, pre, post)) order; column j has room for
// col_ptr[j+1] - col_ptr[j] = (its length at the rebuild) + slack entries, so
// sw_transpose_patch can apply a rewiring update in place.  Count -> scan -> atomic scatter ->
// per-column insertion sort (columns are short; the sort makes the
// nondeterministic scatter order irrelevant).  All kernels early-exit when
// *changed == 0, so "remap only if the matrix changed" (updates.py:367-369)
// is decided on the device and the rebuild can sit in a CUDA graph.
#include "common.cuh"
#include "util.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace {
// grid barrier; a single-block launch (small sheets: no cooperative launch,
// whose set-up costs more than the work) uses the block barrier
__device__ __forceinline__ void gsync(cg::grid_group& grid) {
  if (gridDim.x == 1) __syncthreads();
  else grid.sync();
}


__device__ __forceinline__ bool skip(const int32_t* changed) { return changed && *changed == 0; }

__global__ void k_tr_zero(int32_t* col_length, int N, int32_t* max_len, const int32_t* changed) {
  if (skip(changed)) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) col_length[j] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *max_len = 0;
}

__global__ void k_tr_count(sw_ragged_t m, int32_t* col_length, const int32_t* changed) {
  if (skip(changed)) return;
  const int64_t total = (int64_t)m.num_pre * m.stride;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / m.stride;
    if ((int)(x - i * m.stride) < m.row_length[i]) atomicAdd(&col_length[m.target[x]], 1);
  }
}

__global__ void k_tr_prep(const int32_t* col_length, int32_t* col_ptr, int N, int slack, const int32_t* changed) {
  if (skip(changed)) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x)
    col_ptr[j] = col_length[j] + slack;
}

__global__ void k_tr_scan(int32_t* col_ptr, int N, const int32_t* changed) {
  if (skip(changed)) return;
  // single block; col_ptr[N] receives the total
  __shared__ int32_t warp_sums[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < N; base += blockDim.x) {
    const int x = base + threadIdx.x;
    const int v = x < N ? col_ptr[x] : 0;
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
    if (x < N) col_ptr[x] = before + inc - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) col_ptr[N] = carry;
}

__global__ void k_tr_scatter(sw_ragged_t m, const int32_t* col_ptr, int32_t* cursor, int32_t* src_pre,
                             int32_t* src_slot, int N, const int32_t* changed) {
  if (skip(changed)) return;
  // cursor[j] counts fills of column j (zeroed by the caller-side memset kernel)
  const int64_t total = (int64_t)m.num_pre * m.stride;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / m.stride;
    const int s = (int)(x - i * m.stride);
    if (s < m.row_length[i]) {
      const int j = m.target[x];
      const int pos = col_ptr[j] + atomicAdd(&cursor[j], 1);
      src_pre[pos] = (int32_t)i;
      src_slot[pos] = s;
    }
  }
}

__global__ void k_tr_sort(const int32_t* col_ptr, const int32_t* col_length, int32_t* src_pre, int32_t* src_slot,
                          int N, int32_t* max_len, const int32_t* changed) {
  if (skip(changed)) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
    const int a = col_ptr[j], e = a + col_length[j];
    for (int q = a + 1; q < e; ++q) {
      const int p = src_pre[q], s = src_slot[q];
      int r = q - 1;
      while (r >= a && (src_pre[r] > p || (src_pre[r] == p && src_slot[r] > s))) {
        src_pre[r + 1] = src_pre[r];
        src_slot[r + 1] = src_slot[r];
        --r;
      }
      src_pre[r + 1] = p;
      src_slot[r + 1] = s;
    }
    atomicMax(max_len, e - a);
  }
}

__global__ void k_zero_i32_guard(int32_t* a, int n, const int32_t* changed) {
  if (skip(changed)) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) a[j] = 0;
}

// ---- the whole rebuild in one cooperative launch -------------------------------------
__global__ void __launch_bounds__(512)
k_tr_coop(sw_ragged_t m, int32_t* col_length, int32_t* col_ptr, int32_t* src_pre, int32_t* src_slot,
          int32_t* cursor, int32_t* max_len, const int32_t* changed, int32_t* bsum, int slack,
          int clear_changed) {
  if (skip(changed)) return;   // uniform: every block returns before any grid barrier
  cg::grid_group grid = cg::this_grid();
  const int N = m.num_post;
  const int64_t total = (int64_t)m.num_pre * m.stride;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gn = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = gt; j < N; j += gn) {
    col_length[j] = 0;
    cursor[j] = 0;
  }
  if (gt == 0) *max_len = 0;
  gsync(grid);
  for (int64_t x = gt; x < total; x += gn) {
    const int64_t i = x / m.stride;
    if ((int)(x - i * m.stride) < m.row_length[i]) atomicAdd(&col_length[m.target[x]], 1);
  }
  gsync(grid);
  // exclusive scan: block b owns the contiguous columns [c0, c1)
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry, boff;
  const int per = (N + gridDim.x - 1) / gridDim.x;
  const int c0 = min(N, (int)blockIdx.x * per), c1 = min(N, c0 + per);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto block_scan = [&](bool write) {
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = c0; base < c1; base += blockDim.x) {
      const int x = base + threadIdx.x;
      const int v = x < c1 ? col_length[x] + slack : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(SW_FULL_MASK, inc, o);
        if (lane >= o) inc += t;
      }
      if (lane == 31) wsum[warp] = inc;
      __syncthreads();
      if (warp == 0) {
        int w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(SW_FULL_MASK, w, o);
          if (lane >= o) w += t;
        }
        wsum[lane] = w;
      }
      __syncthreads();
      const int before = carry + (warp ? wsum[warp - 1] : 0);
      if (write && x < c1) col_ptr[x] = boff + before + inc - v;
      __syncthreads();
      if (threadIdx.x == blockDim.x - 1) carry = before + inc;
      __syncthreads();
    }
  };
  if (threadIdx.x == 0) boff = 0;
  block_scan(false);
  if (threadIdx.x == 0) bsum[blockIdx.x] = carry;
  gsync(grid);
  if (threadIdx.x == 0) {
    int o = 0;
    for (int b = 0; b < (int)blockIdx.x; ++b) o += bsum[b];
    boff = o;
    if (blockIdx.x == gridDim.x - 1) col_ptr[N] = o + bsum[blockIdx.x];
  }
  __syncthreads();
  block_scan(true);
  gsync(grid);
  for (int64_t x = gt; x < total; x += gn) {
    const int64_t i = x / m.stride;
    const int s = (int)(x - i * m.stride);
    if (s < m.row_length[i]) {
      const int j = m.target[x];
      const int pos = col_ptr[j] + atomicAdd(&cursor[j], 1);
      src_pre[pos] = (int32_t)i;
      src_slot[pos] = s;
    }
  }
  gsync(grid);
  for (int64_t j = gt; j < N; j += gn) {
    const int a = col_ptr[j], e = a + col_length[j];
    for (int q = a + 1; q < e; ++q) {
      const int p = src_pre[q], s = src_slot[q];
      int r = q - 1;
      while (r >= a && (src_pre[r] > p || (src_pre[r] == p && src_slot[r] > s))) {
        src_pre[r + 1] = src_pre[r];
        src_slot[r + 1] = src_slot[r];
        --r;
      }
      src_pre[r + 1] = p;
      src_slot[r + 1] = s;
    }
    atomicMax(max_len, e - a);
  }
  if (clear_changed) {
    // the gate flag is ours (the patch's overflow flag): reset it once every
    // block has read it
    gsync(grid);
    if (gt == 0) *const_cast<int32_t*>(changed) = 0;
  }
}

int grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" int sw_transpose_rebuild_gated(const sw_ragged_t* m, int32_t* col_length, int32_t* col_ptr,
                                          int32_t* src_pre, int32_t* src_slot, int32_t* cursor,
                                          int32_t* max_len, int32_t* changed, int32_t* block_scratch,
                                          int32_t slack, int32_t clear_changed, void* stream);

extern "C" int sw_transpose_rebuild(const sw_ragged_t* m, int32_t* col_length, int32_t* col_ptr,
                                    int32_t* src_pre, int32_t* src_slot, int32_t* cursor,
                                    int32_t* max_len, const int32_t* changed, int32_t slack, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int N = m->num_post;
  const int64_t total = (int64_t)m->num_pre * m->stride;
  k_tr_zero<<<grid1(N), 256, 0, st>>>(col_length, N, max_len, changed); sw::count_launch();
  k_zero_i32_guard<<<grid1(N), 256, 0, st>>>(cursor, N, changed); sw::count_launch();
  if (total) { k_tr_count<<<grid1(total), 256, 0, st>>>(*m, col_length, changed); sw::count_launch(); }
  k_tr_prep<<<grid1(N), 256, 0, st>>>(col_length, col_ptr, N, slack, changed); sw::count_launch();
  k_tr_scan<<<1, 1024, 0, st>>>(col_ptr, N, changed); sw::count_launch();
  if (total) {
    k_tr_scatter<<<grid1(total), 256, 0, st>>>(*m, col_ptr, cursor, src_pre, src_slot, N, changed); sw::count_launch();
  }
  k_tr_sort<<<grid1(N), 256, 0, st>>>(col_ptr, col_length, src_pre, src_slot, N, max_len, changed); sw::count_launch();
  SW_CHECK_LAUNCH("sw_transpose_rebuild");
  return SW_OK;
}

extern "C" int sw_transpose_rebuild_coop(const sw_ragged_t* m, int32_t* col_length, int32_t* col_ptr,
                                         int32_t* src_pre, int32_t* src_slot, int32_t* cursor,
                                         int32_t* max_len, const int32_t* changed,
                                         int32_t* block_scratch, int32_t slack, void* stream) {
  return sw_transpose_rebuild_gated(m, col_length, col_ptr, src_pre, src_slot, cursor, max_len, const_cast<int32_t*>(changed),
                                    block_scratch, slack, 0, stream);
}

extern "C" int sw_transpose_rebuild_gated(const sw_ragged_t* m, int32_t* col_length, int32_t* col_ptr,
                                          int32_t* src_pre, int32_t* src_slot, int32_t* cursor,
                                          int32_t* max_len, int32_t* changed, int32_t* block_scratch,
                                          int32_t slack, int32_t clear_changed, void* stream) {
  if (!block_scratch) { sw::set_last_error("sw_transpose_rebuild_coop: block scratch required"); return SW_ERR_INVALID_ARG; }
  static int max_blocks = 0;
  if (max_blocks == 0) {
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tr_coop, 512, 0);
    max_blocks = per_sm * sms;
    if (max_blocks > 2048) max_blocks = 2048;
    if (max_blocks < 1) max_blocks = 1;
  }
  const int64_t total = (int64_t)m->num_pre * m->stride;
  int64_t want = (total + 2047) / 2048;
  const int64_t byn = (m->num_post + 511) / 512;
  if (byn > want) want = byn;
  int blocks = (int)(want < 1 ? 1 : (want > max_blocks ? max_blocks : want));
  sw_ragged_t M = *m;
  void* args[] = {(void*)&M, (void*)&col_length, (void*)&col_ptr, (void*)&src_pre, (void*)&src_slot,
                  (void*)&cursor, (void*)&max_len, (void*)&changed, (void*)&block_scratch, (void*)&slack,
                  (void*)&clear_changed};
  if (total <= 65536) {
    // small matrices: one block, block barriers, an ordinary launch
    k_tr_coop<<<1, 512, 0, (cudaStream_t)stream>>>(M, col_length, col_ptr, src_pre, src_slot, cursor, max_len,
                                                    changed, block_scratch, slack, clear_changed);
  } else {
    cudaLaunchCooperativeKernel((const void*)k_tr_coop, dim3(blocks), dim3(512), args, 0, (cudaStream_t)stream);
  }
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_transpose_rebuild_coop");
  return SW_OK;
}

// ---- incremental patch (sw_transpose_patch) ------------------------------------------
// One block.  The rows changed by an update and their removed (pre, post)
// pairs come from the patch log.  Every column the rows touch (their
// current targets and their removed targets) is rebuilt by one warp: its
// entries of unchanged rows are kept in place order, the changed rows'
// current synapses onto it are merged in (pre, slot) order -- exactly the
// column a full rebuild produces.  Overflows (log, slack, per-warp buffer,
// too many changed rows for the row scan) raise *rebuild instead.
namespace {

constexpr int kPatchWarps = 16;
constexpr int kPatchRows = 64;      // changed rows handled by the patch (more: full rebuild)
constexpr int kPatchCol = 256;      // column entries a warp merges in shared memory

__device__ __forceinline__ bool bit_get(const uint32_t* b, int i) { return (b[i >> 5] >> (i & 31)) & 1u; }

__global__ void __launch_bounds__(kPatchWarps * 32)
k_tr_patch(sw_ragged_t m, int32_t* col_length, const int32_t* col_ptr, int32_t* src_pre, int32_t* src_slot,
           int32_t* plog, int cap, int32_t* rebuild, uint32_t* row_bits, uint32_t* col_bits, int32_t* dirty) {
  __shared__ int s_rows[kPatchRows];
  __shared__ int s_nd, s_abort;
  __shared__ int2 s_buf[kPatchWarps][kPatchCol];
  __shared__ int2 s_new[kPatchWarps][kPatchRows];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nt = plog[0], np = plog[1];
  const bool ovf = plog[2] != 0 || nt > cap || np > cap;
  if (nt == 0 && !ovf) {   // nothing changed
    if (tid == 0) plog[1] = 0;
    return;
  }
  if (ovf || nt > kPatchRows) {
    if (tid == 0) { *rebuild = 1; plog[0] = plog[1] = plog[2] = 0; }
    return;
  }
  const int* rows = plog + 4;
  const int* pairs = plog + 4 + cap;
  if (tid == 0) { s_nd = 0; s_abort = 0; }
  // changed rows, ascending (insertion sort of <= kPatchRows ids), and their bitmap
  __shared__ int s_nt;
  if (tid == 0) {
    int n = 0;
    for (int q = 0; q < nt; ++q) {
      const int v = rows[q];
      int r = n - 1;
      while (r >= 0 && s_rows[r] > v) --r;
      if (r >= 0 && s_rows[r] == v) continue;   // listed twice
      for (int t = n - 1; t > r; --t) s_rows[t + 1] = s_rows[t];
      s_rows[r + 1] = v;
      ++n;
    }
    s_nt = n;
  }
  __syncthreads();
  const int nu = s_nt;
  for (int q = tid; q < nu; q += blockDim.x) atomicOr(&row_bits[s_rows[q] >> 5], 1u << (s_rows[q] & 31));
  // dirty columns: removed targets and current targets of the changed rows
  auto mark = [&](int j) {
    const uint32_t b = 1u << (j & 31);
    if (!(atomicOr(&col_bits[j >> 5], b) & b)) dirty[atomicAdd(&s_nd, 1)] = j;
  };
  for (int q = tid; q < np; q += blockDim.x) mark(pairs[2 * q + 1]);
  for (int q = warp; q < nu; q += kPatchWarps) {
    const int i = s_rows[q];
    const int len = m.row_length[i];
    for (int s = lane; s < len; s += 32) mark(m.target[(int64_t)i * m.stride + s]);
  }
  __syncthreads();
  const int nd = s_nd;
  for (int d = warp; d < nd; d += kPatchWarps) {
    const int j = dirty[d];
    // the changed rows' synapses onto j, ascending (rows sorted; slots ascending)
    int nn = 0;
    for (int q = 0; q < nu; ++q) {
      const int i = s_rows[q];
      const int len = m.row_length[i];
      for (int s0 = 0; s0 < len; s0 += 32) {
        const int s = s0 + lane;
        const bool hit = s < len && m.target[(int64_t)i * m.stride + s] == j;
        const unsigned bal = __ballot_sync(SW_FULL_MASK, hit);
        if (hit) {
          const int pos = nn + __popc(bal & sw::lanemask_lt());
          if (pos < kPatchRows) s_new[warp][pos] = make_int2(i, s);
        }
        nn += __popc(bal);
      }
    }
    const int a = col_ptr[j], len0 = col_length[j], room = col_ptr[j + 1] - a;
    // kept entries (rows not changed) keep their order; count them per 32-chunk
    int kept_total = 0;
    for (int q0 = 0; q0 < len0; q0 += 32) {
      const int q = q0 + lane;
      int p = 0, sl = 0;
      bool keep = false;
      if (q < len0) {
        p = src_pre[a + q];
        sl = src_slot[a + q];
        keep = !bit_get(row_bits, p);
      }
      const unsigned bal = __ballot_sync(SW_FULL_MASK, keep);
      if (keep) {
        // output position: kept rank + changed-row entries ordered before it
        int before = 0;
        for (int u = 0; u < nn && u < kPatchRows; ++u) {
          const int2 e = s_new[warp][u];
          before += (e.x < p || (e.x == p && e.y < sl)) ? 1 : 0;
        }
        const int pos = kept_total + __popc(bal & sw::lanemask_lt()) + before;
        if (pos < kPatchCol) s_buf[warp][pos] = make_int2(p, sl);
      }
      kept_total += __popc(bal);
    }
    // the changed rows' entries: own rank + kept entries ordered before
    for (int u = lane; u < nn && u < kPatchRows; u += 32) {
      const int2 e = s_new[warp][u];
      int before = 0;
      for (int q = 0; q < len0; ++q) {
        const int p = src_pre[a + q];
        if (bit_get(row_bits, p)) continue;
        const int sl = src_slot[a + q];
        before += (p < e.x || (p == e.x && sl < e.y)) ? 1 : 0;
      }
      const int pos = u + before;
      if (pos < kPatchCol) s_buf[warp][pos] = e;
    }
    __syncwarp();
    const int L = kept_total + nn;
    if (L > room || L > kPatchCol || nn > kPatchRows) {
      if (lane == 0) atomicExch(&s_abort, 1);
    } else {
      for (int q = lane; q < L; q += 32) {
        src_pre[a + q] = s_buf[warp][q].x;
        src_slot[a + q] = s_buf[warp][q].y;
      }
      if (lane == 0) col_length[j] = L;
    }
    __syncwarp();
  }
  __syncthreads();
  // clear the bitmaps and the log for the next update
  for (int q = tid; q < nu; q += blockDim.x) row_bits[s_rows[q] >> 5] = 0u;
  for (int d = tid; d < nd; d += blockDim.x) col_bits[dirty[d] >> 5] = 0u;
  if (tid == 0) {
    if (s_abort) *rebuild = 1;
    plog[0] = plog[1] = plog[2] = 0;
  }
}

}  // namespace

extern "C" int64_t sw_transpose_patch_scratch_bytes(int32_t num_pre, int32_t num_post) {
  return ((int64_t)(num_pre + 31) / 32 + (num_post + 31) / 32 + num_post) * 4;
}

extern "C" int sw_transpose_patch(const sw_ragged_t* m, int32_t* col_length, const int32_t* col_ptr,
                                  int32_t* src_pre, int32_t* src_slot, int32_t* patch_log, int32_t cap,
                                  int32_t* rebuild, void* scratch, void* stream) {
  if (!m || !patch_log || !rebuild || !scratch || cap < 1) {
    sw::set_last_error("sw_transpose_patch: matrix, patch log, rebuild flag and scratch required");
    return SW_ERR_INVALID_ARG;
  }
  uint32_t* row_bits = (uint32_t*)scratch;                      // zero, left zero
  uint32_t* col_bits = row_bits + (m->num_pre + 31) / 32;       // zero, left zero
  int32_t* dirty = (int32_t*)(col_bits + (m->num_post + 31) / 32);
  k_tr_patch<<<1, kPatchWarps * 32, 0, (cudaStream_t)stream>>>(*m, col_length, col_ptr, src_pre, src_slot,
                                                               patch_log, cap, rebuild, row_bits, col_bits,
                                                               dirty);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_transpose_patch");
  return SW_OK;
}
