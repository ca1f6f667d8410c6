// DEEP R on the padded ragged layout: bitfield init, L1 nudge, eliminate,
// form (device histogram of the host draws + warp-batched row placement).
// Reference: sparsewire/deep_r.py:23-177, bitfield.py:19-96,
// connectivity.py:91-136, updates.py:309-372.
#include "common.cuh"
#include "ragged.cuh"
#include "sm100_async.cuh"

namespace {

constexpr int kWarps = 8;            // warps per block for warp-per-row kernels
constexpr int kThreads = kWarps * 32;

int rows_grid(int64_t rows) {
  int64_t g = (rows + kWarps - 1) / kWarps;
  const int64_t cap = 148 * 64;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

int flat_grid(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  const int64_t cap = 148 * 32;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

__device__ __forceinline__ bool bit_of(const uint64_t* row, int j) {
  return (row[j >> 6] >> (j & 63)) & 1ull;
}

// ---- Bitfield.randomize (bitfield.py:92-96) ----------------------------------
__global__ void k_bf_randomize(sw_bitfield_t bf, uint64_t key, uint64_t tail_mask) {
  const int64_t total = (int64_t)bf.num_pre * bf.words_per_row;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    uint64_t v = sw::draw(key, (uint64_t)x);
    if ((int)(x % bf.words_per_row) == bf.words_per_row - 1) v &= tail_mask;
    bf.words[x] = v;
  }
}

// conn bits := edges; sign bit set for w > 0, cleared for w < 0 (deep_r.py:56-64).
// Two launches, as the reference's two vector calls: phase 0 sets conn and
// the w > 0 sign bits, phase 1 clears the w < 0 ones, so with multapses of
// opposite sign the clear wins deterministically (deep_r.py:62-64).
__global__ void k_deepr_init_bits(sw_ragged_t m, int wp, sw_bitfield_t sign, sw_bitfield_t conn, int phase) {
  const int64_t total = (int64_t)m.num_pre * m.stride;
  const double* w = (const double*)m.planes[wp];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / m.stride;
    const int s = (int)(x - i * m.stride);
    if (s >= m.row_length[i]) continue;
    const int j = m.target[x];
    const uint64_t bit = 1ull << (j & 63);
    const double wv = w[x];
    if (phase == 0) {
      atomicOr((unsigned long long*)&conn.words[i * conn.words_per_row + (j >> 6)], bit);
      if (wv > 0.0) atomicOr((unsigned long long*)&sign.words[i * sign.words_per_row + (j >> 6)], bit);
    } else if (wv < 0.0) {
      atomicAnd((unsigned long long*)&sign.words[i * sign.words_per_row + (j >> 6)], ~bit);
    }
  }
}

// ---- l1_step (deep_r.py:68-77) -------------------------------------------------
__global__ void k_deepr_l1(sw_ragged_t m, int gp, sw_bitfield_t sign, const uint32_t* cache, double l1) {
  const int64_t total = (int64_t)m.num_pre * m.stride;
  double* g = (double*)m.planes[gp];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / m.stride;
    const int s = (int)(x - i * m.stride);
    if (s >= m.row_length[i]) continue;   // padding gets +-0.0 in the reference: no-op
    bool pos;
    if (cache) {
      const int cw = (m.stride + 31) >> 5;
      pos = (cache[i * cw + (s >> 5)] >> (s & 31)) & 1u;
    } else {
      pos = bit_of(sign.words + i * sign.words_per_row, m.target[x]);
    }
    g[x] = __dadd_rn(g[x], pos ? l1 : -l1);
  }
}

// ---- eliminate (deep_r.py:81-99) --------------------------------------------------
// Warp per row.  Mismatch scan (4x unrolled for memory-level parallelism),
// ascending marked-slot list in shared memory, conn-bit clears, then the exact
// chained-removal gather.
__global__ void __launch_bounds__(kThreads)
k_deepr_eliminate(sw_ragged_t m, int wp, sw_bitfield_t sign, sw_bitfield_t conn, int64_t* dormant,
                  uint32_t* cache) {
  extern __shared__ int s_lists[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* list = s_lists + warp * m.stride;
  const double* w = (const double*)m.planes[wp];
  const unsigned lt = sw::lanemask_lt();
  const int64_t step = (int64_t)gridDim.x * kWarps;
  int64_t i = (int64_t)blockIdx.x * kWarps + warp;
  int n_next = (i < m.num_pre) ? m.row_length[i] : 0;
  for (; i < m.num_pre; i += step) {
    const int n = n_next;
    // prefetch the next row's length: the row loop is otherwise a chain of
    // dependent round trips
    if (i + step < m.num_pre) n_next = m.row_length[i + step];
    const int64_t off = i * (int64_t)m.stride;
    const uint64_t* srow = sign.words + i * sign.words_per_row;
    uint64_t* crow = conn.words + i * conn.words_per_row;
    const int cw = (m.stride + 31) >> 5;
    uint32_t* cache_row = cache ? cache + i * (int64_t)cw : nullptr;
    int k = 0;
    constexpr int U = 8;   // 256 slots in flight per warp
    for (int base = 0; base < n; base += 32 * U) {
      int t[U];
      double wv[U];
      uint32_t cwd[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = base + u * 32 + lane;
        t[u] = 0;
        wv[u] = 0.0;
        cwd[u] = 0u;
        if (s < n) {
          t[u] = __ldg(m.target + off + s);
          wv[u] = __ldg(w + off + s);
          if (cache_row) cwd[u] = __ldg(cache_row + (s >> 5));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = base + u * 32 + lane;
        bool bit;
        if (cache_row) bit = (cwd[u] >> (s & 31)) & 1u;
        else bit = (s < n && wv[u] != 0.0) ? ((__ldg(srow + (t[u] >> 6)) >> (t[u] & 63)) & 1ull) : false;
        const bool mis = (s < n) && ((wv[u] < 0.0 && bit) || (wv[u] > 0.0 && !bit));
        if (mis)
          atomicAnd((unsigned long long*)&crow[t[u] >> 6], ~(1ull << (t[u] & 63)));
        const unsigned b = __ballot_sync(SW_FULL_MASK, mis);
        if (mis) list[k + __popc(b & lt)] = s;
        k += __popc(b);
      }
    }
    __syncwarp();
    if (lane == 0) dormant[i] = k;
    if (k > 0) {
      sw::warp_apply_removal(m, off, list, n, k, cache_row);
      if (lane == 0) m.row_length[i] = n - k;
    }
    __syncwarp();
  }
}

// ---- eliminate, vectorised scan (sign cache present, float64 weights, stride % 4 == 0) --
// Same semantics as k_deepr_eliminate.  The mismatch decision needs only the
// weight and the slot-aligned sign bit; the target is read for marked slots
// alone (conn-bit clear, moves), so the scan streams 8 B + 1 bit per synapse.
// Each lane owns 4 consecutive slots (two 16-byte loads) in each half of a
// 256-slot batch, so a warp keeps 2 KB of weights in flight per batch; the
// ascending marked-slot list is rebuilt from four ballots per half.
constexpr int kVW = 8;   // warps per block

__device__ __forceinline__ bool mismatch(double w, uint32_t bit) {
  return (w < 0.0 && bit) || (w > 0.0 && !bit);
}

__global__ void __launch_bounds__(kVW * 32, 5)
k_deepr_elim_vec(sw_ragged_t m, int wp, sw_bitfield_t conn, int64_t* dormant, uint32_t* cache) {
  extern __shared__ int s_lists[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* list = s_lists + warp * m.stride;
  const double* w = (const double*)m.planes[wp];
  const int cw = (m.stride + 31) >> 5;
  const int64_t step = (int64_t)gridDim.x * kVW;
  int64_t i = (int64_t)blockIdx.x * kVW + warp;
  int n_next = (i < m.num_pre) ? m.row_length[i] : 0;
  for (; i < m.num_pre; i += step) {
    const int n = n_next;
    if (i + step < m.num_pre) n_next = m.row_length[i + step];
    const int64_t off = i * (int64_t)m.stride;
    const double2* w2 = reinterpret_cast<const double2*>(w + off);
    const uint32_t* crow = cache + i * (int64_t)cw;
    uint64_t* cbits = conn.words + i * conn.words_per_row;
    int k = 0;
    for (int base = 0; base < n; base += 256) {
      double2 v[4];
      uint32_t word[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s0 = base + h * 128 + lane * 4;
        if (s0 < n) {
          v[2 * h] = __ldcs(w2 + (s0 >> 1));
          v[2 * h + 1] = __ldcs(w2 + (s0 >> 1) + 1);
          word[h] = __ldcs(crow + (s0 >> 5));
        } else {
          v[2 * h] = make_double2(0.0, 0.0);
          v[2 * h + 1] = make_double2(0.0, 0.0);
          word[h] = 0u;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s0 = base + h * 128 + lane * 4;
        const uint32_t wd = word[h] >> (s0 & 31);
        const double x[4] = {v[2 * h].x, v[2 * h].y, v[2 * h + 1].x, v[2 * h + 1].y};
        unsigned mine = 0u;   // bit j: slot s0 + j marked
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (s0 + j < n && mismatch(x[j], (wd >> j) & 1u)) mine |= 1u << j;
        if (__any_sync(SW_FULL_MASK, mine != 0u)) {
          // exclusive prefix of the per-lane counts (ascending slot order)
          const int cnt = __popc(mine);
          int pre = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(SW_FULL_MASK, pre, o);
            if (lane >= o) pre += t;
          }
          const int tot = __shfl_sync(SW_FULL_MASK, pre, 31);
          int pos = k + pre - cnt;
          for (unsigned mm = mine; mm; mm &= mm - 1) list[pos++] = s0 + __ffs(mm) - 1;
          k += tot;
        }
      }
    }
    __syncwarp();
    if (lane == 0) dormant[i] = k;
    if (k > 0) {
      // conn-bit clears of the whole row in one round of target loads
      for (int q = lane; q < k; q += 32) {
        const int t = __ldg(m.target + off + list[q]);
        atomicAnd((unsigned long long*)&cbits[t >> 6], ~(1ull << (t & 63)));
      }
      sw::warp_apply_removal(m, off, list, n, k, cache + i * (int64_t)cw);
      if (lane == 0) m.row_length[i] = n - k;
    }
    __syncwarp();
  }
}

// ---- eliminate in two kernels (sign cache + mark scratch) -------------------------
// k_deepr_elim_scan: pure streaming mismatch scan (weights + sign-cache
// words), warp per row; writes dormant[i] and, for rows with removals, the
// row's marked-slot bitmask marks[i, 0:ceil(n/32)].  k_deepr_elim_apply:
// warp per group of 32 rows, visits only rows with removals: ascending
// marked list from the bitmask, conn-bit clears, the exact chained removal.
// The scan then runs at streaming speed whatever the removal count, and the
// dependent round trips of the removals overlap across many warps.
constexpr int kSW_ = 8;   // warps per block (scan and apply)
constexpr int kSmallK = 8;   // rows with at most this many removals take the per-thread path
constexpr int kMoveBatch = 4;
__host__ __device__ __forceinline__ int small_k(int cw) { return 2 * cw < kSmallK ? 2 * cw : kSmallK; }

__global__ void __launch_bounds__(kSW_ * 32, 6)
k_deepr_elim_scan(sw_ragged_t m, int wp, int64_t* dormant, const uint32_t* cache, uint32_t* marks) {
  __shared__ uint32_t s_mask[kSW_][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* mask = s_mask[warp];
  const double* w = (const double*)m.planes[wp];
  const int cw = (m.stride + 31) >> 5;
  // same test as k_deepr_elim_apply: rows it handles per thread get a slot list
  bool lane_ok = m.n_planes == 4;
  for (int pl = 0; pl < 4 && lane_ok; ++pl) lane_ok = m.plane_bytes[pl] == 8;
  const int64_t step = (int64_t)gridDim.x * kSW_;
  int64_t i = (int64_t)blockIdx.x * kSW_ + warp;
  int n_next = (i < m.num_pre) ? m.row_length[i] : 0;
  mask[lane] = 0u;
  __syncwarp();
  for (; i < m.num_pre; i += step) {
    const int n = n_next;
    if (i + step < m.num_pre) n_next = m.row_length[i + step];
    const int64_t off = i * (int64_t)m.stride;
    const double2* w2 = reinterpret_cast<const double2*>(w + off);
    const uint32_t* crow = cache + i * (int64_t)cw;
    int k = 0;
    for (int base = 0; base < n; base += 256) {
      double2 v[4];
      uint32_t word[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s0 = base + h * 128 + lane * 4;
        if (s0 < n) {
          v[2 * h] = __ldcs(w2 + (s0 >> 1));
          v[2 * h + 1] = __ldcs(w2 + (s0 >> 1) + 1);
          word[h] = __ldcs(crow + (s0 >> 5));
        } else {
          v[2 * h] = make_double2(0.0, 0.0);
          v[2 * h + 1] = make_double2(0.0, 0.0);
          word[h] = 0u;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s0 = base + h * 128 + lane * 4;
        const uint32_t wd = word[h] >> (s0 & 31);
        const double x[4] = {v[2 * h].x, v[2 * h].y, v[2 * h + 1].x, v[2 * h + 1].y};
        unsigned mine = 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (s0 + j < n && mismatch(x[j], (wd >> j) & 1u)) mine |= 1u << j;
        if (__any_sync(SW_FULL_MASK, mine != 0u)) {
          if (mine) atomicOr(&mask[(s0 >> 5) & 31], mine << (s0 & 31));
          k += __reduce_add_sync(SW_FULL_MASK, __popc(mine));
        }
      }
    }
    if (lane == 0) dormant[i] = k;
    if (k > 0) {
      __syncwarp();
      const int nw = (n + 31) >> 5;
      const uint32_t mw = lane < nw ? mask[lane] : 0u;
      if (k <= small_k(cw) && lane_ok) {
        // few removals: the ascending slot list, packed 2 x uint16 per word
        const int c = __popc(mw);
        int pre = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(SW_FULL_MASK, pre, o);
          if (lane >= o) pre += t;
        }
        __syncwarp();
        uint16_t* lst = reinterpret_cast<uint16_t*>(mask);   // reuse the row mask buffer
        int p = pre - c;
        for (uint32_t mm = mw; mm; mm &= mm - 1) lst[p++] = (uint16_t)(lane * 32 + __ffs(mm) - 1);
        __syncwarp();
        if (lane < (k + 1) / 2) marks[i * (int64_t)cw + lane] = mask[lane];
      } else if (lane < nw) {
        marks[i * (int64_t)cw + lane] = mw;
      }
      __syncwarp();
      mask[lane] = 0u;
      __syncwarp();
    }
  }
}

// one thread per row: the exact chained removal of up to kSmallK slots
// (SURVEY App. D1).  The (dst, src) pairs are resolved in registers first,
// then every load of the row (marked targets, source target + planes +
// sign-cache words) is issued before any store.
__device__ __forceinline__ void lane_apply_removal(const sw_ragged_t& m, const sw_bitfield_t& conn,
                                                   uint32_t* cache, const uint32_t* marks, int cw,
                                                   int64_t i, int n, int k) {
  const int64_t off = i * (int64_t)m.stride;
  int mk[kSmallK];
#pragma unroll
  for (int q = 0; q < kSmallK; q += 2) {
    if (q < k) {
      const uint32_t wd = marks[i * (int64_t)cw + q / 2];
      mk[q] = (int)(wd & 0xffffu);
      mk[q + 1] = (int)(wd >> 16);
    }
  }
  const int n2 = n - k;
  int dst[kSmallK], src[kSmallK];
#pragma unroll
  for (int t = 1; t <= kSmallK; ++t) {
    dst[t - 1] = -1;
    if (t > k) continue;
    const int mt = mk[k - t];
    if (mt >= n2) continue;
    int p = n - t;
#pragma unroll 1
    for (int guard = 0; guard <= kSmallK; ++guard) {
      int idx = -1;
#pragma unroll
      for (int q = 0; q < kSmallK; ++q)
        if (q < k && mk[q] == p) idx = q;
      if (idx < 0) break;
      p = n - (k - idx);
    }
    dst[t - 1] = mt;
    src[t - 1] = p;
  }
  // conn clears: every marked slot's target, read before any move
  int tm[kSmallK];
#pragma unroll
  for (int q = 0; q < kSmallK; ++q)
    if (q < k) tm[q] = m.target[off + mk[q]];
  uint64_t* crow = conn.words + i * conn.words_per_row;
#pragma unroll
  for (int q = 0; q < kSmallK; ++q)
    if (q < k) atomicAnd((unsigned long long*)&crow[tm[q] >> 6], ~(1ull << (tm[q] & 63)));
  // moves, kMoveBatch at a time: all loads of a batch, then its stores
  const uint32_t* crow_s = cache + i * (int64_t)cw;
  uint32_t* crow_w = cache + i * (int64_t)cw;
#pragma unroll
  for (int g = 0; g < kSmallK; g += kMoveBatch) {
    if (g >= k) break;
    int st[kMoveBatch];
    uint64_t pv[kMoveBatch][4];
    uint32_t cwd[kMoveBatch];
#pragma unroll
    for (int u = 0; u < kMoveBatch; ++u) {
      const int q = g + u;
      if (dst[q] >= 0) {
        st[u] = m.target[off + src[q]];
#pragma unroll
        for (int pl = 0; pl < 4; ++pl)
          pv[u][pl] = ((const uint64_t*)m.planes[pl])[off + src[q]];
        cwd[u] = crow_s[src[q] >> 5];
      }
    }
#pragma unroll
    for (int u = 0; u < kMoveBatch; ++u) {
      const int q = g + u;
      if (dst[q] >= 0) {
        const int d = dst[q];
        m.target[off + d] = st[u];
#pragma unroll
        for (int pl = 0; pl < 4; ++pl) ((uint64_t*)m.planes[pl])[off + d] = pv[u][pl];
        if ((cwd[u] >> (src[q] & 31)) & 1u) atomicOr(&crow_w[d >> 5], 1u << (d & 31));
        else atomicAnd(&crow_w[d >> 5], ~(1u << (d & 31)));
      }
    }
  }
  m.row_length[i] = n2;
}

__global__ void __launch_bounds__(kSW_ * 32)
k_deepr_elim_apply(sw_ragged_t m, sw_bitfield_t conn, const int64_t* dormant, uint32_t* cache,
                   const uint32_t* marks) {
  extern __shared__ int s_lists[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* list = s_lists + warp * m.stride;
  const int cw = (m.stride + 31) >> 5;
  const unsigned lt = sw::lanemask_lt();
  bool lane_ok = m.n_planes == 4;
  for (int pl = 0; pl < 4 && lane_ok; ++pl) lane_ok = m.plane_bytes[pl] == 8;
  for (int64_t g0 = ((int64_t)blockIdx.x * kSW_ + warp) * 32; g0 < m.num_pre;
       g0 += (int64_t)gridDim.x * kSW_ * 32) {
    const int64_t gi = g0 + lane;
    const int my_k = gi < m.num_pre ? (int)dormant[gi] : 0;
    const int my_n = my_k ? m.row_length[gi] : 0;
    // rows with few removals: one thread per row (four 8-byte planes)
    const int ks = lane_ok ? small_k(cw) : 0;
    if (my_k > 0 && my_k <= ks) lane_apply_removal(m, conn, cache, marks, cw, gi, my_n, my_k);
    unsigned active = __ballot_sync(SW_FULL_MASK, my_k > ks);
    while (active) {
      const int src = __ffs(active) - 1;
      active &= active - 1;
      const int64_t i = g0 + src;
      const int k = __shfl_sync(SW_FULL_MASK, my_k, src);
      const int n = __shfl_sync(SW_FULL_MASK, my_n, src);
      const int64_t off = i * (int64_t)m.stride;
      // ascending marked list from the bitmask (lane = word)
      const int nw = (n + 31) >> 5;
      int pos = 0;
      for (int w0 = 0; w0 < nw; w0 += 32) {
        const uint32_t mw = (w0 + lane < nw) ? marks[i * (int64_t)cw + w0 + lane] : 0u;
        const int c = __popc(mw);
        int pre = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(SW_FULL_MASK, pre, o);
          if (lane >= o) pre += t;
        }
        int p = pos + pre - c;
        for (uint32_t mm = mw; mm; mm &= mm - 1) list[p++] = (w0 + lane) * 32 + __ffs(mm) - 1;
        pos += __shfl_sync(SW_FULL_MASK, pre, 31);
      }
      __syncwarp();
      uint64_t* cbits = conn.words + i * conn.words_per_row;
      for (int q = lane; q < k; q += 32) {
        const int t = __ldg(m.target + off + list[q]);
        atomicAnd((unsigned long long*)&cbits[t >> 6], ~(1ull << (t & 63)));
      }
      sw::warp_apply_removal(m, off, list, n, k, cache + i * (int64_t)cw);
      if (lane == 0) m.row_length[i] = n - k;
      __syncwarp();
    }
  }
  (void)lt;
}

// build the slot-aligned sign cache: bit s of row i = sign(i, target[i, s])
__global__ void k_sign_cache(sw_ragged_t m, sw_bitfield_t sign, uint32_t* cache) {
  const int cw = (m.stride + 31) >> 5;
  const int64_t total = (int64_t)m.num_pre * cw;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / cw;
    const int w0 = (int)(x - i * cw) * 32;
    const int n = m.row_length[i];
    uint32_t v = 0u;
    for (int b = 0; b < 32 && w0 + b < n; ++b) {
      const int j = m.target[i * m.stride + w0 + b];
      v |= (uint32_t)bit_of(sign.words + i * sign.words_per_row, j) << b;
    }
    cache[x] = v;
  }
}

// generic removal of caller-marked slots (remove_slots semantics)
__global__ void __launch_bounds__(kThreads)
k_remove_marked(sw_ragged_t m, const uint8_t* marked, int64_t* removed) {
  extern __shared__ int s_lists[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* list = s_lists + warp * m.stride;
  const unsigned lt = sw::lanemask_lt();
  for (int64_t i = (int64_t)blockIdx.x * kWarps + warp; i < m.num_pre;
       i += (int64_t)gridDim.x * kWarps) {
    const int n = m.row_length[i];
    const int64_t off = i * (int64_t)m.stride;
    int k = 0;
    for (int base = 0; base < n; base += 32) {
      const int s = base + lane;
      const bool mk = s < n && marked[off + s];
      const unsigned b = __ballot_sync(SW_FULL_MASK, mk);
      if (mk) list[k + __popc(b & lt)] = s;
      k += __popc(b);
    }
    __syncwarp();
    if (removed && lane == 0) removed[i] = k;
    if (k > 0) {
      sw::warp_apply_removal(m, off, list, n, k);
      if (lane == 0) m.row_length[i] = n - k;
    }
    __syncwarp();
  }
}

// ---- form: host-phase draws as a device histogram (deep_r.py:110-121) --------------
__global__ void k_sum_i64(const int64_t* x, int64_t n, int64_t* out) {
  int64_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += x[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(SW_FULL_MASK, acc, o);
  __shared__ int64_t part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(SW_FULL_MASK, acc, o);
    if (threadIdx.x == 0 && acc) atomicAdd((unsigned long long*)out, (unsigned long long)acc);
  }
}

// D draws of uniform_int(num_pre) on the host stream: draw c lands in row
// h mod P when valid.  Invalid (rejected) counters are counted; the serial
// fix-up kernel then continues from counter D until D valid draws exist.
// Row-sharded form (world > 1): this rank draws only counters
// [D*rank/world, D*(rank+1)/world) into a histogram over all rows; the
// per-rank histograms are then reduce-scattered by row owner.
__global__ void k_form_hist(int64_t* counters, uint64_t key, uint64_t P, uint64_t rem,
                            int32_t* act, int rank, int world) {
  const int64_t D = counters[0];
  const int64_t c_lo = D * rank / world, c_hi = D * (rank + 1) / world;
  const bool pow2 = (P & (P - 1)) == 0;
  int64_t rej = 0;
  for (int64_t c = c_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < c_hi;
       c += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = sw::draw(key, (uint64_t)c);
    if (sw::draw_valid(h, rem)) {
      const uint64_t r = pow2 ? (h & (P - 1)) : (h % P);
      atomicAdd(act + r, 1);
    } else {
      ++rej;
    }
  }
  if (rej) atomicAdd((unsigned long long*)&counters[2], (unsigned long long)rej);
}

__global__ void k_form_hist_fix(int64_t* counters, uint64_t key, uint64_t P, uint64_t rem,
                                int32_t* act) {
  int64_t need = counters[2];
  uint64_t c = (uint64_t)counters[0];
  while (need > 0) {
    const uint64_t h = sw::draw(key, c++);
    if (sw::draw_valid(h, rem)) { act[h % P] += 1; --need; }
  }
}

// ---- form: row phase (deep_r.py:126-145) ------------------------------
// Warp per row.  Lane l evaluates draw #(ctr + l) of the row stream; the
// reference's sequential inner loop is replayed exactly over the 32 lanes:
// valid draws are iterations, a candidate is placed unless an earlier lane
// of the batch already placed the same post (match_any), the failure streak
// resets per activation and ends it after num_post misses, a full row stops
// all remaining activations without consuming draws.
// One thread per row: the sequential loop of deep_r.py:126-145 verbatim
// (draw by draw with exact rejection, failure streak per activation, full
// row stops all remaining activations without draws).  Posts placed earlier
// in this row are also checked from registers, so the result never depends
// on when the thread's own conn-bit atomics become visible.
constexpr int kFormSmall = 2;

__device__ __forceinline__ void lane_form_row(const sw_ragged_t& m, const sw_bitfield_t& conn,
                                              int excl_diag, uint64_t row_base, int64_t row0, int64_t i,
                                              int acts, int len, int64_t* unplaced, int64_t* counters,
                                              const sw_bitfield_t& sign, uint32_t* cache, int N,
                                              uint64_t rem, bool pow2, int cap) {
  const int64_t off = i * (int64_t)m.stride;
  uint64_t* crow = conn.words + i * conn.words_per_row;
  // row0: global index of local row 0 (row-sharded matrices): the row stream
  // and the diagonal are those of the global row
  const uint64_t key = sw::child_key(row_base, (uint64_t)(row0 + i));
  uint64_t ctr = 0;
  int placed[kFormSmall];
  int np = 0, a = 0, streak = 0, unpl = 0;
  while (a < acts) {
    if (len >= cap) { unpl += acts - a; break; }
    const uint64_t h = sw::draw(key, ctr++);
    if (!sw::draw_valid(h, rem)) continue;   // a rejected draw is not an iteration
    const int j = (int)(pow2 ? (h & (uint64_t)(N - 1)) : (h % (uint64_t)N));
    bool fail = excl_diag && (int64_t)j == row0 + i;
    bool sbit = false;
    if (!fail) {
      const uint64_t cw = __ldcg(crow + (j >> 6));
      if (cache) sbit = (__ldg(sign.words + i * sign.words_per_row + (j >> 6)) >> (j & 63)) & 1ull;
      fail = (cw >> (j & 63)) & 1ull;
#pragma unroll
      for (int q = 0; q < kFormSmall; ++q) fail |= (q < np && placed[q] == j);
    }
    if (fail) {
      if (++streak == N) { ++unpl; ++a; streak = 0; }
      continue;
    }
    m.target[off + len] = j;
    sw::zero_slot(m, off, len);
    atomicOr((unsigned long long*)(crow + (j >> 6)), 1ull << (j & 63));
    if (cache) {
      uint32_t* cr = cache + i * (int64_t)((m.stride + 31) >> 5);
      if (sbit) atomicOr(&cr[len >> 5], 1u << (len & 31));
      else atomicAnd(&cr[len >> 5], ~(1u << (len & 31)));
    }
    placed[np < kFormSmall ? np : kFormSmall - 1] = j;
    ++np;
    ++len;
    ++a;
    streak = 0;
  }
  m.row_length[i] = len;
  unplaced[i] = unpl;
  if (unpl) atomicAdd((unsigned long long*)&counters[1], (unsigned long long)unpl);
}

__global__ void __launch_bounds__(kThreads, 8)
k_deepr_form_rows(sw_ragged_t m, sw_bitfield_t conn, int excl_diag, uint64_t row_base, int64_t row0,
                  const int32_t* act, int64_t* unplaced, int64_t* counters, sw_bitfield_t sign,
                  uint32_t* cache) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = sw::lanemask_lt();
  const int N = m.num_post;
  const uint64_t rem = sw::reject_rem((uint64_t)N);
  const bool pow2 = (N & (N - 1)) == 0;
  const int cap = m.max_row_length;
  // warp handles groups of 32 rows: activations loaded and zero-unplaced
  // written coalesced, then the active rows of the group one by one
  for (int64_t g0 = ((int64_t)blockIdx.x * kWarps + warp) * 32; g0 < m.num_pre;
       g0 += (int64_t)gridDim.x * kWarps * 32) {
    const int64_t gi = g0 + lane;
    const int my_act = gi < m.num_pre ? act[gi] : 0;
    const int my_len = (gi < m.num_pre && my_act) ? m.row_length[gi] : 0;
    if (gi < m.num_pre && my_act == 0) unplaced[gi] = 0;
    // rows with few activations: one thread per row, all 32 rows in flight
    if (my_act > 0 && my_act <= kFormSmall)
      lane_form_row(m, conn, excl_diag, row_base, row0, gi, my_act, my_len, unplaced, counters, sign, cache,
                    N, rem, pow2, cap);
    unsigned active = __ballot_sync(SW_FULL_MASK, my_act > kFormSmall);
    while (active) {
    const int src_lane = __ffs(active) - 1;
    active &= active - 1;
    const int64_t i = g0 + src_lane;
    const int acts = __shfl_sync(SW_FULL_MASK, my_act, src_lane);
    const int64_t off = i * (int64_t)m.stride;
    uint64_t* crow = conn.words + i * conn.words_per_row;
    const uint64_t key = sw::child_key(row_base, (uint64_t)(row0 + i));
    uint64_t ctr = 0;
    int len = __shfl_sync(SW_FULL_MASK, my_len, src_lane);
    int a = 0, streak = 0, unpl = 0;
    while (a < acts) {
      if (len >= cap) { unpl += acts - a; break; }
      // lanes evaluated this batch: when no activation can exhaust its
      // num_post iterations here, only about `need` draws can be used, so
      // later lanes are neither drawn nor probed (the batch then consumes
      // exactly L counters)
      const int need0 = min(acts - a, cap - len);
      const int L = (streak + 32 < N) ? min(32, need0 + 4) : 32;
      const bool live = lane < L;
      const uint64_t h = live ? sw::draw(key, ctr + lane) : 0ull;
      const bool valid = live && sw::draw_valid(h, rem);
      const int j = (int)(pow2 ? (h & (uint64_t)(N - 1)) : (h % (uint64_t)N));
      bool cand = valid && !(excl_diag && (int64_t)j == row0 + i);
      // the candidate's conn word and (for the slot-aligned cache) its sign
      // word are fetched together: one memory round trip per batch
      bool sbit = false;
      if (cand) {
        const uint64_t cwd = __ldcg(crow + (j >> 6));
        if (cache) sbit = (__ldg(sign.words + i * sign.words_per_row + (j >> 6)) >> (j & 63)) & 1ull;
        cand = !((cwd >> (j & 63)) & 1ull);
      }
      const unsigned peers = __match_any_sync(SW_FULL_MASK, cand ? j : (N + lane));
      const bool first = cand && !(peers & lt);
      const unsigned vmask = __ballot_sync(SW_FULL_MASK, valid);
      const unsigned fmask = __ballot_sync(SW_FULL_MASK, first);
      unsigned placed;
      int consumed;   // lanes (counters) consumed by this batch
      if (streak + 32 < N) {
        // fast path: no activation can exhaust its num_post iterations here
        const int need = min(acts - a, cap - len);
        const int nf = __popc(fmask);
        if (nf <= need) {
          placed = fmask;
          consumed = L;
          a += nf;
          len += nf;
          if (fmask) {
            const int hi = 31 - __clz(fmask);
            const unsigned above = (hi == 31) ? 0u : (~0u << (hi + 1));
            streak = __popc(vmask & ~fmask & above);
          } else {
            streak += __popc(vmask);
          }
        } else {
          // lane of the need-th placement
          unsigned f = fmask;
          for (int q = 1; q < need; ++q) f &= f - 1;
          const int L = __ffs(f) - 1;
          placed = fmask & ((L == 31) ? ~0u : ((2u << L) - 1u));
          consumed = L + 1;
          a += need;
          len += need;
          streak = 0;
        }
      } else {
        // exact serial walk over the lanes (small num_post)
        placed = 0u;
        consumed = 32;
        unsigned vm = vmask;
        while (vm) {
          const int l = __ffs(vm) - 1;
          vm &= vm - 1;
          if ((fmask >> l) & 1u) {
            placed |= 1u << l;
            ++a; ++len; streak = 0;
            if (a == acts || len == cap) { consumed = l + 1; break; }
          } else {
            if (++streak == N) {
              ++unpl; ++a; streak = 0;
              if (a == acts) { consumed = l + 1; break; }
            }
          }
        }
      }
      const bool pl = (placed >> lane) & 1u;
      const int slot = len - __popc(placed) + __popc(placed & lt);
      if (pl) {
        m.target[off + slot] = j;
        sw::zero_slot(m, off, slot);
        atomicOr((unsigned long long*)(crow + (j >> 6)), 1ull << (j & 63));
      }
      if (cache) sw::warp_cache_bits(cache + i * (int64_t)((m.stride + 31) >> 5), pl, slot, sbit);
      ctr += (uint64_t)consumed;
      __syncwarp();
    }
    if (lane == 0) {
      m.row_length[i] = len;
      unplaced[i] = unpl;
      if (unpl) atomicAdd((unsigned long long*)&counters[1], (unsigned long long)unpl);
    }
    }
  }
}

int elim_smem(const sw_ragged_t* m) { return kWarps * m->stride * (int)sizeof(int); }

int check_ragged(const sw_ragged_t* m, const char* where) {
  if (!m || m->num_pre < 0 || m->stride < 1 || m->n_planes < 0 || m->n_planes > SW_MAX_PLANES) {
    sw::set_last_error(where);
    return SW_ERR_INVALID_ARG;
  }
  return SW_OK;
}

}  // namespace

extern "C" int sw_bitfield_randomize(const sw_bitfield_t* bf, uint64_t key, void* stream) {
  const int tail = bf->num_post - (bf->words_per_row - 1) * 64;
  const uint64_t mask = tail >= 64 ? ~0ull : ((1ull << tail) - 1ull);
  const int64_t total = (int64_t)bf->num_pre * bf->words_per_row;
  if (total == 0) return SW_OK;
  k_bf_randomize<<<flat_grid(total, 256), 256, 0, (cudaStream_t)stream>>>(*bf, key, mask); sw::count_launch();
  SW_CHECK_LAUNCH("sw_bitfield_randomize");
  return SW_OK;
}

extern "C" int sw_deepr_init_bitfields(const sw_ragged_t* m, int32_t wp, const sw_bitfield_t* sign,
                                       const sw_bitfield_t* conn, uint64_t sign_key, void* stream) {
  if (int s = check_ragged(m, "sw_deepr_init_bitfields: bad matrix")) return s;
  int s = sw_bitfield_randomize(sign, sign_key, stream);
  if (s) return s;
  cudaMemsetAsync(conn->words, 0, (size_t)conn->num_pre * conn->words_per_row * 8, (cudaStream_t)stream);
  const int64_t total = (int64_t)m->num_pre * m->stride;
  if (total == 0) return SW_OK;
  for (int phase = 0; phase < 2; ++phase) {
    k_deepr_init_bits<<<flat_grid(total, 256), 256, 0, (cudaStream_t)stream>>>(*m, wp, *sign, *conn, phase);
    sw::count_launch();
  }
  SW_CHECK_LAUNCH("sw_deepr_init_bitfields");
  return SW_OK;
}

extern "C" int sw_deepr_l1(const sw_ragged_t* m, int32_t gp, const sw_bitfield_t* sign,
                           const uint32_t* sign_slot, double l1, void* stream) {
  if (int s = check_ragged(m, "sw_deepr_l1: bad matrix")) return s;
  if (l1 == 0.0) return SW_OK;   // deep_r.py:74-75
  const int64_t total = (int64_t)m->num_pre * m->stride;
  if (total == 0) return SW_OK;
  k_deepr_l1<<<flat_grid(total, 256), 256, 0, (cudaStream_t)stream>>>(*m, gp, *sign, sign_slot, l1); sw::count_launch();
  SW_CHECK_LAUNCH("sw_deepr_l1");
  return SW_OK;
}

static int set_smem(const void* fn, int bytes) {
  if (bytes > 48 * 1024) {
    if (bytes > 227 * 1024) { sw::set_last_error("row capacity too large for shared-memory slot lists"); return SW_ERR_INVALID_ARG; }
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  }
  return SW_OK;
}

extern "C" int sw_deepr_eliminate(const sw_ragged_t* m, int32_t wp, const sw_bitfield_t* sign,
                                  const sw_bitfield_t* conn, int64_t* dormant, uint32_t* sign_slot,
                                  uint32_t* mark_scratch, void* stream) {
  if (int s = check_ragged(m, "sw_deepr_eliminate: bad matrix")) return s;
  if (m->num_pre == 0) return SW_OK;
  if (sign_slot && mark_scratch && m->plane_bytes[wp] == 8 && m->stride % 4 == 0 &&
      m->stride <= 1024 && ((uintptr_t)m->planes[wp] % 16) == 0) {
    cudaStream_t st = (cudaStream_t)stream;
    int64_t g = (m->num_pre + kSW_ - 1) / kSW_;
    if (g > 148 * 48) g = 148 * 48;
    k_deepr_elim_scan<<<(int)g, kSW_ * 32, 0, st>>>(*m, wp, dormant, sign_slot, mark_scratch); sw::count_launch();
    const int smem = kSW_ * m->stride * (int)sizeof(int);
    if (int s = set_smem((const void*)k_deepr_elim_apply, smem)) return s;
    int64_t g2 = (m->num_pre + kSW_ * 32 - 1) / (kSW_ * 32);
    if (g2 > 148 * 8) g2 = 148 * 8;
    k_deepr_elim_apply<<<(int)g2, kSW_ * 32, smem, st>>>(*m, *conn, dormant, sign_slot, mark_scratch); sw::count_launch();
    SW_CHECK_LAUNCH("sw_deepr_eliminate");
    return SW_OK;
  }
  if (sign_slot && m->plane_bytes[wp] == 8 && m->stride % 4 == 0 &&
      ((uintptr_t)m->planes[wp] % 16) == 0) {
    const int smem = kVW * m->stride * (int)sizeof(int);
    if (int s = set_smem((const void*)k_deepr_elim_vec, smem)) return s;
    int64_t g = (m->num_pre + kVW - 1) / kVW;
    if (g > 148 * 40) g = 148 * 40;
    k_deepr_elim_vec<<<(int)g, kVW * 32, smem, (cudaStream_t)stream>>>(*m, wp, *conn, dormant, sign_slot); sw::count_launch();
    SW_CHECK_LAUNCH("sw_deepr_eliminate");
    return SW_OK;
  }
  const int smem = elim_smem(m);
  if (int s = set_smem((const void*)k_deepr_eliminate, smem)) return s;
  k_deepr_eliminate<<<rows_grid(m->num_pre), kThreads, smem, (cudaStream_t)stream>>>(*m, wp, *sign, *conn, dormant, sign_slot); sw::count_launch();
  SW_CHECK_LAUNCH("sw_deepr_eliminate");
  return SW_OK;
}

extern "C" int sw_deepr_sign_cache_build(const sw_ragged_t* m, const sw_bitfield_t* sign,
                                         uint32_t* sign_slot, void* stream) {
  const int64_t total = (int64_t)m->num_pre * ((m->stride + 31) / 32);
  if (total == 0) return SW_OK;
  k_sign_cache<<<flat_grid(total, 256), 256, 0, (cudaStream_t)stream>>>(*m, *sign, sign_slot); sw::count_launch();
  SW_CHECK_LAUNCH("sw_deepr_sign_cache_build");
  return SW_OK;
}

extern "C" int sw_ragged_remove_marked(const sw_ragged_t* m, const uint8_t* marked, int64_t* removed,
                                       void* stream) {
  if (int s = check_ragged(m, "sw_ragged_remove_marked: bad matrix")) return s;
  if (m->num_pre == 0) return SW_OK;
  const int smem = elim_smem(m);
  if (int s = set_smem((const void*)k_remove_marked, smem)) return s;
  k_remove_marked<<<rows_grid(m->num_pre), kThreads, smem, (cudaStream_t)stream>>>(*m, marked, removed); sw::count_launch();
  SW_CHECK_LAUNCH("sw_ragged_remove_marked");
  return SW_OK;
}

extern "C" int sw_deepr_form_pass(const sw_ragged_t* m, const sw_bitfield_t* conn, int32_t excl_diag,
                                  const int64_t* pending_src, uint64_t host_key, uint64_t row_base,
                                  int32_t* act, int64_t* unplaced, int64_t* counters,
                                  const sw_bitfield_t* sign, uint32_t* sign_slot, void* stream) {
  if (int s = check_ragged(m, "sw_deepr_form_pass: bad matrix")) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t P = m->num_pre;
  cudaMemsetAsync(counters, 0, 4 * sizeof(int64_t), st);
  if (P == 0) return SW_OK;
  cudaMemsetAsync(act, 0, (size_t)P * sizeof(int32_t), st);
  k_sum_i64<<<flat_grid(P, 256), 256, 0, st>>>(pending_src, P, counters); sw::count_launch();
  const uint64_t rem = sw::reject_rem((uint64_t)P);
  k_form_hist<<<148 * 8, 256, 0, st>>>(counters, host_key, (uint64_t)P, rem, act, 0, 1); sw::count_launch();
  if (rem != 0) { k_form_hist_fix<<<1, 1, 0, st>>>(counters, host_key, (uint64_t)P, rem, act); sw::count_launch(); }
  k_deepr_form_rows<<<rows_grid(P), kThreads, 0, st>>>(*m, *conn, excl_diag, row_base, 0, act, unplaced, counters,
      sign ? *sign : sw_bitfield_t{nullptr, 0, 0, 0}, sign ? sign_slot : nullptr); sw::count_launch();
  SW_CHECK_LAUNCH("sw_deepr_form_pass");
  return SW_OK;
}

// Sign-flip injection for the connectivity-update microbenchmark (SURVEY
// 8(d) M-update recipe): valid slot (i, s) flips w when uniform01 draw
// #(i*stride + s) of `key` is below prob.
__global__ void k_flip_signs(sw_ragged_t m, int wp, uint64_t key, double prob) {
  const int64_t total = (int64_t)m.num_pre * m.stride;
  double* w = (double*)m.planes[wp];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / m.stride;
    if ((int)(x - i * m.stride) >= m.row_length[i]) continue;
    if (sw::u01(sw::draw(key, (uint64_t)x)) < prob) w[x] = -w[x];
  }
}

extern "C" int sw_flip_signs(const sw_ragged_t* m, int32_t plane, uint64_t key, double prob, void* stream) {
  const int64_t total = (int64_t)m->num_pre * m->stride;
  if (total == 0) return SW_OK;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_flip_signs<<<(int)g, 256, 0, (cudaStream_t)stream>>>(*m, plane, key, prob); sw::count_launch();
  SW_CHECK_LAUNCH("sw_flip_signs");
  return SW_OK;
}

// ---- row-sharded form pass (SURVEY 8e M-update): the phases of
// sw_deepr_form_pass split at its collectives.  The host all-reduces
// counters[0] (D) after sw_deepr_form_pending, counters[2] (rejected draws)
// after sw_deepr_form_hist_chunk, reduce-scatters the num_pre_global
// histogram by row owner, and all-reduces counters[1] (unplaced) after
// sw_deepr_form_rows_shard.  Integer sums: bit-exact with the unsharded pass.
extern "C" int sw_deepr_form_pending(const int64_t* pending_src, int64_t num_rows, int64_t* counters,
                                     void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(counters, 0, 4 * sizeof(int64_t), st);
  if (num_rows > 0) {
    k_sum_i64<<<flat_grid(num_rows, 256), 256, 0, st>>>(pending_src, num_rows, counters); sw::count_launch();
  }
  SW_CHECK_LAUNCH("sw_deepr_form_pending");
  return SW_OK;
}

extern "C" int sw_deepr_form_hist_chunk(int64_t* counters, uint64_t host_key, int64_t num_pre_global,
                                        int32_t rank, int32_t world, int32_t* act_full, void* stream) {
  if (world < 1 || rank < 0 || rank >= world || num_pre_global < 0) {
    sw::set_last_error("sw_deepr_form_hist_chunk: bad rank/world");
    return SW_ERR_INVALID_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (num_pre_global == 0) return SW_OK;
  cudaMemsetAsync(act_full, 0, (size_t)num_pre_global * sizeof(int32_t), st);
  const uint64_t rem = sw::reject_rem((uint64_t)num_pre_global);
  k_form_hist<<<148 * 8, 256, 0, st>>>(counters, host_key, (uint64_t)num_pre_global, rem, act_full, rank, world);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_deepr_form_hist_chunk");
  return SW_OK;
}

extern "C" int sw_deepr_form_hist_fix(int64_t* counters, uint64_t host_key, int64_t num_pre_global,
                                      int32_t* act_full, void* stream) {
  const uint64_t rem = sw::reject_rem((uint64_t)num_pre_global);
  if (num_pre_global == 0 || rem == 0) return SW_OK;   // no draw can be rejected
  k_form_hist_fix<<<1, 1, 0, (cudaStream_t)stream>>>(counters, host_key, (uint64_t)num_pre_global, rem, act_full);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_deepr_form_hist_fix");
  return SW_OK;
}

extern "C" int sw_deepr_form_rows_shard(const sw_ragged_t* m, const sw_bitfield_t* conn, int32_t excl_diag,
                                        uint64_t row_base, int64_t row0, const int32_t* act, int64_t* unplaced,
                                        int64_t* counters, const sw_bitfield_t* sign, uint32_t* sign_slot,
                                        void* stream) {
  if (int s = check_ragged(m, "sw_deepr_form_rows_shard: bad matrix")) return s;
  if (m->num_pre == 0) return SW_OK;
  k_deepr_form_rows<<<rows_grid(m->num_pre), kThreads, 0, (cudaStream_t)stream>>>(*m, *conn, excl_diag, row_base,
      row0, act, unplaced, counters, sign ? *sign : sw_bitfield_t{nullptr, 0, 0, 0}, sign ? sign_slot : nullptr);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_deepr_form_rows_shard");
  return SW_OK;
}
