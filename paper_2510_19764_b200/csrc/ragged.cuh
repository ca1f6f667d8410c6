// Warp-per-row helpers on the padded ragged layout (connectivity.py:24-136).
#pragma once
#include "common.cuh"

namespace sw {

struct RowView {
  int32_t* target;   // target + i*stride
  int64_t off;       // i*stride, for the planes
};

// Move slot src -> dst in target and every plane (connectivity.py:121-125).
// All source values are loaded before any store, so the loads of one move
// are in flight together.
__device__ __forceinline__ void move_slot(const sw_ragged_t& m, int64_t off, int dst, int src) {
  const int32_t t = m.target[off + src];
  uint64_t v[SW_MAX_PLANES];
#pragma unroll
  for (int p = 0; p < SW_MAX_PLANES; ++p) {
    if (p < m.n_planes)
      v[p] = (m.plane_bytes[p] == 8) ? ((const uint64_t*)m.planes[p])[off + src]
                                     : (uint64_t)((const uint32_t*)m.planes[p])[off + src];
  }
  m.target[off + dst] = t;
#pragma unroll
  for (int p = 0; p < SW_MAX_PLANES; ++p) {
    if (p < m.n_planes) {
      if (m.plane_bytes[p] == 8) ((uint64_t*)m.planes[p])[off + dst] = v[p];
      else ((uint32_t*)m.planes[p])[off + dst] = (uint32_t)v[p];
    }
  }
}

// Zero every plane at one slot (add_synapse, connectivity.py:103-105).
__device__ __forceinline__ void zero_slot(const sw_ragged_t& m, int64_t off, int s) {
#pragma unroll
  for (int p = 0; p < SW_MAX_PLANES; ++p) {
    if (p < m.n_planes) {
      if (m.plane_bytes[p] == 8) ((uint64_t*)m.planes[p])[off + s] = 0ull;
      else ((uint32_t*)m.planes[p])[off + s] = 0u;
    }
  }
}

// Slot-aligned sign-cache update for the slots of one warp instruction
// (warp-uniform call): lanes sharing a cache word are combined, and one lane
// per word issues at most one atomicOr and one atomicAnd.
__device__ __forceinline__ void warp_cache_bits(uint32_t* cache_row, bool active, int slot, bool bit) {
  const int lane = threadIdx.x & 31;
  const int word = active ? (slot >> 5) : -1;
  const unsigned peers = __match_any_sync(0xffffffffu, word);
  const uint32_t b = active ? (1u << (slot & 31)) : 0u;
  const uint32_t s_or = __reduce_or_sync(peers, bit ? b : 0u);
  const uint32_t c_or = __reduce_or_sync(peers, bit ? 0u : b);
  if (active && lane == __ffs(peers) - 1) {
    if (s_or) atomicOr(&cache_row[word], s_or);
    if (c_or) atomicAnd(&cache_row[word], ~c_or);
  }
}

// Exact remove_slots permutation (connectivity.py:130-136).
// list[0..k) holds the marked slots of a row of length n in ASCENDING order.
// The t-th largest marked slot m_t (t = 1..k) that lies below n2 = n - k
// receives the content of resolve(n - t), where resolve(p) follows
// p -> n - rank(p) while p is itself marked.  All sources are >= n2 and all
// destinations < n2, so the gathers are independent and run lane-parallel.
// Padding beyond n2 is left unspecified (the reference leaves stale values).
__device__ __forceinline__ void warp_apply_removal(const sw_ragged_t& m, int64_t off,
                                                   const int* list, int n, int k,
                                                   uint32_t* cache_row = nullptr) {
  const int lane = threadIdx.x & 31;
  const int n2 = n - k;
  for (int t0 = 1; t0 <= k; t0 += 32) {
    const int t = t0 + lane;
    bool moved = false, cbit = false;
    int dst = 0;
    if (t <= k) {
      const int mt = list[k - t];
      if (mt < n2) {
        int p = n - t;
        while (true) {
          // binary search p among marked slots (list ascending)
          int lo = 0, hi = k - 1, q = -1;
          while (lo <= hi) {
            int mid = (lo + hi) >> 1;
            int v = list[mid];
            if (v == p) { q = mid; break; }
            if (v < p) lo = mid + 1; else hi = mid - 1;
          }
          if (q < 0) break;
          p = n - (k - q);   // rank(list[q]) = k - q
        }
        // the slot-aligned sign cache follows the move (sources are all in
        // the tail, destinations below it: no read sees a written word)
        const uint32_t cw = cache_row ? cache_row[p >> 5] : 0u;
        move_slot(m, off, mt, p);
        if (cache_row) {
          cbit = (cw >> (p & 31)) & 1u;
          moved = true;
          dst = mt;
        }
      }
    }
    if (cache_row) warp_cache_bits(cache_row, moved, dst, cbit);
  }
}

}  // namespace sw
