// One 0.1 ms step of the topographic-map model (topomap.py:419-452) as four
// launches with all step state on the device (graph-capturable):
//   k_tm_neurons  Poisson source spikes (neurons.py:189-195, counter =
//                 step*n + node) and the conductance-LIF target update
//                 (neurons.py:137-148) with last step's pending input;
//   k_tm_prop     ordered propagation of both projections through their
//                 transposes into pending (ff then lat, topomap.py:433-437),
//                 fused with the STDP trace decays (plasticity.py:64-66);
//   k_tm_pre      STDP depression of the spiking source rows (ff) and
//                 spiking target rows (lat), then x += 1 (plasticity.py:68-81);
//   k_tm_post     STDP potentiation through the transposes for the spiking
//                 targets (warp per spiking post), then y += 1
//                 (plasticity.py:83-95); step += 1.
#include "common.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#ifndef SW_TM_NODES_PER_CTA
#define SW_TM_NODES_PER_CTA 512
#endif
#ifndef SW_TM_CG_SYNC
#define SW_TM_CG_SYNC 1
#endif

namespace {

__device__ __forceinline__ bool bit(const uint32_t* b, int i) { return (b[i >> 5] >> (i & 31)) & 1u; }

// ---- phase bodies (grid-stride over [t0, n) with step dt) --------------------------
__device__ __forceinline__ void tm_neurons(const sw_topomap_step_t& S, int64_t k, int t0, int dt) {
  const int lane = threadIdx.x & 31;
  const int n = S.n;
  // warp-aligned grid stride so that a warp's 32 nodes form one spike word
  for (int base = t0 & ~31; base < n; base += dt) {
    const int x = base + lane;
    bool src = false, tgt = false;
    // the owned range is word-aligned, so a warp is either owned or not
    const bool own = x >= S.post_lo && x < S.post_hi;
    if (x < n) src = sw::u01(sw::draw(S.poisson_key, (uint64_t)(k * n + x))) < S.p_src[x];
    if (x < n && own) {
      const double gg = __dmul_rn(__dadd_rn(S.g_tot[x], S.pending[x]), S.decay_s);
      S.g_tot[x] = gg;
      const bool active = k > S.ref_until[x];
      const double r = __ddiv_rn(gg, S.g_leak);
      const double vinf = __ddiv_rn(__dadd_rn(S.v_rest, __dmul_rn(r, S.e_exc)), __dadd_rn(1.0, r));
      const double arg = __ddiv_rn(__dmul_rn(-S.h, __dadd_rn(1.0, r)), S.tau_m);
      double vv = active ? __dadd_rn(vinf, __dmul_rn(__dsub_rn(S.V[x], vinf), exp(arg))) : S.v_reset;
      tgt = active && vv >= S.v_theta;
      if (tgt) {
        vv = S.v_reset;
        S.ref_until[x] = k + S.ref_steps;
      }
      S.V[x] = vv;
    }
    const unsigned bs = __ballot_sync(SW_FULL_MASK, src);
    const unsigned bt = __ballot_sync(SW_FULL_MASK, tgt);
    if (lane == 0 && base < n) {
      S.src_bits[base >> 5] = bs;
      if (own) S.tgt_bits[base >> 5] = bt;
    }
  }
}

// Ordered sum over one transpose column (ascending pre): the column's
// source ids and their spike words are loaded kColU at a time (independent
// loads in flight), then the spiking entries are added in column order.
constexpr int kColU = 8;
__device__ __forceinline__ void col_sum(double& acc, int a, int e, const int32_t* src_pre,
                                        const int32_t* src_slot, const uint32_t* bits,
                                        const double* g, int stride) {
  for (int q0 = a; q0 < e; q0 += kColU) {
    int pre[kColU];
    uint32_t wd[kColU];
#pragma unroll
    for (int u = 0; u < kColU; ++u) pre[u] = (q0 + u < e) ? src_pre[q0 + u] : -1;
#pragma unroll
    for (int u = 0; u < kColU; ++u) wd[u] = pre[u] >= 0 ? bits[pre[u] >> 5] : 0u;
#pragma unroll
    for (int u = 0; u < kColU; ++u)
      if ((wd[u] >> (pre[u] & 31)) & 1u)
        acc = __dadd_rn(acc, g[(int64_t)pre[u] * stride + src_slot[q0 + u]]);
  }
}

// the first kColU entries of both columns (ff, then lat) loaded together —
// their pre ids, spike words and (spiking entries) weights — so the two
// columns' round trips overlap; the sums still run ff entries ascending,
// then lat entries ascending (the order col_sum gives)
struct ColBatch {
  double v[kColU];
  unsigned hit;
};
__device__ __forceinline__ void col_load(ColBatch& cb, int a, int e, const int32_t* src_pre, const int32_t* src_slot,
                                         const uint32_t* bits, const double* g, int stride) {
  int pre[kColU];
  uint32_t wd[kColU];
#pragma unroll
  for (int u = 0; u < kColU; ++u) pre[u] = (a + u < e) ? src_pre[a + u] : -1;
#pragma unroll
  for (int u = 0; u < kColU; ++u) wd[u] = pre[u] >= 0 ? bits[pre[u] >> 5] : 0u;
  cb.hit = 0u;
#pragma unroll
  for (int u = 0; u < kColU; ++u) {
    const bool h = (wd[u] >> (pre[u] & 31)) & 1u;
    cb.v[u] = h ? g[(int64_t)pre[u] * stride + src_slot[a + u]] : 0.0;
    cb.hit |= (h ? 1u : 0u) << u;
  }
}
__device__ __forceinline__ void col_add(double& acc, const ColBatch& cb) {
#pragma unroll
  for (int u = 0; u < kColU; ++u)
    if ((cb.hit >> u) & 1u) acc = __dadd_rn(acc, cb.v[u]);
}

__device__ __forceinline__ bool bit_of(const uint32_t* w, int i) { return (w[i >> 5] >> (i & 31)) & 1u; }

// psrc / ptgt (fused period, else null): the previous step's spike words,
// whose trace increments (x of spiking pres, y of spiking posts, += 1) were
// deferred to here, applied before the decay — the same two roundings as the
// increment in that step's STDP phases followed by this step's decay
__device__ __forceinline__ void tm_prop(const sw_topomap_step_t& S, int t0, int dt,
                                        const uint32_t* psrc = nullptr, const uint32_t* ptgt = nullptr) {
  for (int j = t0; j < S.n; j += dt) {
    // trace decays (x per pre, y per post; square model: n pres and n posts)
    double fx = S.ff_x[j], fy = S.ff_y[j], lx = S.lat_x[j], ly = S.lat_y[j];
    if (psrc && bit_of(psrc, j)) fx = __dadd_rn(fx, 1.0);
    if (ptgt && bit_of(ptgt, j)) {
      lx = __dadd_rn(lx, 1.0);
      fy = __dadd_rn(fy, 1.0);
      ly = __dadd_rn(ly, 1.0);
    }
    S.ff_x[j] = __dmul_rn(fx, S.decay_x);
    S.ff_y[j] = __dmul_rn(fy, S.decay_y);
    S.lat_x[j] = __dmul_rn(lx, S.decay_x);
    S.lat_y[j] = __dmul_rn(ly, S.decay_y);
    if (j < S.post_lo || j >= S.post_hi) continue;
    double acc = 0.0;
    const int fa = S.ff_col_ptr[j], fe = fa + S.ff_col_len[j];
    const int la = S.lat_col_ptr[j], le = la + S.lat_col_len[j];
    ColBatch fb, lb;
    col_load(fb, fa, fe, S.ff_src_pre, S.ff_src_slot, S.src_bits, S.ff_g, S.ff_stride);
    col_load(lb, la, le, S.lat_src_pre, S.lat_src_slot, S.tgt_bits, S.lat_g, S.lat_stride);
    col_add(acc, fb);
    col_sum(acc, fa + kColU, fe, S.ff_src_pre, S.ff_src_slot, S.src_bits, S.ff_g, S.ff_stride);
    col_add(acc, lb);
    col_sum(acc, la + kColU, le, S.lat_src_pre, S.lat_src_slot, S.tgt_bits, S.lat_g, S.lat_stride);
    S.pending[j] = acc;
  }
}

__device__ __forceinline__ void depress_row(const int32_t* rl, const int32_t* tg, double* w, int stride,
                                            int i, const double* y, double a_minus, double w_min,
                                            double w_max, int lane) {
  const int len = rl[i];
  const int64_t off = (int64_t)i * stride;
  for (int s = lane; s < len; s += 32) {
    double v = __dsub_rn(w[off + s], __dmul_rn(a_minus, y[tg[off + s]]));
    v = fmax(v, w_min);
    w[off + s] = fmin(v, w_max);
  }
}

// warp w0, w0 + dw, ... over the 2 * words spike words (ff sources, then lat targets)
__device__ __forceinline__ void tm_pre(const sw_topomap_step_t& S, int w0, int dw) {
  const int lane = threadIdx.x & 31;
  const int groups = (S.n + 31) / 32;
  for (int g = w0; g < 2 * groups; g += dw) {
    const bool ff = g < groups;
    const int grp = ff ? g : g - groups;
    unsigned m = ff ? S.src_bits[grp] : S.tgt_bits[grp];
    while (m) {
      const int i = grp * 32 + __ffs(m) - 1;
      m &= m - 1;
      if (ff) depress_row(S.ff_row_length, S.ff_target, S.ff_g, S.ff_stride, i, S.ff_y, S.a_minus, S.w_min, S.w_max, lane);
      else depress_row(S.lat_row_length, S.lat_target, S.lat_g, S.lat_stride, i, S.lat_y, S.a_minus, S.w_min, S.w_max, lane);
      if (lane == 0) {
        if (ff) S.ff_x[i] = __dadd_rn(S.ff_x[i], 1.0);
        else S.lat_x[i] = __dadd_rn(S.lat_x[i], 1.0);
      }
    }
  }
}

// potentiation through the transposes: warp w0, w0 + dw, ... over the
// target spike words; the lanes of a warp share each spiking post's column
// (distinct synapses, so no ordering between them), then y[post] += 1
__device__ __forceinline__ void potentiate_col(int a, int e, const int32_t* src_pre,
                                               const int32_t* src_slot, double* g, int stride,
                                               const double* x, double a_plus, double w_min,
                                               double w_max, int lane) {
  for (int q = a + lane; q < e; q += 32) {
    const int i = src_pre[q];
    const int64_t o = (int64_t)i * stride + src_slot[q];
    double v = __dadd_rn(g[o], __dmul_rn(a_plus, x[i]));
    v = fmax(v, w_min);
    g[o] = fmin(v, w_max);
  }
}

__device__ __forceinline__ void tm_post(const sw_topomap_step_t& S, int w0, int dw) {
  const int lane = threadIdx.x & 31;
  const int words = (S.n + 31) / 32;
  for (int gw = w0; gw < words; gw += dw) {
    unsigned m = S.tgt_bits[gw];
    while (m) {
      const int j = gw * 32 + __ffs(m) - 1;
      m &= m - 1;
      potentiate_col(S.ff_col_ptr[j], S.ff_col_ptr[j] + S.ff_col_len[j], S.ff_src_pre, S.ff_src_slot, S.ff_g,
                     S.ff_stride, S.ff_x, S.a_plus, S.w_min, S.w_max, lane);
      potentiate_col(S.lat_col_ptr[j], S.lat_col_ptr[j] + S.lat_col_len[j], S.lat_src_pre, S.lat_src_slot, S.lat_g,
                     S.lat_stride, S.lat_x, S.a_plus, S.w_min, S.w_max, lane);
      if (lane == 0) {
        S.ff_y[j] = __dadd_rn(S.ff_y[j], 1.0);
        S.lat_y[j] = __dadd_rn(S.lat_y[j], 1.0);
      }
    }
  }
}

// ---- STDP pre and post of one step in one launch (fused period) ----------
// The sequential order is: pre (depress rows of spiking pres with the posts'
// y, then x[pre] += 1), post (potentiate columns of spiking posts with the
// pres' x, then y[post] += 1).  In one launch: the trace increments are
// deferred to the next step's propagation phase (tm_prop psrc / ptgt), the
// pre phase uses y as it is (= before the increment) and, for a synapse
// whose post also spiked, applies the potentiation right after the
// depression with x + 1 of its (spiking) pre; the post phase skips synapses
// whose pre spiked and otherwise uses x as it is (the pre did not spike).
// Every synapse is written by one phase, in the sequential order.
__device__ __forceinline__ void depress_row_fused(const int32_t* rl, const int32_t* tg, double* w, int stride,
                                                  int i, const double* y, const double* x,
                                                  const uint32_t* post_bits, const sw_topomap_step_t& S, int lane) {
  const int len = rl[i];
  const int64_t off = (int64_t)i * stride;
  const double xa = __dadd_rn(x[i], 1.0);
  for (int s = lane; s < len; s += 32) {
    const int j = tg[off + s];
    double v = __dsub_rn(w[off + s], __dmul_rn(S.a_minus, y[j]));
    v = fmin(fmax(v, S.w_min), S.w_max);
    if (bit_of(post_bits, j)) {
      v = __dadd_rn(v, __dmul_rn(S.a_plus, xa));
      v = fmin(fmax(v, S.w_min), S.w_max);
    }
    w[off + s] = v;
  }
}

__device__ __forceinline__ void tm_pre_fused(const sw_topomap_step_t& S, int w0, int dw) {
  const int lane = threadIdx.x & 31;
  const int groups = (S.n + 31) / 32;
  for (int g = w0; g < 2 * groups; g += dw) {
    const bool ff = g < groups;
    const int grp = ff ? g : g - groups;
    unsigned m = ff ? S.src_bits[grp] : S.tgt_bits[grp];
    while (m) {
      const int i = grp * 32 + __ffs(m) - 1;
      m &= m - 1;
      if (ff) depress_row_fused(S.ff_row_length, S.ff_target, S.ff_g, S.ff_stride, i, S.ff_y, S.ff_x, S.tgt_bits, S, lane);
      else depress_row_fused(S.lat_row_length, S.lat_target, S.lat_g, S.lat_stride, i, S.lat_y, S.lat_x, S.tgt_bits, S, lane);
    }
  }
}

__device__ __forceinline__ void potentiate_col_fused(int a, int e, const int32_t* src_pre, const int32_t* src_slot,
                                                     double* g, int stride, const double* x,
                                                     const uint32_t* pre_bits, const sw_topomap_step_t& S,
                                                     int lane) {
  for (int q = a + lane; q < e; q += 32) {
    const int i = src_pre[q];
    if (bit_of(pre_bits, i)) continue;   // done by the pre phase
    const int64_t o = (int64_t)i * stride + src_slot[q];
    double v = __dadd_rn(g[o], __dmul_rn(S.a_plus, x[i]));
    v = fmax(v, S.w_min);
    g[o] = fmin(v, S.w_max);
  }
}

__device__ __forceinline__ void tm_post_fused(const sw_topomap_step_t& S, int w0, int dw) {
  const int lane = threadIdx.x & 31;
  const int words = (S.n + 31) / 32;
  for (int gw = w0; gw < words; gw += dw) {
    unsigned m = S.tgt_bits[gw];
    while (m) {
      const int j = gw * 32 + __ffs(m) - 1;
      m &= m - 1;
      potentiate_col_fused(S.ff_col_ptr[j], S.ff_col_ptr[j] + S.ff_col_len[j], S.ff_src_pre, S.ff_src_slot, S.ff_g,
                           S.ff_stride, S.ff_x, S.src_bits, S, lane);
      potentiate_col_fused(S.lat_col_ptr[j], S.lat_col_ptr[j] + S.lat_col_len[j], S.lat_src_pre, S.lat_src_slot,
                           S.lat_g, S.lat_stride, S.lat_x, S.tgt_bits, S, lane);
    }
  }
}

// per-step spike counts of words [w0, words) step dw, added to cnt[2]
__device__ __forceinline__ void tm_count(const sw_topomap_step_t& S, int w0, int dw, int64_t* cnt) {
  const int words = (S.n + 31) / 32;
  int a = 0, b = 0;
  for (int w = w0; w < words; w += dw) {
    a += __popc(S.src_bits[w]);
    b += __popc(S.tgt_bits[w]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(SW_FULL_MASK, a, o);
    b += __shfl_xor_sync(SW_FULL_MASK, b, o);
  }
  if ((threadIdx.x & 31) == 0 && (a | b)) {
    atomicAdd((unsigned long long*)&cnt[0], (unsigned long long)a);
    atomicAdd((unsigned long long*)&cnt[1], (unsigned long long)b);
  }
}

// ---- one phase per launch (the sharded path splits the step around an all-gather) --
// the per-step kernels start with sw::pdl_enter (common.cuh): launched with
// the PDL attribute, a phase's blocks are scheduled while the previous phase
// drains and wait for its completion before their first access
using sw::pdl_enter;

__global__ void k_tm_neurons(sw_topomap_step_t S) {
  pdl_enter();
  tm_neurons(S, *S.step, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

__global__ void k_tm_prop(sw_topomap_step_t S, int64_t* spike_counts) {
  pdl_enter();
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gn = gridDim.x * blockDim.x;
  tm_prop(S, gt, gn);
  if (spike_counts) tm_count(S, gt, gn, spike_counts);
}

__global__ void k_tm_pre(sw_topomap_step_t S) {
  pdl_enter();
  tm_pre(S, blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), gridDim.x * (blockDim.x >> 5));
}

__global__ void k_tm_post(sw_topomap_step_t S) {
  pdl_enter();
  tm_post(S, blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), gridDim.x * (blockDim.x >> 5));
  // the step counter is read only by the next step's neuron phase
  if (blockIdx.x == 0 && threadIdx.x == 0) *S.step += 1;
}

// ---- fused period (unsharded sheets): 2 launches per step ----------------
// (1) propagation of step t, with the previous step's deferred trace
//     increments and the step counter advanced for the next neuron phase;
// (2) STDP pre and post of step t (tm_pre_fused / tm_post_fused) together
//     with the neuron phase of step t+1 — disjoint data once the spike words
//     alternate between two buffer pairs.
__global__ void k_tm_prop_fused(sw_topomap_step_t S, const uint32_t* psrc, const uint32_t* ptgt,
                                int64_t* spike_counts) {
  pdl_enter();
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gn = gridDim.x * blockDim.x;
  tm_prop(S, gt, gn, psrc, ptgt);
  if (spike_counts) tm_count(S, gt, gn, spike_counts);
  if (blockIdx.x == 0 && threadIdx.x == 0) *S.step += 1;   // read by the next neuron phase only
}

__global__ void k_tm_stdp_neurons(sw_topomap_step_t S, sw_topomap_step_t Sn, int pre_blocks, int post_blocks,
                                  int with_neurons) {
  pdl_enter();
  const int wpb = blockDim.x >> 5, warp = threadIdx.x >> 5;
  if ((int)blockIdx.x < pre_blocks) {
    tm_pre_fused(S, blockIdx.x * wpb + warp, pre_blocks * wpb);
  } else if ((int)blockIdx.x < pre_blocks + post_blocks) {
    tm_post_fused(S, (blockIdx.x - pre_blocks) * wpb + warp, post_blocks * wpb);
  } else if (with_neurons) {
    const int b = blockIdx.x - pre_blocks - post_blocks;
    const int nb = gridDim.x - pre_blocks - post_blocks;
    tm_neurons(Sn, *Sn.step, b * blockDim.x + threadIdx.x, nb * blockDim.x);
  }
}

// the period's last deferred trace increments (no decay)
__global__ void k_tm_trace_flush(sw_topomap_step_t S) {
  pdl_enter();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < S.n; j += gridDim.x * blockDim.x) {
    if (bit_of(S.src_bits, j)) S.ff_x[j] = __dadd_rn(S.ff_x[j], 1.0);
    if (bit_of(S.tgt_bits, j)) {
      S.lat_x[j] = __dadd_rn(S.lat_x[j], 1.0);
      S.ff_y[j] = __dadd_rn(S.ff_y[j], 1.0);
      S.lat_y[j] = __dadd_rn(S.lat_y[j], 1.0);
    }
  }
}


// ---- persistent multi-step kernel ------------------------------------------------------
// n_steps whole steps in one launch: the phases of a step are separated by
// grid-wide barriers (cooperative launch: every CTA resident) — or by
// __syncthreads when one CTA covers the sheet — instead of kernel
// boundaries, so a step costs a few barrier latencies instead of five
// launches.  Same phase bodies, same order, same results as sw_topomap_step.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
#if SW_TM_CG_SYNC
  (void)bar;
  cg::this_grid().sync();
  return;
#endif
  __syncthreads();
  if (gridDim.x > 1) {
    if (threadIdx.x == 0) {
      volatile unsigned* vb = bar;
      const unsigned gen = vb[1];
      __threadfence();
      if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
        bar[0] = 0u;
        __threadfence();
        atomicAdd(&bar[1], 1u);
      } else {
        while (vb[1] == gen) __nanosleep(32);
      }
      __threadfence();
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024)
k_tm_run(sw_topomap_step_t S, int n_steps, int64_t* spike_counts, unsigned* bar) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int gn = gridDim.x * blockDim.x;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x >> 5);
  const int64_t k0 = *S.step;
  grid_barrier(bar);   // everyone has read the step counter
  for (int st = 0; st < n_steps; ++st) {
    const int64_t k = k0 + st;
    tm_neurons(S, k, gw * 32, nw * 32);
    grid_barrier(bar);
    tm_prop(S, gt, gn);
    if (spike_counts) tm_count(S, gt, gn, spike_counts);
    grid_barrier(bar);
    tm_pre(S, gw, nw);
    grid_barrier(bar);
    tm_post(S, gw, nw);
    grid_barrier(bar);
  }
  if (gt == 0) *S.step = k0 + n_steps;
}

// Single-CTA variant for small sheets: the per-node state (LIF, pending
// input, STDP traces, source probabilities), the row lengths, the transpose
// column pointers and the spike words live in shared memory for the whole
// period — the phases' dependent memory round trips become shared-memory
// hits — and are written back at the end.  Synapse arrays (targets,
// transposes, weights) stay in global memory (L1/L2).
struct TmSmem {
  static size_t bytes(int n) {
    const int words = (n + 31) / 32;
    return (size_t)n * 8 * 9 + (size_t)(n + 1) * 4 * 2 + (size_t)n * 4 * 4 + (size_t)words * 4 * 4 + 64;
  }
};

__global__ void __launch_bounds__(512, 1)
k_tm_run_staged(sw_topomap_step_t G, int n_steps, int64_t* spike_counts) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int n = G.n, words = (n + 31) / 32;
  double* d = reinterpret_cast<double*>(sm);
  double *V = d, *gt = d + n, *pend = d + 2 * n, *fx = d + 3 * n, *fy = d + 4 * n, *lx = d + 5 * n,
         *ly = d + 6 * n, *ps = d + 7 * n;
  int64_t* ref = reinterpret_cast<int64_t*>(d + 8 * n);
  int32_t* ip = reinterpret_cast<int32_t*>(d + 9 * n);
  int32_t *fcp = ip, *lcp = ip + (n + 1), *frl = ip + 2 * (n + 1), *lrl = frl + n;
  int32_t *fcl = lrl + n, *lcl = fcl + n;
  // two spike-word buffer pairs: step t's words stay readable while step
  // t+1's neuron phase writes the other pair
  uint32_t *sb = reinterpret_cast<uint32_t*>(lcl + n), *tb = sb + words, *sb1 = tb + words, *tb1 = sb1 + words;
  for (int x = threadIdx.x; x < n; x += blockDim.x) {
    V[x] = G.V[x]; gt[x] = G.g_tot[x]; pend[x] = G.pending[x];
    fx[x] = G.ff_x[x]; fy[x] = G.ff_y[x]; lx[x] = G.lat_x[x]; ly[x] = G.lat_y[x];
    ps[x] = G.p_src[x]; ref[x] = G.ref_until[x];
    frl[x] = G.ff_row_length[x]; lrl[x] = G.lat_row_length[x];
    fcl[x] = G.ff_col_len[x]; lcl[x] = G.lat_col_len[x];
  }
  for (int x = threadIdx.x; x <= n; x += blockDim.x) {
    fcp[x] = G.ff_col_ptr[x];
    lcp[x] = G.lat_col_ptr[x];
  }
  const int64_t k0 = *G.step;
  sw_topomap_step_t S = G;
  S.V = V; S.g_tot = gt; S.pending = pend; S.ff_x = fx; S.ff_y = fy; S.lat_x = lx; S.lat_y = ly;
  S.p_src = ps; S.ref_until = ref; S.ff_row_length = frl; S.lat_row_length = lrl;
  S.ff_col_ptr = fcp; S.lat_col_ptr = lcp; S.ff_col_len = fcl; S.lat_col_len = lcl;
  S.src_bits = sb; S.tgt_bits = tb;
  sw_topomap_step_t S1 = S;
  S1.src_bits = sb1; S1.tgt_bits = tb1;
  __syncthreads();
  const int t = threadIdx.x, nt = blockDim.x;
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // two phases per step (the fused-period order of sw_topomap_steps_fused):
  // propagation with the previous step's deferred trace increments, then
  // STDP pre + post of this step and the neuron phase of the next
  tm_neurons(S, k0, w * 32, nw * 32);
  __syncthreads();
  for (int st = 0; st < n_steps; ++st) {
    const sw_topomap_step_t& Sc = (st & 1) ? S1 : S;
    const sw_topomap_step_t& Sp = (st & 1) ? S : S1;
    tm_prop(Sc, t, nt, st > 0 ? Sp.src_bits : nullptr, st > 0 ? Sp.tgt_bits : nullptr);
    if (spike_counts) tm_count(Sc, t, nt, spike_counts);
    __syncthreads();
    tm_pre_fused(Sc, w, nw);
    tm_post_fused(Sc, w, nw);
    if (st + 1 < n_steps) tm_neurons(Sp, k0 + st + 1, w * 32, nw * 32);
    __syncthreads();
  }
  {
    // the last step's deferred trace increments, its words in the first pair
    const sw_topomap_step_t& Sl = ((n_steps - 1) & 1) ? S1 : S;
    for (int j = t; j < n; j += nt) {
      if (bit_of(Sl.src_bits, j)) fx[j] = __dadd_rn(fx[j], 1.0);
      if (bit_of(Sl.tgt_bits, j)) {
        lx[j] = __dadd_rn(lx[j], 1.0);
        fy[j] = __dadd_rn(fy[j], 1.0);
        ly[j] = __dadd_rn(ly[j], 1.0);
      }
    }
    if ((n_steps - 1) & 1)
      for (int x = t; x < words; x += nt) {
        sb[x] = sb1[x];
        tb[x] = tb1[x];
      }
    __syncthreads();
  }
  for (int x = threadIdx.x; x < n; x += blockDim.x) {
    G.V[x] = V[x]; G.g_tot[x] = gt[x]; G.pending[x] = pend[x];
    G.ff_x[x] = fx[x]; G.ff_y[x] = fy[x]; G.lat_x[x] = lx[x]; G.lat_y[x] = ly[x];
    G.ref_until[x] = ref[x];
  }
  for (int x = threadIdx.x; x < words; x += blockDim.x) {
    G.src_bits[x] = sb[x];
    G.tgt_bits[x] = tb[x];
  }
  if (threadIdx.x == 0) *G.step = k0 + n_steps;
}

int grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

// launch with the programmatic-stream-serialization attribute (PDL; kernels
// start with pdl_enter) for sheets of up to 16 384 nodes (s <= 8: 2.5-4 %
// faster per step; at 65 536 nodes the early-resident dependent blocks cost
// more than the launch latency they hide, -4.5 %); SW_TM_PDL=0 launches
// plainly (measurement)
template <typename... KArgs, typename... Args>
void launch_pdl(int n, void (*kern)(KArgs...), int grid, int block, cudaStream_t st, Args... args) {
  static const int mode = [] { const char* e = getenv("SW_TM_PDL"); return e ? atoi(e) : 1; }();   // 0 off, 2 all sizes
  sw::pdl_launch(mode == 2 || (mode == 1 && n <= 16384), kern, dim3(grid), dim3(block), 0, st, args...);
}

}  // namespace

static int check_step(const sw_topomap_step_t* s) {
  if (s->post_lo < 0 || s->post_hi > s->n || s->post_lo > s->post_hi || (s->post_lo & 31) ||
      ((s->post_hi & 31) && s->post_hi != s->n)) {
    sw::set_last_error("topomap step: post shard must be [lo, hi) on 32-post word boundaries");
    return SW_ERR_INVALID_ARG;
  }
  return SW_OK;
}

extern "C" int sw_topomap_neurons(const sw_topomap_step_t* s, void* stream) {
  if (int e = check_step(s)) return e;
  const int n = s->n;
  if (n <= 0) return SW_OK;
  launch_pdl(n, k_tm_neurons, grid1(n), 256, (cudaStream_t)stream, *s); sw::count_launch();
  SW_CHECK_LAUNCH("sw_topomap_neurons");
  return SW_OK;
}

extern "C" int sw_topomap_synapses(const sw_topomap_step_t* s, int64_t* spike_counts, void* stream) {
  if (int e = check_step(s)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const int n = s->n;
  if (n <= 0) return SW_OK;
  launch_pdl(n, k_tm_prop, grid1(n), 256, st, *s, spike_counts); sw::count_launch();
  int groups = (n + 31) / 32;
  int blocks = (2 * groups + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_pdl(n, k_tm_pre, blocks, 256, st, *s); sw::count_launch();
  int pblocks = (groups + 7) / 8;
  if (pblocks > 148 * 8) pblocks = 148 * 8;
  launch_pdl(n, k_tm_post, pblocks, 256, st, *s); sw::count_launch();
  SW_CHECK_LAUNCH("sw_topomap_synapses");
  return SW_OK;
}

extern "C" int sw_topomap_run_steps(const sw_topomap_step_t* s, int32_t n_steps, int64_t* spike_counts,
                                    uint32_t* barrier_words, void* stream) {
  if (int e = check_step(s)) return e;
  if (s->post_lo != 0 || s->post_hi != s->n) {
    sw::set_last_error("sw_topomap_run_steps: unsharded sheets only (use neurons/synapses)");
    return SW_ERR_INVALID_ARG;
  }
  if (!barrier_words) { sw::set_last_error("sw_topomap_run_steps: barrier words required"); return SW_ERR_INVALID_ARG; }
  const int n = s->n;
  if (n <= 0 || n_steps <= 0) return SW_OK;
  static int max_ctas = 0;
  if (max_ctas == 0) {
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tm_run, 512, 0);
    max_ctas = per_sm * sms;
    if (max_ctas < 1) max_ctas = 1;
  }
  // small sheets: one CTA with the per-node state staged in shared memory
  const size_t sbytes = TmSmem::bytes(n);
  if (n <= 2048 && sbytes <= 200 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute((const void*)k_tm_run_staged, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      attr = true;
    }
    k_tm_run_staged<<<1, 512, sbytes, (cudaStream_t)stream>>>(*s, n_steps, spike_counts);
    sw::count_launch();
    SW_CHECK_LAUNCH("sw_topomap_run_steps");
    return SW_OK;
  }
  // one CTA per SW_TM_NODES_PER_CTA nodes, 512 threads, grid barriers
  int ctas = (n + SW_TM_NODES_PER_CTA - 1) / SW_TM_NODES_PER_CTA;
  if (ctas > max_ctas) ctas = max_ctas;
  sw_topomap_step_t S = *s;
  int ns = n_steps;
  void* args[] = {(void*)&S, (void*)&ns, (void*)&spike_counts, (void*)&barrier_words};
  cudaLaunchCooperativeKernel((const void*)k_tm_run, dim3(ctas), dim3(512), args, 0, (cudaStream_t)stream);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_topomap_run_steps");
  return SW_OK;
}

extern "C" int sw_topomap_steps_fused(const sw_topomap_step_t* s, uint32_t* src_bits_alt, uint32_t* tgt_bits_alt,
                                      int32_t n_steps, int64_t* spike_counts, void* stream) {
  if (int e = check_step(s)) return e;
  if (s->post_lo != 0 || s->post_hi != s->n || !src_bits_alt || !tgt_bits_alt) {
    sw::set_last_error("sw_topomap_steps_fused: unsharded sheets and second spike-word buffers");
    return SW_ERR_INVALID_ARG;
  }
  const int n = s->n;
  if (n <= 0 || n_steps <= 0) return SW_OK;
  cudaStream_t st = (cudaStream_t)stream;
  sw_topomap_step_t S[2] = {*s, *s};
  S[1].src_bits = src_bits_alt;
  S[1].tgt_bits = tgt_bits_alt;
  const int groups = (n + 31) / 32;
  int pre_blocks = (2 * groups + 7) / 8;
  if (pre_blocks > 148 * 8) pre_blocks = 148 * 8;
  int post_blocks = (groups + 7) / 8;
  if (post_blocks > 148 * 8) post_blocks = 148 * 8;
  const int nblocks = grid1(n);
  launch_pdl(n, k_tm_neurons, nblocks, 256, st, S[0]); sw::count_launch();
  for (int t = 0; t < n_steps; ++t) {
    const sw_topomap_step_t& Sc = S[t & 1];
    const uint32_t* psrc = t > 0 ? S[(t - 1) & 1].src_bits : nullptr;
    const uint32_t* ptgt = t > 0 ? S[(t - 1) & 1].tgt_bits : nullptr;
    launch_pdl(n, k_tm_prop_fused, nblocks, 256, st, Sc, psrc, ptgt, spike_counts); sw::count_launch();
    const int with_neurons = t + 1 < n_steps ? 1 : 0;
    launch_pdl(n, k_tm_stdp_neurons, pre_blocks + post_blocks + (with_neurons ? nblocks : 0), 256, st, Sc,
               S[(t + 1) & 1], pre_blocks, post_blocks, with_neurons);
    sw::count_launch();
  }
  const sw_topomap_step_t& Sl = S[(n_steps - 1) & 1];
  launch_pdl(n, k_tm_trace_flush, nblocks, 256, st, Sl); sw::count_launch();
  // the last step's spike words back into the model's buffers
  if ((n_steps - 1) & 1) {
    cudaMemcpyAsync(s->src_bits, src_bits_alt, (size_t)groups * 4, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(s->tgt_bits, tgt_bits_alt, (size_t)groups * 4, cudaMemcpyDeviceToDevice, st);
  }
  SW_CHECK_LAUNCH("sw_topomap_steps_fused");
  return SW_OK;
}

extern "C" int sw_topomap_step(const sw_topomap_step_t* s, int64_t* spike_counts, void* stream) {
  if (int e = sw_topomap_neurons(s, stream)) return e;
  return sw_topomap_synapses(s, spike_counts, stream);
}
