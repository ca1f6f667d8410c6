// The e-prop ALIF classifier forward pass, fused per replica
// (sparsewire/classifier.py:188-234).  Block per replica; one launch runs one
// timestep or a group of n_steps timesteps back to back.  Per step:
//   1. input spikes of the synthetic task from the example's counter stream
//      (classifier.py:63-67: u = uniform01 #(t*NI + k) < p_e[k]); xbar update;
//   2. ascending spike lists (input, hidden) in shared memory; zbar update;
//   3. event-driven ragged propagation: the spiking rows' (post, w) entries
//      are staged in shared memory, bucketed by post (counting sort) and each
//      post's bucket is summed in ascending row order -- per post the
//      ascending-pre float32 sequential sum (classifier.py:208-209 computes
//      the same sums as a dense sgemm on a float32 weight copy); above the
//      staging capacities a warp-serial ordered walk gives the same sums;
//   4. surrogate psi from the pre-step state (neurons.py:69-73);
//   5. leaky readout y, softmax, cross-entropy, d = pi - onehot, pi_sum,
//      learning signal lsig = f32(d @ W_out) (classifier.py:215-223);
//   6. ALIF step with the new currents (neurons.py:60-67).
#include "common.cuh"

#include <cstdlib>
#include <type_traits>

namespace {

// k_clf_step is instantiated for 256 and 512 threads per replica block
// (512 pays off for the 1024-hidden layer, 256 for the 256-hidden one)
constexpr int kThreads = 256;             // auxiliary kernels

constexpr int kStageCap = 2048;   // staged (target, w) entries of the spiking rows
constexpr int kPerThread = 8;     // max rows per thread: (NI + H) <= kThreads * kPerThread

__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Block-wide exclusive scan of two ints (count, length-sum); returns the
// exclusive prefixes for this thread and the totals.
template <int kWarps>
__device__ __forceinline__ void block_scan2(int a, int b, int& ea, int& eb, int& ta, int& tb,
                                            int2* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int xa = __shfl_up_sync(SW_FULL_MASK, ia, o);
    const int xb = __shfl_up_sync(SW_FULL_MASK, ib, o);
    if (lane >= o) { ia += xa; ib += xb; }
  }
  if (lane == 31) wsum[warp] = make_int2(ia, ib);
  __syncthreads();
  int pa = 0, pb = 0;
  ta = 0;
  tb = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const int2 v = wsum[w];
    if (w < warp) { pa += v.x; pb += v.y; }
    ta += v.x;
    tb += v.y;
  }
  ea = pa + ia - a;
  eb = pb + ib - b;
}

// Phase timestamps of one block (clock64), compiled in with -DSW_CLF_PROF;
// read back with sw_debug_clf_prof (tools/timing_breakdown.py).
__device__ long long g_clf_prof[16];
#ifdef SW_CLF_PROF
#define PROF(i) do { if (blockIdx.x == 7 && threadIdx.x == 0) g_clf_prof[i] = clock64(); } while (0)
#else
#define PROF(i) do { } while (0)
#endif

// kCompact: 16-bit row lengths, bucket offsets and sorted-row indices (the
// layout of large layers, to keep 4 blocks per SM); else 32-bit
// kPT: rows of [inputs | hidden] per thread in the spike phase (the host
// picks 4 when NI + H <= 4 * kThreads: smaller per-thread arrays)
template <int kThreads, bool kCompact, int kPT>
__device__ __forceinline__ void clf_step_body(const sw_clf_step_t& P, int scap_arg, int rcap_arg,
                                              bool load_rlen = true) {
  using idx_t = typename std::conditional<kCompact, uint16_t, int>::type;
  // the 32-bit layout uses the compile-time capacities (kStageCap, all rows)
  const int scap = kCompact ? scap_arg : kStageCap;
  const int rcap = kCompact ? rcap_arg : P.num_inputs + P.hidden;
  constexpr int kWarps = kThreads / 32;
  extern __shared__ unsigned char smem_raw[];
  const int H = P.hidden, NI = P.num_inputs, C = P.num_classes;
  const int NT = NI + H;
  // shared-memory layout (clf_smem_bytes on the host mirrors it); scap
  // staged entries and rcap spiking rows are the capacities of the staged
  // propagation path (beyond them: the warp-serial fallback)
  // byte offsets into smem_raw (not integer-cast pointers, which would turn
  // the shared-memory accesses into generic ones)
  size_t o = 0;
  float* acc_ext = (float*)(smem_raw + o); o += (size_t)H * 4;
  float* acc_rec = (float*)(smem_raw + o); o += (size_t)H * 4;
  idx_t* rlen = (idx_t*)(smem_raw + o);   o += (size_t)NT * sizeof(idx_t);    // [NT] row lengths
  o = (o + 3) & ~(size_t)3;
  int* list = (int*)(smem_raw + o);       o += (size_t)NT * 4;                // [NT] spiking rows, ascending
  int* roff = (int*)(smem_raw + o);       o += (size_t)(rcap + 1) * 4;        // [rcap + 1]
  int* st_kr = (int*)(smem_raw + o);      o += (size_t)scap * 4;              // [scap] key | row << 16
  float* st_w = (float*)(smem_raw + o);   o += (size_t)scap * 4;              // [scap]
  idx_t* srow = (idx_t*)(smem_raw + o);   o += (size_t)scap * sizeof(idx_t);  // [scap] sorted by key
  o = (o + 3) & ~(size_t)3;
  float* sw_ = (float*)(smem_raw + o);    o += (size_t)scap * 4;              // [scap]
  idx_t* koff = (idx_t*)(smem_raw + o);   o += (size_t)(2 * H + 1) * sizeof(idx_t);   // [2H + 1] key offsets
  o = (o + 3) & ~(size_t)3;
  int* kcur = (int*)(smem_raw + o);       o += (size_t)2 * H * 4;             // [2H] counts, then cursors
  o = (o + 15) & ~(size_t)15;
  double* yv = (double*)(smem_raw + o);
  double* ypre = yv + 2 * C;                // [C] previous y, pi_sum, b_out (prefetched)
  double* pipre = ypre + C;
  double* bpre = pipre + C;
  double* dv = yv + C;
  __shared__ double s_loss;
  __shared__ int s_label;
  __shared__ int2 wsum[kWarps];
  __shared__ int s_nx, s_nrows, s_total;
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t bH = (int64_t)b * H, bI = (int64_t)b * NI, bC = (int64_t)b * C;

  PROF(0);
  // ALIF state of this thread's first hidden unit, needed only in P6: loaded
  // now so that its latency overlaps the phases before
  const bool h0_ok = threadIdx.x < H;
  const float v0 = h0_ok ? P.v[bH + threadIdx.x] : 0.f;
  const float a0 = h0_ok ? P.a[bH + threadIdx.x] : 0.f;
  const float z0 = h0_ok ? P.z[bH + threadIdx.x] : 0.f;
  // per-replica readout state read only in the readout/softmax phases:
  // asynchronous global->shared copies, waited for at the barrier after P1
  // (32-bit layout only: the compact layout's shared memory is at its budget)
  if constexpr (!kCompact) {
    if ((int)threadIdx.x < C) {
      cp_async8(ypre + threadIdx.x, P.y + bC + threadIdx.x);
      cp_async8(pipre + threadIdx.x, P.pi_sum + bC + threadIdx.x);
      cp_async8(bpre + threadIdx.x, P.b_out + threadIdx.x);
    } else if (threadIdx.x == kThreads - 1) {
      cp_async8(&s_loss, P.loss + b);
      cp_async4(&s_label, P.labels + b);
    }
  }
  // P0: row lengths to shared memory; zero the current accumulators
  // (the row lengths stay in shared memory across the steps of a launch:
  // the connectivity only changes between batches)
  if (load_rlen)
    for (int x = threadIdx.x; x < NT; x += kThreads)
      rlen[x] = (idx_t)((x < NI) ? __ldg(P.in_row_length + x) : __ldg(P.rec_row_length + (x - NI)));
  for (int h = threadIdx.x; h < H; h += kThreads) {
    acc_ext[h] = 0.0f;
    acc_rec[h] = 0.0f;
  }
  // per-key counters of the staged propagation (read after several barriers)
  for (int k = threadIdx.x; k < 2 * H; k += kThreads) kcur[k] = 0;
  // P1: this thread's contiguous chunk of [inputs | hidden]: spike flags,
  // xbar/zbar updates (classifier.py:63-67, 207-213)
  const int per = (NT + kThreads - 1) / kThreads;
  const int x0 = threadIdx.x * per;
  const uint64_t key = P.ex_key[b];
  const uint64_t c0 = (uint64_t)P.t * (uint64_t)NI;
  unsigned flags = 0;
  float tr[kPT], zv[kPT];
  double pv[kPT];
#pragma unroll
  for (int j = 0; j < kPT; ++j) {   // all loads first
    const int x = x0 + j;
    tr[j] = 0.f;
    zv[j] = 0.f;
    pv[j] = 0.0;
    if (j < per && x < NT) {
      if (x < NI) {
        pv[j] = P.p_in[bI + x];
        tr[j] = (P.xbar_in ? P.xbar_in : P.xbar)[bI + x];
      } else {
        zv[j] = P.z[bH + x - NI];
        tr[j] = (P.zbar_in ? P.zbar_in : P.zbar)[bH + x - NI];
      }
    }
  }
  PROF(12);
#pragma unroll
  for (int j = 0; j < kPT; ++j) {
    const int x = x0 + j;
    if (j < per && x < NT) {
      bool f;
      if (x < NI) {
        f = sw::u01(sw::draw(key, c0 + (uint64_t)x)) < pv[j];
        P.xbar[bI + x] = __fadd_rn(__fmul_rn(tr[j], P.alpha), f ? 1.0f : 0.0f);
      } else {
        f = zv[j] != 0.0f;
        P.zbar[bH + x - NI] = __fadd_rn(__fmul_rn(tr[j], P.alpha), zv[j]);
      }
      if (f) flags |= 1u << j;
    }
  }
  PROF(1);
  if constexpr (!kCompact) cp_async_wait_all();
  __syncthreads();   // rlen ready (and the prefetched readout state)
  PROF(2);
  // P2: one block scan -> ascending spike list + staged row offsets
  int cnt = 0, lsum = 0;
  // spiking rows (low 16 bits) and spiking inputs (high 16 bits) in one scan
  for (int j = 0; j < per; ++j)
    if ((flags >> j) & 1u) { cnt += 1 + ((x0 + j < NI) ? 0x10000 : 0); lsum += rlen[x0 + j]; }
  int ecp, el, tcp, tl;
  block_scan2<kWarps>(cnt, lsum, ecp, el, tcp, tl, wsum);
  int ec = ecp & 0xFFFF;
  const int tc = tcp & 0xFFFF;
  for (int j = 0; j < per; ++j) {
    if ((flags >> j) & 1u) {
      list[ec] = x0 + j;
      if constexpr (kCompact) {
        if (ec < rcap) roff[ec] = el;
      } else {
        roff[ec] = el;
      }
      el += rlen[x0 + j];
      ++ec;
    }
  }
  if (threadIdx.x == 0) {
    if (!kCompact || tc <= rcap) roff[tc] = tl;
    s_nrows = tc;
    s_total = tl;
    s_nx = tcp >> 16;
  }
  __syncthreads();
  PROF(3);
  const int nrows = s_nrows, nx = s_nx, nz = nrows - nx;
  
  const int* zl = list + nx;   // hidden entries are NI + h
  const bool staged = kCompact ? (s_total <= scap && nrows <= rcap) : (s_total <= kStageCap);
  // P3: stage every spiking row's (target, w) with coalesced loads; the
  // readout warps also issue their W_out gathers here
  // P3: stage every spiking row's (key = [in|rec] post, row, w) with
  // independent loads (flattened, owning row by binary search) and count
  // entries per key.  P4 turns this into a counting sort by key that is
  // stable in row order, and each thread sums its posts' entries in
  // ascending row (= ascending pre) order: the same float32 sequential sum
  // per post as the reference, without a serial walk over the rows.
  const int T = s_total;
  if (staged) {
    for (int q0 = threadIdx.x; q0 < T; q0 += 4 * kThreads) {
      int tv[4], rv[4];
      float wv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * kThreads;
        tv[u] = 0;
        rv[u] = 0;
        wv[u] = 0.f;
        if (q < T) {
          int lo = 0, hi = nrows - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (roff[mid] <= q) lo = mid; else hi = mid - 1;
          }
          const int x = list[lo];
          const bool in = x < NI;
          const int64_t o = (int64_t)(in ? x : x - NI) * (in ? P.in_stride : P.rec_stride) + (q - roff[lo]);
          tv[u] = __ldg((in ? P.in_target : P.rec_target) + o) + (in ? 0 : H);
          wv[u] = __ldg((in ? P.in_w32 : P.rec_w32) + o);
          rv[u] = lo;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * kThreads;
        if (q < T) {
          st_kr[q] = tv[u] | (rv[u] << 16);
          st_w[q] = wv[u];
          atomicAdd(&kcur[tv[u]], 1);
        }
      }
    }
  }
  PROF(4);
  __syncthreads();
  PROF(5);
  if (staged) {
    // exclusive scan of the 2H key counts (contiguous chunk per thread)
    const int NK = 2 * H;
    const int kper = (NK + kThreads - 1) / kThreads;
    const int k0 = threadIdx.x * kper;
    int loc = 0;
    for (int j = 0; j < kper; ++j) if (k0 + j < NK) loc += kcur[k0 + j];
    int ex, dummy_e, tot, dummy_t;
    block_scan2<kWarps>(loc, 0, ex, dummy_e, tot, dummy_t, wsum);
    for (int j = 0; j < kper; ++j) {
      if (k0 + j < NK) {
        const int c = kcur[k0 + j];
        koff[k0 + j] = (idx_t)ex;
        kcur[k0 + j] = ex;
        ex += c;
      }
    }
    if (threadIdx.x == 0) koff[NK] = (idx_t)tot;
    PROF(10);
    __syncthreads();
    for (int q = threadIdx.x; q < T; q += kThreads) {
      const int kr = st_kr[q];
      const int dst = atomicAdd(&kcur[kr & 0xFFFF], 1);
      srow[dst] = (idx_t)(kr >> 16);
      sw_[dst] = st_w[q];
    }
    PROF(11);
    __syncthreads();
    for (int k = threadIdx.x; k < NK; k += kThreads) {
      const int a = koff[k], e = koff[k + 1];
      // insertion sort of the (few) entries by row, then the ordered sum
      for (int i = a + 1; i < e; ++i) {
        const int r = srow[i];
        const float w = sw_[i];
        int j = i - 1;
        while (j >= a && srow[j] > r) { srow[j + 1] = srow[j]; sw_[j + 1] = sw_[j]; --j; }
        srow[j + 1] = r;
        sw_[j + 1] = w;
      }
      float acc = 0.0f;
      for (int i = a; i < e; ++i) acc = __fadd_rn(acc, sw_[i]);
      if (k < H) acc_ext[k] = acc; else acc_rec[k - H] = acc;
    }
    PROF(15);
  } else {
    // fallback (very many spiking synapses): warp-serial ordered walk
    if (warp == 0) {
      for (int r = 0; r < nx; ++r) {
        const int64_t o = (int64_t)list[r] * P.in_stride;
        for (int c = lane; c < rlen[list[r]]; c += 32) {
          const int t = __ldg(P.in_target + o + c);
          acc_ext[t] = __fadd_rn(acc_ext[t], __ldg(P.in_w32 + o + c));
        }
        __syncwarp();
      }
    } else if (warp == 1) {
      for (int r = nx; r < nrows; ++r) {
        const int64_t o = (int64_t)(list[r] - NI) * P.rec_stride;
        for (int c = lane; c < rlen[list[r]]; c += 32) {
          const int t = __ldg(P.rec_target + o + c);
          acc_rec[t] = __fadd_rn(acc_rec[t], __ldg(P.rec_w32 + o + c));
        }
        __syncwarp();
      }
    }
  }
  // readout y = alpha*y + z @ W_out^T + b (classifier.py:215): up to 4
  // classes per warp, their gathers issued together
  for (int c0 = warp; c0 < C; c0 += 4 * kWarps) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = lane; q < nz; q += 32) {
      const int h = zl[q] - NI;
      double w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * kWarps;
        w[u] = c < C ? __ldg(P.w_out + (int64_t)c * H + h) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += w[u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u * kWarps;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s[u] += __shfl_xor_sync(SW_FULL_MASK, s[u], o);
      if (lane == 0 && c < C)
        yv[c] = kCompact ? __dadd_rn(__dadd_rn(__dmul_rn(P.alpha64, P.y[bC + c]), s[u]), P.b_out[c])
                         : __dadd_rn(__dadd_rn(__dmul_rn(P.alpha64, ypre[c]), s[u]), bpre[c]);
    }
  }
  PROF(6);
  __syncthreads();
  PROF(7);
  // P5: softmax / cross-entropy / d (plasticity.py:156-165, classifier.py:216-219)
  if (warp == 0) {
    double mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmax(mx, yv[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(SW_FULL_MASK, mx, o));
    double se = 0.0;
    double ex[2] = {0.0, 0.0};
    for (int c = lane, u = 0; c < C; c += 32, ++u) {
      const double e = exp(yv[c] - mx);
      if (u < 2) ex[u] = e;
      se += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(SW_FULL_MASK, se, o);
    const int label = kCompact ? P.labels[b] : s_label;
    for (int c = lane, u = 0; c < C; c += 32, ++u) {
      const double pi = (u < 2 ? ex[u] : exp(yv[c] - mx)) / se;
      P.y[bC + c] = yv[c];
      P.pi_sum[bC + c] = (kCompact ? P.pi_sum[bC + c] : pipre[c]) + pi;
      const double dd = pi - (c == label ? 1.0 : 0.0);
      dv[c] = dd;
      P.d[bC + c] = dd;
      if (c == label) P.loss[b] = (kCompact ? P.loss[b] : s_loss) + -log(pi);
    }
  }
  PROF(8);
  __syncthreads();
  PROF(9);
  // P6: surrogate (pre-step state), learning signal, ALIF step
  for (int h = threadIdx.x; h < H; h += kThreads) {
    const bool first = h == (int)threadIdx.x;
    const float vo = first ? v0 : P.v[bH + h];
    const float ao = first ? a0 : P.a[bH + h];
    const float zo = first ? z0 : P.z[bH + h];
    const float thr_o = __fadd_rn(P.v_thr, __fmul_rn(P.beta, ao));
    const float cc = __fdiv_rn(__fsub_rn(vo, thr_o), P.v_thr);
    const float r = __fsub_rn(1.0f, fabsf(cc));
    P.psi[bH + h] = __fmul_rn(0.5f, (r > 0.0f || r != r) ? r : 0.0f);
    // lsig = f32(d @ W_out) (classifier.py:223), classes ascending; the
    // W_out column is loaded 8 classes at a time ahead of the chained sum
    double ls = 0.0;
    for (int c0 = 0; P.lsig && c0 < C; c0 += 8) {
      double wv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) wv[u] = (c0 + u < C) ? __ldg(P.w_out + (int64_t)(c0 + u) * H + h) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c0 + u < C) ls = __fma_rn(dv[c0 + u], wv[u], ls);
    }
    if (P.lsig) P.lsig[bH + h] = __double2float_rn(ls);
    float vv = __fmul_rn(P.alpha, __fsub_rn(vo, __fmul_rn(zo, P.v_thr)));
    vv = __fadd_rn(__fadd_rn(vv, acc_rec[h]), acc_ext[h]);
    const float aa = __fadd_rn(__fmul_rn(P.rho, ao), zo);
    P.v[bH + h] = vv;
    P.a[bH + h] = aa;
    P.z[bH + h] = (vv >= __fadd_rn(P.v_thr, __fmul_rn(P.beta, aa))) ? 1.0f : 0.0f;
  }
  PROF(13);
}

// One launch for n_steps consecutive timesteps (P.n_steps >= 1): the replicas
// are independent within a trial (the weights only change between batches),
// so each block runs its replica's steps back to back, with no inter-kernel
// gap or tail between them.  zbar/xbar/psi/lsig/d are then the bases of
// slot_count contiguous per-step slots ([slot][B][width]); step t writes slot
// t % slot_count and reads the traces of slot (t - 1) % slot_count.
template <int kThreads, bool kCompact, int kPT>
__global__ void __launch_bounds__(kThreads, 1024 / kThreads) k_clf_step(sw_clf_step_t P, int scap, int rcap) {
  if (P.n_steps <= 0) {
    clf_step_body<kThreads, kCompact, kPT>(P, scap, rcap);
    return;
  }
  const int64_t B = P.batch, H = P.hidden, NI = P.num_inputs, C = P.num_classes;
  const int n = P.slot_count;
  for (int s = 0; s < P.n_steps; ++s) {
    sw_clf_step_t Q = P;
    const int t = P.t + s;
    const int64_t cur = t % n, prev = ((t - 1) % n + n) % n;
    Q.t = t;
    Q.zbar = P.zbar + cur * B * H;
    Q.zbar_in = P.zbar + prev * B * H;
    Q.xbar = P.xbar + cur * B * NI;
    Q.xbar_in = P.xbar + prev * B * NI;
    Q.psi = P.psi + cur * B * H;
    Q.lsig = P.lsig ? P.lsig + cur * B * H : nullptr;
    Q.d = P.d + cur * B * C;
    if (s) __syncthreads();   // this block's step s-1 writes are visible to its step s
    clf_step_body<kThreads, kCompact, kPT>(Q, scap, rcap, s == 0);
  }
}

// loss / accuracy of a batch (classifier.py:231-233)
__global__ void k_clf_batch_stats(const double* loss, const double* pi_sum, const int32_t* labels,
                                  int B, int C, double* out2) {
  __shared__ double sl[kThreads];
  __shared__ int sc[kThreads];
  double l = 0.0;
  int correct = 0;
  for (int b = threadIdx.x; b < B; b += kThreads) {
    l += loss[b];
    int best = 0;
    double bv = pi_sum[(int64_t)b * C];
    for (int c = 1; c < C; ++c) {
      const double v = pi_sum[(int64_t)b * C + c];
      if (v > bv) { bv = v; best = c; }
    }
    correct += (best == labels[b]);
  }
  sl[threadIdx.x] = l;
  sc[threadIdx.x] = correct;
  __syncthreads();
  if (threadIdx.x == 0) {
    double L = 0.0;
    int K = 0;
    for (int t = 0; t < kThreads; ++t) { L += sl[t]; K += sc[t]; }
    out2[0] = L;
    out2[1] = (double)K;
  }
}

__global__ void k_f64_to_f32(const double* in, float* out, int64_t n) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    out[x] = __double2float_rn(in[x]);
}

__global__ void k_scale_f64(double* x, int64_t n, double s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __dmul_rn(x[i], s);
}

int grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int sw_debug_clf_prof(long long* out16) {
  return cudaMemcpyFromSymbol(out16, g_clf_prof, 16 * sizeof(long long)) == cudaSuccess ? 0 : SW_ERR_CUDA;
}

// bytes of clf_step_body's shared-memory layout
size_t clf_smem_bytes(int H, int NI, int C, int scap, int rcap, bool compact) {
  const size_t NT = (size_t)NI + H, ix = compact ? 2 : 4;
  size_t o = (size_t)2 * H * 4;                 // acc_ext, acc_rec
  o += NT * ix;                                 // rlen
  o = (o + 3) & ~(size_t)3;
  o += NT * 4 + (size_t)(rcap + 1) * 4;         // list, roff
  o += (size_t)scap * 8;                        // st_kr, st_w
  o += (size_t)scap * ix;                       // srow
  o = (o + 3) & ~(size_t)3;
  o += (size_t)scap * 4;                        // sw_
  o += (size_t)(2 * H + 1) * ix;                // koff
  o = (o + 3) & ~(size_t)3;
  o += (size_t)2 * H * 4;                       // kcur
  o = (o + 15) & ~(size_t)15;
  return o + (size_t)(compact ? 2 : 5) * C * 8 + 16;   // yv, dv (+ ypre, pipre, bpre)
}

int clf_fwd_launch(const sw_clf_step_t* p, void* stream);    // classifier_fwd.cu
int clf_fwd2_launch(const sw_clf_step_t* p, void* stream);   // classifier_fwd2.cu

extern "C" int sw_clf_step(const sw_clf_step_t* p, void* stream) {
  const int H = p->hidden, NI = p->num_inputs, C = p->num_classes;
  if (p->batch <= 0) return SW_OK;
  if (p->n_steps > 0 && p->slot_count < 2) {
    sw::set_last_error("clf_step: n_steps > 0 needs slot_count >= 2 (step t reads slot t-1)");
    return SW_ERR_INVALID_ARG;
  }
  // register-resident forward (classifier_fwd.cu) for layers up to 1024
  // inputs and 1024 hidden units; SW_CLF_KERNEL=staged selects k_clf_step
  static const bool legacy = [] {
    const char* e = getenv("SW_CLF_KERNEL");
    return e && e[0] == 's';
  }();
  if (!legacy && p->in_bits && clf_fwd2_launch(p, stream) == SW_OK) {
    SW_CHECK_LAUNCH("sw_clf_step");
    return SW_OK;
  }
  if (!legacy && clf_fwd_launch(p, stream) == SW_OK) {
    SW_CHECK_LAUNCH("sw_clf_step");
    return SW_OK;
  }
  if (NI + H > kThreads * kPerThread) {
    sw::set_last_error("clf_step: num_inputs + hidden must be <= 2048");
    return SW_ERR_INVALID_ARG;
  }
  // 256-thread blocks (64 registers) reach 4 blocks per SM, i.e. one wave of
  // the batch's replica blocks, if a block's shared memory stays <= ~56 KB:
  // shrink the staged-path capacities (spiking rows, then staged entries;
  // beyond them the warp-serial fallback runs) until it does; else 512-thread
  // blocks.  SW_CLF_THREADS=512 forces the latter (measurement).
  const int NT = NI + H;
  const size_t budget = 56 * 1024;
  int threads = 256, scap = kStageCap, rcap = NT;
  bool compact = false;
  size_t smem = clf_smem_bytes(H, NI, C, scap, rcap, false);
  if (smem > budget) {
    compact = true;
    rcap = NT < 1024 ? NT : 1024;
    smem = clf_smem_bytes(H, NI, C, scap, rcap, true);
    if (smem > budget) { scap = 1536; smem = clf_smem_bytes(H, NI, C, scap, rcap, true); }
  }
  const char* force = getenv("SW_CLF_THREADS");
  if (smem > budget || (force && atoi(force) == 512)) {
    threads = 512;
    compact = false;
    scap = kStageCap;
    rcap = NT;
    smem = clf_smem_bytes(H, NI, C, scap, rcap, false);
  }
  if (smem > 227 * 1024) { sw::set_last_error("clf_step: layer too large"); return SW_ERR_INVALID_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  const bool pt4 = threads == 256 && !compact && NT <= 4 * 256;
  const void* fn = threads == 512 ? (const void*)k_clf_step<512, false, 8>
                   : compact      ? (const void*)k_clf_step<256, true, 8>
                   : pt4          ? (const void*)k_clf_step<256, false, 4>
                                  : (const void*)k_clf_step<256, false, 8>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (threads == 512)
    k_clf_step<512, false, 8><<<p->batch, 512, smem, st>>>(*p, scap, rcap);
  else if (compact)
    k_clf_step<256, true, 8><<<p->batch, 256, smem, st>>>(*p, scap, rcap);
  else if (pt4)
    k_clf_step<256, false, 4><<<p->batch, 256, smem, st>>>(*p, scap, rcap);
  else
    k_clf_step<256, false, 8><<<p->batch, 256, smem, st>>>(*p, scap, rcap);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_clf_step");
  return SW_OK;
}

extern "C" int sw_clf_batch_stats(const double* loss, const double* pi_sum, const int32_t* labels,
                                  int32_t batch, int32_t num_classes, double* out2, void* stream) {
  k_clf_batch_stats<<<1, kThreads, 0, (cudaStream_t)stream>>>(loss, pi_sum, labels, batch, num_classes, out2); sw::count_launch();
  SW_CHECK_LAUNCH("sw_clf_batch_stats");
  return SW_OK;
}

namespace {
struct ZeroArgs {
  char* p[SW_ZERO_MAX_RANGES];
  int64_t n[SW_ZERO_MAX_RANGES];
  int count;
};
// 16-byte stores over each range's aligned body, bytes at its ends
__global__ void k_zero_ranges(const ZeroArgs A) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < A.count; ++r) {
    char* p = A.p[r];
    const int64_t n = A.n[r];
    const int64_t head = min(n, (int64_t)((16 - ((uintptr_t)p & 15)) & 15));
    const int64_t body = (n - head) >> 4;
    uint4* q = reinterpret_cast<uint4*>(p + head);
    for (int64_t x = tid; x < body; x += nt) q[x] = make_uint4(0u, 0u, 0u, 0u);
    const int64_t tail0 = head + body * 16;
    for (int64_t x = tid; x < head; x += nt) p[x] = 0;
    for (int64_t x = tail0 + tid; x < n; x += nt) p[x] = 0;
  }
}
}  // namespace

extern "C" int sw_zero_ranges(void* const* ptrs, const int64_t* bytes, int32_t n, void* stream) {
  if (n < 0 || n > SW_ZERO_MAX_RANGES || (n > 0 && (!ptrs || !bytes))) {
    sw::set_last_error("sw_zero_ranges: 0 <= n <= SW_ZERO_MAX_RANGES");
    return SW_ERR_INVALID_ARG;
  }
  ZeroArgs A{};
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    if (bytes[i] < 0 || (bytes[i] > 0 && !ptrs[i])) {
      sw::set_last_error("sw_zero_ranges: negative size or null range");
      return SW_ERR_INVALID_ARG;
    }
    A.p[A.count] = (char*)ptrs[i];
    A.n[A.count] = bytes[i];
    A.count += bytes[i] > 0;
    total += bytes[i];
  }
  if (total == 0) return SW_OK;
  int64_t g = (total / 16 + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  k_zero_ranges<<<(int)(g < 1 ? 1 : g), 256, 0, (cudaStream_t)stream>>>(A);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_zero_ranges");
  return SW_OK;
}

extern "C" int sw_f64_to_f32(const double* in, float* out, int64_t n, void* stream) {
  if (n <= 0) return SW_OK;
  k_f64_to_f32<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(in, out, n); sw::count_launch();
  SW_CHECK_LAUNCH("sw_f64_to_f32");
  return SW_OK;
}

extern "C" int sw_scale_f64(double* x, int64_t n, double s, void* stream) {
  if (n <= 0) return SW_OK;
  k_scale_f64<<<grid1(n), 256, 0, (cudaStream_t)stream>>>(x, n, s); sw::count_launch();
  SW_CHECK_LAUNCH("sw_scale_f64");
  return SW_OK;
}
