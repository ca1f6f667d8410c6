// One timestep of the e-prop ALIF classifier forward pass, fused per replica
// (sparsewire/classifier.py:188-234).  Block per replica:
//   1. input spikes of the synthetic task from the example's counter stream
//      (classifier.py:63-67: u = uniform01 #(t*NI + k) < p_e[k]); xbar update;
//   2. ascending spike lists (input, hidden) in shared memory; zbar update;
//   3. event-driven ragged propagation: warp 0 walks the spiking input rows,
//      warp 1 the spiking hidden rows, in ascending row order, lanes over a
//      row's slots (targets are distinct within a row), accumulating float32
//      currents in shared memory — per post this is the ascending-pre
//      sequential sum (classifier.py:208-209 computes the same sums as a
//      dense sgemm on a float32 weight copy);
//   4. surrogate psi from the pre-step state (neurons.py:69-73);
//   5. leaky readout y, softmax, cross-entropy, d = pi - onehot, pi_sum,
//      learning signal lsig = f32(d @ W_out) (classifier.py:215-223);
//   6. ALIF step with the new currents (neurons.py:60-67).
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// Block-wide ascending compaction of flags over [0, n): list gets the
// indices with flag set, *count the number.  flag_fn(k) -> bool.
template <typename F>
__device__ void block_compact(int n, F flag_fn, int* list, int* count, int* warp_cnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) *count = 0;
  __syncthreads();
  for (int base = 0; base < n; base += kThreads) {
    const int k = base + threadIdx.x;
    const bool f = (k < n) && flag_fn(k);
    const unsigned b = __ballot_sync(SW_FULL_MASK, f);
    if (lane == 0) warp_cnt[warp] = __popc(b);
    __syncthreads();
    int before = *count;
    for (int w = 0; w < warp; ++w) before += warp_cnt[w];
    if (f) list[before + __popc(b & sw::lanemask_lt())] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < kWarps; ++w) tot += warp_cnt[w];
      *count += tot;
    }
    __syncthreads();
  }
}

// Warp-serial ascending-row accumulation into shared memory.
__device__ void warp_accumulate_rows(const int* list, int n, const int32_t* __restrict__ row_length,
                                     const int32_t* __restrict__ target, const float* __restrict__ w32,
                                     int stride, float* acc) {
  const int lane = threadIdx.x & 31;
  for (int r0 = 0; r0 < n; r0 += 4) {
    int len[4], t[4];
    float w[4];
    int64_t off[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      len[u] = 0;
      t[u] = 0;
      w[u] = 0.f;
      off[u] = 0;
      if (r0 + u < n) {
        const int i = list[r0 + u];
        off[u] = (int64_t)i * stride;
        len[u] = __ldg(row_length + i);
        if (lane < len[u]) {
          t[u] = __ldg(target + off[u] + lane);
          w[u] = __ldg(w32 + off[u] + lane);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (lane < len[u]) acc[t[u]] = __fadd_rn(acc[t[u]], w[u]);
      for (int c = 32 + lane; c < len[u]; c += 32) {
        const int tt = __ldg(target + off[u] + c);
        acc[tt] = __fadd_rn(acc[tt], __ldg(w32 + off[u] + c));
      }
      __syncwarp();
    }
  }
}

constexpr int kStageCap = 4096;   // staged (target, w) entries of the spiking rows

// Ordered adds of staged rows: rows r0..r1-1 of the staged list, each row's
// entries [off[r], off[r+1]) added by the lanes; rows strictly in order.
__device__ __forceinline__ void warp_add_staged(const int* off, int r0, int r1, const int* st_t,
                                                const float* st_w, float* acc) {
  const int lane = threadIdx.x & 31;
  for (int r = r0; r < r1; ++r) {
    for (int q = off[r] + lane; q < off[r + 1]; q += 32) acc[st_t[q]] = __fadd_rn(acc[st_t[q]], st_w[q]);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kThreads) k_clf_step(sw_clf_step_t P) {
  extern __shared__ unsigned char smem_raw[];
  const int H = P.hidden, NI = P.num_inputs, C = P.num_classes;
  float* acc_ext = (float*)smem_raw;
  float* acc_rec = acc_ext + H;
  int* xlist = (int*)(acc_rec + H);
  int* zlist = xlist + NI;
  int* roff = zlist + H;                    // [NI + H + 1] staged row offsets
  int* st_t = roff + NI + H + 1;            // [kStageCap]
  float* st_w = (float*)(st_t + kStageCap); // [kStageCap]
  double* yv = (double*)(((uintptr_t)(st_w + kStageCap) + 15) & ~(uintptr_t)15);
  double* dv = yv + C;
  __shared__ int warp_cnt[kWarps];
  __shared__ int nx, nz;
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t bH = (int64_t)b * H, bI = (int64_t)b * NI, bC = (int64_t)b * C;

  // 1. input spikes (classifier.py:63-67) + xbar (:212-213), one draw per input
  const uint64_t key = P.ex_key[b];
  const uint64_t c0 = (uint64_t)P.t * (uint64_t)NI;
  const double* pin = P.p_in + bI;
  auto xspk = [&](int k) {
    const bool f = sw::u01(sw::draw(key, c0 + (uint64_t)k)) < pin[k];
    P.xbar[bI + k] = __fadd_rn(__fmul_rn(P.xbar[bI + k], P.alpha), f ? 1.0f : 0.0f);
    return f;
  };
  block_compact(NI, xspk, xlist, &nx, warp_cnt);
  // 2. hidden spike list (old z) + zbar (classifier.py:207, 210-211)
  const float* z = P.z + bH;
  block_compact(H, [&](int h) {
    const float zh = z[h];
    P.zbar[bH + h] = __fadd_rn(__fmul_rn(P.zbar[bH + h], P.alpha), zh);
    acc_ext[h] = 0.0f;
    acc_rec[h] = 0.0f;
    return zh != 0.0f;
  }, zlist, &nz, warp_cnt);
  // 3a. lengths of the spiking rows -> staged offsets (warp 0 scan)
  const int nrows = nx + nz;
  for (int r = threadIdx.x; r < nrows; r += kThreads)
    roff[r + 1] = (r < nx) ? __ldg(P.in_row_length + xlist[r]) : __ldg(P.rec_row_length + zlist[r - nx]);
  __syncthreads();
  if (warp == 0) {
    int carry = 0;
    for (int base = 0; base < nrows; base += 32) {
      const int r = base + lane;
      int v = r < nrows ? roff[r + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(SW_FULL_MASK, v, o);
        if (lane >= o) v += t;
      }
      if (r < nrows) roff[r + 1] = carry + v;
      carry += __shfl_sync(SW_FULL_MASK, v, 31);
    }
    if (lane == 0) roff[0] = 0;
  }
  __syncthreads();
  const bool staged = roff[nrows] <= kStageCap;
  // 3b. stage every spiking row's (target, w) with coalesced loads, all warps
  if (staged) {
    for (int r = warp; r < nrows; r += kWarps) {
      const bool in = r < nx;
      const int i = in ? xlist[r] : zlist[r - nx];
      const int64_t o = (int64_t)i * (in ? P.in_stride : P.rec_stride);
      const int32_t* tg = (in ? P.in_target : P.rec_target) + o;
      const float* wv = (in ? P.in_w32 : P.rec_w32) + o;
      const int q0 = roff[r], len = roff[r + 1] - q0;
      for (int c = lane; c < len; c += 32) {
        st_t[q0 + c] = __ldg(tg + c);
        st_w[q0 + c] = __ldg(wv + c);
      }
    }
  }
  __syncthreads();
  // 3c. ordered event-driven accumulation (warp 0: input rows, warp 1: hidden rows)
  if (warp == 0) {
    if (staged) warp_add_staged(roff, 0, nx, st_t, st_w, acc_ext);
    else warp_accumulate_rows(xlist, nx, P.in_row_length, P.in_target, P.in_w32, P.in_stride, acc_ext);
  } else if (warp == 1) {
    if (staged) warp_add_staged(roff, nx, nrows, st_t, st_w, acc_rec);
    else warp_accumulate_rows(zlist, nz, P.rec_row_length, P.rec_target, P.rec_w32, P.rec_stride, acc_rec);
  } else {
    // 5a. readout y = alpha*y + z @ W_out^T + b (classifier.py:215), warps 2.. over classes
    for (int c = warp - 2; c < C; c += kWarps - 2) {
      double s = 0.0;
      for (int q = lane; q < nz; q += 32) s += __ldg(P.w_out + (int64_t)c * H + zlist[q]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(SW_FULL_MASK, s, o);
      if (lane == 0) yv[c] = __dadd_rn(__dadd_rn(__dmul_rn(P.alpha64, P.y[bC + c]), s), P.b_out[c]);
    }
  }
  __syncthreads();
  // 5b. softmax / cross-entropy / d (plasticity.py:156-165, classifier.py:216-219)
  if (warp == 0) {
    double mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmax(mx, yv[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(SW_FULL_MASK, mx, o));
    double se = 0.0;
    for (int c = lane; c < C; c += 32) se += exp(yv[c] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(SW_FULL_MASK, se, o);
    const int label = P.labels[b];
    for (int c = lane; c < C; c += 32) {
      const double pi = exp(yv[c] - mx) / se;
      P.y[bC + c] = yv[c];
      P.pi_sum[bC + c] += pi;
      const double dd = pi - (c == label ? 1.0 : 0.0);
      dv[c] = dd;
      P.d[bC + c] = dd;
      if (c == label) P.loss[b] += -log(pi);
    }
  }
  __syncthreads();
  // 4 + 5c + 6: per hidden neuron
  for (int h = threadIdx.x; h < H; h += kThreads) {
    const float vo = P.v[bH + h], ao = P.a[bH + h], zo = z[h];
    const float thr_o = __fadd_rn(P.v_thr, __fmul_rn(P.beta, ao));
    const float cc = __fdiv_rn(__fsub_rn(vo, thr_o), P.v_thr);
    const float r = __fsub_rn(1.0f, fabsf(cc));
    P.psi[bH + h] = __fmul_rn(0.5f, (r > 0.0f || r != r) ? r : 0.0f);
    double ls = 0.0;
    for (int c = 0; c < C; ++c) ls = __dadd_rn(ls, __dmul_rn(dv[c], __ldg(P.w_out + (int64_t)c * H + h)));
    P.lsig[bH + h] = __double2float_rn(ls);
    float vv = __fmul_rn(P.alpha, __fsub_rn(vo, __fmul_rn(zo, P.v_thr)));
    vv = __fadd_rn(__fadd_rn(vv, acc_rec[h]), acc_ext[h]);
    const float aa = __fadd_rn(__fmul_rn(P.rho, ao), zo);
    P.v[bH + h] = vv;
    P.a[bH + h] = aa;
    P.z[bH + h] = (vv >= __fadd_rn(P.v_thr, __fmul_rn(P.beta, aa))) ? 1.0f : 0.0f;
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

extern "C" int sw_clf_step(const sw_clf_step_t* p, void* stream) {
  const int H = p->hidden, NI = p->num_inputs, C = p->num_classes;
  if (p->batch <= 0) return SW_OK;
  const size_t smem = (size_t)(2 * H) * 4 + (size_t)(NI + H) * 4 + (size_t)(NI + H + 1) * 4 +
                      (size_t)kStageCap * 8 + 16 + (size_t)2 * C * 8;
  if (smem > 48 * 1024) {
    if (smem > 227 * 1024) { sw::set_last_error("clf_step: layer too large"); return SW_ERR_INVALID_ARG; }
    cudaFuncSetAttribute((const void*)k_clf_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  k_clf_step<<<p->batch, kThreads, smem, (cudaStream_t)stream>>>(*p); sw::count_launch();
  SW_CHECK_LAUNCH("sw_clf_step");
  return SW_OK;
}

extern "C" int sw_clf_batch_stats(const double* loss, const double* pi_sum, const int32_t* labels,
                                  int32_t batch, int32_t num_classes, double* out2, void* stream) {
  k_clf_batch_stats<<<1, kThreads, 0, (cudaStream_t)stream>>>(loss, pi_sum, labels, batch, num_classes, out2); sw::count_launch();
  SW_CHECK_LAUNCH("sw_clf_batch_stats");
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
