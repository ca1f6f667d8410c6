// The e-prop ALIF classifier forward pass, block per replica, a group of
// timesteps per launch (sparsewire/classifier.py:196-234).
//
// The replica's own state (v, a, z, zbar, xbar and the input-spike
// thresholds) stays in registers across the steps of a launch: thread t owns
// hidden units [t*HPT, t*HPT + HPT) and inputs [t*IPT, t*IPT + IPT).  Per step:
//   P1  input spikes from the example's counter stream (classifier.py:63-67:
//       uniform01 #(t*NI + k) < p_k, evaluated as the exact integer compare
//       (h >> 11) < ceil(p_k * 2^53)); xbar/zbar updates; one block scan gives
//       the ascending spiking-row lists and their staging offsets;
//   P2  every warp stages spiking rows' (target, w) entries into shared
//       memory (cp.async); then warp 0 sums the input rows and warp 1 the
//       recurrent rows into per-post accumulators, row after row in ascending
//       row order -- the ascending-pre float32 sequential sum per post, with no
//       sort (a row's targets are distinct, so its lanes never collide) --
//       while warps 2.. compute the leaky readout, softmax, cross-entropy and
//       d = pi - onehot (classifier.py:215-219);
//   P3  every thread: surrogate psi from the pre-step state, learning signal
//       lsig = f32(d @ W_out) (classes ascending), ALIF step (neurons.py:60-73).
// The arithmetic of every output is that of k_clf_step (classifier.cu), op for
// op; only the work distribution differs.
#include "common.cuh"
#include "sm100_async.cuh"

#include <cmath>

namespace {

// phase timestamps of block 7, step 3 (tools/fwd_phases.py); armed by sw_debug_fwd_prof
__device__ long long g_fwd_prof[16];
__device__ int g_fwd_prof_on;
#ifdef SW_FWD_PROF
#define FWD_PROF(i) do { if (g_fwd_prof_on && blockIdx.x == 7 && s == 3 && (threadIdx.x & 31) == 0) \
    g_fwd_prof[(i) + 8 * (threadIdx.x >= 32)] = clock64(); } while (0)
#else
#define FWD_PROF(i) do { } while (0)
#endif

constexpr int kT = 256;          // threads per replica block
constexpr int kW = kT / 32;
constexpr int kStage = 2048;     // staged (target, w) entries per step

__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// row groups of the event-driven current sums (see P2b)
__host__ __device__ inline int fwd_groups(int H) {
  return H <= 256 ? 8 : 4;   // classifier_fwd2.cu fwd2_groups: the same groups
}

// bytes of the dynamic shared-memory layout
__host__ __device__ inline size_t fwd_smem_bytes(int H, int NI, int C) {
  const size_t NT = (size_t)NI + H;
  size_t o = 0;
  o += (size_t)fwd_groups(H) * H * 4; // per-group partial sums
  o += NT * 4;                       // rlen
  o += NT * 4;                       // list (spiking rows: inputs, then hidden units NI + h)
  o += (NT + 1) * 4;                 // staging offset per list entry
  o = (o + 15) & ~(size_t)15;
  o += (size_t)kStage * 8;           // staged (target, weight) pairs
  o += 16;                           // staging mbarrier
  o += (size_t)4 * C * 8;            // y, pi_sum, d, b_out
  o += (size_t)NI * 8;               // input-spike thresholds
  return o;
}

template <int HPT, int IPT>
__global__ void __launch_bounds__(kT, 4) k_clf_fwd(sw_clf_step_t P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int H = P.hidden, NI = P.num_inputs, C = P.num_classes;
  const int NT = NI + H;
  size_t o = 0;
  const int G = fwd_groups(H);
  float* part = (float*)(smem_raw + o);    o += (size_t)G * H * 4;
  int* rlen = (int*)(smem_raw + o);        o += (size_t)NT * 4;
  int* list = (int*)(smem_raw + o);        o += (size_t)NT * 4;
  int* soff = (int*)(smem_raw + o);        o += (size_t)(NT + 1) * 4;
  o = (o + 15) & ~(size_t)15;
  int2* st = (int2*)(smem_raw + o);        o += (size_t)kStage * 8;
  uint64_t* sbar = (uint64_t*)(smem_raw + o); o += 16;
  double* yv = (double*)(smem_raw + o);
  double* pis = yv + C;
  double* dv = pis + C;
  double* bo = dv + C;
  uint64_t* thr = (uint64_t*)(bo + C);
  __shared__ int4 wsum[kW];
  __shared__ double s_loss;

  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 32-bit element offsets (B * max(H, NI) * slot_count < 2^31)
  const int bH = b * H, bI = b * NI, bC = b * C;
  const int B = P.batch;
  const bool grouped = P.n_steps > 0;
  const int nsteps = grouped ? P.n_steps : 1;
  const int nslot = grouped ? P.slot_count : 1;

  // ---- launch prologue: replica state into registers / shared memory ----
  for (int x = tid; x < NT; x += kT)
    rlen[x] = (x < NI) ? __ldg(P.in_row_length + x) : __ldg(P.rec_row_length + (x - NI));
  for (int c = tid; c < C; c += kT) {
    yv[c] = P.y[bC + c];
    pis[c] = P.pi_sum[bC + c];
    bo[c] = P.b_out[c];
  }
  if (tid == 0) {
    s_loss = P.loss[b];
    sw::mbar_init(sbar, 1);
    sw::fence_mbar_init();
  }
  for (int x = tid; x < G * H; x += kT) part[x] = 0.0f;
  const float* zin0;
  const float* xin0;
  if (grouped) {
    const int prev = ((P.t - 1) % nslot + nslot) % nslot;
    zin0 = P.zbar + prev * B * H;
    xin0 = P.xbar + prev * B * NI;
  } else {
    zin0 = P.zbar_in ? P.zbar_in : P.zbar;
    xin0 = P.xbar_in ? P.xbar_in : P.xbar;
  }
  float v[HPT], a[HPT], z[HPT], zb[HPT];
  const int h0 = tid * HPT;
#pragma unroll
  for (int j = 0; j < HPT; ++j) {
    const int h = h0 + j;
    const bool ok = h < H;
    v[j] = ok ? P.v[bH + h] : 0.f;
    a[j] = ok ? P.a[bH + h] : 0.f;
    z[j] = ok ? P.z[bH + h] : 0.f;
    zb[j] = ok ? zin0[bH + h] : 0.f;
  }
  float xb[IPT];
  const int x0 = tid * IPT;
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int x = x0 + j;
    const bool ok = x < NI;
    xb[j] = ok ? xin0[bI + x] : 0.f;
    // u01(h) < p  <=>  (h >> 11) < ceil(p * 2^53)  (both sides exact)
    if (ok) thr[x] = (uint64_t)ceil(P.p_in[bI + x] * 0x1p53);
  }
  const uint64_t key = P.ex_key[b];
  const int label = P.labels[b];
  const float alpha = P.alpha, rho = P.rho, beta = P.beta, v_thr = P.v_thr;
  __syncthreads();   // thresholds staged

  uint32_t sphase = 0;
  for (int s = 0; s < nsteps; ++s) {
    const int t = P.t + s;
    const int cur = grouped ? t % nslot : 0;
    float* zbar_o = P.zbar + cur * B * H;
    float* xbar_o = P.xbar + cur * B * NI;
    float* psi_o = P.psi + cur * B * H;
    float* lsig_o = P.lsig + cur * B * H;
    double* d_o = P.d + cur * B * C;

    FWD_PROF(0);
    // ---- P1: spikes, traces, ascending spiking-row lists ----
    unsigned fin = 0, frec = 0;
    int len_in = 0, len_rec = 0;
    const uint64_t c0 = (uint64_t)t * (uint64_t)NI + (uint64_t)x0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const int x = x0 + j;
      if (x < NI) {
        const bool f = (sw::draw(key, c0 + j) >> 11) < thr[x];
        xb[j] = __fadd_rn(__fmul_rn(xb[j], alpha), f ? 1.0f : 0.0f);
        xbar_o[bI + x] = xb[j];
        if (f) { fin |= 1u << j; len_in += (rlen[x] + 1) & ~1; }
      }
    }
#pragma unroll
    for (int j = 0; j < HPT; ++j) {
      const int h = h0 + j;
      if (h < H) {
        zb[j] = __fadd_rn(__fmul_rn(zb[j], alpha), z[j]);
        zbar_o[bH + h] = zb[j];
        if (z[j] != 0.0f) { frec |= 1u << j; len_rec += (rlen[NI + h] + 1) & ~1; }
      }
    }
    // block scan of (input count, input entries, hidden count, hidden entries)
    int4 mine = make_int4(__popc(fin), len_in, __popc(frec), len_rec);
    int4 inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int ax = __shfl_up_sync(SW_FULL_MASK, inc.x, d), ay = __shfl_up_sync(SW_FULL_MASK, inc.y, d);
      const int az = __shfl_up_sync(SW_FULL_MASK, inc.z, d), aw = __shfl_up_sync(SW_FULL_MASK, inc.w, d);
      if (lane >= d) { inc.x += ax; inc.y += ay; inc.z += az; inc.w += aw; }
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();   // B1a
    int4 pre = make_int4(0, 0, 0, 0), tot = make_int4(0, 0, 0, 0);
#pragma unroll
    for (int w = 0; w < kW; ++w) {
      const int4 q = wsum[w];
      if (w < warp) { pre.x += q.x; pre.y += q.y; pre.z += q.z; pre.w += q.w; }
      tot.x += q.x; tot.y += q.y; tot.z += q.z; tot.w += q.w;
    }
    const int nx = tot.x, nz = tot.z, ent = tot.y + tot.w;
    {
      int pos = pre.x + inc.x - mine.x, off = pre.y + inc.y - mine.y;
#pragma unroll
      for (int j = 0; j < IPT; ++j)
        if ((fin >> j) & 1u) { list[pos] = x0 + j; soff[pos] = off; off += (rlen[x0 + j] + 1) & ~1; ++pos; }
      pos = nx + pre.z + inc.z - mine.z;
      off = tot.y + pre.w + inc.w - mine.w;
#pragma unroll
      for (int j = 0; j < HPT; ++j)
        if ((frec >> j) & 1u) { list[pos] = NI + h0 + j; soff[pos] = off; off += (rlen[NI + h0 + j] + 1) & ~1; ++pos; }
    }
    if (tid == 0) soff[nx + nz] = ent;
    const bool staged = ent <= kStage;
    // one mbarrier phase per step: tid 0 expects every staged byte, the
    // row copies complete them
    if (tid == 0 && staged) sw::mbar_arrive_expect_tx(sbar, (uint32_t)ent * 8u);
    __syncthreads();   // B1b: lists and offsets ready
    FWD_PROF(1);

    // ---- P2a: stage the spiking rows' packed (target, w) entries: one bulk
    // copy per row (16-byte multiples: rows padded to even entries) ----
    if (staged) {
      for (int r = tid; r < nx + nz; r += kT) {
        const int x = list[r];
        const bool in = x < NI;
        const int32_t* src = in ? P.in_tw + (int64_t)x * P.in_tw_stride * 2
                                : P.rec_tw + (int64_t)(x - NI) * P.rec_tw_stride * 2;
        const uint32_t bytes = (uint32_t)((rlen[x] + 1) & ~1) * 8u;
        if (bytes) sw::bulk_g2s(st + soff[r], src, bytes, sbar);
      }
    }

    // ---- P2b: readout + softmax (last warp) while the staged rows land ----
    if (warp == kW - 1) {
      // readout y = alpha*y + z @ W_out^T + b (classifier.py:215), lane = class:
      // the spiking hidden units' W_out columns added in ascending unit
      // order; then softmax / cross-entropy / d (plasticity.py:156-165,
      // classifier.py:216-219) on the same lanes
      const int* zl = list + nx;
      for (int c0 = 0; c0 < C; c0 += 32) {
        const int c = c0 + lane;
        if (c < C) {
          double sacc = 0.0;
          const double* wr = P.w_out + (int64_t)c * H - NI;
          for (int q = 0; q < nz; ++q) sacc = __dadd_rn(sacc, __ldg(wr + zl[q]));
          yv[c] = __dadd_rn(__dadd_rn(__dmul_rn(P.alpha64, yv[c]), sacc), bo[c]);
        }
      }
      __syncwarp();
      double mx = -INFINITY;
      for (int c = lane; c < C; c += 32) mx = fmax(mx, yv[c]);
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) mx = fmax(mx, __shfl_xor_sync(SW_FULL_MASK, mx, o2));
      double se = 0.0;
      double ex[2] = {0.0, 0.0};
      for (int c = lane, u = 0; c < C; c += 32, ++u) {
        const double e = exp(yv[c] - mx);
        if (u < 2) ex[u] = e;
        se += e;
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) se += __shfl_xor_sync(SW_FULL_MASK, se, o2);
      for (int c = lane, u = 0; c < C; c += 32, ++u) {
        const double pi = (u < 2 ? ex[u] : exp(yv[c] - mx)) / se;
        pis[c] = pis[c] + pi;
        const double dd = pi - (c == label ? 1.0 : 0.0);
        dv[c] = dd;
        d_o[bC + c] = dd;
        if (c == label) s_loss = s_loss + -log(pi);
      }
    }
    if (staged) sw::mbar_wait(sbar, sphase & 1u);
    sphase += staged ? 1u : 0u;   // one barrier phase per staged step
    FWD_PROF(2);

    // ---- P2c: event-driven currents (classifier.py:208-209 as ragged sums).
    // The ascending spiking rows of a projection are split into G contiguous
    // groups, group g = rows [n*g/G, n*(g+1)/G) summed by warp g into its
    // own partial row (row after row in ascending order, lanes over a row's
    // distinct targets); then per post the group sums are added in group
    // order: sum = ((p_0 + p_1) + ...) + p_{G-1}, every p_g starting from
    // +0.0 (a group without an entry for the post adds +0.0, which changes
    // nothing).  Input rows first, then the recurrent rows. ----
    float aext[HPT], arec[HPT];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int rb = half == 0 ? 0 : nx, n = half == 0 ? nx : nz;
      if (warp < G) {
        float* pg = part + warp * H;
        const int g0 = rb + n * warp / G, g1 = rb + n * (warp + 1) / G;
        for (int r = g0; r < g1; ++r) {
          const int x = list[r];
          const int len = rlen[x];
          const int2* e;
          if (staged) {
            e = st + soff[r];
          } else {
            const bool in = x < NI;
            e = reinterpret_cast<const int2*>(in ? P.in_tw + (int64_t)x * P.in_tw_stride * 2
                                                 : P.rec_tw + (int64_t)(x - NI) * P.rec_tw_stride * 2);
          }
          for (int q = lane; q < len; q += 32) {
            const int2 tw = staged ? e[q] : __ldg(e + q);
            pg[tw.x] = __fadd_rn(pg[tw.x], __int_as_float(tw.y));
          }
          __syncwarp();
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < HPT; ++j) {
        const int h = h0 + j;
        float a0 = 0.0f;
        if (h < H) {
          a0 = part[h];
          part[h] = 0.0f;
          for (int g = 1; g < G; ++g) {
            a0 = __fadd_rn(a0, part[g * H + h]);
            part[g * H + h] = 0.0f;
          }
        }
        if (half == 0) aext[j] = a0; else arec[j] = a0;
      }
      __syncthreads();
      FWD_PROF(3 + half);
    }

    // ---- P3: psi (pre-step state), lsig, ALIF step ----
#pragma unroll
    for (int j = 0; j < HPT; ++j) {
      const int h = h0 + j;
      if (h >= H) continue;
      const float thr_o = __fadd_rn(v_thr, __fmul_rn(beta, a[j]));
      const float cc = __fdiv_rn(__fsub_rn(v[j], thr_o), v_thr);
      const float r = __fsub_rn(1.0f, fabsf(cc));
      psi_o[bH + h] = __fmul_rn(0.5f, (r > 0.0f || r != r) ? r : 0.0f);
      if (P.lsig) {   // NULL: the learning signal is computed by sw_eprop_prep
        double ls = 0.0;
        const double* wc = P.w_out + h;
        int c = 0;
        for (; c + 4 <= C; c += 4) {
          const double w0 = __ldg(wc), w1 = __ldg(wc + H), w2 = __ldg(wc + 2 * H), w3 = __ldg(wc + 3 * H);
          wc += 4 * H;
          ls = __fma_rn(dv[c], w0, ls);
          ls = __fma_rn(dv[c + 1], w1, ls);
          ls = __fma_rn(dv[c + 2], w2, ls);
          ls = __fma_rn(dv[c + 3], w3, ls);
        }
        for (; c < C; ++c, wc += H) ls = __fma_rn(dv[c], __ldg(wc), ls);
        lsig_o[bH + h] = __double2float_rn(ls);
      }
      float vv = __fmul_rn(alpha, __fsub_rn(v[j], __fmul_rn(z[j], v_thr)));
      vv = __fadd_rn(__fadd_rn(vv, arec[j]), aext[j]);
      const float aa = __fadd_rn(__fmul_rn(rho, a[j]), z[j]);
      v[j] = vv;
      a[j] = aa;
      z[j] = (vv >= __fadd_rn(v_thr, __fmul_rn(beta, aa))) ? 1.0f : 0.0f;
    }
    FWD_PROF(5);
    // the next step's P1 reads only this thread's registers and writes the
    // lists after its own barrier B1a, which every thread reaches only after
    // finishing this step's P3
  }

  // ---- launch epilogue: replica state back to HBM ----
#pragma unroll
  for (int j = 0; j < HPT; ++j) {
    const int h = h0 + j;
    if (h < H) {
      P.v[bH + h] = v[j];
      P.a[bH + h] = a[j];
      P.z[bH + h] = z[j];
    }
  }
  __syncthreads();
  for (int c = tid; c < C; c += kT) {
    P.y[bC + c] = yv[c];
    P.pi_sum[bC + c] = pis[c];
  }
  if (tid == 0) P.loss[b] = s_loss;
}

template <int HPT, int IPT>
int launch_fwd(const sw_clf_step_t* p, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute((const void*)k_clf_fwd<HPT, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_clf_fwd<HPT, IPT><<<p->batch, kT, smem, st>>>(*p);
  sw::count_launch();
  return SW_OK;
}

__global__ void k_pack_rows(const int32_t* row_length, const int32_t* target, const double* w, int P,
                            int stride, int tws, int32_t* tw) {
  const int64_t n = (int64_t)P * tws;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(x / tws), q = (int)(x - (int64_t)i * tws);
    const bool ok = q < row_length[i];
    tw[2 * x] = ok ? target[(int64_t)i * stride + q] : 0;
    tw[2 * x + 1] = ok ? __float_as_int(__double2float_rn(w[(int64_t)i * stride + q])) : 0;
  }
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int sw_debug_fwd_prof(int enable, long long* out16) {
  if (out16 && cudaMemcpyFromSymbol(out16, g_fwd_prof, 16 * sizeof(long long)) != cudaSuccess) return SW_ERR_CUDA;
  return cudaMemcpyToSymbol(g_fwd_prof_on, &enable, sizeof(int)) == cudaSuccess ? 0 : SW_ERR_CUDA;
}

extern "C" int sw_clf_pack_rows(const int32_t* row_length, const int32_t* target, const double* w,
                                int32_t num_pre, int32_t stride, int32_t tw_stride, int32_t* tw, void* stream) {
  if (tw_stride < stride || (tw_stride & 1)) {
    sw::set_last_error("sw_clf_pack_rows: tw_stride must be even and >= stride");
    return SW_ERR_INVALID_ARG;
  }
  const int64_t n = (int64_t)num_pre * tw_stride;
  if (n == 0) return SW_OK;
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  k_pack_rows<<<(int)g, 256, 0, (cudaStream_t)stream>>>(row_length, target, w, num_pre, stride, tw_stride, tw);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_clf_pack_rows");
  return SW_OK;
}

// sw_clf_step's fast path (classifier.cu); returns SW_ERR_INVALID_ARG when
// the layer shapes are outside its register layout (the caller then runs
// k_clf_step).
int clf_fwd_launch(const sw_clf_step_t* p, void* stream) {
  const int H = p->hidden, NI = p->num_inputs, C = p->num_classes;
  if (H < 1 || H > 4 * kT || NI < 1 || NI > 4 * kT || C < 1 || !p->in_tw || !p->rec_tw) return SW_ERR_INVALID_ARG;
  const size_t smem = fwd_smem_bytes(H, NI, C);
  if (smem > 200 * 1024) return SW_ERR_INVALID_ARG;
  const int hpt = (H + kT - 1) / kT, ipt = (NI + kT - 1) / kT;
  const int hsel = hpt == 1 ? 1 : (hpt == 2 ? 2 : 4);
  cudaStream_t st = (cudaStream_t)stream;
#define SW_FWD_CASE(HH, II) if (hsel == HH && ipt <= II) return launch_fwd<HH, II>(p, smem, st)
  SW_FWD_CASE(1, 1); SW_FWD_CASE(1, 3); SW_FWD_CASE(1, 4);
  SW_FWD_CASE(2, 3); SW_FWD_CASE(2, 4);
  SW_FWD_CASE(4, 3); SW_FWD_CASE(4, 4);
#undef SW_FWD_CASE
  return SW_ERR_INVALID_ARG;
}
