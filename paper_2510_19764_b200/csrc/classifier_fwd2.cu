// The classifier's trial with the input side precomputed
// (sparsewire/classifier.py:63-67, 196-234).
//
// The input spikes and the input traces xbar do not depend on the network
// state, so two launches per batch (sw_clf_inputs) draw every input spike of
// the trial from the examples' counter streams (u = uniform01 #(t*NI + k) <
// p_k, as the exact integer compare (h >> 11) < ceil(p_k * 2^53)) and runs
// the xbar recursion: spike words in_bits[t][b][k/32] for the forward pass,
// and xbar_t[t][k][b] already in the replica-minor layout the e-prop pass
// reads (no transpose).
//
// The forward kernel (k_clf_fwd2, block per replica, a group of steps per
// launch, state in registers) then only builds its spiking-row lists from
// those words and the hidden spikes:
//   A  hidden spikes -> spike words in unit order (warp ballots), to shared
//      memory and to z_bits for the readout launch; one barrier;
//   C  warp g selects group g of the ascending input rows and group g of
//      the ascending hidden rows straight from the spike words (a popcount
//      scan per warp; G ordered groups by count, no list-building warp and
//      no second barrier) and sums them into its partial rows, reading the
//      packed (target, weight) rows with kRowsAhead rows' loads in flight;
//   D  per post the group partials are added in group order, the ALIF step
//      and the surrogate (neurons.py:60-73).
// The readout / softmax of all the launch's steps then runs as one launch
// (k_clf_readout): the steps' weight sums are independent, so their load
// latencies overlap instead of sitting on the forward pass's step chain.
// Every output is bit-identical to k_clf_fwd's (classifier_fwd.cu): the same
// per-post current sums (groups of the ascending rows, group order), the same
// readout / softmax / ALIF arithmetic.
#include "common.cuh"
#include "sm100_async.cuh"

#include <cmath>
#include <cstdlib>

namespace {

// phase timestamps of block 7, step 3 (tools/fwd_phases.py; sw_debug_fwd2_prof)
// (compiled in with -DSW_FWD_PROF only)
__device__ long long g_fwd2_prof[64];
__device__ int g_fwd2_prof_on;
#ifdef SW_FWD_PROF
#define FWD2_PROF(i) do { if (g_fwd2_prof_on && blockIdx.x == 7 && s == 3 && (threadIdx.x & 31) == 0) \
    g_fwd2_prof[(i) * 8 + (threadIdx.x >> 5)] = clock64(); } while (0)
#else
#define FWD2_PROF(i) do { } while (0)
#endif




// ------------------------------------------------------------- inputs ----
// (1) spike words: block = (replica, kSpkSteps steps), thread = (step, word of
//     32 inputs) flattened so every lane has a word; the replica's spike
//     thresholds ceil(p * 2^53) in shared memory
//     (u01(h) < p  <=>  (h >> 11) < ceil(p * 2^53), both sides exact)
constexpr int kSpkSteps = 32;
__global__ void __launch_bounds__(256) k_clf_spikes(const sw_clf_inputs_t P) {
  extern __shared__ uint64_t s_thr[];
  const int NI = P.num_inputs, W = P.words;
  const int b = blockIdx.x;
  const uint64_t key = __ldg(P.ex_key + b);
  // thresholds as [bit j][word w]: the lanes of a warp (consecutive words)
  // read consecutive entries (a [w][j] layout puts all 32 lanes in one bank)
  for (int x = threadIdx.x; x < NI; x += blockDim.x)
    s_thr[(x & 31) * W + (x >> 5)] = (uint64_t)ceil(__ldg(P.p_in + (int64_t)b * NI + x) * 0x1p53);
  __syncthreads();
  const int t0 = blockIdx.y * kSpkSteps;
  const int items = min(kSpkSteps, P.steps - t0) * W;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int tt = it / W, w = it - tt * W, t = t0 + tt;
    const int n = min(32, NI - w * 32);
    const uint64_t* thr = s_thr + w;
    const uint64_t c0 = (uint64_t)t * (uint64_t)NI + (uint64_t)(w * 32);
    uint32_t bits = 0;
#pragma unroll 4
    for (int j = 0; j < n; ++j)
      if ((sw::draw(key, c0 + j) >> 11) < thr[j * W]) bits |= 1u << j;
    P.in_bits[((int64_t)t * P.batch + b) * W + w] = bits;
  }
}

// (2) the xbar recursion (classifier.py:212-213): block = (word of 32 inputs,
//     32 replicas), warp = input, lane = replica, steps in order; the
//     block's spike words staged through shared memory kXbSteps steps at a
//     time (one load per (step, replica) instead of one per input), double
//     buffered: a chunk's words are loaded into registers before the
//     previous chunk is computed and stored to shared memory after it, so
//     one barrier per chunk and no exposed load latency; xbar written
//     replica-minor
constexpr int kXbSteps = 32;
__global__ void __launch_bounds__(1024) k_clf_xbar(const sw_clf_inputs_t P) {
  __shared__ uint32_t s_w[2][kXbSteps][33];
  const int NI = P.num_inputs;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = blockIdx.x;
  const int b = blockIdx.y * 32 + lane;
  const int x = w * 32 + warp;
  const bool bok = b < P.batch;
  const int64_t plane = (int64_t)NI * P.ldb;
  const int64_t tstride = (int64_t)P.batch * P.words;
  const uint32_t* wp = P.in_bits + (int64_t)(bok ? b : 0) * P.words + w;
  float* out = P.xbar_t + (int64_t)x * P.ldb + b;
  float xb = 0.0f;
  // chunk 0's words
  if (warp < min(kXbSteps, P.steps)) s_w[0][warp][lane] = bok ? __ldg(wp + (int64_t)warp * tstride) : 0u;
  __syncthreads();
  for (int t0 = 0, cb = 0; t0 < P.steps; t0 += kXbSteps, cb ^= 1) {
    const int nt = min(kXbSteps, P.steps - t0);
    // the next chunk's word of this thread, in flight during this chunk
    const int tn = t0 + kXbSteps + warp;
    const uint32_t nxt = (tn < P.steps && bok) ? __ldg(wp + (int64_t)tn * tstride) : 0u;
    if (x < NI) {
      for (int tt = 0; tt < nt; ++tt) {
        const bool sp = (s_w[cb][tt][lane] >> warp) & 1u;
        xb = __fadd_rn(__fmul_rn(xb, P.alpha), sp ? 1.0f : 0.0f);
        out[(int64_t)(t0 + tt) * plane] = bok ? xb : 0.0f;
      }
    }
    if (t0 + kXbSteps < P.steps && warp < kXbSteps) s_w[cb ^ 1][warp][lane] = nxt;
    __syncthreads();
  }
}

// ------------------------------------------------------------ forward ----
// row groups of the current sums: 8 / (hidden units per thread)
__host__ __device__ inline int fwd2_groups(int H) { return H <= 256 ? 8 : 4; }

// per-group row-list capacity: a group holds at most ceil(n / G) rows
__host__ __device__ inline int fwd2_list_cap(int H, int NI) {
  const int G = fwd2_groups(H);
  return (NI + G - 1) / G + (H + G - 1) / G + 2;
}

__host__ __device__ inline size_t fwd2_fixed_bytes(int H, int NI, int n_steps) {
  const size_t NT = (size_t)NI + H;
  size_t o = (size_t)2 * fwd2_groups(H) * H * 4;   // input / hidden partial rows
  o += NT * 2;                                      // rlen (16-bit)
  o += (size_t)fwd2_groups(H) * fwd2_list_cap(H, NI) * 2;   // per-group row lists (16-bit ids)
  o = (o + 3) & ~(size_t)3;
  o += (size_t)((H + 31) / 32) * 4;                 // hidden spike words
  o = (o + 15) & ~(size_t)15;
  o += (size_t)n_steps * ((NI + 31) / 32) * 4;      // the launch's input spike words
  return o;
}

// rows [n*grp/G, n*(grp+1)/G) of the ascending set-bit list of words[0..nw)
// (n = the total set bits) into out[0..), one warp; returns their count.
// Up to 32 words: one load, one scan; more: a counting pass first.
__device__ __forceinline__ int group_rows(const uint32_t* words, int nw, int grp, int G, uint16_t* out, int lane) {
  if (nw <= 32) {
    const uint32_t wd = lane < nw ? words[lane] : 0u;
    const int c = __popc(wd);
    int inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(SW_FULL_MASK, inc, d);
      if (lane >= d) inc += u;
    }
    const int n = __shfl_sync(SW_FULL_MASK, inc, 31);
    const int g0 = n * grp / G, g1 = n * (grp + 1) / G;
    int rank = inc - c;
    if (rank < g1 && rank + c > g0) {
      uint32_t m = wd;
      for (; rank < g0; ++rank) m &= m - 1;   // set bits below the group
      for (; m && rank < g1; m &= m - 1, ++rank) out[rank - g0] = lane * 32 + __ffs(m) - 1;
    }
    __syncwarp();
    return g1 - g0;
  }
  int n = 0;
  for (int w0 = 0; w0 < nw; w0 += 32) {
    const uint32_t wd = w0 + lane < nw ? words[w0 + lane] : 0u;
    n += __reduce_add_sync(SW_FULL_MASK, __popc(wd));
  }
  const int g0 = n * grp / G, g1 = n * (grp + 1) / G;
  int base = 0;
  for (int w0 = 0; w0 < nw && base < g1; w0 += 32) {
    const uint32_t wd = w0 + lane < nw ? words[w0 + lane] : 0u;
    const int c = __popc(wd);
    int inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(SW_FULL_MASK, inc, d);
      if (lane >= d) inc += u;
    }
    int rank = base + inc - c;
    if (rank < g1 && rank + c > g0)
      for (uint32_t m = wd; m; m &= m - 1, ++rank)
        if (rank >= g0 && rank < g1) out[rank - g0] = (w0 + lane) * 32 + __ffs(m) - 1;
    base += __shfl_sync(SW_FULL_MASK, inc, 31);
  }
  __syncwarp();
  return g1 - g0;
}

// both selections at once when the input and the hidden words fit one warp
// (lanes [0, nwi) input words, [nwi, nwi + nwh) hidden words): one scan
__device__ __forceinline__ void group_rows2(const uint32_t* wi, int nwi, const uint32_t* wh, int nwh, int grp,
                                            int G, uint16_t* out_in, int& nin, uint16_t*& out_h, int& nh, int lane) {
  const bool is_in = lane < nwi;
  const uint32_t wd = is_in ? wi[lane] : (lane < nwi + nwh ? wh[lane - nwi] : 0u);
  const int c = __popc(wd);
  int inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(SW_FULL_MASK, inc, d);
    if (lane >= d) inc += u;
  }
  const int n_in = __shfl_sync(SW_FULL_MASK, inc, nwi - 1);
  const int n_h = __shfl_sync(SW_FULL_MASK, inc, 31) - n_in;
  const int a0 = n_in * grp / G, a1 = n_in * (grp + 1) / G;
  const int h0 = n_h * grp / G, h1 = n_h * (grp + 1) / G;
  out_h = out_in + (a1 - a0);
  // this lane's word: ranks within its own list, its group's range
  const int r0 = is_in ? a0 : h0, r1 = is_in ? a1 : h1;
  int rank = inc - c - (is_in ? 0 : n_in);
  uint16_t* out = is_in ? out_in - a0 : out_h - h0;
  const int wbase = (is_in ? lane : lane - nwi) * 32;
  if (rank < r1 && rank + c > r0) {
    uint32_t m = wd;
    for (; rank < r0; ++rank) m &= m - 1;   // set bits below the group
    for (; m && rank < r1; m &= m - 1, ++rank) out[rank] = wbase + __ffs(m) - 1;
  }
  __syncwarp();
  nin = a1 - a0;
  nh = h1 - h0;
}

// dst[target] += weight over the packed rows list[0..nr) in order, one
// warp: lanes 0..kRowsAhead-1 look up a row each (index, length, offset),
// the rows' entries are loaded before any is added (lane = entry), so their
// L2 latencies overlap.  Warp-uniform branches skip the empty row slots of a
// batch and, unless a row of the batch is longer than 32, the long-row code.
constexpr int kRowsAhead = 4;
template <typename IDX>
__device__ __forceinline__ void sum_rows(const IDX* list, int nr, const uint16_t* rl, const int2* base, int stride,
                                         float* dst, int lane) {
  for (int r = 0; r < nr; r += kRowsAhead) {
    const int cnt = min(kRowsAhead, nr - r);
    int my_len = 0, my_off = 0;
    if (lane < cnt) {
      const int x = list[r + lane];
      my_len = rl[x];
      my_off = x * stride;
    }
    const bool longrows = __reduce_max_sync(SW_FULL_MASK, my_len) > 32;
    int2 tw[kRowsAhead];
    int len[kRowsAhead];
#pragma unroll
    for (int u = 0; u < kRowsAhead; ++u) {
      len[u] = __shfl_sync(SW_FULL_MASK, my_len, u);
      const int off = __shfl_sync(SW_FULL_MASK, my_off, u);
      tw[u] = make_int2(0, 0);
      if (lane < len[u]) tw[u] = __ldg(base + off + lane);
    }
    if (!longrows) {
#pragma unroll
      for (int u = 0; u < kRowsAhead; ++u) {
        if (u < cnt) {
          if (lane < len[u]) dst[tw[u].x] = __fadd_rn(dst[tw[u].x], __int_as_float(tw[u].y));
          __syncwarp();
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < kRowsAhead; ++u) {
        if (u < cnt) {
          if (lane < len[u]) dst[tw[u].x] = __fadd_rn(dst[tw[u].x], __int_as_float(tw[u].y));
          const int off = __shfl_sync(SW_FULL_MASK, my_off, u);
          for (int q = lane + 32; q < len[u]; q += 32) {
            const int2 t2 = __ldg(base + off + q);
            dst[t2.x] = __fadd_rn(dst[t2.x], __int_as_float(t2.y));
          }
          __syncwarp();
        }
      }
    }
  }
}

// NTH threads per replica block, HPT hidden units per thread; GT row groups
// (== fwd2_groups(H)), warp w sums group w
template <int NTH, int HPT, int GT>
__global__ void __launch_bounds__(NTH, 1024 / NTH) k_clf_fwd2(sw_clf_step_t P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  sw::pdl_enter();
  constexpr int kT2 = NTH;
  constexpr int G = GT;
  const int H = P.hidden, NI = P.num_inputs;
  const int NT = NI + H;
  const int HW = (H + 31) / 32;
  const int cap = fwd2_list_cap(H, NI);
  size_t o = 0;
  float* pin = (float*)(smem_raw + o);   o += (size_t)G * H * 4;
  float* prc = (float*)(smem_raw + o);   o += (size_t)G * H * 4;
  // 16-bit row lengths and ids: a smaller block leaves more L1 to the e-prop
  // pass running next to it
  uint16_t* rlen = (uint16_t*)(smem_raw + o);   o += (size_t)NT * 2;
  uint16_t* lists = (uint16_t*)(smem_raw + o);  o += (size_t)G * cap * 2;   // [G][cap] this step's rows
  o = (o + 3) & ~(size_t)3;
  uint32_t* zws = (uint32_t*)(smem_raw + o); o += (size_t)HW * 4;       // hidden spike words
  o = (o + 15) & ~(size_t)15;
  uint32_t* wsm = (uint32_t*)(smem_raw + o);   // [n_steps][in_words] spike words

  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bH = b * H;
  const int B = P.batch;
  const int nslot = P.slot_count;
  const int nsteps = P.n_steps;

  for (int x = tid; x < NT; x += kT2)
    rlen[x] = (uint16_t)((x < NI) ? __ldg(P.in_row_length + x) : __ldg(P.rec_row_length + (x - NI)));
  for (int x = tid; x < G * H; x += kT2) { pin[x] = 0.0f; prc[x] = 0.0f; }
  const int prev = ((P.t - 1) % nslot + nslot) % nslot;
  const float* zin0 = P.zbar + prev * B * H;
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
  const float alpha = P.alpha, rho = P.rho, beta = P.beta, v_thr = P.v_thr;
  // the launch's input spike words (all its steps) into shared memory
  for (int x = tid; x < nsteps * P.in_words; x += kT2) {
    const int q = x / P.in_words, w = x - q * P.in_words;
    wsm[x] = __ldg(P.in_bits + ((int64_t)(P.t + q) * B + b) * P.in_words + w);
  }

  int cur = P.t % nslot;
  uint32_t* zw_step = P.z_bits + (int64_t)b * HW;   // this replica's spike words of step s
  for (int s = 0; s < nsteps; ++s, cur = (cur + 1 == nslot) ? 0 : cur + 1) {
    float* zbar_o = P.zbar + cur * B * H;
    float* psi_o = P.psi + cur * B * H;

    FWD2_PROF(0);
    // ---- A: hidden spike words (unit order) to shared memory and to z_bits
    // for the readout launch: thread t holds units HPT*t + j, i.e. bits
    // HPT*(t % (32/HPT)) + j of word t / (32/HPT); the 32/HPT threads of a
    // word OR their bit groups together (butterfly) ----
    {
      uint32_t* zw = zw_step;
      zw_step += (int64_t)B * HW;
      if (HPT == 1) {
        const unsigned hm = __ballot_sync(SW_FULL_MASK, h0 < H && z[0] != 0.0f);
        if (lane == 0 && warp < HW) {
          zws[warp] = hm;
          zw[warp] = hm;
        }
      } else {
        constexpr int TPW = 32 / HPT;   // threads per word
        uint32_t wd = 0;
#pragma unroll
        for (int j = 0; j < HPT; ++j) wd |= (h0 + j < H && z[j] != 0.0f) ? 1u << j : 0u;
        wd <<= HPT * (lane % TPW);
#pragma unroll
        for (int o = 1; o < TPW; o <<= 1) wd |= __shfl_xor_sync(SW_FULL_MASK, wd, o);
        const int q = tid / TPW;
        if (lane % TPW == 0 && q < HW) {
          zws[q] = wd;
          zw[q] = wd;
        }
      }
    }
    // zbar (old z) for the e-prop traces and the readout gradient
#pragma unroll
    for (int j = 0; j < HPT; ++j) {
      const int h = h0 + j;
      if (h < H) {
        zb[j] = __fadd_rn(__fmul_rn(zb[j], alpha), z[j]);
        zbar_o[bH + h] = zb[j];
      }
    }
    __syncthreads();   // B1: hidden spike words (and, at s = 0, the setup) visible
    FWD2_PROF(1);

    // ---- C: warp g selects its group of the ascending input rows and of the
    // ascending hidden rows straight from the spike words, then sums them ----
    if constexpr (2 * G <= NTH / 32) {
      // spare warps (H > 256: G = 4): the input groups on warps 0..G-1, the
      // hidden groups on warps G..2G-1 (separate partial rows, so the same sums)
      if (warp < G) {
        uint16_t* L = lists + warp * cap;
        const int nin = group_rows(wsm + s * P.in_words, P.in_words, warp, G, L, lane);
        sum_rows(L, nin, rlen, reinterpret_cast<const int2*>(P.in_tw), P.in_tw_stride, pin + warp * H, lane);
      } else if (warp < 2 * G) {
        const int g = warp - G;
        uint16_t* Lh = lists + g * cap + (NI + G - 1) / G + 1;
        const int nhd = group_rows(zws, HW, g, G, Lh, lane);
        sum_rows(Lh, nhd, rlen + NI, reinterpret_cast<const int2*>(P.rec_tw), P.rec_tw_stride, prc + g * H,
                 lane);
      }
    } else if (warp < G) {
      uint16_t* L = lists + warp * cap;
      int nin, nhd;
      uint16_t* Lh;
      if (P.in_words + HW <= 32) {
        group_rows2(wsm + s * P.in_words, P.in_words, zws, HW, warp, G, L, nin, Lh, nhd, lane);
      } else {
        nin = group_rows(wsm + s * P.in_words, P.in_words, warp, G, L, lane);
        Lh = L + nin;
        nhd = group_rows(zws, HW, warp, G, Lh, lane);
      }
      FWD2_PROF(4);
      sum_rows(L, nin, rlen, reinterpret_cast<const int2*>(P.in_tw), P.in_tw_stride, pin + warp * H, lane);
      sum_rows(Lh, nhd, rlen + NI, reinterpret_cast<const int2*>(P.rec_tw), P.rec_tw_stride, prc + warp * H,
               lane);
    }
    FWD2_PROF(5);
    __syncthreads();   // B3: partial rows complete
    FWD2_PROF(6);

    // ---- D: group partials in order, ALIF step, surrogate ----
    float aes[HPT], ars[HPT];
    if (HPT > 1 && (H % HPT) == 0) {
      // the thread's HPT consecutive units: one vector load / store per row
      using VecT = typename std::conditional<HPT == 4, float4, float2>::type;
      if (h0 < H) {
        VecT e = *reinterpret_cast<const VecT*>(pin + h0), r = *reinterpret_cast<const VecT*>(prc + h0);
        const VecT zero{};
        *reinterpret_cast<VecT*>(pin + h0) = zero;
        *reinterpret_cast<VecT*>(prc + h0) = zero;
        float* ef = reinterpret_cast<float*>(&e);
        float* rf = reinterpret_cast<float*>(&r);
        for (int g = 1; g < G; ++g) {
          VecT pe = *reinterpret_cast<const VecT*>(pin + g * H + h0);
          VecT pr = *reinterpret_cast<const VecT*>(prc + g * H + h0);
          *reinterpret_cast<VecT*>(pin + g * H + h0) = zero;
          *reinterpret_cast<VecT*>(prc + g * H + h0) = zero;
          const float* pef = reinterpret_cast<const float*>(&pe);
          const float* prf = reinterpret_cast<const float*>(&pr);
#pragma unroll
          for (int j = 0; j < HPT; ++j) {
            ef[j] = __fadd_rn(ef[j], pef[j]);
            rf[j] = __fadd_rn(rf[j], prf[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < HPT; ++j) {
          aes[j] = ef[j];
          ars[j] = rf[j];
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < HPT; ++j) {
        const int h = h0 + j;
        if (h >= H) continue;
        float ae = pin[h], ar = prc[h];
        pin[h] = 0.0f;
        prc[h] = 0.0f;
        for (int g = 1; g < G; ++g) {
          ae = __fadd_rn(ae, pin[g * H + h]);
          ar = __fadd_rn(ar, prc[g * H + h]);
          pin[g * H + h] = 0.0f;
          prc[g * H + h] = 0.0f;
        }
        aes[j] = ae;
        ars[j] = ar;
      }
    }
#pragma unroll
    for (int j = 0; j < HPT; ++j) {
      const int h = h0 + j;
      if (h >= H) continue;
      const float ae = aes[j], ar = ars[j];
      const float thr_o = __fadd_rn(v_thr, __fmul_rn(beta, a[j]));
      const float cc = __fdiv_rn(__fsub_rn(v[j], thr_o), v_thr);
      const float r = __fsub_rn(1.0f, fabsf(cc));
      psi_o[bH + h] = __fmul_rn(0.5f, (r > 0.0f || r != r) ? r : 0.0f);
      float vv = __fmul_rn(alpha, __fsub_rn(v[j], __fmul_rn(z[j], v_thr)));
      vv = __fadd_rn(__fadd_rn(vv, ar), ae);
      const float aa = __fadd_rn(__fmul_rn(rho, a[j]), z[j]);
      v[j] = vv;
      a[j] = aa;
      z[j] = (vv >= __fadd_rn(v_thr, __fmul_rn(beta, aa))) ? 1.0f : 0.0f;
    }
    FWD2_PROF(7);
    // the next step's word writes (A) race with nothing: every warp finished
    // this step's C before B3
  }

#pragma unroll
  for (int j = 0; j < HPT; ++j) {
    const int h = h0 + j;
    if (h < H) {
      P.v[bH + h] = v[j];
      P.a[bH + h] = a[j];
      P.z[bH + h] = z[j];
    }
  }
}

// ------------------------------------------------------------ readout ----
// The readout of a grouped launch's steps (classifier.py:215-219,
// plasticity.py:156-165), block per replica, from the hidden spike words the
// forward launch wrote:
//   1  per step (warp per step), the hidden spike words and the ascending
//      list of spiking units, the list capped at kRoList entries;
//   2  thread per (step, class): s = sum of w_out[c][h] over the step's
//      spiking units in ascending order -- from the list, or for steps with
//      more spikes straight from the words -- (f64, from +0.0, 8 loads in
//      flight); the steps are independent here, so their load latencies
//      overlap; the block's shared memory stays small (no H-sized lists), so
//      more replica blocks per SM and W_out's rows stay in L1;
//   3  warp 0: y = alpha*y + s + b per class, steps in order;
//   4  warp per step: softmax, d = pi - onehot (written to the step's slot);
//   5  warp 0: pi_sum and the loss accumulated in step order.
constexpr int kRoList = 64;
__host__ __device__ inline size_t readout_smem(int n_steps, int H, int C) {
  return (size_t)n_steps * ((H + 31) / 32) * 4 + (size_t)n_steps * (4 + kRoList * 2) + (size_t)n_steps * C * 8 * 3 +
         (size_t)C * 8;
}

__global__ void __launch_bounds__(256) k_clf_readout(const sw_clf_step_t P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  sw::pdl_enter();
  const int H = P.hidden, C = P.num_classes, B = P.batch, n = P.n_steps;
  const int HW = (H + 31) / 32;
  double* s_sum = reinterpret_cast<double*>(smem_raw);      // [n][C]
  double* s_y = s_sum + (size_t)n * C;                      // [n][C]
  double* s_pi = s_y + (size_t)n * C;                       // [n][C]
  double* s_bo = s_pi + (size_t)n * C;                      // [C]
  uint32_t* s_zw = reinterpret_cast<uint32_t*>(s_bo + C);  // [n][HW]
  int* s_cnt = reinterpret_cast<int*>(s_zw + (size_t)n * HW);   // [n]
  uint16_t* s_list = reinterpret_cast<uint16_t*>(s_cnt + n);      // [n][kRoList]
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kW = 8;
  const int bC = b * C;
  const int label = P.labels[b];   // loaded early: read after the sums
  for (int c = tid; c < C; c += blockDim.x) s_bo[c] = P.b_out[c];
  // 1
  for (int t = warp; t < n; t += kW) {
    const uint32_t* zw = P.z_bits + ((int64_t)t * B + b) * HW;
    uint16_t* L = s_list + (size_t)t * kRoList;
    int cnt = 0;
    for (int w0 = 0; w0 < HW; w0 += 32) {
      const uint32_t wd = w0 + lane < HW ? zw[w0 + lane] : 0u;
      if (w0 + lane < HW) s_zw[(size_t)t * HW + w0 + lane] = wd;
      const int c = __popc(wd);
      int inc = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(SW_FULL_MASK, inc, d);
        if (lane >= d) inc += u;
      }
      int p = cnt + inc - c;
      for (uint32_t m = wd; m && p < kRoList; m &= m - 1) L[p++] = (uint16_t)((w0 + lane) * 32 + __ffs(m) - 1);
      cnt += __shfl_sync(SW_FULL_MASK, inc, 31);
    }
    if (lane == 0) s_cnt[t] = cnt;
  }
  __syncthreads();
  // 2
  for (int i = tid; i < n * C; i += blockDim.x) {
    const int t = i / C, c = i - t * C;
    const double* wr = P.w_out + (int64_t)c * H;
    double sacc = 0.0;
    const int cnt = s_cnt[t];
    if (cnt <= kRoList) {
      const uint16_t* L = s_list + (size_t)t * kRoList;
      for (int q0 = 0; q0 < cnt; q0 += 8) {
        double wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) wv[u] = q0 + u < cnt ? __ldg(wr + L[q0 + u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q0 + u < cnt) sacc = __dadd_rn(sacc, wv[u]);
      }
      s_sum[i] = sacc;
      continue;
    }
    const uint32_t* zw = s_zw + (size_t)t * HW;
    int w = 0;
    uint32_t m = zw[0];
    for (;;) {
      // the next 8 spiking units (ascending; -1 past the last)
      int idx[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        while (m == 0u && w + 1 < HW) m = zw[++w];
        idx[u] = m ? w * 32 + __ffs(m) - 1 : -1;
        m &= m - 1;
      }
      double wv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) wv[u] = idx[u] >= 0 ? __ldg(wr + idx[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (idx[u] >= 0) sacc = __dadd_rn(sacc, wv[u]);
      if (idx[7] < 0) break;
    }
    s_sum[i] = sacc;
  }
  __syncthreads();
  // 3
  if (warp == 0) {
    for (int c = lane; c < C; c += 32) {
      double y = P.y[bC + c];
      for (int t = 0; t < n; ++t) {
        y = __dadd_rn(__dadd_rn(__dmul_rn(P.alpha64, y), s_sum[t * C + c]), s_bo[c]);
        s_y[t * C + c] = y;
      }
      P.y[bC + c] = y;
    }
  }
  __syncthreads();
  // 4
  const int nslot = P.slot_count;
  for (int t = warp; t < n; t += kW) {
    const double* yv = s_y + (size_t)t * C;
    double* d_out = P.d + (size_t)((P.t + t) % nslot) * B * C;
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
      s_pi[t * C + c] = pi;
      d_out[bC + c] = pi - (c == label ? 1.0 : 0.0);
    }
  }
  __syncthreads();
  // 5
  if (warp == 0) {
    for (int c = lane; c < C; c += 32) {
      double ps = P.pi_sum[bC + c];
      for (int t = 0; t < n; ++t) ps = ps + s_pi[t * C + c];
      P.pi_sum[bC + c] = ps;
    }
  } else if (warp == 1) {
    // the loss terms -log(pi[t][label]) of the steps in parallel (lane =
    // step), then added in step order by lane 0
    double ls = P.loss[b];
    for (int t0 = 0; t0 < n; t0 += 32) {
      const double term = t0 + lane < n ? -log(s_pi[(t0 + lane) * C + label]) : 0.0;
      for (int u = 0; u < 32 && t0 + u < n; ++u) ls = ls + __shfl_sync(SW_FULL_MASK, term, u);
    }
    if (lane == 0) P.loss[b] = ls;
  }
}

// SW_CLF_PDL=1: the trial's per-group kernels with programmatic dependent launch
inline bool clf_pdl() {
  static const bool on = [] { const char* e = getenv("SW_CLF_PDL"); return e && e[0] == '1'; }();
  return on;
}

template <int NTH, int HPT, int GT>
int launch_fwd2(const sw_clf_step_t* p, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute((const void*)k_clf_fwd2<NTH, HPT, GT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  sw::pdl_launch(clf_pdl(), k_clf_fwd2<NTH, HPT, GT>, dim3(p->batch), dim3(NTH), smem, st, *p);
  sw::count_launch();
  const size_t rsm = readout_smem(p->n_steps, p->hidden, p->num_classes);
  static size_t rsm_attr = 48 * 1024;
  if (rsm > rsm_attr) {
    cudaFuncSetAttribute(k_clf_readout, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
    rsm_attr = rsm;
  }
  sw::pdl_launch(clf_pdl(), k_clf_readout, dim3(p->batch), dim3(256), rsm, st, *p);
  sw::count_launch();
  return SW_OK;
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int sw_debug_fwd2_prof(int enable, long long* out16) {
  if (out16 && cudaMemcpyFromSymbol(out16, g_fwd2_prof, 64 * sizeof(long long)) != cudaSuccess) return SW_ERR_CUDA;
  return cudaMemcpyToSymbol(g_fwd2_prof_on, &enable, sizeof(int)) == cudaSuccess ? 0 : SW_ERR_CUDA;
}

extern "C" int sw_clf_inputs(const sw_clf_inputs_t* p, void* stream) {
  if (!p || p->batch < 1 || p->ldb < p->batch || p->num_inputs < 1 || p->steps < 0 ||
      p->words != (p->num_inputs + 31) / 32) {
    sw::set_last_error("sw_clf_inputs: bad shapes (ldb >= batch, words = ceil(num_inputs / 32))");
    return SW_ERR_INVALID_ARG;
  }
  if (p->steps == 0) return SW_OK;
  const size_t thr_bytes = (size_t)p->words * 32 * 8;
  if (thr_bytes > 200 * 1024) {
    sw::set_last_error("sw_clf_inputs: num_inputs > 25600 (spike thresholds are staged in shared memory)");
    return SW_ERR_INVALID_ARG;
  }
  if (thr_bytes > 48 * 1024)
    cudaFuncSetAttribute(k_clf_spikes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)thr_bytes);
  dim3 grid1(p->batch, (p->steps + kSpkSteps - 1) / kSpkSteps);
  k_clf_spikes<<<grid1, 256, thr_bytes, (cudaStream_t)stream>>>(*p);
  sw::count_launch();
  dim3 grid2(p->words, (p->ldb + 31) / 32);
  k_clf_xbar<<<grid2, 1024, 0, (cudaStream_t)stream>>>(*p);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_clf_inputs");
  return SW_OK;
}

// the grouped forward with precomputed inputs (sw_clf_step with in_bits);
// SW_ERR_INVALID_ARG when the shapes are outside its layout
int clf_fwd2_launch(const sw_clf_step_t* p, void* stream) {
  const int H = p->hidden, NI = p->num_inputs, C = p->num_classes;
  if (p->n_steps < 1 || p->n_steps > 2 * SW_EPROP_MAX_BLOCK || !p->in_bits || !p->z_bits || !p->in_tw || !p->rec_tw || H < 1 || H > 1024 || NI < 1 || C < 1 ||
      NI + H > 65535 || p->in_tw_stride > 65535 || p->rec_tw_stride > 65535 ||   // 16-bit ids and lengths
      readout_smem(p->n_steps, H, C) > 200 * 1024 ||
      p->in_words != (NI + 31) / 32)
    return SW_ERR_INVALID_ARG;
  // 4 replica blocks per SM (512 replicas in one wave): <= 56 KB each
  const size_t smem = fwd2_fixed_bytes(H, NI, p->n_steps);
  if (smem > 56 * 1024) return SW_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (H <= 256) return launch_fwd2<256, 1, 8>(p, smem, st);
  if (H <= 512) return launch_fwd2<256, 2, 4>(p, smem, st);
  return launch_fwd2<256, 4, 4>(p, smem, st);
}
