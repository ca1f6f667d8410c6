// Temporally blocked e-prop update (sparsewire/_kernels.py:15-39 semantics,
// k consecutive timesteps per pass over the eligibility state).
//
// The eligibility recursion of step t+1 needs only eps/ebar after step t and
// step t+1's own inputs (pre trace, psi, lsig), and the forward pass never
// reads eps, ebar or the gradient.  So the trainer runs k forward steps first
// and this kernel then streams every (tile, replica-chunk) of eps/ebar through
// shared memory once for all k steps.  That is 1/k of the HBM traffic of k
// single-step passes.  The pipeline is the one of eprop_fused.cu:
//   warp 0      TMA loader (eps/ebar bulk copies, 3-stage mbarrier ring);
//   warps 2..5  k recursion steps per element, in shared memory; float32
//               gradient terms per step;
//   warp 1      bulk store, and k float64 chains per synapse.  Chain 0
//               continues from the gradient, chains 1..k-1 start at zero, and
//               each chain adds its step's terms in ascending replica order.
//               At the tile's last chunk: grad = ((c0 + c1) + c2) + c3.
// eps and ebar are bit-identical to k single-step passes.  The gradient
// equals the sequential sum for k = 1; for k > 1 it differs only in the
// float64 rounding of that final combination of partial chains.
// Readout gradients (classifier.py:221-222) for the k steps are reduced by
// extra blocks of the same launch.
#include "common.cuh"
#include "sm100_async.cuh"

namespace {

constexpr int kMaxK = 4;
constexpr int kCB = 32;        // replicas per stage
constexpr int kStages = 3;
constexpr int kCompute = 4;
constexpr int kWarps = kCompute + 2;
constexpr int kThreads = kWarps * 32;
constexpr int kBPW = kCB / kCompute;
constexpr int kRowBytes = 32 * 4;

struct SegB {
  const int32_t* pre;
  const int32_t* post;
  const float* trace[kMaxK];   // [B, P] per step
  float* eps;                  // [tiles, B, 32]
  float* ebar;
  double* grad;                // [tiles*32]
  int P;
  int tiles;
};

struct StepsB {
  const float* psi[kMaxK];     // [B, H] per step
  const float* lsig[kMaxK];
  const double* d[kMaxK];      // [B, C] per step (readout)
  const float* zbar[kMaxK];    // [B, H] per step (readout)
  int k;
};

template <int K>
struct Stage {
  float eps[kCB][32];
  float ebar[kCB][32];
  float terms[K][kCB][32];
};

template <int K>
struct Smem {
  Stage<K> st[kStages];
  uint64_t full[kStages];
  uint64_t ready[kStages];
  uint64_t freed[kStages];
  int tile[kStages];
  int ch[kStages];
};

__device__ void readout_block_k(int r, int B, int H, const StepsB& sp, double* g_w_out, double* g_b_out,
                                int C) {
  __shared__ double part[kWarps][33];
  __shared__ double partb[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int htiles = (H + 31) / 32;
  const int c = r / htiles, h = (r % htiles) * 32 + lane;
  double acc = 0.0, accb = 0.0;
  const int per = (B + kWarps - 1) / kWarps;
  const int b0 = warp * per, b1 = min(B, b0 + per);
  for (int k = 0; k < sp.k; ++k) {
    const double* d = sp.d[k];
    const float* zb = sp.zbar[k];
    for (int b = b0; b < b1; b += 8) {
      double dv[8];
      float zv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int bb = b + u;
        dv[u] = bb < b1 ? d[(int64_t)bb * C + c] : 0.0;
        zv[u] = (bb < b1 && h < H) ? zb[(int64_t)bb * H + h] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc = __dadd_rn(acc, __dmul_rn(dv[u], (double)zv[u]));
        accb = __dadd_rn(accb, dv[u]);
      }
    }
  }
  part[warp][lane] = acc;
  if (lane == 0) partb[warp] = accb;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t = __dadd_rn(t, part[w][lane]);
    if (h < H) g_w_out[(int64_t)c * H + h] += t;
    if (lane == 0 && (r % htiles) == 0) {
      double tb = 0.0;
      for (int w = 0; w < kWarps; ++w) tb = __dadd_rn(tb, partb[w]);
      g_b_out[c] += tb;
    }
  }
}

__device__ __forceinline__ const SegB& seg_of(const SegB& s0, const SegB& s1, int tile, int& lt) {
  if (tile < s0.tiles) { lt = tile; return s0; }
  lt = tile - s0.tiles;
  return s1;
}

template <int K>
__global__ void __launch_bounds__(kThreads, 3)
k_eprop_block(SegB s0, SegB s1, StepsB sp, int B, int H, float beta, float rho, float alpha,
              double* g_w_out, double* g_b_out, int C, int ro_blocks, unsigned* tickets) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem<K>& S = *reinterpret_cast<Smem<K>*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if ((int)blockIdx.x < ro_blocks) {
    readout_block_k(blockIdx.x, B, H, sp, g_w_out, g_b_out, C);
  } else {
    const int tiles = s0.tiles + s1.tiles;
    const int nch = (B + kCB - 1) / kCB;
    if (threadIdx.x == 0) {
      for (int s = 0; s < kStages; ++s) {
        sw::mbar_init(&S.full[s], 1);
        sw::mbar_init(&S.ready[s], kCompute);
        sw::mbar_init(&S.freed[s], 1);
      }
      sw::fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
      // ---------------- loader ----------------
      if (lane == 0) {
        const uint64_t pol = sw::policy_evict_first();
        uint32_t k = 0;
        while (true) {
          const int tile = (int)atomicAdd(&tickets[0], 1u);
          if (tile >= tiles) {
            const int slot = k % kStages;
            if (k >= kStages) sw::mbar_wait(&S.freed[slot], ((k / kStages) - 1) & 1);
            S.tile[slot] = -1;
            sw::mbar_arrive(&S.full[slot]);
            break;
          }
          int lt;
          const SegB& sg = seg_of(s0, s1, tile, lt);
          for (int ch = 0; ch < nch; ++ch, ++k) {
            const int slot = k % kStages;
            if (k >= kStages) sw::mbar_wait(&S.freed[slot], ((k / kStages) - 1) & 1);
            S.tile[slot] = tile;
            S.ch[slot] = ch;
            const int nb = min(kCB, B - ch * kCB);
            const uint32_t bytes = (uint32_t)nb * kRowBytes;
            const int64_t off = ((int64_t)lt * B + (int64_t)ch * kCB) * 32;
            sw::mbar_arrive_expect_tx(&S.full[slot], 2 * bytes);
            sw::bulk_g2s_hint(&S.st[slot].eps[0][0], sg.eps + off, bytes, &S.full[slot], pol);
            sw::bulk_g2s_hint(&S.st[slot].ebar[0][0], sg.ebar + off, bytes, &S.full[slot], pol);
          }
        }
      }
    } else if (warp == 1) {
      // ---------------- k ordered float64 chains + bulk store ----------------
      double acc[K];
      const uint64_t pol = sw::policy_evict_first();
      for (uint32_t kk = 0;; ++kk) {
        const int slot = kk % kStages;
        const uint32_t par = (kk / kStages) & 1;
        sw::mbar_wait(&S.full[slot], par);
        const int tile = S.tile[slot];
        if (tile < 0) break;
        const int ch = S.ch[slot];
        sw::mbar_wait(&S.ready[slot], par);
        int lt;
        const SegB& sg = seg_of(s0, s1, tile, lt);
        const int nb = min(kCB, B - ch * kCB);
        if (lane == 0) {
          const int64_t off = ((int64_t)lt * B + (int64_t)ch * kCB) * 32;
          sw::bulk_s2g_hint(sg.eps + off, &S.st[slot].eps[0][0], (uint32_t)nb * kRowBytes, pol);
          sw::bulk_s2g_hint(sg.ebar + off, &S.st[slot].ebar[0][0], (uint32_t)nb * kRowBytes, pol);
          sw::bulk_commit();
        }
        const int e = lt * 32 + lane;
        if (ch == 0) {
          acc[0] = sg.grad[e];
#pragma unroll
          for (int q = 1; q < K; ++q) acc[q] = 0.0;
        }
        const Stage<K>& st = S.st[slot];
        for (int r = 0; r < nb; ++r) {
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (q < sp.k) acc[q] = __dadd_rn(acc[q], (double)st.terms[q][r][lane]);
        }
        if (ch == nch - 1) {
          double g = acc[0];
#pragma unroll
          for (int q = 1; q < K; ++q)
            if (q < sp.k) g = __dadd_rn(g, acc[q]);
          sg.grad[e] = g;
        }
        if (lane == 0) sw::bulk_wait_read0();
        __syncwarp();
        if (lane == 0) sw::mbar_arrive(&S.freed[slot]);
      }
      if (lane == 0) sw::bulk_wait0();
    } else {
      // ---------------- compute: k recursion steps per element ----------------
      const int cw = warp - 2;
      const int bl0 = cw * kBPW;
      int cur_tile = -1, pre = 0, post = 0, P = 0;
      const float* trace[K];
      for (uint32_t kk = 0;; ++kk) {
        const int slot = kk % kStages;
        const uint32_t par = (kk / kStages) & 1;
        sw::mbar_wait(&S.full[slot], par);
        const int tile = S.tile[slot];
        if (tile < 0) break;
        const int ch = S.ch[slot];
        if (tile != cur_tile) {
          int lt;
          const SegB& sg = seg_of(s0, s1, tile, lt);
          pre = __ldg(sg.pre + lt * 32 + lane);
          post = __ldg(sg.post + lt * 32 + lane);
#pragma unroll
          for (int q = 0; q < K; ++q) trace[q] = sg.trace[q];
          P = sg.P;
          cur_tile = tile;
        }
        const int nb = min(kCB, B - ch * kCB);
        Stage<K>& st = S.st[slot];
        for (int u = 0; u < kBPW; ++u) {
          const int bl = bl0 + u;
          if (bl >= nb) break;
          const int64_t b = (int64_t)ch * kCB + bl;
          float zb[K], p[K], l[K];
#pragma unroll
          for (int q = 0; q < K; ++q) {
            if (q < sp.k) {
              zb[q] = __ldg(trace[q] + b * P + pre);
              p[q] = __ldg(sp.psi[q] + b * H + post);
              l[q] = __ldg(sp.lsig[q] + b * H + post);
            }
          }
          float ep = st.eps[bl][lane];
          float eb = st.ebar[bl][lane];
#pragma unroll
          for (int q = 0; q < K; ++q) {
            if (q < sp.k) {
              const float ee = __fmul_rn(p[q], __fsub_rn(zb[q], __fmul_rn(beta, ep)));
              eb = __fadd_rn(__fmul_rn(alpha, eb), ee);
              st.terms[q][bl][lane] = __fmul_rn(l[q], eb);
              ep = __fadd_rn(__fmul_rn(rho, ep), ee);
            }
          }
          st.ebar[bl][lane] = eb;
          st.eps[bl][lane] = ep;
        }
        sw::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) sw::mbar_arrive(&S.ready[slot]);
      }
    }
  }
  // last block out resets the tile ticket (graph replay)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned done = atomicAdd(&tickets[1], 1u);
    if (done == gridDim.x - 1) {
      tickets[0] = 0u;
      tickets[1] = 0u;
      __threadfence();
    }
  }
}

template <int K>
int launch_block(SegB s0, SegB s1, const StepsB& sp, int B, int H, float beta, float rho, float alpha,
                 double* g_w_out, double* g_b_out, int C, int ro_blocks, unsigned* tickets,
                 cudaStream_t st) {
  const int smem = (int)sizeof(Smem<K>);
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute((const void*)k_eprop_block<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eprop_block<K>, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
  }
  const int tiles = s0.tiles + s1.tiles;
  const int workers = tiles ? min(tiles, 148 * per_sm) : 0;
  k_eprop_block<K><<<ro_blocks + workers, kThreads, smem, st>>>(s0, s1, sp, B, H, beta, rho, alpha,
                                                                g_w_out, g_b_out, C, ro_blocks, tickets);
  sw::count_launch();
  return SW_OK;
}

}  // namespace

extern "C" int sw_eprop_fused_block(const sw_eprop_seg_t* segs, int32_t n_segs, const sw_eprop_block_t* blk,
                                    int32_t batch, int32_t hidden, float beta, float rho, float alpha,
                                    double* g_w_out, double* g_b_out, int32_t num_classes,
                                    uint32_t* workspace, void* stream) {
  if (!workspace) { sw::set_last_error("eprop block: workspace (2 zeroed uint32) required"); return SW_ERR_INVALID_ARG; }
  if (n_segs < 1 || n_segs > 2) { sw::set_last_error("eprop block: 1 or 2 segments"); return SW_ERR_INVALID_ARG; }
  if (!blk || blk->k < 1 || blk->k > kMaxK) { sw::set_last_error("eprop block: 1 <= k <= 4 steps"); return SW_ERR_INVALID_ARG; }
  SegB s[2] = {};
  for (int i = 0; i < n_segs; ++i) {
    const sw_eprop_seg_t& q = segs[i];
    if (q.e_pad % 32) { sw::set_last_error("eprop block: e_pad must be a multiple of 32"); return SW_ERR_INVALID_ARG; }
    s[i].pre = q.pre;
    s[i].post = q.post;
    for (int k = 0; k < kMaxK; ++k) s[i].trace[k] = blk->pre_trace[i][k];
    s[i].eps = q.eps;
    s[i].ebar = q.ebar;
    s[i].grad = q.grad;
    s[i].P = q.num_pre;
    s[i].tiles = q.e_pad / 32;
  }
  StepsB sp{};
  sp.k = blk->k;
  for (int k = 0; k < kMaxK; ++k) {
    sp.psi[k] = blk->psi[k];
    sp.lsig[k] = blk->lsig[k];
    sp.d[k] = blk->d[k];
    sp.zbar[k] = blk->zbar[k];
  }
  const bool readout = blk->d[0] && g_w_out && num_classes > 0;
  const int ro_blocks = readout ? num_classes * ((hidden + 31) / 32) : 0;
  if (s[0].tiles + s[1].tiles + ro_blocks == 0 || batch <= 0) return SW_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  switch (blk->k) {
    case 1: rc = launch_block<1>(s[0], s[1], sp, batch, hidden, beta, rho, alpha, g_w_out, g_b_out,
                                 num_classes, ro_blocks, workspace, st); break;
    case 2: rc = launch_block<2>(s[0], s[1], sp, batch, hidden, beta, rho, alpha, g_w_out, g_b_out,
                                 num_classes, ro_blocks, workspace, st); break;
    default: rc = launch_block<4>(s[0], s[1], sp, batch, hidden, beta, rho, alpha, g_w_out, g_b_out,
                                  num_classes, ro_blocks, workspace, st); break;
  }
  if (rc) return rc;
  SW_CHECK_LAUNCH("sw_eprop_fused_block");
  return SW_OK;
}
