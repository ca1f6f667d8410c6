// Fused e-prop hot-path step (sparsewire/_kernels.py:15-39 semantics).
//
// Eligibility state is stored tile-major: eps/ebar[tile][B][32] float32,
// tile = 32 synapses of the per-batch plan order (bucketed by 32-post group,
// then pre, then slot — sw_eprop_plan), so one (tile, replica chunk) is one
// contiguous run that the TMA bulk engine moves with a single copy.
//
// Block = 2 + SW_EPROP_COMPUTE (4) warps, one tile-chunk "stage" at a time through a 4-deep
// shared-memory ring:
//   warp 0      loader:  takes tiles from an atomic ticket, issues
//                        cp.async.bulk global->shared for eps and ebar of
//                        each 32-replica chunk (mbarrier complete_tx) with an
//                        L2 evict-first policy, so the 200 MB/step stream does
//                        not evict the small per-replica state of the forward
//                        kernel;
//   warps 2..5  compute: 8 replicas each per stage — gathers zb/psi/lsig
//                        (L2-resident, 128-byte lines thanks to the plan
//                        order), updates eps/ebar in place in shared memory,
//                        writes the float32 gradient terms;
//   warp 1      ordered sum + store: bulk-stores the updated eps/ebar back to
//                        HBM and folds the terms into the float64 gradient in
//                        ascending replica order (bit-identical to the
//                        reference's b-outer loop), then frees the slot.
// The readout gradients g_w_out += d^T zbar, g_b_out += sum_b d
// (classifier.py:221-222) are reduced by extra blocks of the same launch.
#include "common.cuh"
#include "sm100_async.cuh"

namespace {

struct Seg {
  const int32_t* pre;
  const int32_t* post;
  const float* trace;   // [B, P]
  float* eps;           // [tiles, B, 32]
  float* ebar;
  double* grad;         // [tiles*32]
  int P;
  int tiles;
};

struct ReadoutArgs {
  const double* d;      // [B, C]
  const float* zbar;    // [B, H]
  double* g_w_out;      // [C, H]
  double* g_b_out;      // [C]
  int C;
};

constexpr int kCB = 32;                   // replicas per stage
#ifndef SW_EPROP_STAGES
#define SW_EPROP_STAGES 4
#endif
#ifndef SW_EPROP_MINB
#define SW_EPROP_MINB 4
#endif
#ifndef SW_EPROP_COMPUTE
#define SW_EPROP_COMPUTE 4
#endif
constexpr int kStages = SW_EPROP_STAGES;  // ring depth
constexpr int kCompute = SW_EPROP_COMPUTE; // compute warps
constexpr int kWarps = kCompute + 2;
constexpr int kThreads = kWarps * 32;
constexpr int kBPW = kCB / kCompute;      // replicas per compute warp per stage
constexpr int kRowBytes = 32 * 4;

struct Stage {
  float eps[kCB][32];
  float ebar[kCB][32];
  float terms[kCB][32];
};

struct Smem {
  Stage st[kStages];
  uint64_t full[kStages];
  uint64_t ready[kStages];
  uint64_t freed[kStages];
  int tile[kStages];
  int ch[kStages];
};

__device__ void readout_block(int r, int B, int H, const ReadoutArgs& ro) {
  __shared__ double part[kWarps][33];
  __shared__ double partb[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int htiles = (H + 31) / 32;
  const int c = r / htiles, h = (r % htiles) * 32 + lane;
  double acc = 0.0, accb = 0.0;
  const int per = (B + kWarps - 1) / kWarps;
  const int b0 = warp * per, b1 = min(B, b0 + per);
  for (int b = b0; b < b1; b += 8) {
    double dv[8];
    float zv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int bb = b + u;
      dv[u] = bb < b1 ? ro.d[(int64_t)bb * ro.C + c] : 0.0;
      zv[u] = (bb < b1 && h < H) ? ro.zbar[(int64_t)bb * H + h] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc = __dadd_rn(acc, __dmul_rn(dv[u], (double)zv[u]));
      accb = __dadd_rn(accb, dv[u]);
    }
  }
  part[warp][lane] = acc;
  if (lane == 0) partb[warp] = accb;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t = __dadd_rn(t, part[w][lane]);
    if (h < H) ro.g_w_out[(int64_t)c * H + h] += t;
    if (lane == 0 && (r % htiles) == 0) {
      double tb = 0.0;
      for (int w = 0; w < kWarps; ++w) tb = __dadd_rn(tb, partb[w]);
      ro.g_b_out[c] += tb;
    }
  }
}

__device__ __forceinline__ const Seg& seg_of(const Seg& s0, const Seg& s1, int tile, int& lt) {
  if (tile < s0.tiles) { lt = tile; return s0; }
  lt = tile - s0.tiles;
  return s1;
}

__global__ void __launch_bounds__(kThreads, SW_EPROP_MINB)
k_eprop_fused(Seg s0, Seg s1, const float* __restrict__ psi, const float* __restrict__ lsig,
              int B, int H, float beta, float rho, float alpha, ReadoutArgs ro, int ro_blocks,
              unsigned* tickets) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if ((int)blockIdx.x < ro_blocks) {
    readout_block(blockIdx.x, B, H, ro);
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
          const Seg& sg = seg_of(s0, s1, tile, lt);
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
      // ---------------- ordered float64 sum + bulk store ----------------
      double g = 0.0;
      const uint64_t pol = sw::policy_evict_first();
      for (uint32_t k = 0;; ++k) {
        const int slot = k % kStages;
        const uint32_t par = (k / kStages) & 1;
        sw::mbar_wait(&S.full[slot], par);
        const int tile = S.tile[slot];
        if (tile < 0) break;
        const int ch = S.ch[slot];
        sw::mbar_wait(&S.ready[slot], par);
        int lt;
        const Seg& sg = seg_of(s0, s1, tile, lt);
        const int nb = min(kCB, B - ch * kCB);
        if (lane == 0) {
          const int64_t off = ((int64_t)lt * B + (int64_t)ch * kCB) * 32;
          sw::bulk_s2g_hint(sg.eps + off, &S.st[slot].eps[0][0], (uint32_t)nb * kRowBytes, pol);
          sw::bulk_s2g_hint(sg.ebar + off, &S.st[slot].ebar[0][0], (uint32_t)nb * kRowBytes, pol);
          sw::bulk_commit();
        }
        const int e = lt * 32 + lane;
        if (ch == 0) g = sg.grad[e];
        const float(*tm)[32] = S.st[slot].terms;
        for (int r = 0; r < nb; ++r) g = __dadd_rn(g, (double)tm[r][lane]);
        if (ch == nch - 1) sg.grad[e] = g;
        if (lane == 0) sw::bulk_wait_read0();
        __syncwarp();
        if (lane == 0) sw::mbar_arrive(&S.freed[slot]);
      }
      if (lane == 0) sw::bulk_wait0();
    } else {
      // ---------------- compute ----------------
      const int cw = warp - 2;
      int cur_tile = -1, pre = 0, post = 0;
      const float* trace = nullptr;
      for (uint32_t k = 0;; ++k) {
        const int slot = k % kStages;
        const uint32_t par = (k / kStages) & 1;
        sw::mbar_wait(&S.full[slot], par);
        const int tile = S.tile[slot];
        if (tile < 0) break;
        const int ch = S.ch[slot];
        if (tile != cur_tile) {
          int lt;
          const Seg& sg = seg_of(s0, s1, tile, lt);
          pre = __ldg(sg.pre + lt * 32 + lane);
          post = __ldg(sg.post + lt * 32 + lane);
          trace = sg.trace;
          cur_tile = tile;
        }
        const int P = (tile < s0.tiles) ? s0.P : s1.P;
        const int nb = min(kCB, B - ch * kCB);
        const int bl0 = cw * kBPW;
        float zb[kBPW], p[kBPW], l[kBPW];
        // per-stage base pointers; replica q of this warp is one row further
        const int64_t b0 = (int64_t)ch * kCB + bl0;
        const float* trp = trace + b0 * P + pre;
        const float* psp = psi + b0 * H + post;
        const float* lsp = lsig + b0 * H + post;
        Stage& st = S.st[slot];
        if (bl0 + kBPW <= nb) {
          // full chunk: no per-replica guards
#pragma unroll
          for (int q = 0; q < kBPW; ++q) {
            zb[q] = __ldg(trp + q * P);
            p[q] = __ldg(psp + q * H);
            l[q] = __ldg(lsp + q * H);
          }
#pragma unroll
          for (int q = 0; q < kBPW; ++q) {
            const int bl = bl0 + q;
            const float ep = st.eps[bl][lane];
            const float ee = __fmul_rn(p[q], __fsub_rn(zb[q], __fmul_rn(beta, ep)));
            const float ebn = __fadd_rn(__fmul_rn(alpha, st.ebar[bl][lane]), ee);
            st.ebar[bl][lane] = ebn;
            st.eps[bl][lane] = __fadd_rn(__fmul_rn(rho, ep), ee);
            st.terms[bl][lane] = __fmul_rn(l[q], ebn);
          }
        } else {
#pragma unroll
          for (int q = 0; q < kBPW; ++q) {
            if (bl0 + q < nb) {
              zb[q] = __ldg(trp + q * P);
              p[q] = __ldg(psp + q * H);
              l[q] = __ldg(lsp + q * H);
            }
          }
#pragma unroll
          for (int q = 0; q < kBPW; ++q) {
            const int bl = bl0 + q;
            if (bl < nb) {
              const float ep = st.eps[bl][lane];
              const float ee = __fmul_rn(p[q], __fsub_rn(zb[q], __fmul_rn(beta, ep)));
              const float ebn = __fadd_rn(__fmul_rn(alpha, st.ebar[bl][lane]), ee);
              st.ebar[bl][lane] = ebn;
              st.eps[bl][lane] = __fadd_rn(__fmul_rn(rho, ep), ee);
              st.terms[bl][lane] = __fmul_rn(l[q], ebn);
            }
          }
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

}  // namespace

extern "C" int sw_eprop_fused_step(const sw_eprop_seg_t* segs, int32_t n_segs, const float* psi,
                                   const float* lsig, int32_t batch, int32_t hidden, float beta,
                                   float rho, float alpha, const double* d, const float* zbar,
                                   double* g_w_out, double* g_b_out, int32_t num_classes,
                                   int32_t max_blocks_per_sm, uint32_t* workspace, void* stream) {
  if (!workspace) { sw::set_last_error("eprop: workspace (2 zeroed uint32) required"); return SW_ERR_INVALID_ARG; }
  if (n_segs < 1 || n_segs > 2) { sw::set_last_error("eprop: 1 or 2 segments"); return SW_ERR_INVALID_ARG; }
  Seg s[2] = {};
  for (int k = 0; k < n_segs; ++k) {
    const sw_eprop_seg_t& q = segs[k];
    if (q.e_pad % 32) { sw::set_last_error("eprop: e_pad must be a multiple of 32"); return SW_ERR_INVALID_ARG; }
    s[k] = Seg{q.pre, q.post, q.pre_trace, q.eps, q.ebar, q.grad, q.num_pre, q.e_pad / 32};
  }
  ReadoutArgs ro{d, zbar, g_w_out, g_b_out, num_classes};
  const int ro_blocks = (d && num_classes > 0) ? num_classes * ((hidden + 31) / 32) : 0;
  const int tiles = s[0].tiles + s[1].tiles;
  if (tiles + ro_blocks == 0 || batch <= 0) return SW_OK;
  const int smem = (int)sizeof(Smem);
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute((const void*)k_eprop_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eprop_fused, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
  }
  const int bps = (max_blocks_per_sm > 0 && max_blocks_per_sm < per_sm) ? max_blocks_per_sm : per_sm;
  const int workers = tiles ? min(tiles, 148 * bps) : 0;
  k_eprop_fused<<<ro_blocks + workers, kThreads, smem, (cudaStream_t)stream>>>(
      s[0], s[1], psi, lsig, batch, hidden, beta, rho, alpha, ro, ro_blocks, workspace);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_eprop_fused_step");
  return SW_OK;
}
