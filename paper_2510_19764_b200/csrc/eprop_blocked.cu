// Temporally blocked e-prop update (sparsewire/_kernels.py:15-39 semantics,
// k consecutive timesteps per pass over the eligibility state).
//
// The eligibility recursion of step t+1 needs only eps/ebar after step t and
// step t+1's own inputs (pre trace, psi, lsig), and the forward pass never
// reads eps, ebar or the gradient.  So the trainer runs k forward steps first
// and this kernel then streams every (tile, replica-chunk) of eps/ebar through
// shared memory once for all k steps.  That is 1/k of the HBM traffic of k
// single-step passes.  The pipeline is the one of eprop_fused.cu:
//   warp 0      TMA loader (eps/ebar bulk copies, NS-stage mbarrier ring);
//   warps 2..9  k recursion steps per element, in shared memory; float32
//               gradient terms per step into a separate NT-deep ring (so
//               most of the shared memory holds eps/ebar in flight);
//   warp 1      bulk store, and k float64 chains per synapse.  Chain 0
//               continues from the gradient, chains 1..k-1 start at zero, and
//               each chain adds its step's terms in ascending replica order.
//               At the tile's last chunk: grad = ((c0 + c1) + c2) + c3.
// eps and ebar are bit-identical to k single-step passes.  The gradient
// equals the sequential sum for k = 1; for k > 1 it differs only in the
// float64 rounding of that final combination of partial chains.
// Readout gradients (classifier.py:221-222) for the k steps are reduced by
// extra blocks of the same launch, placed after the streaming workers so
// they fill the SMs idle in the tile-granular tail.
// Timing notes (C1, one B200, graph replay; ablation builds since removed):
// K = 4: the eps/ebar stream alone 35 us (88 % of the measured HBM peak on
// its bytes), the full pass ~98 us.  K = 8 (the trainer's): full pass 179 us;
// without the float64 chains 179 us (hidden behind the recursion); without
// the recursion 98 us; without both 66 us (stream + readout).  With every
// gather forced onto L1-resident lines 172 us: the recursion is issue-bound
// (~15 instructions per element-step at ~2 IPC), not gather-latency-bound
// (see DESIGN.md 4).
#include "common.cuh"
#include "sm100_async.cuh"

#include <cstdio>
#include <cstdlib>

namespace {

constexpr int kMaxK = SW_EPROP_MAX_BLOCK;
#ifndef SW_EPB_UNROLL
#define SW_EPB_UNROLL 1
#endif
constexpr int kEpbUnroll = SW_EPB_UNROLL;
constexpr int kRowBytes = 32 * 4;
constexpr int kMaxWarps = 10;  // readout blocks: all warps of the block split the batch (NC <= 8)

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
  double* ro_scratch;          // split readout partials (NULL: block per class and h-tile)
  int ro_splits;
  int k;
};

// CB replicas per stage, NS stages
template <int K, int CB>
struct Stage {
  float eps[CB][32];
  float ebar[CB][32];
};

// NS eps/ebar stages (held until their bulk store has read them) and a
// separate ring of NT gradient-term buffers (held only until the chain warp
// has added them), so that most of the shared memory holds eps/ebar bytes in
// flight
template <int K, int CB, int NS, int NT>
struct Smem {
  Stage<K, CB> st[NS];
  float terms[NT][K][CB][32];
  uint64_t full[NS];
  uint64_t ready[NS];
  uint64_t freed[NS];
  uint64_t tfree[NT];
  int tile[NS];
  int ch[NS];
};

// part/partb: kMaxWarps*33 + kMaxWarps doubles of the block's dynamic shared
// memory (the streaming blocks' stage ring; no static shared memory, which
// would cost the streaming blocks occupancy)
__device__ void readout_block_k(int r, int B, int H, const StepsB& sp, double* g_w_out, double* g_b_out,
                                int C, double* scratch) {
  double (*part)[33] = reinterpret_cast<double (*)[33]>(scratch);
  double* partb = scratch + kMaxWarps * 33;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int htiles = (H + 31) / 32;
  const int c = r / htiles, h = (r % htiles) * 32 + lane;
  double acc = 0.0, accb = 0.0;
  const int per = (B + nw - 1) / nw;
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
    for (int w = 0; w < nw; ++w) t = __dadd_rn(t, part[w][lane]);
    if (h < H) g_w_out[(int64_t)c * H + h] += t;
    if (lane == 0 && (r % htiles) == 0) {
      double tb = 0.0;
      for (int w = 0; w < nw; ++w) tb = __dadd_rn(tb, partb[w]);
      g_b_out[c] += tb;
    }
  }
}

// Split readout (sp.ro_scratch != NULL): block r = (64-unit h-tile, group
// of kRoCG classes, split s of the k*B (step, replica) pairs).  The block
// stages the d values of its pairs in shared memory (one coalesced pass),
// then every lane accumulates two hidden units (float2 zbar loads, 4 pairs
// in flight) in float64 for the kRoCG classes; the warps take consecutive
// pair ranges and are combined in warp order.  The block writes its partial
// to partial[s][c][h] (ro_scratch[0 : S*C*H]) and partial_b[s][c] (next
// S*C), and the last block of its (h-tile, class group) -- counters after the
// partials, zeroed by the caller and reset here -- adds the S partials in
// split order to g_w_out / g_b_out.  Deterministic; the (step, replica)
// summation order differs from the single-step kernel only in its grouping.
constexpr int kRoCG = 4;
constexpr int kRoH = 64;      // hidden units per readout block (2 per lane)
constexpr int kRoU = 4;
constexpr int kRoFixed = kMaxWarps * kRoCG * kRoH + kMaxWarps * kRoCG + 2;   // doubles before the d stage

__device__ void readout_split(int r, int B, int H, const StepsB& sp, double* g_w_out, double* g_b_out,
                              int C, double* smem, int smem_doubles) {
  double* part = smem;                                   // [kMaxWarps][kRoCG][kRoH]
  double* partb = part + kMaxWarps * kRoCG * kRoH;       // [kMaxWarps][kRoCG]
  unsigned* flag = reinterpret_cast<unsigned*>(partb + kMaxWarps * kRoCG);
  double* sd = smem + kRoFixed;                          // staged d of a pair chunk [pair][kRoCG]
  const int cap = (smem_doubles - kRoFixed) / kRoCG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int S = sp.ro_splits;
  const int ncg = (C + kRoCG - 1) / kRoCG;
  const int sidx = r % S, grp = r / S;
  const int cg = grp % ncg, ht = grp / ncg;
  const int h0 = ht * kRoH + 2 * lane, c0 = cg * kRoCG;
  const bool ok0 = h0 < H, ok1 = h0 + 1 < H;
  const bool vec = (H & 1) == 0;
  const int pairs = sp.k * B;
  const int p0 = (int)((int64_t)pairs * sidx / S), p1 = (int)((int64_t)pairs * (sidx + 1) / S);
  double acc[kRoCG][2], accb[kRoCG];
#pragma unroll
  for (int c = 0; c < kRoCG; ++c) acc[c][0] = acc[c][1] = accb[c] = 0.0;
  for (int q0 = p0; q0 < p1; q0 += cap) {
    const int q1 = min(p1, q0 + cap);
    __syncthreads();
    for (int x = threadIdx.x; x < (q1 - q0) * kRoCG; x += blockDim.x) {
      const int j = q0 + x / kRoCG, c = x % kRoCG;
      const int q = j / B, b = j - q * B;
      sd[x] = c0 + c < C ? __ldg(sp.d[q] + (int64_t)b * C + c0 + c) : 0.0;
    }
    __syncthreads();
    const int per = (q1 - q0 + nw - 1) / nw;
    const int w0 = q0 + warp * per, w1 = min(q1, w0 + per);
    for (int j = w0; j < w1; j += kRoU) {
      float2 zv[kRoU];
#pragma unroll
      for (int u = 0; u < kRoU; ++u) {
        const int jj = min(j + u, w1 - 1);
        const int q = jj / B, b = jj - q * B;
        const float* zr = sp.zbar[q] + (int64_t)b * H + h0;
        if (vec && ok1) {
          zv[u] = __ldg(reinterpret_cast<const float2*>(zr));
        } else {
          zv[u].x = ok0 ? __ldg(zr) : 0.0f;
          zv[u].y = ok1 ? __ldg(zr + 1) : 0.0f;
        }
      }
#pragma unroll
      for (int u = 0; u < kRoU; ++u) {
        if (j + u < w1) {
          const double* dr = sd + (j + u - q0) * kRoCG;
#pragma unroll
          for (int c = 0; c < kRoCG; ++c) {
            const double dv = dr[c];
            acc[c][0] = __dadd_rn(acc[c][0], __dmul_rn(dv, (double)zv[u].x));
            acc[c][1] = __dadd_rn(acc[c][1], __dmul_rn(dv, (double)zv[u].y));
            accb[c] = __dadd_rn(accb[c], dv);
          }
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kRoCG; ++c) {
    part[(warp * kRoCG + c) * kRoH + 2 * lane] = acc[c][0];
    part[(warp * kRoCG + c) * kRoH + 2 * lane + 1] = acc[c][1];
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < kRoCG; ++c) partb[warp * kRoCG + c] = accb[c];
  }
  __syncthreads();
  double* partial = sp.ro_scratch;
  double* partial_b = partial + (int64_t)S * C * H;
  unsigned* cnt = reinterpret_cast<unsigned*>(partial_b + (int64_t)S * C);
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < kRoCG; ++c) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t = __dadd_rn(t, part[(w * kRoCG + c) * kRoH + 2 * lane + i]);
        if (c0 + c < C && h0 + i < H) partial[((int64_t)sidx * C + c0 + c) * H + h0 + i] = t;
      }
      if (lane == 0 && c0 + c < C) {
        double tb = 0.0;
        for (int w = 0; w < nw; ++w) tb = __dadd_rn(tb, partb[w * kRoCG + c]);
        partial_b[(int64_t)sidx * C + c0 + c] = tb;
      }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) *flag = atomicAdd(&cnt[grp], 1u);
    __syncwarp();
    if (*flag == (unsigned)(S - 1)) {
      __threadfence();
#pragma unroll
      for (int c = 0; c < kRoCG; ++c) {
        if (c0 + c >= C) continue;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (h0 + i < H) {
            double t = 0.0;
            for (int x = 0; x < S; ++x)
              t = __dadd_rn(t, __ldcg(partial + ((int64_t)x * C + c0 + c) * H + h0 + i));
            g_w_out[(int64_t)(c0 + c) * H + h0 + i] += t;
          }
        }
        if (ht == 0 && lane == 0) {
          double tb = 0.0;
          for (int x = 0; x < S; ++x) tb = __dadd_rn(tb, __ldcg(partial_b + (int64_t)x * C + c0 + c));
          g_b_out[c0 + c] += tb;
        }
      }
      if (lane == 0) cnt[grp] = 0u;
    }
  }
}

// packed float32x2 (FADD2 / FMUL2 on sm_100): two separately rounded IEEE
// ops.  Only adds, subtracts and the final product (stored, never added)
// are packed: ptxas contracts mul.rn.f32x2 feeding add.rn.f32x2 into FFMA2
// even under -fmad=false, so the products that feed adds stay scalar
// __fmul_rn, which it does not contract.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ const SegB& seg_of(const SegB& s0, const SegB& s1, int tile, int& lt) {
  if (tile < s0.tiles) { lt = tile; return s0; }
  lt = tile - s0.tiles;
  return s1;
}

// resident blocks per SM that the stage ring leaves room for (<= 3): the
// register budget of __launch_bounds__
template <int K, int CB, int NS, int NT>
constexpr int smem_blocks() {
  constexpr int per = (int)sizeof(Smem<K, CB, NS, NT>) + 1024 + 2 * 1024;
  return (233472 / per) < 3 ? ((233472 / per) < 1 ? 1 : 233472 / per) : 3;
}

// KH < K (U == 1 only): the K steps' gathers of a replica are loaded KH
// steps at a time (fewer live registers, more resident warps)
template <int K, int NC, int U, int NS, int CB, int NT, int MB, int KH>
__global__ void __launch_bounds__((NC + 2) * 32, MB > 0 ? MB : smem_blocks<K, CB, NS, NT>())
k_eprop_block(SegB s0, SegB s1, StepsB sp, int B, int H, float beta, float rho, float alpha,
              double* g_w_out, double* g_b_out, int C, int workers, unsigned* tickets) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem<K, CB, NS, NT>& S = *reinterpret_cast<Smem<K, CB, NS, NT>*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // readout blocks come after the streaming workers: they fill the SMs that
  // the tile-granular streaming work leaves idle at its end
  if ((int)blockIdx.x >= workers) {
    if (sp.ro_scratch)
      readout_split(blockIdx.x - workers, B, H, sp, g_w_out, g_b_out, C, reinterpret_cast<double*>(smem_raw),
                    (int)(sizeof(Smem<K, CB, NS, NT>) / sizeof(double)));
    else
      readout_block_k(blockIdx.x - workers, B, H, sp, g_w_out, g_b_out, C, reinterpret_cast<double*>(smem_raw));
  } else {
    const int tiles = s0.tiles + s1.tiles;
    const int nch = (B + CB - 1) / CB;
    if (threadIdx.x == 0) {
      for (int s = 0; s < NS; ++s) {
        sw::mbar_init(&S.full[s], 1);
        sw::mbar_init(&S.ready[s], NC);
        sw::mbar_init(&S.freed[s], 1);
      }
      for (int s = 0; s < NT; ++s) sw::mbar_init(&S.tfree[s], 1);
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
            const int slot = k % NS;
            if (k >= NS) sw::mbar_wait(&S.freed[slot], ((k / NS) - 1) & 1);
            S.tile[slot] = -1;
            sw::mbar_arrive(&S.full[slot]);
            break;
          }
          int lt;
          const SegB& sg = seg_of(s0, s1, tile, lt);
          for (int ch = 0; ch < nch; ++ch, ++k) {
            const int slot = k % NS;
            if (k >= NS) sw::mbar_wait(&S.freed[slot], ((k / NS) - 1) & 1);
            S.tile[slot] = tile;
            S.ch[slot] = ch;
            const int nb = min(CB, B - ch * CB);
            const uint32_t bytes = (uint32_t)nb * kRowBytes;
            const int64_t off = ((int64_t)lt * B + (int64_t)ch * CB) * 32;
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
        const int slot = kk % NS;
        const uint32_t par = (kk / NS) & 1;
        sw::mbar_wait(&S.full[slot], par);
        const int tile = S.tile[slot];
        if (tile < 0) break;
        const int ch = S.ch[slot];
        sw::mbar_wait(&S.ready[slot], par);
        int lt;
        const SegB& sg = seg_of(s0, s1, tile, lt);
        const int nb = min(CB, B - ch * CB);
        if (lane == 0) {
          const int64_t off = ((int64_t)lt * B + (int64_t)ch * CB) * 32;
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
        const float (*terms)[CB][32] = S.terms[kk % NT];
        for (int r = 0; r < nb; ++r) {
#pragma unroll
          for (int q = 0; q < K; ++q)
            acc[q] = __dadd_rn(acc[q], (double)terms[q][r][lane]);
        }
        __syncwarp();
        if (lane == 0) sw::mbar_arrive(&S.tfree[kk % NT]);
        if (ch == nch - 1) {
          double g = acc[0];
#pragma unroll
          for (int q = 1; q < K; ++q) g = __dadd_rn(g, acc[q]);
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
      constexpr int kBPW = CB / NC;
      const int bl0 = cw * kBPW;
      int cur_tile = -1, pre = 0, post = 0, P = 0;
      const float* trace[K];
      for (uint32_t kk = 0;; ++kk) {
        const int slot = kk % NS;
        const uint32_t par = (kk / NS) & 1;
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
        const int nb = min(CB, B - ch * CB);
        Stage<K, CB>& st = S.st[slot];
        float (*terms)[CB][32] = S.terms[kk % NT];
        if (kk >= (uint32_t)NT) sw::mbar_wait(&S.tfree[kk % NT], ((kk / NT) - 1) & 1);
        // K is the exact step count (one instantiation per k), so the K
        // gathers of a replica are issued together ahead of the recursion;
        // 32-bit element offsets, one per replica for all K steps
#pragma unroll kEpbUnroll
        for (int u0 = 0; u0 < kBPW; u0 += U) {
          if constexpr (U == 1 && KH < K) {
            const int bl = bl0 + u0;
            const unsigned b = (unsigned)(ch * CB + min(bl, nb - 1));
            const unsigned ot = b * (unsigned)P + (unsigned)pre;
            const unsigned oh = b * (unsigned)H + (unsigned)post;
            float ep = 0.f, eb = 0.f;
            if (bl < nb) {
              ep = st.eps[bl][lane];
              eb = st.ebar[bl][lane];
            }
#pragma unroll
            for (int q0 = 0; q0 < K; q0 += KH) {
              float zh[KH], ph[KH], lh[KH];
#pragma unroll
              for (int q = 0; q < KH; ++q) {
                zh[q] = __ldg(trace[q0 + q] + ot);
                ph[q] = __ldg(sp.psi[q0 + q] + oh);
                lh[q] = __ldg(sp.lsig[q0 + q] + oh);
              }
              if (bl < nb) {
#pragma unroll
                for (int q = 0; q < KH; ++q) {
                  const float ee = __fmul_rn(ph[q], __fsub_rn(zh[q], __fmul_rn(beta, ep)));
                  eb = __fadd_rn(__fmul_rn(alpha, eb), ee);
                  ep = __fadd_rn(__fmul_rn(rho, ep), ee);
                  terms[q0 + q][bl][lane] = __fmul_rn(lh[q], eb);
                }
              }
            }
            if (bl < nb) {
              st.ebar[bl][lane] = eb;
              st.eps[bl][lane] = ep;
            }
            continue;
          }
          float zb[U][K], p[U][K], l[U][K];
#pragma unroll
          for (int v = 0; v < U; ++v) {
            const unsigned b = (unsigned)(ch * CB + min(bl0 + u0 + v, nb - 1));
            const unsigned ot = b * (unsigned)P + (unsigned)pre;
            const unsigned oh = b * (unsigned)H + (unsigned)post;
#pragma unroll
            for (int q = 0; q < K; ++q) {
              zb[v][q] = __ldg(trace[q] + ot);
              p[v][q] = __ldg(sp.psi[q] + oh);
              l[v][q] = __ldg(sp.lsig[q] + oh);
            }
          }
          if constexpr (U == 2) {
            // two replicas per thread: the adds and the term product packed
            const int ba = bl0 + u0, bb = bl0 + u0 + 1;
            if (ba < nb) {
              const bool okb = bb < nb;
              float epa = st.eps[ba][lane], eba = st.ebar[ba][lane];
              float epb = okb ? st.eps[bb][lane] : 0.f, ebb = okb ? st.ebar[bb][lane] : 0.f;
#pragma unroll
              for (int q = 0; q < K; ++q) {
                float xa, xb;
                up2(sub2(pk2(zb[0][q], zb[1][q]), pk2(__fmul_rn(beta, epa), __fmul_rn(beta, epb))), xa, xb);
                const unsigned long long ee = pk2(__fmul_rn(p[0][q], xa), __fmul_rn(p[1][q], xb));
                const unsigned long long ebn = add2(pk2(__fmul_rn(alpha, eba), __fmul_rn(alpha, ebb)), ee);
                const unsigned long long epn = add2(pk2(__fmul_rn(rho, epa), __fmul_rn(rho, epb)), ee);
                float ta, tb;
                up2(mul2(pk2(l[0][q], l[1][q]), ebn), ta, tb);
                up2(ebn, eba, ebb);
                up2(epn, epa, epb);
                terms[q][ba][lane] = ta;
                if (okb) terms[q][bb][lane] = tb;
              }
              st.ebar[ba][lane] = eba;
              st.eps[ba][lane] = epa;
              if (okb) {
                st.ebar[bb][lane] = ebb;
                st.eps[bb][lane] = epb;
              }
            }
          } else {
#pragma unroll
          for (int v = 0; v < U; ++v) {
            const int bl = bl0 + u0 + v;
            if (bl < nb) {
              float ep = st.eps[bl][lane];
              float eb = st.ebar[bl][lane];
#pragma unroll
              for (int q = 0; q < K; ++q) {
                const float ee = __fmul_rn(p[v][q], __fsub_rn(zb[v][q], __fmul_rn(beta, ep)));
                eb = __fadd_rn(__fmul_rn(alpha, eb), ee);
                ep = __fadd_rn(__fmul_rn(rho, ep), ee);
                terms[q][bl][lane] = __fmul_rn(l[v][q], eb);
              }
              st.ebar[bl][lane] = eb;
              st.eps[bl][lane] = ep;
            }
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

template <int K, int NC, int U, int NS = 3, int CB = 32, int NT = 3, int MB = 0, int KH = K>
int launch_block(SegB s0, SegB s1, const StepsB& sp, int B, int H, float beta, float rho, float alpha,
                 double* g_w_out, double* g_b_out, int C, int ro_blocks, unsigned* tickets,
                 cudaStream_t st) {
  static_assert(NC + 2 <= kMaxWarps && CB % NC == 0, "eprop block configuration");
  static_assert(sizeof(Smem<K, CB, NS, NT>) >= (kRoFixed + 64 * kRoCG) * sizeof(double), "readout scratch");
  const int smem = (int)sizeof(Smem<K, CB, NS, NT>);
  constexpr int threads = (NC + 2) * 32;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute((const void*)k_eprop_block<K, NC, U, NS, CB, NT, MB, KH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eprop_block<K, NC, U, NS, CB, NT, MB, KH>, threads, smem);
    if (per_sm < 1) per_sm = 1;
  }
  const int tiles = s0.tiles + s1.tiles;
  int cap = per_sm;
  if (const char* e = getenv("SW_EPB_PER_SM")) cap = max(1, min(per_sm, atoi(e)));
  const int workers = tiles ? min(tiles, 148 * cap) : 0;
  k_eprop_block<K, NC, U, NS, CB, NT, MB, KH><<<ro_blocks + workers, threads, smem, st>>>(s0, s1, sp, B, H, beta, rho, alpha,
                                                                      g_w_out, g_b_out, C, workers, tickets);
  sw::count_launch();
  return SW_OK;
}


// configuration of the k = 4 kernel: compute warps x stages x replicas per
// stage (SW_EPB_CFG = "NCxNSxCB", for measurement)
int block_cfg() {
  static int cfg = -1;
  if (cfg < 0) {
    cfg = 0;
    if (const char* e = getenv("SW_EPB_CFG")) {
      int nc = 0, ns = 0, cb = 0;
      if (sscanf(e, "%dx%dx%d", &nc, &ns, &cb) == 3)
        cfg = nc * (ns >= 10 ? 10000 : 1000) + ns * 100 + cb;
    }
  }
  return cfg;
}

}  // namespace

extern "C" int64_t sw_eprop_readout_scratch_bytes(int32_t hidden, int32_t num_classes, int32_t splits) {
  if (hidden <= 0 || num_classes <= 0 || splits <= 0) return 0;
  const int64_t groups = (int64_t)((hidden + 31) / 32) * ((num_classes + kRoCG - 1) / kRoCG);
  return 8 * ((int64_t)splits * num_classes * hidden + (int64_t)splits * num_classes) + 4 * groups;
}

extern "C" int sw_eprop_fused_block(const sw_eprop_seg_t* segs, int32_t n_segs, const sw_eprop_block_t* blk,
                                    int32_t batch, int32_t hidden, float beta, float rho, float alpha,
                                    double* g_w_out, double* g_b_out, int32_t num_classes,
                                    uint32_t* workspace, void* stream) {
  if (!workspace) { sw::set_last_error("eprop block: workspace (2 zeroed uint32) required"); return SW_ERR_INVALID_ARG; }
  if (n_segs < 1 || n_segs > 2) { sw::set_last_error("eprop block: 1 or 2 segments"); return SW_ERR_INVALID_ARG; }
  if (!blk || blk->k < 1 || blk->k > kMaxK) { sw::set_last_error("eprop block: 1 <= k <= SW_EPROP_MAX_BLOCK steps"); return SW_ERR_INVALID_ARG; }
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
  // unused steps alias step 0 (the kernel loads them unconditionally)
  for (int i = 0; i < n_segs; ++i)
    for (int k = blk->k; k < kMaxK; ++k) s[i].trace[k] = s[i].trace[0];
  StepsB sp{};
  sp.k = blk->k;
  for (int k = 0; k < kMaxK; ++k) {
    sp.psi[k] = blk->psi[k < blk->k ? k : 0];
    sp.lsig[k] = blk->lsig[k < blk->k ? k : 0];
    sp.d[k] = blk->d[k];
    sp.zbar[k] = blk->zbar[k];
  }
  const bool readout = blk->d[0] && g_w_out && num_classes > 0;
  sp.ro_scratch = blk->ro_scratch;
  sp.ro_splits = blk->ro_splits > 0 ? blk->ro_splits : 1;
  const int htiles = (hidden + 31) / 32;
  const int ro_blocks = !readout ? 0
                        : sp.ro_scratch ? ((hidden + kRoH - 1) / kRoH) * ((num_classes + kRoCG - 1) / kRoCG) * sp.ro_splits
                                        : num_classes * htiles;
  if (s[0].tiles + s[1].tiles + ro_blocks == 0 || batch <= 0) return SW_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
#define SW_EPB_ARGS s[0], s[1], sp, batch, hidden, beta, rho, alpha, g_w_out, g_b_out, num_classes, ro_blocks, workspace, st
  const int cfg = block_cfg();
  switch (blk->k) {
    case 1: rc = launch_block<1, 8, 1>(SW_EPB_ARGS); break;
    case 2: rc = launch_block<2, 8, 1>(SW_EPB_ARGS); break;
    case 3: rc = launch_block<3, 8, 1>(SW_EPB_ARGS); break;
    case 4:
      switch (cfg) {
        case 8332: rc = launch_block<4, 8, 1, 3, 32, 3>(SW_EPB_ARGS); break;
        case 8333: rc = launch_block<4, 8, 2, 4, 32, 2>(SW_EPB_ARGS); break;     // "8x3x33": K=4 packed pairs
        case 8816: rc = launch_block<4, 8, 1, 8, 16, 2>(SW_EPB_ARGS); break;
        default: rc = launch_block<4, 8, 1, 4, 32, 2>(SW_EPB_ARGS); break;
      }
      break;
    case 5: rc = launch_block<5, 4, 1, 4, 16, 2>(SW_EPB_ARGS); break;
    case 6: rc = launch_block<6, 4, 1, 4, 16, 2>(SW_EPB_ARGS); break;
    case 7: rc = launch_block<7, 4, 1, 4, 16, 2>(SW_EPB_ARGS); break;
    default:
      switch (cfg) {
        case 8432: rc = launch_block<8, 8, 1, 4, 32, 2>(SW_EPB_ARGS); break;
        case 4616: rc = launch_block<8, 4, 1, 6, 16, 2>(SW_EPB_ARGS); break;
        case 4432: rc = launch_block<8, 4, 1, 4, 32, 2>(SW_EPB_ARGS); break;
        case 4316: rc = launch_block<8, 4, 1, 3, 16, 2>(SW_EPB_ARGS); break;
        case 4416: rc = launch_block<8, 4, 1, 4, 16, 2>(SW_EPB_ARGS); break;
        case 4417: rc = launch_block<8, 4, 1, 4, 16, 2, 4>(SW_EPB_ARGS); break;      // "4x4x17": the narrow-layer default
        case 4408: rc = launch_block<8, 4, 1, 4, 8, 4, 4>(SW_EPB_ARGS); break;        // "4x4x8": 8 replicas, 4 term buffers
        case 4221: rc = launch_block<8, 4, 1, 2, 16, 2, 5, 4>(SW_EPB_ARGS); break;   // "4x2x21": halves, 5 CTAs/SM
        case 4419: rc = launch_block<8, 4, 2, 4, 16, 2, 4>(SW_EPB_ARGS); break;   // "4x4x19": packed pairs
        case 4420: rc = launch_block<8, 4, 2, 4, 16, 2, 3>(SW_EPB_ARGS); break;   // "4x4x20": packed pairs, <= 113 regs
        // default: <= 85 registers (4 CTAs/SM by registers), so a CTA also
        // fits next to 3 forward blocks of the overlapping k_clf_step launch;
        // wide hidden layers (psi/lsig rows >= 2 KB, more gather misses) gain
        // from 8-replica stages with a 4-deep term ring, i.e. more stages in
        // flight per CTA (C2: 226 -> 203 us; C1 loses 175 -> 185 us with it)
        default:
          if (hidden >= 512) rc = launch_block<8, 4, 1, 4, 8, 4, 4>(SW_EPB_ARGS);
          else rc = launch_block<8, 4, 1, 4, 16, 2, 4>(SW_EPB_ARGS);
          break;
      }
      break;
  }
#undef SW_EPB_ARGS
  if (rc) return rc;
  SW_CHECK_LAUNCH("sw_eprop_fused_block");
  return SW_OK;
}
