// Replica-minor e-prop pass (sparsewire/_kernels.py:15-39 recursion over K
// timesteps per pass; classifier.py:223 learning signal).
//
// Layout: the forward pass writes its per-step vectors replica-major ([B, n]);
// sw_eprop_prep turns a group of K steps into replica-minor copies
// ([n, B]: pre traces, psi) and computes the learning signal
// lsig[h, b] = f32(sum_c d[b, c] * W_out[c, h]) (classes ascending, as the
// forward pass did) straight into that layout.  The pass kernel then gives
// each lane one synapse and R consecutive replicas: the K steps' inputs of
// the lane are three runs of R floats (trace[pre, b0:b0+R], psi[post, ...],
// lsig[post, ...]), loaded with 16-byte vector loads, and the eligibility
// state of the lane is R contiguous floats ([tile][chunk][lane][R]).  Per
// element-step: one 0.75-instruction share of the loads, the eight float32
// operations of the recursion (op for op those of _kernels.py:33-38, so eps
// and ebar are bit-identical to the reference) and one float64 add of the
// gradient term into the lane's accumulator.
//
// Work items are (tile of 8 synapses, split of 64 replicas), statically
// round-robin over the warps; a warp runs an item's 32-replica chunks, writes
// its float64 partial per synapse, and k_grad_reduce adds the splits'
// partials to the gradient in split order: deterministic, and a float64
// regrouping of the reference's replica-ordered sum (within rounding of it).  The plan order of the
// synapses (sw_eprop_plan with shift 0: by post, then pre) makes a warp's
// psi/lsig runs mostly the same address (broadcast) and its trace runs
// distinct 32-byte sectors.
#include "common.cuh"
#include "sm100_async.cuh"

#include <cstdio>
#include <cstdlib>

namespace {

constexpr int kTW = 8;          // warps per pass block

// ---------------------------------------------------------------- prep ----
// Block = (hidden tile of kHT units, replica tile of kBT, step k), 256 threads.
//   A  replica-minor copies: zbar and psi of the tile, and a share of the
//      xbar rows, through a [kBT][kHT + 1] shared tile (coalesced both ways);
//   B  lsig_t[k][h][b] = f32(sum_c d[b][c] * W_out[c][h]), c ascending, one
//      fused multiply-add per class from +0.0 (the forward pass's arithmetic):
//      lane = replica with its d row in registers, W_out[:, tile] in shared
//      memory, each warp kHT/8 hidden units;
//   C  readout-gradient partials over the tile's replicas, b ascending:
//      part[k][bt][c][h] = sum_b d[b][c] * zbar[b][h] (thread = hidden unit x
//      class group) and, in h tile 0, sum_b d[b][c]; k_readout_reduce adds
//      the (k, bt) partials into g_w_out / g_b_out in a fixed order
//      (classifier.py:221-222 summed over the group's steps and replicas; a
//      regrouping of the reference's float64 sums).
constexpr int kHT = 64;
constexpr int kBT = 32;

// the interleaved psi/lsig layout: per group of 4 replicas, 4 psi then 4
// lsig floats; psi of (row, b) at psl_index, its lsig 4 floats later
__host__ __device__ __forceinline__ int64_t psl_index(int64_t row, int64_t L, int b) {
  return (row * L + (b & ~3)) * 2 + (b & 3);
}
constexpr int kMaxC = 32;
// d of the replica tile, class-major with two pad doubles per class row: the
// class-fastest stores of the coalesced d read spread over the banks, and a
// class's replicas b, b+1 (b even) are one 16-byte load
constexpr int kDT = kBT + 2;

__host__ __device__ inline size_t prep_smem_bytes(int C) {
  return (size_t)2 * kBT * (kHT + 1) * 4 + (size_t)C * kHT * 8 + (size_t)kDT * C * 8;
}

// CT: the class count as a compile-time constant (0 = runtime, any count);
// MB: blocks per SM the register budget is sized for
template <int CT, int MB = 1>
__global__ void __launch_bounds__(256, MB) k_prep(const sw_eprop_prep_t P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  sw::pdl_enter();
  float (*tile)[kHT + 1] = reinterpret_cast<float (*)[kHT + 1]>(smem_raw);                       // zbar
  float (*ptile)[kHT + 1] = reinterpret_cast<float (*)[kHT + 1]>(smem_raw + (size_t)kBT * (kHT + 1) * 4);   // psi
  double* ws = reinterpret_cast<double*>(smem_raw + (size_t)2 * kBT * (kHT + 1) * 4);   // [C][kHT]
  const int C = CT ? CT : P.num_classes;
  const int H = P.hidden, NI = P.num_inputs, B = P.batch;
  const int64_t L = P.ldb;
  double* dt = ws + (size_t)C * kHT;                                                  // [C][kDT]
  const int ht = blockIdx.x, bt = blockIdx.y, k = blockIdx.z;
  const int h0 = ht * kHT, b0 = bt * kBT;
  const int nh = min(kHT, H - h0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool ro = P.g_w_out != nullptr;
  const bool want_lsig = (P.lsig_t != nullptr || P.psl_t != nullptr) && P.d[0] != nullptr;

  // ---- A: transposes (psi, zbar of the tile; xbar rows split over the h tiles) ----
  auto load_tile = [&](const float* in, int n, int r0, int nr) {
    for (int x = tid; x < kBT * kHT; x += 256) {
      const int b = x / kHT, r = x % kHT;
      tile[b][r] = (r < nr && b0 + b < B) ? in[(int64_t)(b0 + b) * n + r0 + r] : 0.f;
    }
  };
  auto store_tile = [&](int r0, int nr, float* out) {
    for (int x = tid; x < kBT * kHT; x += 256) {
      const int r = x / kBT, b = x % kBT;
      if (r < nr && b0 + b < L) out[(int64_t)(r0 + r) * L + b0 + b] = tile[b][r];
    }
  };
  const int nht = gridDim.x;
  const int xper = (NI + nht - 1) / nht, x0 = min(NI, ht * xper), x1 = min(NI, x0 + xper);
  for (int r0 = x0; P.xbar[k] && r0 < x1; r0 += kHT) {   // NULL: xbar_t precomputed (sw_clf_inputs)
    load_tile(P.xbar[k], NI, r0, min(kHT, x1 - r0));
    __syncthreads();
    store_tile(r0, min(kHT, x1 - r0), P.xbar_t + (int64_t)k * NI * L);
    __syncthreads();
  }
  // one round of loads: the psi and zbar tiles (through registers, all
  // issued before any shared-memory store), W_out, d, and (deferred
  // reduction) the readout partials this block adds to
  constexpr int kPer = kBT * kHT / 256;
  // with the class count known, W_out's tile columns and the replicas' d
  // rows join the same round (registers, stored after the tiles)
  constexpr int kWPer = CT > 0 ? (CT * kHT + 255) / 256 : 1;
  constexpr int kDPer = CT > 0 ? (kBT * CT + 255) / 256 : 1;
  double wv[kWPer], dv[kDPer];
  {
    float pv[kPer], zv[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int x = tid + u * 256, b = x / kHT, r = x % kHT;
      const bool ok = r < nh && b0 + b < B;
      const int64_t g = (int64_t)(b0 + b) * H + h0 + r;
      pv[u] = ok ? P.psi[k][g] : 0.f;
      zv[u] = ok ? P.zbar[k][g] : 0.f;
    }
    if constexpr (CT > 0) {
      if (want_lsig || ro) {
#pragma unroll
        for (int u = 0; u < kWPer; ++u) {
          const int x = tid + u * 256, c = x / kHT, r = x % kHT;
          wv[u] = (x < CT * kHT && r < nh) ? P.w_out[(int64_t)c * H + h0 + r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kDPer; ++u) {
          const int x = tid + u * 256, b = x / CT, c = x - b * CT;
          dv[u] = (x < kBT * CT && b0 + b < B) ? P.d[k][(int64_t)(b0 + b) * CT + c] : 0.0;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int x = tid + u * 256, b = x / kHT, r = x % kHT;
      ptile[b][r] = pv[u];
      tile[b][r] = zv[u];
    }
  }
  constexpr int CP = (CT > 0 && CT % 4 == 0) ? CT / 4 : 1;
  const int rr = tid % kHT, cg = tid / kHT;   // readout partials: thread = (hidden unit, class group of 4)
  double* part = ro ? P.ro_partial + ((int64_t)k * gridDim.y + bt) * (C * (int64_t)H + C) : nullptr;
  double prev[CP];
#pragma unroll
  for (int u = 0; u < CP; ++u) prev[u] = 0.0;
  if constexpr (CT > 0 && CT % 4 == 0) {
    if (ro && P.defer_reduce && rr < nh) {
#pragma unroll
      for (int u = 0; u < CP; ++u) prev[u] = part[(int64_t)(cg * CP + u) * H + h0 + rr];
    }
  }
  if constexpr (CT > 0) {
    if (want_lsig || ro) {
#pragma unroll
      for (int u = 0; u < kWPer; ++u) {
        const int x = tid + u * 256;
        if (x < CT * kHT) ws[x] = wv[u];
      }
#pragma unroll
      for (int u = 0; u < kDPer; ++u) {
        const int x = tid + u * 256, b = x / CT, c = x - b * CT;
        if (x < kBT * CT) dt[c * kDT + b] = dv[u];
      }
    }
  } else if (want_lsig || ro) {
    for (int x = tid; x < C * kHT; x += 256) {
      const int c = x / kHT, r = x % kHT;
      ws[x] = r < nh ? P.w_out[(int64_t)c * H + h0 + r] : 0.0;
    }
    for (int x = tid; x < kBT * C; x += 256) {   // coalesced read of d, class-major store
      const int b = x / C, c = x - b * C;
      dt[c * kDT + b] = b0 + b < B ? P.d[k][(int64_t)(b0 + b) * C + c] : 0.0;
    }
  }
  __syncthreads();
  for (int x = tid; x < kBT * kHT; x += 256) {
    const int r = x / kBT, b = x % kBT;
    if (r < nh && b0 + b < L) {
      const int64_t row = (int64_t)k * H + h0 + r;
      if (P.psl_t) P.psl_t[psl_index(row, L, b0 + b)] = ptile[b][r];
      else P.psi_t[row * L + b0 + b] = ptile[b][r];
      P.zbar_t[row * L + b0 + b] = tile[b][r];
    }
  }

  // ---- B: learning signal, lane = replica ----
  if (want_lsig) {
    // lsig of (row, replica b0 + lane): lsig_t[row][b], or the lsig half of
    // the interleaved group
    auto lsig_at = [&](int r) -> float* {
      const int64_t row = (int64_t)k * H + h0 + r;
      return P.psl_t ? P.psl_t + psl_index(row, L, b0 + lane) + 4 : P.lsig_t + row * L + b0 + lane;
    };
    if constexpr (CT > 0) {
      double dr[CT];
#pragma unroll
      for (int c = 0; c < CT; ++c) dr[c] = dt[c * kDT + lane];
      // warp w: rows 8w .. 8w+7, four consecutive rows at a time (their
      // W_out values one 32-byte shared load per class), four independent
      // class chains interleaved (W_out's columns past nh are zero)
#pragma unroll 1
      for (int i = 0; i < 2; ++i) {
        const int r0 = warp * 8 + i * 4;
        if (r0 >= nh) break;
        double ls[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int c = 0; c < CT; ++c) {
          const double2* w2 = reinterpret_cast<const double2*>(ws + c * kHT + r0);
          const double2 wa = w2[0], wb = w2[1];
          ls[0] = __fma_rn(dr[c], wa.x, ls[0]);
          ls[1] = __fma_rn(dr[c], wa.y, ls[1]);
          ls[2] = __fma_rn(dr[c], wb.x, ls[2]);
          ls[3] = __fma_rn(dr[c], wb.y, ls[3]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (r0 + q < nh && b0 + lane < L) *lsig_at(r0 + q) = b0 + lane < B ? __double2float_rn(ls[q]) : 0.f;
      }
    } else {
      for (int r = warp; r < nh; r += 8) {
        double ls = 0.0;
        for (int c = 0; c < C; ++c) ls = __fma_rn(dt[c * kDT + lane], ws[c * kHT + r], ls);
        if (b0 + lane < L) *lsig_at(r) = b0 + lane < B ? __double2float_rn(ls) : 0.f;
      }
    }
  }

  // ---- C: readout partials, thread = (hidden unit, class group of 4) ----
  if (ro) {
    const int r = rr;
    if (r < nh) {
      if constexpr (CT > 0 && CT % 4 == 0) {
        double acc[CP];
#pragma unroll
        for (int u = 0; u < CP; ++u) acc[u] = 0.0;
        const double* dg = dt + cg * CP * kDT;
        for (int b = 0; b < kBT; b += 2) {
          const double z0 = (double)tile[b][r], z1 = (double)tile[b + 1][r];
#pragma unroll
          for (int u = 0; u < CP; ++u) {
            const double2 dd = *reinterpret_cast<const double2*>(dg + u * kDT + b);
            acc[u] = __fma_rn(dd.y, z1, __fma_rn(dd.x, z0, acc[u]));
          }
        }
#pragma unroll
        for (int u = 0; u < CP; ++u) {
          double* pp = part + (int64_t)(cg * CP + u) * H + h0 + r;
          *pp = P.defer_reduce ? __dadd_rn(prev[u], acc[u]) : acc[u];
        }
      } else {
        const int cper = (C + 3) / 4, ca = cg * cper, cb = min(C, ca + cper);
        for (int c = ca; c < cb; ++c) {
          double acc = 0.0;
          for (int b = 0; b < kBT; ++b) acc = __fma_rn(dt[c * kDT + b], (double)tile[b][r], acc);
          double* pp = part + (int64_t)c * H + h0 + r;
          *pp = P.defer_reduce ? __dadd_rn(*pp, acc) : acc;
        }
      }
    }
    if (ht == 0 && tid < C) {
      double sb = 0.0;
      for (int b = 0; b < kBT; ++b) sb = __dadd_rn(sb, dt[tid * kDT + b]);
      double* pp = part + (int64_t)C * H + tid;
      *pp = P.defer_reduce ? __dadd_rn(*pp, sb) : sb;
    }
  }
}

// g_w_out[c][h] += sum of the (k, bt) partials; g_b_out likewise.  Block = 32
// outputs; warp w sums the partials of its eighth of the (k, bt) range in
// order, then warp 0 adds the 8 warp sums in order (a fixed grouping).
__global__ void __launch_bounds__(256) k_readout_reduce(const sw_eprop_prep_t P, int nparts) {
  __shared__ double ws8[8][32];
  const int C = P.num_classes, H = P.hidden;
  const int64_t stride = C * (int64_t)H + C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = blockIdx.x * 32 + lane;
  const int q0 = (int)((int64_t)nparts * warp / 8), q1 = (int)((int64_t)nparts * (warp + 1) / 8);
  double s = 0.0;
  if (x < stride) {
    int q = q0;
    for (; q + 8 <= q1; q += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(P.ro_partial + (q + u) * stride + x);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        s = __dadd_rn(s, v[u]);
        P.ro_partial[(q + u) * stride + x] = 0.0;
      }
    }
    for (; q < q1; ++q) {
      s = __dadd_rn(s, __ldcg(P.ro_partial + q * stride + x));
      P.ro_partial[q * stride + x] = 0.0;
    }
  }
  ws8[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && x < stride) {
    double t = ws8[0][lane];
    for (int w = 1; w < 8; ++w) t = __dadd_rn(t, ws8[w][lane]);
    if (x < C * H) P.g_w_out[x] = __dadd_rn(P.g_w_out[x], t);
    else P.g_b_out[x - C * H] = __dadd_rn(P.g_b_out[x - C * H], t);
  }
}

// ---------------------------------------------------------------- pass ----
// A warp = 8 synapses x 32 replicas: lane = 4 * s + g holds synapse s of the
// work item's 8-synapse tile and replicas [b0 + 8g, b0 + 8g + 8) of the
// current 32-replica chunk.  Every input run and state run of a lane is 32
// contiguous bytes (one 256-bit access), and the 4 lanes of a synapse read one
// full 128-byte line: a warp-wide load touches 8 lines (trace: 8 distinct
// pres) or 1-2 lines (psi/lsig: the plan's post order makes the 8 synapses
// share posts), which keeps the L1 tag stage -- the limit of the lane-per-
// synapse form -- off the critical path.
struct TSeg {
  const int32_t* pre;
  const int32_t* post;
  const float* trace[SW_EPROP_MAX_BLOCK];
  float* eps;
  float* ebar;
  double* grad;
  int tiles;             // 8-synapse tiles
};

struct TPass {
  TSeg s[2];
  const float* psi[SW_EPROP_MAX_BLOCK];
  const float* lsig[SW_EPROP_MAX_BLOCK];
  double* partial;       // [tiles][splits][8]
  int ldb, splits, chunks_per_split;
  float beta, rho, alpha;
  unsigned long long nz;   // (-0.0f, -0.0f)
  int defer;               // partials accumulate over passes; sw_eprop_pass_reduce adds them
  int zero;                // eps/ebar start from zero (not read)
  int dbg;   // measurement only (SW_EPT_DBG): 1 = every synapse reads pre/post 0 (L1-resident inputs), 2 = no state traffic
};

// packed float32x2 helpers (add/sub/mul .rn.f32x2, sm_100)
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

// products as fma(a, b, nz) with nz = (-0, -0) from a kernel argument: the
// exact product rounded once (fma with a -0 addend), which ptxas cannot
// contract into a following packed add (it does contract mul.rn.f32x2)
__device__ __forceinline__ unsigned long long pmul2(unsigned long long a, unsigned long long b, unsigned long long nz) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(nz));
  return r;
}
__device__ __forceinline__ void ld256p(unsigned long long (&v)[4], const float* p) {
  asm("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ld256p_cs(unsigned long long (&v)[4], const float* p) {
  asm("ld.global.cs.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}
__device__ __forceinline__ void st256p_cs(float* p, const unsigned long long (&v)[4]) {
  asm volatile("st.global.cs.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(v[0]), "l"(v[1]), "l"(v[2]), "l"(v[3])
               : "memory");
}

// grad[e] += the splits' partials, split order
template <int SPW>
__global__ void k_grad_reduce(const TPass T) {
  const int tiles0 = T.s[0].tiles, tiles = tiles0 + T.s[1].tiles;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < tiles * SPW; x += gridDim.x * blockDim.x) {
    const int tile = x / SPW, sl = x % SPW;
    const bool first = tile < tiles0;
    double* grad = first ? T.s[0].grad : T.s[1].grad;
    const int e = (first ? tile : tile - tiles0) * SPW + sl;
    double gr = grad[e];
    for (int q = 0; q < T.splits; ++q) {
      double* pp = T.partial + ((int64_t)tile * T.splits + q) * SPW + sl;
      gr = __dadd_rn(gr, __ldcg(pp));
      *pp = 0.0;
    }
    grad[e] = gr;
  }
}

// RPL replicas per lane as RPL/2 packed pairs: one 128- or 256-bit access
template <int RPL>
__device__ __forceinline__ void ldp(unsigned long long (&v)[RPL / 2], const float* p) {
  if constexpr (RPL == 8) {
    asm("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
  } else if constexpr (RPL == 2) {
    asm("ld.global.nc.b64 %0, [%1];" : "=l"(v[0]) : "l"(p));
  } else {
    asm("ld.global.nc.v2.b64 {%0,%1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p));
  }
}
template <int RPL>
__device__ __forceinline__ void ldp_cs(unsigned long long (&v)[RPL / 2], const float* p) {
  if constexpr (RPL == 8) {
    asm("ld.global.cs.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
  } else if constexpr (RPL == 2) {
    asm("ld.global.cs.b64 %0, [%1];" : "=l"(v[0]) : "l"(p));
  } else {
    asm("ld.global.cs.v2.b64 {%0,%1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p));
  }
}
template <int RPL>
__device__ __forceinline__ void stp_cs(float* p, const unsigned long long (&v)[RPL / 2]) {
  if constexpr (RPL == 8) {
    asm volatile("st.global.cs.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(v[0]), "l"(v[1]), "l"(v[2]), "l"(v[3])
                 : "memory");
  } else if constexpr (RPL == 2) {
    asm volatile("st.global.cs.b64 [%0], %1;" ::"l"(p), "l"(v[0]) : "memory");
  } else {
    asm volatile("st.global.cs.v2.b64 [%0], {%1,%2};" ::"l"(p), "l"(v[0]), "l"(v[1]) : "memory");
  }
}

// psi and lsig runs of a lane (RPL replicas from replica-minor offset off):
// two loads, or one 32-byte load of the interleaved group (PSL)
template <int RPL, bool PSL>
__device__ __forceinline__ void load_pl(unsigned long long (&pv)[RPL / 2], unsigned long long (&lv)[RPL / 2],
                                        const float* psi, const float* lsig, int64_t off) {
  if constexpr (PSL && RPL == 2) {
    // two replicas (an aligned pair) of a 4-replica group: psi pair, then
    // the lsig pair 4 floats later
    const float* q = psi + ((off & ~3ll) * 2 + (off & 3));
    asm("ld.global.nc.b64 %0, [%1];" : "=l"(pv[0]) : "l"(q));
    asm("ld.global.nc.b64 %0, [%1];" : "=l"(lv[0]) : "l"(q + 4));
  } else if constexpr (PSL) {
    unsigned long long v[4];
    asm("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
        : "l"(psi + 2 * off));
    pv[0] = v[0];
    pv[1] = v[1];
    lv[0] = v[2];
    lv[1] = v[3];
  } else {
    ldp<RPL>(pv, psi + off);
    ldp<RPL>(lv, lsig + off);
  }
}

// SPW synapses per warp (tile), LPS = 32/SPW lanes per synapse, each lane
// RPL = 32/LPS consecutive replicas of the 32-replica chunk; PD: steps of
// inputs loaded ahead of the recursion
// PSL: psi and lsig interleaved per 4-replica group (one 32-byte load per
// step instead of two 16-byte loads; RPL = 4 only)
template <int K, int PD, int SPW, int MB, bool PSL>
__global__ void __launch_bounds__(kTW * 32, MB) k_eprop_t(const TPass T) {
  constexpr int LPS = 32 / SPW, RPL = 32 / LPS, NP = RPL / 2;
  static_assert(!PSL || RPL == 4 || RPL == 2, "interleaved psi/lsig: 2 or 4 replicas per lane");
  sw::pdl_enter();
  const int lane = threadIdx.x & 31;
  const int sl = lane / LPS, g = lane % LPS;
  const int tiles0 = T.s[0].tiles;
  const int tiles = tiles0 + T.s[1].tiles;
  const int items = tiles * T.splits;
  const int nchunk = T.ldb / 32;
  const int64_t L = T.ldb;
  // static assignment of the uniform work items (no ticket atomics): block b
  // owns the contiguous item range [b*items/nb, (b+1)*items/nb) and its warps
  // stride through it, so the warps of a block work on neighbouring tiles of
  // one replica split at a time
  const int nwb = blockDim.x >> 5;
  const int i0 = (int)((int64_t)items * blockIdx.x / gridDim.x), i1 = (int)((int64_t)items * (blockIdx.x + 1) / gridDim.x);
  for (int item = i0 + (threadIdx.x >> 5); item < i1; item += nwb) {
    // split-major item order: the warps working at any moment share replica ranges
    const int split = item / tiles, tile = item - split * tiles;
    const bool first = tile < tiles0;
    const TSeg& S = first ? T.s[0] : T.s[1];
    const int lt = first ? tile : tile - tiles0;
    const int e = lt * SPW + sl;
    int pre = __ldg(S.pre + e), post = __ldg(S.post + e);
    if (T.dbg == 1) pre = post = 0;
    const int c0 = split * T.chunks_per_split, c1 = min(nchunk, c0 + T.chunks_per_split);
    const int64_t tofs = (int64_t)pre * L + g * RPL, pofs = (int64_t)post * L + g * RPL;
    const unsigned long long B2 = pk2(T.beta, T.beta), A2 = pk2(T.alpha, T.alpha), R2 = pk2(T.rho, T.rho);
    const unsigned long long NZ = T.nz;
    double acc = 0.0;
    // state and inputs as packed replica pairs
    unsigned long long ep[NP], eb[NP];
    const int64_t so0 = (((int64_t)lt * nchunk + c0) * 32 + lane) * RPL;
    if (T.dbg == 2 || T.zero) {
      for (int r = 0; r < NP; ++r) ep[r] = eb[r] = 0ull;
    } else {
      ldp_cs<RPL>(ep, S.eps + so0);
      ldp_cs<RPL>(eb, S.ebar + so0);
    }
    for (int c = c0; c < c1; ++c) {
      const int b0 = c * 32;
      const int64_t so = (((int64_t)lt * nchunk + c) * 32 + lane) * RPL;
      unsigned long long zin[K][NP], pin[K][NP], lin[K][NP];
#pragma unroll
      for (int k = 0; k < PD && k < K; ++k) {
        ldp<RPL>(zin[k], S.trace[k] + tofs + b0);
        load_pl<RPL, PSL>(pin[k], lin[k], T.psi[k], T.lsig[k], pofs + b0);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (k + PD < K) {
          ldp<RPL>(zin[k + PD], S.trace[k + PD] + tofs + b0);
          load_pl<RPL, PSL>(pin[k + PD], lin[k + PD], T.psi[k + PD], T.lsig[k + PD], pofs + b0);
        }
        // _kernels.py:33-38 on replica pairs, every op a separately rounded
        // packed f32x2 op: e = psi*(zb - beta*eps); ebar = alpha*ebar + e;
        // grad += f64(lsig*ebar); eps = rho*eps + e
#pragma unroll
        for (int r = 0; r < NP; ++r) {
          const unsigned long long x = sub2(zin[k][r], pmul2(B2, ep[r], NZ));
          const unsigned long long ee = pmul2(pin[k][r], x, NZ);
          eb[r] = add2(pmul2(A2, eb[r], NZ), ee);
          float t0, t1;
          up2(mul2(lin[k][r], eb[r]), t0, t1);
          acc = __dadd_rn(acc, (double)t0);
          acc = __dadd_rn(acc, (double)t1);
          ep[r] = add2(pmul2(R2, ep[r], NZ), ee);
        }
      }
      if (T.dbg != 2) {
        stp_cs<RPL>(S.eps + so, ep);
        stp_cs<RPL>(S.ebar + so, eb);
      }
      if (c + 1 < c1 && T.dbg != 2) {
        if (T.zero) {
#pragma unroll
          for (int r = 0; r < NP; ++r) ep[r] = eb[r] = 0ull;
        } else {
          ldp_cs<RPL>(ep, S.eps + so + 32 * RPL);
          ldp_cs<RPL>(eb, S.ebar + so + 32 * RPL);
        }
      }
    }
    // the synapse's LPS replica groups, added pairwise: (g0 + g1) + (g2 + g3) ...
#pragma unroll
    for (int o = 1; o < LPS; o <<= 1) acc = __dadd_rn(acc, __shfl_xor_sync(SW_FULL_MASK, acc, o));
    // this split's partial; k_grad_reduce adds the splits in order
    if (g == 0) {
      double* pp = T.partial + ((int64_t)tile * T.splits + split) * SPW + sl;
      *pp = T.defer ? __dadd_rn(*pp, acc) : acc;   // deferred: the batch's passes in order
    }
  }
}

}  // namespace

extern "C" int64_t sw_eprop_prep_scratch_bytes(int32_t k, int32_t batch, int32_t hidden, int32_t num_classes) {
  if (k < 1 || batch < 1 || hidden < 1 || num_classes < 1) return 0;
  return (int64_t)k * ((batch + kBT - 1) / kBT) * ((int64_t)num_classes * hidden + num_classes) * 8;
}

extern "C" int sw_eprop_prep(const sw_eprop_prep_t* p, void* stream) {
  if (!p || p->k < 1 || p->k > SW_EPROP_MAX_BLOCK || p->batch < 1 || p->ldb < p->batch || p->ldb % 32) {
    sw::set_last_error("sw_eprop_prep: 1 <= k <= SW_EPROP_MAX_BLOCK, batch >= 1, ldb >= batch, ldb % 32 == 0");
    return SW_ERR_INVALID_ARG;
  }
  if (p->num_classes > kMaxC || (p->g_w_out && (!p->ro_partial || !p->g_b_out || !p->d[0]))) {
    sw::set_last_error("sw_eprop_prep: num_classes <= 32; readout needs d, g_b_out and ro_partial");
    return SW_ERR_INVALID_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = prep_smem_bytes(p->num_classes);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute((const void*)k_prep<0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute((const void*)k_prep<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute((const void*)k_prep<20, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute((const void*)k_prep<20, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  if (smem > 200 * 1024) { sw::set_last_error("sw_eprop_prep: shared memory"); return SW_ERR_INVALID_ARG; }
  // the replica tiles cover ldb (the padding columns are written as zeros)
  dim3 grid((p->hidden + kHT - 1) / kHT, (p->ldb + kBT - 1) / kBT, p->k);
  // register budget for 3 blocks per SM (80 registers; measured: C1 prep
  // 27.9 -> 25.0 us, C2 118.6 -> 96.6 us against the unconstrained 89, and
  // 26.2 / 99.0 us at 4 blocks, which spills); SW_PREP_MB=1|4 (measurement)
  static const int pmb = [] { const char* e = getenv("SW_PREP_MB"); return e ? atoi(e) : 3; }();
  static const bool pdl = [] { const char* e = getenv("SW_CLF_PDL"); return e && e[0] == '1'; }();
  if (p->num_classes == 20 && pmb == 4) sw::pdl_launch(pdl, k_prep<20, 4>, grid, dim3(256), smem, st, *p);
  else if (p->num_classes == 20 && pmb == 1) sw::pdl_launch(pdl, k_prep<20>, grid, dim3(256), smem, st, *p);
  else if (p->num_classes == 20) sw::pdl_launch(pdl, k_prep<20, 3>, grid, dim3(256), smem, st, *p);   // the SHD-shaped task
  else sw::pdl_launch(pdl, k_prep<0, 2>, grid, dim3(256), smem, st, *p);
  sw::count_launch();
  if (p->g_w_out && !p->defer_reduce) {
    const int n = p->num_classes * p->hidden + p->num_classes;
    k_readout_reduce<<<(n + 31) / 32, 256, 0, st>>>(*p, p->k * (int)grid.y);
    sw::count_launch();
  }
  SW_CHECK_LAUNCH("sw_eprop_prep");
  return SW_OK;
}

extern "C" int sw_eprop_prep_reduce(const sw_eprop_prep_t* p, void* stream) {
  if (!p || !p->g_w_out || !p->g_b_out || !p->ro_partial || p->k < 1 || p->ldb < 32) {
    sw::set_last_error("sw_eprop_prep_reduce: readout gradients, partials and the group's k / ldb required");
    return SW_ERR_INVALID_ARG;
  }
  const int n = p->num_classes * p->hidden + p->num_classes;
  k_readout_reduce<<<(n + 31) / 32, 256, 0, (cudaStream_t)stream>>>(*p, p->k * ((p->ldb + kBT - 1) / kBT));
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_eprop_prep_reduce");
  return SW_OK;
}

// synapses per warp of the pass (the plan's state layout, [e_pad/SPW][ldb/32][32][32/(32/SPW)])
constexpr int kSPW = SW_EPROP_PASS_SPW;

extern "C" int32_t sw_eprop_pass_synapses_per_warp(void) { return kSPW; }

extern "C" int64_t sw_eprop_pass_scratch_bytes(int32_t e_pad_total, int32_t ldb) {
  if (e_pad_total <= 0 || ldb <= 0) return 0;
  const int64_t tiles = e_pad_total / kSPW;
  const int64_t splits = (ldb + 63) / 64;
  return tiles * splits * kSPW * 8;
}

extern "C" int sw_eprop_pass(const sw_eprop_tseg_t* segs, int32_t n_segs, const sw_eprop_tpass_t* p,
                             int32_t ldb, float beta, float rho, float alpha, void* stream) {
  if (!p || n_segs < 1 || n_segs > 2 || p->k < 1 || p->k > SW_EPROP_MAX_BLOCK) {
    sw::set_last_error("sw_eprop_pass: 1 or 2 segments, 1 <= k <= SW_EPROP_MAX_BLOCK");
    return SW_ERR_INVALID_ARG;
  }
  if (ldb < 32 || ldb % 32) {
    sw::set_last_error("sw_eprop_pass: ldb (padded batch) must be a positive multiple of 32");
    return SW_ERR_INVALID_ARG;
  }
  if (!p->scratch) {
    sw::set_last_error("sw_eprop_pass: scratch of sw_eprop_pass_scratch_bytes() bytes required");
    return SW_ERR_INVALID_ARG;
  }
  TPass T{};
  int etot = 0;
  for (int i = 0; i < n_segs; ++i) {
    const sw_eprop_tseg_t& q = segs[i];
    if (q.e_pad % 32) { sw::set_last_error("sw_eprop_pass: e_pad must be a multiple of 32"); return SW_ERR_INVALID_ARG; }
    T.s[i].pre = q.pre;
    T.s[i].post = q.post;
    for (int k = 0; k < SW_EPROP_MAX_BLOCK; ++k) T.s[i].trace[k] = q.trace_t[k < p->k ? k : 0];
    T.s[i].eps = q.eps;
    T.s[i].ebar = q.ebar;
    T.s[i].grad = q.grad;
    T.s[i].tiles = q.e_pad / kSPW;
    etot += q.e_pad;
  }
  for (int k = 0; k < SW_EPROP_MAX_BLOCK; ++k) {
    T.psi[k] = p->psi_t[k < p->k ? k : 0];
    T.lsig[k] = p->lsig_t[k < p->k ? k : 0];
  }
  const int tiles = etot / kSPW;
  if (tiles == 0) return SW_OK;
  const int nchunk = ldb / 32;
  T.ldb = ldb;
  T.splits = (ldb + 63) / 64;
  T.chunks_per_split = (nchunk + T.splits - 1) / T.splits;
  T.partial = (double*)p->scratch;
  T.beta = beta;
  T.rho = rho;
  T.alpha = alpha;
  T.nz = 0x8000000080000000ull;
  T.defer = p->defer_reduce != 0;
  T.zero = p->state_zero != 0;
  {
    static const int dbg = [] { const char* e = getenv("SW_EPT_DBG"); return e ? atoi(e) : 0; }();
    T.dbg = dbg;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // variant (SW_EPT_CFG = "1,4": inputs 1 step ahead instead of 2)
  static int cfg = -1;
  if (cfg < 0) {
    cfg = 0;
    if (const char* ev = getenv("SW_EPT_CFG")) {
      int pd = 0, mb = 0;
      if (sscanf(ev, "%d,%d", &pd, &mb) == 2) cfg = pd * 10 + mb;
    }
  }
  const int items = tiles * T.splits;
  auto launch = [&](auto kfn) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kTW * 32, 0);
    if (per_sm < 1) per_sm = 1;
    static const int cap_sm = [] { const char* e = getenv("SW_EPT_PER_SM"); return e ? atoi(e) : 0; }();
    if (cap_sm > 0 && cap_sm < per_sm) per_sm = cap_sm;   // measurement: leave room on the SMs
    int blocks = 148 * per_sm;
    if (blocks * kTW > items) blocks = (items + kTW - 1) / kTW;
    static const bool pdl = [] { const char* e = getenv("SW_CLF_PDL"); return e && e[0] == '1'; }();
    sw::pdl_launch(pdl, kfn, dim3(blocks), dim3(kTW * 32), 0, st, T);
  };
  const int want = cfg ? cfg : 24;
  switch (p->k) {
#define SW_K(KK)                                                                 \
  case KK:                                                                       \
    if (want == 14) launch(k_eprop_t<KK, 1, kSPW, 4, false>);                    \
    else if (p->psl) launch(k_eprop_t<KK, 2, kSPW, 4, true>);                    \
    else launch(k_eprop_t<KK, 2, kSPW, 4, false>);                               \
    break;
    SW_K(1) SW_K(2) SW_K(3) SW_K(4) SW_K(5) SW_K(6) SW_K(7) SW_K(8)
    SW_K(9) SW_K(10) SW_K(11) SW_K(12) SW_K(13) SW_K(14) SW_K(15) SW_K(16)
#undef SW_K
    default: sw::set_last_error("sw_eprop_pass: k"); return SW_ERR_INVALID_ARG;
  }
  sw::count_launch();
  if (!T.defer) {
    const int n = tiles * kSPW;
    k_grad_reduce<kSPW><<<(n + 255) / 256, 256, 0, st>>>(T);
    sw::count_launch();
  }
  SW_CHECK_LAUNCH("sw_eprop_pass");
  return SW_OK;
}

extern "C" int sw_eprop_pass_reduce(const sw_eprop_tseg_t* segs, int32_t n_segs, int32_t ldb, void* scratch,
                                    void* stream) {
  if (n_segs < 1 || n_segs > 2 || ldb < 32 || ldb % 32 || !scratch) {
    sw::set_last_error("sw_eprop_pass_reduce: 1 or 2 segments, ldb a multiple of 32, scratch");
    return SW_ERR_INVALID_ARG;
  }
  TPass T{};
  int etot = 0;
  for (int i = 0; i < n_segs; ++i) {
    T.s[i].grad = segs[i].grad;
    T.s[i].tiles = segs[i].e_pad / kSPW;
    etot += segs[i].e_pad;
  }
  T.splits = (ldb + 63) / 64;
  T.partial = (double*)scratch;
  const int n = etot;
  if (n == 0) return SW_OK;
  k_grad_reduce<kSPW><<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(T);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_eprop_pass_reduce");
  return SW_OK;
}
