// Topographic-map rewiring rule (sparsewire/topomap.py:70-223) on the device.
//
// One rewiring update of one projection = four stream-ordered kernels that
// need no host round trip (so the update can live inside a CUDA graph):
//  1. k_rw_keys:  host/row stream keys folded on the device from the host
//     prefixes fold_key(seed,"host") / fold_key(seed,"row") with
//     (rule_id, update_count, pass 0) (updates.py:313-318, 346-349); bumps
//     update_count; zeroes the per-update counters;
//  2. host phase (topomap.py:101-108): histogram of total_attempts draws of
//     uniform_int(num_pre) on the host stream (exact rejection replay);
//  3. k_rw_rows: thread per row with attempts (topomap.py:142-196):
//     sample_k_distinct (rejection, or partial Fisher-Yates when 2k >= N),
//     ascending selected slots, elimination draws in slot order with
//     p = g < g_theta ? p_dep : p_pot, chained removal (remove_slots order),
//     formation draws for the remaining candidates in ascending post order
//     against the host-built formation-probability LUT (indexed by torus
//     offset), add_synapse at g_init or form_full on RowFull;
//  4. totals / event records for collect() and the device "changed" flag
//     that gates the transpose remap.
#include "common.cuh"
#include "ragged.cuh"
#include "util.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace {
// grid barrier; a single-block launch (small sheets: no cooperative launch,
// whose set-up costs more than the work) uses the block barrier
__device__ __forceinline__ void gsync(cg::grid_group& grid) {
  if (gridDim.x == 1) __syncthreads();
  else grid.sync();
}


constexpr int kKMax = 64;   // attempts per row handled by one thread
constexpr int kTotals = 16;  // totals[] words: see sw_rewire_update

__global__ void k_rw_keys(uint64_t host_prefix, uint64_t row_prefix, int32_t rule_id,
                          int64_t* update_count, uint64_t* keys, int64_t* totals, int32_t* changed) {
  const uint64_t u = (uint64_t)*update_count;
  keys[0] = sw::fold_int(sw::fold_int(sw::fold_int(host_prefix, (uint64_t)rule_id), u), 0);
  keys[1] = sw::fold_int(sw::fold_int(sw::fold_int(row_prefix, (uint64_t)rule_id), u), 0);
  *update_count = (int64_t)u + 1;
  for (int k = 0; k < kTotals; ++k) totals[k] = 0;
  *changed = 0;
}

__device__ __forceinline__ int torus_offset(int i, int j, int side) {
  const int xi = i % side, yi = i / side, xj = j % side, yj = j / side;
  return (xj - xi + side) % side + side * ((yj - yi + side) % side);
}

struct RwArgs {
  sw_ragged_t m;
  int gp;                       // weight plane index
  const int32_t* attempts;
  const uint64_t* keys;         // [host, row_base]
  const double* form_lut;       // [N] by torus offset
  const double* dist_lut;       // [N] by torus offset
  int side;
  double g_theta, p_dep, p_pot, g_init;
  int64_t* totals;              // [0]=removed [1]=kept [2]=formed [3]=missed [4]=full [5]=attempts [7]=error
                                // [8]=blocks done [9]=heavy rows
  int32_t* changed;
  const int32_t* ev_off;        // [P] exclusive scan of attempts (or null)
  int8_t* ev_kind;              // 1 = elimination, 2 = formation
  double* ev_d;
  int32_t* heavy;               // rows with kKMax < attempts <= N, then the heavy-row scratch (or null)
  int64_t heavy_cap;
  int32_t* plog;                // sw_transpose_patch log (or null): [0] rows, [1] pairs, [2] overflow
  int32_t pcap;
  int32_t block_totals = 0;     // counters summed per block before the atomics (large sheets)
};

// patch log: a removed (pre, post) pair, then (at the row's end) the row itself
__device__ __forceinline__ void plog_pair(const RwArgs& A, int i, int j) {
  if (!A.plog) return;
  const int k = atomicAdd(&A.plog[1], 1);
  if (k < A.pcap) {
    A.plog[4 + A.pcap + 2 * k] = i;
    A.plog[4 + A.pcap + 2 * k + 1] = j;
  } else {
    A.plog[2] = 1;
  }
}
__device__ __forceinline__ void plog_row(const RwArgs& A, int i) {
  if (!A.plog) return;
  const int k = atomicAdd(&A.plog[0], 1);
  if (k < A.pcap) A.plog[4 + k] = i;
  else A.plog[2] = 1;
}

__device__ __forceinline__ int fy_get(const int* key, const int* val, int n, int p) {
  for (int q = 0; q < n; ++q) if (key[q] == p) return val[q];
  return p;
}

// the per-row counters (removed, kept, formed, missed, full, attempts) are
// summed per thread, then (block_totals: sheets of more than 16 384 rows) per
// block in shared memory, one atomic per counter and block: one atomic per
// counter and row serialised the rows with attempts on six L2 addresses
// (s16 +5 %); on smaller sheets the block reduction costs more than it saves
__device__ __forceinline__ void rw_add_totals(const RwArgs& A, const unsigned long long (&c)[6]) {
  __shared__ unsigned long long s_tot[32][6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  unsigned long long v[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    v[q] = c[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(SW_FULL_MASK, v[q], o);
  }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 6; ++q) s_tot[warp][q] = v[q];
  __syncthreads();
  if (threadIdx.x < 6) {
    unsigned long long t = 0;
    for (int w = 0; w < nw; ++w) t += s_tot[w][threadIdx.x];
    if (t) atomicAdd((unsigned long long*)&A.totals[threadIdx.x], t);
  }
  __syncthreads();
}

__device__ __forceinline__ void rw_rows(const RwArgs& A, int64_t t0, int64_t dt) {
  const sw_ragged_t& m = A.m;
  const int N = m.num_post;
  unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};
  for (int i = (int)t0; i < m.num_pre; i += (int)dt) {
    const int k = A.attempts[i];
    if (k == 0) continue;
    if (k > N || (k > kKMax && !A.heavy)) { atomicAdd((unsigned long long*)&A.totals[7], 1ull); continue; }
    if (k > kKMax) {   // deferred to the serial heavy-row path (rw_heavy_rows)
      const unsigned long long h = atomicAdd((unsigned long long*)&A.totals[9], 1ull);
      if ((int64_t)h < A.heavy_cap) A.heavy[h] = i;
      continue;
    }
    const uint64_t key = sw::child_key(A.keys[1], (uint64_t)i);
    uint64_t ctr = 0;
    int cand[kKMax];
    // sample_k_distinct (rng.py:116-141)
    if (2 * k < N) {
      const uint64_t rem = sw::reject_rem((uint64_t)N);
      int filled = 0;
      while (filled < k) {
        const int v = (int)sw::uniform_int_seq(key, ctr, (uint64_t)N, rem);
        bool seen = false;
        for (int q = 0; q < filled; ++q) seen |= (cand[q] == v);
        if (!seen) cand[filled++] = v;
      }
    } else {
      int fk[2 * kKMax], fv[2 * kKMax], nf = 0;
      for (int q = 0; q < k; ++q) {
        const uint64_t nn = (uint64_t)(N - q);
        const int j = q + (int)sw::uniform_int_seq(key, ctr, nn, sw::reject_rem(nn));
        const int vq = fy_get(fk, fv, nf, q), vj = fy_get(fk, fv, nf, j);
        // set(q, vj); set(j, vq)
        int t;
        for (t = 0; t < nf && fk[t] != q; ++t) {}
        if (t == nf) { fk[nf] = q; ++nf; }
        fv[t] = vj;
        for (t = 0; t < nf && fk[t] != j; ++t) {}
        if (t == nf) { fk[nf] = j; ++nf; }
        fv[t] = vq;
      }
      for (int q = 0; q < k; ++q) cand[q] = fy_get(fk, fv, nf, q);
    }
    const int64_t off = (int64_t)i * m.stride;
    double* g = (double*)m.planes[A.gp];
    int n = m.row_length[i];
    // selected slots (ascending) and which candidates are connected
    int sel[kKMax];
    int ns = 0;
    unsigned long long conn = 0ull;
    for (int s = 0; s < n && ns < k; ++s) {
      const int t = m.target[off + s];
      for (int q = 0; q < k; ++q) {
        if (cand[q] == t) { sel[ns++] = s; conn |= 1ull << q; break; }
      }
    }
    // elimination draws in slot order (topomap.py:163-175)
    unsigned long long hit = 0ull;
    for (int q = 0; q < ns; ++q) {
      const double u = sw::u01(sw::draw(key, ctr++));
      const double p = g[off + sel[q]] < A.g_theta ? A.p_dep : A.p_pot;
      if (u < p) hit |= 1ull << q;
    }
    const int removed = __popcll(hit), kept = ns - removed;
    int ev = A.ev_kind ? A.ev_off[i] : 0;
    if (A.ev_kind) {
      for (int q = 0; q < ns; ++q)
        if ((hit >> q) & 1ull) {
          A.ev_kind[ev] = 1;
          A.ev_d[ev] = A.dist_lut[torus_offset(i, m.target[off + sel[q]], A.side)];
          ++ev;
        }
    }
    for (int q = 0; q < ns; ++q)
      if ((hit >> q) & 1ull) plog_pair(A, i, m.target[off + sel[q]]);
    // chained removal, descending slots (connectivity.py:130-136)
    for (int q = ns - 1; q >= 0; --q) {
      if (!((hit >> q) & 1ull)) continue;
      const int last = n - 1;
      if (sel[q] != last) sw::move_slot(m, off, sel[q], last);
      n = last;
    }
    // remaining candidates, ascending post (topomap.py:177-193)
    int rem_[kKMax];
    int nr = 0;
    for (int q = 0; q < k; ++q) {
      if ((conn >> q) & 1ull) continue;
      const int v = cand[q];
      int r = nr++;
      while (r > 0 && rem_[r - 1] > v) { rem_[r] = rem_[r - 1]; --r; }
      rem_[r] = v;
    }
    int formed = 0, missed = 0, full = 0;
    for (int q = 0; q < nr; ++q) {
      const int j = rem_[q];
      const int o = torus_offset(i, j, A.side);
      const double u = sw::u01(sw::draw(key, ctr++));
      if (!(u < A.form_lut[o])) { ++missed; continue; }
      if (n >= m.max_row_length) { ++full; continue; }
      m.target[off + n] = j;
      sw::zero_slot(m, off, n);
      g[off + n] = A.g_init;
      ++n;
      ++formed;
      if (A.ev_kind) {
        A.ev_kind[ev] = 2;
        A.ev_d[ev] = A.dist_lut[o];
        ++ev;
      }
    }
    if (A.ev_kind)
      for (; ev < A.ev_off[i] + k; ++ev) A.ev_kind[ev] = 0;
    m.row_length[i] = n;
    cnt[0] += (unsigned long long)removed;
    cnt[1] += (unsigned long long)kept;
    cnt[2] += (unsigned long long)formed;
    cnt[3] += (unsigned long long)missed;
    cnt[4] += (unsigned long long)full;
    cnt[5] += (unsigned long long)k;
    if (removed + formed) {
      *A.changed = 1;
      plog_row(A, i);
    }
  }
  if (A.block_totals) {
    rw_add_totals(A, cnt);
  } else {
#pragma unroll
    for (int q = 0; q < 6; ++q)
      if (cnt[q]) atomicAdd((unsigned long long*)&A.totals[q], cnt[q]);
  }
}

// One row with kKMax < k <= N attempts, serially, with the attempt set as a
// bitmap over the posts (the reference's own attempt-bitfield formulation,
// topomap.py:142-196): same draws in the same order as rw_rows.  Scratch
// after the heavy-row list: W bitmap words, then N int32 (Fisher-Yates
// array, reused for the selected slots).  Such rows are vanishingly rare
// (10 s^2 attempts over 256 s^2 rows per update) but must not change the
// result (KTooLarge only for k > N, as bitfield.py:67-77).
__device__ void rw_row_heavy(const RwArgs& A, int i) {
  const sw_ragged_t& m = A.m;
  const int N = m.num_post;
  const int W = (N + 63) >> 6;
  uint64_t* bits = reinterpret_cast<uint64_t*>(A.heavy + ((A.heavy_cap + 1) & ~1LL));
  int32_t* arr = reinterpret_cast<int32_t*>(bits + W);
  const int k = A.attempts[i];
  const uint64_t key = sw::child_key(A.keys[1], (uint64_t)i);
  uint64_t ctr = 0;
  for (int w = 0; w < W; ++w) bits[w] = 0ull;
  if (2 * k < N) {
    const uint64_t rem = sw::reject_rem((uint64_t)N);
    int filled = 0;
    while (filled < k) {
      const int v = (int)sw::uniform_int_seq(key, ctr, (uint64_t)N, rem);
      const uint64_t b = 1ull << (v & 63);
      if (!(bits[v >> 6] & b)) { bits[v >> 6] |= b; ++filled; }
    }
  } else {
    for (int q = 0; q < N; ++q) arr[q] = q;
    for (int q = 0; q < k; ++q) {
      const uint64_t nn = (uint64_t)(N - q);
      const int j = q + (int)sw::uniform_int_seq(key, ctr, nn, sw::reject_rem(nn));
      const int t = arr[q]; arr[q] = arr[j]; arr[j] = t;
    }
    for (int q = 0; q < k; ++q) bits[arr[q] >> 6] |= 1ull << (arr[q] & 63);
  }
  const int64_t off = (int64_t)i * m.stride;
  double* g = (double*)m.planes[A.gp];
  int n = m.row_length[i];
  // selected slots ascending; elimination draws in slot order; hit = sign bit
  int ns = 0;
  for (int s = 0; s < n; ++s) {
    const int t = m.target[off + s];
    if ((bits[t >> 6] >> (t & 63)) & 1ull) arr[ns++] = s;
  }
  int removed = 0;
  int ev = A.ev_kind ? A.ev_off[i] : 0;
  for (int q = 0; q < ns; ++q) {
    const int s = arr[q];
    const int t = m.target[off + s];
    const double u = sw::u01(sw::draw(key, ctr++));
    const double p = g[off + s] < A.g_theta ? A.p_dep : A.p_pot;
    bits[t >> 6] &= ~(1ull << (t & 63));
    if (u < p) {
      arr[q] = -1 - s;
      ++removed;
      plog_pair(A, i, t);
      if (A.ev_kind) { A.ev_kind[ev] = 1; A.ev_d[ev] = A.dist_lut[torus_offset(i, t, A.side)]; ++ev; }
    }
  }
  for (int q = ns - 1; q >= 0; --q) {
    if (arr[q] >= 0) continue;
    const int s = -1 - arr[q], last = n - 1;
    if (s != last) sw::move_slot(m, off, s, last);
    n = last;
  }
  int formed = 0, missed = 0, full = 0;
  for (int w = 0; w < W; ++w) {
    uint64_t word = bits[w];
    while (word) {
      const int j = (w << 6) + __ffsll((long long)word) - 1;
      word &= word - 1;
      const int o = torus_offset(i, j, A.side);
      const double u = sw::u01(sw::draw(key, ctr++));
      if (!(u < A.form_lut[o])) { ++missed; continue; }
      if (n >= m.max_row_length) { ++full; continue; }
      m.target[off + n] = j;
      sw::zero_slot(m, off, n);
      g[off + n] = A.g_init;
      ++n;
      ++formed;
      if (A.ev_kind) { A.ev_kind[ev] = 2; A.ev_d[ev] = A.dist_lut[o]; ++ev; }
    }
  }
  if (A.ev_kind)
    for (; ev < A.ev_off[i] + k; ++ev) A.ev_kind[ev] = 0;
  m.row_length[i] = n;
  A.totals[0] += removed;
  A.totals[1] += ns - removed;
  A.totals[2] += formed;
  A.totals[3] += missed;
  A.totals[4] += full;
  A.totals[5] += k;
  if (removed + formed) {
    *A.changed = 1;
    plog_row(A, i);
  }
}

// The last block to finish its rows runs the deferred heavy rows (if any):
// no extra launch or grid barrier on the common path.
__device__ __forceinline__ void rw_heavy_tail(const RwArgs& A) {
  if (!A.heavy) return;
  __syncthreads();
  if (threadIdx.x != 0) return;
  __threadfence();
  const unsigned long long prev = atomicAdd((unsigned long long*)&A.totals[8], 1ull);
  if (prev != gridDim.x - 1) return;
  __threadfence();
  const int64_t nh = *(volatile int64_t*)&A.totals[9];
  if (nh > A.heavy_cap) { atomicAdd((unsigned long long*)&A.totals[7], 1ull); return; }
  for (int64_t h = 0; h < nh; ++h) rw_row_heavy(A, ((volatile int32_t*)A.heavy)[h]);
}

__global__ void k_rw_rows(RwArgs A) {
  rw_rows(A, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
  rw_heavy_tail(A);
}

// One rewiring update in one cooperative launch (keys, host-phase
// histogram, row phase behind grid barriers) when no per-attempt events are
// recorded: one graph node per rule instead of five.
__global__ void __launch_bounds__(256)
k_rw_fused(RwArgs A, uint64_t host_prefix, uint64_t row_prefix, int32_t rule_id, int64_t* update_count,
           uint64_t* keys, int32_t* attempts, int64_t total_attempts, int64_t* rej) {
  cg::grid_group grid = cg::this_grid();
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gn = (int64_t)gridDim.x * blockDim.x;
  const uint64_t u = (uint64_t)*update_count;
  const uint64_t hk = sw::fold_int(sw::fold_int(sw::fold_int(host_prefix, (uint64_t)rule_id), u), 0);
  const uint64_t P = (uint64_t)A.m.num_pre;
  for (int64_t i = gt; i < (int64_t)P; i += gn) attempts[i] = 0;
  if (gt == 0) {
    keys[0] = hk;
    keys[1] = sw::fold_int(sw::fold_int(sw::fold_int(row_prefix, (uint64_t)rule_id), u), 0);
    for (int k = 0; k < kTotals; ++k) A.totals[k] = 0;
    *A.changed = 0;
    *rej = 0;
  }
  gsync(grid);
  if (gt == 0) *update_count = (int64_t)u + 1;
  const uint64_t rem = sw::reject_rem(P);
  const bool pow2 = (P & (P - 1)) == 0;
  int64_t r = 0;
  for (int64_t c = gt; c < total_attempts; c += gn) {
    const uint64_t h = sw::draw(hk, (uint64_t)c);
    if (sw::draw_valid(h, rem)) atomicAdd(attempts + (pow2 ? (h & (P - 1)) : (h % P)), 1);
    else ++r;
  }
  if (r) atomicAdd((unsigned long long*)rej, (unsigned long long)r);
  gsync(grid);
  if (gt == 0 && *rej) {
    // rejected draws (probability < P / 2^64): continue the stream serially
    int64_t need = *rej;
    uint64_t c = (uint64_t)total_attempts;
    while (need > 0) {
      const uint64_t h = sw::draw(hk, c++);
      if (sw::draw_valid(h, rem)) { attempts[h % P] += 1; --need; }
    }
  }
  if (rem != 0) gsync(grid);
  rw_rows(A, gt, gn);
  rw_heavy_tail(A);
}

__global__ void k_copy_i32(const int32_t* a, int32_t* b, int n) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) b[x] = a[x];
}

int grid1(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

// heavy-row list entries: at most total_attempts / (kKMax + 1) rows
int64_t heavy_cap(const sw_rewire_params_t* prm) { return prm->total_attempts / (kKMax + 1) + 1; }

}  // namespace

extern "C" int64_t sw_rewire_scratch_bytes(int32_t num_post, int64_t total_attempts) {
  const int64_t cap = total_attempts / (kKMax + 1) + 1;
  const int64_t W = ((int64_t)num_post + 63) / 64;
  return ((cap + 1) & ~1LL) * 4 + W * 8 + (int64_t)num_post * 4;
}

extern "C" int sw_rewire_update(const sw_ragged_t* m, int32_t weight_plane, const sw_rewire_params_t* prm,
                                int32_t* attempts, int64_t* update_count, uint64_t* keys,
                                int64_t* totals, int32_t* changed, int64_t* rej, int32_t* ev_off,
                                int8_t* ev_kind, double* ev_d, int32_t forced_attempts, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int P = m->num_pre;
  if (prm->patch_log) cudaMemsetAsync(prm->patch_log, 0, 4 * sizeof(int32_t), st);   // this update's log
  if (!forced_attempts && !ev_kind && P > 0) {
    static int max_blocks = 0;
    if (max_blocks == 0) {
      int per_sm = 0, sms = 0, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rw_fused, 256, 0);
      max_blocks = per_sm * sms;
      if (max_blocks < 1) max_blocks = 1;
    }
    int blocks = grid1(P);
    if (blocks > max_blocks) blocks = max_blocks;
    RwArgs A{*m, weight_plane, attempts, keys, prm->form_lut, prm->dist_lut, prm->side,
             prm->g_theta, prm->p_dep, prm->p_pot, prm->g_init, totals, changed, nullptr, nullptr, nullptr,
             (int32_t*)prm->scratch, heavy_cap(prm), prm->patch_log, prm->patch_cap, P > 16384 ? 1 : 0};
    uint64_t hp = prm->host_prefix, rp = prm->row_prefix;
    int32_t rid = prm->rule_id;
    int64_t ta = prm->total_attempts;
    void* args[] = {(void*)&A, (void*)&hp, (void*)&rp, (void*)&rid, (void*)&update_count, (void*)&keys,
                    (void*)&attempts, (void*)&ta, (void*)&rej};
    if (P <= 256) {
      // small sheets: one block, block barriers, an ordinary launch
      k_rw_fused<<<1, 256, 0, st>>>(A, hp, rp, rid, update_count, keys, attempts, ta, rej);
    } else {
      cudaLaunchCooperativeKernel((const void*)k_rw_fused, dim3(blocks), dim3(256), args, 0, st);
    }
    sw::count_launch();
    SW_CHECK_LAUNCH("sw_rewire_update");
    return SW_OK;
  }
  k_rw_keys<<<1, 1, 0, st>>>(prm->host_prefix, prm->row_prefix, prm->rule_id, update_count, keys,
                             totals, changed); sw::count_launch();
  if (!forced_attempts) {
    cudaMemsetAsync(attempts, 0, (size_t)P * sizeof(int32_t), st);
    cudaMemsetAsync(rej, 0, sizeof(int64_t), st);
    if (prm->total_attempts > 0 && P > 0) {
      int64_t blocks = (prm->total_attempts + 255) / 256;
      if (blocks > 148 * 8) blocks = 148 * 8;
      sw::k_hist_draws_dk<<<(int)blocks, 256, 0, st>>>(prm->total_attempts, keys, (uint64_t)P, attempts, rej); sw::count_launch();
      if (sw::reject_rem((uint64_t)P) != 0) {
        sw::k_hist_fix_dk<<<1, 1, 0, st>>>(prm->total_attempts, keys, (uint64_t)P, attempts, rej); sw::count_launch();
      }
    }
  }
  if (ev_kind) {
    k_copy_i32<<<grid1(P), 256, 0, st>>>(attempts, ev_off, P); sw::count_launch();
    sw::k_scan_excl_i32<<<1, 1024, 0, st>>>(ev_off, P, nullptr); sw::count_launch();
  }
  RwArgs A{*m, weight_plane, attempts, keys, prm->form_lut, prm->dist_lut, prm->side,
           prm->g_theta, prm->p_dep, prm->p_pot, prm->g_init, totals, changed, ev_off, ev_kind, ev_d,
           (int32_t*)prm->scratch, heavy_cap(prm), prm->patch_log, prm->patch_cap, P > 16384 ? 1 : 0};
  if (P > 0) { k_rw_rows<<<grid1(P), 256, 0, st>>>(A); sw::count_launch(); }
  SW_CHECK_LAUNCH("sw_rewire_update");
  return SW_OK;
}

namespace {
__global__ void k_tm_log(const int64_t* update, const int64_t* ta, const int64_t* tb, int64_t* log,
                         int64_t cap) {
  int64_t idx = *update - 1;
  idx = idx < 0 ? 0 : (idx >= cap ? cap - 1 : idx);
  log[idx * 4 + 0] = ta[0];
  log[idx * 4 + 1] = ta[2];
  log[idx * 4 + 2] = tb[0];
  log[idx * 4 + 3] = tb[2];
}
}  // namespace

extern "C" int sw_topomap_log(const int64_t* update_count, const int64_t* totals_a,
                              const int64_t* totals_b, int64_t* log, int64_t cap, void* stream) {
  if (cap <= 0) return SW_OK;
  k_tm_log<<<1, 1, 0, (cudaStream_t)stream>>>(update_count, totals_a, totals_b, log, cap);
  sw::count_launch();
  SW_CHECK_LAUNCH("sw_topomap_log");
  return SW_OK;
}
