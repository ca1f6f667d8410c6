// Small shared device kernels: single-block exclusive scan and the
// "host-phase" histogram of D uniform_int draws (deep_r.py:119-120,
// topomap.py:104-105: counters 0..D-1 of one stream, rejected draws
// replayed serially past D so exactly the first D valid draws count).
#pragma once
#include "common.cuh"

namespace sw {

// single-block exclusive scan of n int32 (in place); *total = sum
__global__ void k_scan_excl_i32(int32_t* a, int n, int32_t* total);

// histogram of D draws of uniform_int(P) on stream `key`; rejected draws
// are counted in *rej (device) and replayed by k_hist_fix
__global__ void k_hist_draws(int64_t D, uint64_t key, uint64_t P, uint64_t rem, int32_t* act,
                             int64_t* rej);
__global__ void k_hist_fix(int64_t D, uint64_t key, uint64_t P, uint64_t rem, int32_t* act,
                           const int64_t* rej);

// fold one integer part into a key (rng.py:60)
__host__ __device__ __forceinline__ uint64_t fold_int(uint64_t acc, uint64_t part) {
  return mix64(acc ^ mix64(part + 0x9Eull));
}

}  // namespace sw

namespace sw {
// k_hist_draws with the stream key read from device memory
__global__ void k_hist_draws_dk(int64_t D, const uint64_t* key, uint64_t P, int32_t* act, int64_t* rej);
__global__ void k_hist_fix_dk(int64_t D, const uint64_t* key, uint64_t P, int32_t* act, const int64_t* rej);
}  // namespace sw
