// Shared device helpers for the sm_100a structural-plasticity kernels.
//
// RNG: the reference's counter-based SplitMix64 streams
// (sparsewire/rng.py:28-33 mix64, :84-86 child_key, :88-96 draws,
//  :98-104 uniform01, :106-114 uniform_int with exact rejection).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/sparsewire_b200.h"

#define SW_GOLDEN 0x9E3779B97F4A7C15ull
#define SW_CHILD_SALT 0x632BE59BD9B4E019ull
#define SW_FULL_MASK 0xffffffffu

namespace sw {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// draw #c of the stream with key K (rng.py:88-91)
__host__ __device__ __forceinline__ uint64_t draw(uint64_t key, uint64_t c) {
  return mix64(key + c * SW_GOLDEN);
}

__host__ __device__ __forceinline__ uint64_t child_key(uint64_t key, uint64_t idx) {
  return mix64(key ^ mix64(idx + SW_CHILD_SALT));
}

// uniform01 = (h >> 11) * 2^-53, exact in double (rng.py:98-104)
__host__ __device__ __forceinline__ double u01(uint64_t h) {
  return (double)(h >> 11) * 0x1p-53;
}

// uniform_int(n) accepts h < 2^64 - (2^64 mod n) (rng.py:110-114).
// Returns the threshold r = 2^64 mod n; a draw is valid iff r == 0 or h < 2^64 - r.
__host__ __device__ __forceinline__ uint64_t reject_rem(uint64_t n) {
  return (0ull - n) % n;   // (2^64 - n) mod n == 2^64 mod n
}
__host__ __device__ __forceinline__ bool draw_valid(uint64_t h, uint64_t rem) {
  return rem == 0 || h < (0ull - rem);
}

// Sequential uniform_int on a private counter (exact reference semantics).
__device__ __forceinline__ uint64_t uniform_int_seq(uint64_t key, uint64_t& ctr,
                                                    uint64_t n, uint64_t rem) {
  while (true) {
    uint64_t h = draw(key, ctr++);
    if (draw_valid(h, rem)) return h % n;
  }
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// error flag word shared by the kernels of one call (first error wins)
__device__ __forceinline__ void raise_flag(int* flag, int code) {
  if (flag) atomicCAS(flag, 0, code);
}

}  // namespace sw

// ---- host-side error plumbing -------------------------------------------------
namespace sw {
void set_last_error(const char* msg);
int check_launch(const char* where);
void count_launch();
}  // namespace sw

#define SW_CHECK_LAUNCH(name) do { int _s = sw::check_launch(name); if (_s) return _s; } while (0)

// ---- programmatic dependent launch -----------------------------------------
// A kernel launched with pdl_launch may be scheduled while the previous
// kernel in the stream drains; it must call pdl_enter() before touching
// anything that kernel writes (griddepcontrol.wait: the previous grid has
// completed and its memory is visible), and lets its own successor be
// scheduled (launch_dependents).  Without the attribute both are no-ops.
namespace sw {
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(bool on, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}
}  // namespace sw
