// Library plumbing (error string, ABI version) and the counter-RNG entry points.
#include <cstdio>
#include <cstring>
#include <atomic>
#include "common.cuh"

namespace sw {
static thread_local char g_last_error[512] = "";
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_last_error(const char* msg) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
}

int check_launch(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
    set_last_error(buf);
    return SW_ERR_CUDA;
  }
  return SW_OK;
}
}  // namespace sw

extern "C" int sw_abi_version(void) { return SW_ABI_VERSION; }
extern "C" const char* sw_last_error(void) { return sw::g_last_error; }
extern "C" long long sw_launch_count(void) { return sw::g_launches.load(); }

__global__ void k_rng_selftest(uint64_t* out) {
  out[0] = sw::mix64(0);
  out[1] = sw::mix64(1);
  out[2] = sw::mix64(SW_GOLDEN);
}

extern "C" int sw_rng_selftest(uint64_t* out3, void* stream) {
  k_rng_selftest<<<1, 1, 0, (cudaStream_t)stream>>>(out3); sw::count_launch();
  SW_CHECK_LAUNCH("sw_rng_selftest");
  return SW_OK;
}

__global__ void k_rng_u64(uint64_t key, uint64_t c0, int64_t n, uint64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sw::draw(key, c0 + (uint64_t)i);
}

__global__ void k_rng_u01(uint64_t key, uint64_t c0, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sw::u01(sw::draw(key, c0 + (uint64_t)i));
}

__global__ void k_rng_child(uint64_t key, int64_t n, uint64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sw::child_key(key, (uint64_t)i);
}

__global__ void k_rng_uint_seq(uint64_t key, uint64_t n, int64_t count, uint64_t* out) {
  uint64_t ctr = 0, rem = sw::reject_rem(n);
  for (int64_t i = 0; i < count; ++i) out[i] = sw::uniform_int_seq(key, ctr, n, rem);
  out[count] = ctr;
}

static int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

extern "C" int sw_rng_u64(uint64_t key, uint64_t counter0, int64_t n, uint64_t* out, void* stream) {
  if (n <= 0) return SW_OK;
  k_rng_u64<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(key, counter0, n, out); sw::count_launch();
  SW_CHECK_LAUNCH("sw_rng_u64");
  return SW_OK;
}

extern "C" int sw_rng_uniform01(uint64_t key, uint64_t counter0, int64_t n, double* out, void* stream) {
  if (n <= 0) return SW_OK;
  k_rng_u01<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(key, counter0, n, out); sw::count_launch();
  SW_CHECK_LAUNCH("sw_rng_uniform01");
  return SW_OK;
}

extern "C" int sw_rng_child_keys(uint64_t key, int64_t n, uint64_t* out, void* stream) {
  if (n <= 0) return SW_OK;
  k_rng_child<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(key, n, out); sw::count_launch();
  SW_CHECK_LAUNCH("sw_rng_child_keys");
  return SW_OK;
}

extern "C" int sw_rng_uniform_int_seq(uint64_t key, uint64_t n, int64_t count, uint64_t* out, void* stream) {
  if (n == 0 || count < 0) { sw::set_last_error("uniform_int: n must be positive"); return SW_ERR_INVALID_ARG; }
  k_rng_uint_seq<<<1, 1, 0, (cudaStream_t)stream>>>(key, n, count, out); sw::count_launch();
  SW_CHECK_LAUNCH("sw_rng_uniform_int_seq");
  return SW_OK;
}
