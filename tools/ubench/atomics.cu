// Throughput probes for the propagation design (not product code):
// global f64 RED to random addresses in a 512 KB output, shared-memory f64
// atomics, DSMEM (cluster) f64 red, non-atomic smem RMW.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

__global__ void k_red_global(double* out, int n_per_thread, int mask) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < n_per_thread; ++k) { s = hsh(s + k); atomicAdd(out + (s & mask), 1.0); }
}
__global__ void k_red_global_f32(float* out, int n_per_thread, int mask) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < n_per_thread; ++k) { s = hsh(s + k); atomicAdd(out + (s & mask), 1.0f); }
}
__global__ void k_atom_smem(double* out, int n_per_thread) {
  extern __shared__ double acc[];   // 16384 doubles
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < n_per_thread; ++k) { s = hsh(s + k); atomicAdd(acc + (s & 16383), 1.0); }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = acc[0];
}
__global__ void k_atom_smem_u64(unsigned long long* out, int n_per_thread) {
  extern __shared__ unsigned long long acu[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) acu[i] = 0;
  __syncthreads();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < n_per_thread; ++k) { s = hsh(s + k); atomicAdd(acu + (s & 16383), 1ull); }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = acu[0];
}
// non-atomic RMW where each warp owns a disjoint smem slice (upper bound for owner-computes)
__global__ void k_rmw_smem(double* out, int n_per_thread) {
  extern __shared__ double acc[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* my = acc + w * 512;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < n_per_thread; ++k) { s = hsh(s + k); int a = ((s & 15) << 5) | lane; my[a] += 1.0; }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = acc[0];
}
__global__ void __cluster_dims__(4, 1, 1) k_dsmem_red(double* out, int n_per_thread) {
  extern __shared__ double acc[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) acc[i] = 0;
  cl.sync();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < n_per_thread; ++k) {
    s = hsh(s + k);
    double* remote = cl.map_shared_rank(acc, (s >> 14) & 3);
    atomicAdd(remote + (s & 16383), 1.0);
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = acc[0];
}

int main() {
  double* out; cudaMalloc(&out, 1 << 24); cudaMemset(out, 0, 1 << 24);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 4, threads = 512, npt = 256;
  const double total = (double)blocks * threads * npt;
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    cudaError_t e = cudaGetLastError();
    printf("%-28s %8.3f ms  %8.1f G ops/s  %s\n", name, ms, total / (ms * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
  };
  run("red.global.f64 64K", [&] { k_red_global<<<blocks, threads>>>(out, npt, 65535); });
  run("red.global.f64 1M", [&] { k_red_global<<<blocks, threads>>>(out, npt, (1 << 20) - 1); });
  run("red.global.f32 64K", [&] { k_red_global_f32<<<blocks, threads>>>((float*)out, npt, 65535); });
  cudaFuncSetAttribute(k_atom_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k_atom_smem_u64, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k_rmw_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k_dsmem_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  run("atom.shared.f64 16K", [&] { k_atom_smem<<<148, 1024, 131072>>>(out, npt * 2); });
  run("atom.shared.u64 16K", [&] { k_atom_smem_u64<<<148, 1024, 131072>>>((unsigned long long*)out, npt * 2); });
  run("smem RMW owned", [&] { k_rmw_smem<<<148, 1024, 131072>>>(out, npt * 2); });
  run("dsmem red.f64 cluster4", [&] { k_dsmem_red<<<148, 1024, 131072>>>(out, npt * 2); });
  return 0;
}
