// Microbenchmark: u32 atomic-add throughput on B200 for the vote accumulator design.
// Measures (1) shared-memory atomics, random and lane-consecutive addresses,
// (2) global RED into an L2-resident 1 MiB grid, (3) DSMEM atomics to a peer CTA
// of a 2-CTA cluster. Prints one JSON line per case.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int kWords = 47104;  // 184 KB of u32 counters
constexpr int kIters = 4096;

__device__ __forceinline__ uint32_t xs(uint32_t x) {
  x ^= x << 13; x ^= x >> 17; x ^= x << 5; return x;
}

template <int MODE>  // 0 random, 1 consecutive, 2 no atomic (address gen only)
__global__ void __launch_bounds__(1024, 1) smem_atom(uint32_t* out) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t st = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 7919u;
  uint32_t acc = 0;
  #pragma unroll 8
  for (int it = 0; it < kIters; ++it) {
    st = xs(st);
    uint32_t a;
    if (MODE == 1) a = ((it * 1024u + threadIdx.x) * 1u) % kWords;
    else a = st % kWords;
    if (MODE == 2) acc += a;
    else atomicAdd(&s[a], (st >> 31) + 1u);
  }
  __syncthreads();
  uint32_t sum = acc;
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) sum += s[i];
  atomicAdd(out, sum);
}

__global__ void __launch_bounds__(1024, 1) gmem_red(uint32_t* grid, uint32_t* out) {
  uint32_t st = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 7919u;
  #pragma unroll 8
  for (int it = 0; it < kIters / 4; ++it) {
    st = xs(st);
    atomicAdd(&grid[st & (262144 - 1)], (st >> 31) + 1u);
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024, 1) dsmem_atom(uint32_t* out) {
  extern __shared__ uint32_t s[];
  cg::cluster_group cluster = cg::this_cluster();
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) s[i] = 0;
  cluster.sync();
  const unsigned peer = cluster.block_rank() ^ 1u;
  uint32_t* ps = cluster.map_shared_rank(s, peer);
  uint32_t st = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 7919u;
  #pragma unroll 8
  for (int it = 0; it < kIters / 4; ++it) {
    st = xs(st);
    atomicAdd(&ps[st % kWords], (st >> 31) + 1u);
  }
  cluster.sync();
  uint32_t sum = 0;
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) sum += s[i];
  atomicAdd(out, sum);
}

template <typename K>
float time_it(K launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *out, *grid;
  CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&grid, 262144 * 4));
  const size_t smem = kWords * 4;
  CK(cudaFuncSetAttribute(smem_atom<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(smem_atom<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(smem_atom<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(dsmem_atom, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const double n_smem = double(sms) * 1024 * kIters;
  float t0 = time_it([&] { smem_atom<0><<<sms, 1024, smem>>>(out); }, 10);
  CK(cudaGetLastError());
  float t1 = time_it([&] { smem_atom<1><<<sms, 1024, smem>>>(out); }, 10);
  float t2 = time_it([&] { smem_atom<2><<<sms, 1024, smem>>>(out); }, 10);
  const double n_g = double(sms) * 4 * 1024 * (kIters / 4);
  float t3 = time_it([&] { gmem_red<<<sms * 4, 1024>>>(grid, out); }, 10);
  CK(cudaGetLastError());
  const double n_d = double(sms) * 1024 * (kIters / 4);
  float t4 = time_it([&] { dsmem_atom<<<sms, 1024, smem>>>(out); }, 10);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  printf("{\"case\":\"smem_atomic_random\",\"ms\":%.4f,\"atomics_per_s\":%.4e}\n", t0, n_smem / (t0 * 1e-3));
  printf("{\"case\":\"smem_atomic_consecutive\",\"ms\":%.4f,\"atomics_per_s\":%.4e}\n", t1, n_smem / (t1 * 1e-3));
  printf("{\"case\":\"smem_addrgen_only\",\"ms\":%.4f,\"ops_per_s\":%.4e}\n", t2, n_smem / (t2 * 1e-3));
  printf("{\"case\":\"gmem_red_random_1MiB\",\"ms\":%.4f,\"atomics_per_s\":%.4e}\n", t3, n_g / (t3 * 1e-3));
  printf("{\"case\":\"dsmem_atomic_peer_random\",\"ms\":%.4f,\"atomics_per_s\":%.4e}\n", t4, n_d / (t4 * 1e-3));
  return 0;
}
