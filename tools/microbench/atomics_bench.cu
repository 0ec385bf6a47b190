// Shared-memory atomic throughput of the B200 (the roofline denominator of the vote kernel).
// Built as a shared library (tools/microbench/libsmem_atomics.so); bench.py measures the peak
// live on the box: conflict-free u32 atomicAdd with lane-distinct addresses in one 184 KB
// region per SM, 1024 threads/SM, address generation by a single IADD/LOP per atomic.
// Also a standalone main() for ad-hoc runs (-DSTANDALONE).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace {
constexpr int kWords = 47104;  // 184 KB of u32 counters
constexpr int kIters = 8192;

// lane-distinct, bank-conflict-free addresses: word = (base + it*stride + tid) & mask
__global__ void __launch_bounds__(1024, 1) smem_atom_peak(uint32_t* out, int iters) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const uint32_t mask = 32767;  // 128 KB window inside the region
  uint32_t a = threadIdx.x;
  const uint32_t inc = threadIdx.x & 1 ? 2u : 1u;
#pragma unroll 16
  for (int it = 0; it < iters; ++it) {
    atomicAdd(&s[a], inc);
    a = (a + 1024u + 32u) & mask;
  }
  __syncthreads();
  uint32_t sum = 0;
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) sum += s[i];
  if (sum == 0xFFFFFFFFu) *out = sum;
}
}  // namespace

extern "C" int smem_atomic_peak(int device, double* atomics_per_s, double* ms_out) {
  if (cudaSetDevice(device) != cudaSuccess) return 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  uint32_t* out;
  if (cudaMalloc(&out, 4) != cudaSuccess) return 2;
  const size_t smem = kWords * 4;
  cudaFuncSetAttribute(smem_atom_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) smem_atom_peak<<<sms, 1024, smem>>>(out, kIters);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    smem_atom_peak<<<sms, 1024, smem>>>(out, kIters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (e != cudaSuccess) return 3;
  *atomics_per_s = (double)sms * 1024.0 * kIters / (best * 1e-3);
  *ms_out = best;
  return 0;
}

#ifdef STANDALONE
int main() {
  double r, ms;
  const int st = smem_atomic_peak(0, &r, &ms);
  printf("{\"status\":%d,\"smem_atomics_per_s\":%.4e,\"ms\":%.4f}\n", st, r, ms);
  return st;
}
#endif
