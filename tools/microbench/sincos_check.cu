// Dev check: CUDA sincos() is bit-identical to sin() and cos() on [-pi, pi] (peak_angle_kernel
// relies on it). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ../_bin/sincos_check sincos_check.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
__global__ void k(const double* x, int n, unsigned long long* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s1 = sin(x[i]), c1 = cos(x[i]), s2, c2;
  sincos(x[i], &s2, &c2);
  if (__double_as_longlong(s1) != __double_as_longlong(s2) || __double_as_longlong(c1) != __double_as_longlong(c2)) atomicAdd(bad, 1ull);
}
int main() {
  const int n = 1 << 24;
  double* h = new double[n];
  uint64_t st = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; h[i] = -M_PI + 2 * M_PI * ((st >> 11) * (1.0 / 9007199254740992.0)); }
  h[0] = M_PI; h[1] = -M_PI; h[2] = 0.0; h[3] = M_PI / 2;
  double* d; unsigned long long* b; cudaMalloc(&d, n * 8); cudaMalloc(&b, 8); cudaMemset(b, 0, 8);
  cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(d, n, b);
  unsigned long long hb; cudaMemcpy(&hb, b, 8, cudaMemcpyDeviceToHost);
  printf("sincos vs sin/cos mismatches: %llu of %d\n", hb, n);
  return 0;
}
