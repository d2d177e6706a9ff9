// Calibration microbenchmarks (B200): cost of %globaltimer reads, generic vs
// shared loads, and a small smem reduction loop at 544 threads/CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

__global__ void k_timer(unsigned long long* out) {
  unsigned long long c0 = clock64();
  unsigned long long a = gt();
  unsigned long long b = gt();
  unsigned long long c1 = clock64();
  for (int i = 0; i < 10; ++i) b = gt();
  unsigned long long c2 = clock64();
  if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = c2 - c1; out[2] = b - a; }
}

template <bool kGeneric>
__global__ void __launch_bounds__(544, 1) k_loop(float* out, int S, int m, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  float* base;
  if (kGeneric) base = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  else base = reinterpret_cast<float*>(raw);
  for (int i = threadIdx.x; i < 40000; i += blockDim.x) base[i] = i * 0.5f;
  __syncthreads();
  unsigned long long c0 = clock64();
  float acc = 0.f;
  float* vals = base + S * m;
  for (int jj = threadIdx.x; jj < m; jj += blockDim.x) {
    const float* src = base + (jj / 128) * S * 128 + (jj % 128);
    float v = 0.f;
#pragma unroll 8
    for (int s = 0; s < S; ++s) v += src[s * 128];
    vals[jj] = v;
    acc = fmaxf(acc, v);
  }
  __syncthreads();
  unsigned long long c1 = clock64();
  float es = 0.f;
  for (int jj = threadIdx.x; jj < m; jj += blockDim.x) es += expf(vals[jj] - acc);
  __syncthreads();
  unsigned long long c2 = clock64();
  float es2 = 0.f;
  for (int jj = threadIdx.x; jj < m; jj += blockDim.x) es2 += __expf(vals[jj] - acc);
  __syncthreads();
  unsigned long long c3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + es + es2;
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 64 * 8);
  float* o; cudaMalloc(&o, 1 << 20);
  unsigned long long h[8];
  k_timer<<<1, 32>>>(d); cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  k_timer<<<1, 32>>>(d); cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("globaltimer: 2 reads %llu cyc, 10 reads %llu cyc, delta between first two %llu ns\n", h[0], h[1], h[2]);
  cudaFuncSetAttribute(k_loop<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_loop<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int rep = 0; rep < 2; ++rep) {
    k_loop<true><<<1, 544, 180000>>>(o, 6, 3072, d); cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("generic ptr: sum %llu cyc, expf %llu cyc, __expf %llu cyc\n", h[0], h[1], h[2]);
    k_loop<false><<<1, 544, 180000>>>(o, 6, 3072, d); cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("shared ptr : sum %llu cyc, expf %llu cyc, __expf %llu cyc\n", h[0], h[1], h[2]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
