// Same-kernel write -> grid barrier -> read of another SM's fresh data (B200).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}

template <int WMODE>
__global__ void __launch_bounds__(544, 1) rw(float4* buf, unsigned* ctr, int per, long long* cyc, float* out) {
  const int G = gridDim.x;
  float4* mine = buf + (long long)blockIdx.x * 544 * per;
  for (int i = 0; i < per; ++i) {
    float4 v = make_float4(i, blockIdx.x, threadIdx.x, 1.f);
    if (WMODE == 0) __stcg(mine + i * 544 + threadIdx.x, v);
    else mine[i * 544 + threadIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(ctr, 1u);
    while (ld_acq(ctr) < (unsigned)G) __nanosleep(32);
  }
  __syncthreads();
  long long c0 = clock64();
  const float4* other = buf + (long long)((blockIdx.x + 37) % G) * 544 * per;
  float4 x[8];
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) if (i < per) x[i] = __ldcg(other + i * 544 + threadIdx.x);
#pragma unroll
  for (int i = 0; i < 8; ++i) if (i < per) acc += x[i].x + x[i].y;
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  out[blockIdx.x * 544 + threadIdx.x] = acc;
}

int main() {
  float4* buf; cudaMalloc(&buf, 16 << 20);
  unsigned* ctr; cudaMalloc(&ctr, 4);
  long long* cyc; cudaMalloc(&cyc, 256 * 8);
  float* out; cudaMalloc(&out, 256 * 544 * 4);
  long long h[256];
  for (int wm = 0; wm < 2; ++wm)
    for (int G : {60, 148}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(ctr, 0, 4);
        if (wm == 0) rw<0><<<G, 544>>>(buf, ctr, 8, cyc, out); else rw<1><<<G, 544>>>(buf, ctr, 8, cyc, out);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, cyc, G * 8, cudaMemcpyDeviceToHost);
      long long mx = 0, mn = 1ll << 60; for (int i = 0; i < G; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
      printf("store %s G=%3d: read-after-barrier of 68 KB/CTA: min %lld max %lld cycles (%.2f us)\n",
             wm == 0 ? "st.cg" : "st   ", G, mn, mx, mx / 1.965e3);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
