// Per-SM L2 read throughput on B200: G CTAs x 544 threads each read `per_cta`
// bytes of an L2-resident buffer (written just before by all SMs), with
// (0) ld.global.cg float4, all loads of a thread issued before use, (1) the
// same with 4 loads per thread in flight, (2) cp.async 16 B into shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void writer(float4* buf, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    buf[i] = make_float4(i, i + 1, i + 2, i + 3);
}

template <int MODE, int PER>
__global__ void __launch_bounds__(544, 1) reader(const float4* buf, int per_thread, float* out, long long* cyc) {
  extern __shared__ float4 sm[];
  const float4* base = buf + (long long)blockIdx.x * 544 * per_thread;
  long long c0 = clock64();
  float4 acc = make_float4(0, 0, 0, 0);
  if (MODE == 0) {
    float4 x[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) x[i] = __ldcg(base + i * 544 + threadIdx.x);
#pragma unroll
    for (int i = 0; i < PER; ++i) { acc.x += x[i].x; acc.y += x[i].y; }
  } else if (MODE == 1) {
    for (int i0 = 0; i0 < PER; i0 += 4) {
      float4 x[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) x[i] = __ldcg(base + (i0 + i) * 544 + threadIdx.x);
#pragma unroll
      for (int i = 0; i < 4; ++i) { acc.x += x[i].x; acc.y += x[i].y; }
    }
  } else {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      unsigned dst = (unsigned)__cvta_generic_to_shared(sm + i * 544 + threadIdx.x);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(base + i * 544 + threadIdx.x) : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int i = 0; i < PER; ++i) { float4 x = sm[i * 544 + threadIdx.x]; acc.x += x.x; acc.y += x.y; }
  }
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  out[blockIdx.x * 544 + threadIdx.x] = acc.x + acc.y;
}

template <int MODE, int PER>
void run(const float4* buf, float* out, long long* dcyc, int G) {
  cudaFuncSetAttribute(reader<MODE, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  long long h[256];
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9; long long med = 0;
  for (int rep = 0; rep < 5; ++rep) {
    writer<<<592, 256>>>((float4*)buf, 8ll << 20 >> 4);
    cudaEventRecord(e0);
    reader<MODE, PER><<<G, 544, MODE == 2 ? PER * 544 * 16 : 0>>>(buf, PER, out, dcyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
    cudaMemcpy(h, dcyc, G * 8, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < G; ++i) mx = h[i] > mx ? h[i] : mx; med = mx;
  }
  const double bytes = (double)PER * 544 * 16;
  printf("mode %d per-thread %2d  G=%3d  bytes/CTA %6.0f KB  kernel %.2f us  max CTA cycles %lld (%.2f us) -> %.1f GB/s per SM\n",
         MODE, PER, G, bytes / 1024, best * 1e3, med, med / 1.965e3, bytes / (med / 1.965));
}

int main() {
  float4* buf; cudaMalloc(&buf, 8 << 20);
  float* out; cudaMalloc(&out, 256 * 544 * 4);
  long long* dcyc; cudaMalloc(&dcyc, 256 * 8);
  for (int G : {1, 60, 148}) {
    run<0, 8>(buf, out, dcyc, G);
    run<1, 8>(buf, out, dcyc, G);
    run<2, 8>(buf, out, dcyc, G);
    run<0, 4>(buf, out, dcyc, G);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
