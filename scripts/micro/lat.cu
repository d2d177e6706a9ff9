// Latency probes on B200: dependent global loads (L2-resident data written by
// other SMs), CREDUX round trip, shuffle round trip.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void writer(unsigned* buf, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) buf[i] = (unsigned)(((long long)i * 7919 + 13) % n);
}

__global__ void probe(const unsigned* buf, unsigned long long* out, int n) {
  if (blockIdx.x != 0) return;
  const int lane = threadIdx.x & 31;
  unsigned x = lane;
  // 1. dependent __ldcg chain (L2 hits)
  long long c0 = clock64();
  for (int i = 0; i < 64; ++i) x = __ldcg(buf + x);
  long long c1 = clock64();
  // 2. dependent __ldg chain
  for (int i = 0; i < 64; ++i) x = __ldg(buf + (x ^ 1u) % n);
  long long c2 = clock64();
  // 3. CREDUX chain
  unsigned y = x;
  for (int i = 0; i < 64; ++i) y = __reduce_max_sync(0xffffffffu, y + lane) - lane;
  long long c3 = clock64();
  // 4. shuffle chain
  for (int i = 0; i < 64; ++i) y = __shfl_xor_sync(0xffffffffu, y, 1 + (i & 15)) + 1;
  long long c4 = clock64();
  // 5. dependent LDS chain
  __shared__ unsigned s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 31 + 7) & 1023;
  __syncwarp();
  unsigned z = lane;
  long long c5 = clock64();
  for (int i = 0; i < 64; ++i) z = s[z];
  long long c6 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (c1 - c0) / 64; out[1] = (c2 - c1) / 64; out[2] = (c3 - c2) / 64; out[3] = (c4 - c3) / 64;
    out[4] = (c6 - c5) / 64; out[5] = x + y + z;
  }
}

int main() {
  const int n = 1 << 24;  // 64 MB: L2 resident
  unsigned* buf; cudaMalloc(&buf, n * 4ull);
  unsigned long long* d; cudaMalloc(&d, 64);
  unsigned long long h[6];
  for (int rep = 0; rep < 3; ++rep) {
    writer<<<148 * 4, 256>>>(buf, n);
    probe<<<1, 32>>>(buf, d, n);
    cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: ldcg(L2) %llu  ldg %llu  credux %llu  shfl %llu  lds %llu\n", h[0], h[1], h[2], h[3], h[4]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
