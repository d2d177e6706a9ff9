// Cold-HBM gather of |I| = 3072 random 8 KB rows of a 128256 x 4096 bf16
// matrix (the Llama head's active rows, 25.2 MB) into shared memory, B200:
// which load path and which work split reach the HBM roofline?
//   M0 cp.async 16 B, K-split (24 tiles of 128 rows x S splits), 8-stage ring
//   M1 TMA tile::gather4 (SW128), K-split, 8-stage ring, one issuing thread
//   M2 TMA tile::gather4, row split (148 CTAs x ~21 full rows), all in flight
//   M3 LDG.128 to registers, row split, all in flight
//   M4 cp.async.bulk (1-D, 8 KB per row), row split, all in flight
//   M5 cp.async 16 B, row split, all in flight
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather gather.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

constexpr int V = 128256, D = 4096, M = 3072;
constexpr int kThreads = 512;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t par) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(done) : "r"(b), "r"(par) : "memory");
  } while (!done);
}
__device__ __forceinline__ void g4(uint32_t dst, const CUtensorMap* tm, int col, int r0, int r1, int r2, int r3,
                                   uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(dst), "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar) : "memory");
}

struct Args {
  const uint16_t* w;
  const int* ids;   // this launch's id set
  int S;
  float* sink;
  unsigned long long* t;  // per-CTA end time
};

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) gather_kernel(Args a, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (sa(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bars[16];
  __shared__ int rid[256];
  const int tid = threadIdx.x;
  float acc = 0.f;
  if (tid == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    a.t[512 + blockIdx.x] = t0;
  }
  if (MODE == 9) {
  } else if (MODE == 10 || MODE == 11) {
    // the head's stage pattern: UT tiles of 128 rows x a K chunk, plus 60 hidden-state
    // rows (64-row stage, 4 zero-filled) from a small L2-resident H, 8-stage budget of 192 KB
    constexpr int UT = MODE == 11 ? 2 : 1;
    constexpr int kStage = UT * 16384 + 8192;
    constexpr int kSt = (196608 / kStage) > 8 ? 8 : 196608 / kStage;
    const int unit = blockIdx.x / a.S, split = blockIdx.x % a.S;
    const int KB = D / 64, kb0 = split * KB / a.S, kb1 = (split + 1) * KB / a.S, nk = kb1 - kb0;
    if (tid < 128 * UT) rid[tid] = a.ids[unit * 128 * UT + tid];
    __syncthreads();
    const int lr = tid >> 3;
    const int swz = ((tid & 7) ^ (lr & 7)) << 4;
    const uint16_t* hbase = a.w + (long long)(V - 64) * D;  // H: 60 rows near the end of W (L2-resident after the first CTAs)
    for (int q = 0; q < nk; ++q) {
      const uint32_t st = sa(sm + (q % kSt) * kStage);
      const int col = (kb0 + q) * 64;
#pragma unroll
      for (int i = 0; i < 2 * UT; ++i) {
        const int ur = (i >> 1) * 128 + lr + 64 * (i & 1);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + (i >> 1) * 16384 + (lr + 64 * (i & 1)) * 128 + swz),
                     "l"(a.w + (long long)rid[ur] * D + (tid & 7) * 8 + col) : "memory");
      }
      if (lr < 64)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(st + UT * 16384 + lr * 128 + swz),
                     "l"(hbase + (long long)lr * D + (tid & 7) * 8 + col), "r"(lr < 60 ? 16 : 0) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(kSt - 1) : "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    acc = reinterpret_cast<float*>(sm)[tid];
  } else if (MODE == 8) {
    // K-split, M0's lane mapping (8 threads per 128-B row piece), every stage in flight at once
    const int tile = blockIdx.x / a.S, split = blockIdx.x % a.S;
    const int KB = D / 64, kb0 = split * KB / a.S, kb1 = (split + 1) * KB / a.S, nk = kb1 - kb0;
    if (tid < 128) rid[tid] = a.ids[tile * 128 + tid];
    __syncthreads();
    const int lr = tid >> 3;
    const int swz = ((tid & 7) ^ (lr & 7)) << 4;
    const uint16_t* rp0 = a.w + (long long)rid[lr] * D + (tid & 7) * 8;
    const uint16_t* rp1 = a.w + (long long)rid[lr + 64] * D + (tid & 7) * 8;
    for (int q = 0; q < nk; ++q) {
      const uint32_t st = sa(sm + q * 16384);
      const int col = (kb0 + q) * 64;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + lr * 128 + swz), "l"(rp0 + col) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + (lr + 64) * 128 + swz), "l"(rp1 + col) : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    acc = reinterpret_cast<float*>(sm)[tid];
  } else if (MODE == 6 || MODE == 7) {
    // K-split, 128 rows x [kb0, kb1): M6 ring of 4 x 32 KB stages (256 B per row per stage,
    // 64 B contiguous per thread); M7 everything in flight at once (up to 13 K-blocks = 208 KB)
    const int tile = blockIdx.x / a.S, split = blockIdx.x % a.S;
    const int KB = D / 64, kb0 = split * KB / a.S, kb1 = (split + 1) * KB / a.S, nk = kb1 - kb0;
    if (tid < 128) rid[tid] = a.ids[tile * 128 + tid];
    __syncthreads();
    const int r = tid >> 2, cg = (tid & 3) * 4;  // row, first of 4 chunks within a 256-B (2-block) span
    const uint16_t* rp = a.w + (long long)rid[r] * D;
    for (int q = 0; q < nk; q += 2) {
      const int stage = MODE == 6 ? (q / 2) % 4 : q / 2;
      const uint32_t st = sa(sm + stage * 32768);
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int c = cg + c4, blk = c >> 3, ch = c & 7;
        if (q + blk < nk) {
          const uint32_t dst = st + blk * 16384 + r * 128 + ((ch ^ (r & 7)) << 4);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(rp + (kb0 + q + blk) * 64 + ch * 8) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (MODE == 6) asm volatile("cp.async.wait_group 3;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    acc = reinterpret_cast<float*>(sm)[tid];
  } else if (MODE == 0 || MODE == 1) {
    const int tile = blockIdx.x / a.S, split = blockIdx.x % a.S;
    const int KB = D / 64, kb0 = split * KB / a.S, kb1 = (split + 1) * KB / a.S, nk = kb1 - kb0;
    if (tid < 128) rid[tid] = a.ids[tile * 128 + tid];
    if (tid == 0) {
      for (int s = 0; s < 8; ++s) mbar_init(sa(&bars[s]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (MODE == 0) {
      const int lr = tid >> 3;
      const int swz = ((tid & 7) ^ (lr & 7)) << 4;
      const uint16_t* rp0 = a.w + (long long)rid[lr] * D + (tid & 7) * 8;
      const uint16_t* rp1 = a.w + (long long)rid[lr + 64] * D + (tid & 7) * 8;
      for (int q = 0; q < nk; ++q) {
        const uint32_t st = sa(sm + (q % 8) * 16384);
        const int col = (kb0 + q) * 64;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + lr * 128 + swz), "l"(rp0 + col) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + (lr + 64) * 128 + swz), "l"(rp1 + col) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 7;" ::: "memory");
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      acc = reinterpret_cast<float*>(sm)[tid];
    } else {
      if (tid == 0) {
        for (int q = 0; q < nk; ++q) {
          const int s = q % 8;
          if (q >= 8) mbar_wait(sa(&bars[s]), ((q / 8) - 1) & 1);
          const uint32_t st = sa(sm + s * 16384);
          mbar_expect(sa(&bars[s]), 16384);
          const int col = (kb0 + q) * 64;
          for (int r = 0; r < 128; r += 4)
            g4(st + r * 128, &tm, col, rid[r], rid[r + 1], rid[r + 2], rid[r + 3], sa(&bars[s]));
        }
        for (int q = nk - 8 > 0 ? nk - 8 : 0; q < nk; ++q) mbar_wait(sa(&bars[q % 8]), (q / 8) & 1);
      }
      __syncthreads();
      acc = reinterpret_cast<float*>(sm)[tid];
    }
  } else {
    // row split: CTA c owns rows [c*M/G, (c+1)*M/G)
    const int G = gridDim.x;
    const int r0 = (int)((long long)blockIdx.x * M / G), r1 = (int)((long long)(blockIdx.x + 1) * M / G);
    const int nr = r1 - r0;  // 20 or 21
    if (tid < 24) rid[tid] = a.ids[r0 + (tid < nr ? tid : nr - 1)];
    if (tid == 0) {
      mbar_init(sa(&bars[0]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (MODE == 2) {
      if (tid == 0) {
        const int ng = (nr + 3) / 4;  // gather4 groups
        mbar_expect(sa(&bars[0]), ng * 4 * D * 2);
        for (int kb = 0; kb < D / 64; ++kb)
          for (int gq = 0; gq < ng; ++gq)
            g4(sa(sm + kb * (24 * 128) + gq * 512), &tm, kb * 64, rid[4 * gq], rid[4 * gq + 1], rid[4 * gq + 2],
               rid[4 * gq + 3], sa(&bars[0]));
        mbar_wait(sa(&bars[0]), 0);
      }
      __syncthreads();
      acc = reinterpret_cast<float*>(sm)[tid];
    } else if (MODE == 3) {
      // 21 rows x 512 chunks of 16 B: chunk c of row r
      uint4 x[21];
#pragma unroll
      for (int i = 0; i < 21; ++i) {
        const int r = i < nr ? i : nr - 1;
        x[i] = __ldcs(reinterpret_cast<const uint4*>(a.w + (long long)rid[r] * D) + tid);
      }
#pragma unroll
      for (int i = 0; i < 21; ++i) acc += __uint_as_float(x[i].x ^ x[i].w);
    } else if (MODE == 4) {
      if (tid == 0) {
        mbar_expect(sa(&bars[0]), nr * D * 2);
        for (int r = 0; r < nr; ++r)
          asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(sa(sm + r * D * 2)), "l"(a.w + (long long)rid[r] * D), "r"(D * 2), "r"(sa(&bars[0]))
                       : "memory");
        mbar_wait(sa(&bars[0]), 0);
      }
      __syncthreads();
      acc = reinterpret_cast<float*>(sm)[tid];
    } else {
      for (int r = 0; r < nr; ++r)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(sm + r * D * 2 + tid * 16)),
                     "l"(a.w + (long long)rid[r] * D + tid * 8) : "memory");
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      acc = reinterpret_cast<float*>(sm)[tid];
    }
  }
  if (acc == 1234.5f) a.sink[tid] = acc;
  __syncthreads();
  if (tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.t[blockIdx.x] = t;
  }
}

__global__ void flush_kernel(uint4* p, long long n, int v) {
  // read-only flush: evicts L2 with clean lines (a write flush leaves dirty lines whose
  // write-back would be charged to the next kernel)
  unsigned acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc ^= __ldcg(p + i).x;
  if (acc == 0x12345678u + v) p[0].y = acc;
}
__global__ void empty_kernel(Args a) {
  if (a.sink == nullptr && threadIdx.x == 9999) a.t[0] = 0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  uint16_t* w;
  cudaMalloc(&w, (size_t)V * D * 2);
  cudaMemset(w, 0x3c, (size_t)V * D * 2);
  std::vector<int> perm(V);  // first R*M entries: R disjoint id sets
  for (int i = 0; i < V; ++i) perm[i] = i;
  std::mt19937 rng(1);
  std::shuffle(perm.begin(), perm.end(), rng);
  int* ids;
  constexpr int R = 24;  // disjoint id sets, rotated in the graph runs
  cudaMalloc(&ids, (size_t)R * M * 4);
  cudaMemcpy(ids, perm.data(), (size_t)R * M * 4, cudaMemcpyHostToDevice);
  uint4* fl;
  const long long fl_n = (512ll << 20) / 16;
  cudaMalloc(&fl, fl_n * 16);
  float* sink;
  cudaMalloc(&sink, 4096);
  unsigned long long* t;
  cudaMalloc(&t, 1024 * 8);

  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)V};
  cuuint64_t gstr[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("tensor map encode: %d\n", (int)cr);

  Args a{w, ids, 6, sink, t};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int grid, int smem, int S, bool cold) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    a.S = S;
    std::vector<float> ms;
    for (int rep = 0; rep < 25; ++rep) {
      if (cold) flush_kernel<<<592, 512>>>(fl, fl_n, rep);
      cudaEventRecord(e0);
      kern<<<grid, kThreads, smem>>>(a, tm);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float x;
      cudaEventElapsedTime(&x, e0, e1);
      if (rep >= 3) ms.push_back(x * 1e3f);
    }
    std::sort(ms.begin(), ms.end());
    cudaError_t err = cudaGetLastError();
    std::vector<unsigned long long> h(1024);
    cudaMemcpy(h.data(), t, 1024 * 8, cudaMemcpyDeviceToHost);
    unsigned long long s0 = ~0ull, e1m = 0;
    for (int i = 0; i < grid; ++i) { s0 = std::min(s0, h[512 + i]); e1m = std::max(e1m, h[i]); }
    const double span = (e1m - s0) * 1e-3;
    // graph: 48 launches over 24 disjoint id sets (cold by rotation), with PDL
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t gr; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 48; ++i) {
      Args b = a; b.ids = ids + (size_t)(i % R) * M;
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem; cfg.stream = s;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kern, b, tm);
    }
    cudaStreamEndCapture(s, &gr);
    cudaGraphInstantiate(&ge, gr, 0);
    std::vector<float> gm;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
      float x; cudaEventElapsedTime(&x, e0, e1); gm.push_back(x * 1e3f / 48);
    }
    std::sort(gm.begin(), gm.end());
    printf("%-30s grid %3d S %d %s: event med %6.2f us | in-kernel span %6.2f us (%5.0f GB/s) | graph %6.2f us/launch (%5.0f GB/s) %s\n",
           name, grid, S, cold ? "cold" : "warm", ms[ms.size() / 2], span, (double)M * D * 2 / (span * 1e3), gm[3],
           (double)M * D * 2 / (gm[3] * 1e3), err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaGraphExecDestroy(ge); cudaGraphDestroy(gr); cudaStreamDestroy(s);
  };
  {
    std::vector<float> ms;
    for (int rep = 0; rep < 25; ++rep) {
      cudaEventRecord(e0);
      empty_kernel<<<148, kThreads, 200 * 1024>>>(a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float x;
      cudaEventElapsedTime(&x, e0, e1);
      ms.push_back(x * 1e3f);
    }
    std::sort(ms.begin(), ms.end());
    printf("empty kernel 148 CTAs: med %.2f us\n", ms[12]);
  }
  run("M9 empty (launch floor)", gather_kernel<9>, 148, 200 * 1024, 1, true);
  for (int cold = 1; cold >= 0; --cold) {
    for (int S : {5}) {
      run("M0 cp.async k-split ring", gather_kernel<0>, 24 * S, 8 * 16384 + 1024, S, cold);
      run("M1 tma gather4 k-split ring", gather_kernel<1>, 24 * S, 8 * 16384 + 1024, S, cold);
    }
    run("M8 cp.async k-split ALL in flight", gather_kernel<8>, 120, 13 * 16384 + 1024, 5, cold);
    run("M10 head pattern +H, 24x5", gather_kernel<10>, 120, 196608 + 1024, 5, cold);
    run("M10 head pattern +H, 24x6", gather_kernel<10>, 144, 196608 + 1024, 6, cold);
    run("M11 head pattern +H, 2 tiles/CTA, 12x8", gather_kernel<11>, 96, 196608 + 1024, 8, cold);
    run("M11 head pattern +H, 2 tiles/CTA, 12x12", gather_kernel<11>, 144, 196608 + 1024, 12, cold);
    run("M6 cp.async k-split ring4x32K", gather_kernel<6>, 120, 4 * 32768 + 1024, 5, cold);
    run("M7 cp.async k-split all-in-flight", gather_kernel<7>, 120, 7 * 32768 + 1024, 5, cold);
    run("M2 tma gather4 row-split", gather_kernel<2>, 148, 64 * 24 * 128 + 1024, 1, cold);
    run("M3 ldg.128 row-split", gather_kernel<3>, 148, 1024, 1, cold);
    run("M4 bulk 1-D rows row-split", gather_kernel<4>, 148, 21 * 8192 + 1024, 1, cold);
    run("M5 cp.async row-split", gather_kernel<5>, 148, 21 * 8192 + 1024, 1, cold);
    if (!cold) break;
  }
  // the same K-split gathers with every 3072-id set sorted ascending (the slot
  // table's order after init): a 128-row tile then spans ~1/24 of the vocabulary
  for (int r = 0; r < R; ++r) std::sort(perm.begin() + (size_t)r * M, perm.begin() + (size_t)(r + 1) * M);
  cudaMemcpy(ids, perm.data(), (size_t)R * M * 4, cudaMemcpyHostToDevice);
  run("M0 ring, SORTED ids", gather_kernel<0>, 120, 8 * 16384 + 1024, 5, true);
  run("M8 all in flight, SORTED ids", gather_kernel<8>, 120, 13 * 16384 + 1024, 5, true);
  run("M5 row-split, SORTED ids", gather_kernel<5>, 148, 21 * 8192 + 1024, 1, true);
  return 0;
}
