// a3+a4 on the 5th-generation tensor cores (tcgen05.mma, accumulators in TMEM).
//
//   logits[b][i][j] = sum_c W[row(ids_b[j])][c] * H[b][i][c]     (Eq. 2 on I)
//
// The paper gathers the active rows into a dense repack buffer on a copy
// stream and then runs a dense GEMM.  Here the gather is fused into
// the contraction's load stage instead: each 128-row tile of active rows is
// pulled straight from W_head with 16-byte cp.async into 128B-swizzled shared
// memory (the UMMA K-major SW128 layout), so the weight bytes cross HBM exactly
// once and no repack buffer is written.
//
// Tile: UMMA M = 128 active rows (A operand), N = NT >= n draft nodes (B
// operand, zero-padded), K = 64 per stage (one 128-byte swizzle atom).  D lives
// in TMEM (NT fp32 columns x 128 lanes).
//
// Work split: T = sum_b ceil(n_active_b / 128) tiles are read from device
// memory (no host sync).  With T < #SMs every tile is split along K into
// S = floor(#SMs / T) uniform chunks (one unit per CTA); partial tiles are
// reduced in a fixed order (split 0, 1, ..., S-1) by the S CTAs of the tile,
// each reducing a slice of its rows, so equal rows give bit-equal logits.  With
// T >= #SMs, S = 1 and CTAs loop over whole tiles.  The kernel is launched
// cooperatively (all CTAs co-resident), which makes the split-K spin-wait safe.
//
// Warp roles (160 threads): warps 0-3 load (cp.async) and run the epilogue
// (tcgen05.ld, one TMEM lane = one active row per thread); warp 4 allocates
// TMEM and one elected lane issues the MMAs.
#include <cuda.h>

#include "common.cuh"
#include "internal.h"

namespace nanospec {

namespace {

constexpr int kBM = 128;          // active rows per tile (UMMA M)
constexpr int kBK = 64;           // K per stage (bf16 -> 128 bytes)
constexpr int kLoadWarps = 4;
constexpr int kThreads = (kLoadWarps + 1) * 32;
constexpr int kSmemBudget = 200 * 1024;
constexpr int kMaxSMs = 256;

struct TcArgs {
  HeadProblem p;
  float* part;          // [units][NT][128] fp32 split-K partials
  unsigned* arrive;     // [max tiles] split-K arrival counters (zero between launches)
  unsigned* done;       // [max tiles]
  int max_tiles;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128B-swizzled UMMA shared-memory descriptor (SM100 format):
// start>>4 [0,14), LBO>>4 [16,30) (unused for SW128 K-major: 1), SBO>>4 [32,46)
// = 1024 B between 8-row groups, version 1 at [46,48), layout SWIZZLE_128B (2)
// at [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, N, M.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t ld_acquire(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------------ work split
struct Split {
  int tiles;  // total row tiles over all sequences
  int S;      // K chunks per tile
  int units;  // tiles * S
};

__device__ __forceinline__ Split compute_split(const HeadProblem& p, int grid, int kb) {
  Split s;
  int t = 0;
  for (int b = 0; b < p.batch; ++b) {
    int m = p.nact_base[(long long)b * p.nact_stride];
    m = m < 0 ? 0 : (m > p.max_ids ? p.max_ids : m);
    t += (m + kBM - 1) / kBM;
  }
  s.tiles = t;
  s.S = t >= grid || t == 0 ? 1 : min(kb, grid / t);
  s.units = t * s.S;
  return s;
}

// tile index -> (sequence, first row, valid rows)
__device__ __forceinline__ void locate_tile(const HeadProblem& p, int tile, int& seq, int& row0, int& rows) {
  int t = tile;
  for (int b = 0; b < p.batch; ++b) {
    int m = p.nact_base[(long long)b * p.nact_stride];
    m = m < 0 ? 0 : (m > p.max_ids ? p.max_ids : m);
    int nt = (m + kBM - 1) / kBM;
    if (t < nt) {
      seq = b;
      row0 = t * kBM;
      rows = min(kBM, m - row0);
      return;
    }
    t -= nt;
  }
  seq = 0;
  row0 = 0;
  rows = 0;
}

template <int NT>
struct Cfg {
  static constexpr int kABytes = kBM * kBK * 2;   // 16 KB
  static constexpr int kBBytes = NT * kBK * 2;    // NT * 128 B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStageBytes) > 8 ? 8 : (kSmemBudget / kStageBytes);
  static constexpr int kTmemCols = NT < 32 ? 32 : NT;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 2048 /*barriers, row table*/;
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) head_tc_kernel(TcArgs a) {
  using C = Cfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* tiles_base = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  // bars[0..S) full, [S..2S) empty, [2S] tmem_full, [2S+1] tmem_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 2);
  const uint16_t** row_ptr = reinterpret_cast<const uint16_t**>(tmem_slot + 2);  // [128]

  const HeadProblem& p = a.p;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int KB = p.d / kBK;

  const Split sp = compute_split(p, gridDim.x, KB);

  if (tid == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(smem_u32(&bars[s]), kLoadWarps * 32);          // full: every loader thread arrives
      mbar_init(smem_u32(&bars[C::kStages + s]), 1);           // empty: one tcgen05.commit
    }
    mbar_init(smem_u32(&bars[2 * C::kStages]), 1);             // tmem_full
    mbar_init(smem_u32(&bars[2 * C::kStages + 1]), kLoadWarps * 32);  // tmem_empty
    fence_proxy_async();
  }
  if (warp == kLoadWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = make_idesc(kBM, NT);

  int it = 0;      // pipeline iteration counter across units (same sequence in every role)
  int local = 0;   // units processed by this CTA
  for (int u = blockIdx.x; u < sp.units; u += gridDim.x, ++local) {
    const int tile = u / sp.S, split = u - (u / sp.S) * sp.S;
    const int kb0 = split * KB / sp.S, kb1 = (split + 1) * KB / sp.S;
    const int nk = kb1 - kb0;
    int seq, row0, rows;
    locate_tile(p, tile, seq, row0, rows);

    if (warp < kLoadWarps) {
      // ---------------- producers: gather rows of W_head + H into SW128 stages
      asm volatile("bar.sync 1, %0;" ::"n"(kLoadWarps * 32));  // previous unit done with row_ptr
      if (tid < kBM) {
        const int j = row0 + tid;
        const uint16_t* rp = nullptr;
        if (tid < rows) {
          const int32_t g = p.ids_base[(long long)seq * p.ids_stride + j];
          const long long r = p.n_shards > 1 ? g / p.n_shards : g;
          rp = p.w + r * p.ldw;
        }
        row_ptr[tid] = rp;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kLoadWarps * 32));
      const uint16_t* hseq = p.h + (long long)seq * p.n * p.d;
      for (int q = 0; q < nk + C::kStages - 1; ++q) {
        if (q < nk) {
          const int g_it = it + q;
          const int stage = g_it % C::kStages;
          if (g_it >= C::kStages) mbar_wait(smem_u32(&bars[C::kStages + stage]), ((g_it / C::kStages) - 1) & 1);
          const uint32_t sA = smem_u32(tiles_base + stage * C::kStageBytes);
          const uint32_t sB = sA + C::kABytes;
          const int kcol = (kb0 + q) * kBK;
#pragma unroll
          for (int i = 0; i < (kBM * 8) / (kLoadWarps * 32); ++i) {
            const int ch = i * (kLoadWarps * 32) + tid;
            const int r = ch >> 3, c = ch & 7;
            const uint16_t* rp = row_ptr[r];
            const uint32_t dst = sA + r * 128 + ((c ^ (r & 7)) << 4);
            cp_async16(dst, rp ? (const void*)(rp + kcol + c * 8) : (const void*)p.w, rp ? 16u : 0u);
          }
#pragma unroll
          for (int i = 0; i < (NT * 8 + kLoadWarps * 32 - 1) / (kLoadWarps * 32); ++i) {
            const int ch = i * (kLoadWarps * 32) + tid;
            if (ch < NT * 8) {
              const int r = ch >> 3, c = ch & 7;
              const bool ok = r < p.n;
              const uint32_t dst = sB + r * 128 + ((c ^ (r & 7)) << 4);
              cp_async16(dst, ok ? (const void*)(hseq + (long long)r * p.d + kcol + c * 8) : (const void*)p.h,
                         ok ? 16u : 0u);
            }
          }
        }
        cp_async_commit();
        if (q >= C::kStages - 1) {
          const int jq = q - (C::kStages - 1);
          cp_async_wait<C::kStages - 1>();
          fence_proxy_async();
          mbar_arrive(smem_u32(&bars[(it + jq) % C::kStages]));
        }
      }
      // ---------------- epilogue: TMEM -> registers -> logits or split-K partials
      mbar_wait(smem_u32(&bars[2 * C::kStages]), local & 1);
      tc_fence_after();
      const int r = warp * 32 + lane;  // TMEM lane == tile row
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < NT && c0 < p.n; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);
        if (sp.S == 1) {
          if (r < rows) {
#pragma unroll
            for (int c = 0; c < 16; ++c)
              if (c0 + c < p.n) p.logits[((long long)seq * p.n + c0 + c) * p.max_ids + row0 + r] = v[c];
          }
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c0 + c < p.n) a.part[((long long)u * NT + c0 + c) * kBM + r] = v[c];
        }
      }
      tc_fence_before();
      mbar_arrive(smem_u32(&bars[2 * C::kStages + 1]));
    } else {
      // ---------------- MMA issuer (warp 4, one lane)
      if (local > 0) {
        mbar_wait(smem_u32(&bars[2 * C::kStages + 1]), (local - 1) & 1);
        tc_fence_after();
      }
      for (int q = 0; q < nk; ++q) {
        const int g_it = it + q;
        const int stage = g_it % C::kStages;
        mbar_wait(smem_u32(&bars[stage]), (g_it / C::kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sA = smem_u32(tiles_base + stage * C::kStageBytes);
          const uint32_t sB = sA + C::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            umma_bf16(tmem, sw128_desc(sA + kk * 32), sw128_desc(sB + kk * 32), idesc, (q | kk) ? 1u : 0u);
          }
          umma_commit(smem_u32(&bars[C::kStages + stage]));
          if (q == nk - 1) umma_commit(smem_u32(&bars[2 * C::kStages]));
        }
        __syncwarp();
      }
    }
    it += nk;

    if (sp.S > 1) {
      // ---------------- fixed-order split-K reduction, distributed over the tile's CTAs
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        atomicAdd(&a.arrive[tile], 1u);
        while (ld_acquire(&a.arrive[tile]) < (unsigned)sp.S) __nanosleep(64);
      }
      __syncthreads();
      const int s0 = split * kBM / sp.S, s1 = (split + 1) * kBM / sp.S;
      const int nr = s1 - s0;
      const int total = nr * p.n;
      for (int idx = tid; idx < total; idx += kThreads) {
        const int c = idx / nr;
        const int rr = s0 + (idx - c * nr);
        if (rr < rows) {
          float acc = 0.f;
          for (int s = 0; s < sp.S; ++s) acc += __ldcg(&a.part[((long long)(tile * sp.S + s) * NT + c) * kBM + rr]);
          p.logits[((long long)seq * p.n + c) * p.max_ids + row0 + rr] = acc;
        }
      }
      __syncthreads();
      if (tid == 0) {
        unsigned old = atomicAdd(&a.done[tile], 1u);
        if (old == (unsigned)sp.S - 1) {
          a.arrive[tile] = 0u;
          a.done[tile] = 0u;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kLoadWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols));
  }
}

template <int NT>
cudaError_t launch_nt(const HeadProblem& p, void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream) {
  using C = Cfg<NT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(head_tc_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = num_sms < kMaxSMs ? num_sms : kMaxSMs;
  TcArgs a;
  a.p = p;
  const int max_tiles = p.batch * ((p.max_ids + kBM - 1) / kBM);
  char* s = (char*)scratch;
  a.arrive = (unsigned*)s;
  a.done = (unsigned*)(s + sizeof(unsigned) * (size_t)max_tiles);
  size_t off = (sizeof(unsigned) * 2 * (size_t)max_tiles + 255) / 256 * 256;
  a.part = (float*)(s + off);
  a.max_tiles = max_tiles;
  if (off + (size_t)kMaxSMs * NT * kBM * sizeof(float) > scratch_bytes) return cudaErrorInvalidValue;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeCooperative;
  attrs[0].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, head_tc_kernel<NT>, a);
}

}  // namespace

size_t head_tc_scratch_bytes(int batch, int max_ids, int n) {
  const size_t max_tiles = (size_t)batch * ((max_ids + kBM - 1) / kBM);
  int nt = n <= 16 ? 16 : n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256;
  return (sizeof(unsigned) * 2 * max_tiles + 255) / 256 * 256 + (size_t)kMaxSMs * nt * kBM * sizeof(float);
}

cudaError_t launch_head_tc(const HeadProblem& p, void* scratch, size_t scratch_bytes, int num_sms,
                           cudaStream_t stream) {
  if (p.d % kBK != 0 || p.n < 1 || p.n > 256 || p.ldw % 8 != 0) return cudaErrorNotSupported;
  if (p.n <= 16) return launch_nt<16>(p, scratch, scratch_bytes, num_sms, stream);
  if (p.n <= 32) return launch_nt<32>(p, scratch, scratch_bytes, num_sms, stream);
  if (p.n <= 64) return launch_nt<64>(p, scratch, scratch_bytes, num_sms, stream);
  if (p.n <= 128) return launch_nt<128>(p, scratch, scratch_bytes, num_sms, stream);
  return launch_nt<256>(p, scratch, scratch_bytes, num_sms, stream);
}

}  // namespace nanospec
