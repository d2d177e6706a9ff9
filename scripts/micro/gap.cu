// Back-to-back dependent kernels in a CUDA graph (B200): time per tiny kernel,
// with and without programmatic dependent launch (PDL).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(int* x, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicAdd(x, 1);
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

int main() {
  int* x; cudaMalloc(&x, 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int blocks : {1, 148}) for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 200; ++i) {
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(512); cfg.stream = s;
      cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      a[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = a; cfg.numAttrs = pdl;
      cudaLaunchKernelEx(&cfg, tiny, x, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("blocks %3d pdl %d: %.2f us per dependent kernel\n", blocks, pdl, ms * 1e3 / 200);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
