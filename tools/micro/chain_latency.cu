// Kernel-boundary cost in a CUDA graph: a chain of N light kernels (148 CTAs x
// 256 threads, each reading the previous kernel's output), with
//   mode 0: plain stream order, mode 1: PDL (griddepcontrol.wait),
//   mode 2: PDL launch + a release/acquire completion counter instead of the wait.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_latency chain_latency.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void chain_kernel(const float *in, float *out, int *cnt, int k, int mode, int work) {
  if (mode >= 1) asm volatile("griddepcontrol.launch_dependents;" :::);
  if (mode == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (mode == 2 && k > 0) {
    if (threadIdx.x == 0) {
      int v;
      do {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt + k - 1) : "memory");
      } while (v < (int)gridDim.x);
    }
    __syncthreads();
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float v = __ldcg(in + i);
  for (int w = 0; w < work; ++w) v = v * 0.999f + 1.0f;
  __stcg(out + i, v + 1.0f);
  if (mode == 2) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt + k) : "memory");
  }
}

int main(int argc, char **argv) {
  const int N = 200, G = 148, T = 256;
  float *buf[2];
  int *cnt;
  cudaMalloc(&buf[0], G * T * 4);
  cudaMalloc(&buf[1], G * T * 4);
  cudaMemset(buf[0], 0, G * T * 4);
  cudaMalloc(&cnt, N * 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int work : {0, 2000}) {
    for (int mode = 0; mode < 3; ++mode) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      cudaMemsetAsync(cnt, 0, N * 4, st);
      for (int k = 0; k < N; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(T);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = mode >= 1 && k > 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, chain_kernel, (const float *)buf[k & 1], buf[(k + 1) & 1], cnt, k, mode,
                           (k & 1) ? 0 : work);
      }
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st);
      cudaStreamSynchronize(st);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("work %4d (every other kernel) mode %d (%s): %.2f us per kernel  [%s]\n", work, mode,
             mode == 0 ? "stream order" : mode == 1 ? "PDL wait" : "PDL launch + counter", ms * 1e3 / 10 / N,
             cudaGetErrorString(cudaGetLastError()));
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  return 0;
}
