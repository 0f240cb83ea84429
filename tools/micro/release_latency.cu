// PDL release latency after a producer grid that ends with a burst of stores:
// producer (148 CTAs x 192 threads) writes `kb` KB per CTA with st.global.cg
// (as the deferred stream-K GEMM writes its partial slots) and stamps its exit;
// the consumer (256 CTAs, launched with programmatic serialization) stamps after
// griddepcontrol.wait and after its first dependent load.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o release_latency release_latency.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void producer(float *ws, int per_cta_floats, unsigned long long *tm, int mode) {
  asm volatile("griddepcontrol.launch_dependents;" :::);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float *dst = ws + (size_t)blockIdx.x * per_cta_floats;
  for (int i = threadIdx.x; i < per_cta_floats; i += blockDim.x) {
    if (mode == 0) __stcg(dst + i, (float)i);
    else dst[i] = (float)i;
  }
  __syncthreads();
  if (threadIdx.x == 0) tm[blockIdx.x] = gt();
}

__global__ void consumer(const float *ws, int per_cta_floats, unsigned long long *tm) {
  asm volatile("griddepcontrol.launch_dependents;" :::);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const unsigned long long t1 = gt();
  float v = __ldcg(ws + (size_t)(blockIdx.x % 148) * per_cta_floats + threadIdx.x);
  __syncthreads();
  const unsigned long long t2 = gt();
  if (threadIdx.x == 0) {
    tm[2 * blockIdx.x] = t1;
    tm[2 * blockIdx.x + 1] = t2 + (v == -1.f);
  }
}

int main() {
  float *ws;
  unsigned long long *tp, *tc;
  cudaMalloc(&ws, 148 * 64 * 1024);
  cudaMalloc(&tp, 148 * 8);
  cudaMalloc(&tc, 512 * 8);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int mode = 0; mode < 2; ++mode)
    for (int kb : {1, 8, 32, 64}) {
      const int per = kb * 256;
      std::vector<double> rel, rel2;
      for (int rep = 0; rep < 6; ++rep) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.stream = st;
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(192);
        cudaLaunchKernelEx(&cfg, producer, ws, per, tp, mode);
        cfg.gridDim = dim3(256);
        cfg.blockDim = dim3(128);
        cudaLaunchKernelEx(&cfg, consumer, (const float *)ws, per, tc);
        cudaStreamSynchronize(st);
        std::vector<unsigned long long> hp(148), hc(512);
        cudaMemcpy(hp.data(), tp, 148 * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hc.data(), tc, 512 * 8, cudaMemcpyDeviceToHost);
        const unsigned long long pend = *std::max_element(hp.begin(), hp.end());
        unsigned long long w = ~0ull, l = 0;
        for (int c = 0; c < 256; ++c) {
          w = std::min(w, hc[2 * c]);
          l = std::max(l, hc[2 * c + 1]);
        }
        if (rep >= 2) {
          rel.push_back(((double)w - (double)pend) / 1e3);
          rel2.push_back(((double)l - (double)pend) / 1e3);
        }
      }
      printf("%s %3d KB/CTA (%5.1f MB): consumer wait passed %+.2f us, first load done (max) %+.2f us after producer end\n",
             mode ? "st     " : "st.cg  ", kb, 148.0 * kb / 1024, rel[rel.size() / 2], rel2[rel2.size() / 2]);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
