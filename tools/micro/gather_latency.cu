// L2 gather cost: 256 CTAs x 128 threads each sum NL independent 4-byte (or
// 16-byte) loads from a 5 MB fp32 buffer resident in L2, as the deferred
// split-K consumers do. Per-CTA time from globaltimer, median over CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_latency gather_latency.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// the deferred split-K slot layout [slot][token][128]: thread reads slot 2k of token b (blockIdx % 32),
// SLOT_MAJOR = 0: the alternative [token][slot][128]
template <int NL, int SLOT_MAJOR>
__global__ void gather_slots(const float *ws, float *out, unsigned long long *tm) {
  __syncthreads();
  const unsigned long long t0 = gt();
  const int i = threadIdx.x & 63, b = blockIdx.x % 32, h = threadIdx.x >> 6;
  float f[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const int slot = 2 * (k + 9 * h + (blockIdx.x / 32) * 3);
    const size_t row = SLOT_MAJOR ? (size_t)slot * 32 + b : (size_t)b * 296 + slot;
    f[k] = __ldcg(ws + row * 128 + i);
  }
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < NL; ++k) acc += f[k];
  __syncthreads();
  const unsigned long long t1 = gt();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) tm[blockIdx.x] = t1 - t0;
}

template <int NL, int SM>
void run_slots(float *ws, float *out, unsigned long long *tm) {
  for (int rep = 0; rep < 3; ++rep) gather_slots<NL, SM><<<256, 128>>>(ws, out, tm);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(256);
  cudaMemcpy(h.data(), tm, 256 * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  printf("slots %s NL=%3d: median %.2f us, max %.2f us\n", SM ? "[slot][token][128]" : "[token][slot][128]", NL,
         h[128] / 1e3, h[255] / 1e3);
}

template <int NL, int MODE>  // MODE 0: ld.cg 4 B, 1: ld (default) 4 B, 2: ld.cg 16 B (NL / 4 loads)
__global__ void gather(const float *ws, float *out, unsigned long long *tm, int stride) {
  __syncthreads();
  const unsigned long long t0 = gt();
  const int i = threadIdx.x & 63;
  float acc = 0.f;
  if (MODE == 2) {
    float4 f[NL / 4];
#pragma unroll
    for (int k = 0; k < NL / 4; ++k)
      f[k] = __ldcg(reinterpret_cast<const float4 *>(ws + (size_t)((blockIdx.x * 7 + k * 131) % 4096) * stride) + i);
#pragma unroll
    for (int k = 0; k < NL / 4; ++k) acc += f[k].x + f[k].y + f[k].z + f[k].w;
  } else {
    float f[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const float *src = ws + (size_t)((blockIdx.x * 7 + k * 131) % 4096) * stride + i;
      f[k] = MODE == 0 ? __ldcg(src) : *src;
    }
#pragma unroll
    for (int k = 0; k < NL; ++k) acc += f[k];
  }
  __syncthreads();
  const unsigned long long t1 = gt();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) tm[blockIdx.x] = t1 - t0;
}

// the producer: 148 CTAs write the buffer with st.cg (as the stream-K GEMM writes its partial slots)
__global__ void produce(float *ws, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) __stcg(ws + i, (float)i);
}

template <int NL, int MODE>
void run_after_write(float *ws, float *out, unsigned long long *tm, const char *name) {
  for (int rep = 0; rep < 3; ++rep) {
    produce<<<148, 256>>>(ws, 4096 * 320);
    gather<NL, MODE><<<256, 128>>>(ws, out, tm, 320);
  }
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(256);
  cudaMemcpy(h.data(), tm, 256 * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  printf("%-14s NL=%3d after a st.cg producer: median %.2f us, max %.2f us\n", name, NL, h[128] / 1e3, h[255] / 1e3);
}

template <int NL, int MODE>
void run(const float *ws, float *out, unsigned long long *tm, const char *name) {
  for (int rep = 0; rep < 3; ++rep) gather<NL, MODE><<<256, 128>>>(ws, out, tm, 320);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(256);
  cudaMemcpy(h.data(), tm, 256 * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  printf("%-14s NL=%3d: median %.2f us, max %.2f us\n", name, NL, h[128] / 1e3, h[255] / 1e3);
}

int main() {
  float *ws, *out;
  unsigned long long *tm;
  cudaMalloc(&ws, 4096 * 320 * 4 + 4096);
  cudaMemset(ws, 0, 4096 * 320 * 4 + 4096);
  cudaMalloc(&out, 256 * 128 * 4);
  cudaMalloc(&tm, 256 * 8);
  run<8, 0>(ws, out, tm, "ld.cg 4B");
  run<32, 0>(ws, out, tm, "ld.cg 4B");
  run<64, 0>(ws, out, tm, "ld.cg 4B");
  run<8, 1>(ws, out, tm, "ld 4B");
  run<32, 1>(ws, out, tm, "ld 4B");
  run<64, 1>(ws, out, tm, "ld 4B");
  run<32, 2>(ws, out, tm, "ld.cg 16B");
  run<64, 2>(ws, out, tm, "ld.cg 16B");
  run_slots<32, 1>(ws, out, tm);
  run_slots<64, 1>(ws, out, tm);
  run_slots<32, 0>(ws, out, tm);
  run_slots<64, 0>(ws, out, tm);
  run_after_write<8, 0>(ws, out, tm, "ld.cg 4B");
  run_after_write<64, 0>(ws, out, tm, "ld.cg 4B");
  run_after_write<64, 2>(ws, out, tm, "ld.cg 16B");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
