// Does a kernel that stored to a PEER GPU's memory release its PDL dependents later?
// A (148 CTAs) optionally stores 4 KB per CTA to peer memory (NVLink) early, spins ~10 us, stamps its exit;
// B (PDL dependent) stamps after griddepcontrol.wait. Needs 2 GPUs with P2P.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peer_release peer_release.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void kern_a(float *dst, int mode, unsigned long long *tm) {
  asm volatile("griddepcontrol.launch_dependents;" :::);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (mode) {
    float4 *d = reinterpret_cast<float4 *>(dst) + blockIdx.x * 256;
    d[threadIdx.x] = make_float4(1.f, 2.f, 3.f, 4.f);
  }
  const unsigned long long t0 = gt();
  while (gt() - t0 < 10000) {
  }
  __syncthreads();
  if (threadIdx.x == 0) tm[blockIdx.x] = gt();
}

__global__ void kern_b(unsigned long long *tm) {
  asm volatile("griddepcontrol.launch_dependents;" :::);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) tm[blockIdx.x] = gt();
}

int main() {
  int can = 0;
  cudaDeviceCanAccessPeer(&can, 0, 1);
  if (!can) { printf("no P2P\n"); return 0; }
  cudaSetDevice(1);
  float *peer;
  cudaMalloc(&peer, 148 * 4096);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  float *local;
  cudaMalloc(&local, 148 * 4096);
  unsigned long long *ta, *tb;
  cudaMalloc(&ta, 148 * 8);
  cudaMalloc(&tb, 148 * 8);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const char *names[3] = {"no stores", "local stores", "peer (NVLink) stores"};
  for (int mode = 0; mode < 3; ++mode) {
    std::vector<double> d;
    for (int rep = 0; rep < 8; ++rep) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cfg.stream = st;
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(256);
      cudaLaunchKernelEx(&cfg, kern_a, mode == 2 ? peer : local, mode ? 1 : 0, ta);
      cudaLaunchKernelEx(&cfg, kern_b, tb);
      cudaStreamSynchronize(st);
      std::vector<unsigned long long> ha(148), hb(148);
      cudaMemcpy(ha.data(), ta, 148 * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(hb.data(), tb, 148 * 8, cudaMemcpyDeviceToHost);
      const double aend = (double)*std::max_element(ha.begin(), ha.end());
      const double bw = (double)*std::min_element(hb.begin(), hb.end());
      if (rep >= 2) d.push_back((bw - aend) / 1e3);
    }
    std::sort(d.begin(), d.end());
    printf("A with %-22s: B's wait passes %+.2f us after A's last CTA exit (median of %zu)\n", names[mode],
           d[d.size() / 2], d.size());
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
