// Fused TP all-reduce + residual + RMSNorm over NVLink peer memory (decode).
//
// Replaces, for decode-sized messages, the NCCL all-reduce that follows each
// row-parallel projection (the reference models it as 4 BSP
// supersteps per layer, costs.py:123-147) together with the residual add and
// the next RMSNorm that consume it. Each TP rank's O/down GEMM writes its fp32
// partial into its own peer-visible slot (cudaIpc-exported); this kernel then,
// per token row (one CTA):
//   1. publishes "row t of my partial is ready" by writing the call's epoch
//      into flag[site][t][my rank] of EVERY rank (NVLink stores, release.sys);
//   2. waits until all ranks' flags for row t carry the epoch (acquire.sys,
//      bounded spin -> trap rather than hang);
//   3. reads every rank's partial row over NVLink (peer loads, 16 B vectors),
//      sums them in rank order -- identical bits on every rank, so the
//      replicated residual stream stays replicated -- adds the residual and
//      writes x and rmsnorm(x) * gain.
// One launch replaces NCCL all-reduce + hx_residual_add_rmsnorm; the message
// never round-trips through a staging buffer. Epochs: per call site, bumped by
// the site's last CTA, so graph replays and repeated requests never need a reset.
#include <cstring>

#include "hx_common.cuh"

namespace hx {

constexpr int kMaxTP = 8;

struct ArPeers {
  const float *part[kMaxTP];  // rank r's partial slot [n_tok][hidden] (peer-mapped; own = local)
  int *flags[kMaxTP];         // rank r's flag array [sites][max_tok][kMaxTP] (peer-mapped)
};

__device__ __forceinline__ void st_release_sys(int *p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int *p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename TO>
__global__ void __launch_bounds__(1024)
    tp_ar_rmsnorm_kernel(float *x, ArPeers peers, int rank, int tp, int site, int max_tok, int *site_state,
                         const float *gain, TO *out, int hidden, float eps) {
  pdl_trigger();
  pdl_wait();  // this rank's partial (previous kernel) is complete
  __shared__ float red[32];
  __shared__ int s_epoch;
  const int t = blockIdx.x;
  int *state = site_state + 2 * site;  // [epoch, done-CTAs]
  if (threadIdx.x == 0) {
    const int e = *(volatile int *)state + 1;
    s_epoch = e;
    __threadfence_system();  // partial writes (previous kernel) before the flags
    for (int r = 0; r < tp; ++r)
      st_release_sys(peers.flags[r] + ((size_t)site * max_tok + t) * kMaxTP + rank, e);
  }
  __syncthreads();
  const int e = s_epoch;
  if (threadIdx.x < tp) {
    const int *f = peers.flags[rank] + ((size_t)site * max_tok + t) * kMaxTP + threadIdx.x;
    for (uint32_t spins = 0; ld_acquire_sys(f) < e; ++spins)
      if (spins > (1u << 26)) __trap();  // a peer never arrived: fail loudly, never hang
  }
  __syncthreads();
  constexpr int MAXV = 2;  // hidden <= 8192
  float4 v[MAXV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int n = (i * 1024 + threadIdx.x) * 4;
    if (n >= hidden) continue;
    float4 acc = *reinterpret_cast<const float4 *>(x + (size_t)t * hidden + n);
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < tp; ++r) {  // rank order: identical result on every rank
      const float4 p = __ldcv(reinterpret_cast<const float4 *>(peers.part[r] + (size_t)t * hidden + n));
      sum.x += p.x; sum.y += p.y; sum.z += p.z; sum.w += p.w;
    }
    acc.x += sum.x; acc.y += sum.y; acc.z += sum.z; acc.w += sum.w;
    *reinterpret_cast<float4 *>(x + (size_t)t * hidden + n) = acc;
    v[i] = acc;
    ss += acc.x * acc.x + acc.y * acc.y + acc.z * acc.z + acc.w * acc.w;
  }
  if (out) {
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    float tot = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot += red[i];
    const float inv = 1.0f / sqrtf(tot / (float)hidden + eps);
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int n = (i * 1024 + threadIdx.x) * 4;
      if (n >= hidden) continue;
      const float4 g = *reinterpret_cast<const float4 *>(gain + n);
      TO *o = out + (size_t)t * hidden + n;
      o[0] = from_f32<TO>((v[i].x * inv) * g.x);
      o[1] = from_f32<TO>((v[i].y * inv) * g.y);
      o[2] = from_f32<TO>((v[i].z * inv) * g.z);
      o[3] = from_f32<TO>((v[i].w * inv) * g.w);
    }
  }
  // the site's last CTA publishes the epoch for the next call of this site
  __syncthreads();
  if (threadIdx.x == 0) {
    const int done = atomicAdd(state + 1, 1);
    if (done == (int)gridDim.x - 1) {
      state[1] = 0;
      *(volatile int *)state = e;
    }
  }
}

}  // namespace hx

using namespace hx;

extern "C" int hx_ipc_alloc(void **ptr, size_t bytes) {
  if (!ptr || !bytes) return HX_ERR_ARG;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, bytes);
  return e == cudaSuccess ? 0 : (int)e;
}

extern "C" int hx_ipc_free(void *ptr) { return (int)cudaFree(ptr); }

extern "C" int hx_ipc_handle(void *ptr, void *handle64) {
  if (!ptr || !handle64) return HX_ERR_ARG;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) return (int)e;
  static_assert(sizeof(h) == 64, "ipc handle size");
  memcpy(handle64, &h, 64);
  return 0;
}

extern "C" int hx_ipc_open(const void *handle64, void **peer_ptr) {
  if (!handle64 || !peer_ptr) return HX_ERR_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  return (int)cudaIpcOpenMemHandle(peer_ptr, h, cudaIpcMemLazyEnablePeerAccess);
}

extern "C" int hx_ipc_close(void *peer_ptr) { return (int)cudaIpcCloseMemHandle(peer_ptr); }

extern "C" int hx_tp_allreduce_residual_rmsnorm(float *x, const float *const *parts, int *const *flags, int rank,
                                                int tp, int site, int max_tok, int *site_state, const float *gain,
                                                void *out, int out_dtype, int n_tok, int hidden, float eps,
                                                hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!x || !parts || !flags || !site_state || tp < 1 || tp > kMaxTP || rank < 0 || rank >= tp ||
      n_tok > max_tok || hidden % 4 || hidden > 8192 || (out && !gain))
    return HX_ERR_ARG;
  ArPeers p{};
  for (int r = 0; r < tp; ++r) {
    p.part[r] = parts[r];
    p.flags[r] = flags[r];
  }
  cudaStream_t st = as_stream(stream);
  if (out_dtype == HX_BF16)
    return launch(tp_ar_rmsnorm_kernel<__nv_bfloat16>, dim3(n_tok), dim3(1024), 0, st, x, p, rank, tp, site, max_tok,
                  site_state, gain, (__nv_bfloat16 *)out, hidden, eps);
  return launch(tp_ar_rmsnorm_kernel<float>, dim3(n_tok), dim3(1024), 0, st, x, p, rank, tp, site, max_tok,
                site_state, gain, (float *)out, hidden, eps);
}
