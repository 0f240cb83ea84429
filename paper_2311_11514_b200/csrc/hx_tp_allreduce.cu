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

unsigned long long *hx_trace_slots(size_t n);  // hx_gemm.cu (hx_debug_trace)

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


// ---------------------------------------------------------------------------
// Push ("one-shot, flag-free") variant. The pull kernel above pays three
// dependent NVLink trips per call (flag store -> peer flag observed -> remote
// loads). Here every rank PUSHES its partial row into every peer's inbox with
// plain remote stores and each receiver polls its own LOCAL inbox until the
// data itself is there: an inbox element holds the sentinel -0.0f (0x80000000)
// until a peer's store lands (pushed values are sanitised -0.0 -> +0.0, which
// cannot change any sum). One one-way NVLink trip per call, no fences.
// Inbox per rank: [2 buffers][tp senders][max_tok][hidden] fp32; call k uses
// buffer k & 1 and every element is re-armed in place right after it is read
// (a peer writes buffer k & 1 again only at call k + 2, which needs this
// rank's call k + 1 data, pushed after this kernel has completed).
// One token row = a cluster of AR_CL CTAs, each owning hidden / AR_CL features,
// so the push/poll traffic spreads over 4x the SMs; the RMS sum of squares is
// combined across the cluster through DSMEM. Call counters are per CTA:
// state[c] counts the calls CTA c (= token row t, feature slice c % AR_CL)
// took part in -- every inbox location is always served by the same CTA index
// on every rank, so no cross-CTA atomics sit on the kernel's completion path.
struct ArInbox {
  float *box[kMaxTP];  // rank r's inbox (peer-mapped; own = local)
};

constexpr uint32_t kSentinel = 0x80000000u;
constexpr int AR_CL = 4;

__device__ __forceinline__ uint4 ld_volatile_u4(const void *p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool has_sentinel(const uint4 &v) {
  return v.x == kSentinel || v.y == kSentinel || v.z == kSentinel || v.w == kSentinel;
}

// bf16 payload (PL = __nv_bfloat16): each partial is rounded to bf16 once
// (every rank, its own partial included, so all ranks sum identical values in
// rank order, accumulating in fp32): half the NVLink bytes of the fp32 payload.
// Inbox halfwords are armed with the bf16 sentinel 0x8000 (-0.0), pushed -0.0 is
// sent as +0.0.
template <typename PL>
struct ArPayload;
template <>
struct ArPayload<float> {
  static constexpr int V = 4;  // elements per 16-byte vector
  __device__ static bool armed(const uint4 &u) { return has_sentinel(u); }
  __device__ static uint4 sentinel() { return make_uint4(kSentinel, kSentinel, kSentinel, kSentinel); }
  __device__ static uint4 pack(const float *v) {  // -0.0 -> +0.0 (bitwise), value-preserving
    return make_uint4(__float_as_uint(v[0] + 0.0f), __float_as_uint(v[1] + 0.0f), __float_as_uint(v[2] + 0.0f),
                      __float_as_uint(v[3] + 0.0f));
  }
  __device__ static void unpack(const uint4 &u, float *v) {
    v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y); v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
  }
};
template <>
struct ArPayload<__nv_bfloat16> {
  static constexpr int V = 8;
  static constexpr uint32_t S2 = 0x80008000u;
  __device__ static bool has16(uint32_t w) { return (w & 0xFFFFu) == 0x8000u || (w >> 16) == 0x8000u; }
  __device__ static bool armed(const uint4 &u) { return has16(u.x) || has16(u.y) || has16(u.z) || has16(u.w); }
  __device__ static uint4 sentinel() { return make_uint4(S2, S2, S2, S2); }
  __device__ static uint32_t pk2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    uint32_t w = *reinterpret_cast<uint32_t *>(&h);
    if ((w & 0xFFFFu) == 0x8000u) w &= 0xFFFF0000u;  // -0.0 -> +0.0
    if ((w >> 16) == 0x8000u) w &= 0x0000FFFFu;
    return w;
  }
  __device__ static uint4 pack(const float *v) {
    return make_uint4(pk2(v[0], v[1]), pk2(v[2], v[3]), pk2(v[4], v[5]), pk2(v[6], v[7]));
  }
  __device__ static void unpack(const uint4 &u, float *v) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};

template <typename TO, typename PL>
__global__ void __launch_bounds__(256)
    tp_ar_push_rmsnorm_kernel(float *x, const float *own, ArInbox ib, int rank, int tp, int max_tok, int *state,
                              const float *gain, TO *out, int hidden, float eps, SKView skv,
                              unsigned long long *trace) {
  pdl_trigger();
  // hx_debug_trace: start, wait done, end, smid | 1 << 41, partial read, pushed, peers arrived, summed
  unsigned long long *tr = trace ? trace + 8 * blockIdx.x : nullptr;
  auto stamp = [&](int f) {
    if (tr && threadIdx.x == 0) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tt));
      tr[f] = tt;
    }
  };
  stamp(0);
  __shared__ float red[8];
  __shared__ float parts[AR_CL];
  const unsigned cr = cluster_rank();
  const int t = blockIdx.x / AR_CL;
  const int per = hidden / AR_CL, base = (int)cr * per;
  const size_t row = (size_t)hidden;
  if (out) cluster_arrive_relaxed();  // matched by the wait before the first DSMEM store (every CTA started)
  if (out && threadIdx.x < per / 32)   // the gain is a weight: pull this CTA's slice into L1 before the wait
    asm volatile("prefetch.global.L1 [%0];" ::"l"(gain + base + threadIdx.x * 32));
  constexpr int V = ArPayload<PL>::V;   // features per 16-byte vector
  constexpr int NV = 2048 / (256 * V);  // vectors per thread: <= 2048 features per CTA (hidden <= 8192)
  constexpr int NQ = NV * V / 4;        // float4 reads of this rank's partial per thread
  // deferred GEMM (skv.ws): the contributor ranges of this thread's tiles, before the wait
  SkTile sti[NQ];
  int sn[NQ];
  bool sact[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    sn[q] = base + ((q / (V / 4)) * 256 + threadIdx.x) * V + (q % (V / 4)) * 4;
    sact[q] = sn[q] < base + per;
    sti[q] = SkTile{0, -1, 0};
    if (skv.ws && sact[q]) sti[q] = sk_tile(skv, sn[q] / kSkRows);
  }
  pdl_wait();  // this rank's partial (previous kernel) is complete
  stamp(1);
  if (tr && threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    tr[3] = sm | (1ull << 41);
  }
  const int call = *(volatile int *)(state + blockIdx.x);
  const int buf = call & 1;
  // inbox element index of (buffer, sender r, token t, feature n); payload elements of PL
  PL *mine = reinterpret_cast<PL *>(ib.box[rank]);
  auto at = [&](PL *box, int r, int n) { return box + (((size_t)buf * tp + r) * max_tok + t) * row + n; };
  float p[NV][V];
  // this rank's partial: plain, or (skv.ws: the O/down GEMM was deferred,
  // HX_LINEAR_DEFER_REDUCE) its split tiles summed from the partial slots in CTA
  // order -- the fix-up's bits -- every load of the thread in flight together
  float4 f4[NQ], x4[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q)  // the residual row too: its loads overlap the push and the poll
    if (sact[q]) x4[q] = *reinterpret_cast<const float4 *>(x + (size_t)t * row + sn[q]);
  if (skv.ws) {
    sk_gather_n<NQ>(skv, sti, own, (long)row, t, sn, sact, f4);
  } else {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (sact[q]) f4[q] = __ldcs(reinterpret_cast<const float4 *>(own + (size_t)t * row + sn[q]));
  }
  stamp(4);
  // 1. push my partial slice of row t to every peer (remote stores, fire and forget)
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int n = base + (i * 256 + threadIdx.x) * V;
    if (n >= base + per) continue;
#pragma unroll
    for (int j = 0; j < V; j += 4) {
      const float4 f = f4[i * (V / 4) + j / 4];
      p[i][j] = f.x; p[i][j + 1] = f.y; p[i][j + 2] = f.z; p[i][j + 3] = f.w;
    }
    const uint4 w = ArPayload<PL>::pack(p[i]);
    ArPayload<PL>::unpack(w, p[i]);  // this rank sums exactly the values its peers receive
    for (int r = 0; r < tp; ++r)
      if (r != rank) *reinterpret_cast<uint4 *>(at(reinterpret_cast<PL *>(ib.box[r]), rank, n)) = w;
  }
  stamp(5);
  // 2. poll my inbox for every peer's slice, re-arm it in place, sum in rank order
  //    (bitwise identical on all ranks), residual
  const uint4 s4 = ArPayload<PL>::sentinel();
  float ss = 0.f;
  float v[NV][V];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int n = base + (i * 256 + threadIdx.x) * V;
    if (n >= base + per) continue;
    float sum[V];
#pragma unroll
    for (int j = 0; j < V; ++j) sum[j] = 0.f;
    for (int r = 0; r < tp; ++r) {
      float q[V];
      if (r != rank) {
        PL *src = at(mine, r, n);
        uint4 u = ld_volatile_u4(src);
        for (uint32_t spins = 0; ArPayload<PL>::armed(u); ++spins) {
          if (spins > (1u << 26)) __trap();  // a peer never arrived: fail loudly, never hang
          u = ld_volatile_u4(src);
        }
        *reinterpret_cast<uint4 *>(src) = s4;
        ArPayload<PL>::unpack(u, q);
      } else {
#pragma unroll
        for (int j = 0; j < V; ++j) q[j] = p[i][j];
      }
#pragma unroll
      for (int j = 0; j < V; ++j) sum[j] += q[j];
    }
#pragma unroll
    for (int j = 0; j < V; j += 4) {
      float4 acc = x4[i * (V / 4) + j / 4];
      acc.x += sum[j]; acc.y += sum[j + 1]; acc.z += sum[j + 2]; acc.w += sum[j + 3];
      *reinterpret_cast<float4 *>(x + (size_t)t * row + n + j) = acc;
      v[i][j] = acc.x; v[i][j + 1] = acc.y; v[i][j + 2] = acc.z; v[i][j + 3] = acc.w;
      ss += acc.x * acc.x + acc.y * acc.y + acc.z * acc.z + acc.w * acc.w;
    }
  }
  stamp(6);
  // 3. RMSNorm across the cluster (DSMEM), same summation order in every CTA
  if (out) {
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    cluster_wait();
    if (threadIdx.x == 0) {  // this CTA's sum of squares into every cluster CTA's parts[rank]
      float s2 = 0.f;
      for (int i = 0; i < 8; ++i) s2 += red[i];
      for (int c = 0; c < AR_CL; ++c) dsmem_st_f32(&parts[cr], c, s2);
    }
    cluster_sync_all();  // every CTA's stores into this CTA's parts[] are visible; no remote reads follow
    float tot = 0.f;
    for (int c = 0; c < AR_CL; ++c) tot += parts[c];   // same order in every CTA
    const float inv = 1.0f / sqrtf(tot / (float)hidden + eps);
    TO *o = out + (size_t)t * row;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int n = base + (i * 256 + threadIdx.x) * V;
      if (n >= base + per) continue;
#pragma unroll
      for (int j = 0; j < V; j += 4) {
        const float4 g = __ldg(reinterpret_cast<const float4 *>(gain + n + j));
        store4(o + n + j, (v[i][j] * inv) * g.x, (v[i][j + 1] * inv) * g.y, (v[i][j + 2] * inv) * g.z,
               (v[i][j + 3] * inv) * g.w);
      }
    }
  }
  __syncthreads();  // every thread has read `call`
  if (threadIdx.x == 0) *(volatile int *)(state + blockIdx.x) = call + 1;
  stamp(2);
}

__global__ void fill_u32_kernel(uint32_t *p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
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

extern "C" size_t hx_tp_inbox_bytes_ex(int tp, int max_tok, int hidden, int payload_dtype) {
  return (size_t)2 * tp * max_tok * hidden * (payload_dtype == HX_BF16 ? 2 : 4);
}

extern "C" size_t hx_tp_inbox_bytes(int tp, int max_tok, int hidden) {
  return hx_tp_inbox_bytes_ex(tp, max_tok, hidden, HX_F32);
}

extern "C" int hx_tp_inbox_init_ex(void *inbox, int tp, int max_tok, int hidden, int payload_dtype,
                                   hx_stream_t stream) {
  if (!inbox || tp < 1 || max_tok < 1 || hidden < 1) return HX_ERR_ARG;
  // load the kernels before any rank spins in them (lazy loading, see hx_handoff_inbox_init)
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, tp_ar_push_rmsnorm_kernel<float, float>);
  cudaFuncGetAttributes(&fa, tp_ar_push_rmsnorm_kernel<__nv_bfloat16, float>);
  cudaFuncGetAttributes(&fa, tp_ar_push_rmsnorm_kernel<float, __nv_bfloat16>);
  cudaFuncGetAttributes(&fa, tp_ar_push_rmsnorm_kernel<__nv_bfloat16, __nv_bfloat16>);
  const size_t n = hx_tp_inbox_bytes_ex(tp, max_tok, hidden, payload_dtype) / 4;
  fill_u32_kernel<<<296, 256, 0, as_stream(stream)>>>((uint32_t *)inbox, n,
                                                       payload_dtype == HX_BF16 ? 0x80008000u : kSentinel);
  return launch_status();
}

extern "C" int hx_tp_inbox_init(void *inbox, int tp, int max_tok, int hidden, hx_stream_t stream) {
  return hx_tp_inbox_init_ex(inbox, tp, max_tok, hidden, HX_F32, stream);
}

static int ar_push(float *x, const float *own_part, void *const *inboxes, int rank, int tp, int max_tok, int *state,
                   const float *gain, void *out, int out_dtype, int n_tok, int hidden, float eps, int payload_dtype,
                   const SKView &skv, hx_stream_t stream) {
  if (n_tok == 0) return 0;
  const int V = payload_dtype == HX_BF16 ? 8 : 4;
  if (!x || !own_part || !inboxes || !state || tp < 1 || tp > kMaxTP || rank < 0 || rank >= tp ||
      n_tok > max_tok || hidden % (V * AR_CL) || hidden > 8192 || (out && !gain) ||
      (payload_dtype != HX_F32 && payload_dtype != HX_BF16))
    return HX_ERR_ARG;
  ArInbox ib{};
  for (int r = 0; r < tp; ++r) ib.box[r] = reinterpret_cast<float *>(inboxes[r]);
  cudaStream_t st = as_stream(stream);
  const dim3 grid(n_tok * AR_CL);
  unsigned long long *tr = hx_trace_slots((size_t)grid.x);
#define HX_AR(TO, PL)                                                                                              \
  return launch_cluster(tp_ar_push_rmsnorm_kernel<TO, PL>, grid, dim3(256), 0, st, AR_CL, x, own_part, ib, rank, tp, \
                        max_tok, state, gain, (TO *)out, hidden, eps, skv, tr)
  if (payload_dtype == HX_BF16) {
    if (out_dtype == HX_BF16) HX_AR(__nv_bfloat16, __nv_bfloat16);
    HX_AR(float, __nv_bfloat16);
  }
  if (out_dtype == HX_BF16) HX_AR(__nv_bfloat16, float);
  HX_AR(float, float);
#undef HX_AR
}

extern "C" int hx_tp_allreduce_push_residual_rmsnorm_ex(float *x, const float *own_part, void *const *inboxes, int rank,
                                                        int tp, int max_tok, int *state, const float *gain, void *out,
                                                        int out_dtype, int n_tok, int hidden, float eps,
                                                        int payload_dtype, hx_stream_t stream) {
  return ar_push(x, own_part, inboxes, rank, tp, max_tok, state, gain, out, out_dtype, n_tok, hidden, eps,
                 payload_dtype, SKView{}, stream);
}

extern "C" int hx_tp_allreduce_push_residual_rmsnorm_sk(float *x, const float *own_part, const void *gemm_workspace,
                                                        int k_dim, void *const *inboxes, int rank, int tp, int max_tok,
                                                        int *state, const float *gain, void *out, int out_dtype,
                                                        int n_tok, int hidden, float eps, int payload_dtype,
                                                        hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!gemm_workspace || k_dim <= 0) return HX_ERR_ARG;
  SKView skv;
  const int rc = sk_view_for(n_tok, hidden, k_dim, gemm_workspace, &skv);
  if (rc) return rc;
  return ar_push(x, own_part, inboxes, rank, tp, max_tok, state, gain, out, out_dtype, n_tok, hidden, eps,
                 payload_dtype, skv, stream);
}

extern "C" int hx_tp_allreduce_push_residual_rmsnorm(float *x, const float *own_part, float *const *inboxes, int rank,
                                                     int tp, int max_tok, int *state, const float *gain, void *out,
                                                     int out_dtype, int n_tok, int hidden, float eps,
                                                     hx_stream_t stream) {
  return hx_tp_allreduce_push_residual_rmsnorm_ex(x, own_part, reinterpret_cast<void *const *>(inboxes), rank, tp,
                                                  max_tok, state, gain, out, out_dtype, n_tok, hidden, eps, HX_F32,
                                                  stream);
}
