// Attention and the paged KV cache: RoPE + KV append,
// split-KV decode attention over pages with an in-kernel combine, and causal
// prefill attention. The decode kernel is HBM-bound on the KV read (8-15% of
// the decode step's bytes); the prefill kernel is a tiled
// flash-style CUDA-core kernel (attention is ~1-6% of prefill FLOPs).
//
// Paged layout: cache[block][kv_head][page][hd]; token position p of seq b
// lives in block block_table[b * max_blocks + p / page] at slot p % page.
#include <cstdlib>

#include "hx_common.cuh"

namespace hx {

// tensor-core variants (hx_attention_mma.cu)
int launch_prefill_mma(const void *q, const void *kc, const void *vc, const int32_t *bt, const int32_t *sl, void *o,
                       int batch, int s, int hq, int hkv, int hd, int page, int maxb, cudaStream_t st);
int launch_decode_mma(int G, int hd, dim3 grid, const void *q, const void *kc, const void *vc, const int32_t *bt,
                      const int32_t *sl, void *o, int hkv, int page, int maxb, float *ws, int *cnt, cudaStream_t st);
int launch_decode_tma(int G, dim3 grid, const void *q, const void *kc, const void *vc, const int32_t *bt,
                      const int32_t *sl, void *o, int hkv, int maxb, float *ws, int *cnt, bool rope, float theta,
                      cudaStream_t st, int ns, const SKView *skv = nullptr, long ldq = 0);
static int g_attn_tma = [] {
  const char *e = getenv("HX_ATTN_TMA");
  return e ? atoi(e) : 1;
}();
static int g_attn_mma = [] {
  const char *e = getenv("HX_ATTN_MMA");
  return e ? atoi(e) : 1;
}();
// smallest GQA group routed to the tensor-core decode kernel (1 = MHA too)
static int g_attn_mma_min_group = [] {
  const char *e = getenv("HX_ATTN_MMA_MIN_G");
  return e ? atoi(e) : 1;  // measured: MHA through the cp.async/mma kernel is also faster
}();

__device__ __forceinline__ size_t page_index(const int32_t *bt, int b, int pos, int max_blocks, int page,
                                             int hkv, int kvh, int hd) {
  const int blk = bt[(size_t)b * max_blocks + pos / page];
  return (((size_t)blk * hkv + kvh) * page + pos % page) * hd;
}

// ------------------------------------------------------------- RoPE + append
// One CTA per token: the (cos, sin) of the token's position are computed once
// into smem (the same fp32 arithmetic per pair index as everywhere else) and
// shared by all q / k heads; threads then sweep (head, 4 rotate-half pairs)
// tasks with 4-element vector loads and stores (v heads: plain copy into the
// page). The old (token, head) grid launched 96 tiny CTAs per token with
// scalar accesses and recomputed the transcendental per head.
template <typename T, int VEC>
__global__ void __launch_bounds__(256)
    rope_append_kernel(const T *qkv, T *q_out, T *kc, T *vc, const int32_t *bt, const int32_t *seq_lens,
                       int prefill_len, int hq, int hkv, int hd, int page, int max_blocks, float theta) {
  struct alignas(VEC * sizeof(T)) Vec { T v[VEC]; };
  __shared__ float2 csn[128];  // hd <= 256
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const int b = prefill_len ? t / prefill_len : t;
  const int pos = seq_lens[b] + (prefill_len ? t % prefill_len : 0);
  const int half = hd / 2;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float inv_freq = 1.0f / powf(theta, (float)(2 * i) / (float)hd);
    float sn, cs;
    sincosf((float)pos * inv_freq, &sn, &cs);
    csn[i] = make_float2(cs, sn);
  }
  __syncthreads();
  const int nh = hq + 2 * hkv, per = half / VEC;
  const T *row = qkv + (size_t)t * nh * hd;
  for (int task = threadIdx.x; task < nh * per; task += blockDim.x) {
    const int h = task / per, i = (task % per) * VEC;
    const Vec x1 = *reinterpret_cast<const Vec *>(row + (size_t)h * hd + i);
    const Vec x2 = *reinterpret_cast<const Vec *>(row + (size_t)h * hd + half + i);
    T *dst;
    if (h >= hq + hkv) {
      dst = vc + page_index(bt, b, pos, max_blocks, page, hkv, h - hq - hkv, hd);
      *reinterpret_cast<Vec *>(dst + i) = x1;
      *reinterpret_cast<Vec *>(dst + half + i) = x2;
      continue;
    }
    dst = h < hq ? q_out + ((size_t)t * hq + h) * hd : kc + page_index(bt, b, pos, max_blocks, page, hkv, h - hq, hd);
    Vec y1, y2;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const float2 c = csn[i + j];
      const float2 y = rope_rot(to_f32(x1.v[j]), to_f32(x2.v[j]), c.x, c.y);  // x cos + rotate_half(x) sin
      y1.v[j] = from_f32<T>(y.x);
      y2.v[j] = from_f32<T>(y.y);
    }
    *reinterpret_cast<Vec *>(dst + i) = y1;
    *reinterpret_cast<Vec *>(dst + half + i) = y2;
  }
}

// ------------------------------------------------------------- decode
// CTA = (seq b, kv head, split); 4 warps; a "lane group" of LG = HD / V lanes
// owns one token at a time (V = elements per 16-byte load), so a warp works on
// 32 / LG tokens concurrently and every lane issues U independent K and V
// 16-byte loads per iteration.
constexpr int DEC_THREADS = 128;

template <typename T, int HD, int G>
__global__ void __launch_bounds__(DEC_THREADS)
    attn_decode_kernel(const T *q, const T *kc, const T *vc, const int32_t *bt, const int32_t *seq_lens,
                       T *o, int hkv, int page, int max_blocks, float scale, float *ws, int *counters) {
  pdl_trigger();
  pdl_wait();
  constexpr int V = Vec16<T>::N;
  constexpr int LG = HD / V;
  constexpr int GPW = 32 / LG;
  constexpr int NG = (DEC_THREADS / 32) * GPW;
  constexpr int U = G <= 2 ? 8 : 4;  // 2*U independent 16-byte loads in flight per lane
  const int b = blockIdx.x / hkv, kvh = blockIdx.x % hkv;
  const int split = blockIdx.y, splits = gridDim.y;
  const int hq = hkv * G;
  const int ctx = seq_lens[b] + 1;
  const int chunk = (ctx + splits - 1) / splits;
  const int t0 = split * chunk, t1 = min(ctx, t0 + chunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp * GPW + lane / LG, gl = lane % LG;
  const int d0 = gl * V;

  float qv[G][V];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    Vec16<T>::load(q + ((size_t)b * hq + kvh * G + g) * HD + d0, qv[g]);
#pragma unroll
    for (int j = 0; j < V; ++j) qv[g][j] *= scale;
  }
  float m[G], l[G], acc[G][V];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) acc[g][j] = 0.f;
  }
  const int32_t *btb = bt + (size_t)b * max_blocks;
  for (int base = t0; base < t1; base += NG * U) {  // warp-uniform trip count (shuffles below)
    uint4 kraw[U], vraw[U];  // raw 16-byte vectors: all loads issued before any use
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int p = base + u * NG + grp;
      ok[u] = p < t1;
      if (ok[u]) {
        const size_t off = (((size_t)btb[p / page] * hkv + kvh) * page + p % page) * HD + d0;
        kraw[u] = __ldg(reinterpret_cast<const uint4 *>(kc + off));
        vraw[u] = __ldg(reinterpret_cast<const uint4 *>(vc + off));
      } else {
        kraw[u] = make_uint4(0, 0, 0, 0);
        vraw[u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float kv[V], vv[V];
      Vec16<T>::load(reinterpret_cast<const T *>(&kraw[u]), kv);
      Vec16<T>::load(reinterpret_cast<const T *>(&vraw[u]), vv);
      float s[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float a = 0.f;
#pragma unroll
        for (int j = 0; j < V; ++j) a = fmaf(qv[g][j], kv[j], a);
#pragma unroll
        for (int off = LG / 2; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        s[g] = a;
      }
      if (!ok[u]) continue;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float mn = fmaxf(m[g], s[g]);
        const float corr = __expf(m[g] - mn);
        const float pr = __expf(s[g] - mn);
        l[g] = l[g] * corr + pr;
#pragma unroll
        for (int j = 0; j < V; ++j) acc[g][j] = fmaf(pr, vv[j], acc[g][j] * corr);
        m[g] = mn;
      }
    }
  }

  // combine the NG lane groups of this CTA
  __shared__ float sm_m[NG][G], sm_l[NG][G];
  __shared__ float sm_acc[NG][G][HD];
  if (gl == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) { sm_m[grp][g] = m[g]; sm_l[grp][g] = l[g]; }
  }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int j = 0; j < V; ++j) sm_acc[grp][g][d0 + j] = acc[g][j];
  __syncthreads();
  // per (g, d): merge groups -> (M, L, A) for this split
  const size_t pair = (size_t)b * hkv + kvh;
  for (int w = threadIdx.x; w < G * HD; w += DEC_THREADS) {
    const int g = w / HD, d = w % HD;
    float M = -INFINITY;
    for (int i = 0; i < NG; ++i) M = fmaxf(M, sm_m[i][g]);
    float L = 0.f, A = 0.f;
    if (M != -INFINITY) {
      for (int i = 0; i < NG; ++i) {
        const float c = __expf(sm_m[i][g] - M);
        L += sm_l[i][g] * c;
        A += sm_acc[i][g][d] * c;
      }
    }
    if (splits == 1) {
      o[((size_t)b * hq + kvh * G + g) * HD + d] = from_f32<T>(A / L);
    } else {
      float *part = ws + ((pair * splits + split) * G + g) * (HD + 2);
      part[d] = A;
      if (d == 0) { part[HD] = M; part[HD + 1] = L; }
    }
  }
  if (splits == 1) return;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int tk = ticket_acq_rel(&counters[pair]);
    s_last = tk == splits - 1;
    if (s_last) counters[pair] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  for (int w = threadIdx.x; w < G * HD; w += DEC_THREADS) {
    const int g = w / HD, d = w % HD;
    float M = -INFINITY;
    for (int s = 0; s < splits; ++s) M = fmaxf(M, __ldcg(ws + ((pair * splits + s) * G + g) * (HD + 2) + HD));
    float L = 0.f, A = 0.f;
    for (int s = 0; s < splits; ++s) {
      const float *part = ws + ((pair * splits + s) * G + g) * (HD + 2);
      const float ms = __ldcg(part + HD);
      if (ms == -INFINITY) continue;
      const float c = __expf(ms - M);
      L += __ldcg(part + HD + 1) * c;
      A += __ldcg(part + d) * c;
    }
    o[((size_t)b * hq + kvh * G + g) * HD + d] = from_f32<T>(A / L);
  }
}

// ------------------------------------------------------------- prefill
// CTA = (64 queries, q head, seq); 256 threads; fp32 smem tiles; online softmax.
constexpr int PF_BQ = 64, PF_BK = 64, PF_THREADS = 256;

template <typename T, int HD>
__global__ void __launch_bounds__(PF_THREADS)
    attn_prefill_kernel(const T *q, const T *kc, const T *vc, const int32_t *bt, const int32_t *seq_lens,
                        T *o, int s_len, int hq, int hkv, int page, int max_blocks, float scale) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  float *Qs = sm;                         // [BQ][HD]
  float *Ks = Qs + PF_BQ * HD;            // [BK][HD + 1]
  float *Vs = Ks + PF_BK * (HD + 1);      // [BK][HD]
  float *Ps = Vs + PF_BK * HD;            // [BQ][BK + 1]
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (hq / hkv);
  const int p0 = seq_lens[b];
  const int q0 = qt * PF_BQ;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  constexpr int DPT = HD / 16;  // output dims per thread
  for (int i = tid; i < PF_BQ * HD; i += PF_THREADS) {
    const int r = i / HD, d = i % HD;
    const int qi = q0 + r;
    Qs[i] = qi < s_len ? to_f32(q[(((size_t)b * s_len + qi) * hq + h) * HD + d]) * scale : 0.f;
  }
  float m[4], l[4], acc[4][DPT];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    m[i] = -INFINITY;
    l[i] = 0.f;
#pragma unroll
    for (int j = 0; j < DPT; ++j) acc[i][j] = 0.f;
  }
  const int q_last = min(s_len, q0 + PF_BQ) - 1;
  for (int k0 = 0; k0 <= q_last; k0 += PF_BK) {
    __syncthreads();
    for (int i = tid; i < PF_BK * HD; i += PF_THREADS) {
      const int r = i / HD, d = i % HD;
      const int kj = k0 + r;
      float kvk = 0.f, kvv = 0.f;
      if (kj < s_len) {
        const size_t off = page_index(bt, b, p0 + kj, max_blocks, page, hkv, kvh, HD) + d;
        kvk = to_f32(kc[off]);
        kvv = to_f32(vc[off]);
      }
      Ks[r * (HD + 1) + d] = kvk;
      Vs[r * HD + d] = kvv;
    }
    __syncthreads();
    // S = Q K^T for rows ty*4+i, cols tx*4+j
    float s[4][4] = {};
    for (int d = 0; d < HD; ++d) {
      float a[4], kk[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Qs[(ty * 4 + i) * HD + d];
#pragma unroll
      for (int j = 0; j < 4; ++j) kk[j] = Ks[(tx * 4 + j) * (HD + 1) + d];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = fmaf(a[i], kk[j], s[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int qi = q0 + ty * 4 + i;
      float rmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int kj = k0 + tx * 4 + j;
        if (kj > qi || kj >= s_len) s[i][j] = -INFINITY;
        rmax = fmaxf(rmax, s[i][j]);
      }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, off));
      const float mn = fmaxf(m[i], rmax);
      const float corr = mn == -INFINITY ? 1.f : __expf(m[i] - mn);
      float rs = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float pr = mn == -INFINITY ? 0.f : __expf(s[i][j] - mn);
        Ps[(ty * 4 + i) * (PF_BK + 1) + tx * 4 + j] = pr;
        rs += pr;
      }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, off);
      l[i] = l[i] * corr + rs;
      m[i] = mn;
#pragma unroll
      for (int j = 0; j < DPT; ++j) acc[i][j] *= corr;
    }
    __syncthreads();
    for (int c = 0; c < PF_BK; ++c) {
      float vv[DPT];
#pragma unroll
      for (int j = 0; j < DPT; ++j) vv[j] = Vs[c * HD + tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float pr = Ps[(ty * 4 + i) * (PF_BK + 1) + c];
#pragma unroll
        for (int j = 0; j < DPT; ++j) acc[i][j] = fmaf(pr, vv[j], acc[i][j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int qi = q0 + ty * 4 + i;
    if (qi >= s_len) continue;
    T *dst = o + (((size_t)b * s_len + qi) * hq + h) * HD;
#pragma unroll
    for (int j = 0; j < DPT; ++j) dst[tx + 16 * j] = from_f32<T>(acc[i][j] / l[i]);
  }
}

static int decode_splits(int batch, int hkv, int max_ctx) {
  // one wave: the tensor-core kernel keeps 2 CTAs (2 x 64 KB of K/V in flight)
  // per SM, so splits = floor(2 * 148 / pairs) -- more would add a second,
  // mostly idle wave; each split still streams several 64-key blocks
  const int pairs = batch * hkv;
  static const int target = [] {  // CTAs per wave (2 per SM); HX_ATTN_CTAS overrides (tuning)
    const char *e = getenv("HX_ATTN_CTAS");
    return e ? atoi(e) : 2 * 148;
  }();
  int s = target / pairs;
  const int cap = (max_ctx + 63) / 64;
  s = s < cap ? s : cap;
  return s < 1 ? 1 : s;
}

// TMA decode kernel plan. Default: 2 CTAs per SM (4 warps, 3-deep ring), whose
// ~100 KB of smem lets a CTA become resident next to the preceding QKV GEMM's
// CTA under PDL and stream its KV pages during the GEMM's tail. HX_ATTN_NS=6:
// one 8-warp CTA per SM with a 6-deep ring and only as many splits as fill the
// 148 SMs (fewer splits, shorter combine: faster in isolation at 64-128 (batch,
// kv-head) pairs, but it cannot overlap the GEMM -- measured slower in the
// 70B TP=2 decode step, 8.73 vs 8.56 ms per 40 layers).
static int tma_decode_splits(int batch, int hkv, int max_ctx, int *ns) {
  const int pairs = batch * hkv;
  static const int env_ns = [] {
    const char *e = getenv("HX_ATTN_NS");
    return e ? atoi(e) : 0;
  }();
  const int cap = (max_ctx + 63) / 64;
  int s, n;
  if (env_ns == 6) {
    n = 6;
    s = 148 / pairs;
  } else if (env_ns == 2) {  // 2-deep ring, ~71 KB: 3 CTAs per SM
    n = 2;
    s = 3 * 148 / pairs;
  } else {
    n = 3;
    s = decode_splits(batch, hkv, max_ctx);
  }
  s = s < cap ? s : cap;
  *ns = n;
  return s < 1 ? 1 : s;
}

template <typename T, int HD>
static int launch_decode_g(int G, dim3 grid, const void *q, const void *kc, const void *vc, const int32_t *bt,
                           const int32_t *sl, void *o, int hkv, int page, int maxb, float scale, float *ws,
                           int *cnt, cudaStream_t st) {
#define HX_DEC(GG)                                                                                      \
  return launch(attn_decode_kernel<T, HD, GG>, dim3(grid), dim3(DEC_THREADS), 0, st, (const T *)q, (const T *)kc, (const T *)vc, bt, \
                                                              sl, (T *)o, hkv, page, maxb, scale, ws, cnt)
  switch (G) {
    case 1: HX_DEC(1); break;
    case 2: HX_DEC(2); break;
    case 4: HX_DEC(4); break;
    case 8: HX_DEC(8); break;
    case 16:
      if constexpr (sizeof(T) == 4) {  // bf16 G=16 always takes the tensor-core kernel
        HX_DEC(16);
      } else {
        return HX_ERR_UNSUPPORTED;
      }
    default: return HX_ERR_UNSUPPORTED;
  }
#undef HX_DEC
  return launch_status();
}

}  // namespace hx

using namespace hx;

extern "C" int hx_rope_kv_append(const void *qkv, void *q_out, void *k_cache, void *v_cache,
                                 const int32_t *block_table, const int32_t *seq_lens, int dtype, int n_tok,
                                 int prefill_len, int hq, int hkv, int hd, int page_size, int max_blocks,
                                 float theta, hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!qkv || !q_out || !k_cache || !v_cache || !block_table || !seq_lens || hd % 2 || page_size <= 0)
    return HX_ERR_ARG;
  if (hd > 256) return HX_ERR_UNSUPPORTED;
  cudaStream_t st = as_stream(stream);
  const dim3 grid(n_tok);
  const int half = hd / 2;
#define HX_ROPE(T, V)                                                                                            \
  return launch(rope_append_kernel<T, V>, grid, dim3(256), 0, st, (const T *)qkv, (T *)q_out, (T *)k_cache,     \
                (T *)v_cache, block_table, seq_lens, prefill_len, hq, hkv, hd, page_size, max_blocks, theta)
  if (dtype == HX_BF16) {
    if (half % 4 == 0) HX_ROPE(__nv_bfloat16, 4);
    HX_ROPE(__nv_bfloat16, 1);
  }
  if (half % 4 == 0) HX_ROPE(float, 4);
  HX_ROPE(float, 1);
#undef HX_ROPE
  return launch_status();
}

extern "C" size_t hx_attn_decode_workspace(int batch, int hq, int hkv, int hd, int max_ctx) {
  int ns;
  const int s0 = decode_splits(batch, hkv, max_ctx), s1 = tma_decode_splits(batch, hkv, max_ctx, &ns);
  const int s = s0 > s1 ? s0 : s1;
  if (s <= 1) return 0;
  const size_t counters = kTicketBytes;
  return counters + (size_t)batch * hkv * s * (hq / hkv) * (hd + 2) * sizeof(float);
}

extern "C" int hx_attn_decode_paged(const void *q, const void *k_cache, const void *v_cache,
                                    const int32_t *block_table, const int32_t *seq_lens, void *o, int dtype,
                                    int batch, int hq, int hkv, int hd, int page_size, int max_blocks,
                                    int max_ctx, void *workspace, size_t workspace_bytes, hx_stream_t stream) {
  if (batch == 0) return 0;
  if (!q || !k_cache || !v_cache || !block_table || !seq_lens || !o || hq % hkv) return HX_ERR_ARG;
  const int G = hq / hkv;
  const bool tma = dtype == HX_BF16 && hd == 128 && page_size == 64 && g_attn_tma &&
                   (G == 1 || G == 2 || G == 4 || G == 8 || G == 16);
  int ns = 3;
  const int splits = tma ? tma_decode_splits(batch, hkv, max_ctx, &ns) : decode_splits(batch, hkv, max_ctx);
  float *ws = nullptr;
  int *cnt = nullptr;
  if (splits > 1) {
    if (!workspace || workspace_bytes < hx_attn_decode_workspace(batch, hq, hkv, hd, max_ctx))
      return HX_ERR_WORKSPACE;
    if (batch * hkv > kMaxTickets) return HX_ERR_UNSUPPORTED;
    const size_t counters = kTicketBytes;
    cnt = reinterpret_cast<int *>(workspace);
    ws = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(workspace) + counters);
  }
  dim3 grid(batch * hkv, splits);
  const float scale = 1.0f / sqrtf((float)hd);
  if (tma)
    return launch_decode_tma(G, grid, q, k_cache, v_cache, block_table, seq_lens, o, hkv, max_blocks, ws, cnt, false,
                             0.f, as_stream(stream), ns);
  if (dtype == HX_BF16 && G >= g_attn_mma_min_group && (hd == 64 || hd == 128) && g_attn_mma)  // tensor cores
    return launch_decode_mma(G, hd, grid, q, k_cache, v_cache, block_table, seq_lens, o, hkv, page_size, max_blocks,
                             ws, cnt, as_stream(stream));
  cudaStream_t st = as_stream(stream);
#define HX_ARGS grid, q, k_cache, v_cache, block_table, seq_lens, o, hkv, page_size, max_blocks, scale, ws, cnt, st
  if (dtype == HX_BF16) {
    switch (hd) {
      case 32: return launch_decode_g<__nv_bfloat16, 32>(G, HX_ARGS);
      case 64: return launch_decode_g<__nv_bfloat16, 64>(G, HX_ARGS);
      case 128: return launch_decode_g<__nv_bfloat16, 128>(G, HX_ARGS);
    }
  } else {
    switch (hd) {
      case 32: return launch_decode_g<float, 32>(G, HX_ARGS);
      case 64: return launch_decode_g<float, 64>(G, HX_ARGS);
      case 128: return launch_decode_g<float, 128>(G, HX_ARGS);
    }
  }
#undef HX_ARGS
  return HX_ERR_UNSUPPORTED;
}

extern "C" int hx_attn_decode_rope_append(const void *qkv, void *k_cache, void *v_cache, const int32_t *block_table,
                                          const int32_t *seq_lens, void *o, int dtype, int batch, int hq, int hkv,
                                          int hd, int page_size, int max_blocks, int max_ctx, float theta,
                                          void *workspace, size_t workspace_bytes, hx_stream_t stream) {
  if (batch == 0) return 0;
  if (!qkv || !k_cache || !v_cache || !block_table || !seq_lens || !o || hq % hkv) return HX_ERR_ARG;
  const int G = hq / hkv;
  if (dtype != HX_BF16 || hd != 128 || page_size != 64 || !g_attn_tma ||
      !(G == 1 || G == 2 || G == 4 || G == 8 || G == 16))
    return HX_ERR_UNSUPPORTED;
  int ns = 3;
  const int splits = tma_decode_splits(batch, hkv, max_ctx, &ns);
  float *ws = nullptr;
  int *cnt = nullptr;
  if (splits > 1) {
    if (!workspace || workspace_bytes < hx_attn_decode_workspace(batch, hq, hkv, hd, max_ctx))
      return HX_ERR_WORKSPACE;
    if (batch * hkv > kMaxTickets) return HX_ERR_UNSUPPORTED;
    cnt = reinterpret_cast<int *>(workspace);
    ws = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(workspace) + kTicketBytes);
  }
  return launch_decode_tma(G, dim3(batch * hkv, splits), qkv, k_cache, v_cache, block_table, seq_lens, o, hkv,
                           max_blocks, ws, cnt, true, theta, as_stream(stream), ns);
}

extern "C" int hx_attn_decode_rope_append_sk(const float *qkv32, int ld_qkv, const void *gemm_workspace, int k_dim,
                                             void *k_cache, void *v_cache, const int32_t *block_table,
                                             const int32_t *seq_lens, void *o, int batch, int hq, int hkv, int hd,
                                             int page_size, int max_blocks, int max_ctx, float theta, void *workspace,
                                             size_t workspace_bytes, hx_stream_t stream) {
  if (batch == 0) return 0;
  if (!qkv32 || !gemm_workspace || !k_cache || !v_cache || !block_table || !seq_lens || !o || hq % hkv ||
      ld_qkv < (hq + 2 * hkv) * hd || k_dim <= 0)
    return HX_ERR_ARG;
  const int G = hq / hkv;
  if (hd != 128 || page_size != 64 || !g_attn_tma || !(G == 1 || G == 2 || G == 4 || G == 8 || G == 16))
    return HX_ERR_UNSUPPORTED;
  SKView skv;
  int rc = sk_view_for(batch, (hq + 2 * hkv) * hd, k_dim, gemm_workspace, &skv);
  if (rc) return rc;
  int ns = 3;
  const int splits = tma_decode_splits(batch, hkv, max_ctx, &ns);
  if (ns == 6) return HX_ERR_UNSUPPORTED;
  float *ws = nullptr;
  int *cnt = nullptr;
  if (splits > 1) {
    if (!workspace || workspace_bytes < hx_attn_decode_workspace(batch, hq, hkv, hd, max_ctx))
      return HX_ERR_WORKSPACE;
    if (batch * hkv > kMaxTickets) return HX_ERR_UNSUPPORTED;
    cnt = reinterpret_cast<int *>(workspace);
    ws = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(workspace) + kTicketBytes);
  }
  return launch_decode_tma(G, dim3(batch * hkv, splits), qkv32, k_cache, v_cache, block_table, seq_lens, o, hkv,
                           max_blocks, ws, cnt, true, theta, as_stream(stream), ns, &skv, ld_qkv);
}

template <typename T, int HD>
static int launch_prefill(const void *q, const void *kc, const void *vc, const int32_t *bt, const int32_t *sl,
                          void *o, int batch, int s, int hq, int hkv, int page, int maxb, cudaStream_t st) {
  const size_t smem = sizeof(float) * (PF_BQ * HD + PF_BK * (HD + 1) + PF_BK * HD + PF_BQ * (PF_BK + 1));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_kernel<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((s + PF_BQ - 1) / PF_BQ, hq, batch);
  return launch(attn_prefill_kernel<T, HD>, dim3(grid), dim3(PF_THREADS), smem, st, (const T *)q, (const T *)kc, (const T *)vc, bt, sl,
                                                             (T *)o, s, hq, hkv, page, maxb,
                                                             1.0f / sqrtf((float)HD));
  return launch_status();
}

extern "C" int hx_attn_prefill(const void *q, const void *k_cache, const void *v_cache, const int32_t *block_table,
                               const int32_t *seq_lens, void *o, int dtype, int batch, int s, int hq, int hkv,
                               int hd, int page_size, int max_blocks, hx_stream_t stream) {
  if (batch == 0 || s == 0) return 0;
  if (!q || !k_cache || !v_cache || !block_table || !seq_lens || !o || hq % hkv) return HX_ERR_ARG;
  cudaStream_t st = as_stream(stream);
#define HX_PF(T, D) return launch_prefill<T, D>(q, k_cache, v_cache, block_table, seq_lens, o, batch, s, hq, hkv, page_size, max_blocks, st)
  if (dtype == HX_BF16 && (hd == 64 || hd == 128) && g_attn_mma)
    return launch_prefill_mma(q, k_cache, v_cache, block_table, seq_lens, o, batch, s, hq, hkv, hd, page_size,
                              max_blocks, st);
  if (dtype == HX_BF16) {
    switch (hd) {
      case 32: HX_PF(__nv_bfloat16, 32);
      case 64: HX_PF(__nv_bfloat16, 64);
      case 128: HX_PF(__nv_bfloat16, 128);
    }
  } else {
    switch (hd) {
      case 32: HX_PF(float, 32);
      case 64: HX_PF(float, 64);
      case 128: HX_PF(float, 128);
    }
  }
#undef HX_PF
  return HX_ERR_UNSUPPORTED;
}
