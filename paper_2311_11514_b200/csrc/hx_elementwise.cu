// Row-wise / element-wise kernels of the layer (PAPER.md:121-151 with Llama-2
// specifics): embedding gather, RMSNorm, the fused "+ residual, then RMSNorm"
// that follows each TP all-reduce, SwiGLU, greedy argmax (vocab-parallel) and
// the per-step sequence-length advance. All are HBM/latency bound: one CTA per
// token row, 16-byte vector accesses, fp32 math.
#include <cstdlib>

#include "hx_common.cuh"

namespace hx {

unsigned long long g_launches = 0;

void set_max_carveout(const void *fn) {
  const char *e = getenv("HX_MAX_CARVEOUT");
  if (e && atoi(e) == 0) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
}
int g_pdl = [] {  // HX_PDL=0 turns programmatic dependent launch off (A/B)
  const char *e = getenv("HX_PDL");
  return e ? atoi(e) : 1;
}();

constexpr int ROW_THREADS = 256;

template <typename T>
__global__ void embed_kernel(const int32_t *ids, const T *table, float *x, int hidden, int vocab) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  int id = ids[t];
  id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);
  const T *src = table + (size_t)id * hidden;
  float *dst = x + (size_t)t * hidden;
  constexpr int V = Vec16<T>::N;
  for (int i = threadIdx.x * V; i < hidden; i += blockDim.x * V) {
    float v[V];
    Vec16<T>::load(src + i, v);
#pragma unroll
    for (int j = 0; j < V; j += 4) Vec16<float>::store(dst + i + j, v + j);
  }
}

__device__ __forceinline__ float block_sum(float v, float *red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// x += delta (if delta); out = x / sqrt(mean(x^2) + eps) * gain (if out)
template <typename TO>
__global__ void __launch_bounds__(ROW_THREADS)
    add_rmsnorm_kernel(float *x, long ldx, const float *delta, const float *gain, TO *out, int hidden,
                       float eps) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  const int t = blockIdx.x;
  float *xr = x + (size_t)t * ldx;
  const float *dr = delta ? delta + (size_t)t * hidden : nullptr;
  constexpr int MAXV = 8;  // hidden <= 8 * 4 * 256 = 8192
  float v[MAXV][4], d[MAXV][4], g[MAXV][4];
  // issue every load (x, delta, gain) before the first use
#pragma unroll
  for (int r = 0; r < MAXV; ++r) {
    const int i = (r * ROW_THREADS + threadIdx.x) * 4;
    if (i < hidden) {
      Vec16<float>::load(xr + i, v[r]);
      if (dr) Vec16<float>::load(dr + i, d[r]);
      if (out) Vec16<float>::load(gain + i, g[r]);
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int r = 0; r < MAXV; ++r) {
    const int i = (r * ROW_THREADS + threadIdx.x) * 4;
    if (i < hidden) {
      if (dr) {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[r][j] += d[r][j];
        Vec16<float>::store(xr + i, v[r]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) ss = fmaf(v[r][j], v[r][j], ss);
    }
  }
  if (!out) return;
  const float tot = block_sum(ss, red);
  const float inv = 1.0f / sqrtf(tot / (float)hidden + eps);
  TO *o = out + (size_t)t * hidden;
#pragma unroll
  for (int r = 0; r < MAXV; ++r) {
    const int i = (r * ROW_THREADS + threadIdx.x) * 4;
    if (i < hidden) {
      store4(o + i, (v[r][0] * inv) * g[r][0], (v[r][1] * inv) * g[r][1], (v[r][2] * inv) * g[r][2],
             (v[r][3] * inv) * g[r][3]);
    }
  }
}

template <typename T>
__global__ void swiglu_kernel(const T *gu, T *out, int inter) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.y;
  const T *g = gu + (size_t)t * 2 * inter;
  const T *u = g + inter;
  T *o = out + (size_t)t * inter;
  constexpr int V = Vec16<T>::N;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * V;
  if (i >= inter) return;
  float gv[V], uv[V], r[V];
  Vec16<T>::load(g + i, gv);
  Vec16<T>::load(u + i, uv);
#pragma unroll
  for (int j = 0; j < V; ++j) r[j] = (gv[j] / (1.0f + expf(-gv[j]))) * uv[j];
  Vec16<T>::store(o + i, r);
}

__device__ __forceinline__ unsigned long long pack_key(float v, int idx) {
  uint32_t b = __float_as_uint(v);
  uint32_t ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // unsigned-monotone
  ord ^= 0x80000000u;                                           // signed-monotone
  return ((unsigned long long)ord << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)idx);
}

__global__ void __launch_bounds__(1024)
    argmax_kernel(const float *logits, long long *keys, int n_cols, int ld, int offset) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const float *row = logits + (size_t)t * ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < n_cols; i += blockDim.x) {  // i ascending: strict > keeps the first
    const float v = row[i];
    if (v > best || bi == 0x7fffffff) { best = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sv[w] = best; si[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
      if (sv[i] > best || (sv[i] == best && si[i] < bi)) { best = sv[i]; bi = si[i]; }
    keys[t] = (long long)pack_key(best, bi + offset);
  }
}

__global__ void argmax_finalize_kernel(const long long *keys, int32_t *ids, int32_t *history,
                                       int32_t *step, int s_out, int n_tok, int bump) {
  pdl_trigger();
  pdl_wait();
  const int t = threadIdx.x + blockIdx.x * blockDim.x;
  const int st = history ? *step : 0;
  if (t < n_tok) {
    const uint32_t lo = (uint32_t)((unsigned long long)keys[t] & 0xFFFFFFFFull);
    const int id = (int)(0xFFFFFFFFu - lo);
    ids[t] = id;
    if (history && st < s_out) history[(size_t)t * s_out + st] = id;
  }
  if (history && bump) {
    __syncthreads();
    if (t == 0) *step = st + 1;
  }
}

// No early pdl_trigger: dependents launch only once seq_lens is final, so any
// later kernel may read seq_lens (and KV pages below it) before its own
// griddepcontrol.wait -- the decode attention prefetches pages that way.
__global__ void advance_kernel(int32_t *seq_lens, int batch, int n) {
  pdl_wait();
  const int b = threadIdx.x + blockIdx.x * blockDim.x;
  if (b < batch) seq_lens[b] += n;
}

}  // namespace hx

using namespace hx;

extern "C" int hx_version(void) { return 1; }

extern "C" void hx_set_pdl(int enabled) { g_pdl = enabled ? 1 : 0; }

extern "C" uint64_t hx_launch_count(void) { return g_launches; }

extern "C" const char *hx_error_string(int code) {
  switch (code) {
    case HX_OK: return "ok";
    case HX_ERR_ARG: return "hx: bad argument";
    case HX_ERR_UNSUPPORTED: return "hx: unsupported shape/dtype";
    case HX_ERR_WORKSPACE: return "hx: workspace too small";
    case HX_ERR_DRIVER: return "hx: cuTensorMapEncodeTiled unavailable or failed";
    default: return cudaGetErrorString((cudaError_t)code);
  }
}

extern "C" int hx_embed(const int32_t *ids, const void *table, int table_dtype, float *x, int n_tok,
                        int hidden, int vocab, hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!ids || !table || !x || hidden % 8) return HX_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  if (table_dtype == HX_BF16)
    return launch(embed_kernel<__nv_bfloat16>, dim3(n_tok), dim3(128), 0, st, ids, (const __nv_bfloat16 *)table, x, hidden, vocab);
  else
    return launch(embed_kernel<float>, dim3(n_tok), dim3(128), 0, st, ids, (const float *)table, x, hidden, vocab);
  return launch_status();
}

static int add_rmsnorm(float *x, long ldx, const float *delta, const float *gain, void *out, int out_dtype,
                       int n_tok, int hidden, float eps, hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!x || hidden % 4 || hidden > 8 * 4 * ROW_THREADS || ldx < hidden || ldx % 4) return HX_ERR_ARG;
  if (out && !gain) return HX_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  if (out_dtype == HX_BF16)
    return launch(add_rmsnorm_kernel<__nv_bfloat16>, dim3(n_tok), dim3(ROW_THREADS), 0, st, x, ldx, delta, gain, (__nv_bfloat16 *)out,
                                                                     hidden, eps);
  else
    return launch(add_rmsnorm_kernel<float>, dim3(n_tok), dim3(ROW_THREADS), 0, st, x, ldx, delta, gain, (float *)out, hidden, eps);
  return launch_status();
}

extern "C" int hx_rmsnorm(const float *x, int ldx, const float *gain, void *out, int out_dtype, int n_tok,
                          int hidden, float eps, hx_stream_t stream) {
  if (!out) return HX_ERR_ARG;
  return add_rmsnorm(const_cast<float *>(x), ldx, nullptr, gain, out, out_dtype, n_tok, hidden, eps, stream);
}

extern "C" int hx_residual_add_rmsnorm(float *x, const float *delta, const float *gain, void *out,
                                       int out_dtype, int n_tok, int hidden, float eps,
                                       hx_stream_t stream) {
  if (!delta) return HX_ERR_ARG;
  return add_rmsnorm(x, hidden, delta, gain, out, out_dtype, n_tok, hidden, eps, stream);
}

extern "C" int hx_swiglu(const void *gu, void *out, int dtype, int n_tok, int inter, hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!gu || !out || inter % 8) return HX_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  const int V = dtype == HX_BF16 ? 8 : 4;
  dim3 grid((inter / V + 127) / 128, n_tok);
  if (dtype == HX_BF16)
    return launch(swiglu_kernel<__nv_bfloat16>, dim3(grid), dim3(128), 0, st, (const __nv_bfloat16 *)gu, (__nv_bfloat16 *)out, inter);
  else
    return launch(swiglu_kernel<float>, dim3(grid), dim3(128), 0, st, (const float *)gu, (float *)out, inter);
  return launch_status();
}

extern "C" int hx_advance(int32_t *seq_lens, int batch, int n, hx_stream_t stream) {
  if (batch == 0) return 0;
  if (!seq_lens) return HX_ERR_ARG;
  return launch(advance_kernel, dim3((batch + 127) / 128), dim3(128), 0, as_stream(stream), seq_lens, batch, n);
  return launch_status();
}

extern "C" int hx_argmax_partial(const float *logits, int64_t *keys, int n_tok, int n_cols, int ld,
                                 int vocab_offset, hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!logits || !keys || n_cols <= 0 || ld < n_cols) return HX_ERR_ARG;
  return launch(argmax_kernel, dim3(n_tok), dim3(1024), 0, as_stream(stream), logits, (long long *)keys, n_cols, ld, vocab_offset);
  return launch_status();
}

extern "C" int hx_argmax_finalize(const int64_t *keys, int32_t *ids, int32_t *history, int32_t *step,
                                  int s_out, int n_tok, int bump_step, hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!keys || !ids || (history && !step) || n_tok > 1024) return HX_ERR_ARG;
  return launch(argmax_finalize_kernel, dim3(1), dim3(1024), 0, as_stream(stream), (const long long *)keys, ids, history, step,
                                                            s_out, n_tok, bump_step);
  return launch_status();
}

extern "C" size_t hx_kv_bytes(int dtype, int layers, int num_blocks, int hkv_rank, int page_size, int hd) {
  const size_t el = dtype == HX_BF16 ? 2 : 4;
  return 2 * el * (size_t)layers * num_blocks * hkv_rank * page_size * hd;
}
