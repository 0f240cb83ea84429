// Tensor-core attention for bf16 mode: warp-level
// m16n8k16 MMAs with the online softmax kept in registers.
//
//   attn_prefill_mma_kernel: causal prefill, CTA = 64 queries x 1 head x 1
//     sequence, 4 warps x 16 query rows; K/V 64-key blocks gathered from the
//     paged cache with cp.async into a double-buffered smem ring.
//   attn_decode_mma_kernel: GQA decode (group G >= 2), CTA = (seq, kv head,
//     split); the G query heads of the group form one 16-row query tile (rows
//     >= G are zero), so each K/V byte read from HBM feeds G heads on the
//     tensor core; the 4 warps take 16-key slices of each 64-key block and are
//     merged in smem, splits through the workspace (last-CTA ticket).
// Both are HBM/L2-bound on K/V; fp32 mode and MHA decode use the CUDA-core
// kernels in hx_attention.cu.
#include <cstdlib>

#include <climits>

#include "hx_common.cuh"

namespace hx {

constexpr int AM_BQ = 64, AM_BKV = 64, AM_THREADS = 128;
constexpr int DEC_NS = 3;  // decode K/V ring depth: 2 blocks (64 KB) in flight per CTA, 2 CTAs/SM

template <int HD>
struct AttnSmem {
  static constexpr int LD = HD + 8;  // 16-byte pad: conflict-free ldmatrix rows
  static constexpr int TILE = AM_BKV * LD;
};

// gather a 64-key block of K and V rows (positions p0 + k0 ..) into smem
template <int HD, int THREADS = AM_THREADS>
__device__ __forceinline__ void load_kv_block(__nv_bfloat16 *ks, __nv_bfloat16 *vs, const __nv_bfloat16 *kc,
                                              const __nv_bfloat16 *vc, const int32_t *btb, int p0, int k0,
                                              int klim, int page, int hkv, int kvh) {
  constexpr int LD = AttnSmem<HD>::LD;
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < AM_BKV * CH; i += THREADS) {
    const int r = i / CH, c = (i % CH) * 8;
    const int kj = k0 + r;
    __nv_bfloat16 *kd = ks + r * LD + c, *vd = vs + r * LD + c;
    if (kj < klim) {
      const int pos = p0 + kj;
      const size_t off = (((size_t)btb[pos / page] * hkv + kvh) * page + pos % page) * HD + c;
      cp_async16(kd, kc + off);
      cp_async16(vd, vc + off);
    } else {
      *reinterpret_cast<uint4 *>(kd) = make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4 *>(vd) = make_uint4(0, 0, 0, 0);
    }
  }
}

// S[16 x 8*NT] = Q[16 x HD] . K[keys 16*kr .. , HD]^T for NT n-tiles (NT even)
template <int HD, int NT>
__device__ __forceinline__ void qk_tiles(float (*s)[4], const uint32_t (*qf)[4], const __nv_bfloat16 *ks,
                                         int key_base, int lane) {
  constexpr int LD = AttnSmem<HD>::LD;
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) s[j][e] = 0.f;
#pragma unroll
  for (int jj = 0; jj < NT / 2; ++jj) {
#pragma unroll
    for (int c = 0; c < HD / 16; ++c) {
      const int row = key_base + 16 * jj + (lane & 7) + 8 * (lane >> 4);
      const int col = 16 * c + 8 * ((lane >> 3) & 1);
      uint32_t b0, b1, b2, b3;
      ldsm_x4(smem_u32(ks + row * LD + col), b0, b1, b2, b3);
      mma_bf16_16816(s[2 * jj], qf[c], b0, b1);
      mma_bf16_16816(s[2 * jj + 1], qf[c], b2, b3);
    }
  }
}

// O[16 x HD] += P[16 x 16*KC] . V[keys key_base .., HD]; P from the S tiles
template <int HD, int KC>
__device__ __forceinline__ void pv_tiles(float (*o)[4], const float (*p)[4], const __nv_bfloat16 *vs, int key_base,
                                         int lane) {
  constexpr int LD = AttnSmem<HD>::LD;
#pragma unroll
  for (int kk = 0; kk < KC; ++kk) {
    uint32_t a[4];
    a[0] = pack_bf16(p[2 * kk][0], p[2 * kk][1]);
    a[1] = pack_bf16(p[2 * kk][2], p[2 * kk][3]);
    a[2] = pack_bf16(p[2 * kk + 1][0], p[2 * kk + 1][1]);
    a[3] = pack_bf16(p[2 * kk + 1][2], p[2 * kk + 1][3]);
#pragma unroll
    for (int n = 0; n < HD / 8; n += 2) {
      const int row = key_base + 16 * kk + (lane & 7) + 8 * ((lane >> 3) & 1);
      const int col = 8 * n + 8 * (lane >> 4);
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(smem_u32(vs + row * LD + col), b0, b1, b2, b3);
      mma_bf16_16816(o[n], a, b0, b1);
      mma_bf16_16816(o[n + 1], a, b2, b3);
    }
  }
}

// online softmax over NT n-tiles of S (rows g / g+8 of the warp tile);
// s is replaced by p = exp2(s * sl2 - m) and l accumulates per-thread partials
template <int NT, int HDT>
__device__ __forceinline__ void online_softmax(float (*s)[4], float (*o)[4], float *m, float *l, float sl2) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < NT; ++j) mx = fmaxf(mx, fmaxf(s[j][2 * h], s[j][2 * h + 1]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mn = fmaxf(m[h], mx * sl2);
    const float base = mn == -INFINITY ? 0.f : mn;
    const float corr = exp2f(m[h] - base);
    float rs = 0.f;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      s[j][2 * h] = exp2f(s[j][2 * h] * sl2 - base);
      s[j][2 * h + 1] = exp2f(s[j][2 * h + 1] * sl2 - base);
      rs += s[j][2 * h] + s[j][2 * h + 1];
    }
    l[h] = l[h] * corr + rs;
    m[h] = mn;
#pragma unroll
    for (int n = 0; n < HDT; ++n) {
      o[n][2 * h] *= corr;
      o[n][2 * h + 1] *= corr;
    }
  }
}

// ------------------------------------------------------------------ prefill
// NW warps x 16 query rows per CTA (BQ = 16 NW); K/V 64-key blocks double
// buffered with cp.async and shared by all NW warps (NW = 8: half the K/V smem
// traffic per query row of NW = 4, 16 warps per SM at 2 CTAs/SM)
template <int HD, int NW>
__global__ void __launch_bounds__(32 * NW)
    attn_prefill_mma_kernel(const __nv_bfloat16 *q, const __nv_bfloat16 *kc, const __nv_bfloat16 *vc,
                            const int32_t *bt, const int32_t *seq_lens, __nv_bfloat16 *o, int s_len, int hq,
                            int hkv, int page, int max_blocks, float sl2) {
  pdl_trigger();
  pdl_wait();
  constexpr int LD = AttnSmem<HD>::LD;
  extern __shared__ __align__(128) uint8_t smraw[];
  __nv_bfloat16 *qs = reinterpret_cast<__nv_bfloat16 *>(smraw);
  constexpr int BQ = 16 * NW, THREADS = 32 * NW;
  __nv_bfloat16 *ks = qs + BQ * LD;  // [2][BKV][LD]
  __nv_bfloat16 *vs = ks + 2 * AttnSmem<HD>::TILE;
  const int nqt = gridDim.x;
  const int qt = nqt - 1 - blockIdx.x;  // heaviest (last) query tiles first
  const int h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (hq / hkv);
  const int p0 = seq_lens[b];
  const int q0 = qt * BQ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int32_t *btb = bt + (size_t)b * max_blocks;

  constexpr int CH = HD / 8;
  for (int i = threadIdx.x; i < BQ * CH; i += THREADS) {
    const int r = i / CH, c = (i % CH) * 8;
    __nv_bfloat16 *d = qs + r * LD + c;
    if (q0 + r < s_len)
      cp_async16(d, q + (((size_t)b * s_len + q0 + r) * hq + h) * HD + c);
    else
      *reinterpret_cast<uint4 *>(d) = make_uint4(0, 0, 0, 0);
  }
  const int q_hi = min(s_len, q0 + BQ);
  const int nblk = (q_hi + AM_BKV - 1) / AM_BKV;
  load_kv_block<HD, THREADS>(ks, vs, kc, vc, btb, p0, 0, s_len, page, hkv, kvh);
  cp_async_commit();

  uint32_t qf[HD / 16][4];
  float oacc[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) oacc[n][e] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  const int qa = q0 + 16 * warp + g;  // this thread's two query rows: qa, qa + 8

  for (int kb = 0; kb < nblk; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nblk) {
      load_kv_block<HD, THREADS>(ks + (buf ^ 1) * AttnSmem<HD>::TILE, vs + (buf ^ 1) * AttnSmem<HD>::TILE, kc, vc, btb, p0,
                        (kb + 1) * AM_BKV, s_len, page, hkv, kvh);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int c = 0; c < HD / 16; ++c) {
        const int row = 16 * warp + (lane & 7) + 8 * ((lane >> 3) & 1);
        const int col = 16 * c + 8 * (lane >> 4);
        ldsm_x4(smem_u32(qs + row * LD + col), qf[c][0], qf[c][1], qf[c][2], qf[c][3]);
      }
    }
    const __nv_bfloat16 *kb_s = ks + buf * AttnSmem<HD>::TILE;
    const __nv_bfloat16 *vb_s = vs + buf * AttnSmem<HD>::TILE;
    const int k0 = kb * AM_BKV;
    if (k0 <= q0 + 16 * warp + 15) {  // warp-uniform causal skip of fully masked blocks
      float s[8][4];
      qk_tiles<HD, 8>(s, qf, kb_s, 0, lane);
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int kj = k0 + 8 * j + 2 * t4 + (e & 1);
          const int qi = qa + 8 * (e >> 1);
          if (kj > qi || kj >= s_len) s[j][e] = -INFINITY;
        }
      online_softmax<8, HD / 8>(s, oacc, m, l, sl2);
      pv_tiles<HD, 4>(oacc, s, vb_s, 0, lane);
    }
    __syncthreads();
  }
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 1);
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 2);
  }
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int qi = qa + 8 * hh;
    if (qi >= s_len) continue;
    const float inv = 1.f / l[hh];
    __nv_bfloat16 *dst = o + (((size_t)b * s_len + qi) * hq + h) * HD;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
      *reinterpret_cast<uint32_t *>(dst + 8 * n + 2 * t4) = pack_bf16(oacc[n][2 * hh] * inv, oacc[n][2 * hh + 1] * inv);
  }
}

// ------------------------------------------------------------------ decode (GQA)
template <int HD, int G>
__global__ void __launch_bounds__(AM_THREADS)
    attn_decode_mma_kernel(const __nv_bfloat16 *q, const __nv_bfloat16 *kc, const __nv_bfloat16 *vc,
                           const int32_t *bt, const int32_t *seq_lens, __nv_bfloat16 *o, int hkv, int page,
                           int max_blocks, float sl2, float *ws, int *counters) {
  pdl_trigger();
  pdl_wait();
  constexpr int LD = AttnSmem<HD>::LD;
  extern __shared__ __align__(128) uint8_t smraw[];
  __nv_bfloat16 *qs = reinterpret_cast<__nv_bfloat16 *>(smraw);  // [16][LD]
  __nv_bfloat16 *ks = qs + 16 * LD;                                // [DEC_NS][BKV][LD]
  __nv_bfloat16 *vs = ks + DEC_NS * AttnSmem<HD>::TILE;
  float *red = reinterpret_cast<float *>(ks);  // [4 warps][16 rows][HD + 2], reuses K/V after the loop
  const int b = blockIdx.x / hkv, kvh = blockIdx.x % hkv;
  const int split = blockIdx.y, splits = gridDim.y;
  const int hq = hkv * G;
  const int ctx = seq_lens[b] + 1;
  const int chunk = (ctx + splits - 1) / splits;
  const int t0 = split * chunk, t1 = min(ctx, t0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int32_t *btb = bt + (size_t)b * max_blocks;

  constexpr int CH = HD / 8;
  for (int i = threadIdx.x; i < 16 * CH; i += AM_THREADS) {
    const int r = i / CH, c = (i % CH) * 8;
    __nv_bfloat16 *d = qs + r * LD + c;
    if (r < G)
      cp_async16(d, q + ((size_t)b * hq + kvh * G + r) * HD + c);
    else
      *reinterpret_cast<uint4 *>(d) = make_uint4(0, 0, 0, 0);
  }
  // DEC_NS-deep cp.async ring of 64-key K/V blocks (group 0 also carries Q)
  const int nblk = t1 > t0 ? (t1 - t0 + AM_BKV - 1) / AM_BKV : 0;
#pragma unroll
  for (int i = 0; i < DEC_NS - 1; ++i) {
    if (i < nblk)
      load_kv_block<HD>(ks + i * AttnSmem<HD>::TILE, vs + i * AttnSmem<HD>::TILE, kc, vc, btb, 0, t0 + i * AM_BKV, t1,
                        page, hkv, kvh);
    cp_async_commit();
  }
  uint32_t qf[HD / 16][4];
  float oacc[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) oacc[n][e] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  if (nblk == 0) {
    cp_async_wait<0>();
    __syncthreads();
  }
  for (int kb = 0; kb < nblk; ++kb) {
    cp_async_wait<DEC_NS - 2>();  // block kb (and, at kb = 0, Q) has landed
    __syncthreads();               // ... and every warp is done with block kb - 1's buffer
    if (kb == 0) {
#pragma unroll
      for (int c = 0; c < HD / 16; ++c) {
        const int row = (lane & 7) + 8 * ((lane >> 3) & 1);
        const int col = 16 * c + 8 * (lane >> 4);
        ldsm_x4(smem_u32(qs + row * LD + col), qf[c][0], qf[c][1], qf[c][2], qf[c][3]);
      }
    }
    const int nb = kb + DEC_NS - 1;
    if (nb < nblk)
      load_kv_block<HD>(ks + (nb % DEC_NS) * AttnSmem<HD>::TILE, vs + (nb % DEC_NS) * AttnSmem<HD>::TILE, kc, vc,
                        btb, 0, t0 + nb * AM_BKV, t1, page, hkv, kvh);
    cp_async_commit();
    const int buf = kb % DEC_NS;
    const int k0 = t0 + kb * AM_BKV + 16 * warp;  // this warp's 16 keys
    if (k0 < t1) {
      float s[2][4];
      qk_tiles<HD, 2>(s, qf, ks + buf * AttnSmem<HD>::TILE, 16 * warp, lane);
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (k0 + 8 * j + 2 * t4 + (e & 1) >= t1) s[j][e] = -INFINITY;
      online_softmax<2, HD / 8>(s, oacc, m, l, sl2);
      pv_tiles<HD, 1>(oacc, s, vs + buf * AttnSmem<HD>::TILE, 16 * warp, lane);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // all warps done with K/V before `red` reuses that smem
  // merge the 4 warps: per row (head) m, l and O
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 1);
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 2);
  }
  float *wr = red + (size_t)warp * 16 * (HD + 2);
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int r = g + 8 * hh;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      wr[r * (HD + 2) + 8 * n + 2 * t4] = oacc[n][2 * hh];
      wr[r * (HD + 2) + 8 * n + 2 * t4 + 1] = oacc[n][2 * hh + 1];
    }
    if (t4 == 0) {
      wr[r * (HD + 2) + HD] = m[hh];
      wr[r * (HD + 2) + HD + 1] = l[hh];
    }
  }
  __syncthreads();
  const size_t pair = (size_t)b * hkv + kvh;
  for (int w = threadIdx.x; w < G * HD; w += AM_THREADS) {
    const int r = w / HD, d = w % HD;
    float M = -INFINITY;
#pragma unroll
    for (int i = 0; i < 4; ++i) M = fmaxf(M, red[(i * 16 + r) * (HD + 2) + HD]);
    float L = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float c = exp2f(red[(i * 16 + r) * (HD + 2) + HD] - M);
        L += red[(i * 16 + r) * (HD + 2) + HD + 1] * c;
        A += red[(i * 16 + r) * (HD + 2) + d] * c;
      }
    }
    if (splits == 1) {
      o[((size_t)b * hq + kvh * G + r) * HD + d] = __float2bfloat16_rn(A / L);
    } else {
      float *part = ws + ((pair * splits + split) * G + r) * (HD + 2);
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
  for (int w = threadIdx.x; w < G * HD; w += AM_THREADS) {
    const int r = w / HD, d = w % HD;
    float M = -INFINITY;
    for (int s2 = 0; s2 < splits; ++s2) M = fmaxf(M, __ldcg(ws + ((pair * splits + s2) * G + r) * (HD + 2) + HD));
    float L = 0.f, A = 0.f;
    for (int s2 = 0; s2 < splits; ++s2) {
      const float *part = ws + ((pair * splits + s2) * G + r) * (HD + 2);
      const float ms = __ldcg(part + HD);
      if (ms == -INFINITY) continue;
      const float c = exp2f(ms - M);
      L += __ldcg(part + HD + 1) * c;
      A += __ldcg(part + d) * c;
    }
    o[((size_t)b * hq + kvh * G + r) * HD + d] = __float2bfloat16_rn(A / L);
  }
}

// ------------------------------------------------------------------ decode, TMA-fed (hd 128, page 64)
// Same math as attn_decode_mma_kernel, but each 64-key block of one KV head --
// one contiguous 16 KB page slice in the paged layout -- arrives by TMA (two
// 64-column 128B-swizzled boxes for K, two for V) into a DEC_NS-deep mbarrier
// ring: 4 instructions per block instead of 2048 cp.async, so the warps only
// issue ldmatrix / mma / softmax. ldmatrix addresses apply the same XOR swizzle.
unsigned long long *hx_trace_slots(size_t n);  // hx_gemm.cu (hx_debug_trace)
__device__ __forceinline__ unsigned long long attn_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t sw128_addr(uint32_t base, int r, int col) {
  const int half = col >> 6, chunk = (col & 63) >> 3;
  return base + half * 8192 + r * 128 + ((chunk ^ (r & 7)) << 4) + ((col & 7) << 1);
}

// DEF (with ROPE): the QKV projection was a deferred stream-K GEMM
// (HX_LINEAR_DEFER_REDUCE, fp32 output `q` with row pitch ldq): its split tiles
// are summed here from the GEMM's partial slots, in CTA order, and rounded to
// bf16 -- the bits the GEMM's own fix-up would have stored -- so the GEMM ends
// without its serial fix-up tail. A head is one 128-row tile; its contributor
// range (tl) is computed once per CTA before the dependency wait. A thread
// gathers features i0..i0+3 and i0+64..i0+67 of one head (a RoPE rotate-half
// quad pair) with 16-byte loads, every contributor's loads in flight together.
__device__ __forceinline__ void gather_quad_pair(const SKView &v, const float *y, long ldy, int b, int head, int i0,
                                                 const SkTile &ti, float (&lo)[4], float (&hi)[4]) {
  float4 l = make_float4(0.f, 0.f, 0.f, 0.f), h = l;
  if (ti.whole()) {
    const float *src = y + (long)b * ldy + head * kSkRows + i0;
    l = *reinterpret_cast<const float4 *>(src);
    h = *reinterpret_cast<const float4 *>(src + 64);
  } else {
    constexpr int MAXC = 10;
    for (int cb = ti.c_first; cb <= ti.c_last; cb += MAXC) {
      float4 fl[MAXC], fh[MAXC];
#pragma unroll
      for (int k = 0; k < MAXC; ++k)
        if (cb + k <= ti.c_last) {
          const float *src = v.ws + ((size_t)ti.slot(cb + k) * v.BN + b) * kSkRows + i0;
          fl[k] = __ldcg(reinterpret_cast<const float4 *>(src));
          fh[k] = __ldcg(reinterpret_cast<const float4 *>(src + 64));
        }
#pragma unroll
      for (int k = 0; k < MAXC; ++k)
        if (cb + k <= ti.c_last) {
          l.x += fl[k].x; l.y += fl[k].y; l.z += fl[k].z; l.w += fl[k].w;
          h.x += fh[k].x; h.y += fh[k].y; h.z += fh[k].z; h.w += fh[k].w;
        }
    }
  }
  const float lv[4] = {l.x, l.y, l.z, l.w}, hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {  // the bf16 value the GEMM would have stored
    lo[j] = __bfloat162float(__float2bfloat16_rn(lv[j]));
    hi[j] = __bfloat162float(__float2bfloat16_rn(hv[j]));
  }
}

template <int G, bool ROPE, int NS, int BPI, bool CL, bool DEF = false>
__global__ void __launch_bounds__(AM_THREADS * BPI)
    attn_decode_tma_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                           const __nv_bfloat16 *q, const int32_t *bt, const int32_t *seq_lens, __nv_bfloat16 *o,
                           int hkv, int max_blocks, float sl2, float *ws, int *counters, __nv_bfloat16 *kc,
                           __nv_bfloat16 *vc, float theta, SKView skv, long ldq, unsigned long long *trace, int prewait) {
  constexpr int HD = 128, LD = HD + 8, PAGE = 64;
  constexpr uint32_t BLK = PAGE * HD * 2;  // 16 KB per tensor per block
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *ring = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  // ring: [NS][K 16 KB | V 16 KB]; then Q tile; then barriers
  __nv_bfloat16 *qs = reinterpret_cast<__nv_bfloat16 *>(ring + NS * 2 * BLK);
  uint64_t *full = reinterpret_cast<uint64_t *>(qs + 16 * LD);
  float *red = reinterpret_cast<float *>(ring);  // [4 warps][16][HD + 2], reuses the ring at the end
  float *mypart = red + 4 * BPI * 16 * (HD + 2);  // [G][HD + 2] this split's combined partial (CL)
  __shared__ int s_last;
  pdl_trigger();
  // hx_debug_trace: start, wait done, end, smid | 1 << 40, q ready, loop done, partials combined, nblk
  unsigned long long *tr = trace ? trace + 8 * (blockIdx.x + (size_t)blockIdx.y * gridDim.x) : nullptr;
  auto stamp = [&](int f) {
    if (tr && threadIdx.x == 0) tr[f] = attn_globaltimer();
  };
  stamp(0);
  // CL: the splits of one (batch, kv-head) pair form a thread-block cluster and
  // combine through DSMEM; otherwise grid.y = splits and the last split to
  // finish (ticket) combines through the workspace
  const int splits = CL ? (int)cluster_nctarank() : (int)gridDim.y;
  const int split = CL ? (int)cluster_rank() : (int)blockIdx.y;
  const int pidx = CL ? (int)blockIdx.x / splits : (int)blockIdx.x;
  const int b = pidx / hkv, kvh = pidx % hkv;
  const int hq = hkv * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  // Before waiting on the producer of q / the new token's K,V: seq_lens and the
  // block table are only written by hx_advance (which lets dependents launch only
  // at its exit) and by the host, and every position < seq_lens[b] was appended in
  // an earlier step -- so the pages wholly before the new token's page stream in
  // while the QKV GEMM is still running.
  const int pos = seq_lens[b];  // the new token's position
  const int ctx = pos + 1;
  int chunk = (ctx + splits - 1) / splits;
  chunk = (chunk + PAGE - 1) / PAGE * PAGE;  // page-aligned split ranges
  const int t0 = split * chunk, t1 = min(ctx, t0 + chunk);
  const int nblk = t1 > t0 ? (t1 - t0 + PAGE - 1) / PAGE : 0;
  const int32_t *btb = bt + (size_t)b * max_blocks;
  const int safe = min(nblk, max(0, pos / PAGE - t0 / PAGE));  // blocks not holding the new token
  const uint64_t pol = l2_policy_evict_first();  // each K/V byte is read once per step
  // this CTA's block-table entries, fetched by many threads at once (one
  // dependent L2 round trip instead of one per TMA issue of thread 0)
  constexpr int kMaxBt = 64;  // 64-key blocks per split (contexts up to 4096 tokens per split)
  __shared__ int bts[kMaxBt];
  for (int i = threadIdx.x; i < nblk && i < kMaxBt; i += AM_THREADS * BPI) bts[i] = btb[t0 / PAGE + i];
  // DEF: the contributor ranges of this pair's G q heads, its k head and v head
  // (GEMM geometry only -- independent of the producer's data)
  __shared__ SkTile s_tiles[DEF ? G + 2 : 1];
  if constexpr (DEF) {
    if (threadIdx.x < G + 2) {
      const int h = threadIdx.x < G ? kvh * G + threadIdx.x : hq + (threadIdx.x == G ? 0 : hkv) + kvh;
      s_tiles[threadIdx.x] = sk_tile(skv, h);
    }
  }
  // RoPE angles of the new position (pos is known before the wait): feature
  // threadIdx % 64 (ROPE), features 4 (threadIdx % 16) + 0..3 (DEF)
  float rope_sn = 0.f, rope_cs = 0.f;
  float qsn[4], qcs[4];
  if constexpr (DEF) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float inv_freq = 1.0f / powf(theta, (float)(2 * (4 * (threadIdx.x & 15) + j)) / 128.0f);
      sincosf((float)pos * inv_freq, &qsn[j], &qcs[j]);
    }
  } else if constexpr (ROPE) {
    const float inv_freq = 1.0f / powf(theta, (float)(2 * (threadIdx.x & 63)) / 128.0f);
    sincosf((float)pos * inv_freq, &rope_sn, &rope_cs);
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int s = i % NS;
    const int row = ((i < kMaxBt ? bts[i] : btb[t0 / PAGE + i]) * hkv + kvh) * PAGE;
    uint8_t *kd = ring + s * 2 * BLK, *vd = kd + BLK;
    mbar_arrive_expect_tx(&full[s], 2 * BLK);
    tma_load_2d(kd, &tmk, &full[s], 0, row, pol);
    tma_load_2d(kd + BLK / 2, &tmk, &full[s], 64, row, pol);
    tma_load_2d(vd, &tmv, &full[s], 0, row, pol);
    tma_load_2d(vd + BLK / 2, &tmv, &full[s], 64, row, pol);
  };
  const int pre = min(min(NS, prewait), safe);
  if (threadIdx.x == 0) {
    tma_prefetch(&tmk);
    tma_prefetch(&tmv);
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    for (int i = 0; i < pre; ++i) issue(i);
  }
  pdl_wait();
  stamp(1);
  if (tr && threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    tr[3] = sm | (1ull << 40);
    tr[7] = (unsigned long long)nblk | ((unsigned long long)split << 16);
    tr[2] = 0;
  }
  if constexpr (DEF) {
    static_assert(ROPE, "the deferred QKV path is the fused RoPE + KV-append path");
    const float *y = reinterpret_cast<const float *>(q);
    const int i0 = 4 * (threadIdx.x & 15);
    for (int e = threadIdx.x; e < (16 - G) * (HD / 8); e += AM_THREADS * BPI)  // zero padding rows G..15
      *reinterpret_cast<uint4 *>(qs + (G + e / (HD / 8)) * LD + (e % (HD / 8)) * 8) = make_uint4(0, 0, 0, 0);
    for (int r = threadIdx.x >> 4; r < G; r += AM_THREADS * BPI / 16) {
      float lo[4], hi[4];
      gather_quad_pair(skv, y, ldq, b, kvh * G + r, i0, s_tiles[r], lo, hi);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 yy = rope_rot(lo[j], hi[j], qcs[j], qsn[j]);
        qs[r * LD + i0 + j] = __float2bfloat16_rn(yy.x);
        qs[r * LD + i0 + 64 + j] = __float2bfloat16_rn(yy.y);
      }
    }
    if (t0 <= pos && pos < t1 && threadIdx.x < 32) {  // threads 0-15: the new k, 16-31: the new v
      const size_t slot = (((size_t)btb[pos / PAGE] * hkv + kvh) * PAGE + pos % PAGE) * HD;
      const bool is_k = threadIdx.x < 16;
      float lo[4], hi[4];
      gather_quad_pair(skv, y, ldq, b, (is_k ? hq : hq + hkv) + kvh, i0, s_tiles[is_k ? G : G + 1], lo, hi);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (is_k) {
          const float2 yy = rope_rot(lo[j], hi[j], qcs[j], qsn[j]);
          kc[slot + i0 + j] = __float2bfloat16_rn(yy.x);
          kc[slot + i0 + 64 + j] = __float2bfloat16_rn(yy.y);
        } else {
          vc[slot + i0 + j] = __float2bfloat16_rn(lo[j]);
          vc[slot + i0 + 64 + j] = __float2bfloat16_rn(hi[j]);
        }
      }
      fence_proxy_async_global();  // the page is about to be read back by TMA
    }
  } else if constexpr (ROPE) {
    // q rows straight from the packed qkv row, rotated here (rotate-half pairs
    // (i, i + 64), same fp32 arithmetic as rope_append_kernel); the CTA whose
    // range holds the new token also rotates its k and appends k, v to the page
    const int i = threadIdx.x & 63;
    const __nv_bfloat16 *row = q + (size_t)b * (hq + 2 * hkv) * HD;
    const float sn = rope_sn, cs = rope_cs;
    constexpr int STEP = AM_THREADS * BPI / 64;   // q rows per pass
    constexpr int NR = (16 + STEP - 1) / STEP;   // passes
    __nv_bfloat16 x1r[NR], x2r[NR];
    const int r0 = threadIdx.x >> 6;
#pragma unroll
    for (int k = 0; k < NR; ++k) {  // every load in flight before any is used
      const int r = r0 + k * STEP;
      if (r < G) {
        x1r[k] = row[(kvh * G + r) * HD + i];
        x2r[k] = row[(kvh * G + r) * HD + i + 64];
      }
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      const int r = r0 + k * STEP;
      if (r >= 16) continue;
      float y1 = 0.f, y2 = 0.f;
      if (r < G) {
        const float2 y = rope_rot(to_f32(x1r[k]), to_f32(x2r[k]), cs, sn);
        y1 = y.x;
        y2 = y.y;
      }
      qs[r * LD + i] = __float2bfloat16_rn(y1);
      qs[r * LD + i + 64] = __float2bfloat16_rn(y2);
    }
    if (t0 <= pos && pos < t1) {
      const size_t slot = (((size_t)btb[pos / PAGE] * hkv + kvh) * PAGE + pos % PAGE) * HD;
      if (threadIdx.x < 64) {
        const float x1 = to_f32(row[(hq + kvh) * HD + i]), x2 = to_f32(row[(hq + kvh) * HD + i + 64]);
        const float2 y = rope_rot(x1, x2, cs, sn);
        kc[slot + i] = __float2bfloat16_rn(y.x);
        kc[slot + i + 64] = __float2bfloat16_rn(y.y);
      } else {
        vc[slot + i] = row[(hq + hkv + kvh) * HD + i];
        vc[slot + i + 64] = row[(hq + hkv + kvh) * HD + i + 64];
      }
      fence_proxy_async_global();  // the page is about to be read back by TMA
    }
  } else {
    for (int i = threadIdx.x; i < 16 * (HD / 8); i += AM_THREADS * BPI) {
      const int r = i / (HD / 8), c = (i % (HD / 8)) * 8;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < G) v = *reinterpret_cast<const uint4 *>(q + ((size_t)b * hq + kvh * G + r) * HD + c);
      *reinterpret_cast<uint4 *>(qs + r * LD + c) = v;
    }
  }
  __syncthreads();
  stamp(4);
  int issued = pre;  // meaningful in thread 0 only
  if (threadIdx.x == 0)
    for (; issued < NS && issued < nblk; ++issued) issue(issued);
  uint32_t qf[HD / 16][4];
#pragma unroll
  for (int c = 0; c < HD / 16; ++c) {
    const int row = (lane & 7) + 8 * ((lane >> 3) & 1);
    const int col = 16 * c + 8 * (lane >> 4);
    ldsm_x4(smem_u32(qs + row * LD + col), qf[c][0], qf[c][1], qf[c][2], qf[c][3]);
  }
  float oacc[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) oacc[n][e] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  // BPI blocks per iteration: warp w takes 16 keys of block kb0 + w / 4
  const int wb = warp >> 2, wk = warp & 3;
  for (int kb0 = 0; kb0 < nblk; kb0 += BPI) {
    if (kb0 > 0) __syncthreads();  // every warp is done with the previous iteration's stages
    if (threadIdx.x == 0)
      for (; issued < nblk && issued < kb0 + NS; ++issued) issue(issued);
    const int kb = kb0 + wb;
    const int s = kb % NS;
    const int k0 = t0 + kb * PAGE + 16 * wk;  // this warp's 16 keys
    if (kb < nblk) mbar_wait(&full[s], (kb / NS) & 1);
    const uint32_t kbase = smem_u32(ring + s * 2 * BLK), vbase = kbase + BLK;
    if (kb < nblk && k0 < t1) {
      float sc[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[j][e] = 0.f;
#pragma unroll
      for (int c = 0; c < HD / 16; ++c) {
        const int row = 16 * wk + (lane & 7) + 8 * (lane >> 4);
        const int col = 16 * c + 8 * ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sw128_addr(kbase, row, col), b0, b1, b2, b3);
        mma_bf16_16816(sc[0], qf[c], b0, b1);
        mma_bf16_16816(sc[1], qf[c], b2, b3);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (k0 + 8 * j + 2 * t4 + (e & 1) >= t1) sc[j][e] = -INFINITY;
      online_softmax<2, HD / 8>(sc, oacc, m, l, sl2);
      uint32_t a[4];
      a[0] = pack_bf16(sc[0][0], sc[0][1]);
      a[1] = pack_bf16(sc[0][2], sc[0][3]);
      a[2] = pack_bf16(sc[1][0], sc[1][1]);
      a[3] = pack_bf16(sc[1][2], sc[1][3]);
#pragma unroll
      for (int n = 0; n < HD / 8; n += 2) {
        const int row = 16 * wk + (lane & 7) + 8 * ((lane >> 3) & 1);
        const int col = 8 * n + 8 * (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sw128_addr(vbase, row, col), b0, b1, b2, b3);
        mma_bf16_16816(oacc[n], a, b0, b1);
        mma_bf16_16816(oacc[n + 1], a, b2, b3);
      }
    }
  }
  __syncthreads();  // ring no longer read: `red` may overwrite it
  stamp(5);
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 1);
    l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], 2);
  }
  float *wr = red + (size_t)warp * 16 * (HD + 2);
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int r = g + 8 * hh;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      wr[r * (HD + 2) + 8 * n + 2 * t4] = oacc[n][2 * hh];
      wr[r * (HD + 2) + 8 * n + 2 * t4 + 1] = oacc[n][2 * hh + 1];
    }
    if (t4 == 0) {
      wr[r * (HD + 2) + HD] = m[hh];
      wr[r * (HD + 2) + HD + 1] = l[hh];
    }
  }
  __syncthreads();
  const size_t pair = (size_t)b * hkv + kvh;
  for (int w = threadIdx.x; w < G * HD; w += AM_THREADS * BPI) {
    const int r = w / HD, d = w % HD;
    float M = -INFINITY;
#pragma unroll
    for (int i = 0; i < 4 * BPI; ++i) M = fmaxf(M, red[(i * 16 + r) * (HD + 2) + HD]);
    float L = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int i = 0; i < 4 * BPI; ++i) {
        const float c = exp2f(red[(i * 16 + r) * (HD + 2) + HD] - M);
        L += red[(i * 16 + r) * (HD + 2) + HD + 1] * c;
        A += red[(i * 16 + r) * (HD + 2) + d] * c;
      }
    }
    if (splits == 1) {
      o[((size_t)b * hq + kvh * G + r) * HD + d] = __float2bfloat16_rn(A / L);
    } else {
      float *part = CL ? mypart + r * (HD + 2) : ws + ((pair * splits + split) * G + r) * (HD + 2);
      part[d] = A;
      if (d == 0) { part[HD] = M; part[HD + 1] = L; }
    }
  }
  if (splits == 1) {
    stamp(2);
    return;
  }
  if constexpr (CL) {
    // every split's (A, M, L) sits in its own smem: combine across the cluster
    // over DSMEM, each CTA producing an interleaved 1/splits of the outputs
    cluster_sync_all();
    stamp(6);
    for (int w = split * AM_THREADS * BPI + threadIdx.x; w < G * HD; w += splits * AM_THREADS * BPI) {
      const int r = w / HD, d = w % HD;
      constexpr int MAXS = 8;  // cluster splits are 2..8
      float ms[MAXS], ls[MAXS], as[MAXS];
#pragma unroll
      for (int c2 = 0; c2 < MAXS; ++c2) {  // all remote loads in flight before any is used
        if (c2 < splits) {
          ms[c2] = dsmem_ld_f32(mypart + r * (HD + 2) + HD, c2);
          ls[c2] = dsmem_ld_f32(mypart + r * (HD + 2) + HD + 1, c2);
          as[c2] = dsmem_ld_f32(mypart + r * (HD + 2) + d, c2);
        }
      }
      float M = -INFINITY;
#pragma unroll
      for (int c2 = 0; c2 < MAXS; ++c2)
        if (c2 < splits) M = fmaxf(M, ms[c2]);
      float L = 0.f, A = 0.f;
#pragma unroll
      for (int c2 = 0; c2 < MAXS; ++c2) {
        if (c2 >= splits || ms[c2] == -INFINITY) continue;
        const float cf = exp2f(ms[c2] - M);
        L += ls[c2] * cf;
        A += as[c2] * cf;
      }
      o[((size_t)b * hq + kvh * G + r) * HD + d] = __float2bfloat16_rn(A / L);
    }
    cluster_sync_all();  // peers have read this CTA's partial before it exits
    stamp(2);
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int tk = ticket_acq_rel(&counters[pair]);
    s_last = tk == splits - 1;
    if (s_last) counters[pair] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  // combine the splits: all (m, l) pairs into smem first, then one scale per
  // (row, split), then the rows with every split's loads independent (the
  // split-combine tail is latency-bound: no load may wait on another)
  float *ml = red;                       // [splits][G] x (m -> scale, l)
  float *lsum = red + 2 * G * splits;    // [G]
  const float *wsp = ws + pair * splits * G * (HD + 2);
  for (int i = threadIdx.x; i < G * splits; i += AM_THREADS * BPI) {
    const float2 v = __ldcg(reinterpret_cast<const float2 *>(wsp + (size_t)i * (HD + 2) + HD));
    ml[2 * i] = v.x;
    ml[2 * i + 1] = v.y;
  }
  __syncthreads();
  if (threadIdx.x < G) {
    const int r = threadIdx.x;
    float M = -INFINITY;
    for (int s2 = 0; s2 < splits; ++s2) M = fmaxf(M, ml[2 * (s2 * G + r)]);
    float L = 0.f;
    for (int s2 = 0; s2 < splits; ++s2) {
      const float ms = ml[2 * (s2 * G + r)];
      const float c = ms == -INFINITY ? 0.f : exp2f(ms - M);
      L += ml[2 * (s2 * G + r) + 1] * c;
      ml[2 * (s2 * G + r)] = c;
    }
    lsum[r] = L;
  }
  __syncthreads();
#pragma unroll 4
  for (int w = threadIdx.x; w < G * HD / 2; w += AM_THREADS * BPI) {
    const int r = w / (HD / 2), d = (w % (HD / 2)) * 2;
    float2 A = make_float2(0.f, 0.f);
    for (int s2 = 0; s2 < splits; ++s2) {
      const float c = ml[2 * (s2 * G + r)];
      if (c == 0.f) continue;
      const float2 p = __ldcg(reinterpret_cast<const float2 *>(wsp + (size_t)(s2 * G + r) * (HD + 2) + d));
      A.x += p.x * c;
      A.y += p.y * c;
    }
    const float L = lsum[r];
    __nv_bfloat16 *dst = o + ((size_t)b * hq + kvh * G + r) * HD + d;
    dst[0] = __float2bfloat16_rn(A.x / L);
    dst[1] = __float2bfloat16_rn(A.y / L);
  }
}

template <int G, bool ROPE, int NS, int BPI, bool CL = false, bool DEF = false>
static int launch_decode_tma_g(dim3 grid, const CUtensorMap &mk, const CUtensorMap &mv, const void *q,
                               const int32_t *bt, const int32_t *sl, void *o, int hkv, int maxb, float *ws, int *cnt,
                               void *kc, void *vc, float theta, cudaStream_t st, const SKView &skv = SKView{},
                               long ldq = 0) {
  const size_t smem = 1024 + NS * 2 * 16384 + 16 * 136 * 2 + NS * 8 + 16;
  auto kern = attn_decode_tma_kernel<G, ROPE, NS, BPI, CL, DEF>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const float sl2 = 1.4426950408889634f / sqrtf(128.f);
  unsigned long long *tr = hx_trace_slots((size_t)grid.x * grid.y);
  static const int prewait = [] {  // KV blocks streamed before the dependency wait (HX_ATTN_PREWAIT, tuning)
    const char *e = getenv("HX_ATTN_PREWAIT");
    return e ? atoi(e) : NS;
  }();
  if constexpr (CL)
    return launch_cluster(kern, dim3(grid.x * grid.y), dim3(AM_THREADS * BPI), smem, st, (int)grid.y, mk, mv,
                          (const __nv_bfloat16 *)q, bt, sl, (__nv_bfloat16 *)o, hkv, maxb, sl2, ws, cnt,
                          (__nv_bfloat16 *)kc, (__nv_bfloat16 *)vc, theta, skv, ldq, tr, prewait);
  return launch(kern, grid, dim3(AM_THREADS * BPI), smem, st, mk, mv, (const __nv_bfloat16 *)q, bt, sl,
                (__nv_bfloat16 *)o, hkv, maxb, sl2, ws, cnt, (__nv_bfloat16 *)kc, (__nv_bfloat16 *)vc, theta, skv, ldq,
                tr, prewait);
}

static const int g_attn_cluster = [] {  // split-KV combine over DSMEM clusters (HX_ATTN_CLUSTER=0: workspace)
  const char *e = getenv("HX_ATTN_CLUSTER");
  return e ? atoi(e) : 1;
}();

// kc/vc: [num_blocks][hkv][64][128] bf16. rope: q is the packed qkv row and the
// new token's k (rotated) and v are appended by the kernel itself.
int launch_decode_tma(int G, dim3 grid, const void *q, const void *kc, const void *vc, const int32_t *bt,
                      const int32_t *sl, void *o, int hkv, int maxb, float *ws, int *cnt, bool rope, float theta,
                      cudaStream_t st, int ns, const SKView *skv, long ldq) {
  CUtensorMap mk, mv;
  // the pool size is not part of the C-ABI: declare 2^28 rows (64 GB of K); only
  // rows of blocks named by the block table are ever addressed
  const long rows = 1l << 28;
  int rc = make_tma_bf16_sw128(&mk, kc, rows, 128, 128, 64);
  if (!rc) rc = make_tma_bf16_sw128(&mv, vc, rows, 128, 128, 64);
  if (rc) return rc;
  void *k = const_cast<void *>(kc), *v = const_cast<void *>(vc);
  if (skv) {  // deferred QKV (fused RoPE + KV append), 3-deep ring, 1 block per iteration
    if (!rope || ns == 6) return HX_ERR_UNSUPPORTED;
#define HX_TMA_DEF(GG)                                                                                              \
  if (ns == 2)                                                                                                     \
    return grid.y >= 2 && grid.y <= 8                                                                              \
               ? launch_decode_tma_g<GG, true, 2, 1, true, true>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, \
                                                                 theta, st, *skv, ldq)                             \
               : launch_decode_tma_g<GG, true, 2, 1, false, true>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k,  \
                                                                  v, theta, st, *skv, ldq);                        \
  if (grid.y >= 2 && grid.y <= 8 && g_attn_cluster)                                                               \
    return launch_decode_tma_g<GG, true, 3, 1, true, true>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, \
                                                           st, *skv, ldq);                                          \
  return launch_decode_tma_g<GG, true, 3, 1, false, true>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, \
                                                          st, *skv, ldq)
    switch (G) {
      case 1: HX_TMA_DEF(1);
      case 2: HX_TMA_DEF(2);
      case 4: HX_TMA_DEF(4);
      case 8: HX_TMA_DEF(8);
      case 16: HX_TMA_DEF(16);
    }
#undef HX_TMA_DEF
    return HX_ERR_UNSUPPORTED;
  }
#define HX_TMA_G(GG)                                                                                               \
  if (ns == 2 && rope)                                                                                             \
    return grid.y >= 2 && grid.y <= 8                                                                              \
               ? launch_decode_tma_g<GG, true, 2, 1, true>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, st) \
               : launch_decode_tma_g<GG, true, 2, 1>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, st);      \
  if (ns == 6)                                                                                                     \
    return rope ? launch_decode_tma_g<GG, true, 6, 2>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, st) \
                : launch_decode_tma_g<GG, false, 6, 2>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, st); \
  if (grid.y >= 2 && grid.y <= 8 && g_attn_cluster)                                                               \
    return rope ? launch_decode_tma_g<GG, true, 3, 1, true>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, st) \
                : launch_decode_tma_g<GG, false, 3, 1, true>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, st); \
  return rope ? launch_decode_tma_g<GG, true, 3, 1>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, st)   \
              : launch_decode_tma_g<GG, false, 3, 1>(grid, mk, mv, q, bt, sl, o, hkv, maxb, ws, cnt, k, v, theta, st)
  switch (G) {
    case 1: HX_TMA_G(1);
    case 2: HX_TMA_G(2);
    case 4: HX_TMA_G(4);
    case 8: HX_TMA_G(8);
    case 16: HX_TMA_G(16);
  }
#undef HX_TMA_G
  return HX_ERR_UNSUPPORTED;
}

template <int HD, int NW>
static size_t prefill_smem() {
  return sizeof(__nv_bfloat16) * (16 * NW * AttnSmem<HD>::LD + 4 * AttnSmem<HD>::TILE);
}
template <int HD>
static size_t decode_smem() {
  static_assert(sizeof(float) * 4 * 16 * (HD + 2) <= sizeof(__nv_bfloat16) * 2 * DEC_NS * AttnSmem<HD>::TILE,
                "red alias");
  return sizeof(__nv_bfloat16) * (16 * AttnSmem<HD>::LD + 2 * DEC_NS * AttnSmem<HD>::TILE);
}

template <int HD, int NW>
static int launch_prefill_mma_hd(const void *q, const void *kc, const void *vc, const int32_t *bt, const int32_t *sl,
                                 void *o, int batch, int s, int hq, int hkv, int page, int maxb, cudaStream_t st) {
  const size_t smem = prefill_smem<HD, NW>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_mma_kernel<HD, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const float sl2 = 1.4426950408889634f / sqrtf((float)HD);
  dim3 grid((s + 16 * NW - 1) / (16 * NW), hq, batch);
  return launch(attn_prefill_mma_kernel<HD, NW>, grid, dim3(32 * NW), smem, st, (const __nv_bfloat16 *)q,
                (const __nv_bfloat16 *)kc, (const __nv_bfloat16 *)vc, bt, sl, (__nv_bfloat16 *)o, s, hq, hkv, page,
                maxb, sl2);
}

static const int g_pf_warps = [] {  // prefill attention warps per CTA (HX_PF_WARPS=4 | 8)
  const char *e = getenv("HX_PF_WARPS");
  return e ? atoi(e) : 8;
}();

int launch_prefill_mma(const void *q, const void *kc, const void *vc, const int32_t *bt, const int32_t *sl, void *o,
                       int batch, int s, int hq, int hkv, int hd, int page, int maxb, cudaStream_t st) {
  if (hd == 128)
    return g_pf_warps == 4 ? launch_prefill_mma_hd<128, 4>(q, kc, vc, bt, sl, o, batch, s, hq, hkv, page, maxb, st)
                           : launch_prefill_mma_hd<128, 8>(q, kc, vc, bt, sl, o, batch, s, hq, hkv, page, maxb, st);
  if (hd == 64)
    return g_pf_warps == 4 ? launch_prefill_mma_hd<64, 4>(q, kc, vc, bt, sl, o, batch, s, hq, hkv, page, maxb, st)
                           : launch_prefill_mma_hd<64, 8>(q, kc, vc, bt, sl, o, batch, s, hq, hkv, page, maxb, st);
  return HX_ERR_UNSUPPORTED;
}

template <int HD, int G>
static int launch_decode_mma_g(dim3 grid, const void *q, const void *kc, const void *vc, const int32_t *bt,
                               const int32_t *sl, void *o, int hkv, int page, int maxb, float *ws, int *cnt,
                               cudaStream_t st) {
  const size_t smem = decode_smem<HD>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_mma_kernel<HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const float sl2 = 1.4426950408889634f / sqrtf((float)HD);
  return launch(attn_decode_mma_kernel<HD, G>, grid, dim3(AM_THREADS), smem, st, (const __nv_bfloat16 *)q,
                (const __nv_bfloat16 *)kc, (const __nv_bfloat16 *)vc, bt, sl, (__nv_bfloat16 *)o, hkv, page, maxb,
                sl2, ws, cnt);
}

int launch_decode_mma(int G, int hd, dim3 grid, const void *q, const void *kc, const void *vc, const int32_t *bt,
                      const int32_t *sl, void *o, int hkv, int page, int maxb, float *ws, int *cnt, cudaStream_t st) {
#define HX_DM(HDV, GV) \
  if (hd == HDV && G == GV) return launch_decode_mma_g<HDV, GV>(grid, q, kc, vc, bt, sl, o, hkv, page, maxb, ws, cnt, st)
  HX_DM(128, 1); HX_DM(128, 2); HX_DM(128, 4); HX_DM(128, 8); HX_DM(128, 16);
  HX_DM(64, 1); HX_DM(64, 2); HX_DM(64, 4); HX_DM(64, 8); HX_DM(64, 16);
#undef HX_DM
  return HX_ERR_UNSUPPORTED;
}

}  // namespace hx
