// Causal prefill attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// The attention of PAPER.md:121-131 for a whole prompt (no earlier context):
// o = softmax(q k^T / sqrt(hd) + causal) v per head. One CTA owns 128 query
// rows of one (sequence, head) and walks the 128-key blocks up to the diagonal:
//   warp 0   TMA producer: Q once; per block K (two 64-key pages of the paged
//            cache) and V^T (from the prefill's transposed-V scratch) into a
//            2-stage ring, 128B-swizzled, one mbarrier per stage;
//   warp 1   MMA issuer (one thread): S_j = Q K_j^T into one of two TMEM
//            accumulators (M=128, N=128, K=16 x 8), then PV_j = P_j V_j into
//            one of two more -- S_{j+1} is issued before PV_j so QK^T of the
//            next block overlaps the softmax of this one;
//   warps 2-5 softmax, one query row per thread (TMEM lane = row): row max
//            and exp2 straight from TMEM, P_j (bf16) written to smem in the
//            UMMA K-major layout, and O kept in registers: O = (O + PV_{j-1})
//            * exp2(m_{j-1} - m_j) before P_j is released (online softmax).
// TMEM holds 4 x 128 fp32 columns (S0, S1, PV0, PV1) = the whole 512.
// Unsupported shapes (hd != 128, s % 128, page != 64, earlier context) are
// refused; the engine then uses the mma.sync kernel (hx_attention_mma.cu).
#include <cstdlib>

#include "hx_common.cuh"

namespace hx {

constexpr int TC_ROWS = 128;
constexpr uint32_t TC_HALF = 128 * 128;  // [128 rows x 64 bf16] SW128 half tile (16 KB)
constexpr uint32_t TC_TILE = 2 * TC_HALF;

int make_tma_bf16_sw128(CUtensorMap *map, const void *ptr, long rows, int cols, long pitch, int box_rows);

// 32 lanes x 32 bit x 16 columns, without the wait (batch several, then tmem_wait_ld)
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// byte offset of element (r, c) of a [128 x 128] bf16 tile stored as two
// 128B-swizzled K-major halves (columns 0-63, 64-127)
__device__ __forceinline__ uint32_t tc_off(int r, int c) {
  return (c >> 6) * TC_HALF + r * 128 + (((((c & 63) >> 3)) ^ (r & 7)) << 4) + ((c & 7) << 1);
}

__global__ void __launch_bounds__(192, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                           const __grid_constant__ CUtensorMap tmv, const int32_t *bt, __nv_bfloat16 *o, int s_len,
                           int hq, int hkv, int max_blocks, float sl2) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t *qs = sm;                      // Q [128 x 128]
  uint8_t *kv = sm + TC_TILE;            // stage st: K at kv + 2*st*TILE, V^T at + TILE
  uint8_t *ps = sm + 5 * TC_TILE;        // P [128 x 128]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 6 * TC_TILE);
  uint64_t *q_full = bar, *kv_full = bar + 1, *kv_empty = bar + 3, *s_full = bar + 5, *s_empty = bar + 7,
           *p_full = bar + 9, *pv_full = bar + 10, *pv_empty = bar + 12;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 14);

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = gridDim.x - 1 - blockIdx.x;  // heaviest query tiles first
  const int h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (hq / hkv);
  const int q0 = qt * TC_ROWS;
  const int nblk = qt + 1;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmq);
    tma_prefetch(&tmk);
    tma_prefetch(&tmv);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
      mbar_init(&pv_full[i], 1);
      mbar_init(&pv_empty[i], 128);
    }
    mbar_init(p_full, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_last();
      pdl_wait();  // q, the K pages and V^T come from the preceding kernels
      mbar_arrive_expect_tx(q_full, TC_TILE);
      for (int hh = 0; hh < 2; ++hh)
        tma_load_2d(qs + hh * TC_HALF, &tmq, q_full, h * 128 + hh * 64, b * s_len + q0, pol);
      const int32_t *btb = bt + (size_t)b * max_blocks;
      for (int j = 0; j < nblk; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        uint8_t *ks = kv + 2 * st * TC_TILE, *vs = ks + TC_TILE;
        mbar_arrive_expect_tx(&kv_full[st], 2 * TC_TILE);
        for (int pg = 0; pg < 2; ++pg) {
          const int row = (btb[2 * j + pg] * hkv + kvh) * 64;
          for (int hh = 0; hh < 2; ++hh)
            tma_load_2d(ks + hh * TC_HALF + pg * 64 * 128, &tmk, &kv_full[st], hh * 64, row, pol);
        }
        for (int hh = 0; hh < 2; ++hh)
          tma_load_2d(vs + hh * TC_HALF, &tmv, &kv_full[st], j * 128 + hh * 64, (b * hkv + kvh) * 128, pol);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, 128);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        if (j >= 2) mbar_wait(&s_empty[st], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint8_t *ks = kv + 2 * st * TC_TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tmem + st * 128, umma_desc_sw128(qs + (kk >> 2) * TC_HALF) + 2 * (kk & 3),
                    umma_desc_sw128(ks + (kk >> 2) * TC_HALF) + 2 * (kk & 3), idesc, kk > 0 ? 1u : 0u);
        umma_commit(&s_full[st]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) issue_s(j + 1);
        const int st = j & 1;
        mbar_wait(p_full, j & 1);
        if (j >= 2) mbar_wait(&pv_empty[st], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint8_t *vs = kv + (2 * st + 1) * TC_TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tmem + 256 + st * 128, umma_desc_sw128(ps + (kk >> 2) * TC_HALF) + 2 * (kk & 3),
                    umma_desc_sw128(vs + (kk >> 2) * TC_HALF) + 2 * (kk & 3), idesc, kk > 0 ? 1u : 0u);
        umma_commit(&pv_full[st]);
        umma_commit(&kv_empty[st]);
      }
    }
  } else {
    // softmax warps: TMEM lane quarter = warp % 4, one query row per thread
    const int qq = warp & 3;
    const int r = qq * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qq * 32) << 16);
    float O[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) O[c] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nblk; ++j) {
      const int st = j & 1;
      const bool diag = j == qt;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float mx = -INFINITY;
#pragma unroll
      for (int c1 = 0; c1 < 128; c1 += 64) {
        float v[64];
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) tmem_ld16_nw(trow + st * 128 + c1 + c0, v + c0);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 64; ++k)
          if (!diag || c1 + k <= r) mx = fmaxf(mx, v[k]);
      }
      const float m_new = fmaxf(m, mx * sl2);
      const float corr = exp2f(m - m_new);  // m = -inf on the first block: corr = 0, O and l are 0
      if (j > 0) {  // fold PV_{j-1} (relative to m) into O, rescale to m_new
        const int pb = (j - 1) & 1;
        mbar_wait(&pv_full[pb], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c1 = 0; c1 < 128; c1 += 32) {
          float v[32];
          tmem_ld16_nw(trow + 256 + pb * 128 + c1, v);
          tmem_ld16_nw(trow + 256 + pb * 128 + c1 + 16, v + 16);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) O[c1 + k] = (O[c1 + k] + v[k]) * corr;
        }
        tc_fence_before();
        mbar_arrive(&pv_empty[pb]);
      }
      l *= corr;
      // P_j = exp2(S * sl2 - m_new) -> bf16 -> smem (UMMA K-major, 128B swizzle)
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 16) {
        float v[16];
        tmem_ld16(trow + st * 128 + c0, v);  // (pass 2 keeps one load in flight: O holds 128 registers)
        uint32_t pk[8];
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const float p0 = (!diag || c0 + k <= r) ? exp2f(v[k] * sl2 - m_new) : 0.f;
          const float p1 = (!diag || c0 + k + 1 <= r) ? exp2f(v[k + 1] * sl2 - m_new) : 0.f;
          l += p0 + p1;
          pk[k >> 1] = pack_bf16(p0, p1);
        }
        *reinterpret_cast<uint4 *>(ps + tc_off(r, c0)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4 *>(ps + tc_off(r, c0 + 8)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      tc_fence_before();
      mbar_arrive(&s_empty[st]);
      fence_proxy_async_smem();  // P (generic-proxy stores) -> the tensor core's async proxy
      mbar_arrive(p_full);
      m = m_new;
    }
    const int pb = (nblk - 1) & 1;
    mbar_wait(&pv_full[pb], ((nblk - 1) >> 1) & 1);
    tc_fence_after();
#pragma unroll
    for (int c0 = 0; c0 < 128; c0 += 16) {
      float v[16];
      tmem_ld16(trow + 256 + pb * 128 + c0, v);
#pragma unroll
      for (int k = 0; k < 16; ++k) O[c0 + k] += v[k];
    }
    const float inv = 1.0f / l;
    __nv_bfloat16 *dst = o + ((size_t)(b * s_len + q0 + r) * hq + h) * 128;
#pragma unroll
    for (int c0 = 0; c0 < 128; c0 += 8) {
      uint4 u;
      u.x = pack_bf16(O[c0] * inv, O[c0 + 1] * inv);
      u.y = pack_bf16(O[c0 + 2] * inv, O[c0 + 3] * inv);
      u.z = pack_bf16(O[c0 + 4] * inv, O[c0 + 5] * inv);
      u.w = pack_bf16(O[c0 + 6] * inv, O[c0 + 7] * inv);
      *reinterpret_cast<uint4 *>(dst + c0) = u;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------------ persistent variant
// The one-tile kernel above is latency-bound: 1024 short CTAs (1-4 key blocks
// at 7B s=512) in ~7 waves, each paying the barrier/TMEM set-up, the first TMA
// round trip and its drain alone (ncu: 9 % tensor pipe, the top stalls are the
// mbarrier waits and CTAs waiting to exit). Here one CTA per SM walks the
// (query tile, head, sequence) items heaviest first (item c, c + G, ...): the
// producer loads the next item's Q (once the previous item's last S MMA has
// read the Q buffer: q_empty) and K/V blocks while the current item is still
// in its softmax / PV / epilogue, and every mbarrier phase is tracked by a
// global block counter across items. Roles, TMEM map and numerics per item
// are those of attn_prefill_tc_kernel.
__global__ void __launch_bounds__(192, 1)
    attn_prefill_tcp_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                            const __grid_constant__ CUtensorMap tmv, const int32_t *bt, __nv_bfloat16 *o, int s_len,
                            int hq, int hkv, int max_blocks, float sl2, int batch) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t *qs = sm;
  uint8_t *kv = sm + TC_TILE;
  uint8_t *ps = sm + 5 * TC_TILE;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 6 * TC_TILE);
  uint64_t *q_full = bar, *kv_full = bar + 1, *kv_empty = bar + 3, *s_full = bar + 5, *s_empty = bar + 7,
           *p_full = bar + 9, *pv_full = bar + 10, *pv_empty = bar + 12, *q_empty = bar + 14;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 15);

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = s_len / TC_ROWS;
  const int per_tile = hq * batch;
  const int n_items = nq * per_tile;
  const int G = gridDim.x;
  // item -> (query tile, head, sequence), heaviest query tiles first
  auto decode_item = [&](int item, int &qt, int &h, int &b) {
    qt = nq - 1 - item / per_tile;
    const int rem = item % per_tile;
    h = rem % hq;
    b = rem / hq;
  };

  if (threadIdx.x == 0) {
    tma_prefetch(&tmq);
    tma_prefetch(&tmk);
    tma_prefetch(&tmv);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
      mbar_init(&pv_full[i], 1);
      mbar_init(&pv_empty[i], 128);
    }
    mbar_init(p_full, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_last();
      pdl_wait();  // q, the K pages and V^T come from the preceding kernels
      int g = 0, it = 0;
      for (int item = blockIdx.x; item < n_items; item += G, ++it) {
        int qt, h, b;
        decode_item(item, qt, h, b);
        const int kvh = h / (hq / hkv);
        if (it > 0) mbar_wait(q_empty, (it - 1) & 1);  // the previous item's S MMAs have read Q
        mbar_arrive_expect_tx(q_full, TC_TILE);
        for (int hh = 0; hh < 2; ++hh)
          tma_load_2d(qs + hh * TC_HALF, &tmq, q_full, h * 128 + hh * 64, b * s_len + qt * TC_ROWS, pol);
        const int32_t *btb = bt + (size_t)b * max_blocks;
        for (int j = 0; j <= qt; ++j, ++g) {
          const int st = g & 1;
          if (g >= 2) mbar_wait(&kv_empty[st], ((g >> 1) & 1) ^ 1);
          uint8_t *ks = kv + 2 * st * TC_TILE, *vs = ks + TC_TILE;
          mbar_arrive_expect_tx(&kv_full[st], 2 * TC_TILE);
          for (int pg = 0; pg < 2; ++pg) {
            const int row = (btb[2 * j + pg] * hkv + kvh) * 64;
            for (int hh = 0; hh < 2; ++hh)
              tma_load_2d(ks + hh * TC_HALF + pg * 64 * 128, &tmk, &kv_full[st], hh * 64, row, pol);
          }
          for (int hh = 0; hh < 2; ++hh)
            tma_load_2d(vs + hh * TC_HALF, &tmv, &kv_full[st], j * 128 + hh * 64, (b * hkv + kvh) * 128, pol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, 128);
      auto issue_s = [&](int gs) {
        const int st = gs & 1;
        mbar_wait(&kv_full[st], (gs >> 1) & 1);
        if (gs >= 2) mbar_wait(&s_empty[st], ((gs >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint8_t *ks = kv + 2 * st * TC_TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tmem + st * 128, umma_desc_sw128(qs + (kk >> 2) * TC_HALF) + 2 * (kk & 3),
                    umma_desc_sw128(ks + (kk >> 2) * TC_HALF) + 2 * (kk & 3), idesc, kk > 0 ? 1u : 0u);
        umma_commit(&s_full[st]);
      };
      int g = 0, it = 0;
      for (int item = blockIdx.x; item < n_items; item += G, ++it) {
        int qt, h, b;
        decode_item(item, qt, h, b);
        const int nblk = qt + 1;
        mbar_wait(q_full, it & 1);
        issue_s(g);
        if (nblk == 1) umma_commit(q_empty);
        for (int j = 0; j < nblk; ++j) {
          const int gb = g + j;
          if (j + 1 < nblk) {
            issue_s(gb + 1);
            if (j + 2 == nblk) umma_commit(q_empty);  // the item's last S MMA has been issued
          }
          const int st = gb & 1;
          mbar_wait(p_full, gb & 1);
          if (gb >= 2) mbar_wait(&pv_empty[st], ((gb >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint8_t *vs = kv + (2 * st + 1) * TC_TILE;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + 256 + st * 128, umma_desc_sw128(ps + (kk >> 2) * TC_HALF) + 2 * (kk & 3),
                      umma_desc_sw128(vs + (kk >> 2) * TC_HALF) + 2 * (kk & 3), idesc, kk > 0 ? 1u : 0u);
          umma_commit(&pv_full[st]);
          umma_commit(&kv_empty[st]);
        }
        g += nblk;
      }
    }
  } else {
    const int qq = warp & 3;
    const int r = qq * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qq * 32) << 16);
    int g = 0;
    for (int item = blockIdx.x; item < n_items; item += G) {
      int qt, h, b;
      decode_item(item, qt, h, b);
      const int nblk = qt + 1;
      float O[128];
#pragma unroll
      for (int c = 0; c < 128; ++c) O[c] = 0.f;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nblk; ++j) {
        const int gb = g + j;
        const int st = gb & 1;
        const bool diag = j == qt;
        mbar_wait(&s_full[st], (gb >> 1) & 1);
        tc_fence_after();
        float mx = -INFINITY;
#pragma unroll
        for (int c1 = 0; c1 < 128; c1 += 64) {
          float v[64];
#pragma unroll
          for (int c0 = 0; c0 < 64; c0 += 16) tmem_ld16_nw(trow + st * 128 + c1 + c0, v + c0);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 64; ++k)
            if (!diag || c1 + k <= r) mx = fmaxf(mx, v[k]);
        }
        const float m_new = fmaxf(m, mx * sl2);
        const float corr = exp2f(m - m_new);
        if (j > 0) {  // fold PV_{gb-1} into O, rescale to m_new (also frees the P buffer)
          const int pg = gb - 1;
          const int pb = pg & 1;
          mbar_wait(&pv_full[pb], (pg >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c1 = 0; c1 < 128; c1 += 32) {
            float v[32];
            tmem_ld16_nw(trow + 256 + pb * 128 + c1, v);
            tmem_ld16_nw(trow + 256 + pb * 128 + c1 + 16, v + 16);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 32; ++k) O[c1 + k] = (O[c1 + k] + v[k]) * corr;
          }
          tc_fence_before();
          mbar_arrive(&pv_empty[pb]);
        }
        l *= corr;
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 16) {
          float v[16];
          tmem_ld16(trow + st * 128 + c0, v);
          uint32_t pk[8];
#pragma unroll
          for (int k = 0; k < 16; k += 2) {
            const float p0 = (!diag || c0 + k <= r) ? exp2f(v[k] * sl2 - m_new) : 0.f;
            const float p1 = (!diag || c0 + k + 1 <= r) ? exp2f(v[k + 1] * sl2 - m_new) : 0.f;
            l += p0 + p1;
            pk[k >> 1] = pack_bf16(p0, p1);
          }
          *reinterpret_cast<uint4 *>(ps + tc_off(r, c0)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4 *>(ps + tc_off(r, c0 + 8)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
        tc_fence_before();
        mbar_arrive(&s_empty[st]);
        fence_proxy_async_smem();
        mbar_arrive(p_full);
        m = m_new;
      }
      const int lg = g + nblk - 1;
      const int pb = lg & 1;
      mbar_wait(&pv_full[pb], (lg >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 16) {
        float v[16];
        tmem_ld16(trow + 256 + pb * 128 + c0, v);
#pragma unroll
        for (int k = 0; k < 16; ++k) O[c0 + k] += v[k];
      }
      tc_fence_before();
      mbar_arrive(&pv_empty[pb]);  // the last PV buffer is read: the next item may reuse it
      const float inv = 1.0f / l;
      __nv_bfloat16 *dst = o + ((size_t)(b * s_len + qt * TC_ROWS + r) * hq + h) * 128;
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 8) {
        uint4 u;
        u.x = pack_bf16(O[c0] * inv, O[c0 + 1] * inv);
        u.y = pack_bf16(O[c0 + 2] * inv, O[c0 + 3] * inv);
        u.z = pack_bf16(O[c0 + 4] * inv, O[c0 + 5] * inv);
        u.w = pack_bf16(O[c0 + 6] * inv, O[c0 + 7] * inv);
        *reinterpret_cast<uint4 *>(dst + c0) = u;
      }
      g += nblk;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// vt[((b * hkv + h) * 128 + d) * s + i] = v of token (b, i), kv head h, dim d,
// read from the packed qkv rows; 64 x 64 tiles through smem with 4-byte
// (bf16 pair) accesses on both sides
__global__ void __launch_bounds__(256)
    prefill_vt_kernel(const __nv_bfloat16 *qkv, __nv_bfloat16 *vt, int s_len, int hq, int hkv) {
  pdl_trigger();
  pdl_wait();
  __shared__ __nv_bfloat16 tile[64][66];  // [token][dim]
  const int i0 = blockIdx.x * 64, d0 = blockIdx.y * 64;
  const int bh = blockIdx.z, b = bh / hkv, h = bh % hkv;
  const size_t row_w = (size_t)(hq + 2 * hkv) * 128;
  const __nv_bfloat16 *src = qkv + (size_t)(b * s_len + i0) * row_w + (hq + hkv + h) * 128 + d0;
  for (int e = threadIdx.x; e < 64 * 32; e += 256) {
    const int t = e >> 5, dp = (e & 31) * 2;
    const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162 *>(src + t * row_w + dp);
    tile[t][dp] = v.x;
    tile[t][dp + 1] = v.y;
  }
  __syncthreads();
  __nv_bfloat16 *dst = vt + ((size_t)bh * 128 + d0) * s_len + i0;
  for (int e = threadIdx.x; e < 64 * 32; e += 256) {
    const int d = e >> 5, tp = (e & 31) * 2;
    __nv_bfloat162 v;
    v.x = tile[tp][d];
    v.y = tile[tp + 1][d];
    *reinterpret_cast<__nv_bfloat162 *>(dst + (size_t)d * s_len + tp) = v;
  }
}

}  // namespace hx

using namespace hx;

extern "C" int hx_prefill_vt(const void *qkv, void *vt, int batch, int s_len, int hq, int hkv, int hd,
                             hx_stream_t stream) {
  if (batch == 0) return 0;
  if (!qkv || !vt || hd != 128 || s_len % 64 || hq % hkv) return HX_ERR_UNSUPPORTED;
  return launch(prefill_vt_kernel, dim3(s_len / 64, 2, batch * hkv), dim3(256), 0, as_stream(stream),
                (const __nv_bfloat16 *)qkv, (__nv_bfloat16 *)vt, s_len, hq, hkv);
}

extern "C" int hx_attn_prefill_tc(const void *q, const void *k_cache, const void *vt, const int32_t *block_table,
                                  void *o, int batch, int s_len, int hq, int hkv, int hd, int page_size,
                                  int max_blocks, hx_stream_t stream) {
  if (batch == 0) return 0;
  if (!q || !k_cache || !vt || !block_table || !o || hq % hkv) return HX_ERR_ARG;
  if (hd != 128 || page_size != 64 || s_len % 128 || s_len / 64 > max_blocks) return HX_ERR_UNSUPPORTED;
  CUtensorMap mq, mk, mv;
  int rc = make_tma_bf16_sw128(&mq, q, (long)batch * s_len, hq * 128, (long)hq * 128, 128);
  if (!rc) rc = make_tma_bf16_sw128(&mk, k_cache, 1l << 28, 128, 128, 64);
  if (!rc) rc = make_tma_bf16_sw128(&mv, vt, (long)batch * hkv * 128, s_len, s_len, 128);
  if (rc) return rc;
  const size_t smem = 1024 + 6 * TC_TILE + 16 * 8 + 16;
  const float sl2 = 1.4426950408889634f / sqrtf(128.f);
  static const bool persistent = [] {  // HX_PREFILL_TC_P=0: one CTA per (query tile, head, sequence)
    const char *e = getenv("HX_PREFILL_TC_P");
    return e ? atoi(e) != 0 : true;
  }();
  if (persistent) {
    static bool attrp = false;
    if (!attrp) {
      cudaFuncSetAttribute(attn_prefill_tcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attrp = true;
    }
    const int items = (s_len / 128) * hq * batch;
    return launch(attn_prefill_tcp_kernel, dim3(items < 148 ? items : 148), dim3(192), smem, as_stream(stream), mq, mk,
                  mv, block_table, (__nv_bfloat16 *)o, s_len, hq, hkv, max_blocks, sl2, batch);
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  return launch(attn_prefill_tc_kernel, dim3(s_len / 128, hq, batch), dim3(192), smem, as_stream(stream), mq, mk, mv,
                block_table, (__nv_bfloat16 *)o, s_len, hq, hkv, max_blocks, sl2);
}
