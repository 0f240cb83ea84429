// hx_linear: the TP column/row-parallel projections (QKV, O, gate/up, down,
// lm_head). Replaces the weight-scan and FLOP terms of the reference cost
// model (pkg/src/heteroplan/costs.py:114-119).
//
// bf16: one tcgen05 kernel computes D[M, N] = A[M, K] . B[N, K]^T with both
// operands K-major, staged by TMA (128B swizzle) through a STAGES-deep
// mbarrier ring, accumulated in TMEM by one elected thread, and drained by 4
// epilogue warps (tcgen05.ld 32x32b). The host picks the orientation:
//   decode  (n_tok <= 64): A = weights (M = out features, 128-row tiles),
//            B = activations (N = 16/32/64 tokens): a weight-streaming,
//            HBM-bound kernel, stream-K: one persistent CTA per SM streams
//            an equal share of the (tile, k-block) units; the last CTA of a
//            tile (atomic ticket) reduces the fp32 partials in CTA order
//            (deterministic), or the consumer kernel does (DEFER_REDUCE).
//   prefill (n_tok > 64):  A = activations (M = 128 tokens), B = weights
//            (N = 256 features): tensor-bound, one 128x256 fp32 tile in TMEM.
// Weights may be pre-packed (hx_pack_weight) into [N/128][K/64][128][64]
// tiles so every 16 KB TMA box is one contiguous HBM stream. Under PDL the
// producer issues the first STAGES weight tiles before griddepcontrol.wait:
// weights never depend on the previous kernel, so their HBM latency overlaps
// the previous kernel's tail.
// fp32 mode (parity with the CPU oracle) uses a CUDA-core kernel.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "hx_common.cuh"

namespace hx {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int kNumSMs = 148;
constexpr uint32_t TILE_BYTES = BM * BK * 2;  // one packed 128x64 weight tile

struct GemmArgs {
  void *c;
  long ldm, ldn;  // C[m * ldm + n * ldn]
  int M, N, K;
  int c_bf16;
  int accumulate;
  int kb_total;
  int kb_per_split;
  int a_is_weight;
  int w_packed;
  float *ws;
  int *counters;
};

// plain output descriptor, passed by value (registers): C[m * ldm + n * ldn]
struct OutDesc {
  void *c;
  long ldm, ldn;
  int M, N, c_bf16, accumulate;
};
__device__ __forceinline__ OutDesc out_of(const GemmArgs &p) {
  return OutDesc{p.c, p.ldm, p.ldn, p.M, p.N, p.c_bf16, p.accumulate};
}

__device__ __forceinline__ void store_chunk(const OutDesc p, int m, int n0, const float *v) {
  if (m >= p.M) return;
  if (p.c_bf16) {
    __nv_bfloat16 *c = reinterpret_cast<__nv_bfloat16 *>(p.c);
    if (p.ldn == 1 && n0 + 16 <= p.N && ((p.ldm * m + n0) & 7) == 0) {
      Vec16<__nv_bfloat16>::store(c + m * p.ldm + n0, v);
      Vec16<__nv_bfloat16>::store(c + m * p.ldm + n0 + 8, v + 8);
      return;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (n0 + j < p.N) c[m * p.ldm + (long)(n0 + j) * p.ldn] = __float2bfloat16_rn(v[j]);
  } else {
    float *c = reinterpret_cast<float *>(p.c);
    if (p.ldn == 1 && !p.accumulate && n0 + 16 <= p.N && ((p.ldm * m + n0) & 3) == 0) {
#pragma unroll
      for (int j = 0; j < 16; j += 4) Vec16<float>::store(c + m * p.ldm + n0 + j, v + j);
      return;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (n0 + j < p.N) {
        float *dst = c + m * p.ldm + (long)(n0 + j) * p.ldn;
        *dst = p.accumulate ? *dst + v[j] : v[j];
      }
    }
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tm_a,
                        const __grid_constant__ CUtensorMap tm_b, const __grid_constant__ GemmArgs p) {
  constexpr uint32_t A_BYTES = BM * BK * 2;
  constexpr uint32_t B_BYTES = BN * BK * 2;
  constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sa = smem;
  uint8_t *sb = smem + STAGES * A_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(sb + STAGES * B_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *accf = empty + STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accf + 1);
  __shared__ int s_last;

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterisation: CTAs launched together cover a GM x (~148 / GM)
  // block of tiles, so the activation rows and weight columns they share are
  // read from HBM once and re-used from L2 (m-major order re-reads all of X for
  // every weight tile once M outgrows one wave)
  constexpr int GM = 16;
  const int Mt = gridDim.x, Nt = gridDim.y;
  const int pid = blockIdx.y * Mt + blockIdx.x;
  const int first_m = (pid / (GM * Nt)) * GM;
  const int gm = min(Mt - first_m, GM);
  const int tm = first_m + (pid % (GM * Nt)) % gm;
  const int tn = (pid % (GM * Nt)) / gm;
  const int m0 = tm * BM, n0 = tn * BN;
  const int split = blockIdx.z, splits = gridDim.z;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_a);
    tma_prefetch(&tm_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // TMA producer
    const uint64_t pol_w = l2_policy_evict_first(), pol_x = l2_policy_evict_last();
    // weight operand: A (decode) or B (prefill); packed tiles are row blocks of a [*, 64] tensor
    auto load_w = [&](uint8_t *dst, int kb) {
      if (p.a_is_weight) {
        if (p.w_packed) tma_load_2d(dst, &tm_a, &full[(dst - sa) / A_BYTES], 0, (tm * p.kb_total + kb) * BM, pol_w);
        else tma_load_2d(dst, &tm_a, &full[(dst - sa) / A_BYTES], kb * BK, m0, pol_w);
      } else {
        uint64_t *bar = &full[(dst - sb) / B_BYTES];
        if (p.w_packed) {
#pragma unroll
          for (int h = 0; h < BN / BM; ++h)
            tma_load_2d(dst + h * TILE_BYTES, &tm_b, bar, 0, ((tn * (BN / BM) + h) * p.kb_total + kb) * BM, pol_w);
        } else {
          tma_load_2d(dst, &tm_b, bar, kb * BK, n0, pol_w);
        }
      }
    };
    auto load_x = [&](int s, int kb) {
      if (p.a_is_weight) tma_load_2d(sb + s * B_BYTES, &tm_b, &full[s], kb * BK, n0, pol_x);
      else tma_load_2d(sa + s * A_BYTES, &tm_a, &full[s], kb * BK, m0, pol_x);
    };
    auto wbuf = [&](int s) { return p.a_is_weight ? sa + s * A_BYTES : sb + s * B_BYTES; };
    // prologue: weight tiles of the first stages go out before the dependency wait
    const int pre = min(nkb, STAGES);
    for (int i = 0; i < pre; ++i) {
      mbar_arrive_expect_tx(&full[i], A_BYTES + B_BYTES);
      load_w(wbuf(i), kb0 + i);
    }
    pdl_wait();
    for (int i = 0; i < pre; ++i) load_x(i, kb0 + i);
    for (int i = pre; i < nkb; ++i) {
      const int s = i % STAGES;
      mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
      load_w(wbuf(s), kb0 + i);
      load_x(s, kb0 + i);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer: 4 x (128 x BN x 16) per 64-wide K block
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      tc_fence_after();
      const uint64_t ad = umma_desc_sw128(sa + s * A_BYTES);
      const uint64_t bd = umma_desc_sw128(sb + s * B_BYTES);
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk)
        umma_bf16(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : 0u);
      umma_commit(&empty[s]);
    }
    umma_commit(accf);
  }
  __syncwarp();

  // ---- epilogue: warp w owns TMEM lanes [32w, 32w + 32) = tile rows
  mbar_wait(accf, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  const int m = m0 + row;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  if (splits == 1) {
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      tmem_ld16(trow + c, v);
      store_chunk(out_of(p), m, n0 + c, v);
    }
  } else {
    const int tile = tn * Mt + tm;
    float *mine = p.ws + ((size_t)(tile * splits + split) * BM + row) * BN;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      tmem_ld16(trow + c, v);
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        __stcg(reinterpret_cast<float4 *>(mine + c + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int t = ticket_acq_rel(&p.counters[tile]);
      s_last = (t == splits - 1);
      if (s_last) p.counters[tile] = 0;  // re-arm for the next launch / graph replay
    }
    __syncthreads();
    if (s_last) {
      const float *base = p.ws + ((size_t)tile * splits * BM + row) * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.f;
        for (int s = 0; s < splits; ++s) {
          const float *src = base + (size_t)s * BM * BN + c;
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            float4 f = __ldcg(reinterpret_cast<const float4 *>(src + j));
            acc[j] += f.x; acc[j + 1] += f.y; acc[j + 2] += f.z; acc[j + 3] += f.w;
          }
        }
        store_chunk(out_of(p), m, n0 + c, acc);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ------------------------------------------------------------------ persistent prefill GEMM
// Prefill (token-major) Y = X W^T on whole 128 x BN tiles, persistent: one CTA
// per SM walks the tiles blockIdx.x, blockIdx.x + G, ... in the grouped
// raster order of gemm_bf16_tc_kernel. Warp 0 streams the A (activation) and B
// (packed weight) K-blocks of all its tiles through one mbarrier ring without
// a per-tile refill; warp 1 issues the MMAs of tile k into TMEM buffer k & 1
// while warps 2-5 drain tile k - 1 from the other buffer (2 x BN = 512 TMEM
// columns), so the epilogue and the next tile's pipeline fill hide behind the
// tensor core instead of running between CTAs.
template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    gemm_tc_persistent_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                              const __grid_constant__ GemmArgs p) {
  constexpr uint32_t A_BYTES = BM * BK * 2;
  constexpr uint32_t B_BYTES = BN * BK * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sa = smem;
  uint8_t *sb = smem + STAGES * A_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(sb + STAGES * B_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;   // [2]
  uint64_t *tempty = tfull + 2;       // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int GM = 16;
  const int Mt = (p.M + BM - 1) / BM, Nt = (p.N + BN - 1) / BN;
  const int tiles = Mt * Nt, G = gridDim.x;
  const int nkb = p.kb_total;
  auto tile_mn = [&](int pid, int &tm, int &tn) {  // grouped rasterisation (L2 reuse of X rows / W columns)
    const int first_m = (pid / (GM * Nt)) * GM;
    const int gm = min(Mt - first_m, GM);
    tm = first_m + (pid % (GM * Nt)) % gm;
    tn = (pid % (GM * Nt)) / gm;
  };

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_a);
    tma_prefetch(&tm_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = l2_policy_evict_first(), pol_x = l2_policy_evict_last();
      auto load_w = [&](int s, int tn, int kb) {
        if (p.w_packed) {
#pragma unroll
          for (int h = 0; h < BN / BM; ++h)
            tma_load_2d(sb + s * B_BYTES + h * TILE_BYTES, &tm_b, &full[s], 0,
                        ((tn * (BN / BM) + h) * p.kb_total + kb) * BM, pol_w);
        } else {
          tma_load_2d(sb + s * B_BYTES, &tm_b, &full[s], kb * BK, tn * BN, pol_w);
        }
      };
      auto load_x = [&](int s, int tm, int kb) { tma_load_2d(sa + s * A_BYTES, &tm_a, &full[s], kb * BK, tm * BM, pol_x); };
      int i = 0;
      bool first = true;
      for (int pid = blockIdx.x; pid < tiles; pid += G) {
        int tm, tn;
        tile_mn(pid, tm, tn);
        int kb = 0;
        if (first) {  // the first tile's weight blocks go out before the dependency wait
          const int pre = min(nkb, STAGES);
          for (int j = 0; j < pre; ++j) {
            mbar_arrive_expect_tx(&full[j], A_BYTES + B_BYTES);
            load_w(j, tn, j);
          }
          pdl_wait();
          for (int j = 0; j < pre; ++j) load_x(j, tm, j);
          i = kb = pre;
          first = false;
        }
        for (; kb < nkb; ++kb, ++i) {
          const int s = i % STAGES;
          mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
          load_w(s, tn, kb);
          load_x(s, tm, kb);
        }
      }
      if (first) pdl_wait();  // no tile (never: grid <= tiles), keep the PDL contract
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int i = 0, lt = 0;
      for (int pid = blockIdx.x; pid < tiles; pid += G, ++lt) {
        const int buf = lt & 1;
        mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * BN;
        for (int kb = 0; kb < nkb; ++kb, ++i) {
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(sa + s * A_BYTES);
          const uint64_t bd = umma_desc_sw128(sb + s * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16(acc, ad + 2 * kk, bd + 2 * kk, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[buf]);
      }
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quarters (warp % 4): tile rows
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const OutDesc od = out_of(p);
    int lt = 0;
    for (int pid = blockIdx.x; pid < tiles; pid += G, ++lt) {
      int tm, tn;
      tile_mn(pid, tm, tn);
      const int buf = lt & 1;
      mbar_wait(&tfull[buf], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + buf * BN;
      const int m = tm * BM + row;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(trow + c, v);
        store_chunk(od, m, tn * BN + c, v);
      }
      tc_fence_before();
      mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 2 * BN);
}

// ------------------------------------------------------------------ stream-K decode
// Persistent weight-streaming GEMM for decode (A = weights, 128-row tiles;
// B = the n_tok <= 64 activation rows). The tiles x K-blocks unit space is
// cut into one contiguous, equal range per CTA (2 CTAs/SM), so every CTA
// streams the same number of 16 KB weight tiles with one uninterrupted TMA
// pipeline across tile boundaries -- no wave quantisation, no per-tile
// pipeline refill. Warp roles: 0 = TMA producer, 1 = MMA issuer (TMEM
// accumulator double-buffered across segments), 2..5 = epilogue. A segment
// covering a whole tile stores straight to C; partial segments (at most the
// first and last of each CTA) go to a workspace slot, and the tile's last
// contributor (atomic ticket) sums the slots in CTA order (deterministic).
struct SKArgs {
  void *c;
  long ldm, ldn;
  int M, N;
  int c_bf16, accumulate, w_packed;
  int defer;  // HX_LINEAR_DEFER_REDUCE: leave split tiles as partial slots (no ticket)
  int KB, units;
  float *ws;
  int *counters;
  unsigned long long *trace;  // optional per-CTA timeline (hx_debug_trace): start, wait done, end, smid
  int l2pf;                   // weight tiles beyond the smem ring prefetched into L2 before the PDL wait
  int prewait;                // ring stages whose weight tiles are requested before the PDL wait
  const uint8_t *w_ptr;       // packed weights (for the epilogue warps' L2 prefetch)
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}

// c * units < 2^31 for every decode shape (units <= 4096 tiles x 172 K-blocks, G <= 296)

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 2)
    gemm_streamk_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                        const __grid_constant__ SKArgs p) {
  constexpr uint32_t A_BYTES = BM * BK * 2;
  constexpr uint32_t B_BYTES = BN * BK * 2;
  constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : 128);
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sa = smem;
  uint8_t *sb = smem + STAGES * A_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(sb + STAGES * B_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;   // [2]
  uint64_t *tempty = tfull + 2;       // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  __shared__ int s_last;

  pdl_trigger();
  const unsigned long long t_start = p.trace ? globaltimer() : 0ull;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;
  const int u0 = sk_start(c, p.units, G), u1 = sk_start(c + 1, p.units, G);

  if (threadIdx.x == 0) {
    tma_prefetch(&tm_w);
    tma_prefetch(&tm_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = l2_policy_evict_first(), pol_x = l2_policy_evict_last();
      auto load_w = [&](int s, int u) {
        const int t = u / p.KB, kb = u % p.KB;
        if (p.w_packed) tma_load_2d(sa + s * A_BYTES, &tm_w, &full[s], 0, u * BM, pol_w);
        else tma_load_2d(sa + s * A_BYTES, &tm_w, &full[s], kb * BK, t * BM, pol_w);
      };
      auto load_x = [&](int s, int u) { tma_load_2d(sb + s * B_BYTES, &tm_x, &full[s], (u % p.KB) * BK, 0, pol_x); };
      const int n = u1 - u0;
      const int pre = min(n, STAGES);
      const int pw = min(pre, p.prewait);
      for (int i = 0; i < pw; ++i) {  // weights first: they do not depend on the previous kernel
        mbar_arrive_expect_tx(&full[i], A_BYTES + B_BYTES);
        load_w(i, u0 + i);
      }
      pdl_wait();
      if (p.trace) p.trace[8 * c + 1] = globaltimer();
      for (int i = 0; i < pw; ++i) load_x(i, u0 + i);
      for (int i = pw; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], A_BYTES + B_BYTES);
        load_w(i, u0 + i);
        load_x(i, u0 + i);
      }
      for (int i = pre; i < n; ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
        load_w(s, u0 + i);
        load_x(s, u0 + i);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int i = 0, seg = 0;
      for (int u = u0; u < u1; ++seg) {
        const int t = u / p.KB;
        const int ue = min(u1, (t + 1) * p.KB);
        const int buf = seg & 1;
        mbar_wait(&tempty[buf], ((seg >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * BN;
        for (int first = 1; u < ue; ++u, ++i, first = 0) {
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(sa + s * A_BYTES);
          const uint64_t bd = umma_desc_sw128(sb + s * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16(acc, ad + 2 * kk, bd + 2 * kk, idesc, (first && kk == 0) ? 0u : 1u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[buf]);
      }
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quarters (warp % 4)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int etid = threadIdx.x - 64;  // 0..127
    // Idle until the first accumulator: pull the weight tiles beyond the
    // producer's smem ring into L2 (plain LSU prefetches, so they never queue
    // in front of the TMA loads the MMA waits for), letting HBM stream this
    // GEMM's weights while the previous kernel (norm, all-reduce) is short of
    // bytes; after the PDL wait those tiles arrive at L2 speed.
    if (p.l2pf && p.w_packed) {
      const int i0 = min(u1 - u0, STAGES), i1 = min(u1 - u0, STAGES + p.l2pf);
      constexpr int LINES = BM * BK * 2 / 128;  // 128 B lines per 16 KB tile
      for (int l = etid; l < (i1 - i0) * LINES; l += 128) {
        const uint8_t *a = p.w_ptr + (size_t)(u0 + i0 + l / LINES) * (BM * BK * 2) + (l % LINES) * 128;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
      }
    }
    int seg = 0;
    for (int u = u0; u < u1; ++seg) {
      const int t = u / p.KB;
      const int kb_lo = u - t * p.KB;
      const int ue = min(u1, (t + 1) * p.KB);
      const int kb_hi = ue - t * p.KB;
      u = ue;
      const int buf = seg & 1;
      mbar_wait(&tfull[buf], (seg >> 1) & 1);
      if (p.trace && etid == 0) p.trace[8 * c + (seg == 0 ? 4 : 6)] = globaltimer();
      tc_fence_after();
      const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + buf * BN;
      const int m = t * BM + row;
      const OutDesc ga{p.c, p.ldm, p.ldn, p.M, p.N, p.c_bf16, p.accumulate};
      const bool whole = (kb_lo == 0 && kb_hi == p.KB);
      // partial tile: slot 2c (this CTA's first segment) or 2c+1 (its last)
      // slot layout is token-major, ws[slot][token][row]: a warp's 32 rows are
      // contiguous for every token, so stores here and loads in the reducers coalesce
      float *mine = p.ws + (size_t)(2 * c + (seg == 0 ? 0 : 1)) * BM * BN + row;
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 16) {
        float v[16];
        tmem_ld16(tacc + cc, v);
        if (whole) {
          store_chunk(ga, m, cc, v);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) __stcg(mine + (size_t)(cc + j) * BM, v[j]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[buf]);
      if (whole || p.defer) continue;  // deferred: the consuming kernel sums the slots
      // release the partial (one thread, after the CTA-level barrier; acq_rel
      // fences are cumulative through bar.sync) and take a ticket
      named_bar_sync(1, 128);
      if (p.trace && etid == 0) p.trace[8 * c + 5] = globaltimer();
      const int c_first = sk_owner(t * p.KB, p.units, G);
      const int c_last = sk_owner((t + 1) * p.KB - 1, p.units, G);
      if (etid == 0) {
        const int tk = ticket_acq_rel(&p.counters[t]);
        s_last = (tk == c_last - c_first);
        if (s_last) p.counters[t] = 0;
      }
      named_bar_sync(1, 128);
      if (p.trace && etid == 0) p.trace[8 * c + 7] = globaltimer();
      if (s_last) {
#pragma unroll 1
        for (int ch = 0; ch < BN; ch += 16) {
          float acc[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = 0.f;
          // all contributors' partials are requested before any is summed (one L2
          // round trip instead of one per contributor), then added in CTA order
          constexpr int MAXC = 6;
          for (int cb = c_first; cb <= c_last; cb += MAXC) {
            float f[MAXC][16];
#pragma unroll
            for (int i = 0; i < MAXC; ++i) {
              const int cc = cb + i;
              if (cc <= c_last) {
                // tile t is the first segment of cc unless cc started before the tile (c_first only)
                const int sl = 2 * cc + (cc == c_first && sk_start(cc, p.units, G) < t * p.KB ? 1 : 0);
                const float *src = p.ws + (size_t)sl * BM * BN + (size_t)ch * BM + row;
#pragma unroll
                for (int j = 0; j < 16; ++j) f[i][j] = __ldcg(src + (size_t)j * BM);
              }
            }
#pragma unroll
            for (int i = 0; i < MAXC; ++i) {
              if (cb + i <= c_last) {
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] += f[i][j];
              }
            }
          }
          store_chunk(ga, m, ch, acc);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
  if (p.trace && threadIdx.x == 0) {
    p.trace[8 * c + 0] = t_start;
    p.trace[8 * c + 2] = globaltimer();
    p.trace[8 * c + 3] = smid();
  }
}

// ------------------------------------------------------------------ deferred split-K consumer
// x[t, :] += Y[t, :], Y = the preceding deferred stream-K GEMM's fp32 output:
// whole tiles straight from y, split tiles summed from the partial slots in CTA
// order (identical arithmetic to the in-kernel fixup); then the RMSNorm of x.
// This moves the split-K reduction (two dependent L2 round trips under a
// saturated memory system) off the GEMM's critical tail into a kernel that
// reads its input anyway.
constexpr int SK_CL = 4;

template <typename TO>
__global__ void __launch_bounds__(256)
    sk_residual_rmsnorm_kernel(float *x, const float *y, long ldy, SKView v, const float *gain, TO *out, int hidden,
                               float eps) {
  // one row = a cluster of SK_CL CTAs (each owns hidden / SK_CL features); the
  // RMS sum of squares is combined across the cluster through DSMEM
  pdl_trigger();
  __shared__ float red[8];
  __shared__ float parts[SK_CL];
  const unsigned cr = cluster_rank();
  const int t = blockIdx.x / SK_CL;
  const int per = hidden / SK_CL, base = (int)cr * per;
  float *xr = x + (size_t)t * hidden;
  if (out) cluster_arrive_relaxed();  // matched by the wait before the first DSMEM store (every CTA started)
  constexpr int MAXV = 2;  // hidden <= SK_CL * 2 * 4 * 256 = 8192
  float4 xv[MAXV], dv[MAXV], gv[MAXV];
  // the gain is a weight: fetch it before waiting on the producer GEMM
  // (batching the two gathers with sk_gather_n measured 1 % slower at 7B)
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int n = base + (i * 256 + threadIdx.x) * 4;
    if (out && n < base + per) gv[i] = __ldg(reinterpret_cast<const float4 *>(gain + n));
  }
  pdl_wait();
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int n = base + (i * 256 + threadIdx.x) * 4;
    if (n < base + per) {
      xv[i] = *reinterpret_cast<const float4 *>(xr + n);
      dv[i] = sk_gather4(v, y, ldy, t, n);
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int n = base + (i * 256 + threadIdx.x) * 4;
    if (n < base + per) {
      xv[i].x += dv[i].x; xv[i].y += dv[i].y; xv[i].z += dv[i].z; xv[i].w += dv[i].w;
      *reinterpret_cast<float4 *>(xr + n) = xv[i];
      ss += xv[i].x * xv[i].x + xv[i].y * xv[i].y + xv[i].z * xv[i].z + xv[i].w * xv[i].w;
    }
  }
  if (!out) return;  // uniform across the cluster
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  cluster_wait();
  if (threadIdx.x == 0) {  // this CTA's sum of squares into every cluster CTA's parts[rank]
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += red[i];
    for (int c = 0; c < SK_CL; ++c) dsmem_st_f32(&parts[cr], c, s);
  }
  cluster_sync_all();  // every CTA's stores into this CTA's parts[] are visible; no remote reads follow
  float tot = 0.f;
  for (int c = 0; c < SK_CL; ++c) tot += parts[c];  // same order in every CTA
  const float inv = 1.0f / sqrtf(tot / (float)hidden + eps);
  TO *o = out + (size_t)t * hidden;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int n = base + (i * 256 + threadIdx.x) * 4;
    if (n < base + per) {
      const float4 g = gv[i];
      store4(o + n, (xv[i].x * inv) * g.x, (xv[i].y * inv) * g.y, (xv[i].z * inv) * g.z, (xv[i].w * inv) * g.w);
    }
  }
}

// SwiGLU consumer of a deferred gate/up GEMM (fp32 y [n_tok][2 inter]): gate
// and up gathered like the residual consumer (whole tiles from y, split tiles
// from the partial slots in CTA order), rounded to bf16 exactly where the
// in-kernel fix-up would have stored them, then silu(gate) * up as in
// hx_swiglu -- identical bits, without the GEMM's fix-up tail.
__global__ void __launch_bounds__(256)
    sk_swiglu_kernel(const float *y, long ldy, SKView v, __nv_bfloat16 *out, long ld_out, int inter) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.y;
  const int f = (blockIdx.x * 256 + threadIdx.x) * 4;
  if (f >= inter) return;
  const float4 g = sk_gather4(v, y, ldy, t, f);
  const float4 u = sk_gather4(v, y, ldy, t, f + inter);
  const float gv[4] = {g.x, g.y, g.z, g.w}, uv[4] = {u.x, u.y, u.z, u.w};
  float r[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float gb = __bfloat162float(__float2bfloat16_rn(gv[j]));
    const float ub = __bfloat162float(__float2bfloat16_rn(uv[j]));
    r[j] = (gb / (1.0f + expf(-gb))) * ub;
  }
  store4(out + (size_t)t * ld_out + f, r[0], r[1], r[2], r[3]);
}

// ------------------------------------------------------------------ packing
// dst[(t * KB + kb) * 128 * 64 + r * 64 + c] = src[(t * 128 + r) * K + kb * 64 + c] (0 if OOB)
__global__ void pack_weight_kernel(const __nv_bfloat16 *__restrict__ src, __nv_bfloat16 *__restrict__ dst,
                                   int N, int K, int KB) {
  // no pdl_trigger(): a dependent GEMM prefetches weight tiles before its
  // griddepcontrol.wait, so it must not start until the packed weights exist
  pdl_wait();
  const size_t tile = blockIdx.x;  // t * KB + kb
  const int t = (int)(tile / KB), kb = (int)(tile % KB);
  for (int e = threadIdx.x * 8; e < BM * BK; e += blockDim.x * 8) {
    const int r = e / BK, c = e % BK;
    const int n = t * BM + r, k = kb * BK + c;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (n < N && k + 8 <= K) {
      v = *reinterpret_cast<const uint4 *>(src + (size_t)n * K + k);
    } else if (n < N) {
      __nv_bfloat16 tmp[8];
      for (int j = 0; j < 8; ++j) tmp[j] = k + j < K ? src[(size_t)n * K + k + j] : __float2bfloat16_rn(0.f);
      v = *reinterpret_cast<uint4 *>(tmp);
    }
    *reinterpret_cast<uint4 *>(dst + tile * BM * BK + e) = v;
  }
}

// ------------------------------------------------------------------ fp32 SIMT
// Y[t, n] = sum_k X[t, k] W[n, k]; 64x64 tile, 256 threads x (4x4).
__global__ void __launch_bounds__(256)
    gemm_f32_simt_kernel(const float *__restrict__ w, const float *__restrict__ x, float *y,
                         int n_tok, int n_out, int K, int ldy, int accumulate) {
  pdl_trigger();
  pdl_wait();
  __shared__ float xs[16][64 + 4];
  __shared__ float ws[16][64 + 4];
  const int t0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int r = i / 16, kk = i % 16;
      const int t = t0 + r, n = n0 + r, k = k0 + kk;
      xs[kk][r] = (t < n_tok && k < K) ? x[(size_t)t * K + k] : 0.f;
      ws[kk][r] = (n < n_out && k < K) ? w[(size_t)n * K + k] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = xs[kk][ty * 4 + i];
        b[i] = ws[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + ty * 4 + i;
    if (t >= n_tok) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < n_out) {
        float *dst = y + (size_t)t * ldy + n;
        *dst = accumulate ? *dst + acc[i][j] : acc[i][j];
      }
    }
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static int get_encode() {
  std::call_once(g_encode_once, [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode ? 0 : HX_ERR_DRIVER;
}

// 2-D bf16 tensor [rows, cols] row-major with row pitch `pitch` elements;
// box = box_rows x 64 columns, 128B swizzle.
static int make_map(CUtensorMap *map, const void *ptr, long rows, int cols, long pitch, int box_rows) {
  if (get_encode()) return HX_ERR_DRIVER;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : HX_ERR_DRIVER;
}

int make_tma_bf16_sw128(CUtensorMap *map, const void *ptr, long rows, int cols, long pitch, int box_rows) {
  return make_map(map, ptr, rows, cols, pitch, box_rows);
}

template <int BN, int STAGES>
static size_t smem_bytes() {
  return 1024 + STAGES * (BM * BK * 2 + BN * BK * 2) + (2 * STAGES + 1) * 8 + 16;
}

template <int BN, int STAGES>
static int launch_tc(const CUtensorMap &ma, const CUtensorMap &mb, const GemmArgs &p, int splits,
                     cudaStream_t st) {
  const size_t smem = smem_bytes<BN, STAGES>();
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(gemm_bf16_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr_done = true;
  }
  dim3 grid((p.M + BM - 1) / BM, (p.N + BN - 1) / BN, splits);
  return launch(gemm_bf16_tc_kernel<BN, STAGES>, grid, dim3(128), smem, st, ma, mb, p);
}

struct Plan {
  bool decode;
  int bn;
  int splits;
  int kb_per;
  int tiles;
};

static Plan plan_gemm(int n_tok, int n_out, int K) {
  Plan pl{};
  const int kb = (K + BK - 1) / BK;
  pl.decode = n_tok <= 64;
  if (pl.decode) {
    pl.bn = n_tok <= 16 ? 16 : (n_tok <= 32 ? 32 : 64);
    pl.tiles = (n_out + BM - 1) / BM;
    const int slots = 2 * kNumSMs;
    double best = -1.0;
    pl.splits = 1;
    pl.kb_per = kb;
    for (int s = 1; s <= 16; ++s) {
      const int per = (kb + s - 1) / s;
      if (per < 4 && s > 1) break;
      const int se = (kb + per - 1) / per;
      const int ctas = pl.tiles * se;
      const double eff = (double)ctas / (double)(((ctas + slots - 1) / slots) * slots);
      if (eff > best + 0.02) {
        best = eff;
        pl.splits = se;
        pl.kb_per = per;
      }
    }
  } else {
    pl.bn = 256;
    pl.tiles = ((n_tok + BM - 1) / BM) * ((n_out + 255) / 256);
    pl.splits = 1;
    pl.kb_per = kb;
  }
  return pl;
}

}  // namespace hx

using namespace hx;

// The stream-K decode GEMM is persistent: one CTA per SM (see launch_sk).
// persistent stream-K grid: one CTA per SM (HX_SK_CTAS overrides, e.g. 296 = 2 per SM)
static int sk_ctas() {
  static const int n = [] {
    const char *e = getenv("HX_SK_CTAS");
    return e ? atoi(e) : kNumSMs;
  }();
  return n;
}
static int sk_grid(int units) { return std::min(units, sk_ctas()); }

// debug timeline: 8 u64 per stream-K CTA (start, dependency-wait done, end, smid,
// seg0 accumulator ready, seg0 epilogue done, last-seg accumulator ready, #segments)
static unsigned long long *g_trace = nullptr;
static size_t g_trace_cap = 0, g_trace_pos = 0;

// n CTA slots of the same trace for another traced kernel (decode attention), or null
namespace hx {
unsigned long long *hx_trace_slots(size_t n);
}
unsigned long long *hx::hx_trace_slots(size_t n) {
  if (!g_trace || g_trace_pos + n > g_trace_cap) return nullptr;
  unsigned long long *t = g_trace + 8 * g_trace_pos;
  g_trace_pos += n;
  return t;
}

extern "C" size_t hx_linear_workspace(int dtype, int n_tok, int n_out, int k_dim) {
  if (dtype != HX_BF16) return 0;
  Plan pl = plan_gemm(n_tok, n_out, k_dim);
  if (pl.decode) {  // stream-K: two partial slots per CTA
    const int units = pl.tiles * ((k_dim + BK - 1) / BK);
    return kTicketBytes + (size_t)2 * sk_grid(units) * BM * pl.bn * sizeof(float);
  }
  if (pl.splits <= 1) return 0;
  return kTicketBytes + (size_t)pl.tiles * pl.splits * BM * pl.bn * sizeof(float);
}

template <int BN, int STAGES>
static int launch_sk(const CUtensorMap &mw, const CUtensorMap &mx, const SKArgs &p, cudaStream_t st) {
  // The request is floored at just over half an SM's shared memory so that
  // exactly one stream-K CTA lands on every SM: when two fit, the block
  // scheduler may stack two CTAs of the same launch on one SM (measured +0.11
  // ms per 7B decode step). Smaller kernels (norms, attention) still co-reside
  // under PDL.
  const size_t kOneCtaPerSm = sk_ctas() > kNumSMs ? 0 : 116 * 1024;
  const size_t smem = std::max<size_t>(kOneCtaPerSm, 1024 + STAGES * (BM * BK * 2 + BN * BK * 2) + (2 * STAGES + 4) * 8 + 32);
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(gemm_streamk_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_done = true;
  }
  return launch(gemm_streamk_kernel<BN, STAGES>, dim3(sk_grid(p.units)), dim3(192), smem, st, mw, mx, p);
}

namespace hx {
// The deferred-reduction view of hx_linear(n_tok, n_out, k_dim) with workspace ws.
int sk_view_for(int n_tok, int n_out, int k_dim, const void *workspace, SKView *v) {
  Plan pl = plan_gemm(n_tok, n_out, k_dim);
  if (!pl.decode) return HX_ERR_UNSUPPORTED;
  v->ws = reinterpret_cast<const float *>(reinterpret_cast<const uint8_t *>(workspace) + kTicketBytes);
  v->KB = (k_dim + BK - 1) / BK;
  v->units = pl.tiles * v->KB;
  v->G = sk_grid(v->units);
  v->BN = pl.bn;
  return 0;
}
}  // namespace hx

extern "C" int hx_splitk_residual_rmsnorm(float *x, const float *y, int ldy, const void *workspace, int n_tok,
                                          int n_out, int k_dim, const float *gain, void *out, int out_dtype,
                                          float eps, hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!x || !y || !workspace || n_out % 4 || n_out > 8 * 4 * 256 || ldy % 4 || (out && !gain)) return HX_ERR_ARG;
  Plan pl = plan_gemm(n_tok, n_out, k_dim);
  if (!pl.decode) return HX_ERR_UNSUPPORTED;
  SKView v;
  v.ws = reinterpret_cast<const float *>(reinterpret_cast<const uint8_t *>(workspace) + kTicketBytes);
  v.KB = (k_dim + BK - 1) / BK;
  v.units = pl.tiles * v.KB;
  v.G = sk_grid(v.units);
  v.BN = pl.bn;
  cudaStream_t st = as_stream(stream);
  if (n_out % (SK_CL * 4)) return HX_ERR_UNSUPPORTED;
  if (out_dtype == HX_BF16)
    return launch_cluster(sk_residual_rmsnorm_kernel<__nv_bfloat16>, dim3(n_tok * SK_CL), dim3(256), 0, st, SK_CL, x,
                          y, (long)ldy, v, gain, (__nv_bfloat16 *)out, n_out, eps);
  return launch_cluster(sk_residual_rmsnorm_kernel<float>, dim3(n_tok * SK_CL), dim3(256), 0, st, SK_CL, x, y,
                        (long)ldy, v, gain, (float *)out, n_out, eps);
}

extern "C" int hx_splitk_swiglu(const float *y, int ldy, const void *workspace, int n_tok, int inter, int k_dim,
                                void *out, int ld_out, hx_stream_t stream) {
  if (n_tok == 0) return 0;
  if (!y || !workspace || !out || inter % 4 || ldy % 4 || ld_out % 4 || ldy < 2 * inter) return HX_ERR_ARG;
  Plan pl = plan_gemm(n_tok, 2 * inter, k_dim);
  if (!pl.decode) return HX_ERR_UNSUPPORTED;
  SKView v;
  v.ws = reinterpret_cast<const float *>(reinterpret_cast<const uint8_t *>(workspace) + kTicketBytes);
  v.KB = (k_dim + BK - 1) / BK;
  v.units = pl.tiles * v.KB;
  v.G = sk_grid(v.units);
  v.BN = pl.bn;
  return launch(sk_swiglu_kernel, dim3((inter / 4 + 255) / 256, n_tok), dim3(256), 0, as_stream(stream), y, (long)ldy,
                v, (__nv_bfloat16 *)out, (long)ld_out, inter);
}

extern "C" size_t hx_debug_trace(void *buf, size_t records) {
  const size_t used = g_trace_pos;
  g_trace = reinterpret_cast<unsigned long long *>(buf);
  g_trace_cap = buf ? records : 0;
  g_trace_pos = 0;
  return used;
}

extern "C" size_t hx_packed_weight_elems(int n_out, int k_dim) {
  return (size_t)((n_out + BM - 1) / BM) * ((k_dim + BK - 1) / BK) * BM * BK;
}

extern "C" int hx_pack_weight(const void *w, void *packed, int n_out, int k_dim, hx_stream_t stream) {
  if (!w || !packed || n_out <= 0 || k_dim <= 0 || k_dim % 8) return HX_ERR_ARG;
  const int KB = (k_dim + BK - 1) / BK;
  const int tiles = ((n_out + BM - 1) / BM) * KB;
  return launch(pack_weight_kernel, dim3(tiles), dim3(256), 0, as_stream(stream), (const __nv_bfloat16 *)w,
                (__nv_bfloat16 *)packed, n_out, k_dim, KB);
}

extern "C" int hx_linear(const void *w, const void *x, void *y, int dtype, int y_dtype, int n_tok, int n_out,
                         int k_dim, int ldy, int flags, void *workspace, size_t workspace_bytes, hx_stream_t stream) {
  if (n_tok <= 0 || n_out <= 0 || k_dim <= 0) return n_tok == 0 ? 0 : HX_ERR_ARG;
  if (!w || !x || !y || ldy < n_out) return HX_ERR_ARG;
  const int accumulate = flags & HX_LINEAR_ACCUMULATE;
  const int packed = (flags & HX_LINEAR_PACKED) ? 1 : 0;
  cudaStream_t st = as_stream(stream);
  if (dtype == HX_F32) {
    if (y_dtype != HX_F32 || packed) return HX_ERR_UNSUPPORTED;
    dim3 grid((n_out + 63) / 64, (n_tok + 63) / 64);
    return launch(gemm_f32_simt_kernel, grid, dim3(256), 0, st, (const float *)w, (const float *)x, (float *)y,
                  n_tok, n_out, k_dim, ldy, accumulate);
  }
  if (dtype != HX_BF16) return HX_ERR_ARG;
  if (k_dim % 8) return HX_ERR_UNSUPPORTED;  // TMA row pitch must be 16B aligned
  if (accumulate && y_dtype != HX_F32) return HX_ERR_UNSUPPORTED;
  Plan pl = plan_gemm(n_tok, n_out, k_dim);
  GemmArgs p{};
  p.c = y;
  p.K = k_dim;
  p.c_bf16 = (y_dtype == HX_BF16);
  p.accumulate = accumulate;
  p.kb_total = (k_dim + BK - 1) / BK;
  p.kb_per_split = pl.kb_per;
  p.w_packed = packed;
  CUtensorMap ma, mb;
  int rc;
  const long packed_rows = (long)((n_out + BM - 1) / BM) * p.kb_total * BM;
  if (pl.decode) {
    rc = packed ? make_map(&ma, w, packed_rows, BK, BK, BM) : make_map(&ma, w, n_out, k_dim, k_dim, BM);
    if (rc) return rc;
    if ((rc = make_map(&mb, x, n_tok, k_dim, k_dim, pl.bn))) return rc;
    SKArgs sk{};
    static const int l2pf = [] {
      const char *e = getenv("HX_GEMM_L2PF");
      return e ? atoi(e) : 16;
    }();
    static const int l2pf_all = [] {
      const char *e = getenv("HX_GEMM_L2PF_ALL");
      return e ? atoi(e) : 0;
    }();
    sk.l2pf = ((flags & HX_LINEAR_L2_PREFETCH) || l2pf_all) ? l2pf : 0;
    sk.w_ptr = reinterpret_cast<const uint8_t *>(w);
    sk.c = y; sk.ldm = 1; sk.ldn = ldy; sk.M = n_out; sk.N = n_tok;
    sk.c_bf16 = p.c_bf16; sk.accumulate = accumulate; sk.w_packed = packed;
    sk.defer = (flags & HX_LINEAR_DEFER_REDUCE) ? 1 : 0;
    if (sk.defer && (p.c_bf16 || accumulate)) return HX_ERR_UNSUPPORTED;
    sk.KB = p.kb_total; sk.units = pl.tiles * p.kb_total;
    const size_t need = hx_linear_workspace(dtype, n_tok, n_out, k_dim);
    if (!workspace || workspace_bytes < need) return HX_ERR_WORKSPACE;
    if (pl.tiles > kMaxTickets) return HX_ERR_UNSUPPORTED;
    sk.counters = reinterpret_cast<int *>(workspace);
    sk.ws = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(workspace) + kTicketBytes);
    const size_t g = (size_t)sk_grid(sk.units);
    static const int prewait = [] {  // HX_SK_PREWAIT: ring stages streamed before the PDL wait (tuning)
      const char *e = getenv("HX_SK_PREWAIT");
      return e ? atoi(e) : 64;
    }();
    sk.prewait = prewait;
    if (g_trace && g_trace_pos + g <= g_trace_cap) {
      sk.trace = g_trace + 8 * g_trace_pos;
      g_trace_pos += g;
    }
    // ring depths 6 / 5 / 4 (BN 16 / 32 / 64): deeper rings (HX_SK_STAGES 8-12,
    // HX_SK32_STAGES 7-9 in round 1) measured neutral and were dropped
    switch (pl.bn) {
      case 16: return launch_sk<16, 6>(ma, mb, sk, st);
      case 32: return launch_sk<32, 5>(ma, mb, sk, st);
      default: return launch_sk<64, 4>(ma, mb, sk, st);
    }
  } else {
    p.M = n_tok; p.N = n_out; p.ldm = ldy; p.ldn = 1; p.a_is_weight = 0;
    if ((rc = make_map(&ma, x, n_tok, k_dim, k_dim, BM))) return rc;
    rc = packed ? make_map(&mb, w, packed_rows, BK, BK, BM) : make_map(&mb, w, n_out, k_dim, k_dim, pl.bn);
    if (rc) return rc;
  }
  if (pl.splits > 1) {
    const size_t need = hx_linear_workspace(dtype, n_tok, n_out, k_dim);
    if (!workspace || workspace_bytes < need) return HX_ERR_WORKSPACE;
    if (pl.tiles > kMaxTickets) return HX_ERR_UNSUPPORTED;
    p.counters = reinterpret_cast<int *>(workspace);
    p.ws = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(workspace) + kTicketBytes);
  }
  static const int persistent = [] {  // 0: one CTA per tile (round-1 kernel); 2: every shape <= 4096 tiles
    const char *e = getenv("HX_GEMM_PERSISTENT");
    return e ? atoi(e) : 1;
  }();
  // measured in the engine (same-box A/B, profiles/r02/prefill_gemm_persistent.txt):
  // 7B one-shot prefill (4096 token rows) 54.2 -> 51.9 ms persistent; C3 asym
  // (2048-row micro-batches, <= 1024 tiles) 67.0 -> 64.5 ms; but 70B [1,1]
  // micro-batched gate/up (2048 x 57344, 3584 tiles) costs 2415 -> 2529 ms when
  // persistent, and one-shot 32768-row GEMMs (>= 8192 tiles) lose 10-20 %. So:
  // persistent up to 1024 tiles, and for >= 4096-row GEMMs up to 4096 tiles.
  const int n_tiles = ((p.M + BM - 1) / BM) * ((p.N + 255) / 256);
  if (persistent && pl.bn == 256 && pl.splits == 1 && !p.a_is_weight && n_tiles <= 4096 &&
      (n_tiles <= 1024 || p.M >= 4096 || persistent == 2)) {
    constexpr int STG = 4;
    const size_t smem = 1024 + STG * (BM * BK * 2 + 256 * BK * 2) + (2 * STG + 4) * 8 + 16;
    static bool attr_done = false;
    if (!attr_done) {
      cudaFuncSetAttribute(gemm_tc_persistent_kernel<256, STG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      attr_done = true;
    }
    const int tiles = ((p.M + BM - 1) / BM) * ((p.N + 255) / 256);
    return launch(gemm_tc_persistent_kernel<256, STG>, dim3(std::min(tiles, kNumSMs)), dim3(192), smem, st, ma, mb,
                  p);
  }
  switch (pl.bn) {
    case 16: return launch_tc<16, 6>(ma, mb, p, pl.splits, st);
    case 32: return launch_tc<32, 6>(ma, mb, p, pl.splits, st);
    case 64: return launch_tc<64, 5>(ma, mb, p, pl.splits, st);
    default: return launch_tc<256, 4>(ma, mb, p, pl.splits, st);
  }
}
