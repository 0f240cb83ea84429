// Shared helpers for the hx_* sm_100a kernels: dtype traits, launch
// bookkeeping and the Blackwell PTX wrappers (mbarrier, TMA, tcgen05/TMEM).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hx_api.h"

namespace hx {

extern unsigned long long g_launches;

// Every split-K / split-KV workspace starts with a fixed-size array of ticket
// counters (zeroed once by the caller, re-armed by the kernels), so kernels of
// different shapes sharing one workspace never overlay partials on tickets.
constexpr size_t kTicketBytes = 16384;
constexpr int kMaxTickets = (int)(kTicketBytes / sizeof(int));

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  ++g_launches;
  return e == cudaSuccess ? 0 : (int)e;
}

inline cudaStream_t as_stream(hx_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: every hx kernel triggers its dependents at
// entry and waits (griddepcontrol.wait) before touching data written by the
// previous kernel, so a kernel's launch, prologue and -- for the decode GEMM --
// its first weight-tile loads overlap the previous kernel's tail. Captured
// into CUDA graphs as programmatic edges. The one exception is hx_advance (the
// only kernel that writes seq_lens): it never triggers early, so any later
// kernel may read seq_lens and the KV pages below it before its own wait.
extern int g_pdl;

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Every hx kernel runs with the maximum shared-memory carveout so the SM's
// L1/smem split never has to be reconfigured (which drains the SM) between
// consecutive kernels: a PDL-launched successor can become co-resident with
// its predecessor's tail.
void set_max_carveout(const void *fn);

// PDL launch with a thread-block cluster of `cluster_x` CTAs along x
template <typename... KArgs, typename... Args>
inline int launch_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          int cluster_x, Args &&...args) {
  static bool configured = false;
  if (!configured) {
    set_max_carveout(reinterpret_cast<const void *>(kern));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  ++g_launches;
  if (e != cudaSuccess) return (int)e;
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

// cluster helpers: rank in cluster, DSMEM read of another CTA's shared float, cluster barrier
__device__ __forceinline__ unsigned cluster_nctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ float dsmem_ld_f32(const float *local_addr, unsigned cta) {
  uint32_t remote;
  const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(local_addr));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(cta));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}
__device__ __forceinline__ void dsmem_st_f32(float *local_addr, unsigned cta, float v) {
  uint32_t remote;
  const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(local_addr));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(cta));
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(v) : "memory");
}
// split cluster barrier: arrive early (no ordering), wait before the first DSMEM access
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// host: 2-D bf16 TMA map [rows, cols] (row pitch in elements), box = box_rows
// rows x 64 columns (128 B), 128B swizzle (hx_gemm.cu)
int make_tma_bf16_sw128(CUtensorMap *map, const void *ptr, long rows, int cols, long pitch, int box_rows);

template <typename... KArgs, typename... Args>
inline int launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                  Args &&...args) {
  static bool configured = false;  // one flag per kernel instantiation
  if (!configured) {
    set_max_carveout(reinterpret_cast<const void *>(kern));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  ++g_launches;
  if (e != cudaSuccess) return (int)e;
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
// rotate-half RoPE of the pair (x1, x2) = (x[i], x[i + hd/2]) by angle (cos c, sin s).
// Explicit _rn ops: no FMA contraction, so every kernel that rotates (and the
// numpy oracle, which rounds each product) produces the same bits.
__device__ __forceinline__ float2 rope_rot(float x1, float x2, float c, float s) {
  return make_float2(__fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, s)), __fadd_rn(__fmul_rn(x2, c), __fmul_rn(x1, s)));
}
// four consecutive outputs in one vector store (dst 4-element aligned)
__device__ __forceinline__ void store4(float *dst, float a, float b, float c, float d) {
  *reinterpret_cast<float4 *>(dst) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void store4(__nv_bfloat16 *dst, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t *>(&lo);
  u.y = *reinterpret_cast<uint32_t *>(&hi);
  *reinterpret_cast<uint2 *>(dst) = u;
}

// 16-byte vector of T: 4 floats or 8 bf16.
template <typename T> struct Vec16;
template <> struct Vec16<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void load(const float *p, float *out) {
    float4 v = *reinterpret_cast<const float4 *>(p);
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  }
  __device__ __forceinline__ static void store(float *p, const float *in) {
    *reinterpret_cast<float4 *>(p) = make_float4(in[0], in[1], in[2], in[3]);
  }
};
template <> struct Vec16<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void load(const __nv_bfloat16 *p, float *out) {
    uint4 v = *reinterpret_cast<const uint4 *>(p);
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      out[2 * i] = f.x; out[2 * i + 1] = f.y;
    }
  }
  __device__ __forceinline__ static void store(__nv_bfloat16 *p, const float *in) {
    uint4 v;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(in[2 * i], in[2 * i + 1]);
    *reinterpret_cast<uint4 *>(p) = v;
  }
};

// Split-K / split-KV ticket: acq_rel fence + atomic increment by one thread.
// Writers: all threads store their partials, bar.sync, then one thread takes
// the ticket (the fence releases the CTA's stores, cumulative through the
// barrier). The thread drawing the last ticket has acquired every partial;
// after the next bar.sync its CTA reads them with ld.cg. Much cheaper than a
// sequentially consistent __threadfence() in every thread.
__device__ __forceinline__ int ticket_acq_rel(int *counter) {
  int old;
  asm volatile("fence.acq_rel.gpu;\n\tatom.global.add.s32 %0, [%1], 1;\n\tfence.acq_rel.gpu;"
               : "=r"(old)
               : "l"(counter)
               : "memory");
  return old;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- PTX: mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order this thread's generic-proxy global stores before later async-proxy (TMA) reads
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Bounded wait: a pipeline bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spins = 0;; ++spins) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (spins > (1u << 28)) __trap();
  }
}

// ---------------------------------------------------------------- warp MMA (attention)
// m16n8k16 bf16 -> f32 warp MMA and ldmatrix; used by the attention kernels,
// whose per-tile shapes (16-row query tiles, 8-wide key/dim tiles) map onto
// warp-level fragments with the softmax kept in registers.
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16_16816(float *d, const uint32_t *a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- PTX: TMA
// bring one TMA box of a 2-D tensor into L2 (no smem, no barrier)
__device__ __forceinline__ void tma_prefetch_l2_2d(const CUtensorMap *map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y)
               : "memory");
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

// ---------------------------------------------------------------- PTX: tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate)
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, K-major, 128B swizzle: rows of 128 B, 8-row
// core groups 1024 B apart (SBO), version 1 (sm_100), layout SWIZZLE_128B = 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(const void *smem_tile) {
  uint64_t addr = smem_u32(smem_tile);
  return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor: bf16 x bf16 -> f32, both K-major, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// ---------------------------------------------------------------- stream-K partition
// The persistent decode GEMM (hx_gemm.cu) splits units = (128-row tile, 64-wide
// K block) evenly over G CTAs: CTA c owns [sk_start(c), sk_start(c + 1)). A
// tile covered by one CTA is written whole; a tile split across CTAs leaves
// fp32 partials in workspace slots 2c (c's first segment) / 2c + 1 (its last),
// laid out [slot][token][128 rows]. Consumers of a deferred GEMM
// (HX_LINEAR_DEFER_REDUCE) sum those partials in CTA order -- the same
// arithmetic as the in-kernel fix-up, so the bits are identical.
constexpr int kSkRows = 128;

__device__ __forceinline__ int sk_start(int c, int units, int G) { return (int)((unsigned)(c * units) / (unsigned)G); }

// first CTA whose range contains unit u: the largest c with sk_start(c) <= u,
// i.e. c * units < (u + 1) * G (one division; every CTA owns >= 1 unit)
__device__ __forceinline__ int sk_owner(int u, int units, int G) {
  return min(G - 1, (int)(((unsigned)(u + 1) * (unsigned)G - 1u) / (unsigned)units));
}

struct SKView {
  const float *ws;  // partial slots (workspace + kTicketBytes)
  int units, KB, G, BN;
};

// host: the view of hx_linear(n_tok, n_out, k_dim) deferred into `workspace`
int sk_view_for(int n_tok, int n_out, int k_dim, const void *workspace, SKView *v);

// tile tt of a deferred GEMM: CTAs c_first..c_last contributed; c_first's
// partial sits in slot0 (2 c_first, or 2 c_first + 1 when the tile is the last
// segment of a range that began before it), every later contributor began
// inside the tile (its first segment, slot 2 c); one contributor = a whole tile
// stored straight to y
struct SkTile {
  int c_first, c_last, slot0;
  __device__ __forceinline__ bool whole() const { return c_first == c_last; }
  __device__ __forceinline__ int slot(int c) const { return c == c_first ? slot0 : 2 * c; }
};

__device__ __forceinline__ SkTile sk_tile(const SKView &v, int tt) {
  SkTile t;
  t.c_first = sk_owner(tt * v.KB, v.units, v.G);
  t.c_last = sk_owner((tt + 1) * v.KB - 1, v.units, v.G);
  t.slot0 = 2 * t.c_first + (sk_start(t.c_first, v.units, v.G) < tt * v.KB ? 1 : 0);
  return t;
}

// NQ float4 gathers at once (features n[q]..n[q]+3 of token t): the tiles'
// contributor ranges ti[q] are computed by the caller (before its dependency
// wait -- they are GEMM geometry, not data) and every item's contributor loads
// are in flight together; per item the sum is sk_gather4's (CTA order from 0).
template <int NQ>
__device__ __forceinline__ void sk_gather_n(const SKView &v, const SkTile (&ti)[NQ], const float *y, long ldy, int t,
                                            const int (&n)[NQ], const bool (&act)[NQ], float4 (&out)[NQ]) {
  constexpr int MAXC = 8;
  int cl[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    out[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    cl[q] = -1;
    if (act[q]) {
      if (ti[q].whole()) out[q] = *reinterpret_cast<const float4 *>(y + (long)t * ldy + n[q]);
      else cl[q] = ti[q].c_last;
    }
  }
  for (int base = 0;; base += MAXC) {
    float4 f[NQ][MAXC];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int k = 0; k < MAXC; ++k) {
        const int cc = ti[q].c_first + base + k;
        if (cc <= cl[q])
          f[q][k] = __ldcg(reinterpret_cast<const float4 *>(v.ws + ((size_t)ti[q].slot(cc) * v.BN + t) * kSkRows +
                                                            n[q] % kSkRows));
      }
    bool more = false;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
#pragma unroll
      for (int k = 0; k < MAXC; ++k)
        if (ti[q].c_first + base + k <= cl[q]) {
          out[q].x += f[q][k].x; out[q].y += f[q][k].y; out[q].z += f[q][k].z; out[q].w += f[q][k].w;
        }
      more |= ti[q].c_first + base + MAXC <= cl[q];
    }
    if (!more) break;
  }
}

__device__ __forceinline__ float4 sk_gather4(const SKView &v, const float *y, long ldy, int t, int n) {
  const int tt = n / kSkRows, r = n % kSkRows;
  const SkTile ti = sk_tile(v, tt);
  if (ti.whole()) return *reinterpret_cast<const float4 *>(y + (long)t * ldy + n);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  constexpr int MAXC = 8;  // all contributors' loads in flight together
  for (int cb = ti.c_first; cb <= ti.c_last; cb += MAXC) {
    float4 f[MAXC];
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      const int cc = cb + i;
      if (cc <= ti.c_last)
        f[i] = __ldcg(reinterpret_cast<const float4 *>(v.ws + ((size_t)ti.slot(cc) * v.BN + t) * kSkRows + r));
    }
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      if (cb + i <= ti.c_last) {
        acc.x += f[i].x; acc.y += f[i].y; acc.z += f[i].z; acc.w += f[i].w;
      }
    }
  }
  return acc;
}

}  // namespace hx
