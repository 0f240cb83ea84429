// Inter-stage reshard over NVLink P2P (decode): stage j -> stage j+1 hidden
// state hand-off and the last stage -> stage 0 token-id return.
//
// Replaces the paper's leader send + TP-group broadcast (the
// reference models it as pp_comm_cost over the fastest cross link,
// costs.py:150-165). After stage j's row-parallel all-reduce every TP rank holds
// the identical hidden state, so receiver r' of stage j+1 takes it from sender
// r' mod TP_j (topology.py): a TP_j -> TP_{j+1} reshard in which each receiver
// gets exactly one message and no rank broadcasts.
//
// Transport: the sender kernel STORES the rows straight into the receiver's
// inbox over NVLink (cudaIpc-mapped); the receiver kernel polls its own local
// inbox until the data itself has landed -- every 32-bit word of an armed
// inbox holds the sentinel 0x80000000 (-0.0f / INT_MIN) and pushed words equal
// to it are sent as 0 (fp32 -0.0 -> +0.0, value-preserving; ids are >= 0). One
// one-way NVLink trip, no flags, no fences, no host involvement: both kernels
// live inside the stages' decode CUDA graphs and the GPUs synchronise among
// themselves. Inbox = 3 buffers of max_words; hand-off k uses buffer k % 3 and
// the receiver re-arms buffer (k + 2) % 3 (consumed at k - 1; the sender cannot
// reach k + 2 before the receiver has finished k + 1, because the next step's
// input depends on the receiver's output through the token loop). Each side
// keeps its own call counter (int[2], zeroed) in device memory.
#include "hx_common.cuh"

namespace hx {

constexpr int kMaxDst = 8;
constexpr uint32_t kHandoffSentinel = 0x80000000u;

struct HandoffDsts {
  uint32_t *box[kMaxDst];
};

__device__ __forceinline__ uint32_t hand_clean(uint32_t v) { return v == kHandoffSentinel ? 0u : v; }

__device__ __forceinline__ void bump_call(int *state, int call) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int done = atomicAdd(state + 1, 1);
    if (done == (int)gridDim.x - 1) {
      state[1] = 0;
      *(volatile int *)state = call + 1;
    }
  }
}

__global__ void __launch_bounds__(256)
    handoff_push_kernel(const uint32_t *__restrict__ src, HandoffDsts d, int n_dst, size_t words, size_t max_words,
                        int *state) {
  pdl_trigger();
  pdl_wait();  // src was written by the previous kernel
  const int call = *(volatile int *)state;
  const size_t base = (size_t)(call % 3) * max_words;
  const size_t nv = words / 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    uint4 v = __ldcs(reinterpret_cast<const uint4 *>(src) + i);
    v.x = hand_clean(v.x); v.y = hand_clean(v.y); v.z = hand_clean(v.z); v.w = hand_clean(v.w);
    for (int k = 0; k < n_dst; ++k) reinterpret_cast<uint4 *>(d.box[k] + base)[i] = v;
  }
  for (size_t i = nv * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += stride) {
    const uint32_t v = hand_clean(src[i]);
    for (int k = 0; k < n_dst; ++k) d.box[k][base + i] = v;
  }
  bump_call(state, call);
}

__device__ __forceinline__ uint4 ld_volatile_v4(const uint4 *p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(256)
    handoff_pull_kernel(uint32_t *__restrict__ dst, uint32_t *inbox, size_t words, size_t max_words, int *state) {
  pdl_trigger();
  pdl_wait();  // the previous kernel may still read dst
  const int call = *(volatile int *)state;
  const uint32_t *buf = inbox + (size_t)(call % 3) * max_words;
  uint32_t *rearm = inbox + (size_t)((call + 2) % 3) * max_words;
  const size_t nv = words / 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const uint4 s4 = make_uint4(kHandoffSentinel, kHandoffSentinel, kHandoffSentinel, kHandoffSentinel);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    const uint4 *p = reinterpret_cast<const uint4 *>(buf) + i;
    uint4 v = ld_volatile_v4(p);
    for (uint32_t spins = 0; v.x == kHandoffSentinel || v.y == kHandoffSentinel || v.z == kHandoffSentinel ||
                             v.w == kHandoffSentinel;
         ++spins) {
      if (spins > (1u << 26)) __trap();  // the sender never arrived: fail loudly, never hang
      v = ld_volatile_v4(p);
    }
    reinterpret_cast<uint4 *>(dst)[i] = v;
  }
  for (size_t i = nv * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += stride) {
    uint32_t v = ld_volatile_u32(buf + i);
    for (uint32_t spins = 0; v == kHandoffSentinel; ++spins) {
      if (spins > (1u << 26)) __trap();
      v = ld_volatile_u32(buf + i);
    }
    dst[i] = v;
  }
  // re-arm the buffer consumed by the previous hand-off (the whole buffer: sizes may vary)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < max_words / 4; i += stride)
    reinterpret_cast<uint4 *>(rearm)[i] = s4;
  for (size_t i = (max_words / 4) * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < max_words; i += stride)
    rearm[i] = kHandoffSentinel;
  bump_call(state, call);
}

// ------------------------------------------------------------- credit-based stream (prefill)
// The prefill's stage j pushes micro-batch after micro-batch without waiting for
// stage j+1, so the decode protocol's "the sender cannot lap the receiver"
// argument does not hold. Flow control by credits: the inbox carries a credit
// word after its 3 buffers (kCreditOffset); the receiver, after copying
// hand-off k out of buffer k % 3 and re-arming that buffer in place, publishes
// credit = k + 1 (release, system scope); the sender's hand-off k first waits
// (acquire, over NVLink) until credit >= k - 2, i.e. buffer k % 3 was drained.
__device__ __forceinline__ int ld_acquire_sys_s32(const int *p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_s32(int *p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__host__ __device__ __forceinline__ int *credit_word(uint32_t *inbox, size_t max_words) {
  return reinterpret_cast<int *>(inbox + 3 * max_words);
}

__global__ void __launch_bounds__(256)
    handoff_push_credit_kernel(const uint32_t *__restrict__ src, uint32_t *box, size_t words, size_t max_words,
                               int *state) {
  pdl_trigger();
  pdl_wait();  // src was written by the previous kernel
  const int call = *(volatile int *)state;
  if (threadIdx.x == 0) {
    const int *credit = credit_word(box, max_words);
    for (uint32_t spins = 0; ld_acquire_sys_s32(credit) < call - 2; ++spins)
      if (spins > (1u << 26)) __trap();  // the receiver never drained: fail loudly, never hang
  }
  __syncthreads();
  uint32_t *dst = box + (size_t)(call % 3) * max_words;
  const size_t nv = words / 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    uint4 v = __ldcs(reinterpret_cast<const uint4 *>(src) + i);
    v.x = hand_clean(v.x); v.y = hand_clean(v.y); v.z = hand_clean(v.z); v.w = hand_clean(v.w);
    reinterpret_cast<uint4 *>(dst)[i] = v;
  }
  for (size_t i = nv * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += stride)
    dst[i] = hand_clean(src[i]);
  bump_call(state, call);
}

__global__ void __launch_bounds__(256)
    handoff_pull_credit_kernel(uint32_t *__restrict__ dst, uint32_t *inbox, size_t words, size_t max_words,
                               int *state) {
  pdl_trigger();
  pdl_wait();  // the previous kernel may still read dst
  const int call = *(volatile int *)state;
  uint32_t *buf = inbox + (size_t)(call % 3) * max_words;
  const size_t nv = words / 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const uint4 s4 = make_uint4(kHandoffSentinel, kHandoffSentinel, kHandoffSentinel, kHandoffSentinel);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    uint4 *p = reinterpret_cast<uint4 *>(buf) + i;
    uint4 v = ld_volatile_v4(p);
    for (uint32_t spins = 0; v.x == kHandoffSentinel || v.y == kHandoffSentinel || v.z == kHandoffSentinel ||
                             v.w == kHandoffSentinel;
         ++spins) {
      if (spins > (1u << 26)) __trap();
      v = ld_volatile_v4(p);
    }
    reinterpret_cast<uint4 *>(dst)[i] = v;
    *p = s4;  // drained: re-arm in place
  }
  for (size_t i = nv * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += stride) {
    uint32_t v = ld_volatile_u32(buf + i);
    for (uint32_t spins = 0; v == kHandoffSentinel; ++spins) {
      if (spins > (1u << 26)) __trap();
      v = ld_volatile_u32(buf + i);
    }
    dst[i] = v;
    buf[i] = kHandoffSentinel;
  }
  // every CTA's re-arm stores are visible before the last CTA hands the buffer back
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const int done = atomicAdd(state + 1, 1);
    if (done == (int)gridDim.x - 1) {
      state[1] = 0;
      *(volatile int *)state = call + 1;
      __threadfence_system();
      st_release_sys_s32(credit_word(inbox, max_words), call + 1);
    }
  }
}

__global__ void handoff_fill_kernel(uint32_t *p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = kHandoffSentinel;
}

static int handoff_grid(size_t words) {
  const size_t per = 256 * 4 * 2;  // ~2 uint4 per thread
  size_t g = (words + per - 1) / per;
  return (int)(g < 1 ? 1 : (g > 148 ? 148 : g));
}

}  // namespace hx

using namespace hx;

// 3 buffers of max_words words, then the credit word of the flow-controlled (prefill) protocol
extern "C" size_t hx_handoff_inbox_bytes(size_t max_words) { return 3 * max_words * sizeof(uint32_t) + 128; }

extern "C" int hx_handoff_inbox_init(void *inbox, size_t max_words, hx_stream_t stream) {
  if (!inbox || !max_words || max_words % 4) return HX_ERR_ARG;
  cudaMemsetAsync(credit_word((uint32_t *)inbox, max_words), 0, 128, as_stream(stream));
  // Load both ends of the protocol now: under CUDA lazy loading the first launch
  // of a kernel loads its module, which cannot complete while a spinning pull
  // occupies the device -- a pull launched before the push's first-ever launch in
  // the same context (single-GPU emulation) would then never see its data.
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, handoff_push_kernel);
  cudaFuncGetAttributes(&fa, handoff_pull_kernel);
  cudaFuncGetAttributes(&fa, handoff_push_credit_kernel);
  cudaFuncGetAttributes(&fa, handoff_pull_credit_kernel);
  handoff_fill_kernel<<<148, 256, 0, as_stream(stream)>>>((uint32_t *)inbox, 3 * max_words);
  return launch_status();
}

extern "C" int hx_handoff_push(const void *src, void *const *dst_inboxes, int n_dst, size_t words, size_t max_words,
                               int *state, hx_stream_t stream) {
  if (!src || !dst_inboxes || n_dst < 1 || n_dst > kMaxDst || !state || max_words % 4 || words > max_words ||
      (uintptr_t)src % 16)
    return HX_ERR_ARG;
  if (words == 0) return 0;
  HandoffDsts d{};
  for (int k = 0; k < n_dst; ++k) d.box[k] = (uint32_t *)dst_inboxes[k];
  return launch(handoff_push_kernel, dim3(handoff_grid(words)), dim3(256), 0, as_stream(stream),
                (const uint32_t *)src, d, n_dst, words, max_words, state);
}

extern "C" int hx_handoff_pull(void *dst, void *inbox, size_t words, size_t max_words, int *state,
                               hx_stream_t stream) {
  if (!dst || !inbox || !state || max_words % 4 || words > max_words || (uintptr_t)dst % 16) return HX_ERR_ARG;
  if (words == 0) return 0;
  return launch(handoff_pull_kernel, dim3(handoff_grid(max_words)), dim3(256), 0, as_stream(stream),
                (uint32_t *)dst, (uint32_t *)inbox, words, max_words, state);
}

extern "C" int hx_handoff_push_credit(const void *src, void *dst_inbox, size_t words, size_t max_words, int *state,
                                      hx_stream_t stream) {
  if (!src || !dst_inbox || !state || max_words % 4 || words > max_words || (uintptr_t)src % 16) return HX_ERR_ARG;
  if (words == 0) return 0;
  return launch(handoff_push_credit_kernel, dim3(handoff_grid(words)), dim3(256), 0, as_stream(stream),
                (const uint32_t *)src, (uint32_t *)dst_inbox, words, max_words, state);
}

extern "C" int hx_handoff_pull_credit(void *dst, void *inbox, size_t words, size_t max_words, int *state,
                                      hx_stream_t stream) {
  if (!dst || !inbox || !state || max_words % 4 || words > max_words || (uintptr_t)dst % 16) return HX_ERR_ARG;
  if (words == 0) return 0;
  return launch(handoff_pull_credit_kernel, dim3(handoff_grid(words)), dim3(256), 0, as_stream(stream),
                (uint32_t *)dst, (uint32_t *)inbox, words, max_words, state);
}
