// common.cuh -- shared device helpers for the Binar Sort sm_100a kernels.
//
// Key model (reference semantics, keys.py:35-93, kernels.py:63,69):
//   * a word x of W bits carries its sort key in the low `width` bits, read
//     MSB-first from bit width-1 (UnsignedCodec), after the codec transform
//     (SignedCodec: flip the sign bit; Float64Codec: IEEE total order);
//   * the GPU works on the *normalised encoded key* nk = enc(x) << (W-width),
//     so digit j (0 = most significant) is (nk >> (W-8-8j)) & 0xFF.  A
//     digit pass over 8 bits computes exactly the buckets that 8 levels of
//     the reference's binary recursion compute (SURVEY §7 design sketch).
//   * the data moved is always the raw word x: no transform passes.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bs {

constexpr int WARP = 32;

// Debug build (-DBS_DEBUG_CHECKS, libbinarsort_b200_debug.so): every global
// and staging write of the sort kernels checks its index; a violation sets bit
// 3 of the sort's status word (bs_sort_status) instead of trapping, so the
// test suite can run the whole parity corpus against the checked build.
#ifdef BS_DEBUG_CHECKS
#define BS_DCHECK(ctl, cond)                                   \
  do {                                                         \
    if (!(cond)) atomicOr(&(ctl)->error, 8u);                  \
  } while (0)
#else
#define BS_DCHECK(ctl, cond) \
  do {                       \
  } while (0)
#endif

template <int VB> struct ValT { using T = uint32_t; };
template <> struct ValT<8> { using T = uint64_t; };

__host__ __device__ __forceinline__ uint64_t min64(uint64_t a, uint64_t b) { return a < b ? a : b; }

template <typename K> struct KeyTraits;
template <> struct KeyTraits<uint32_t> {
  static constexpr int BITS = 32;
  __device__ __forceinline__ static int clz(uint32_t x) { return __clz(x); }
};
template <> struct KeyTraits<uint64_t> {
  static constexpr int BITS = 64;
  __device__ __forceinline__ static int clz(uint64_t x) { return __clzll(x); }
};

// Codec transform, keys.py:51-93.  KIND 0 unsigned, 1 signed, 2 float.
template <typename K, int KIND>
__device__ __forceinline__ K encode(K x) {
  constexpr int W = KeyTraits<K>::BITS;
  constexpr K MSB = K(1) << (W - 1);
  if constexpr (KIND == 0) {
    return x;
  } else if constexpr (KIND == 1) {
    return x ^ MSB;
  } else {
    K m = K(0) - (x >> (W - 1));  // all ones iff sign bit set
    return x ^ (m | MSB);
  }
}

// Per-launch view of the key geometry.
template <typename K, int KIND>
struct KeyGeom {
  int shift0;  // W - width_eff
  // SignedCodec(width) flips bit width-1 of the low-width word (keys.py:51-58):
  // after the shift that is the word's top bit, so any width works.
  __device__ __forceinline__ K norm(K x) const {
    constexpr K MSB = K(1) << (KeyTraits<K>::BITS - 1);
    if constexpr (KIND == 0) return x << shift0;
    else if constexpr (KIND == 1) return (x << shift0) ^ MSB;
    else return encode<K, KIND>(x) << shift0;
  }
  __device__ __forceinline__ static uint32_t digit_of_norm(K nk, int dig) {
    constexpr int W = KeyTraits<K>::BITS;
    return uint32_t(nk >> (W - 8 - 8 * dig)) & 0xFFu;
  }
  __device__ __forceinline__ uint32_t digit(K x, int dig) const {
    return digit_of_norm(norm(x), dig);
  }
};

// Digit `dig` of a raw word, precomputed shifts: ((enc(x) << l) >> r) & 0xFF,
// with the signed codec's sign flip folded into digit 0.
template <typename K, int KIND>
struct DigitFn {
  int l, r;
  uint32_t flip;
  __device__ __forceinline__ DigitFn(int shift0, int dig)
      : l(shift0), r(KeyTraits<K>::BITS - 8 - 8 * dig), flip((KIND == 1 && dig == 0) ? 0x80u : 0u) {}
  __device__ __forceinline__ uint32_t operator()(K x) const {
    const K e = (KIND == 2) ? encode<K, 2>(x) : x;
    return (uint32_t((e << l) >> r) & 0xFFu) ^ flip;
  }
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// atomicOr on shared memory issued under a predicate (no branch around it);
// returns the old word, or 0 when `on` is false
__device__ __forceinline__ uint32_t atom_or_shared_if(uint32_t *p, uint32_t v, bool on) {
  uint32_t old = 0;
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q atom.shared.or.b32 %0, [%1], %2;\n\t}"
      : "+r"(old)
      : "r"(a), "r"(v), "r"(uint32_t(on))
      : "memory");
  return old;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Peers of this lane among the lanes in `active` that hold the same 8-bit
// digit: 8 warp ballots, one per bit plane (the north_star's ballot/popc
// ranking).  Result includes the lane itself when it is active.
__device__ __forceinline__ uint32_t match_digit8(uint32_t d, uint32_t active) {
  uint32_t peers = active;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t bb = __ballot_sync(0xFFFFFFFFu, bit);
    peers &= bit ? bb : ~bb;
  }
  return peers;
}

// Stable warp-level ranking of KPT elements per lane by 8-bit digit.
// Element layout: chunk j / lane l  <->  warp-local index 32*j + l.
// whist: this warp's 256 counters in shared memory, zero on entry; on exit
// whist[d] = number of this warp's valid elements with digit d.
// rank[j] = stable rank of element (j, lane) among this warp's elements of
// the same digit.  `nvalid` = number of valid warp-local elements (prefix).
template <int KPT>
__device__ __forceinline__ void warp_rank(const uint32_t (&dig)[KPT], int nvalid,
                                          uint32_t *whist, uint32_t (&rank)[KPT]) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const int idx = 32 * j + lane;
    const bool valid = idx < nvalid;
    if (32 * j >= nvalid) {  // warp-uniform: nothing left
      rank[j] = 0;
      continue;
    }
    const uint32_t active = __ballot_sync(0xFFFFFFFFu, valid);
    const uint32_t d = dig[j];
    const uint32_t peers = match_digit8(d, active);
    const uint32_t below = __popc(peers & lt);
    uint32_t old = 0;
    if (valid && below == 0) {
      old = whist[d];
      whist[d] = old + __popc(peers);
    }
    const int leader = __ffs(peers) - 1;
    old = __shfl_sync(0xFFFFFFFFu, old, valid ? leader : lane);
    rank[j] = old + below;
    __syncwarp();
  }
}

// Block-wide exclusive scan of one value per thread for the first 256 threads
// (digit counts).  `scratch` needs 256/32 + 1 words.  Returns the exclusive
// prefix; *total (optional) gets the sum.  All BLOCK threads must call.
template <int BLOCK>
__device__ __forceinline__ uint32_t scan256_excl(uint32_t v, uint32_t *scratch) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t x = (tid < 256) ? v : 0u;
  uint32_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (tid < 256 && lane == 31) scratch[w] = incl;
  __syncthreads();
  if (tid < 32) {
    uint32_t s = (lane < 8) ? scratch[lane] : 0u;
    uint32_t si = s;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xFFFFFFFFu, si, o);
      if (lane >= o) si += y;
    }
    if (lane < 8) scratch[lane] = si - s;
  }
  __syncthreads();
  uint32_t r = (tid < 256) ? scratch[w] + incl - x : 0u;
  __syncthreads();
  return r;
}

template <typename T>
__device__ __forceinline__ T warp_or(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_and(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v &= __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

}  // namespace bs

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) global -> shared, completed on
// an mbarrier.  Used to double-buffer tiles/tasks so the next one streams in
// while the current one is ranked and scattered.
// ---------------------------------------------------------------------------
namespace bs {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order earlier generic-proxy accesses of shared memory before async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// barrier among the first NT threads of the CTA (id 1; id 0 is __syncthreads)
template <int NT>
__device__ __forceinline__ void named_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Programmatic dependent launch: a kernel launched with the programmatic
// stream-serialisation attribute may start while the previous kernel in the
// stream drains; it must wait here before touching anything that kernel
// produces or reads.  A no-op for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Bulk shared -> global store (async proxy), tracked by the issuing thread's
// bulk async-groups.  Addresses 16-byte aligned, size a multiple of 16.
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the issuing thread's stores have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// ... and have completed (writes performed)
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Producer-side wait: back off between polls so a spinning producer lane does
// not steal issue slots from the consumer warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
  // try_wait with a suspend-time hint: the waiting thread is descheduled
  // until the phase completes (or ~1 ms passes) instead of polling
  asm volatile(
      "{\n .reg .pred p;\n WAITS_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      " @!p bra WAITS_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Span of elements [0, cnt) of `src` widened to the enclosing 16-byte aligned
// granules (an over-read that stays inside granules holding valid elements,
// so it never crosses a page).  `head` = element offset of src[0] in it.
struct Span {
  const void *base;
  uint32_t bytes;
  uint32_t head;
};
template <typename T>
__device__ __forceinline__ Span span16(const T *src, uint32_t cnt) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  const uintptr_t a0 = a & ~uintptr_t(15);
  const uintptr_t a1 = (a + uintptr_t(cnt) * sizeof(T) + 15) & ~uintptr_t(15);
  return Span{reinterpret_cast<const void *>(a0), uint32_t(a1 - a0), uint32_t((a - a0) / sizeof(T))};
}

}  // namespace bs
