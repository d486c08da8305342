// metrics_impl.cuh -- K6: the reference's Metrics as a closed form over the
// sorted output, one coalesced read of the keys.
//
// For the baseline recursive sort (kernels.sort_words, kernels.py:88-126)
// started at `depth0` on n >= 2 keys of effective width w, with sorted
// normalised keys s_i and lcp_i = min(w, clz(s_i ^ s_{i+1})):
//   L_i        = min(w, 1 + max(lcp_{i-1}, lcp_i))      (missing -> -1)
//   extractions = sum L_i                (bits examined per element)
//   swaps       = sum popcount(top L_i bits of s_i)   (each bit-1 element is
//                 swapped once per partition that examines it, kernels.py:70-74)
//   calls       = 1 + sum max(0, min(lcp_i, w-1) - lcp_{i-1}) + #{lcp_i < w}
//                 (internal trie nodes + branch nodes)
//   max_depth   = depth0 + max L_i
#pragma once

#include "common.cuh"

namespace bs {

template <typename K, int KIND, int BLOCK, int IPT>
__global__ void __launch_bounds__(BLOCK) metrics_kernel(const K *__restrict__ keys, uint64_t n,
                                                        int shift0, int w, int64_t depth0,
                                                        unsigned long long *counters) {
  constexpr int W = KeyTraits<K>::BITS;
  const KeyGeom<K, KIND> g{shift0};
  __shared__ unsigned long long s_red[4][BLOCK / 32];
  unsigned long long ext = 0, sw = 0, calls = 0, lmax = 0;
  const uint64_t chunk = uint64_t(BLOCK) * IPT;
  for (uint64_t base = uint64_t(blockIdx.x) * chunk; base < n; base += uint64_t(gridDim.x) * chunk) {
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const uint64_t i = base + uint64_t(j) * BLOCK + threadIdx.x;
      if (i >= n) break;
      const K si = g.norm(keys[i]);
      int lp = -1, lc = -1;  // lcp_{i-1}, lcp_i
      if (i > 0) {
        const K x = g.norm(keys[i - 1]) ^ si;
        lp = x ? min(w, KeyTraits<K>::clz(x)) : w;
      }
      if (i + 1 < n) {
        const K x = si ^ g.norm(keys[i + 1]);
        lc = x ? min(w, KeyTraits<K>::clz(x)) : w;
      }
      const int Li = min(w, 1 + max(lp, lc));
      ext += Li;
      sw += (Li > 0) ? __popcll((unsigned long long)(uint64_t(si) >> (W - Li))) : 0;
      if (i + 1 < n) {
        calls += max(0, min(lc, w - 1) - lp);
        calls += (lc < w) ? 1 : 0;
      }
      lmax = max(lmax, (unsigned long long)Li);
    }
  }
  // block reduce
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ext += __shfl_xor_sync(0xFFFFFFFFu, ext, o);
    sw += __shfl_xor_sync(0xFFFFFFFFu, sw, o);
    calls += __shfl_xor_sync(0xFFFFFFFFu, calls, o);
    lmax = max(lmax, __shfl_xor_sync(0xFFFFFFFFu, lmax, o));
  }
  if (lane == 0) {
    s_red[0][wid] = ext;
    s_red[1][wid] = sw;
    s_red[2][wid] = calls;
    s_red[3][wid] = lmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0, b = 0, c = 0, m = 0;
    for (int i = 0; i < BLOCK / 32; ++i) {
      a += s_red[0][i];
      b += s_red[1][i];
      c += s_red[2][i];
      m = max(m, s_red[3][i]);
    }
    atomicAdd(&counters[0], a);
    atomicAdd(&counters[1], b);
    atomicAdd(&counters[2], c);
    atomicMax(&counters[3], m + (unsigned long long)depth0);
  }
}

// the "+1" of the calls formula (the root call) is added once by this kernel
__global__ void metrics_root_kernel(unsigned long long *counters) { atomicAdd(&counters[2], 1ull); }

}  // namespace bs
