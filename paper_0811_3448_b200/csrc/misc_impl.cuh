// misc_impl.cuh -- the smaller kernels of the C ABI:
//   * exact reference partition pass (kernels.partition_words, kernels.py:56-77)
//     through its closed form;
//   * range_sorted_words (kernels.py:80-85);
//   * multi-GPU front-end device steps: strided key sampling and a stable
//     partition into 2R-1 splitter classes (replaces variants._prepartition,
//     variants.py:124-148, as the step before the NCCL all-to-all-v).
#pragma once

#include "common.cuh"

namespace bs {

// ---------------------------------------------------------------------------
// Simple device scan of per-block counts (reduce-then-scan, one CTA).
// ---------------------------------------------------------------------------
__global__ void scan_blocks_kernel(uint32_t *counts, uint32_t nblocks, uint32_t *total) {
  // exclusive scan in place, single CTA of 1024 threads
  __shared__ uint32_t s[1024];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < nblocks; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = (i < nblocks) ? counts[i] : 0u;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      uint32_t t = (int(threadIdx.x) >= o) ? s[threadIdx.x - o] : 0u;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nblocks) counts[i] = carry + s[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += s[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

// ---------------------------------------------------------------------------
// Exact partition pass.  With b_i the bit of element i at `pos` and Z the
// number of zeros (split = Z):
//  * zero region i < Z: keeps e_i if b_i == 0; the k-th L-one (bit-1 element
//    at a position < Z) is replaced by the k-th R-zero (bit-0 element at a
//    position >= Z, counted from the right end);
//  * one region: offset n-1 gets L-one #0; offset q-1 (Z < q <= n-1) gets e_q
//    if b_q == 1, else L-one #(1 + #zeros in (q, n)).
// swaps = n - Z (every bit-1 element is swapped exactly once), extractions = n.
// ---------------------------------------------------------------------------
constexpr int PART_BLOCK = 256;
constexpr int PART_IPT = 16;
constexpr int PART_CHUNK = PART_BLOCK * PART_IPT;

template <typename K>
__device__ __forceinline__ uint32_t bit_at(K x, int pos, int width) {
  // (u64(x) << pos) & (1 << (width-1)), kernels.py:63,69
  const uint64_t msb = uint64_t(1) << (width - 1);
  return ((uint64_t(x) << pos) & msb) ? 1u : 0u;
}

template <typename K>
__global__ void part_count_kernel(const K *keys, uint64_t n, int pos, int width, uint32_t *bcount) {
  __shared__ uint32_t s[PART_BLOCK / 32];
  const uint64_t base = uint64_t(blockIdx.x) * PART_CHUNK;
  uint32_t c = 0;
  for (int j = 0; j < PART_IPT; ++j) {
    const uint64_t i = base + uint64_t(j) * PART_BLOCK + threadIdx.x;
    if (i < n) c += bit_at(keys[i], pos, width) ^ 1u;  // zeros
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < PART_BLOCK / 32; ++i) t += s[i];
    bcount[blockIdx.x] = t;
  }
}

// exclusive zero-prefix per element, computed per chunk sequentially per
// thread-block (chunk order = element order): block-level scan of zeros.
template <typename K>
__device__ __forceinline__ void chunk_zero_prefix(const K *keys, uint64_t n, int pos, int width,
                                                  uint32_t block_excl, uint32_t (&zp)[PART_IPT],
                                                  uint32_t (&bit)[PART_IPT], uint32_t *s_warp) {
  // thread t owns elements base + t*IPT + j (blocked, contiguous per thread)
  const uint64_t base = uint64_t(blockIdx.x) * PART_CHUNK + uint64_t(threadIdx.x) * PART_IPT;
  uint32_t run = 0;
  for (int j = 0; j < PART_IPT; ++j) {
    const uint64_t i = base + j;
    bit[j] = (i < n) ? bit_at(keys[i], pos, width) : 1u;
    zp[j] = run;
    run += (i < n) ? (bit[j] ^ 1u) : 0u;
  }
  // block exclusive scan of `run`
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = run;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int i = 0; i < PART_BLOCK / 32; ++i) {
      uint32_t t = s_warp[i];
      s_warp[i] = acc;
      acc += t;
    }
  }
  __syncthreads();
  const uint32_t texcl = block_excl + s_warp[w] + incl - run;
  for (int j = 0; j < PART_IPT; ++j) zp[j] += texcl;
}

// zp = #zeros in [0, i).  For i < Z: #ones in [0,i) = i - zp.  For i >= Z:
// #zeros in (i, n) = Z - zp - (b_i==0).
template <typename K>
__global__ void part_index_kernel(const K *keys, uint64_t n, int pos, int width,
                                  const uint32_t *bexcl, const uint32_t *Zp, uint32_t *lone,
                                  uint32_t *zpos) {
  __shared__ uint32_t s_warp[PART_BLOCK / 32];
  uint32_t zp[PART_IPT], bit[PART_IPT];
  chunk_zero_prefix(keys, n, pos, width, bexcl[blockIdx.x], zp, bit, s_warp);
  const uint32_t Z = *Zp;
  const uint64_t base = uint64_t(blockIdx.x) * PART_CHUNK + uint64_t(threadIdx.x) * PART_IPT;
  for (int j = 0; j < PART_IPT; ++j) {
    const uint64_t i = base + j;
    if (i >= n) break;
    // L-ones: bit-1 elements the low cursor examines fresh, i.e. positions
    // [0, Z] (position Z only when it holds a one); rank = #ones before.
    if (i <= Z && bit[j]) lone[uint32_t(i) - zp[j]] = uint32_t(i);
    // R-zeros: bit-0 elements at positions >= Z, ranked from the right end.
    if (i >= Z && !bit[j]) zpos[Z - zp[j] - 1u] = uint32_t(i);
  }
}

template <typename K, int VB>
__global__ void part_gather_kernel(const K *src, K *dst, const void *vsrc_, void *vdst_, uint64_t n,
                                   int pos, int width, const uint32_t *bexcl, const uint32_t *Zp,
                                   const uint32_t *lone, const uint32_t *zpos) {
  using V = typename ValT<VB>::T;
  const V *vsrc = static_cast<const V *>(vsrc_);
  V *vdst = static_cast<V *>(vdst_);
  auto mv = [&](uint64_t to, uint64_t from) {
    dst[to] = src[from];
    if constexpr (VB != 0) vdst[to] = vsrc[from];
  };
  __shared__ uint32_t s_warp[PART_BLOCK / 32];
  uint32_t zp[PART_IPT], bit[PART_IPT];
  chunk_zero_prefix(src, n, pos, width, bexcl[blockIdx.x], zp, bit, s_warp);
  const uint32_t Z = *Zp;
  const uint64_t base = uint64_t(blockIdx.x) * PART_CHUNK + uint64_t(threadIdx.x) * PART_IPT;
  for (int j = 0; j < PART_IPT; ++j) {
    const uint64_t i = base + j;
    if (i >= n) break;
    if (i < Z) {
      mv(i, bit[j] ? uint64_t(zpos[uint32_t(i) - zp[j]]) : i);
    } else {
      // element i is q for target offset q-1 (q > Z); offset n-1 handled below
      if (i > Z) {
        const uint32_t zeros_after = Z - zp[j] - (bit[j] ^ 1u);
        mv(i - 1, bit[j] ? i : uint64_t(lone[1u + zeros_after]));
      }
      if (i == n - 1) mv(n - 1, lone[0]);
    }
  }
}

__global__ void part_finish_kernel(const uint32_t *Zp, uint64_t n, int64_t *split,
                                   unsigned long long *counters) {
  const uint32_t Z = *Zp;
  if (split) *split = int64_t(Z);
  if (counters) {
    atomicAdd(&counters[0], (unsigned long long)n);
    atomicAdd(&counters[1], (unsigned long long)(n - Z));
  }
}

// ---------------------------------------------------------------------------
// range_sorted_words: flag stays 1 unless some adjacent pair is decreasing.
// ---------------------------------------------------------------------------
template <typename K>
__global__ void range_sorted_kernel(const K *keys, uint64_t n, int32_t *flag) {
  bool ok = true;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i + 1 < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    ok &= !(keys[i] > keys[i + 1]);
  if (!__all_sync(0xFFFFFFFFu, ok) && (threadIdx.x & 31) == 0) *flag = 0;
}

// ---------------------------------------------------------------------------
// Multi-GPU helpers.
// ---------------------------------------------------------------------------
template <typename K, int KIND>
__global__ void sample_kernel(const K *keys, uint64_t n, int shift0, uint64_t count, K *out) {
  const KeyGeom<K, KIND> g{shift0};
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t idx = ((2 * i + 1) * n) / (2 * count);
    out[i] = g.norm(keys[idx]);
  }
}

// class of a normalised key against R-1 sorted normalised splitters:
// 2*#{s_j < key} + [key equals some s_j].  Class 2j holds keys strictly
// between s_{j-1} and s_j, class 2j+1 keys equal to s_j; with duplicate
// splitters a tied key takes the class of the first equal splitter.
template <typename K>
__device__ __forceinline__ uint32_t split_class(K nk, const K *spl, int nsp) {
  uint32_t lt = 0, eq = 0;
  for (int j = 0; j < nsp; ++j) {
    const K s = spl[j];
    lt += (s < nk) ? 1u : 0u;
    eq |= (s == nk) ? 1u : 0u;
  }
  return 2u * lt + eq;
}

constexpr int SPLIT_BLOCK = 256;
constexpr int SPLIT_KPT = 16;
constexpr int SPLIT_TILE = SPLIT_BLOCK * SPLIT_KPT;

// R <= 8 ranks: at most 7 splitters, held in registers (no shared loads per key)
constexpr int SPLIT_MAXSP = 7;
constexpr int SPLIT_HIST_TPB = 4;  // tiles per split_hist_kernel CTA

// Class of a normalised key against the (<= 7, sorted) splitters held in
// shared memory padded to 8 with the maximum word: branchless lower bound
// (3 probes) for #{s_j < key}, then one probe for "equals a splitter".
// Same classes as split_class().
template <typename K>
struct SplitClass {
  const K *s;  // shared, 8 entries
  int nsp;
  __device__ __forceinline__ uint32_t cls(K nk) const {
    uint32_t lt = 0;
#pragma unroll
    for (uint32_t step = 4; step > 0; step >>= 1)
      if (s[lt + step - 1] < nk) lt += step;
    const uint32_t eq = (int(lt) < nsp && s[lt] == nk) ? 1u : 0u;
    return 2u * lt + eq;
  }
};

template <typename K>
__device__ __forceinline__ void load_splitters(K *s_spl, const K *spl, int nsp) {
  if (threadIdx.x < SPLIT_MAXSP + 1) s_spl[threadIdx.x] = int(threadIdx.x) < nsp ? spl[threadIdx.x] : ~K(0);
}

// Fast path: a 256-entry table on the key's top byte.  Entry t holds the
// class of every key whose top byte is t when no splitter lies in that byte
// range (all but <= 7 entries), else 0xFF (take the binary search).
template <typename K>
struct SplitLUT {
  const uint8_t *tab;  // shared, 256 entries
  SplitClass<K> sc;
  __device__ __forceinline__ uint32_t cls(K nk) const {
    constexpr int W = int(sizeof(K)) * 8;
    const uint32_t c = tab[uint32_t(nk >> (W - 8))];
    return c != 0xFFu ? c : sc.cls(nk);
  }
};

// build the table (call with >= 256 threads after the splitters are in shared memory + a barrier)
template <typename K>
__device__ __forceinline__ void build_split_lut(uint8_t *tab, const SplitClass<K> &sc) {
  constexpr int W = int(sizeof(K)) * 8;
  const uint32_t t = threadIdx.x;
  if (t < 256) {
    const K lo = K(t) << (W - 8), hi = lo | (~K(0) >> 8);
    const uint32_t a = sc.cls(lo), b = sc.cls(hi);
    tab[t] = (a == b && (a & 1u) == 0u) ? uint8_t(a) : uint8_t(0xFF);
  }
}

// Per-tile class counts.  Each thread counts its 16 keys in packed 8-bit
// fields (classes 0-7 / 8-15 in two 64-bit words), the warp sums 16-bit
// fields with shuffles, and one shared atomic per class and warp folds the
// warps: no same-address shared atomics per key (16 classes would serialise).
template <typename K, int KIND>
__global__ void __launch_bounds__(SPLIT_BLOCK) split_hist_kernel(const K *keys, uint64_t n, int shift0,
                                                                 const K *spl, int nsp,
                                                                 uint32_t *tile_hist /* [ntiles][16] */) {
  const KeyGeom<K, KIND> g{shift0};
  __shared__ uint32_t h[16];
  __shared__ K s_spl[SPLIT_MAXSP + 1];
  __shared__ uint8_t s_tab[256];
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 16) h[tid] = 0;
  load_splitters(s_spl, spl, nsp);
  const SplitClass<K> sc{s_spl, nsp};
  __syncthreads();
  build_split_lut(s_tab, sc);
  const SplitLUT<K> sr{s_tab, sc};
  __syncthreads();
  // SPLIT_HIST_TPB consecutive tiles per CTA (the table build is amortised)
  const uint64_t ntiles = (n + SPLIT_TILE - 1) / SPLIT_TILE;
  for (uint64_t t = uint64_t(blockIdx.x) * SPLIT_HIST_TPB;
       t < min64(ntiles, uint64_t(blockIdx.x + 1) * SPLIT_HIST_TPB); ++t) {
    const uint64_t base = t * SPLIT_TILE;
    const int cnt = int(min64(SPLIT_TILE, n - base));
    // all loads first (no per-key branch between them), then classify
    K x[SPLIT_KPT];
#pragma unroll
    for (int j = 0; j < SPLIT_KPT; ++j) {
      const int e = j * SPLIT_BLOCK + tid;
      x[j] = e < cnt ? keys[base + e] : K(0);
    }
    uint64_t lo = 0, hi = 0;
#pragma unroll
    for (int j = 0; j < SPLIT_KPT; ++j) {
      const uint32_t c = sr.cls(g.norm(x[j]));
      const uint64_t inc = (j * SPLIT_BLOCK + tid < cnt) ? (1ull << (8 * (c & 7u))) : 0ull;
      if (c < 8u) lo += inc;
      else hi += inc;
    }
    // widen to 16-bit fields (a warp holds up to 32*16 = 512 per class)
    uint64_t f[4] = {lo & 0x00FF00FF00FF00FFull, (lo >> 8) & 0x00FF00FF00FF00FFull, hi & 0x00FF00FF00FF00FFull,
                     (hi >> 8) & 0x00FF00FF00FF00FFull};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) f[q] += __shfl_xor_sync(0xFFFFFFFFu, f[q], o);
    if (lane < 16) {  // lane c reports class c
      // f[0]: classes 0,2,4,6  f[1]: 1,3,5,7  f[2]: 8,10,12,14  f[3]: 9,11,13,15
      const int c = lane;
      const uint64_t word = (c >> 3) ? ((c & 1) ? f[3] : f[2]) : ((c & 1) ? f[1] : f[0]);
      const uint32_t v = uint32_t(word >> (16 * ((c & 7) >> 1))) & 0xFFFFu;
      if (v) atomicAdd(&h[c], v);
    }
    __syncthreads();
    if (tid < 16) {
      tile_hist[size_t(t) * 16 + tid] = h[tid];
      h[tid] = 0;
    }
    __syncthreads();
  }
}

template <typename K, int VB, int KIND>
__global__ void __launch_bounds__(SPLIT_BLOCK) split_scatter_kernel(
    const K *keys, const void *vals_, uint64_t n, int shift0, const K *spl, int nsp,
    const uint32_t *tile_off, K *out_keys, void *out_vals_) {
  using V = typename ValT<VB>::T;
  const V *vals = static_cast<const V *>(vals_);
  V *out_vals = static_cast<V *>(out_vals_);
  constexpr int NW = SPLIT_BLOCK / 32;
  const KeyGeom<K, KIND> g{shift0};
  __shared__ uint32_t whist_all[NW * 256];
  __shared__ uint32_t tstart[256];
  __shared__ K s_spl[16];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid < nsp) s_spl[tid] = spl[tid];
  uint32_t *whist = whist_all + w * 256;
  for (int i = lane; i < 256; i += 32) whist[i] = 0;
  __syncthreads();
  const uint64_t base = uint64_t(blockIdx.x) * SPLIT_TILE;
  const int cnt = int(min64(SPLIT_TILE, n - base));
  const int wbase = w * 32 * SPLIT_KPT;
  const int nvw = max(0, min(32 * SPLIT_KPT, cnt - wbase));
  K x[SPLIT_KPT];
  V v[SPLIT_KPT];
  uint32_t dg[SPLIT_KPT], rk[SPLIT_KPT];
#pragma unroll
  for (int j = 0; j < SPLIT_KPT; ++j) {
    const int e = wbase + 32 * j + lane;
    x[j] = 0;
    dg[j] = 0;
    if (e < cnt) {
      x[j] = keys[base + e];
      if constexpr (VB != 0) v[j] = vals[base + e];
      dg[j] = split_class(g.norm(x[j]), s_spl, nsp);
    }
  }
  warp_rank<SPLIT_KPT>(dg, nvw, whist, rk);
  __syncthreads();
  uint32_t total = 0;
  if (tid < 256) {
    uint32_t s = 0;
    for (int ww = 0; ww < NW; ++ww) {
      const uint32_t cc = whist_all[ww * 256 + tid];
      whist_all[ww * 256 + tid] = s;
      s += cc;
    }
    total = s;
  }
  (void)total;
  __syncthreads();
  if (tid < 16) tstart[tid] = tile_off[size_t(blockIdx.x) * 16 + tid];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < SPLIT_KPT; ++j) {
    const int e = wbase + 32 * j + lane;
    if (e < cnt) {
      const uint32_t d = dg[j];
      const uint64_t o = uint64_t(tstart[d]) + whist[d] + rk[j];
      out_keys[o] = x[j];
      if constexpr (VB != 0) out_vals[o] = v[j];
    }
  }
}

// ---------------------------------------------------------------------------
// Parallel class-major scan of the per-tile class counts (replaces a serial
// one-warp walk over all tiles): chunk sums -> one CTA scans the chunk sums
// per class -> every chunk scans its own tiles.  tile_hist[t][c] becomes the
// shard-local position of tile t's first class-c element in the class-major
// order (class bases included).
// ---------------------------------------------------------------------------
constexpr int SCAN_TPT = 4;                      // tiles per thread
constexpr int SCAN_CHUNK = SCAN_TPT * 256;       // tiles per chunk (256-thread CTAs)

__device__ __forceinline__ void load_row16(const uint32_t *row, uint32_t (&c)[16]) {
  const uint4 *r = reinterpret_cast<const uint4 *>(row);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 v = r[q];
    c[4 * q] = v.x, c[4 * q + 1] = v.y, c[4 * q + 2] = v.z, c[4 * q + 3] = v.w;
  }
}

__global__ void __launch_bounds__(256) split_chunk_sum_kernel(const uint32_t *tile_hist, uint32_t ntiles,
                                                              uint32_t *chunk_sum /* [nchunks][16] */) {
  __shared__ uint32_t s[8][16];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = 0;
  const uint32_t t0 = blockIdx.x * SCAN_CHUNK + uint32_t(tid) * SCAN_TPT;
#pragma unroll
  for (int k = 0; k < SCAN_TPT; ++k) {
    if (t0 + k < ntiles) {
      uint32_t c[16];
      load_row16(tile_hist + size_t(t0 + k) * 16, c);
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] += c[q];
    }
  }
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    uint32_t v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) s[w][c] = v;
  }
  __syncthreads();
  if (tid < 16) {
    uint32_t v = 0;
    for (int i = 0; i < 8; ++i) v += s[i][tid];
    chunk_sum[size_t(blockIdx.x) * 16 + tid] = v;
  }
}

// one CTA of 16 warps: warp c scans class c over the chunks (in place ->
// exclusive in-class chunk bases); then class bases (class-major) and totals
__global__ void __launch_bounds__(512) split_top_scan_kernel(uint32_t *chunk_sum, uint32_t nchunks, int ncls,
                                                             unsigned long long *class_counts,
                                                             uint32_t *class_base /* [16] */) {
  __shared__ uint32_t tot[16];
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  uint32_t run = 0;
  for (uint32_t i0 = 0; i0 < nchunks; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t v = i < nchunks ? chunk_sum[size_t(i) * 16 + c] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    if (i < nchunks) chunk_sum[size_t(i) * 16 + c] = run + incl - v;
    run += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
  if (lane == 0) tot[c] = run;
  __syncthreads();
  if (threadIdx.x == 0) {
    class_base[32] = 0u;  // split_exchange_kernel's completion ticket
    uint32_t b = 0;
    for (int k = 0; k < 16; ++k) {
      class_base[k] = b;
      if (k < ncls) class_counts[k] = tot[k];
      b += tot[k];
    }
  }
}

__global__ void __launch_bounds__(256) split_chunk_scan_kernel(uint32_t *tile_hist, uint32_t ntiles,
                                                               const uint32_t *chunk_sum,
                                                               const uint32_t *class_base) {
  __shared__ uint32_t s[8][16];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t t0 = blockIdx.x * SCAN_CHUNK + uint32_t(tid) * SCAN_TPT;
  uint32_t acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = 0;
#pragma unroll
  for (int k = 0; k < SCAN_TPT; ++k) {
    if (t0 + k < ntiles) {
      uint32_t c[16];
      load_row16(tile_hist + size_t(t0 + k) * 16, c);
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] += c[q];
    }
  }
  uint32_t ex[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    uint32_t incl = acc[c];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    ex[c] = incl - acc[c];
    if (lane == 31) s[w][c] = incl;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    uint32_t b = class_base[c] + chunk_sum[size_t(blockIdx.x) * 16 + c];
    for (int i = 0; i < w; ++i) b += s[i][c];
    ex[c] += b;
  }
#pragma unroll
  for (int k = 0; k < SCAN_TPT; ++k) {
    if (t0 + k < ntiles) {
      uint32_t c[16];
      uint32_t *row = tile_hist + size_t(t0 + k) * 16;
      load_row16(row, c);
      uint4 *r = reinterpret_cast<uint4 *>(row);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        r[q] = make_uint4(ex[4 * q], ex[4 * q + 1], ex[4 * q + 2], ex[4 * q + 3]);
        ex[4 * q] += c[4 * q], ex[4 * q + 1] += c[4 * q + 1], ex[4 * q + 2] += c[4 * q + 2],
            ex[4 * q + 3] += c[4 * q + 3];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Fused destination partition + exchange (the all-to-all-v of SURVEY §8e
// step 4 folded into the partition of step 2).  Every element's position in
// the GLOBAL class-major order is known once the class counts of all ranks
// are (gpos = shard-local class-major position + delta[class], delta from the
// host); destination rank d owns global positions [bounds[d], bounds[d+1]),
// so the element is stored straight into d's receive buffer at
// gpos - bounds[d] -- a peer (NVLink / NVSwitch) store for d != this rank.
// A tile is staged in shared memory in class order first, so consecutive
// threads store consecutive addresses of each class run.  Key-value: stable
// (a class's elements keep shard order -- stable ballot ranking -- and ranks'
// blocks are in rank order via delta).  Keys only: within a class, elements
// are ranked by their arrival slot on a shared class counter, so the order
// of tied keys (and which destination gets which copies of a tie class split
// across ranks) is unspecified; the receiver's sort orders them anyway, and
// with width < word bits keys tied on the low bits may come out in a
// different order from run to run.
// ---------------------------------------------------------------------------
template <typename K, int VB>
struct ExchangeSmem {
  using V = typename ValT<VB>::T;
  static constexpr size_t keys_off = 0;
  static constexpr size_t vals_off = sizeof(K) * SPLIT_TILE;
  static constexpr size_t bytes = vals_off + (VB ? sizeof(V) * SPLIT_TILE : 0);
};

template <typename K, int VB, int KIND>
__global__ void __launch_bounds__(SPLIT_BLOCK, sizeof(K) + VB <= 4 ? 4 : sizeof(K) + VB <= 8 ? 3 : 2) split_exchange_kernel(
    const K *keys, const void *vals_, uint64_t n, int shift0, const K *spl, int nsp, const uint32_t *tile_off,
    const long long *delta, const unsigned long long *bounds, int nranks, K *const *dst_keys,
    void *const *dst_vals, uint32_t *ticket) {
  using V = typename ValT<VB>::T;
  using S = ExchangeSmem<K, VB>;
  constexpr int NW = SPLIT_BLOCK / 32;
  extern __shared__ __align__(16) unsigned char xsm[];
  K *stage = reinterpret_cast<K *>(xsm + S::keys_off);
  V *vstage = reinterpret_cast<V *>(xsm + S::vals_off);
  __shared__ uint32_t wrun[NW][16];
  __shared__ uint32_t tb[17];
  __shared__ long long s_g[16];  // global position of tile position i in class c: s_g[c] + i
  __shared__ unsigned long long s_bnd[9];
  __shared__ K *s_dk[8];
  __shared__ V *s_dv[8];
  const KeyGeom<K, KIND> g{shift0};
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ncls = 2 * nsp + 1;
  __shared__ K s_spl[SPLIT_MAXSP + 1];
  __shared__ uint8_t s_tab[256];
  // once per CTA (the grid is persistent: a CTA takes tiles blockIdx.x,
  // blockIdx.x + gridDim.x, ...): splitters, class table, boundaries, tables
  load_splitters(s_spl, spl, nsp);
  const SplitClass<K> sc{s_spl, nsp};
  if (tid <= nranks) s_bnd[tid] = bounds[tid];
  if (tid < nranks) {
    s_dk[tid] = dst_keys[tid];
    if constexpr (VB != 0) s_dv[tid] = static_cast<V *>(dst_vals[tid]);
  }
  __syncthreads();
  build_split_lut(s_tab, sc);
  const SplitLUT<K> sr{s_tab, sc};
  const V *vals = static_cast<const V *>(vals_);
  const int wbase = w * 32 * SPLIT_KPT;
  const uint32_t lt = lanemask_lt();
  const uint32_t ntiles = uint32_t((n + SPLIT_TILE - 1) / SPLIT_TILE);
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
  for (int i = tid; i < NW * 16; i += SPLIT_BLOCK) (&wrun[0][0])[i] = 0;
  __syncthreads();  // also: the previous tile's write-out has left the staging buffer; the table is built
  const uint64_t base = uint64_t(tile) * SPLIT_TILE;
  const int cnt = int(min64(SPLIT_TILE, n - base));
  K x[SPLIT_KPT];
  V v[SPLIT_KPT];
  uint32_t dr[SPLIT_KPT];  // class | rank-in-warp << 8
  // all loads first (the ranking below is warp-collective, so loads inside
  // it would wait one by one)
#pragma unroll
  for (int j = 0; j < SPLIT_KPT; ++j) {
    const int e = wbase + 32 * j + lane;
    x[j] = K(0);
    if (e < cnt) {
      x[j] = keys[base + e];
      if constexpr (VB != 0) v[j] = vals[base + e];
    }
  }
  if constexpr (VB == 0) {
    // keys only: order inside a class is immaterial (the receiver sorts) --
    // the rank is the arrival slot on the warp's own class counter
#pragma unroll
    for (int j = 0; j < SPLIT_KPT; ++j) {
      const int e = wbase + 32 * j + lane;
      if (e < cnt) {
        const uint32_t d = sr.cls(g.norm(x[j]));
        dr[j] = d | (atomicAdd(&wrun[w][d], 1u) << 8);
      }
    }
  } else
#pragma unroll
  for (int j = 0; j < SPLIT_KPT; ++j) {
    const int e = wbase + 32 * j + lane;
    const bool valid = e < cnt;
    const uint32_t d = valid ? sr.cls(g.norm(x[j])) : 0u;
    // stable rank among this warp's elements of the same class (element
    // order j-major, lane-minor): 4 ballots match the class's 4 bits
    uint32_t peers = __ballot_sync(0xFFFFFFFFu, valid);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t bb = __ballot_sync(0xFFFFFFFFu, bit);
      peers &= bit ? bb : ~bb;
    }
    const uint32_t below = __popc(peers & lt);
    uint32_t old = 0;
    if (valid && below == 0) {
      old = wrun[w][d];
      wrun[w][d] = old + __popc(peers);
    }
    old = __shfl_sync(0xFFFFFFFFu, old, valid ? __ffs(peers) - 1 : lane);
    dr[j] = d | ((old + below) << 8);
    __syncwarp();
  }
  __syncthreads();
  if (w == 0) {  // warp 0, lane c < 16: per-warp exclusive prefixes of class c, then the tile's class bases
    uint32_t run = 0;
    if (lane < 16)
      for (int i = 0; i < NW; ++i) {
        const uint32_t c = wrun[i][lane];
        wrun[i][lane] = run;
        run += c;
      }
    uint32_t incl = run;  // inclusive scan over the 16 classes (lanes >= 16 hold 0)
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane < 16) {
      tb[lane + 1] = incl;
      if (lane == 0) tb[0] = 0;
      // shard class-major position -> global position
      s_g[lane] = (long long)tile_off[size_t(tile) * 16 + lane] + (lane < ncls ? delta[lane] : 0) -
                  (long long)(incl - run);
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < SPLIT_KPT; ++j) {
    const int e = wbase + 32 * j + lane;
    if (e < cnt) {
      const uint32_t d = dr[j] & 0xFFu;
      const uint32_t p = tb[d] + wrun[w][d] + (dr[j] >> 8);
      stage[p] = x[j];
      if constexpr (VB != 0) vstage[p] = v[j];
    }
  }
  __syncthreads();
  // Write-out by segments: the tile's positions, in class order, map to
  // increasing global positions; cutting them at class starts and at the
  // destination boundaries gives <= 15 + 7 segments, each a contiguous run
  // with one destination and one offset.  One thread lists the segments,
  // then each warp stores 32 consecutive positions per step.
  __shared__ uint32_t seg_start[24];
  __shared__ K *seg_kp[24];  // segment k: position i of the tile goes to seg_kp[k][i]
  __shared__ V *seg_vp[24];
  __shared__ int s_nseg;
  if (w == 0) {
    // lane c < 16 cuts class c's run [tb[c], tb[c+1]) at the destination
    // boundaries that fall inside it; a scan over the lanes places its
    // segments in the list (class order == position order)
    uint32_t a0 = 0, b0 = 0;
    long long gc = 0;
    int d0 = 0, nseg = 0;
    if (lane < 16) {
      a0 = tb[lane], b0 = tb[lane + 1], gc = s_g[lane];
      if (b0 > a0) {
        const unsigned long long gfirst = (unsigned long long)(gc + (long long)a0);
        const unsigned long long glast = (unsigned long long)(gc + (long long)b0) - 1ull;
        while (d0 + 1 < nranks && gfirst >= s_bnd[d0 + 1]) ++d0;
        int d1 = d0;
        while (d1 + 1 < nranks && glast >= s_bnd[d1 + 1]) ++d1;
        nseg = d1 - d0 + 1;
      }
    }
    int incl = nseg;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    int k = incl - nseg;
    uint32_t i = a0;
    for (int d = d0; d < d0 + nseg; ++d, ++k) {
      const long long off = gc - (long long)s_bnd[d];
      seg_start[k] = i;
      seg_kp[k] = s_dk[d] + off;
      if constexpr (VB != 0) seg_vp[k] = s_dv[d] + off;
      if (d + 1 < nranks) i = uint32_t(min64(uint64_t(b0), uint64_t(s_bnd[d + 1] - (unsigned long long)gc)));
    }
    if (lane == 15) {
      seg_start[incl] = uint32_t(cnt);  // sentinel
      s_nseg = incl;
    }
  }
  __syncthreads();
  // segment by segment: consecutive threads store consecutive addresses of one destination
  const int nseg_all = s_nseg;
  for (int k = 0; k < nseg_all; ++k) {
    const uint32_t e0 = seg_start[k + 1];
    K *const pk = seg_kp[k];
    if constexpr (VB != 0) {
      V *const pv = seg_vp[k];
      for (uint32_t i = seg_start[k] + uint32_t(tid); i < e0; i += SPLIT_BLOCK) {
        pk[i] = stage[i];
        pv[i] = vstage[i];
      }
    } else {
      for (uint32_t i = seg_start[k] + uint32_t(tid); i < e0; i += SPLIT_BLOCK) pk[i] = stage[i];
    }
  }
  }  // tiles
  // The receivers are ordered after this grid by stream order on this GPU
  // plus a collective later in the stream.  Release chain, explicit: every
  // CTA's stores (cumulative through the barrier) are ordered by a GPU-scope
  // fence before its ticket; the last CTA to take a ticket has observed all
  // of them and issues ONE system-scope fence -- instead of a system fence
  // per CTA, which holds the CTA's SM slot until its peer stores drain.
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(ticket, 1u) == gridDim.x - 1u) __threadfence_system();
  }
}

}  // namespace bs
