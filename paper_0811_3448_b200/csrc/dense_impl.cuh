// dense_impl.cuh -- K4a: dense keys-only local sort by bitmap enumeration.
//
// A dense task (planned by plan_kernel) holds keys that all equal `common`
// outside one bit span [lb, lb+span) of the normalised key (span <= 16): the
// common case after two 8-bit MSD levels of full-width keys, where each
// reference recursion node below the second digit (kernels.py:88-126) sorts
// ~2^12 keys that differ only in their low 16 bits.  Because a key is fully
// determined by its span bits, the sorted task is a function of the MULTISET
// of span values only -- so the kernel never moves keys, it counts them:
//
//   insert:     every key is read once from the TMA-filled input slot and sets
//               its bit in the presence bitmap B1 with one shared atomicOr.
//               A key that finds its bit set is a repeat: the second copy sets
//               B2, the third B3, later ones go to a small overflow list; a
//               an overflow entry also marks its word in the summary bitmap OF.
//               The input slot is released to the producer warp right here.
//   count/scan: thread t owns bitmap words 4t..4t+3 (one uint4 of B1):
//               popc(B1) [+ popc(B2) + popc(B3) + listed overflow copies for
//               marked words] -> block exclusive scan -> t's output offset.
//   enumerate:  the owner walks its words' set bits (top down, filling its
//               output run from the end) and
//               writes value = denorm(common | (32q + b) << lb), repeated by
//               its multiplicity, into the staging buffer (clearing B1/B2/B3
//               as it goes), which one thread then stores with a bulk async
//               copy (TMA) while the block moves on to the next task.
//
// Per key that is one sequential shared load, one shared atomic and one
// shared store; per task one read of B1 -- against the reference's
// partition loop (kernels.py:56-77) that touches every key once per bit.
// A producer warp streams tasks in through an NSLOT-deep TMA ring.
// A task with more repeats than the overflow list holds is handed to the
// general local sort (small variant) or to the next MSD level as an ordinary
// bucket (big variant), so the kernel is exact for any input.
#pragma once

#include "sort_impl.cuh"

namespace bs {

// index of the highest set bit (m != 0): one FLO
__device__ __forceinline__ uint32_t msb_index(uint32_t m) {
  uint32_t b;
  asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(m));
  return b;
}

template <typename K, int BLOCK, int CAP, int NSLOT>
struct DenseSmem {
  static constexpr int NW = 2048;                          // 2^16 values / 32
  static constexpr int NS = NW / 32;                       // summary words
  static constexpr int DUPCAP = CAP > 8192 ? 1024 : 256;  // fourth+ copies
  static constexpr size_t kbuf = (sizeof(K) * CAP + 32 + 15) & ~size_t(15);
  static constexpr size_t dbuf_off = 0;
  static constexpr size_t stg_off = dbuf_off + NSLOT * kbuf;  // staging (+16: alignment shift)
  // structure-of-arrays bitmaps: random words spread over all 32 banks
  static constexpr size_t b1_off = stg_off + kbuf + 16;
  static constexpr size_t b2_off = b1_off + sizeof(uint32_t) * NW;
  static constexpr size_t b3_off = b2_off + sizeof(uint32_t) * NW;
  static constexpr size_t of_off = b3_off + sizeof(uint32_t) * NW;  // word has overflow entries
  static constexpr size_t dup_off = of_off + sizeof(uint32_t) * NS;
  static constexpr size_t misc_off = dup_off + sizeof(uint32_t) * DUPCAP;
  static constexpr size_t bars_off = misc_off + sizeof(uint32_t) * 64;
  static constexpr size_t info_off = bars_off + sizeof(uint64_t) * 2 * NSLOT;
  static constexpr size_t bytes = info_off + sizeof(InFlight) * NSLOT;
};

template <typename K, int KIND, int BLOCK, int CAP, int NSLOT, bool BIG>
__global__ void __launch_bounds__(BLOCK + 32, BIG ? 1 : 2) dense_kernel(Ws ws, int L) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  using S = DenseSmem<K, BLOCK, CAP, NSLOT>;
  static_assert(S::NW == 4 * BLOCK, "thread t owns bitmap words 4t..4t+3");
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t *B1 = reinterpret_cast<uint32_t *>(smem + S::b1_off);
  uint32_t *B2 = reinterpret_cast<uint32_t *>(smem + S::b2_off);
  uint32_t *B3 = reinterpret_cast<uint32_t *>(smem + S::b3_off);
  uint32_t *OF = reinterpret_cast<uint32_t *>(smem + S::of_off);
  uint32_t *dup = reinterpret_cast<uint32_t *>(smem + S::dup_off);
  uint32_t *misc = reinterpret_cast<uint32_t *>(smem + S::misc_off);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S::bars_off);
  uint64_t *empty = full + NSLOT;
  InFlight *info = reinterpret_cast<InFlight *>(smem + S::info_off);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  // Small dense tasks: the whole list, after all levels.  Big ones: the tasks
  // planned at level L, right after scatter(L), so one that overflows can
  // still be pushed to level L+1 as an ordinary bucket.
  const uint32_t k0 = BIG ? (L > 0 ? ws.ctl->dbig_end[L - 1] : 0u) : 0u;
  const uint32_t nt = min(BIG ? ws.ctl->dbig_end[L] : ws.ctl->ndtasks, ws.maxtasks / 2) - min(k0, ws.maxtasks / 2);
  if (blockIdx.x >= nt) return;
  // big tasks are stored from the back of the list
  auto task_at = [&](uint32_t k) -> const DTask & {
    return ws.dtasks[BIG ? ws.maxtasks - 1 - (k0 + k) : k];
  };
  if (tid == BLOCK) {
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (w == BLOCK / 32) {  // ---------------- producer warp ----------------
    if (lane != 0) return;
    uint32_t ti = blockIdx.x;
    DTask nxt = task_at(ti);  // task records are fetched one task ahead
    for (uint32_t i = 0;; ++i) {
      const int s = int(i % NSLOT);
      const DTask t = nxt;
      const uint32_t tn = ti + gridDim.x;
      if (tn < nt) nxt = task_at(tn);
      if (i >= NSLOT) mbar_wait_sleep(&empty[s], ((i / NSLOT) - 1) & 1u);
      InFlight f{};
      f.idx = ti;
      if (ti < nt) {
        f.start = t.start;
        f.cnt = t.count;
        f.digit = t.meta;  // lb | span << 8 | parity << 16 | digit << 20
        f.parity = (t.meta >> 16) & 1u;
        const uint64_t cm = t.common;
        f.headv = uint32_t(cm);  // the common bits travel in headv:tile0
        f.tile0 = uint32_t(cm >> 32);
        const Span sk = span16(static_cast<const K *>(ws.keys[f.parity]) + f.start, f.cnt);
        f.headk = sk.head;
        info[s] = f;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[s], sk.bytes);
        bulk_g2s(smem + S::dbuf_off + s * S::kbuf, sk.base, sk.bytes, &full[s]);
      } else {
        info[s] = f;
        mbar_arrive(&full[s]);
        return;
      }
      ti = tn;
    }
  }

  // ---------------- consumers ----------------
  constexpr int NWARP = BLOCK / 32;
  constexpr int EPG = 16 / int(sizeof(K));  // keys per 16-byte granule
  constexpr int NDUP = 32;                  // misc[NDUP]: overflow count
  constexpr int GPT = (CAP / EPG + 2 + BLOCK - 1) / BLOCK;  // granules per thread (incl. head shift)
  // every bitmap starts clear; afterwards owners clear what they used
  for (int q = tid; q < S::NW / 4; q += BLOCK) {
    reinterpret_cast<uint4 *>(B1)[q] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4 *>(B2)[q] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4 *>(B3)[q] = make_uint4(0, 0, 0, 0);
  }
  if (tid < S::NS) OF[tid] = 0;
  if (tid == 0) misc[NDUP] = 0;
  named_sync<BLOCK>();
  const KeyGeom<K, KIND> g{0};
  for (uint32_t i = 0;; ++i) {
    const int s = int(i % NSLOT);
    mbar_wait(&full[s], (i / NSLOT) & 1u);
    const InFlight f = info[s];
    if (f.idx >= nt) break;
    const int n = int(f.cnt);
    const int lb = int(f.digit & 0xFFu), span = int((f.digit >> 8) & 0xFFu);
    const uint32_t vmask = (span >= 32) ? 0xFFFFFFFFu : ((1u << span) - 1u);
    const K common = K((uint64_t(f.tile0) << 32) | f.headv);
    // ---- insert: one presence atomic per key, 16-byte granules ----
    const K *slot = reinterpret_cast<const K *>(smem + S::dbuf_off + s * S::kbuf);
    const int head = int(f.headk);
    const int ngr = (head + n + EPG - 1) / EPG;
    {
      // third and later copies (rare): B3, then the overflow list
      auto third_copy = [&](uint32_t idx) {
        const uint32_t q = idx >> 5, bit = 1u << (idx & 31u);
        if (atomicOr(&B3[q], bit) & bit) {
          const uint32_t sl = atomicAdd(&misc[NDUP], 1u);
          if (sl < uint32_t(S::DUPCAP)) dup[sl] = idx;
          atomicOr(&OF[q >> 5], 1u << (q & 31u));
        }
      };
#pragma unroll
      for (int u = 0; u < GPT; ++u) {
        const int gi = tid + u * BLOCK;
        if (gi >= ngr) break;
        const uint4 v = reinterpret_cast<const uint4 *>(slot)[gi];
        K kk[EPG];
        if constexpr (sizeof(K) == 4) {
          kk[0] = K(v.x), kk[1] = K(v.y), kk[2 % EPG] = K(v.z), kk[3 % EPG] = K(v.w);
        } else {
          kk[0] = K((uint64_t(v.y) << 32) | v.x);
          kk[1 % EPG] = K((uint64_t(v.w) << 32) | v.z);
        }
        const int e0 = gi * EPG - head;
        // all presence atomics of the granule first, one rare branch after
        uint32_t idx[EPG], rep = 0;
#pragma unroll
        for (int j = 0; j < EPG; ++j) {
          idx[j] = uint32_t(g.norm(kk[j]) >> lb) & vmask;
          const bool ok = e0 + j >= 0 && e0 + j < n;
          const uint32_t bit = ok ? (1u << (idx[j] & 31u)) : 0u;
          if (atomicOr(&B1[idx[j] >> 5], bit) & bit) rep |= 1u << j;
        }
        // second copies: ~3% of the keys, so nearly every warp has some --
        // predicated atomics, no divergent branch
        uint32_t third = 0;
#pragma unroll
        for (int j = 0; j < EPG; ++j) {
          const uint32_t bit = 1u << (idx[j] & 31u);
          if (atom_or_shared_if(&B2[idx[j] >> 5], bit, (rep >> j) & 1u) & bit) third |= 1u << j;
        }
        if (third) {
#pragma unroll
          for (int j = 0; j < EPG; ++j)
            if ((third >> j) & 1u) third_copy(idx[j]);
        }
      }
    }
    named_sync<BLOCK>();  // S1: bitmaps complete, slot consumed
    if (tid == 0) mbar_arrive(&empty[s]);
    const uint32_t ndup = misc[NDUP];
    if (ndup > uint32_t(S::DUPCAP)) {
      // too many repeats: hand the task to the general local sort (small) or
      // to the next MSD level as an ordinary bucket (big)
      if (tid == 0) {
        if (BIG) push_bucket(ws, L, f.start, f.cnt, (f.digit >> 20) & 0xFu, f.parity & 1u);
        else emit_tasks(ws, f.start, f.cnt, f.parity & 1u);
      }
      named_sync<BLOCK>();
      for (int q = tid; q < S::NW / 4; q += BLOCK) {
        reinterpret_cast<uint4 *>(B1)[q] = make_uint4(0, 0, 0, 0);
        reinterpret_cast<uint4 *>(B2)[q] = make_uint4(0, 0, 0, 0);
        reinterpret_cast<uint4 *>(B3)[q] = make_uint4(0, 0, 0, 0);
      }
      if (tid < S::NS) OF[tid] = 0;
      if (tid == 0) misc[NDUP] = 0;
      named_sync<BLOCK>();
      continue;
    }
    // ---- count + scan: thread t owns words 4t..4t+3 ----
    const int nw = span <= 7 ? 4 : (1 << (span - 5));
    const bool own = 4 * tid < nw;
    uint4 b1 = make_uint4(0, 0, 0, 0);
    uint32_t of = 0;  // 4-bit mask of this thread's words with overflow entries
    uint4 b2 = make_uint4(0, 0, 0, 0), b3 = make_uint4(0, 0, 0, 0);
    if (own) {
      b1 = reinterpret_cast<const uint4 *>(B1)[tid];
      b2 = reinterpret_cast<const uint4 *>(B2)[tid];
      b3 = reinterpret_cast<const uint4 *>(B3)[tid];
      of = (OF[tid >> 3] >> (4 * (tid & 7))) & 0xFu;
    }
    uint32_t cw[4] = {uint32_t(__popc(b1.x) + __popc(b2.x) + __popc(b3.x)),
                      uint32_t(__popc(b1.y) + __popc(b2.y) + __popc(b3.y)),
                      uint32_t(__popc(b1.z) + __popc(b2.z) + __popc(b3.z)),
                      uint32_t(__popc(b1.w) + __popc(b2.w) + __popc(b3.w))};
    if (of)
      for (uint32_t t = 0; t < ndup; ++t) {
        const uint32_t q = dup[t] >> 5;
        if ((q >> 2) == uint32_t(tid)) {
          const uint32_t jj = q & 3u;
          cw[0] += jj == 0u, cw[1] += jj == 1u, cw[2] += jj == 2u, cw[3] += jj == 3u;
        }
      }
    const uint32_t c = cw[0] + cw[1] + cw[2] + cw[3];
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) misc[w] = incl;
    // the previous task's staging store must have left shared memory before
    // this task's enumeration overwrites it
    if (tid == 0) bulk_wait_read0();
    named_sync<BLOCK>();  // S2
    const uint32_t wt = lane < NWARP ? misc[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < NWARP; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += y;
    }
    const uint32_t pos = __shfl_sync(0xFFFFFFFFu, wi - wt, w) + incl - c;
    // summary words are read (above) before S2; clear them for the next task
    if (tid < S::NS) OF[tid] = 0;
    if (tid == 0) misc[NDUP] = 0;
    // ---- enumerate into the staging buffer (shifted to the output's 16-byte phase) ----
    K *dst = static_cast<K *>(ws.keys[0]) + f.start;
    const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(dst) & 15u);
    K *stg = reinterpret_cast<K *>(smem + S::stg_off + mis);
    if (own) {
      // Walk the owned words from the top bit down, writing the run backwards
      // from its end (FLO yields the bit index directly).  A second copy is a
      // predicated store; words with third or later copies (rare) take the
      // general loop.
      BS_DCHECK(ws.ctl, pos + c <= uint32_t(n));
      K *pe = stg + (pos + c);
      const uint32_t w1[4] = {b1.x, b1.y, b1.z, b1.w};
      const uint32_t w2[4] = {b2.x, b2.y, b2.z, b2.w};
      const uint32_t w3[4] = {b3.x, b3.y, b3.z, b3.w};
      const bool plain = KIND == 0 && lb == 0;
#pragma unroll
      for (int j = 3; j >= 0; --j) {
        uint32_t m = w1[j];
        const uint32_t e2 = w2[j];
        const uint32_t q = uint32_t(tid) * 4u + uint32_t(j);
        const K hw = common | (K(q * 32u) << lb);
        if (w3[j] == 0u) {
          if (plain) {
            if (m) do {
                const uint32_t b = msb_index(m);
                m ^= 1u << b;
                const K v = hw | K(b);
                const uint32_t r = (e2 >> b) & 1u;
                pe[-1] = v;
                if (r) pe[-2] = v;
                pe -= 1u + r;
              } while (m);
          } else {
            if (m) do {
                const uint32_t b = msb_index(m);
                m ^= 1u << b;
                const K v = denorm<K, KIND>(hw | (K(b) << lb));
                const uint32_t r = (e2 >> b) & 1u;
                pe[-1] = v;
                if (r) pe[-2] = v;
                pe -= 1u + r;
              } while (m);
          }
        } else {
          while (m) {
            const uint32_t b = msb_index(m);
            m ^= 1u << b;
            const K v = denorm<K, KIND>(hw | (K(b) << lb));
            *--pe = v;
            if ((e2 >> b) & 1u) {
              *--pe = v;
              if ((w3[j] >> b) & 1u) {
                *--pe = v;
                if ((of >> j) & 1u)
                  for (uint32_t t = 0; t < ndup; ++t)
                    if (dup[t] == q * 32u + b) *--pe = v;
              }
            }
          }
        }
      }
      if (b1.x | b1.y | b1.z | b1.w) reinterpret_cast<uint4 *>(B1)[tid] = make_uint4(0, 0, 0, 0);
      if (b2.x | b2.y | b2.z | b2.w) reinterpret_cast<uint4 *>(B2)[tid] = make_uint4(0, 0, 0, 0);
      if (b3.x | b3.y | b3.z | b3.w) reinterpret_cast<uint4 *>(B3)[tid] = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();  // staging writes -> visible to the bulk copy
    named_sync<BLOCK>();       // S3
    // ---- store: 16-byte-aligned middle by one bulk copy, ragged ends by threads ----
    BS_DCHECK(ws.ctl, f.start + uint64_t(n) <= ws.n && n <= CAP);
    {
      const int h = min(n, mis ? int((16u - mis) / sizeof(K)) : 0);
      const int m = ((n - h) / EPG) * EPG;
      if (tid == 0 && m > 0) {
        bulk_s2g(dst + h, stg + h, uint32_t(m) * uint32_t(sizeof(K)));
        bulk_commit();
      }
      if (tid < h) dst[tid] = stg[tid];
      if (h + m + tid < n) dst[h + m + tid] = stg[h + m + tid];
    }
  }
  if (tid == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------
// K4a, small tasks (<= CAP keys): the same counting sort arranged for
// occupancy.  256 consumers own 8 bitmap words each (half the warps pay the
// per-task scan / barrier overhead), two presence bitmaps (third and later
// copies go to the overflow list), and the output is staged IN the consumed
// input slot, so a CTA needs 2 slots + 16 KB of bitmaps (~54 KB) and four
// CTAs share an SM: while one waits at a barrier or for its copy, three others
// insert or enumerate.  A slot is handed back to the producer warp once the
// bulk store that reads it has drained (checked one task later, after that
// task's insert phase).
// ---------------------------------------------------------------------------
template <typename K, int BLOCK, int CAP, int NSLOT>
struct Dense2Smem {
  static constexpr int NW = 2048;     // 2^16 values / 32
  static constexpr int NS = NW / 32;  // summary words
  static constexpr int DUPCAP = 512;  // third+ copies
  static constexpr size_t kbuf = (sizeof(K) * CAP + 48 + 15) & ~size_t(15);
  static constexpr size_t dbuf_off = 0;
  static constexpr size_t b1_off = dbuf_off + NSLOT * kbuf;
  static constexpr size_t b2_off = b1_off + sizeof(uint32_t) * NW;
  static constexpr size_t of_off = b2_off + sizeof(uint32_t) * NW;
  static constexpr size_t dup_off = of_off + sizeof(uint32_t) * NS;
  static constexpr size_t misc_off = dup_off + sizeof(uint32_t) * DUPCAP;
  static constexpr size_t bars_off = misc_off + sizeof(uint32_t) * 64;
  static constexpr size_t info_off = bars_off + sizeof(uint64_t) * 2 * NSLOT;
  static constexpr size_t bytes = info_off + sizeof(InFlight) * NSLOT;
};

template <typename K, int KIND, int BLOCK, int CAP, int NSLOT>
__global__ void __launch_bounds__(BLOCK + 32, 4) dense2_kernel(Ws ws) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  using S = Dense2Smem<K, BLOCK, CAP, NSLOT>;
  constexpr int WPT = S::NW / BLOCK;  // bitmap words per thread
  static_assert(WPT == 8, "thread t owns bitmap words 8t..8t+7");
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t *B1 = reinterpret_cast<uint32_t *>(smem + S::b1_off);
  uint32_t *B2 = reinterpret_cast<uint32_t *>(smem + S::b2_off);
  uint32_t *OF = reinterpret_cast<uint32_t *>(smem + S::of_off);
  uint32_t *dup = reinterpret_cast<uint32_t *>(smem + S::dup_off);
  uint32_t *misc = reinterpret_cast<uint32_t *>(smem + S::misc_off);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S::bars_off);
  uint64_t *empty = full + NSLOT;
  InFlight *info = reinterpret_cast<InFlight *>(smem + S::info_off);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t nt = min(ws.ctl->ndtasks, ws.maxtasks / 2);
  if (blockIdx.x >= nt) return;
  if (tid == BLOCK) {
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (w == BLOCK / 32) {  // ---------------- producer warp ----------------
    if (lane != 0) return;
    uint32_t ti = blockIdx.x;
    DTask nxt = ws.dtasks[ti];  // task records are fetched one task ahead
    for (uint32_t i = 0;; ++i) {
      const int s = int(i % NSLOT);
      const DTask t = nxt;
      const uint32_t tn = ti + gridDim.x;
      if (tn < nt) nxt = ws.dtasks[tn];
      if (i >= NSLOT) mbar_wait_sleep(&empty[s], ((i / NSLOT) - 1) & 1u);
      InFlight f{};
      f.idx = ti;
      if (ti < nt) {
        f.start = t.start;
        f.cnt = t.count;
        f.digit = t.meta;  // lb | span << 8 | parity << 16 | digit << 20
        f.parity = (t.meta >> 16) & 1u;
        const uint64_t cm = t.common;
        f.headv = uint32_t(cm);  // the common bits travel in headv:tile0
        f.tile0 = uint32_t(cm >> 32);
        const Span sk = span16(static_cast<const K *>(ws.keys[f.parity]) + f.start, f.cnt);
        f.headk = sk.head;
        info[s] = f;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[s], sk.bytes);
        bulk_g2s(smem + S::dbuf_off + s * S::kbuf, sk.base, sk.bytes, &full[s]);
      } else {
        info[s] = f;
        mbar_arrive(&full[s]);
        return;
      }
      ti = tn;
    }
  }

  // ---------------- consumers ----------------
  constexpr int NWARP = BLOCK / 32;
  constexpr int EPG = 16 / int(sizeof(K));  // keys per 16-byte granule
  constexpr int NDUP = 32;                  // misc[NDUP]: overflow count
  constexpr int GPT = (CAP / EPG + 2 + BLOCK - 1) / BLOCK;  // granules per thread (incl. head shift)
  // every bitmap starts clear; afterwards owners clear what they used
  for (int q = tid; q < S::NW / 4; q += BLOCK) {
    reinterpret_cast<uint4 *>(B1)[q] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4 *>(B2)[q] = make_uint4(0, 0, 0, 0);
  }
  if (tid < S::NS) OF[tid] = 0;
  if (tid == 0) misc[NDUP] = 0;
  named_sync<BLOCK>();
  const KeyGeom<K, KIND> g{0};
  int pending = -1;  // tid 0: slot whose bulk store has not been waited for yet
  for (uint32_t i = 0;; ++i) {
    const int s = int(i % NSLOT);
    mbar_wait(&full[s], (i / NSLOT) & 1u);
    const InFlight f = info[s];
    if (f.idx >= nt) break;
    const int n = int(f.cnt);
    const int lb = int(f.digit & 0xFFu), span = int((f.digit >> 8) & 0xFFu);
    const uint32_t vmask = (span >= 32) ? 0xFFFFFFFFu : ((1u << span) - 1u);
    const K common = K((uint64_t(f.tile0) << 32) | f.headv);
    unsigned char *slotb = smem + S::dbuf_off + s * S::kbuf;
    // ---- insert: one presence atomic per key, 16-byte granules ----
    const K *slot = reinterpret_cast<const K *>(slotb);
    const int head = int(f.headk);
    const int ngr = (head + n + EPG - 1) / EPG;
    {
      // third and later copies: the overflow list
      auto later_copy = [&](uint32_t idx) {
        const uint32_t q = idx >> 5;
        const uint32_t sl = atomicAdd(&misc[NDUP], 1u);
        if (sl < uint32_t(S::DUPCAP)) dup[sl] = idx;
        atomicOr(&OF[q >> 5], 1u << (q & 31u));
      };
      // granules [g_lo, g_hi) lie wholly inside the task: no per-key bounds
      const int g_lo = (head + EPG - 1) / EPG, g_hi = (head + n) / EPG;
#pragma unroll
      for (int u = 0; u < GPT; ++u) {
        const int gi = tid + u * BLOCK;
        if (gi >= ngr) break;
        const uint4 v = reinterpret_cast<const uint4 *>(slot)[gi];
        K kk[EPG];
        if constexpr (sizeof(K) == 4) {
          kk[0] = K(v.x), kk[1] = K(v.y), kk[2 % EPG] = K(v.z), kk[3 % EPG] = K(v.w);
        } else {
          kk[0] = K((uint64_t(v.y) << 32) | v.x);
          kk[1 % EPG] = K((uint64_t(v.w) << 32) | v.z);
        }
        uint32_t idx[EPG], bit[EPG], rep = 0;
        if (gi >= g_lo && gi < g_hi) {
#pragma unroll
          for (int j = 0; j < EPG; ++j) {
            idx[j] = uint32_t(g.norm(kk[j]) >> lb) & vmask;
            bit[j] = 1u << (idx[j] & 31u);
            if (atomicOr(&B1[idx[j] >> 5], bit[j]) & bit[j]) rep |= 1u << j;
          }
        } else {
          const int e0 = gi * EPG - head;
#pragma unroll
          for (int j = 0; j < EPG; ++j) {
            idx[j] = uint32_t(g.norm(kk[j]) >> lb) & vmask;
            const bool ok = e0 + j >= 0 && e0 + j < n;
            bit[j] = ok ? (1u << (idx[j] & 31u)) : 0u;
            if (atomicOr(&B1[idx[j] >> 5], bit[j]) & bit[j]) rep |= 1u << j;
          }
        }
        // second copies (~3% of the keys), later ones (rare)
        if (rep) {
#pragma unroll
          for (int j = 0; j < EPG; ++j)
            if ((rep >> j) & 1u)
              if (atomicOr(&B2[idx[j] >> 5], bit[j]) & bit[j]) later_copy(idx[j]);
        }
      }
    }
    named_sync<BLOCK>();  // S1: bitmaps complete, input keys consumed
    if (tid == 0 && pending >= 0) {
      // the previous task's bulk store has left its slot by now: hand it back
      bulk_wait_read0();
      mbar_arrive(&empty[pending]);
      pending = -1;
    }
    const uint32_t ndup = misc[NDUP];
    if (ndup > uint32_t(S::DUPCAP)) {
      // too many repeats: hand the task to the general local sort
      if (tid == 0) {
        emit_tasks(ws, f.start, f.cnt, f.parity & 1u);
        mbar_arrive(&empty[s]);
      }
      named_sync<BLOCK>();
      for (int q = tid; q < S::NW / 4; q += BLOCK) {
        reinterpret_cast<uint4 *>(B1)[q] = make_uint4(0, 0, 0, 0);
        reinterpret_cast<uint4 *>(B2)[q] = make_uint4(0, 0, 0, 0);
      }
      if (tid < S::NS) OF[tid] = 0;
      if (tid == 0) misc[NDUP] = 0;
      named_sync<BLOCK>();
      continue;
    }
    // ---- count + scan: thread t owns words 8t..8t+7 ----
    const int nw = span <= 8 ? 8 : (1 << (span - 5));
    const bool own = WPT * tid < nw;
    uint32_t w1[WPT], w2[WPT];
#pragma unroll
    for (int j = 0; j < WPT; ++j) w1[j] = w2[j] = 0;
    uint32_t of = 0;  // 8-bit mask of this thread's words with overflow entries
    if (own) {
      const uint4 a0 = reinterpret_cast<const uint4 *>(B1)[2 * tid], a1 = reinterpret_cast<const uint4 *>(B1)[2 * tid + 1];
      const uint4 c0 = reinterpret_cast<const uint4 *>(B2)[2 * tid], c1 = reinterpret_cast<const uint4 *>(B2)[2 * tid + 1];
      w1[0] = a0.x, w1[1] = a0.y, w1[2] = a0.z, w1[3] = a0.w, w1[4] = a1.x, w1[5] = a1.y, w1[6] = a1.z, w1[7] = a1.w;
      w2[0] = c0.x, w2[1] = c0.y, w2[2] = c0.z, w2[3] = c0.w, w2[4] = c1.x, w2[5] = c1.y, w2[6] = c1.z, w2[7] = c1.w;
      if (ndup) of = (OF[tid >> 2] >> (8 * (tid & 3))) & 0xFFu;
    }
    const bool any2 = (w2[0] | w2[1] | w2[2] | w2[3] | w2[4] | w2[5] | w2[6] | w2[7]) != 0u;
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < WPT; ++j) c += uint32_t(__popc(w1[j]));
    if (any2) {
#pragma unroll
      for (int j = 0; j < WPT; ++j) c += uint32_t(__popc(w2[j]));
    }
    if (of)
      for (uint32_t t = 0; t < ndup; ++t) c += ((dup[t] >> 5) / uint32_t(WPT)) == uint32_t(tid);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) misc[w] = incl;
    named_sync<BLOCK>();  // S2
    const uint32_t wt = lane < NWARP ? misc[lane] : 0u;
    uint32_t wi = wt;
#pragma unroll
    for (int o = 1; o < NWARP; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += y;
    }
    const uint32_t pos = __shfl_sync(0xFFFFFFFFu, wi - wt, w) + incl - c;
    // the summary words and the counter were read before S2; clear them for the
    // next task (its insert phase starts after S3)
    if (ndup) {
      if (tid < S::NS) OF[tid] = 0;
      if (tid == 0) misc[NDUP] = 0;
    }
    // ---- enumerate into the consumed slot (shifted to the output's 16-byte phase) ----
    K *dst = static_cast<K *>(ws.keys[0]) + f.start;
    const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(dst) & 15u);
    K *stg = reinterpret_cast<K *>(slotb + mis);
    if (own) {
      // Walk the owned words from the lowest bit up, writing the run forwards.
      // The loop-carried state is the mask alone (m &= m - 1); the bit index
      // (FLO, a long-latency pipe) hangs off the isolated bit, so consecutive
      // iterations pipeline.  A second copy is a predicated store; words with
      // listed copies (rare) take the general loop.
      BS_DCHECK(ws.ctl, pos + c <= uint32_t(n));
      K *pe = stg + pos;
      const bool plain = KIND == 0 && lb == 0;
#pragma unroll
      for (int j = 0; j < WPT; ++j) {
        uint32_t m = w1[j];
        const uint32_t e2 = w2[j];
        const uint32_t q = uint32_t(tid) * uint32_t(WPT) + uint32_t(j);
        const K hw = common | (K(q * 32u) << lb);
        if (((of >> j) & 1u) == 0u) {
          if (plain) {
            while (m) {
              const uint32_t t = m - 1u;
              const uint32_t bit = m & ~t;
              m &= t;
              const K v = hw | K(msb_index(bit));
              pe[0] = v;
              if (e2 & bit) pe[1] = v;
              pe += (e2 & bit) ? 2 : 1;
            }
          } else {
            while (m) {
              const uint32_t t = m - 1u;
              const uint32_t bit = m & ~t;
              m &= t;
              const K v = denorm<K, KIND>(hw | (K(msb_index(bit)) << lb));
              pe[0] = v;
              if (e2 & bit) pe[1] = v;
              pe += (e2 & bit) ? 2 : 1;
            }
          }
        } else {
          while (m) {
            const uint32_t t = m - 1u;
            const uint32_t bit = m & ~t;
            m &= t;
            const uint32_t b = msb_index(bit);
            const K v = denorm<K, KIND>(hw | (K(b) << lb));
            *pe++ = v;
            if (e2 & bit) {
              *pe++ = v;
              for (uint32_t t2 = 0; t2 < ndup; ++t2)
                if (dup[t2] == q * 32u + b) *pe++ = v;
            }
          }
        }
      }
      BS_DCHECK(ws.ctl, pe == stg + pos + c);
      if (c) {
        reinterpret_cast<uint4 *>(B1)[2 * tid] = make_uint4(0, 0, 0, 0);
        reinterpret_cast<uint4 *>(B1)[2 * tid + 1] = make_uint4(0, 0, 0, 0);
        if (any2) {
          reinterpret_cast<uint4 *>(B2)[2 * tid] = make_uint4(0, 0, 0, 0);
          reinterpret_cast<uint4 *>(B2)[2 * tid + 1] = make_uint4(0, 0, 0, 0);
        }
      }
    }
    fence_proxy_async_smem();  // staging writes -> visible to the bulk copy
    named_sync<BLOCK>();       // S3
    // ---- store: 16-byte-aligned middle by one bulk copy, ragged ends by threads ----
    BS_DCHECK(ws.ctl, f.start + uint64_t(n) <= ws.n && n <= CAP);
    {
      const int h = min(n, mis ? int((16u - mis) / sizeof(K)) : 0);
      const int m = ((n - h) / EPG) * EPG;
      if (tid == 0) {
        if (m > 0) {
          bulk_s2g(dst + h, stg + h, uint32_t(m) * uint32_t(sizeof(K)));
          bulk_commit();
        }
        pending = s;
      }
      if (tid < h) dst[tid] = stg[tid];
      if (h + m + tid < n) dst[h + m + tid] = stg[h + m + tid];
    }
  }
  if (tid == 0) bulk_wait0();
}

}  // namespace bs
