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
//               B2, the third (big tasks only) B3, later ones go to a small
//               overflow list; an overflow entry also marks its word in the
//               summary bitmap OF.
//   count/scan: thread t owns WPT consecutive bitmap words: popc(B1) [+ B2,
//               B3, listed copies of marked words] -> block exclusive scan ->
//               t's output offset.
//   enumerate:  the owner walks its words' set bits (lowest first) and writes
//               value = denorm(common | (32q + b) << lb), repeated by its
//               multiplicity, clearing the bitmaps as it goes.  The output is
//               staged IN the consumed input slot (its keys are dead after the
//               insert phase), which one thread then stores with a bulk async
//               copy (TMA) while the block moves on to the next task; the slot
//               goes back to the producer warp once that copy has drained
//               (checked one task later, after that task's insert phase).
//
// Per key that is one sequential shared load, one shared atomic and one
// shared store; per task one read of the bitmaps -- against the reference's
// partition loop (kernels.py:56-77) that touches every key once per bit.
// A producer warp streams tasks in through an NSLOT-deep TMA ring.
//
// Two instantiations.  Small tasks (<= 4608 keys): 256 consumers x 8 words,
// two bitmaps, 2 slots -- ~55 KB per CTA, so four CTAs share an SM and one's
// barriers and copy waits hide behind the others.  Big tasks (u32, <= 18432
// keys, e.g. the level-2 nodes of 2^30-key inputs): 512 consumers x 4 words,
// three bitmaps, one slot (two CTAs per SM cover each other's copy waits),
// launched per level right after scatter(L).
// A task with more repeats than the overflow list holds is handed to the
// general local sort (if it fits one of its tasks) or to the next MSD level as
// an ordinary bucket (big tasks beyond that), so the kernel is exact for any
// input.
#pragma once

#include "sort_impl.cuh"

namespace bs {

// index of the highest set bit (m != 0): one FLO
__device__ __forceinline__ uint32_t msb_index(uint32_t m) {
  uint32_t b;
  asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(m));
  return b;
}

template <typename K, int BLOCK, int CAP, int NSLOT, bool BIG>
struct DenseSmem {
  static constexpr int NW = 2048;     // 2^16 values / 32
  static constexpr int NS = NW / 32;  // summary words
  static constexpr int NB = BIG ? 3 : 2;  // presence bitmaps (copies held before the overflow list)
  static constexpr int DUPCAP = BIG ? 1024 : 64;
  static constexpr size_t kbuf = (sizeof(K) * CAP + 48 + 15) & ~size_t(15);
  static constexpr size_t dbuf_off = 0;
  // structure-of-arrays bitmaps: random words spread over all 32 banks
  static constexpr size_t b1_off = dbuf_off + NSLOT * kbuf;
  static constexpr size_t b2_off = b1_off + sizeof(uint32_t) * NW;
  static constexpr size_t b3_off = b2_off + sizeof(uint32_t) * NW;
  static constexpr size_t of_off = b3_off + (BIG ? sizeof(uint32_t) * NW : 0);  // word has overflow entries
  static constexpr size_t dup_off = of_off + sizeof(uint32_t) * NS;
  static constexpr size_t misc_off = dup_off + sizeof(uint32_t) * DUPCAP;
  static constexpr size_t bars_off = misc_off + sizeof(uint32_t) * 64;
  static constexpr size_t info_off = bars_off + sizeof(uint64_t) * 2 * NSLOT;
  static constexpr size_t bytes = info_off + sizeof(InFlight) * NSLOT;
};

template <typename K, int KIND, int BLOCK, int CAP, int NSLOT, bool BIG>
__global__ void __launch_bounds__(BLOCK + 32, BIG ? 2 : 4) dense_kernel(Ws ws, int L) {
  pdl_wait();  // programmatic dependent launch: previous kernel's writes visible
  if (ws_failed(ws)) return;
  using S = DenseSmem<K, BLOCK, CAP, NSLOT, BIG>;
  constexpr int WPT = S::NW / BLOCK;  // bitmap words per thread
  static_assert(WPT == 2 || WPT == 4 || WPT == 8, "thread t owns bitmap words WPT*t .. WPT*t + WPT-1");
  constexpr bool HAS3 = BIG;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t *B1 = reinterpret_cast<uint32_t *>(smem + S::b1_off);
  uint32_t *B2 = reinterpret_cast<uint32_t *>(smem + S::b2_off);
  uint32_t *B3 = reinterpret_cast<uint32_t *>(smem + S::b3_off);  // HAS3 only
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
  auto clear_all = [&]() {
    for (int q = tid; q < S::NW / 4; q += BLOCK) {
      reinterpret_cast<uint4 *>(B1)[q] = make_uint4(0, 0, 0, 0);
      reinterpret_cast<uint4 *>(B2)[q] = make_uint4(0, 0, 0, 0);
      if constexpr (HAS3) reinterpret_cast<uint4 *>(B3)[q] = make_uint4(0, 0, 0, 0);
    }
    if (tid < S::NS) OF[tid] = 0;
    if (tid == 0) misc[NDUP] = 0;
  };
  // every bitmap starts clear; afterwards owners clear what they used
  clear_all();
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
      // copies beyond the bitmaps: the overflow list
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
        // second copies (a few % of the keys), later ones (rare)
        if (rep) {
#pragma unroll
          for (int j = 0; j < EPG; ++j)
            if ((rep >> j) & 1u)
              if (atomicOr(&B2[idx[j] >> 5], bit[j]) & bit[j]) {
                if constexpr (HAS3) {
                  if (atomicOr(&B3[idx[j] >> 5], bit[j]) & bit[j]) later_copy(idx[j]);
                } else {
                  later_copy(idx[j]);
                }
              }
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
      // too many repeats: hand the task to the general local sort (small) or
      // to the next MSD level as an ordinary bucket (big)
      if (tid == 0) {
        // (only ranges the local sort cannot take become buckets: the bucket
        // and tile lists are sized for buckets of more than local_max keys)
        if (BIG && f.cnt > ws.local_max) push_bucket(ws, L, f.start, f.cnt, (f.digit >> 20) & 0xFu, f.parity & 1u);
        else emit_tasks(ws, f.start, f.cnt, f.parity & 1u);
        mbar_arrive(&empty[s]);
      }
      named_sync<BLOCK>();
      clear_all();
      named_sync<BLOCK>();
      continue;
    }
    // ---- count + scan: thread t owns words WPT*t .. WPT*t + WPT-1 ----
    const int nw = span <= 5 ? 1 : (1 << (span - 5));
    const bool own = WPT * tid < nw;
    uint32_t w1[WPT], w2[WPT], w3[HAS3 ? WPT : 1];
#pragma unroll
    for (int j = 0; j < WPT; ++j) w1[j] = w2[j] = 0;
#pragma unroll
    for (int j = 0; j < (HAS3 ? WPT : 1); ++j) w3[j] = 0;
    uint32_t of = 0;  // WPT-bit mask of this thread's words with overflow entries
    auto load_words = [&](const uint32_t *B, uint32_t *dst) {
      if constexpr (WPT == 2) {
        const uint2 a = reinterpret_cast<const uint2 *>(B)[tid];
        dst[0] = a.x, dst[1] = a.y;
      } else {
#pragma unroll
        for (int h = 0; h < WPT / 4; ++h) {
          const uint4 a = reinterpret_cast<const uint4 *>(B)[(WPT / 4) * tid + h];
          dst[4 * h] = a.x, dst[4 * h + 1] = a.y, dst[4 * h + 2] = a.z, dst[4 * h + 3] = a.w;
        }
      }
    };
    auto zero_words = [&](uint32_t *B) {
      if constexpr (WPT == 2) {
        reinterpret_cast<uint2 *>(B)[tid] = make_uint2(0, 0);
      } else {
#pragma unroll
        for (int h = 0; h < WPT / 4; ++h) reinterpret_cast<uint4 *>(B)[(WPT / 4) * tid + h] = make_uint4(0, 0, 0, 0);
      }
    };
    if (own) {
      load_words(B1, w1);
      load_words(B2, w2);
      if constexpr (HAS3) load_words(B3, w3);
      if (ndup) of = (OF[(WPT * tid) >> 5] >> ((WPT * tid) & 31)) & ((1u << WPT) - 1u);
    }
    uint32_t any2 = 0, any3 = 0;
#pragma unroll
    for (int j = 0; j < WPT; ++j) any2 |= w2[j];
    if constexpr (HAS3) {
#pragma unroll
      for (int j = 0; j < WPT; ++j) any3 |= w3[j];
    }
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < WPT; ++j) c += uint32_t(__popc(w1[j]));
    if (any2) {
#pragma unroll
      for (int j = 0; j < WPT; ++j) c += uint32_t(__popc(w2[j]));
    }
    if constexpr (HAS3) {
      if (any3) {
#pragma unroll
        for (int j = 0; j < WPT; ++j) c += uint32_t(__popc(w3[j]));
      }
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
      // iterations pipeline.  Repeats are predicated stores; words with listed
      // copies (rare) take the general loop.
      BS_DCHECK(ws.ctl, pos + c <= uint32_t(n));
      K *pe = stg + pos;
      const bool plain = KIND == 0 && lb == 0;
#pragma unroll
      for (int j = 0; j < WPT; ++j) {
        uint32_t m = w1[j];
        const uint32_t e2 = w2[j];
        const uint32_t e3 = HAS3 ? w3[j] : 0u;
        const uint32_t q = uint32_t(tid) * uint32_t(WPT) + uint32_t(j);
        const K hw = common | (K(q * 32u) << lb);
        if (((of >> j) & 1u) == 0u) {
          while (m) {
            const uint32_t t = m - 1u;
            const uint32_t bit = m & ~t;
            m &= t;
            const K v = plain ? (hw | K(msb_index(bit))) : denorm<K, KIND>(hw | (K(msb_index(bit)) << lb));
            pe[0] = v;
            if (e2 & bit) pe[1] = v;
            if constexpr (HAS3) {
              if (e3 & bit) pe[2] = v;
              pe += 1 + ((e2 & bit) ? 1 : 0) + ((e3 & bit) ? 1 : 0);
            } else {
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
              if (!HAS3 || (e3 & bit)) {
                if constexpr (HAS3) *pe++ = v;
                for (uint32_t t2 = 0; t2 < ndup; ++t2)
                  if (dup[t2] == q * 32u + b) *pe++ = v;
              }
            }
          }
        }
      }
      BS_DCHECK(ws.ctl, pe == stg + pos + c);
      if (c) {
        zero_words(B1);
        if (any2) zero_words(B2);
        if constexpr (HAS3) {
          if (any3) zero_words(B3);
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
      if constexpr (NSLOT == 1) {
        // single slot: it must be free before the next task can be loaded, so
        // thread 0 also copies the ragged ends and waits for the bulk store to
        // leave the slot (the SM's other CTA covers the wait)
        if (tid == 0) {
          if (m > 0) {
            bulk_s2g(dst + h, stg + h, uint32_t(m) * uint32_t(sizeof(K)));
            bulk_commit();
          }
          for (int e = 0; e < h; ++e) dst[e] = stg[e];
          for (int e = h + m; e < n; ++e) dst[e] = stg[e];
          bulk_wait_read0();
          mbar_arrive(&empty[s]);
        }
      } else {
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
  }
  if (tid == 0) bulk_wait0();
}

}  // namespace bs
