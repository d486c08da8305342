/*
 * binarsort_b200.h -- C ABI of the B200-native Binar Sort hot path.
 *
 * The reference (arxiv 0811.3448, package `binarsort`) routes a 1-D word
 * array to its numba kernel module through `KeyCodec.words_view`
 * (/root/reference/pkg/src/binarsort/keys.py:140-149,175-178) and then calls
 *
 *     kernels.sort_words(words, 0, n-1, 0, width, False, 0, 0, False, counters, 1)
 *
 * (core.py:213-219, kernels.py:88-126).  The entry points below replace that
 * kernel-module ABI (kernels.py:52-172) for device-resident buffers.  All
 * pointers named `keys`, `vals`, `ws`, `counters` are DEVICE pointers; `stream`
 * is a cudaStream_t (NULL = legacy default stream).  No call allocates device
 * memory, keeps global mutable state, or synchronises the stream unless it
 * says so; calls on distinct streams with distinct buffers are independent.
 *
 * Status codes map onto the reference's exception types in the Python shim:
 *   BS_ERR_VALUE  -> ValueError      (bad configuration, keys.py:164-165 etc.)
 *   BS_ERR_ASSERT -> AssertionError  (contract violation, core.py:102-105)
 *   BS_ERR_CUDA / BS_ERR_WORKSPACE / BS_ERR_INTERNAL -> RuntimeError
 * bs_last_error() returns a thread-local message for the last failing call.
 */
#ifndef BINARSORT_B200_H
#define BINARSORT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BS_OK 0
#define BS_ERR_VALUE 1
#define BS_ERR_ASSERT 2
#define BS_ERR_CUDA 3
#define BS_ERR_WORKSPACE 4
#define BS_ERR_INTERNAL 5

/* key_kind: the codec's order-preserving word transform (keys.py:51-93). */
#define BS_KEY_UNSIGNED 0 /* UnsignedCodec(width): identity, low `width` bits  */
#define BS_KEY_SIGNED 1   /* SignedCodec(width): flip bit width-1 (two's compl.) */
#define BS_KEY_FLOAT 2    /* Float64Codec: IEEE-754 total-order transform       */

/* Library version (major*10000 + minor*100 + patch). */
int bs_version(void);

/* 1 in the bounds-checked build (libbinarsort_b200_debug.so), else 0. */
int bs_debug_checks(void);

/* Thread-local message for the last non-BS_OK return on this thread. */
const char *bs_last_error(void);

/*
 * Workspace bytes bs_sort needs for n elements (replaces nothing in the
 * reference: the numba kernel is in-place; the GPU MSD ping-pongs through a
 * second buffer of n*(key_bytes+val_bytes) plus O(n/1024) bucket metadata).
 * key_bytes in {4, 8}; val_bytes in {0, 4, 8}.
 */
size_t bs_workspace_bytes(uint64_t n, int key_bytes, int val_bytes);

/*
 * Device status of the last sort that used workspace `ws` (bs_sort or
 * bs_sort_from): enqueues on `stream` a 4-byte copy of the sort's overflow
 * flag into *status (device or pinned host memory).  0 = OK; otherwise bit 0
 * bucket-list overflow, bit 1 tile-map overflow, bit 2 task-list overflow --
 * work was dropped and the output is NOT sorted -- and, in the bounds-checked
 * build (libbinarsort_b200_debug.so, -DBS_DEBUG_CHECKS), bit 3 = a write
 * index failed its check.  The capacities are sized so
 * this cannot happen for any input (Geometry in binarsort_b200.cu); the flag
 * is the loud failure path that proves it (the Python shim raises
 * RuntimeError).  No reference counterpart: the numba kernels cannot run out
 * of work-list space (kernels.py:88-126 recurses on the call stack).
 */
int bs_sort_status(const void *ws, int32_t *status, void *stream);
/* Byte offset of that status word inside the workspace: a caller that
 * synchronises the stream anyway can read it in place (no copy launched). */
size_t bs_sort_status_offset(void);

/*
 * Test hook: cap the work-list capacities (buckets, tiles, tasks) of the
 * sorts this thread launches next; 0 = no cap.  Caps only shrink the lists, so
 * any workspace sized by bs_workspace_bytes stays valid.  Used by the
 * forced-overflow test to prove bs_sort_status reports dropped work.
 */
void bs_debug_capacity(uint32_t max_buckets, uint32_t max_tiles, uint32_t max_tasks);

/*
 * Sort keys[0..n) (and vals[0..n) alongside, if vals != NULL) in place into
 * nondecreasing codec order.  Replaces kernels.sort_words(arr, lower, upper,
 * pos, width, False, 0, 0, False, counters, depth) (kernels.py:88-126) for the
 * sub-range arr[lower..upper]: pass keys = arr + lower, n = upper-lower+1,
 * start_pos = pos.  The sort key of a word is its low `width` bits read from
 * bit (width-1-start_pos) down to bit 0 (kernels.py:63,69), after the
 * key_kind transform.
 *
 * Keys-only output is the unique nondecreasing sequence, hence bit-exact with
 * the reference.  With vals the sort is STABLE (ties keep input order), which
 * is exactly the order the reference produces on packed (key<<32|index) words
 * (SURVEY §8c).  `counters`, if non-NULL, is a device int64[4] that receives
 * the reference Metrics {bit_extractions, swaps, recursive_calls, max_depth}
 * of the baseline recursive sort started at `depth` (closed form over the
 * sorted output); it is written asynchronously.
 */
int bs_sort(void *keys, void *vals, uint64_t n, int key_bytes, int val_bytes,
            int width, int start_pos, int key_kind, void *ws, size_t ws_bytes,
            void *stream, int64_t *counters, int64_t depth);

/*
 * bs_sort plus phase timing (bench instrumentation; SYNCHRONISES `stream`):
 * times the phases [init, {hist(L), plan(L), scatter(L)} for each level L,
 * local sort] with CUDA events on `stream`, writes up to `nphases` durations
 * in milliseconds to phase_ms and the number written to *nrecorded.
 */
int bs_sort_profiled(void *keys, void *vals, uint64_t n, int key_bytes,
                     int val_bytes, int width, int start_pos, int key_kind,
                     void *ws, size_t ws_bytes, void *stream, int64_t *counters,
                     int64_t depth, float *phase_ms, int nphases, int *nrecorded);

/*
 * bs_sort from a separate source: sorts src_keys[0..n) (+src_vals) into
 * keys[0..n) (+vals), using the source buffers as the MSD ping-pong copy (their
 * contents are destroyed).  Same order, stability and arguments as bs_sort;
 * ws must hold bs_sort_from_workspace_bytes(n, ...), which has no n-element
 * copy.  The multi-GPU front end sorts each rank's receive buffer this way
 * (the receive buffer stays registered for peer access; the result lands in
 * a fresh caller buffer).  Replaces the local sort after the exchange in
 * variants.sort_parallel (variants.py:195-206).
 */
size_t bs_sort_from_workspace_bytes(uint64_t n, int key_bytes, int val_bytes);
int bs_sort_from(void *src_keys, void *src_vals, void *keys, void *vals, uint64_t n,
                 int key_bytes, int val_bytes, int width, int start_pos,
                 int key_kind, void *ws, size_t ws_bytes, void *stream);
/* Number of kernels bs_sort launches for this shape (for launch accounting). */
int bs_sort_launches(uint64_t n, int key_bytes, int width, int start_pos,
                     int with_counters);

/*
 * Reference Metrics of kernels.sort_words over an ALREADY SORTED device array
 * (the K6 closed form).  Adds into the device int64[4]
 * `counters` with Metrics.merge semantics (core.py:60-77): counts add,
 * max_depth takes the max.  ws must hold bs_metrics_workspace_bytes(n).
 */
size_t bs_metrics_workspace_bytes(uint64_t n);
int bs_metrics(const void *sorted_keys, uint64_t n, int key_bytes, int width,
               int start_pos, int key_kind, int64_t depth, void *ws,
               size_t ws_bytes, void *stream, int64_t *counters);

/*
 * One reference partition pass (kernels.partition_words, kernels.py:56-77) on
 * keys[0..n) at bit `pos`, reproducing the reference's exact (unstable)
 * two-cursor permutation via its closed form; vals (may be
 * NULL) receive the same permutation.  The bit is read from the raw word as
 * (x << pos) & (1 << (width-1)) (kernels.py:63,69).  Writes the split index
 * (relative to keys) to *split_dev (device int64) and adds n extractions and
 * the swap count into counters (device int64[4], may be NULL).  ws must hold
 * bs_partition_workspace_bytes(n, key_bytes, val_bytes).
 */
size_t bs_partition_workspace_bytes(uint64_t n, int key_bytes, int val_bytes);
int bs_partition_words(void *keys, void *vals, uint64_t n, int key_bytes,
                       int val_bytes, int width, int pos, void *ws,
                       size_t ws_bytes, void *stream, int64_t *split_dev,
                       int64_t *counters);

/*
 * kernels.range_sorted_words (kernels.py:80-85): writes 1 to *flag_dev
 * (device int32) iff keys[0..n) is nondecreasing as unsigned words.
 */
int bs_range_sorted(const void *keys, uint64_t n, int key_bytes, void *stream,
                    int32_t *flag_dev);

/* ---------------------------------------------------------------------------
 * Multi-GPU front end (replaces variants.sort_parallel's serial top-bit
 * pre-partition + thread pool, variants.py:124-229).  The host issues the
 * small collectives (sample and class-count all-gathers) over NCCL; the data
 * moves either through bs_split_exchange (fused partition + peer-memory
 * stores, the product path) or through bs_split_by_splitters + an NCCL
 * all-to-all-v (baseline).  These are the per-rank device steps.
 * ------------------------------------------------------------------------- */

/*
 * Stable partition of keys[0..n) (+vals) into 2*R-1 destination classes given
 * R-1 nondecreasing splitter words (device, already key_kind-encoded and
 * normalised to the top of the word): class 2j = keys strictly between
 * splitter j-1 and splitter j, class 2j+1 = keys equal to splitter j.  The
 * result goes to out_keys/out_vals (device, n elements) and the 2R-1 class
 * counts to class_counts (device uint64).  ws: bs_split_workspace_bytes.
 */
size_t bs_split_workspace_bytes(uint64_t n, int key_bytes, int val_bytes, int nranks);
int bs_split_by_splitters(const void *keys, const void *vals, uint64_t n,
                          int key_bytes, int val_bytes, int width,
                          int key_kind, const void *splitters, int nranks,
                          void *out_keys, void *out_vals, uint64_t *class_counts,
                          void *ws, size_t ws_bytes, void *stream);

/*
 * Fused destination partition + exchange over peer memory (one kernel instead
 * of partition -> ncclAllToAllv):
 *   bs_split_count: per-tile class histogram and class-major scan of keys
 *     against the splitters (as bs_split_by_splitters); writes the 2R-1 class
 *     counts (device uint64) and keeps the tile offsets in ws for
 *   bs_split_exchange: with delta[c] = (global class-major position of this
 *     rank's first class-c element) - (its shard-local class-major position)
 *     and bounds[0..R] (destination d owns global positions [bounds[d],
 *     bounds[d+1])), stores every element at dst_keys[d][gpos - bounds[d]]
 *     (dst_vals alike).  dst_keys / dst_vals are DEVICE arrays of R device
 *     pointers, normally peer mappings of the other ranks' receive buffers
 *     (bs_ipc_open).  Call with the same ws right after bs_split_count on the
 *     same keys.  The grid ends with a system-scope fence; the caller orders
 *     the receivers after it (stream order + a collective).
 *     With vals the exchange is stable (class, then source rank, then shard
 *     index).  Keys only, the order of elements within a class (and which
 *     copies of a tie class land on which destination) is unspecified: they
 *     are ranked by arrival on a shared counter, and the receiver's sort
 *     orders them.  Keys tied on their low `width` bits may therefore arrive
 *     in a run-dependent order.  nranks <= 8 (one NVSwitch node).
 * delta: device int64[2R-1]; bounds: device uint64[R+1].
 */
int bs_split_count(const void *keys, uint64_t n, int key_bytes, int width,
                   int key_kind, const void *splitters, int nranks,
                   uint64_t *class_counts, void *ws, size_t ws_bytes, void *stream);
int bs_split_exchange(const void *keys, const void *vals, uint64_t n,
                      int key_bytes, int val_bytes, int width, int key_kind,
                      const void *splitters, int nranks, const int64_t *delta,
                      const uint64_t *bounds, void *const *dst_keys,
                      void *const *dst_vals, void *ws, size_t ws_bytes,
                      void *stream);
/*
 * Peer-mapped receive buffers (CUDA IPC; one process per GPU on an
 * NVLink/NVSwitch node).  bs_ipc_alloc allocates `bytes` of device memory and
 * writes its export handle (bs_ipc_handle_bytes() bytes) to `handle`;
 * bs_ipc_open maps another process's handle (peer access enabled lazily);
 * bs_ipc_close unmaps; bs_ipc_free releases an allocation of this process.
 */
size_t bs_ipc_handle_bytes(void);
int bs_ipc_alloc(size_t bytes, void **ptr, void *handle);
int bs_ipc_open(const void *handle, void **ptr);
int bs_ipc_close(void *ptr);
int bs_ipc_free(void *ptr);
/*
 * Gather `count` uniformly strided samples of the encoded, normalised sort key
 * (device, key_bytes words) from keys[0..n): sample i is element
 * floor((2i+1)*n/(2*count)).
 */
int bs_sample_keys(const void *keys, uint64_t n, int key_bytes, int width,
                   int key_kind, uint64_t count, void *out_samples,
                   void *stream);

/* -------------------------------------------------------------------------
 * Exact reference-order engine.  Replays the reference recursion bit level
 * by bit level with the exact two-cursor permutation of every partition
 * (kernels.py:56-77), so the output -- including the
 * order of keys equal in the examined bits, and values carried alongside --
 * and the counters are the reference's own for every drive form:
 *
 *   mode 0  kernels.sort_words(arr, lo, up, start_pos, width, passthrough_loop,
 *           check_after, streak, checked, counters, depth)   (kernels.py:88-126)
 *           -- core.sort / variants.sort_optimized / binar_sort_range
 *   mode 1  kernels.sort_words_iterative(arr, lo, up, width, counters)
 *           (kernels.py:129-172; max_depth = stack high-water mark)
 *   mode 2  core._sort_levels (core.py:146-180): a sortedness scan before every
 *           partition, one call per partition; `on_level` is called after each
 *           level's kernels are enqueued (sort_with_observer)
 *   mode 3  variants.sort_parallel (variants.py:162-229): `par_levels` levels
 *           of _prepartition, then sort_words per bucket from pos=par_levels
 *
 * The sort key is (enc(x) << pos) & (1 << (width-1)) with enc the key_kind
 * transform of the raw word; sortedness scans compare whole encoded words,
 * like range_sorted_words (kernels.py:80-85).  counters (device int64[4], may
 * be NULL) is overwritten.  n < 2^32 - 1.  Slower than bs_sort (width passes
 * of ~40 bytes per element instead of ~4 digit passes): bs_sort is the
 * product path wherever the tie order cannot be observed.
 * ------------------------------------------------------------------------- */
typedef void (*bs_level_fn)(void *ctx, int pos);
size_t bs_exact_workspace_bytes(uint64_t n, int key_bytes, int val_bytes);
int bs_exact_sort(void *keys, void *vals, uint64_t n, int key_bytes, int val_bytes,
                  int width, int start_pos, int key_kind, int mode,
                  int passthrough_loop, int check_after, int streak, int checked,
                  int par_levels, int64_t depth, void *ws, size_t ws_bytes,
                  void *stream, int64_t *counters, bs_level_fn on_level, void *ctx);
/*
 * Start positions (ascending, relative to keys) of the engine's current
 * segments -- the reference observer's (lower, upper) list (core.py:175-180)
 * -- written to starts (device uint32[n]); their number to *count (device).
 * Call from on_level (same ws, n, key_bytes, val_bytes, stream).
 */
int bs_exact_boundaries(const void *ws, uint64_t n, int key_bytes, int val_bytes,
                        uint32_t *starts, uint32_t *count, void *stream);
/*
 * The array's current contents after `levels_done` levels -- what the
 * reference observer reads from the partially sorted sequence between levels
 * (core.py:175-180; cli.py:160-185 prints them) -- gathered into out_keys
 * (device, n words).  Call from on_level with the same keys/ws/n/widths.
 */
int bs_exact_snapshot(const void *keys, const void *ws, uint64_t n, int key_bytes, int val_bytes,
                      int levels_done, void *out_keys, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* BINARSORT_B200_H */
