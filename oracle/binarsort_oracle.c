/*
 * oracle/binarsort_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference Binar Sort word kernels, used as the
 * CPU checker for the CUDA product path and as the CPU baseline in bench.py
 * (cpu_baseline kind "port").  Nothing in paper_0811_3448_b200/ links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do.
 *
 * Every function follows the reference numba kernels line by line
 * (/root/reference/pkg/src/binarsort/kernels.py) so that outputs AND the
 * four-slot counter array {extractions, swaps, calls, max_depth} match the
 * reference exactly (pinned against tests/golden/, generated from the
 * reference itself by tests/golden/make_golden.py).
 *
 * Word types: u32 and u64 arrays (the reference's numba kernels are
 * instantiated for both dtypes).  Bit extraction is `(u64(x) << pos) & msb`
 * with msb = 1 << (width-1), exactly kernels.py:63,69.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define EXTRACTIONS 0
#define SWAPS 1
#define CALLS 2
#define MAX_DEPTH 3

/* ---------------------------------------------------------------------------
 * partition_words -- kernels.py:56-77.  Two-cursor in-place partition of
 * arr[lower..upper] on bit `pos`; returns the split index.
 * ------------------------------------------------------------------------- */
#define DEF_PARTITION(T, SUF)                                                   \
int64_t or_partition_words_##SUF(T *arr, int64_t lower, int64_t upper,          \
                                 int64_t pos, int64_t width, int64_t *counters) \
{                                                                               \
    const uint64_t msb = (uint64_t)1 << (uint64_t)(width - 1);                  \
    const uint64_t shift = (uint64_t)pos;                                       \
    int64_t lo = lower, hi = upper;                                             \
    int64_t ext = 0, sw = 0;                                                    \
    while (lo < hi + 1) {                                                       \
        ext++;                                                                  \
        if (((uint64_t)arr[lo] << shift) & msb) {                               \
            T tmp = arr[hi];                                                    \
            arr[hi] = arr[lo];                                                  \
            arr[lo] = tmp;                                                      \
            sw++;                                                               \
            hi--;                                                               \
        } else {                                                                \
            lo++;                                                               \
        }                                                                       \
    }                                                                           \
    counters[EXTRACTIONS] += ext;                                               \
    counters[SWAPS] += sw;                                                      \
    return lo;                                                                  \
}

/* range_sorted_words -- kernels.py:80-85. */
#define DEF_RANGE_SORTED(T, SUF)                                                \
int or_range_sorted_words_##SUF(const T *arr, int64_t lower, int64_t upper)    \
{                                                                               \
    for (int64_t i = lower; i < upper; i++)                                     \
        if (arr[i] > arr[i + 1]) return 0;                                      \
    return 1;                                                                   \
}

/* sort_words -- kernels.py:88-126 (recursive dispatch, pass-through loop,
 * sortedness check after `check_after` consecutive pass-throughs). */
#define DEF_SORT(T, SUF)                                                        \
void or_sort_words_##SUF(T *arr, int64_t lower, int64_t upper, int64_t pos,     \
                         int64_t width, int passthrough_loop,                  \
                         int64_t check_after, int64_t streak, int checked,      \
                         int64_t *counters, int64_t depth)                      \
{                                                                               \
    counters[CALLS] += 1;                                                       \
    if (depth > counters[MAX_DEPTH]) counters[MAX_DEPTH] = depth;               \
    for (;;) {                                                                  \
        if (pos == width || upper < lower + 1) return;                          \
        int64_t split = or_partition_words_##SUF(arr, lower, upper, pos,        \
                                                 width, counters);              \
        if (split == lower || split == upper + 1) {                             \
            streak += 1;                                                        \
            if (check_after > 0 && streak >= check_after && !checked) {         \
                checked = 1;                                                    \
                if (or_range_sorted_words_##SUF(arr, lower, upper)) return;     \
            }                                                                   \
            if (passthrough_loop) { pos += 1; continue; }                       \
            or_sort_words_##SUF(arr, lower, upper, pos + 1, width,              \
                                passthrough_loop, check_after, streak, checked, \
                                counters, depth + 1);                           \
            return;                                                             \
        }                                                                       \
        or_sort_words_##SUF(arr, lower, split - 1, pos + 1, width,              \
                            passthrough_loop, check_after, 0, 0, counters,      \
                            depth + 1);                                         \
        or_sort_words_##SUF(arr, split, upper, pos + 1, width,                  \
                            passthrough_loop, check_after, 0, 0, counters,      \
                            depth + 1);                                         \
        return;                                                                 \
    }                                                                           \
}

/* sort_words_iterative -- kernels.py:129-172 (explicit stack, lower side
 * popped first; counters[3] = stack high-water mark). */
#define DEF_SORT_ITER(T, SUF)                                                   \
void or_sort_words_iterative_##SUF(T *arr, int64_t lower, int64_t upper,        \
                                   int64_t width, int64_t *counters)            \
{                                                                               \
    int64_t cap = 2 * (width + 1) + 2;                                          \
    int64_t (*stack)[3] = malloc(sizeof(int64_t[3]) * (size_t)cap);             \
    stack[0][0] = lower; stack[0][1] = upper; stack[0][2] = 0;                  \
    int64_t top = 1, high_water = 1;                                            \
    while (top > 0) {                                                           \
        top -= 1;                                                               \
        int64_t lo_ = stack[top][0], up_ = stack[top][1], pos = stack[top][2];  \
        counters[CALLS] += 1;                                                   \
        int64_t split = or_partition_words_##SUF(arr, lo_, up_, pos, width,     \
                                                 counters);                     \
        if (pos + 1 == width) continue;                                         \
        if (split == lo_ || split == up_ + 1) {                                 \
            stack[top][0] = lo_; stack[top][1] = up_; stack[top][2] = pos + 1;  \
            top += 1;                                                           \
        } else {                                                                \
            if (up_ > split) {                                                  \
                stack[top][0] = split; stack[top][1] = up_;                     \
                stack[top][2] = pos + 1; top += 1;                              \
            }                                                                   \
            if (split - 1 > lo_) {                                              \
                stack[top][0] = lo_; stack[top][1] = split - 1;                 \
                stack[top][2] = pos + 1; top += 1;                              \
            }                                                                   \
        }                                                                       \
        if (top > high_water) high_water = top;                                 \
    }                                                                           \
    if (high_water > counters[MAX_DEPTH]) counters[MAX_DEPTH] = high_water;     \
    free(stack);                                                                \
}

DEF_PARTITION(uint32_t, u32)
DEF_PARTITION(uint64_t, u64)
DEF_RANGE_SORTED(uint32_t, u32)
DEF_RANGE_SORTED(uint64_t, u64)
DEF_SORT(uint32_t, u32)
DEF_SORT(uint64_t, u64)
DEF_SORT_ITER(uint32_t, u32)
DEF_SORT_ITER(uint64_t, u64)

/* ---------------------------------------------------------------------------
 * sort_parallel -- variants.py:162-229, word path (variants.py:184-209).
 * Sequential level-synchronous pre-partition of the top `levels` bits
 * (_prepartition, variants.py:124-148), then a pool of `workers` threads sorts
 * the disjoint buckets with sort_words(.., pos=levels, .., depth=levels+1).
 * Buckets are handed out in order from a shared cursor (ThreadPoolExecutor.map
 * semantics).  `metrics` receives {extractions, swaps, calls, max_depth} with
 * Metrics.merge semantics (core.py:60-77).
 * ------------------------------------------------------------------------- */
typedef struct {
    void *arr;
    int is64;
    int64_t width, levels;
    int64_t (*ranges)[2];
    int64_t nranges;
    int64_t next;            /* shared cursor, guarded by mu */
    pthread_mutex_t mu;
    int64_t *bucket_counters; /* nranges x 4 */
} par_job_t;

static void *par_worker(void *p)
{
    par_job_t *job = (par_job_t *)p;
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int64_t i = job->next++;
        pthread_mutex_unlock(&job->mu);
        if (i >= job->nranges) break;
        int64_t *c = job->bucket_counters + 4 * i;
        if (job->is64)
            or_sort_words_u64((uint64_t *)job->arr, job->ranges[i][0], job->ranges[i][1],
                              job->levels, job->width, 0, 0, 0, 0, c, job->levels + 1);
        else
            or_sort_words_u32((uint32_t *)job->arr, job->ranges[i][0], job->ranges[i][1],
                              job->levels, job->width, 0, 0, 0, 0, c, job->levels + 1);
    }
    return NULL;
}

static int bit_length(int64_t v)
{
    int b = 0;
    while (v > 0) { b++; v >>= 1; }
    return b;
}

int or_sort_parallel(void *arr, int is64, int64_t n, int64_t width,
                     int64_t workers, int64_t *metrics)
{
    memset(metrics, 0, 4 * sizeof(int64_t));
    if (workers < 1) return -1;
    if (n <= 1 || width == 0) return 0;
    int64_t levels = bit_length(workers - 1);
    if (levels > width) levels = width;
    /* _prepartition */
    int64_t cap = (int64_t)1 << levels;
    int64_t (*ranges)[2] = malloc(sizeof(int64_t[2]) * (size_t)(cap + 1));
    int64_t (*nxt)[2] = malloc(sizeof(int64_t[2]) * (size_t)(cap + 1));
    int64_t nr = 1;
    ranges[0][0] = 0; ranges[0][1] = n - 1;
    int64_t pre[4] = {0, 0, 0, 0};
    for (int64_t pos = 0; pos < levels; pos++) {
        int64_t nn = 0;
        for (int64_t r = 0; r < nr; r++) {
            int64_t lo = ranges[r][0], up = ranges[r][1];
            if (up <= lo) { nxt[nn][0] = lo; nxt[nn][1] = up; nn++; continue; }
            metrics[CALLS] += 1;
            int64_t split = is64
                ? or_partition_words_u64((uint64_t *)arr, lo, up, pos, width, pre)
                : or_partition_words_u32((uint32_t *)arr, lo, up, pos, width, pre);
            if (split == lo || split == up + 1) {
                nxt[nn][0] = lo; nxt[nn][1] = up; nn++;
            } else {
                nxt[nn][0] = lo; nxt[nn][1] = split - 1; nn++;
                nxt[nn][0] = split; nxt[nn][1] = up; nn++;
            }
        }
        memcpy(ranges, nxt, sizeof(int64_t[2]) * (size_t)nn);
        nr = nn;
        if (pos + 1 > metrics[MAX_DEPTH]) metrics[MAX_DEPTH] = pos + 1;
    }
    metrics[EXTRACTIONS] += pre[EXTRACTIONS];
    metrics[SWAPS] += pre[SWAPS];
    /* work = buckets with more than one element */
    int64_t nw = 0;
    for (int64_t r = 0; r < nr; r++)
        if (ranges[r][1] > ranges[r][0]) { nxt[nw][0] = ranges[r][0]; nxt[nw][1] = ranges[r][1]; nw++; }
    par_job_t job;
    job.arr = arr; job.is64 = is64; job.width = width; job.levels = levels;
    job.ranges = nxt; job.nranges = nw; job.next = 0;
    pthread_mutex_init(&job.mu, NULL);
    job.bucket_counters = calloc((size_t)(4 * (nw > 0 ? nw : 1)), sizeof(int64_t));
    int64_t nthreads = (workers == 1 || nw <= 1) ? 1 : (workers < nw ? workers : nw);
    if (nthreads == 1) {
        par_worker(&job);
    } else {
        pthread_t *th = malloc(sizeof(pthread_t) * (size_t)nthreads);
        for (int64_t t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, par_worker, &job);
        for (int64_t t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
        free(th);
    }
    for (int64_t i = 0; i < nw; i++) {
        int64_t *c = job.bucket_counters + 4 * i;
        metrics[EXTRACTIONS] += c[EXTRACTIONS];
        metrics[SWAPS] += c[SWAPS];
        metrics[CALLS] += c[CALLS];
        if (c[MAX_DEPTH] > metrics[MAX_DEPTH]) metrics[MAX_DEPTH] = c[MAX_DEPTH];
    }
    pthread_mutex_destroy(&job.mu);
    free(job.bucket_counters);
    free(ranges);
    free(nxt);
    return 0;
}
