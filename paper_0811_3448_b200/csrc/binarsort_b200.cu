// binarsort_b200.cu -- host side of the C ABI declared in include/binarsort_b200.h.
//
// Launch sequence of bs_sort (all on the caller's stream, no host sync):
//   memset(ctl) ; init ; for L in 0..ndig: { hist(L) ; plan(L) ; scatter(L) } ;
//   local ; [metrics]
// Levels that have no buckets exit immediately on the device.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/binarsort_b200.h"
#include "metrics_impl.cuh"
#include "misc_impl.cuh"
#include "sort_impl.cuh"
#include "dense_impl.cuh"
#include "exact_impl.cuh"
#include "spread_impl.cuh"

namespace bs {

static thread_local std::string g_err;

// Optional phase events (bs_sort_profiled): thread-local, set for one call.
static thread_local cudaEvent_t *t_ev = nullptr;
static thread_local int t_nev = 0, t_iev = 0;
static inline void mark(cudaStream_t st) {
  if (t_ev && t_iev < t_nev) cudaEventRecord(t_ev[t_iev++], st);
}

static int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define BS_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(BS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// Launch with programmatic stream serialisation: the kernel may be scheduled
// while its predecessor in the stream drains (every kernel of the sort starts
// with pdl_wait()), hiding most of the launch gap between dependent kernels.
template <typename... KArgs, typename... Args>
static cudaError_t pdl_launch(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Per-device one-time setup (function attributes, grid sizes) is keyed by the
// current device, so one process may sort on several GPUs.
constexpr int MAX_DEV = 64;

static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < MAX_DEV ? dev : 0;
}

static int num_sms() {
  static int sms[MAX_DEV] = {};
  static std::once_flag once[MAX_DEV];
  const int dev = current_device();
  std::call_once(once[dev], [dev] {
    cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    if (sms[dev] <= 0) sms[dev] = 148;
  });
  return sms[dev];
}

// ----- tuning (per record width) --------------------------------------------
// Scatter tiles and local-sort capacity by record bytes (key + value):
//   4 B  (u32 keys):              tile 512x22 = 11264 (per-tile barriers, scan and digit atomics amortised over
//                                 more keys, 176-byte runs; 23+ keys per thread spill), local 512x16 = 8192
//   8-12 B (u64 keys, KV):         tile 256x16 = 4096 (KV: 256x14, 3 CTAs/SM), local 512x16 = 8192 (u64 keys only: 512x9 = 4608, 2 CTAs/SM)
//   16 B (u64 keys + u64 values):  tile 256x16 = 4096, local 512x8  = 4096
// (local capacity is bounded by two TMA input buffers in 227 KB of smem)
struct Tune {
  int sc_block, sc_kpt, lc_block, lc_kpt;
};
//   8 B keys only: local 512x9, two CTAs per SM (one task's barriers hide behind the other's work: cfg3-zipf 6.95 -> 6.45 ms)
constexpr Tune tune_for(int kb, int vb) {
  return (kb + vb) <= 4   ? Tune{512, 22, 512, 16}
         : vb == 0        ? Tune{256, 16, 512, 9}
         : (kb + vb) < 16 ? Tune{256, 14, 512, 16}
                          : Tune{256, 16, 512, 8};
}

struct Geometry {
  uint64_t n;
  int kb, vb;
  uint32_t tile, local_max, group_min;
  uint32_t maxb, maxtiles, maxtasks;
  int ndig;
};

// bs_debug_capacity: thread-local caps on the work lists (0 = none)
static thread_local uint32_t t_cap_b = 0, t_cap_t = 0, t_cap_k = 0;

static Geometry geometry(uint64_t n, int kb, int vb, int width_eff) {
  Geometry g{};
  g.n = n;
  g.kb = kb;
  g.vb = vb;
  const Tune tn = tune_for(kb, vb);
  g.tile = uint32_t(tn.sc_block * tn.sc_kpt);
  g.local_max = uint32_t(tn.lc_block * tn.lc_kpt);
  g.group_min = g.local_max / 8;
  g.ndig = (width_eff + 7) / 8;
  const uint64_t maxb = n / (uint64_t(g.local_max) + 1) + 2;
  const uint64_t maxtiles = n / g.tile + maxb + 2;
  const uint64_t maxtasks = 3 * n / g.group_min + n / g.local_max + uint64_t(g.ndig + 2) * maxb + 1024;
  g.maxb = uint32_t(maxb);
  g.maxtiles = uint32_t(maxtiles);
  g.maxtasks = uint32_t(maxtasks);
  return g;
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t ctl, buckets[2], bhist[2], bor[2], band[2], tile_bucket[2], status, toff, hist16, h16part, tasks, tasks2, dtasks,
      keys, vals, total;
};

static Layout layout(const Geometry &g, bool own_copy = true) {
  Layout l{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align_up(bytes);
    return o;
  };
  l.ctl = take(sizeof(Ctl));
  for (int p = 0; p < 2; ++p) {
    l.buckets[p] = take(sizeof(Bucket) * g.maxb);
    l.bhist[p] = take(sizeof(uint32_t) * 256 * size_t(g.maxb));
    l.bor[p] = take(sizeof(uint64_t) * g.maxb);
    l.band[p] = take(sizeof(uint64_t) * g.maxb);
    l.tile_bucket[p] = take(sizeof(uint32_t) * g.maxtiles);
  }
  l.status = take(sizeof(uint32_t) * 256 * size_t(g.maxtiles));
  l.toff = take(g.vb ? sizeof(uint32_t) * 256 * size_t(g.maxtiles) : 0);
  l.hist16 = take(sizeof(uint32_t) * 65536);
  l.h16part = take(sizeof(uint32_t) * 32768 * size_t(H16_MAXCTA));
  l.tasks = take(sizeof(Task) * g.maxtasks);
  l.tasks2 = take(g.vb == 0 && g.kb == 8 ? sizeof(Task) * g.maxtasks : 0);
  l.dtasks = take(g.vb == 0 ? sizeof(DTask) * g.maxtasks : 0);
  // the ping-pong copy (bs_sort_from uses the caller's source buffer instead)
  l.keys = take(own_copy ? size_t(g.kb) * g.n : 0);
  l.vals = take(own_copy ? size_t(g.vb) * g.n : 0);
  l.total = off;
  return l;
}

template <typename F>
static int max_active(F kernel, int block, size_t smem) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, block, smem);
  return nb > 0 ? nb : 1;
}

template <typename K, int VB, int KIND>
static int run_sort(void *keys, void *vals, uint64_t n, int width_eff, void *wsp, size_t ws_bytes,
                    cudaStream_t st, void *src_keys = nullptr, void *src_vals = nullptr) {
  const int kb = int(sizeof(K));
  Geometry geo = geometry(n, kb, VB, width_eff);
  const Layout lay = layout(geo, src_keys == nullptr);
  // test caps shrink the lists inside an unchanged layout (the flag reports it)
  if (t_cap_b) geo.maxb = geo.maxb < t_cap_b ? geo.maxb : t_cap_b;
  if (t_cap_t) geo.maxtiles = geo.maxtiles < t_cap_t ? geo.maxtiles : t_cap_t;
  if (t_cap_k) geo.maxtasks = geo.maxtasks < t_cap_k ? geo.maxtasks : t_cap_k;
  if (ws_bytes < lay.total)
    return fail(BS_ERR_WORKSPACE, "workspace too small: need " + std::to_string(lay.total) +
                                      " bytes, got " + std::to_string(ws_bytes));
  char *base = static_cast<char *>(wsp);
  Ws ws{};
  ws.ctl = reinterpret_cast<Ctl *>(base + lay.ctl);
  for (int p = 0; p < 2; ++p) {
    ws.buckets[p] = reinterpret_cast<Bucket *>(base + lay.buckets[p]);
    ws.bhist[p] = reinterpret_cast<uint32_t *>(base + lay.bhist[p]);
    ws.bor[p] = reinterpret_cast<uint64_t *>(base + lay.bor[p]);
    ws.band[p] = reinterpret_cast<uint64_t *>(base + lay.band[p]);
    ws.tile_bucket[p] = reinterpret_cast<uint32_t *>(base + lay.tile_bucket[p]);
  }
  ws.status = reinterpret_cast<uint32_t *>(base + lay.status);
  ws.toff = reinterpret_cast<uint32_t *>(base + lay.toff);
  ws.hist16 = reinterpret_cast<uint32_t *>(base + lay.hist16);
  ws.h16part = reinterpret_cast<uint32_t *>(base + lay.h16part);
  ws.tasks = reinterpret_cast<Task *>(base + lay.tasks);
  ws.tasks2 = reinterpret_cast<Task *>(base + lay.tasks2);
  ws.dtasks = reinterpret_cast<DTask *>(base + lay.dtasks);
  ws.keys[0] = keys;
  ws.keys[1] = src_keys ? src_keys : base + lay.keys;
  ws.vals[0] = vals;
  ws.vals[1] = VB ? (src_keys ? src_vals : base + lay.vals) : nullptr;
  ws.root_parity = src_keys ? 1u : 0u;
  ws.n = n;
  ws.maxb = geo.maxb;
  ws.maxtiles = geo.maxtiles;
  ws.maxtasks = geo.maxtasks;
  ws.tile = geo.tile;
  ws.local_max = geo.local_max;
  ws.group_min = geo.group_min;
  ws.ndig = geo.ndig;
  ws.shift0 = int(sizeof(K) * 8) - width_eff;
  ws.kbits = int(sizeof(K) * 8);
  ws.stable = VB != 0;
  ws.dense = (VB == 0 && width_eff == int(sizeof(K) * 8)) ? 1 : 0;

  constexpr Tune TN = tune_for(int(sizeof(K)), VB);
  constexpr int SC_BLOCK = TN.sc_block, SKPT = TN.sc_kpt, LC_BLOCK = TN.lc_block, LC_KPT = TN.lc_kpt;
  constexpr int HI_BLOCK = SC_BLOCK, HKPT = SKPT;  // histogram tiles == scatter tiles
  using SS = ScatterSmem<K, VB, KIND, SC_BLOCK, SKPT>;
  // keys-only scatter ring: two tile slots (4-byte keys: 2 x 44 KB, 2 CTAs/SM; a third slot of 8192-key
  // tiles measured 0.605 ms per cfg2 pass, two slots of 11264-key tiles 0.580 ms)
  constexpr int SC_NBUF = 2;
  using SW = ScatterWsSmem<K, KIND, SC_BLOCK, SKPT, SC_NBUF>;
  using LS = LocalSmem<K, VB, KIND, LC_BLOCK, LC_KPT>;
  constexpr bool WSPEC = VB == 0;  // keys-only: warp-specialised scatter
  auto sc = scatter_kernel<K, VB, KIND, SC_BLOCK, SKPT>;
  auto sw = scatter_ws_kernel<K, KIND, SC_BLOCK, SKPT, SC_NBUF>;
  // dense local sort (bitmap enumeration): small tasks 256 consumers, 4608
  // keys, 2-slot ring (4 CTAs/SM); big variant (u32 only) 512 consumers,
  // 18432-key tasks (e.g. 2^30-key inputs), one slot, 2 CTAs/SM
    constexpr int DN_BLOCK = 256, DN_CAP = 4608, DN_SLOTS = 2;
  constexpr int DB_BLOCK = 512, DB_CAP = sizeof(K) == 4 ? 18432 : 6144, DB_SLOTS = 1;
  using DS = DenseSmem<K, DN_BLOCK, DN_CAP, DN_SLOTS, false>;
  using DB = DenseSmem<K, DB_BLOCK, DB_CAP, DB_SLOTS, true>;
  auto dk = dense_kernel<K, KIND, DN_BLOCK, DN_CAP, DN_SLOTS, false>;
  auto db = dense_kernel<K, KIND, DB_BLOCK, DB_CAP, DB_SLOTS, true>;
  ws.dense_max = DN_CAP;
  ws.dense_big_max = sizeof(K) == 4 ? DB_CAP : 0;
  auto lc = local_kernel<K, VB, KIND, LC_BLOCK, LC_KPT>;
  // keys-only 64-bit: spread tasks go to spread_kernel first (1024 x 8 = local_max)
  constexpr bool SPREAD = VB == 0 && sizeof(K) == 8;
  // 512 x 9 = 4608-key slots (~107 KB): two CTAs per SM, so one task's barriers hide behind the
  // other's work; local tasks larger than a slot stay on local_kernel
  constexpr int SP_BLOCK = 512, SP_KPT = 9;
  static_assert(!SPREAD || SP_BLOCK * SP_KPT <= LC_BLOCK * LC_KPT, "spread tasks are local tasks");
  using SPS = SpreadSmem<K, SP_BLOCK, SP_KPT>;
  auto sp = spread_kernel<K, KIND, SP_BLOCK, SP_KPT>;
  auto hk = hist_kernel<K, KIND, HI_BLOCK, HKPT>;
  constexpr int H16_BLOCK = 1024;
  constexpr size_t H16_SMEM = 32768 * sizeof(uint32_t);
  auto h16 = hist16_kernel<K, KIND, H16_BLOCK>;
  struct Setup {
    int sc_grid, lc_grid, hk_grid, dk_grid, db_grid, sp_grid;
    cudaError_t attr_err;
  };
  static Setup setup[MAX_DEV];
  static std::once_flag once[MAX_DEV];
  const int dev = current_device();
  int &sc_grid = setup[dev].sc_grid, &lc_grid = setup[dev].lc_grid, &hk_grid = setup[dev].hk_grid,
      &dk_grid = setup[dev].dk_grid, &db_grid = setup[dev].db_grid, &sp_grid = setup[dev].sp_grid;
  cudaError_t &attr_err = setup[dev].attr_err;
  std::call_once(once[dev], [&] {
    cudaError_t e1 = cudaFuncSetAttribute(sc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SS::bytes));
    cudaError_t e2 = cudaFuncSetAttribute(lc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(LS::bytes));
    cudaError_t e3 = cudaFuncSetAttribute(sw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SW::bytes));
    cudaError_t e4 = VB == 0 ? cudaFuncSetAttribute(dk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(DS::bytes))
                             : cudaSuccess;
    if (VB == 0 && e4 == cudaSuccess)
      e4 = cudaFuncSetAttribute(db, cudaFuncAttributeMaxDynamicSharedMemorySize, int(DB::bytes));
    db_grid = VB == 0 ? num_sms() * max_active(db, DB_BLOCK + 32, DB::bytes) : 0;
    attr_err = e1 != cudaSuccess ? e1 : (e2 != cudaSuccess ? e2 : (e3 != cudaSuccess ? e3 : e4));
    dk_grid = VB == 0 ? num_sms() * max_active(dk, DN_BLOCK + 32, DS::bytes) : 0;
    sc_grid = WSPEC ? num_sms() * max_active(sw, SC_BLOCK + 32, SW::bytes)
                    : num_sms() * max_active(sc, SC_BLOCK, SS::bytes);
    lc_grid = num_sms() * max_active(lc, LC_BLOCK, LS::bytes);
    hk_grid = num_sms() * max_active(hk, HI_BLOCK, 0);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(h16, cudaFuncAttributeMaxDynamicSharedMemorySize, int(H16_SMEM));
    if (SPREAD && attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(sp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SPS::bytes));
    sp_grid = SPREAD ? num_sms() * max_active(sp, SP_BLOCK, SPS::bytes) : 0;
  });
  if (attr_err != cudaSuccess) return fail(BS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));

  mark(st);
  BS_CUDA(cudaMemsetAsync(ws.ctl, 0, sizeof(Ctl), st));
  {
    const uint32_t ntiles = uint32_t((n + geo.tile - 1) / geo.tile);
    const int g = int(min64((ntiles + 255) / 256 + 1, 4096));
    BS_CUDA(pdl_launch(init_kernel<K, KIND>, g, 256, 0, st, ws));
  }
  mark(st);
  if (n > geo.local_max) {
    const int nlev = geo.ndig + 1;
    for (int L = 0; L < nlev; ++L) {
      // keys-only: level 0 counts digit pairs (hist16), so level 1 needs no
      // histogram pass; stable sorts count per tile at every level instead
      if (L == 0 && VB == 0) {
        const int parts = num_sms() < H16_MAXCTA ? num_sms() : H16_MAXCTA;
        BS_CUDA(pdl_launch(h16, parts, H16_BLOCK, H16_SMEM, st, ws));
        BS_CUDA(pdl_launch(hist16_reduce_kernel, 32768 / 4 / 64, 256, 0, st, ws, parts));
      }
      else BS_CUDA(pdl_launch(hk, hk_grid, HI_BLOCK, 0, st, ws, L));
      mark(st);
      BS_CUDA(pdl_launch(plan_kernel<K>, num_sms() * 4, 256, 0, st, ws, L));
      if (L == 0 && VB == 0 && ws.dense)  // whole-input counting, when plan(0) chose it
        BS_CUDA(pdl_launch(gen16_kernel<K, KIND>, num_sms() * 8, 256, 0, st, ws));
      if constexpr (VB != 0) BS_CUDA(pdl_launch(tile_scan_kernel, num_sms() * 8, 256, 0, st, ws, L));
      mark(st);
      if constexpr (WSPEC) BS_CUDA(pdl_launch(sw, sc_grid, SC_BLOCK + 32, SW::bytes, st, ws, L));
      else BS_CUDA(pdl_launch(sc, sc_grid, SC_BLOCK, SS::bytes, st, ws, L));
      if constexpr (VB == 0) {
        // big dense children of this level (their data is in place now)
        if (ws.dense && ws.dense_big_max && L < nlev - 1)
          BS_CUDA(pdl_launch(db, db_grid, DB_BLOCK + 32, DB::bytes, st, ws, L));
      }
      BS_CUDA(pdl_launch(expand_kernel, num_sms() * 4, 256, 0, st, ws, L + 1));
      mark(st);
    }
  }
  if constexpr (VB == 0) {
    if (ws.dense) BS_CUDA(pdl_launch(dk, dk_grid, DN_BLOCK + 32, DS::bytes, st, ws, 0));
  }
  if constexpr (SPREAD) {
    BS_CUDA(pdl_launch(sp, sp_grid, SP_BLOCK, SPS::bytes, st, ws));
    BS_CUDA(pdl_launch(lc, lc_grid, LC_BLOCK, LS::bytes, st, ws, 1));
  } else {
    BS_CUDA(pdl_launch(lc, lc_grid, LC_BLOCK, LS::bytes, st, ws, 0));
  }
  mark(st);
  BS_CUDA(cudaGetLastError());
  return BS_OK;
}

template <typename K, int KIND>
static int run_metrics(const void *keys, uint64_t n, int width_eff, int64_t depth0, int64_t *counters,
                       cudaStream_t st) {
  if (n < 2) return BS_OK;
  constexpr int BLOCK = 256, IPT = 8;
  const uint64_t chunks = (n + BLOCK * IPT - 1) / (BLOCK * IPT);
  const int grid = int(min64(chunks, uint64_t(num_sms()) * 8));
  metrics_kernel<K, KIND, BLOCK, IPT><<<grid, BLOCK, 0, st>>>(
      static_cast<const K *>(keys), n, int(sizeof(K) * 8) - width_eff, width_eff, depth0,
      reinterpret_cast<unsigned long long *>(counters));
  metrics_root_kernel<<<1, 1, 0, st>>>(reinterpret_cast<unsigned long long *>(counters));
  BS_CUDA(cudaGetLastError());
  return BS_OK;
}

static int check_common(int key_bytes, int val_bytes, int width, int start_pos, int key_kind) {
  if (key_bytes != 4 && key_bytes != 8) return fail(BS_ERR_VALUE, "key_bytes must be 4 or 8");
  if (val_bytes != 0 && val_bytes != 4 && val_bytes != 8) return fail(BS_ERR_VALUE, "val_bytes must be 0, 4 or 8");
  if (width < 1 || width > key_bytes * 8)
    return fail(BS_ERR_VALUE, "unsupported word width " + std::to_string(width));
  if (start_pos < 0 || start_pos > width) return fail(BS_ERR_ASSERT, "bit position out of codec width");
  if (key_kind == BS_KEY_SIGNED && width < 2) return fail(BS_ERR_VALUE, "unsupported word width " + std::to_string(width));
  if (key_kind == BS_KEY_FLOAT && (key_bytes != 8 || width != 64))
    return fail(BS_ERR_VALUE, "float keys are 64-bit words of width 64");
  if (key_kind < 0 || key_kind > 2) return fail(BS_ERR_VALUE, "unknown key_kind");
  return BS_OK;
}

}  // namespace bs

using namespace bs;

extern "C" {

int bs_version(void) { return 200; }

int bs_debug_checks(void) {
#ifdef BS_DEBUG_CHECKS
  return 1;
#else
  return 0;
#endif
}

const char *bs_last_error(void) { return g_err.c_str(); }

size_t bs_workspace_bytes(uint64_t n, int key_bytes, int val_bytes) {
  if ((key_bytes != 4 && key_bytes != 8) || (val_bytes != 0 && val_bytes != 4 && val_bytes != 8)) return 0;
  return layout(geometry(n, key_bytes, val_bytes, key_bytes * 8)).total;
}

int bs_sort(void *keys, void *vals, uint64_t n, int key_bytes, int val_bytes, int width, int start_pos,
            int key_kind, void *ws, size_t ws_bytes, void *stream, int64_t *counters, int64_t depth) {
  int rc = check_common(key_bytes, val_bytes, width, start_pos, key_kind);
  if (rc) return rc;
  if (n >= (uint64_t(1) << 30) + 1) return fail(BS_ERR_VALUE, "n > 2^30 elements per call is not supported");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int width_eff = width - start_pos;
  // the sign bit lies above the effective key once start_pos > 0
  if (key_kind == BS_KEY_SIGNED && start_pos > 0) key_kind = BS_KEY_UNSIGNED;
  if (counters) BS_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(int64_t), st));
  if (n <= 1 || width_eff == 0) return BS_OK;  // nothing to move (core.py:207-212)
  if (val_bytes != 0 && vals == nullptr) return fail(BS_ERR_VALUE, "val_bytes > 0 but vals is NULL");
  if (val_bytes == 0) vals = nullptr;
#define BS_DISPATCH_V(K, KIND)                                                                  \
  do {                                                                                          \
    if (val_bytes == 0) rc = run_sort<K, 0, KIND>(keys, vals, n, width_eff, ws, ws_bytes, st);  \
    else if (val_bytes == 4) rc = run_sort<K, 4, KIND>(keys, vals, n, width_eff, ws, ws_bytes, st); \
    else rc = run_sort<K, 8, KIND>(keys, vals, n, width_eff, ws, ws_bytes, st);                 \
  } while (0)
  if (key_bytes == 4) {
    if (key_kind == BS_KEY_UNSIGNED) BS_DISPATCH_V(uint32_t, 0);
    else BS_DISPATCH_V(uint32_t, 1);
  } else {
    if (key_kind == BS_KEY_UNSIGNED) BS_DISPATCH_V(uint64_t, 0);
    else if (key_kind == BS_KEY_SIGNED) BS_DISPATCH_V(uint64_t, 1);
    else BS_DISPATCH_V(uint64_t, 2);
  }
#undef BS_DISPATCH_V
  if (rc) return rc;
  if (counters) return bs_metrics(keys, n, key_bytes, width, start_pos, key_kind, depth, nullptr, 0, stream, counters);
  return BS_OK;
}

int bs_sort_status(const void *ws, int32_t *status, void *stream) {
  if (!ws || !status) return fail(BS_ERR_VALUE, "ws and status must be non-NULL");
  // Ctl sits at offset 0 of every sort workspace (layout())
  const char *flag = static_cast<const char *>(ws) + offsetof(Ctl, error);
  BS_CUDA(cudaMemcpyAsync(status, flag, sizeof(int32_t), cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return BS_OK;
}

size_t bs_sort_status_offset(void) { return offsetof(Ctl, error); }

void bs_debug_capacity(uint32_t max_buckets, uint32_t max_tiles, uint32_t max_tasks) {
  t_cap_b = max_buckets;
  t_cap_t = max_tiles;
  t_cap_k = max_tasks;
}

size_t bs_sort_from_workspace_bytes(uint64_t n, int key_bytes, int val_bytes) {
  if ((key_bytes != 4 && key_bytes != 8) || (val_bytes != 0 && val_bytes != 4 && val_bytes != 8)) return 0;
  return layout(geometry(n, key_bytes, val_bytes, key_bytes * 8), false).total;
}

int bs_sort_from(void *src_keys, void *src_vals, void *keys, void *vals, uint64_t n, int key_bytes, int val_bytes,
                 int width, int start_pos, int key_kind, void *ws, size_t ws_bytes, void *stream) {
  int rc = check_common(key_bytes, val_bytes, width, start_pos, key_kind);
  if (rc) return rc;
  if (n >= (uint64_t(1) << 30) + 1) return fail(BS_ERR_VALUE, "n > 2^30 elements per call is not supported");
  if (n > 0 && (src_keys == nullptr || keys == nullptr)) return fail(BS_ERR_VALUE, "NULL key buffer");
  if (val_bytes != 0 && n > 0 && (src_vals == nullptr || vals == nullptr))
    return fail(BS_ERR_VALUE, "val_bytes > 0 but a value buffer is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int width_eff = width - start_pos;
  if (key_kind == BS_KEY_SIGNED && start_pos > 0) key_kind = BS_KEY_UNSIGNED;
  if (n <= 1 || width_eff == 0) {  // nothing to order: the result is the source
    if (n) BS_CUDA(cudaMemcpyAsync(keys, src_keys, n * key_bytes, cudaMemcpyDeviceToDevice, st));
    if (n && val_bytes) BS_CUDA(cudaMemcpyAsync(vals, src_vals, n * val_bytes, cudaMemcpyDeviceToDevice, st));
    return BS_OK;
  }
  if (val_bytes == 0) vals = src_vals = nullptr;
#define BS_DISPATCH_F(K, KIND)                                                                             \
  do {                                                                                                     \
    if (val_bytes == 0) rc = run_sort<K, 0, KIND>(keys, vals, n, width_eff, ws, ws_bytes, st, src_keys, src_vals); \
    else if (val_bytes == 4) rc = run_sort<K, 4, KIND>(keys, vals, n, width_eff, ws, ws_bytes, st, src_keys, src_vals); \
    else rc = run_sort<K, 8, KIND>(keys, vals, n, width_eff, ws, ws_bytes, st, src_keys, src_vals);      \
  } while (0)
  if (key_bytes == 4) {
    if (key_kind == BS_KEY_UNSIGNED) BS_DISPATCH_F(uint32_t, 0);
    else BS_DISPATCH_F(uint32_t, 1);
  } else {
    if (key_kind == BS_KEY_UNSIGNED) BS_DISPATCH_F(uint64_t, 0);
    else if (key_kind == BS_KEY_SIGNED) BS_DISPATCH_F(uint64_t, 1);
    else BS_DISPATCH_F(uint64_t, 2);
  }
#undef BS_DISPATCH_F
  return rc;
}

int bs_sort_profiled(void *keys, void *vals, uint64_t n, int key_bytes, int val_bytes, int width, int start_pos,
                     int key_kind, void *ws, size_t ws_bytes, void *stream, int64_t *counters, int64_t depth,
                     float *phase_ms, int nphases, int *nrecorded) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nev = nphases + 1;
  cudaEvent_t evs[64];
  if (nev > 64 || nphases < 1) return fail(BS_ERR_VALUE, "nphases must be in [1, 63]");
  for (int i = 0; i < nev; ++i) BS_CUDA(cudaEventCreate(&evs[i]));
  t_ev = evs;
  t_nev = nev;
  t_iev = 0;
  const int rc = bs_sort(keys, vals, n, key_bytes, val_bytes, width, start_pos, key_kind, ws, ws_bytes, stream,
                         counters, depth);
  const int rec = t_iev;
  t_ev = nullptr;
  t_nev = t_iev = 0;
  if (rc == BS_OK) {
    BS_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i + 1 < rec; ++i) BS_CUDA(cudaEventElapsedTime(&phase_ms[i], evs[i], evs[i + 1]));
  }
  for (int i = 0; i < nev; ++i) cudaEventDestroy(evs[i]);
  if (nrecorded) *nrecorded = rec > 0 ? rec - 1 : 0;
  return rc;
}

int bs_sort_launches(uint64_t n, int key_bytes, int width, int start_pos, int with_counters) {
  const int width_eff = width - start_pos;
  if (n <= 1 || width_eff <= 0) return 0;
  const Geometry g = geometry(n, key_bytes, 0, width_eff);
  int k = 3 + (key_bytes == 8 ? 1 : 0);  // init + dense + local (+ spread for 64-bit keys)
  // per level hist/plan/scatter/expand (+ big dense), + the level-0 hist16 reduce and gen16
  if (n > g.local_max) k += 4 * (g.ndig + 1) + (key_bytes == 4 ? g.ndig : 0) + 1 + (width_eff == key_bytes * 8 ? 1 : 0);
  if (with_counters) k += 2;
  return k;
}

size_t bs_metrics_workspace_bytes(uint64_t) { return 0; }

int bs_metrics(const void *sorted_keys, uint64_t n, int key_bytes, int width, int start_pos, int key_kind,
               int64_t depth, void *, size_t, void *stream, int64_t *counters) {
  int rc = check_common(key_bytes, 0, width, start_pos, key_kind);
  if (rc) return rc;
  if (!counters) return fail(BS_ERR_VALUE, "counters is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int width_eff = width - start_pos;
  if (key_kind == BS_KEY_SIGNED && start_pos > 0) key_kind = BS_KEY_UNSIGNED;
  if (n < 2 || width_eff == 0) return BS_OK;
  if (key_bytes == 4) {
    if (key_kind == BS_KEY_UNSIGNED) return run_metrics<uint32_t, 0>(sorted_keys, n, width_eff, depth, counters, st);
    return run_metrics<uint32_t, 1>(sorted_keys, n, width_eff, depth, counters, st);
  }
  if (key_kind == BS_KEY_UNSIGNED) return run_metrics<uint64_t, 0>(sorted_keys, n, width_eff, depth, counters, st);
  if (key_kind == BS_KEY_SIGNED) return run_metrics<uint64_t, 1>(sorted_keys, n, width_eff, depth, counters, st);
  return run_metrics<uint64_t, 2>(sorted_keys, n, width_eff, depth, counters, st);
}

size_t bs_partition_workspace_bytes(uint64_t n, int key_bytes, int val_bytes) {
  const uint64_t nblk = (n + PART_CHUNK - 1) / PART_CHUNK;
  return align_up(size_t(key_bytes) * n) + align_up(size_t(val_bytes) * n) +
         2 * align_up(sizeof(uint32_t) * (n + 1)) + align_up(sizeof(uint32_t) * (nblk + 1)) + 256;
}

int bs_partition_words(void *keys, void *vals, uint64_t n, int key_bytes, int val_bytes, int width, int pos,
                       void *ws, size_t ws_bytes, void *stream, int64_t *split_dev, int64_t *counters) {
  if (key_bytes != 4 && key_bytes != 8) return fail(BS_ERR_VALUE, "key_bytes must be 4 or 8");
  if (val_bytes != 0 && val_bytes != 4 && val_bytes != 8) return fail(BS_ERR_VALUE, "val_bytes must be 0, 4 or 8");
  if (val_bytes != 0 && vals == nullptr) return fail(BS_ERR_VALUE, "val_bytes > 0 but vals is NULL");
  if (width < 1 || width > 64) return fail(BS_ERR_VALUE, "unsupported word width");
  if (n == 0) return fail(BS_ERR_ASSERT, "partition requires a non-empty range");
  if (pos < 0 || pos >= width) return fail(BS_ERR_ASSERT, "bit position out of codec width");
  if (n >= (uint64_t(1) << 32)) return fail(BS_ERR_VALUE, "n too large");
  if (ws_bytes < bs_partition_workspace_bytes(n, key_bytes, val_bytes))
    return fail(BS_ERR_WORKSPACE, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char *b = static_cast<char *>(ws);
  void *copy = b;
  b += align_up(size_t(key_bytes) * n);
  void *vcopy = b;
  b += align_up(size_t(val_bytes) * n);
  uint32_t *lone = reinterpret_cast<uint32_t *>(b);
  b += align_up(sizeof(uint32_t) * (n + 1));
  uint32_t *zpos = reinterpret_cast<uint32_t *>(b);
  b += align_up(sizeof(uint32_t) * (n + 1));
  uint32_t *bcnt = reinterpret_cast<uint32_t *>(b);
  const uint64_t nblk = (n + PART_CHUNK - 1) / PART_CHUNK;
  uint32_t *Zp = bcnt + nblk;
  BS_CUDA(cudaMemcpyAsync(copy, keys, size_t(key_bytes) * n, cudaMemcpyDeviceToDevice, st));
  if (val_bytes) BS_CUDA(cudaMemcpyAsync(vcopy, vals, size_t(val_bytes) * n, cudaMemcpyDeviceToDevice, st));
  auto go = [&](auto tag, auto vbc) -> int {
    using K = decltype(tag);
    constexpr int VB = decltype(vbc)::value;
    const K *src = static_cast<const K *>(copy);
    part_count_kernel<K><<<unsigned(nblk), PART_BLOCK, 0, st>>>(src, n, pos, width, bcnt);
    scan_blocks_kernel<<<1, 1024, 0, st>>>(bcnt, uint32_t(nblk), Zp);
    part_index_kernel<K><<<unsigned(nblk), PART_BLOCK, 0, st>>>(src, n, pos, width, bcnt, Zp, lone, zpos);
    part_gather_kernel<K, VB><<<unsigned(nblk), PART_BLOCK, 0, st>>>(src, static_cast<K *>(keys), vcopy, vals, n,
                                                                     pos, width, bcnt, Zp, lone, zpos);
    part_finish_kernel<<<1, 1, 0, st>>>(Zp, n, split_dev, reinterpret_cast<unsigned long long *>(counters));
    BS_CUDA(cudaGetLastError());
    return BS_OK;
  };
  using I0 = std::integral_constant<int, 0>;
  using I4 = std::integral_constant<int, 4>;
  using I8 = std::integral_constant<int, 8>;
  if (key_bytes == 4) {
    if (val_bytes == 0) return go(uint32_t(0), I0{});
    if (val_bytes == 4) return go(uint32_t(0), I4{});
    return go(uint32_t(0), I8{});
  }
  if (val_bytes == 0) return go(uint64_t(0), I0{});
  if (val_bytes == 4) return go(uint64_t(0), I4{});
  return go(uint64_t(0), I8{});
}

int bs_range_sorted(const void *keys, uint64_t n, int key_bytes, void *stream, int32_t *flag_dev) {
  if (key_bytes != 4 && key_bytes != 8) return fail(BS_ERR_VALUE, "key_bytes must be 4 or 8");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int32_t one = 1;
  BS_CUDA(cudaMemcpyAsync(flag_dev, &one, sizeof(one), cudaMemcpyHostToDevice, st));
  if (n < 2) return BS_OK;
  const int grid = int(min64((n + 255) / 256, uint64_t(num_sms()) * 8));
  if (key_bytes == 4)
    range_sorted_kernel<uint32_t><<<grid, 256, 0, st>>>(static_cast<const uint32_t *>(keys), n, flag_dev);
  else
    range_sorted_kernel<uint64_t><<<grid, 256, 0, st>>>(static_cast<const uint64_t *>(keys), n, flag_dev);
  BS_CUDA(cudaGetLastError());
  return BS_OK;
}

size_t bs_split_workspace_bytes(uint64_t n, int, int, int) {
  const uint64_t ntiles = (n + SPLIT_TILE - 1) / SPLIT_TILE;
  const uint64_t nchunks = (ntiles + SCAN_CHUNK - 1) / SCAN_CHUNK;
  return align_up(sizeof(uint32_t) * 16 * (ntiles + 1)) + align_up(sizeof(uint32_t) * 16 * (nchunks + 1)) +
         align_up(sizeof(uint32_t) * 16);
}

}  // extern "C"

namespace bs {

template <typename F>
static int split_dispatch(int key_bytes, int key_kind, int val_bytes, F &&go) {
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  using I4 = std::integral_constant<int, 4>;
  using I8 = std::integral_constant<int, 8>;
  auto by_v = [&](auto ktag, auto kindc) -> int {
    if (val_bytes == 0) return go(ktag, kindc, I0{});
    if (val_bytes == 4) return go(ktag, kindc, I4{});
    return go(ktag, kindc, I8{});
  };
  if (key_bytes == 4) return key_kind == 0 ? by_v(uint32_t(0), I0{}) : by_v(uint32_t(0), I1{});
  if (key_kind == 0) return by_v(uint64_t(0), I0{});
  if (key_kind == 1) return by_v(uint64_t(0), I1{});
  return by_v(uint64_t(0), I2{});
}

struct SplitWs {
  uint32_t *tile_hist, *chunk_sum, *class_base;
  uint32_t ntiles, nchunks;
};

static SplitWs split_ws(void *ws, uint64_t n) {
  SplitWs w{};
  w.ntiles = uint32_t((n + SPLIT_TILE - 1) / SPLIT_TILE);
  w.nchunks = (w.ntiles + SCAN_CHUNK - 1) / SCAN_CHUNK;
  char *b = static_cast<char *>(ws);
  w.tile_hist = reinterpret_cast<uint32_t *>(b);
  b += align_up(sizeof(uint32_t) * 16 * (uint64_t(w.ntiles) + 1));
  w.chunk_sum = reinterpret_cast<uint32_t *>(b);
  b += align_up(sizeof(uint32_t) * 16 * (uint64_t(w.nchunks) + 1));
  w.class_base = reinterpret_cast<uint32_t *>(b);
  return w;
}

static int split_check(uint64_t n, int key_bytes, int val_bytes, int width, int key_kind, int nranks,
                       size_t ws_bytes) {
  int rc = check_common(key_bytes, val_bytes, width, 0, key_kind);
  if (rc) return rc;
  if (nranks < 1 || nranks > 8) return fail(BS_ERR_VALUE, "nranks must be in [1, 8]");
  if (n >= (uint64_t(1) << 32)) return fail(BS_ERR_VALUE, "n too large");
  if (ws_bytes < bs_split_workspace_bytes(n, key_bytes, val_bytes, nranks))
    return fail(BS_ERR_WORKSPACE, "workspace too small");
  return BS_OK;
}

// class histogram per tile + parallel class-major scan (tile offsets stay in ws)
static int split_count(const void *keys, uint64_t n, int key_bytes, int width, int key_kind, const void *splitters,
                       int nranks, uint64_t *class_counts, void *ws, cudaStream_t st) {
  const int ncls = 2 * nranks - 1, nsp = nranks - 1;
  BS_CUDA(cudaMemsetAsync(class_counts, 0, sizeof(uint64_t) * ncls, st));
  if (n == 0) return BS_OK;
  const SplitWs w = split_ws(ws, n);
  const int shift0 = key_bytes * 8 - width;
  return split_dispatch(key_bytes, key_kind, 0, [&](auto ktag, auto kindc, auto) -> int {
    using K = decltype(ktag);
    constexpr int KIND = decltype(kindc)::value;
    split_hist_kernel<K, KIND><<<(w.ntiles + SPLIT_HIST_TPB - 1) / SPLIT_HIST_TPB, SPLIT_BLOCK, 0, st>>>(
        static_cast<const K *>(keys), n, shift0,
                                                                 static_cast<const K *>(splitters), nsp, w.tile_hist);
    split_chunk_sum_kernel<<<w.nchunks, 256, 0, st>>>(w.tile_hist, w.ntiles, w.chunk_sum);
    split_top_scan_kernel<<<1, 512, 0, st>>>(w.chunk_sum, w.nchunks, ncls,
                                             reinterpret_cast<unsigned long long *>(class_counts), w.class_base);
    split_chunk_scan_kernel<<<w.nchunks, 256, 0, st>>>(w.tile_hist, w.ntiles, w.chunk_sum, w.class_base);
    BS_CUDA(cudaGetLastError());
    return BS_OK;
  });
}

}  // namespace bs

extern "C" {

int bs_split_by_splitters(const void *keys, const void *vals, uint64_t n, int key_bytes, int val_bytes,
                          int width, int key_kind, const void *splitters, int nranks, void *out_keys,
                          void *out_vals, uint64_t *class_counts, void *ws, size_t ws_bytes, void *stream) {
  int rc = split_check(n, key_bytes, val_bytes, width, key_kind, nranks, ws_bytes);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = split_count(keys, n, key_bytes, width, key_kind, splitters, nranks, class_counts, ws, st);
  if (rc || n == 0) return rc;
  const SplitWs w = split_ws(ws, n);
  const int shift0 = key_bytes * 8 - width, nsp = nranks - 1;
  return split_dispatch(key_bytes, key_kind, val_bytes, [&](auto ktag, auto kindc, auto vbc) -> int {
    using K = decltype(ktag);
    constexpr int KIND = decltype(kindc)::value;
    constexpr int VB = decltype(vbc)::value;
    split_scatter_kernel<K, VB, KIND><<<w.ntiles, SPLIT_BLOCK, 0, st>>>(
        static_cast<const K *>(keys), vals, n, shift0, static_cast<const K *>(splitters), nsp, w.tile_hist,
        static_cast<K *>(out_keys), out_vals);
    BS_CUDA(cudaGetLastError());
    return BS_OK;
  });
}

int bs_split_count(const void *keys, uint64_t n, int key_bytes, int width, int key_kind, const void *splitters,
                   int nranks, uint64_t *class_counts, void *ws, size_t ws_bytes, void *stream) {
  int rc = split_check(n, key_bytes, 0, width, key_kind, nranks, ws_bytes);
  if (rc) return rc;
  return split_count(keys, n, key_bytes, width, key_kind, splitters, nranks, class_counts, ws,
                     static_cast<cudaStream_t>(stream));
}

int bs_split_exchange(const void *keys, const void *vals, uint64_t n, int key_bytes, int val_bytes, int width,
                      int key_kind, const void *splitters, int nranks, const int64_t *delta,
                      const uint64_t *bounds, void *const *dst_keys, void *const *dst_vals, void *ws,
                      size_t ws_bytes, void *stream) {
  int rc = split_check(n, key_bytes, val_bytes, width, key_kind, nranks, ws_bytes);
  if (rc) return rc;
  if (val_bytes != 0 && (vals == nullptr || dst_vals == nullptr))
    return fail(BS_ERR_VALUE, "val_bytes > 0 but vals or dst_vals is NULL");
  if (n == 0) return BS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const SplitWs w = split_ws(ws, n);
  const int shift0 = key_bytes * 8 - width, nsp = nranks - 1;
  return split_dispatch(key_bytes, key_kind, val_bytes, [&](auto ktag, auto kindc, auto vbc) -> int {
    using K = decltype(ktag);
    constexpr int KIND = decltype(kindc)::value;
    constexpr int VB = decltype(vbc)::value;
    auto kern = split_exchange_kernel<K, VB, KIND>;
    const size_t smem = ExchangeSmem<K, VB>::bytes;
    BS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    // persistent grid: the per-CTA setup (splitters, class table) is paid once per resident CTA
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SPLIT_BLOCK, smem);
    const unsigned grid = unsigned(min64(w.ntiles, uint64_t(num_sms()) * uint64_t(per_sm > 0 ? per_sm : 1)));
    kern<<<grid, SPLIT_BLOCK, smem, st>>>(static_cast<const K *>(keys), vals, n, shift0,
                                              static_cast<const K *>(splitters), nsp, w.tile_hist,
                                              reinterpret_cast<const long long *>(delta),
                                              reinterpret_cast<const unsigned long long *>(bounds), nranks,
                                              reinterpret_cast<K *const *>(dst_keys), dst_vals, w.class_base + 32);
    BS_CUDA(cudaGetLastError());
    return BS_OK;
  });
}

size_t bs_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int bs_ipc_alloc(size_t bytes, void **ptr, void *handle) {
  if (!ptr || !handle) return fail(BS_ERR_VALUE, "ptr and handle must be non-NULL");
  *ptr = nullptr;
  BS_CUDA(cudaMalloc(ptr, bytes ? bytes : 1));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, *ptr);
  if (e != cudaSuccess) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return fail(BS_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  }
  std::memcpy(handle, &h, sizeof(h));
  return BS_OK;
}

int bs_ipc_open(const void *handle, void **ptr) {
  if (!ptr || !handle) return fail(BS_ERR_VALUE, "ptr and handle must be non-NULL");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  BS_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return BS_OK;
}

int bs_ipc_close(void *ptr) {
  BS_CUDA(cudaIpcCloseMemHandle(ptr));
  return BS_OK;
}

int bs_ipc_free(void *ptr) {
  BS_CUDA(cudaFree(ptr));
  return BS_OK;
}

int bs_sample_keys(const void *keys, uint64_t n, int key_bytes, int width, int key_kind, uint64_t count,
                   void *out_samples, void *stream) {
  int rc = check_common(key_bytes, 0, width, 0, key_kind);
  if (rc) return rc;
  if (n == 0 || count == 0) return BS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int shift0 = key_bytes * 8 - width;
  const int grid = int(min64((count + 255) / 256, 1024));
  if (key_bytes == 4) {
    if (key_kind == 0)
      sample_kernel<uint32_t, 0><<<grid, 256, 0, st>>>(static_cast<const uint32_t *>(keys), n, shift0, count,
                                                      static_cast<uint32_t *>(out_samples));
    else
      sample_kernel<uint32_t, 1><<<grid, 256, 0, st>>>(static_cast<const uint32_t *>(keys), n, shift0, count,
                                                      static_cast<uint32_t *>(out_samples));
  } else {
    if (key_kind == 0)
      sample_kernel<uint64_t, 0><<<grid, 256, 0, st>>>(static_cast<const uint64_t *>(keys), n, shift0, count,
                                                      static_cast<uint64_t *>(out_samples));
    else if (key_kind == 1)
      sample_kernel<uint64_t, 1><<<grid, 256, 0, st>>>(static_cast<const uint64_t *>(keys), n, shift0, count,
                                                      static_cast<uint64_t *>(out_samples));
    else
      sample_kernel<uint64_t, 2><<<grid, 256, 0, st>>>(static_cast<const uint64_t *>(keys), n, shift0, count,
                                                      static_cast<uint64_t *>(out_samples));
  }
  BS_CUDA(cudaGetLastError());
  return BS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Exact reference-order engine (exact_impl.cuh): host driver.
// ---------------------------------------------------------------------------
namespace bs {

struct ExLayout {
  size_t copy, vcopy, seg, tab0, tab1, lone, zpos, bcnt, ctr, total;
  uint64_t nblk;
};

static ExLayout ex_layout(uint64_t n, int kb, int vb) {
  ExLayout l{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes);
    return o;
  };
  l.nblk = (n + ex::EX_CHUNK - 1) / ex::EX_CHUNK;
  l.ctr = take(4 * sizeof(unsigned long long));
  l.bcnt = take(sizeof(uint32_t) * (l.nblk + 1));
  l.seg = take(sizeof(uint32_t) * n);
  l.tab0 = take(sizeof(ex::SegT) * n);
  l.tab1 = take(sizeof(ex::SegT) * n);
  l.lone = take(sizeof(uint32_t) * (n + 1));
  l.zpos = take(sizeof(uint32_t) * (n + 1));
  l.copy = take(size_t(kb) * n);
  l.vcopy = take(size_t(vb) * n);
  l.total = off;
  return l;
}

template <typename K, int VB>
static int run_exact(void *keys, void *vals, uint64_t n, int width, int pos0, int key_kind, int mode, int loop,
                     int check_after, int streak0, int checked0, int par_levels, int64_t depth0, void *wsp,
                     size_t ws_bytes, cudaStream_t st, int64_t *counters, bs_level_fn on_level, void *ctx) {
  const ExLayout l = ex_layout(n, int(sizeof(K)), VB);
  if (ws_bytes < l.total)
    return fail(BS_ERR_WORKSPACE, "workspace too small: need " + std::to_string(l.total) + " bytes, got " +
                                      std::to_string(ws_bytes));
  char *b = static_cast<char *>(wsp);
  ex::Ex e{};
  e.keys[0] = keys;
  e.keys[1] = b + l.copy;
  e.vals[0] = vals;
  e.vals[1] = VB ? b + l.vcopy : nullptr;
  e.seg = reinterpret_cast<uint32_t *>(b + l.seg);
  e.tab[0] = reinterpret_cast<ex::SegT *>(b + l.tab0);
  e.tab[1] = reinterpret_cast<ex::SegT *>(b + l.tab1);
  e.lone = reinterpret_cast<uint32_t *>(b + l.lone);
  e.zpos = reinterpret_cast<uint32_t *>(b + l.zpos);
  e.bcnt = reinterpret_cast<uint32_t *>(b + l.bcnt);
  e.ctr = counters ? reinterpret_cast<unsigned long long *>(counters)
                   : reinterpret_cast<unsigned long long *>(b + l.ctr);
  e.n = n;
  e.width = width;
  e.kind = key_kind;
  e.mode = mode;
  e.loop = loop;
  e.check_after = check_after;
  e.par_levels = par_levels;
  e.depth0 = mode == ex::M_PAR ? 0 : depth0;
  const int nlev = width - pos0;
  // root record and counters before the first level (see exact_impl.cuh)
  int64_t c0[4] = {0, 0, 0, 0};
  uint32_t rbits = 0;
  if (mode == ex::M_REC) {  // the root call (kernels.py:100-102)
    c0[2] = 1;
    c0[3] = depth0;
    rbits = (n >= 2 && nlev > 0) ? ex::F_ACTIVE : 0u;
    if (checked0) rbits |= ex::F_CHECKED;
  } else if (mode == ex::M_ITER) {  // the stack holds the root (kernels.py:138-142)
    c0[3] = 1;
    rbits = (n >= 1 && nlev > 0) ? ex::F_ACTIVE : 0u;
  } else if (mode == ex::M_LEVELS) {  // core.py:157: segments = [(lower, upper, upper > lower)]
    rbits = n >= 2 ? (ex::F_ACTIVE | ex::F_CHECK) : 0u;
  } else {  // sort_parallel: prepartition levels (variants.py:181-193), then bucket calls
    if (n >= 2) {
      c0[3] = par_levels;
      if (par_levels == 0) {  // one bucket: sort_words(words, 0, n-1, 0, width, ..., 1)
        c0[2] = 1;
        c0[3] = 1;
      }
    }
    rbits = (n >= 2 && nlev > 0) ? ex::F_ACTIVE : 0u;
  }
  const uint32_t rdep = (mode == ex::M_PAR && par_levels == 0) ? 1u : 0u;
  const ex::SegT root{uint32_t(n), ex::pack(rbits, uint32_t(streak0), rdep, 0), 0, 0};
  BS_CUDA(cudaMemcpyAsync(e.ctr, c0, sizeof(c0), cudaMemcpyHostToDevice, st));
  if (n == 0) return BS_OK;
  const unsigned g1 = unsigned(min64((n + 255) / 256, uint64_t(1) << 30));
  const unsigned gchunk = unsigned(l.nblk);
  ex::ex_init_kernel<<<unsigned(min64((n + 255) / 256, uint64_t(num_sms()) * 16)), 256, 0, st>>>(e, root);
  const bool checks = (mode == ex::M_REC && check_after > 0) || mode == ex::M_LEVELS;
  for (int L = 0; L < nlev; ++L) {
    const int pos = pos0 + L, par = L & 1, cur = L & 1;
    if (checks) ex::ex_check_kernel<K><<<g1, 256, 0, st>>>(e, par, cur);
    ex::ex_count_kernel<K><<<gchunk, ex::EX_BLOCK, 0, st>>>(e, pos, par, cur);
    scan_blocks_kernel<<<1, 1024, 0, st>>>(e.bcnt, uint32_t(l.nblk), nullptr);
    ex::ex_bounds_kernel<K><<<gchunk, ex::EX_BLOCK, 0, st>>>(e, pos, par, cur);
    ex::ex_plan_kernel<<<g1, 256, 0, st>>>(e, L, pos, cur);
    ex::ex_index_kernel<K><<<gchunk, ex::EX_BLOCK, 0, st>>>(e, pos, par, cur);
    ex::ex_gather_kernel<K, VB><<<gchunk, ex::EX_BLOCK, 0, st>>>(e, pos, par, cur);
    BS_CUDA(cudaGetLastError());
    if (on_level) on_level(ctx, pos);
  }
  const int fcur = nlev & 1;
  if (mode == ex::M_REC && check_after > 0) {  // scans flagged by the last level
    ex::ex_check_kernel<K><<<g1, 256, 0, st>>>(e, fcur, fcur);
    ex::ex_resolve_kernel<<<g1, 256, 0, st>>>(e, fcur);
  }
  ex::ex_finalize_kernel<K, VB><<<unsigned(min64((n + 255) / 256, uint64_t(num_sms()) * 16)), 256, 0, st>>>(
      e, fcur, uint32_t(nlev & 1));
  BS_CUDA(cudaGetLastError());
  return BS_OK;
}

}  // namespace bs

extern "C" {

size_t bs_exact_workspace_bytes(uint64_t n, int key_bytes, int val_bytes) {
  if ((key_bytes != 4 && key_bytes != 8) || (val_bytes != 0 && val_bytes != 4 && val_bytes != 8)) return 0;
  return ex_layout(n, key_bytes, val_bytes).total;
}

int bs_exact_sort(void *keys, void *vals, uint64_t n, int key_bytes, int val_bytes, int width, int start_pos,
                  int key_kind, int mode, int passthrough_loop, int check_after, int streak, int checked,
                  int par_levels, int64_t depth, void *ws, size_t ws_bytes, void *stream, int64_t *counters,
                  bs_level_fn on_level, void *ctx) {
  if (key_bytes != 4 && key_bytes != 8) return fail(BS_ERR_VALUE, "key_bytes must be 4 or 8");
  if (val_bytes != 0 && val_bytes != 4 && val_bytes != 8) return fail(BS_ERR_VALUE, "val_bytes must be 0, 4 or 8");
  if (width < 1 || width > key_bytes * 8) return fail(BS_ERR_VALUE, "unsupported word width " + std::to_string(width));
  if (start_pos < 0 || start_pos > width) return fail(BS_ERR_ASSERT, "bit position past codec width");
  if (key_kind < 0 || key_kind > 2) return fail(BS_ERR_VALUE, "unknown key_kind");
  if (key_kind == BS_KEY_SIGNED && width < 2) return fail(BS_ERR_VALUE, "unsupported word width " + std::to_string(width));
  if (key_kind == BS_KEY_FLOAT && width != 64) return fail(BS_ERR_VALUE, "float keys are 64-bit words of width 64");
  if (mode < 0 || mode > 3) return fail(BS_ERR_VALUE, "unknown exact mode");
  if (check_after < 0) return fail(BS_ERR_VALUE, "sortedness_check_after must be >= 0");
  if (par_levels < 0 || par_levels > width || (mode == 3 && start_pos != 0))
    return fail(BS_ERR_VALUE, "bad prepartition levels");
  if (n >= (uint64_t(1) << 32) - 1) return fail(BS_ERR_VALUE, "n too large for the exact engine");
  if (n > 0 && keys == nullptr) return fail(BS_ERR_VALUE, "NULL key buffer");
  if (val_bytes != 0 && n > 0 && vals == nullptr) return fail(BS_ERR_VALUE, "val_bytes > 0 but vals is NULL");
  if (depth < 0 || depth > 120) return fail(BS_ERR_VALUE, "depth out of range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (val_bytes == 0) vals = nullptr;
  streak = streak < 0 ? 0 : (streak > 255 ? 255 : streak);
#define BS_EX(K)                                                                                                    \
  do {                                                                                                              \
    if (val_bytes == 0)                                                                                             \
      return run_exact<K, 0>(keys, vals, n, width, start_pos, key_kind, mode, passthrough_loop, check_after, streak, \
                             checked, par_levels, depth, ws, ws_bytes, st, counters, on_level, ctx);                \
    if (val_bytes == 4)                                                                                             \
      return run_exact<K, 4>(keys, vals, n, width, start_pos, key_kind, mode, passthrough_loop, check_after, streak, \
                             checked, par_levels, depth, ws, ws_bytes, st, counters, on_level, ctx);                \
    return run_exact<K, 8>(keys, vals, n, width, start_pos, key_kind, mode, passthrough_loop, check_after, streak,   \
                           checked, par_levels, depth, ws, ws_bytes, st, counters, on_level, ctx);                  \
  } while (0)
  if (key_bytes == 4) BS_EX(uint32_t);
  BS_EX(uint64_t);
#undef BS_EX
}

int bs_exact_snapshot(const void *keys, const void *ws, uint64_t n, int key_bytes, int val_bytes, int levels_done,
                      void *out_keys, void *stream) {
  if (!ws || !out_keys || (n > 0 && !keys)) return fail(BS_ERR_VALUE, "keys, ws and out_keys must be non-NULL");
  if (key_bytes != 4 && key_bytes != 8) return fail(BS_ERR_VALUE, "key_bytes must be 4 or 8");
  if (n == 0) return BS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const ExLayout l = ex_layout(n, key_bytes, val_bytes);
  char *b = static_cast<char *>(const_cast<void *>(ws));
  ex::Ex e{};
  e.keys[0] = const_cast<void *>(keys);
  e.keys[1] = b + l.copy;
  e.seg = reinterpret_cast<uint32_t *>(b + l.seg);
  e.tab[0] = reinterpret_cast<ex::SegT *>(b + l.tab0);
  e.tab[1] = reinterpret_cast<ex::SegT *>(b + l.tab1);
  e.n = n;
  const int cur = levels_done & 1;
  const unsigned grid = unsigned(min64((n + 255) / 256, uint64_t(num_sms()) * 16));
  if (key_bytes == 4)
    ex::ex_snapshot_kernel<uint32_t><<<grid, 256, 0, st>>>(e, cur, uint32_t(cur), static_cast<uint32_t *>(out_keys));
  else
    ex::ex_snapshot_kernel<uint64_t><<<grid, 256, 0, st>>>(e, cur, uint32_t(cur), static_cast<uint64_t *>(out_keys));
  BS_CUDA(cudaGetLastError());
  return BS_OK;
}

int bs_exact_boundaries(const void *ws, uint64_t n, int key_bytes, int val_bytes, uint32_t *starts, uint32_t *count,
                        void *stream) {
  if (!ws || !starts || !count) return fail(BS_ERR_VALUE, "ws, starts and count must be non-NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 0) {
    BS_CUDA(cudaMemsetAsync(count, 0, sizeof(uint32_t), st));
    return BS_OK;
  }
  const ExLayout l = ex_layout(n, key_bytes, val_bytes);
  const char *b = static_cast<const char *>(ws);
  const uint32_t *seg = reinterpret_cast<const uint32_t *>(b + l.seg);
  // the chunk counts reuse the engine's bcnt array (the level's kernels are done with it)
  uint32_t *bcnt = reinterpret_cast<uint32_t *>(const_cast<char *>(b) + l.bcnt);
  ex::ex_starts_count_kernel<<<unsigned(l.nblk), ex::EX_BLOCK, 0, st>>>(seg, n, bcnt);
  scan_blocks_kernel<<<1, 1024, 0, st>>>(bcnt, uint32_t(l.nblk), count);
  ex::ex_starts_write_kernel<<<unsigned(l.nblk), ex::EX_BLOCK, 0, st>>>(seg, n, bcnt, starts);
  BS_CUDA(cudaGetLastError());
  return BS_OK;
}

}  // extern "C"

