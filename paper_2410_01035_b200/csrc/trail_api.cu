// trail_api.cu — the C ABI of libtrail.so (include/trail.h): argument validation, the
// create-time constants (computed in fp64 on the host), workspace ownership, layer-1
// regime planning, NCCL all-gather of records (NCCL loaded at run time), profiling.
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <vector>
#include <new>

#include "trail_internal.cuh"

using namespace trail;

struct trail_ctx {
  Ctx c;
};

namespace {

constexpr int kGemvMaxN = 16;   // AUTO: GEMV up to this many requests (bf16)

#define TRAIL_CUDA(expr)                                                     \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      fprintf(stderr, "[trail] %s failed: %s\n", #expr, cudaGetErrorString(_e)); \
      return TRAIL_ERR_CUDA;                                                 \
    }                                                                        \
  } while (0)

struct ProfScope {
  Ctx &c;
  int slot = -1;
  cudaStream_t s;
  int kid_ = -1;
  unsigned flags_ = 0;
  ProfScope(Ctx &c_, int kid, cudaStream_t s_) : c(c_), s(s_) {
    if (!c.prof) return;
    if (c.prof_mode == 2) {
      kid_ = kid;
      c.last_used[kid] = true;
      // while a graph is being captured, record as an external event node so every
      // replay re-records the event; outside capture a plain record
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(s, &cs);
      flags_ = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
      cudaEventRecordWithFlags(c.last_ev[kid][0], s, flags_);
    } else if (c.prof_n < c.prof_cap) {
      slot = c.prof_n++;
      c.prof_kid[slot] = kid;
      cudaEventRecord(c.prof_ev[2 * slot], s);
    }
  }
  ~ProfScope() {
    if (kid_ >= 0) cudaEventRecordWithFlags(c.last_ev[kid_][1], s, flags_);
    else if (slot >= 0) cudaEventRecord(c.prof_ev[2 * slot + 1], s);
  }
};

void plan_l1(const Ctx &c, int n, int *mode, int *bn, int *splits, bool planning = false) {
  int m = c.cfg.l1_mode;
  if (c.dtype == TRAIL_F32) {
    // fp32: the 3xTF32 tensor-core layer 1 (K2t) unless the CUDA-core GEMV is forced
    // AUTO keeps the CUDA-core GEMV K2a: measured at configs[0], K2t's launch is shorter
    // (14.4 vs 18.2 us) but the step is longer (median 38.9 vs 32.8 us);
    // TRAIL_FP32_L1=tf32 makes AUTO pick K2t (A/B runs)
    static const bool tf32_env = [] {
      const char *e = getenv("TRAIL_FP32_L1");
      return e && e[0] == 't';
    }();
    const bool tf32_ok = tf32_supported(c) || (planning && c.H % 128 == 0 && c.d % 4 == 0);
    if ((m == TRAIL_L1_TF32 || (m == TRAIL_L1_AUTO && tf32_env)) && tf32_ok) {
      *mode = TRAIL_L1_TF32;
      *bn = 0;
      *splits = tf32_splits(c);
      return;
    }
    m = TRAIL_L1_GEMV;
  }
  else if (m == TRAIL_L1_AUTO) m = (n <= kGemvMaxN) ? TRAIL_L1_GEMV : TRAIL_L1_UMMA;
  if (m == TRAIL_L1_UMMA && c.cfg.l1_mode == TRAIL_L1_AUTO && wide_supported(c) && n >= wide_min_n())
    m = TRAIL_L1_WIDE;
  if (m == TRAIL_L1_WIDE && !wide_supported(c)) m = TRAIL_L1_UMMA;
  if (m == TRAIL_L1_WIDE) {
    *mode = TRAIL_L1_WIDE;
    *bn = 512;
    *splits = 1;
    return;
  }
  if (m == TRAIL_L1_UMMA) {
    *mode = TRAIL_L1_UMMA;
    *bn = 128;
    *splits = fused_splits(c, n);
    return;
  }
  if (m == TRAIL_L1_GEMV) {
    // about one CTA per SM (64 hidden rows x one K range each); K ranges a multiple of 8
    // elements and small enough that both operand slices fit in shared memory
    const int ctas_x = c.H / 64;
    int s = std::max(1, c.num_sms / ctas_x);
    const int kmax = (200 * 1024 - 512 - 16384) / (128 * (int)c.esize) - 16;
    s = std::max(s, (c.d + kmax - 1) / kmax);
    s = std::min(s, std::max(1, c.d / 8));
    const int kchunk = ((c.d + s - 1) / s + 7) / 8 * 8;
    s = (c.d + kchunk - 1) / kchunk;
    *mode = TRAIL_L1_GEMV;
    *bn = 0;
    *splits = s;
  } else {
    const int b = (n > 1024 && umma_max_bn(c) == 256) ? 256 : 128;
    const int tiles = ((n + 127) / 128) * (c.H / b);
    const int kblocks = c.d / 64;
    *mode = TRAIL_L1_UMMA_UNFUSED;
    *bn = b;
    *splits = std::max(1, std::min(kblocks, c.num_sms / std::max(1, tiles)));
  }
}

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void *lib = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char *(*errStr)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi &nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
      api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.lib) break;
    }
    if (api.lib) {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(api.lib, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(api.lib, "ncclCommInitRank");
      api.allGather = (decltype(api.allGather))dlsym(api.lib, "ncclAllGather");
      api.commDestroy = (decltype(api.commDestroy))dlsym(api.lib, "ncclCommDestroy");
      api.errStr = (decltype(api.errStr))dlsym(api.lib, "ncclGetErrorString");
      api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.commDestroy;
    }
  }
  return api;
}

trail_status set_device(const Ctx &c) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) return TRAIL_ERR_CUDA;
  if (cur != c.device && cudaSetDevice(c.device) != cudaSuccess) return TRAIL_ERR_CUDA;
  return TRAIL_OK;
}

void free_ctx(Ctx &c) {
  void *ptrs[] = {c.w1, c.b1, c.w2, c.b2, c.consts, c.lq, c.meta, c.dev_err, c.xs,
                  c.partial, c.rec_local, c.rec_all, c.zpart, c.arrive_cnt, c.trace,
                  c.rank_sorted, c.rank_cnt, c.pool_head, c.pool_tail, c.pool_cnt, c.bk_ws,
                  c.chunk_acc, c.chunk_cnt, c.xmix, c.iota};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  if (c.ev_fork) cudaEventDestroy(c.ev_fork);
  if (c.ev_join) cudaEventDestroy(c.ev_join);
  if (c.side) cudaStreamDestroy(c.side);
  if (c.prof_ev) {
    for (int i = 0; i < 2 * c.prof_cap; ++i) cudaEventDestroy(c.prof_ev[i]);
    delete[] c.prof_ev;
    delete[] c.prof_kid;
  }
  for (int i = 0; i < TRAIL_K_COUNT; ++i)
    for (int j = 0; j < 2; ++j)
      if (c.last_ev[i][j]) cudaEventDestroy(c.last_ev[i][j]);
  if (c.nccl_comm && nccl().ok) nccl().commDestroy((ncclComm_t)c.nccl_comm);
}

size_t partial_elems_needed(const Ctx &c) {
  size_t best = 0;
  for (int n = 1; n <= c.cfg.max_requests; ++n) {
    for (int forced = 0; forced < 2; ++forced) {
      Ctx tmp_c;
      tmp_c.cfg = c.cfg;
      // bf16: the GEMV and unfused tcgen05 plans; fp32: the GEMV and 3xTF32 plans
      tmp_c.cfg.l1_mode = forced ? TRAIL_L1_GEMV
                                 : (c.dtype == TRAIL_F32 ? TRAIL_L1_TF32 : TRAIL_L1_UMMA_UNFUSED);
      tmp_c.d = c.d; tmp_c.H = c.H; tmp_c.dtype = c.dtype; tmp_c.num_sms = c.num_sms;
      int mode, bn, s;
      plan_l1(tmp_c, n, &mode, &bn, &s, true);
      best = std::max(best, (size_t)s * (size_t)n * (size_t)c.H);
    }
  }
  return best;
}

}  // namespace

// =============================================================================== ABI
extern "C" {

int32_t trail_abi_version(void) { return TRAIL_ABI_VERSION; }

const char *trail_status_string(trail_status s) {
  switch (s) {
    case TRAIL_OK: return "ok";
    case TRAIL_WARN_OVER_BUDGET: return "forced set exceeds the KV budget or run cap";
    case TRAIL_ERR_INVALID: return "invalid argument";
    case TRAIL_ERR_CUDA: return "CUDA error";
    case TRAIL_ERR_NOMEM: return "out of memory";
    case TRAIL_ERR_CAPACITY: return "capacity exceeded";
    case TRAIL_ERR_NCCL: return "NCCL unavailable or failed";
    case TRAIL_ERR_STATE: return "invalid handle state";
    case TRAIL_ERR_UNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

trail_status trail_create(const trail_config *cfg, trail_handle *out) {
  if (!cfg || !out) return TRAIL_ERR_INVALID;
  *out = nullptr;
  const trail_config &g = *cfg;
  if (g.dtype != TRAIL_F32 && g.dtype != TRAIL_BF16) return TRAIL_ERR_INVALID;
  if (g.k < 1 || g.k > kMaxBins) return TRAIL_ERR_INVALID;
  if (g.hidden < 128 || g.hidden > kMaxHidden || g.hidden % 128) return TRAIL_ERR_INVALID;
  if (g.d <= 0 || (g.dtype == TRAIL_BF16 ? g.d % 64 : g.d % 8)) return TRAIL_ERR_INVALID;
  if (!g.w1 || !g.b1 || !g.w2 || !g.b2 || !g.bin_edges) return TRAIL_ERR_INVALID;
  if (!(g.c >= 0.0)) return TRAIL_ERR_INVALID;   // rejects NaN and negatives
  if (g.max_slots <= 0 || g.max_requests <= 0 || g.max_sched < 0) return TRAIL_ERR_INVALID;
  if (g.max_requests > (1 << 18)) return TRAIL_ERR_INVALID;   // K1 offset search bound
  if (g.world_size < 1) return TRAIL_ERR_INVALID;
  if (g.l1_mode < 0 || g.l1_mode > 5) return TRAIL_ERR_INVALID;
  if (g.l1_mode >= TRAIL_L1_UMMA && g.l1_mode <= TRAIL_L1_WIDE && g.dtype != TRAIL_BF16)
    return TRAIL_ERR_UNSUPPORTED;
  if (g.l1_mode == TRAIL_L1_TF32 && g.dtype != TRAIL_F32) return TRAIL_ERR_UNSUPPORTED;
  // every selection runs in one thread-block cluster: 16 x 8192 records (8 x 8192 where a
  // 16-CTA cluster cannot be resident; checked again after select_prepare)
  if ((int64_t)g.max_sched * g.world_size > 16 * 8192) return TRAIL_ERR_CAPACITY;
  const int k = g.k;
  const double *e = g.bin_edges;
  if (!(e[0] >= 0.0)) return TRAIL_ERR_INVALID;
  for (int i = 0; i < k; ++i)
    if (!(e[i + 1] - e[i] >= 1.0) || !isfinite(e[i + 1])) return TRAIL_ERR_INVALID;
  double prior[kMaxBins];
  if (g.prior) {
    double s = 0;
    for (int i = 0; i < k; ++i) {
      if (!(g.prior[i] >= 0.0)) return TRAIL_ERR_INVALID;
      s += g.prior[i];
    }
    if (fabs(s - 1.0) > 1e-6) return TRAIL_ERR_INVALID;
    for (int i = 0; i < k; ++i) prior[i] = g.prior[i] / s;
  } else {
    for (int i = 0; i < k; ++i) prior[i] = 1.0 / k;
  }

  trail_ctx *h = new (std::nothrow) trail_ctx();
  if (!h) return TRAIL_ERR_NOMEM;
  Ctx &c = h->c;
  c.cfg = g;
  c.device = g.device;
  c.d = g.d; c.H = g.hidden; c.k = k; c.dtype = g.dtype;
  c.esize = g.dtype == TRAIL_BF16 ? 2 : 4;
  c.world = g.world_size;
  auto fail = [&](trail_status st) { free_ctx(c); delete h; return st; };
  if (cudaSetDevice(c.device) != cudaSuccess) return fail(TRAIL_ERR_CUDA);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c.device) != cudaSuccess) return fail(TRAIL_ERR_CUDA);
  if (prop.major < 10) {
    fprintf(stderr, "[trail] device %d is sm_%d%d; this library is built for sm_100a\n", c.device,
            prop.major, prop.minor);
    return fail(TRAIL_ERR_UNSUPPORTED);
  }
  c.num_sms = prop.multiProcessorCount;

  // ---- constants in fp64
  HeadConsts &hc = c.host_consts;
  memset(&hc, 0, sizeof(hc));
  hc.k = k;
  hc.H = c.H;
  double prior_L = 0.0;
  for (int i = 0; i < kMaxBins; ++i) {
    if (i < k) {
      const double m = (e[i] + e[i + 1]) * 0.5;
      const double w = e[i + 1] - e[i];
      hc.m[i] = (float)m;
      hc.log_stay[i] = (float)log(1.0 - 1.0 / w);
      hc.log_move[i] = (i + 1 < k) ? (float)log(1.0 / (e[i + 2] - e[i + 1])) : -INFINITY;
      hc.log_prior[i] = prior[i] > 0 ? (float)log(prior[i]) : -INFINITY;
      if (isinf(g.c)) {
        hc.thr_tab[i] = 0xFFFFFFFFu;
      } else {
        const double t = floor(g.c * m);
        hc.thr_tab[i] = t >= 4294967295.0 ? 0xFFFFFFFEu : (uint32_t)t;
      }
      prior_L += prior[i] * m;
    } else {
      hc.m[i] = 0.f; hc.log_stay[i] = -INFINITY; hc.log_move[i] = -INFINITY;
      hc.log_prior[i] = -INFINITY; hc.thr_tab[i] = 0xFFFFFFFFu;
    }
  }
  hc.prior_L = (float)prior_L;
  hc.dyn_c = -1.f;            // static threshold floor(c r) unless trail_set_threshold_mode

  // ---- device memory
  const size_t w1_bytes = (size_t)c.H * c.d * c.esize;
#define ALLOC(ptr, bytes) \
  if (cudaMalloc((void **)&(ptr), (bytes)) != cudaSuccess) return fail(TRAIL_ERR_NOMEM)
  ALLOC(c.w1, w1_bytes);
  ALLOC(c.b1, c.H * sizeof(float));
  ALLOC(c.w2, (size_t)k * c.H * sizeof(float));
  ALLOC(c.b2, k * sizeof(float));
  ALLOC(c.consts, sizeof(HeadConsts));
  ALLOC(c.lq, (size_t)g.max_slots * k * sizeof(float));
  ALLOC(c.meta, (size_t)g.max_slots * sizeof(SlotMeta));
  ALLOC(c.dev_err, sizeof(uint32_t));
  ALLOC(c.xs, (size_t)g.max_requests * c.d * c.esize);
  c.partial_elems = partial_elems_needed(c);
  ALLOC(c.partial, c.partial_elems * sizeof(float));
  const int max_sched = std::max(1, g.max_sched);
  ALLOC(c.rec_local, (size_t)max_sched * sizeof(Record));
  ALLOC(c.rec_all, (size_t)max_sched * c.world * sizeof(Record));
  ALLOC(c.pool_head, (size_t)pool_grid(c) * c.d * sizeof(float));
  ALLOC(c.pool_tail, (size_t)pool_grid(c) * c.d * sizeof(float));
  ALLOC(c.pool_cnt, (size_t)g.max_requests * sizeof(uint32_t));
  if (cudaMemset(c.pool_cnt, 0, (size_t)g.max_requests * sizeof(uint32_t)) != cudaSuccess)
    return fail(TRAIL_ERR_CUDA);
  ALLOC(c.rank_sorted, (size_t)std::min(max_sched * c.world, kRankMaxRecords) * sizeof(Record));
  ALLOC(c.rank_cnt, 16 * sizeof(uint32_t));
  if (cudaMemset(c.rank_cnt, 0, 16 * sizeof(uint32_t)) != cudaSuccess) return fail(TRAIL_ERR_CUDA);
  c.bk_cap = max_sched * c.world;
  ALLOC(c.bk_ws, bucket_workspace_bytes(c.bk_cap));
  if (cudaMemset(c.bk_ws, 0, bucket_workspace_bytes(c.bk_cap)) != cudaSuccess)
    return fail(TRAIL_ERR_CUDA);
  const size_t m_tiles = ((size_t)g.max_requests + 127) / 128;
  if (c.dtype == TRAIL_BF16) {
    ALLOC(c.zpart, (size_t)g.max_requests * (c.H / 128) * k * sizeof(float));
    ALLOC(c.arrive_cnt, m_tiles * 16 * sizeof(uint32_t));
    if (cudaMemset(c.arrive_cnt, 0, m_tiles * 16 * sizeof(uint32_t)) != cudaSuccess)
      return fail(TRAIL_ERR_CUDA);
  }
#undef ALLOC
  if (cudaMemcpy(c.w1, g.w1, w1_bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c.b1, g.b1, c.H * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c.w2, g.w2, (size_t)k * c.H * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c.b2, g.b2, k * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c.consts, &hc, sizeof(hc), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(c.lq, 0, (size_t)g.max_slots * k * sizeof(float)) != cudaSuccess ||
      cudaMemset(c.meta, 0, (size_t)g.max_slots * sizeof(SlotMeta)) != cudaSuccess ||
      cudaMemset(c.dev_err, 0, sizeof(uint32_t)) != cudaSuccess ||
      cudaMemset(c.xs, 0, (size_t)g.max_requests * c.d * c.esize) != cudaSuccess)
    return fail(TRAIL_ERR_CUDA);
  if (umma_prepare(c) != cudaSuccess || head_prepare(c) != cudaSuccess ||
      pool_prepare() != cudaSuccess || gemv_prepare(c) != cudaSuccess || tf32_prepare(c) != cudaSuccess ||
      fused_prepare(c) != cudaSuccess || wide_prepare(c) != cudaSuccess ||
      select_prepare(c) != cudaSuccess)
    return fail(TRAIL_ERR_CUDA);
  if ((int64_t)max_sched * c.world > select_cluster_capacity()) return fail(TRAIL_ERR_CAPACITY);
  if (cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming) != cudaSuccess)
    return fail(TRAIL_ERR_CUDA);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(TRAIL_ERR_CUDA);
  *out = h;
  return TRAIL_OK;
}

trail_status trail_destroy(trail_handle h) {
  if (!h) return TRAIL_ERR_INVALID;
  set_device(h->c);
  cudaDeviceSynchronize();
  free_ctx(h->c);
  delete h;
  return TRAIL_OK;
}

trail_status trail_trace_enable(trail_handle h, int32_t max_ctas) {
  if (!h || max_ctas < 0) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  if (c.trace) {
    TRAIL_CUDA(cudaDeviceSynchronize());
    cudaFree(c.trace);
    c.trace = nullptr;
    c.trace_cap = 0;
  }
  if (max_ctas == 0) return TRAIL_OK;
  if (cudaMalloc((void **)&c.trace, (size_t)max_ctas * 16 * sizeof(uint64_t)) != cudaSuccess)
    return TRAIL_ERR_NOMEM;
  TRAIL_CUDA(cudaMemset(c.trace, 0, (size_t)max_ctas * 16 * sizeof(uint64_t)));
  c.trace_cap = max_ctas;
  return TRAIL_OK;
}

trail_status trail_trace_read(trail_handle h, uint64_t *host_out, int32_t max_ctas) {
  if (!h || !host_out || max_ctas < 0) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (!c.trace) return TRAIL_ERR_STATE;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  TRAIL_CUDA(cudaDeviceSynchronize());
  const size_t nb = (size_t)std::min(max_ctas, c.trace_cap) * 16 * sizeof(uint64_t);
  TRAIL_CUDA(cudaMemcpy(host_out, c.trace, nb, cudaMemcpyDeviceToHost));
  return TRAIL_OK;
}

trail_status trail_set_l1_mode(trail_handle h, int32_t l1_mode) {
  if (!h || l1_mode < 0 || l1_mode > 5) return TRAIL_ERR_INVALID;
  if (l1_mode >= TRAIL_L1_UMMA && l1_mode <= TRAIL_L1_WIDE && h->c.dtype != TRAIL_BF16)
    return TRAIL_ERR_UNSUPPORTED;
  if (l1_mode == TRAIL_L1_TF32 && h->c.dtype != TRAIL_F32) return TRAIL_ERR_UNSUPPORTED;
  h->c.cfg.l1_mode = l1_mode;
  return TRAIL_OK;
}

trail_status trail_set_prefill_start(trail_handle h, int32_t first_prefill) {
  if (!h || first_prefill < -1) return TRAIL_ERR_INVALID;
  h->c.prefill_start = first_prefill;
  return TRAIL_OK;
}

trail_status trail_set_w1_l2_persist(trail_handle h, int32_t enable) {
  if (!h || enable < 0 || enable > 1) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  const size_t w1_bytes = (size_t)c.H * c.d * c.esize;
  if (enable) {
    int max_persist = 0, max_window = 0;
    if (cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c.device) !=
            cudaSuccess ||
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c.device) !=
            cudaSuccess)
      return TRAIL_ERR_CUDA;
    if (max_persist <= 0 || max_window <= 0) return TRAIL_ERR_UNSUPPORTED;
    const size_t set_aside = std::min(w1_bytes, (size_t)max_persist);
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, set_aside) != cudaSuccess)
      return TRAIL_ERR_CUDA;
    c.w1_window.base_ptr = c.w1;
    c.w1_window.num_bytes = std::min(w1_bytes, (size_t)max_window);
    c.w1_window.hitRatio = std::min(1.0f, (float)set_aside / (float)c.w1_window.num_bytes);
    c.w1_window.hitProp = cudaAccessPropertyPersisting;
    c.w1_window.missProp = cudaAccessPropertyStreaming;
    c.w1_persist = true;
  } else {
    c.w1_persist = false;
    if (cudaCtxResetPersistingL2Cache() != cudaSuccess ||
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0) != cudaSuccess)
      return TRAIL_ERR_CUDA;
  }
  return TRAIL_OK;
}

trail_status trail_set_fill_mode(trail_handle h, int32_t mode) {
  if (!h || mode < 0 || mode > 1) return TRAIL_ERR_INVALID;
  h->c.fill_mode = mode;
  return TRAIL_OK;
}

trail_status trail_set_threshold_mode(trail_handle h, int32_t mode) {
  if (!h || mode < 0 || mode > 1) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  c.host_consts.dyn_c = mode == 1 ? (float)std::min(c.cfg.c, 1e30) : -1.f;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(c.consts, &c.host_consts, sizeof(HeadConsts), cudaMemcpyHostToDevice) != cudaSuccess)
    return TRAIL_ERR_CUDA;
  return TRAIL_OK;
}

trail_status trail_set_rows_hint(trail_handle h, int64_t rows) {
  if (!h || rows < 0) return TRAIL_ERR_INVALID;
  h->c.rows_hint = rows;
  return TRAIL_OK;
}

trail_status trail_plan_l1(trail_handle h, int32_t n, int32_t *l1_mode_out, int32_t *splits_out) {
  if (!h || n < 0) return TRAIL_ERR_INVALID;
  int mode, bn, s;
  plan_l1(h->c, std::max(1, n), &mode, &bn, &s);
  if (l1_mode_out) *l1_mode_out = mode;
  if (splits_out) *splits_out = s;
  return TRAIL_OK;
}

static trail_status predict_body(Ctx &c, const void *emb, int64_t emb_ld,
                                 const int32_t *row_offsets, const uint32_t *request_ids,
                                 const uint8_t *is_prefill, const float *prior_override, int32_t n,
                                 float *posteriors, float *expected_remaining, cudaStream_t s);

trail_status trail_predict_step(trail_handle h, const void *emb, int64_t emb_ld,
                                const int32_t *row_offsets, const uint32_t *request_ids,
                                const uint8_t *is_prefill, const float *prior_override,
                                int32_t n, float *posteriors, float *expected_remaining,
                                trail_stream stream) {
  if (!h) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (n < 0) return TRAIL_ERR_INVALID;
  if (n == 0) return TRAIL_OK;
  if (n > c.cfg.max_requests) return TRAIL_ERR_CAPACITY;
  if (!emb || !row_offsets || !request_ids || !is_prefill) return TRAIL_ERR_INVALID;
  if (emb_ld < c.d || (emb_ld * (int64_t)c.esize) % 16 != 0 || ((uintptr_t)emb) % 16 != 0)
    return TRAIL_ERR_INVALID;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  return predict_body(c, emb, emb_ld, row_offsets, request_ids, is_prefill, prior_override, n,
                      posteriors, expected_remaining, (cudaStream_t)stream);
}

trail_status trail_predict_step_layers(trail_handle h, const void *const *embs,
                                       const float *layer_weights, int32_t n_layers,
                                       int64_t emb_ld, const int32_t *row_offsets,
                                       const uint32_t *request_ids, const uint8_t *is_prefill,
                                       const float *prior_override, int32_t n, float *posteriors,
                                       float *expected_remaining, trail_stream stream) {
  if (!h) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (n < 0 || n_layers < 1 || n_layers > kMaxLayers || !embs || !layer_weights)
    return TRAIL_ERR_INVALID;
  if (n == 0) return TRAIL_OK;
  if (n > c.cfg.max_requests) return TRAIL_ERR_CAPACITY;
  if (!row_offsets || !request_ids || !is_prefill) return TRAIL_ERR_INVALID;
  if (emb_ld < c.d || (emb_ld * (int64_t)c.esize) % 16 != 0) return TRAIL_ERR_INVALID;
  double wsum = 0.0;
  for (int l = 0; l < n_layers; ++l) {
    if (!embs[l] || ((uintptr_t)embs[l]) % 16 != 0) return TRAIL_ERR_INVALID;
    if (!(layer_weights[l] >= 0.f) || !std::isfinite(layer_weights[l])) return TRAIL_ERR_INVALID;
    wsum += (double)layer_weights[l];
  }
  if (!(wsum > 0.0)) return TRAIL_ERR_INVALID;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  if (!c.xmix) {   // lazily: [max_requests][d] probe inputs + the one-row-per-request offsets
    if (cudaMalloc(&c.xmix, (size_t)c.cfg.max_requests * c.d * c.esize) != cudaSuccess ||
        cudaMalloc(&c.iota, ((size_t)c.cfg.max_requests + 1) * sizeof(int32_t)) != cudaSuccess)
      return TRAIL_ERR_NOMEM;
    std::vector<int32_t> io((size_t)c.cfg.max_requests + 1);
    for (size_t i = 0; i < io.size(); ++i) io[i] = (int32_t)i;
    if (cudaMemcpy(c.iota, io.data(), io.size() * sizeof(int32_t), cudaMemcpyHostToDevice) !=
        cudaSuccess)
      return TRAIL_ERR_CUDA;
  }
  MixArgs ma = {};
  ma.L = n_layers;
  for (int l = 0; l < n_layers; ++l) {
    ma.emb[l] = embs[l];
    ma.a[l] = (double)layer_weights[l] / wsum;
  }
  cudaStream_t s = (cudaStream_t)stream;
  {
    ProfScope p(c, TRAIL_K_POOL, s);
    TRAIL_CUDA(launch_layer_mix(c, ma, emb_ld, row_offsets, n, s));
  }
  return predict_body(c, c.xmix, c.d, c.iota, request_ids, is_prefill, prior_override, n,
                      posteriors, expected_remaining, s);
}

namespace {
struct L1Window {        // scope of the layer-1 launches of one predict step
  explicit L1Window(const Ctx &c) { tl_l1_window = c.w1_persist ? &c.w1_window : nullptr; }
  ~L1Window() { tl_l1_window = nullptr; }
};
}  // namespace

static trail_status predict_body(Ctx &c, const void *emb, int64_t emb_ld,
                                 const int32_t *row_offsets, const uint32_t *request_ids,
                                 const uint8_t *is_prefill, const float *prior_override, int32_t n,
                                 float *posteriors, float *expected_remaining, cudaStream_t s) {
  int mode, bn, splits;
  plan_l1(c, n, &mode, &bn, &splits);
  if (mode != TRAIL_L1_UMMA && mode != TRAIL_L1_WIDE && (size_t)splits * n * c.H > c.partial_elems)
    return TRAIL_ERR_CAPACITY;
  if (mode == TRAIL_L1_WIDE && c.side && c.prefill_start > 0 && c.prefill_start < n) {
    // decode / prefill split (trail_set_prefill_start, opt-in): the CTA pairs take the decode
    // tiles [0, t) on 2*(t/256) SMs at once; the side stream pools the tail's prompts on the
    // remaining SMs and runs the tail [t, n) through the split-K kernel.  Measured at
    // configs[3]: K2d 158 -> 144 us, but the side path (K1 on 22 SMs 98 us + K2c 81 us) is
    // longer than K1 + K2d in series, so the step gets slower (239 -> 250 us); kept as an
    // opt-in for batches with fewer prompt rows or parts with more spare SMs
    const int t = (c.prefill_start / 256) * 256;     // whole CTA-pair tiles
    const int nt = n - t;
    const int pairs = (t + 255) / 256;
    const int spare = c.num_sms - 2 * pairs;
    const int tiles_tail = ((nt + 127) / 128) * (c.H / 128);
    if (t >= 256 && spare >= 8 && tiles_tail <= spare) {
      TRAIL_CUDA(cudaEventRecord(c.ev_fork, s));
      TRAIL_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
      {
        ProfScope p(c, TRAIL_K_POOL, c.side);
        TRAIL_CUDA(launch_pool(c, emb, emb_ld, row_offsets + t, nt, 0, c.side, spare));
      }
      L1Window l1w(c);          // W1 access-policy window (if enabled) on the layer-1 launches
      {
        ProfScope p(c, TRAIL_K_GEMV, c.side);   // (profiling slot of the tail's layer 1)
        const int sp = std::max(1, std::min(spare / tiles_tail, c.d / 64));
        TRAIL_CUDA(launch_fused_predict(c, emb, emb_ld, row_offsets + t, nt, std::min(sp, 16),
                                        request_ids + t, is_prefill + t,
                                        prior_override ? prior_override + (int64_t)t * c.k : nullptr,
                                        posteriors ? posteriors + (int64_t)t * c.k : nullptr,
                                        expected_remaining ? expected_remaining + t : nullptr,
                                        c.side));
      }
      TRAIL_CUDA(cudaEventRecord(c.ev_join, c.side));
      {
        ProfScope p(c, TRAIL_K_UMMA, s);
        TRAIL_CUDA(launch_wide_predict(c, emb, emb_ld, row_offsets, t, request_ids, is_prefill,
                                       prior_override, posteriors, expected_remaining, s, 1));
      }
      TRAIL_CUDA(cudaStreamWaitEvent(s, c.ev_join, 0));
      return TRAIL_OK;
    }
  }
  {
    ProfScope p(c, TRAIL_K_POOL, s);
    // decode rows are gathered from emb by every layer-1 kernel except the unfused GEMM
    TRAIL_CUDA(launch_pool(c, emb, emb_ld, row_offsets, n, mode == TRAIL_L1_UMMA_UNFUSED ? 1 : 0, s));
  }
  L1Window l1w(c);              // W1 access-policy window (if enabled) on the layer-1 launches
  if (mode == TRAIL_L1_WIDE) {   // layer 1 + layer 2 + head, CTA pairs over the whole hidden width
    ProfScope p(c, TRAIL_K_UMMA, s);
    TRAIL_CUDA(launch_wide_predict(c, emb, emb_ld, row_offsets, n, request_ids, is_prefill,
                                   prior_override, posteriors, expected_remaining, s));
    return TRAIL_OK;
  }
  if (mode == TRAIL_L1_UMMA) {   // layer 1 + layer 2 + head in one kernel
    ProfScope p(c, TRAIL_K_UMMA, s);
    TRAIL_CUDA(launch_fused_predict(c, emb, emb_ld, row_offsets, n, splits, request_ids,
                                    is_prefill, prior_override,
                                    posteriors, expected_remaining, s));
    return TRAIL_OK;
  }
  if (mode == TRAIL_L1_GEMV) {
    ProfScope p(c, TRAIL_K_GEMV, s);
    TRAIL_CUDA(launch_gemv_l1(c, emb, emb_ld, row_offsets, n, splits, s));
  } else if (mode == TRAIL_L1_TF32) {
    ProfScope p(c, TRAIL_K_GEMV, s);   // (the layer-1 profiling slot of the fp32 path)
    TRAIL_CUDA(launch_tf32_l1(c, emb, emb_ld, row_offsets, n, s));
  } else {
    ProfScope p(c, TRAIL_K_UMMA, s);
    TRAIL_CUDA(launch_umma_l1(c, n, bn, splits, s));
  }
  tl_l1_window = nullptr;        // the head reads no W1
  {
    ProfScope p(c, TRAIL_K_HEAD, s);
    TRAIL_CUDA(launch_head(c, n, splits, request_ids, is_prefill, prior_override, posteriors,
                           expected_remaining, s));
  }
  return TRAIL_OK;
}

trail_status trail_prefill_chunk(trail_handle h, const void *emb, int64_t emb_ld,
                                 const int32_t *row_offsets, const uint32_t *request_ids,
                                 const uint8_t *is_final, int32_t n, void *pooled,
                                 int64_t pooled_ld, trail_stream stream) {
  if (!h || n < 0) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (n == 0) return TRAIL_OK;
  if (!emb || !row_offsets || !request_ids || !is_final || !pooled) return TRAIL_ERR_INVALID;
  if (emb_ld < c.d || pooled_ld < c.d || (emb_ld * (int64_t)c.esize) % 16 != 0 ||
      (pooled_ld * (int64_t)c.esize) % 16 != 0 || ((uintptr_t)emb) % 16 != 0 ||
      ((uintptr_t)pooled) % 16 != 0)
    return TRAIL_ERR_INVALID;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  TRAIL_CUDA(launch_prefill_chunk(c, emb, emb_ld, row_offsets, request_ids, is_final, n, pooled,
                                  pooled_ld, (cudaStream_t)stream));
  return TRAIL_OK;
}

trail_status trail_time_update(trail_handle h, const uint32_t *request_ids, int32_t n,
                               int32_t steps, float *posteriors, float *expected_remaining,
                               trail_stream stream) {
  if (!h || n < 0 || steps < 0) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (n == 0) return TRAIL_OK;
  if (!request_ids) return TRAIL_ERR_INVALID;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope p(c, TRAIL_K_HEAD, s);
  TRAIL_CUDA(launch_time_update(c, request_ids, n, steps, posteriors, expected_remaining, s));
  return TRAIL_OK;
}

trail_status trail_schedule_pack(trail_handle h, const uint32_t *request_ids,
                                 const uint32_t *arrival_seq, const int32_t *kv_blocks,
                                 const uint8_t *is_running, int32_t n, int32_t capacity,
                                 void *records, trail_stream stream) {
  if (!h || n < 0 || capacity < n) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (capacity == 0) return TRAIL_OK;
  if (!records || (n > 0 && (!request_ids || !arrival_seq || !kv_blocks || !is_running)))
    return TRAIL_ERR_INVALID;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope p(c, TRAIL_K_PACK, s);
  TRAIL_CUDA(launch_pack(c, request_ids, arrival_seq, kv_blocks, is_running, n, (Record *)records,
                         capacity, s));
  return TRAIL_OK;
}

trail_status trail_schedule_select(trail_handle h, const void *records, int32_t n_records,
                                   int64_t kv_budget, int32_t max_run, uint32_t *run_ids,
                                   uint32_t *preempt_ids, uint32_t *admit_ids,
                                   int32_t *counts, trail_stream stream) {
  if (!h || n_records < 0 || max_run < 0) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (!counts || (n_records > 0 && (!records || !run_ids || !preempt_ids || !admit_ids)))
    return TRAIL_ERR_INVALID;
  if ((int64_t)n_records > (int64_t)std::max(1, c.cfg.max_sched) * c.world)
    return TRAIL_ERR_CAPACITY;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope p(c, TRAIL_K_SELECT, s);
  TRAIL_CUDA(launch_select(c, (const Record *)records, n_records, kv_budget, max_run, run_ids,
                           preempt_ids, admit_ids, counts, s));
  return TRAIL_OK;
}

trail_status trail_schedule_step(trail_handle h, const uint32_t *request_ids,
                                 const uint32_t *arrival_seq, const int32_t *kv_blocks,
                                 const uint8_t *is_running, int32_t n, int64_t kv_budget,
                                 int32_t max_run, uint32_t *run_ids, uint32_t *preempt_ids,
                                 uint32_t *admit_ids, int32_t *counts, trail_stream stream) {
  if (!h || n < 0 || max_run < 0) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (n > std::max(0, c.cfg.max_sched)) return TRAIL_ERR_CAPACITY;
  if (!counts || !run_ids || !preempt_ids || !admit_ids) return TRAIL_ERR_INVALID;
  if (n > 0 && (!request_ids || !arrival_seq || !kv_blocks || !is_running))
    return TRAIL_ERR_INVALID;
  if (c.world > 1 && !c.nccl_comm) return TRAIL_ERR_STATE;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  if (!c.nccl_comm && n <= select_local_capacity()) {
    // local selection: the record build is fused into the selection kernel
    ProfScope p(c, TRAIL_K_SELECT, s);
    TRAIL_CUDA(launch_select_local(c, request_ids, arrival_seq, kv_blocks, is_running, n,
                                   kv_budget, max_run, run_ids, preempt_ids, admit_ids, counts,
                                   s));
    return TRAIL_OK;
  }
  const int npad = c.nccl_comm ? std::max(1, c.cfg.max_sched) : n;
  {
    ProfScope p(c, TRAIL_K_PACK, s);
    TRAIL_CUDA(launch_pack(c, request_ids, arrival_seq, kv_blocks, is_running, n, c.rec_local,
                           npad, s));
  }
  const Record *sel_in = c.rec_local;
  int total = n;
  if (c.nccl_comm) {
    NcclApi &api = nccl();
    ProfScope p(c, TRAIL_K_GATHER, s);
    ncclResult_t r = api.allGather(c.rec_local, c.rec_all, (size_t)npad * sizeof(Record),
                                   ncclUint8, (ncclComm_t)c.nccl_comm, s);
    if (r != ncclSuccess) {
      fprintf(stderr, "[trail] ncclAllGather: %s\n", api.errStr ? api.errStr(r) : "?");
      return TRAIL_ERR_NCCL;
    }
    sel_in = c.rec_all;
    total = npad * c.world;
  }
  ProfScope p(c, TRAIL_K_SELECT, s);
  TRAIL_CUDA(launch_select(c, sel_in, total, kv_budget, max_run, run_ids, preempt_ids, admit_ids,
                           counts, s));
  return TRAIL_OK;
}

trail_status trail_release(trail_handle h, const uint32_t *request_ids, int32_t n,
                           trail_stream stream) {
  if (!h || n < 0) return TRAIL_ERR_INVALID;
  if (n == 0) return TRAIL_OK;
  if (!request_ids) return TRAIL_ERR_INVALID;
  if (set_device(h->c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  TRAIL_CUDA(launch_release(h->c, request_ids, n, (cudaStream_t)stream));
  return TRAIL_OK;
}

trail_status trail_read_state(trail_handle h, const uint32_t *request_ids, int32_t n, float *L,
                              uint32_t *age, uint32_t *threshold, uint8_t *seen,
                              float *posterior, trail_stream stream) {
  if (!h || n < 0) return TRAIL_ERR_INVALID;
  if (n == 0) return TRAIL_OK;
  if (!request_ids) return TRAIL_ERR_INVALID;
  if (set_device(h->c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  TRAIL_CUDA(launch_read_state(h->c, request_ids, n, L, age, threshold, seen, posterior,
                               (cudaStream_t)stream));
  return TRAIL_OK;
}

trail_status trail_nccl_unique_id(void *id_out) {
  if (!id_out) return TRAIL_ERR_INVALID;
  NcclApi &api = nccl();
  if (!api.ok) return TRAIL_ERR_NCCL;
  ncclUniqueId id;
  if (api.getUniqueId(&id) != ncclSuccess) return TRAIL_ERR_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return TRAIL_OK;
}

trail_status trail_comm_init(trail_handle h, const void *id, int32_t rank, int32_t world_size) {
  if (!h || !id || rank < 0 || world_size < 1 || rank >= world_size) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (world_size != c.world) return TRAIL_ERR_INVALID;
  if (c.nccl_comm) return TRAIL_ERR_STATE;
  NcclApi &api = nccl();
  if (!api.ok) return TRAIL_ERR_NCCL;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  ncclResult_t r = api.commInitRank(&comm, world_size, uid, rank);
  if (r != ncclSuccess) {
    fprintf(stderr, "[trail] ncclCommInitRank: %s\n", api.errStr ? api.errStr(r) : "?");
    return TRAIL_ERR_NCCL;
  }
  c.nccl_comm = comm;
  c.rank = rank;
  return TRAIL_OK;
}

trail_status trail_device_errors(trail_handle h, uint32_t *bits_out, int32_t clear) {
  if (!h || !bits_out) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
  TRAIL_CUDA(cudaDeviceSynchronize());
  TRAIL_CUDA(cudaMemcpy(bits_out, c.dev_err, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  if (clear) TRAIL_CUDA(cudaMemset(c.dev_err, 0, sizeof(uint32_t)));
  return TRAIL_OK;
}

trail_status trail_profile_enable(trail_handle h, int32_t enable) {
  if (!h) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (enable == 2) {
    if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
    for (int i = 0; i < TRAIL_K_COUNT; ++i)
      for (int j = 0; j < 2; ++j)
        if (!c.last_ev[i][j]) TRAIL_CUDA(cudaEventCreate(&c.last_ev[i][j]));
    c.prof_mode = 2;
    c.prof = true;
    return TRAIL_OK;
  }
  c.prof_mode = enable ? 1 : 0;
  if (enable && !c.prof_ev) {
    if (set_device(c) != TRAIL_OK) return TRAIL_ERR_CUDA;
    c.prof_cap = 8192;
    c.prof_ev = new (std::nothrow) cudaEvent_t[2 * c.prof_cap];
    c.prof_kid = new (std::nothrow) int[c.prof_cap];
    if (!c.prof_ev || !c.prof_kid) return TRAIL_ERR_NOMEM;
    for (int i = 0; i < 2 * c.prof_cap; ++i) TRAIL_CUDA(cudaEventCreate(&c.prof_ev[i]));
  }
  c.prof = enable != 0;
  return TRAIL_OK;
}

trail_status trail_profile_read(trail_handle h, int32_t kid, double *total_ms, int64_t *launches,
                                int32_t reset) {
  if (!h || kid < 0 || kid >= TRAIL_K_COUNT) return TRAIL_ERR_INVALID;
  Ctx &c = h->c;
  if (c.prof_mode == 2) {   // duration of the most recent launch of `kid`
    double ms = 0.0;
    int64_t cnt = 0;
    if (c.last_used[kid]) {
      float f = 0.f;
      TRAIL_CUDA(cudaEventSynchronize(c.last_ev[kid][1]));
      TRAIL_CUDA(cudaEventElapsedTime(&f, c.last_ev[kid][0], c.last_ev[kid][1]));
      ms = f;
      cnt = 1;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = cnt;
    return TRAIL_OK;
  }
  if (c.prof_n > 0) {
    TRAIL_CUDA(cudaEventSynchronize(c.prof_ev[2 * (c.prof_n - 1) + 1]));
    for (int i = 0; i < c.prof_n; ++i) {
      float ms = 0.f;
      TRAIL_CUDA(cudaEventElapsedTime(&ms, c.prof_ev[2 * i], c.prof_ev[2 * i + 1]));
      c.prof_ms[c.prof_kid[i]] += ms;
      c.prof_cnt[c.prof_kid[i]] += 1;
    }
    c.prof_n = 0;
  }
  if (total_ms) *total_ms = c.prof_ms[kid];
  if (launches) *launches = c.prof_cnt[kid];
  if (reset) {
    for (int i = 0; i < TRAIL_K_COUNT; ++i) { c.prof_ms[i] = 0; c.prof_cnt[i] = 0; }
  }
  return TRAIL_OK;
}

}  // extern "C"

namespace trail {
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("TRAIL_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// Selection kernel: default = multi-CTA rank counting (k_rank.cu) up to its capacity;
// TRAIL_SELECT=radix / bitonic forces the single-CTA radix or bitonic kernels (comparisons).
int select_impl() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("TRAIL_SELECT");
    v = (e && e[0] == 'c') ? 2 : 0;   // "cluster": the single-cluster kernel for every size
  }
  return v;
}
int select_local_capacity() { return select_cluster_capacity(); }
cudaError_t launch_select_local(const Ctx &c, const uint32_t *ids, const uint32_t *arrival,
                                const int32_t *kv, const uint8_t *running, int n, int64_t budget,
                                int max_run, uint32_t *run, uint32_t *pre, uint32_t *adm,
                                int32_t *counts, cudaStream_t s) {
  return launch_select_any(c, nullptr, c.rec_local, ids, arrival, kv, running, n, budget,
                           max_run, run, pre, adm, counts, s);
}
}  // namespace trail
