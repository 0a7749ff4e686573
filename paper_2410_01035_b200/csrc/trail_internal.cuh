// trail_internal.cuh — shared definitions of libtrail.so (CUDA path only; the oracle
// under oracle/ shares nothing with this file).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/trail.h"

namespace trail {

constexpr int kMaxBins = 32;      // one warp lane per bin in the head kernel
constexpr int kMaxHidden = 512;   // TMEM columns (fp32) of one 128-row accumulator
constexpr int kRecordBytes = 16;
constexpr uint32_t kPadKey = 0xFFFFFFFFu;

// Per-slot state (16 B) + log-posterior row [k] kept separately.
struct SlotMeta {
  float L;          // expected remaining length L_t
  uint32_t age;     // decode iterations since the first observation (D-11)
  uint32_t thr;     // floor(c * r) (D-10); 0xFFFFFFFF = never frozen
  uint32_t flags;   // bit0 = observed
};

struct Record {     // 16-byte record exchanged between ranks (row a4/a5)
  uint32_t keybits; // (!forced) << 31 | fp32 bits of the key
  uint32_t arrival;
  uint32_t kv;
  uint32_t gid;     // (id_base + slot) & 0x7FFFFFFF | running << 31
};

// Constants uploaded once at create (device copies).
struct HeadConsts {
  float m[kMaxBins];        // bin midpoints m_i
  float log_stay[kMaxBins]; // log(1 - 1/w_i)          (T_ii, D-1)
  float log_move[kMaxBins]; // log(1/w_{i+1}), -inf at i = k-1  (T_{i,i+1})
  float log_prior[kMaxBins];// log pi_i
  uint32_t thr_tab[kMaxBins];// floor(c * m_i) (fp64 on host), 0xFFFFFFFF for c = inf
  float prior_L;            // E_pi[L] (D-24)
  int k;
  int H;
  float dyn_c;              // < 0: static threshold floor(c r); else the dynamic
                            // variant: forced iff a >= c (a + L_t)
};

// Dynamic-threshold variant: the smallest integer age a with a >= c (a + L), i.e.
// a >= c L / (1 - c) for c < 1 (never for c >= 1), recomputed whenever L changes and stored
// as the slot threshold, so every selection kernel keeps testing a >= thr.
__host__ __device__ __forceinline__ uint32_t dynamic_threshold(float c, float L) {
  if (!(c < 1.f)) return 0xFFFFFFFFu;
  const float t = ceilf(c * L / (1.f - c));
  return t >= 4294967040.f ? 0xFFFFFFFEu : (t <= 0.f ? 0u : (uint32_t)t);
}

// Row a4 (record build): key = L_t of the slot (E_pi[L] if never observed, D-24); forced =
// running & observed & a >= threshold (rank -inf); a bad slot id keys +inf
// (sorts last, never displaces a valid request) and a negative KV counts 0, both flagged.
__device__ __forceinline__ Record build_record(uint32_t slot, uint32_t arrival, int32_t kvb,
                                               bool run, const SlotMeta *__restrict__ meta,
                                               const HeadConsts *__restrict__ cst,
                                               int max_slots, uint32_t id_base,
                                               uint32_t *__restrict__ err) {
  if (kvb < 0) { atomicOr(err, TRAIL_DEV_NEG_KV); kvb = 0; }
  float key = cst->prior_L;
  bool forced = false;
  if (slot < (uint32_t)max_slots) {
    const SlotMeta mt = meta[slot];
    if (mt.flags & 1u) {
      key = mt.L;
      forced = run && (mt.age >= mt.thr);
    }
  } else {
    atomicOr(err, TRAIL_DEV_BAD_ID);
    key = INFINITY;
  }
  uint32_t kb;
  if (isfinite(key) && key >= 0.f) {
    kb = __float_as_uint(key) & 0x7FFFFFFFu;
  } else {
    if (slot < (uint32_t)max_slots) atomicOr(err, TRAIL_DEV_NONFIN);
    kb = 0x7F800000u;
  }
  Record r;
  r.keybits = (forced ? 0u : 0x80000000u) | kb;
  r.arrival = arrival;
  r.kv = (uint32_t)kvb;
  r.gid = ((id_base + slot) & 0x7FFFFFFFu) | (run ? 0x80000000u : 0u);
  return r;
}

struct Ctx {
  trail_config cfg;
  int device = 0;
  int d = 0, H = 0, k = 0, dtype = 0;
  size_t esize = 2;            // bytes per W1/embedding element
  // weights
  void *w1 = nullptr;          // [H][d] dtype
  float *b1 = nullptr, *w2 = nullptr, *b2 = nullptr;
  HeadConsts *consts = nullptr;   // device
  HeadConsts host_consts;
  // state
  float *lq = nullptr;         // [max_slots][k]
  SlotMeta *meta = nullptr;    // [max_slots]
  uint32_t *dev_err = nullptr; // sticky bits
  // workspaces
  void *xs = nullptr;          // [max_requests][d] staged embeddings (dtype)
  float *partial = nullptr;    // [S][n][H] layer-1 split-K partials
  size_t partial_elems = 0;
  float *zpart = nullptr;      // [max_requests][H/128][k] fused kernel: layer-2 partial logits
  uint32_t *arrive_cnt = nullptr;  // [m_tiles][16] fused kernel: column-tile arrival counters
  uint64_t *trace = nullptr;   // diagnostics: per-CTA phase timestamps (trail_trace_enable)
  int trace_cap = 0;           // CTAs the trace buffer holds (16 u64 each)
  int fused_max_clusters[17] = {};
  float *chunk_acc = nullptr;       // [max_slots][d] chunked-prefill running sums (lazy)
  uint32_t *chunk_cnt = nullptr;    // [max_slots] rows accumulated so far
  void *xmix = nullptr;             // [max_requests][d] multi-layer probe inputs (lazy)
  int32_t *iota = nullptr;          // [max_requests + 1] 0, 1, 2, ... (one row per request)
  float *pool_head = nullptr;       // [pool_grid][d] K1 partial sums (request began earlier)
  float *pool_tail = nullptr;       // [pool_grid][d] K1 partial sums (request continues)
  uint32_t *pool_cnt = nullptr;     // [max_requests] K1 per-request chunk arrival counters
  void *bk_ws = nullptr;            // bucketed selection workspace (k_bucket.cu)
  int bk_cap = 0;                   // records it holds
  Record *rank_sorted = nullptr;    // [max_sched * world] rank-select scatter target
  uint32_t *rank_cnt = nullptr;     // rank-select CTA completion counter  // fused kernel: resident clusters of size s (occupancy)
  Record *rec_local = nullptr; // [max_sched]
  Record *rec_all = nullptr;   // [max_sched * world]
  // TMA descriptors (bf16 path)
  CUtensorMap tmap_x, tmap_w128, tmap_w256;
  CUtensorMap tmap_w_gemv;                       // W1, 16-byte x 64-row boxes (K2a)
  bool have_tmap_gemv = false;
  CUtensorMap tmap_w_tf32;                       // fp32 SW128 maps (K2t): W1 128-row boxes,
  CUtensorMap tmap_xs_tf32[3], tmap_e_tf32[3];   // xs / caller rows in 1-, 4-, 32-row boxes
  bool have_tmap_tf32 = false;
  const void *tmap_e_tf32_ptr = nullptr;
  int64_t tmap_e_tf32_ld = 0;
  CUtensorMap tmap_xs1, tmap_xs4, tmap_xs32;     // xs rows, boxes 64 x {1, 4, 32} (fused gather)
  CUtensorMap tmap_emb, tmap_emb4, tmap_emb32;   // caller's embeddings, same boxes; re-encoded
                                                 // whenever emb / ld change
  const void *tmap_emb_ptr = nullptr;
  int64_t tmap_emb_ld = 0;
  bool have_tmaps = false;
  int num_sms = 148;
  int64_t rows_hint = 0;        // trail_set_rows_hint: embedding rows of the next predict steps
  int fill_mode = 0;            // trail_set_fill_mode: 0 strict prefix (D-15), 1 first-fit
  bool w1_persist = false;      // trail_set_w1_l2_persist
  int prefill_start = -1;       // trail_set_prefill_start: requests before it are single-row
  cudaStream_t side = nullptr;  // the prefill tail's stream (decode/prefill split)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaAccessPolicyWindow w1_window = {};
  // NCCL
  void *nccl_comm = nullptr;
  int rank = 0, world = 1;
  // profiling
  bool prof = false;
  int prof_n = 0;
  cudaEvent_t *prof_ev = nullptr;   // pairs
  int *prof_kid = nullptr;
  int prof_cap = 0;
  double prof_ms[TRAIL_K_COUNT] = {0};
  int64_t prof_cnt[TRAIL_K_COUNT] = {0};
  // mode 2 (graph-friendly): one fixed event pair per kernel id, re-recorded every launch
  // (also by CUDA-graph event-record nodes captured while profiling)
  int prof_mode = 0;
  cudaEvent_t last_ev[TRAIL_K_COUNT][2] = {};
  bool last_used[TRAIL_K_COUNT] = {};
};

// ---------------------------------------------------------------- launchers (host)
// K1.  write_singles = 0: single-row requests are not copied to xs (the fused tcgen05
// kernel gathers those rows straight from emb)
cudaError_t launch_pool(const Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                        int write_singles, cudaStream_t s, int grid = 0);
int pool_grid(const Ctx &c);
bool pool_use_bulk();
cudaError_t pool_prepare();
cudaError_t gemv_prepare(Ctx &c);
bool encode_plain_2d(CUtensorMap *m, const void *base, bool bf16, uint64_t cols, uint64_t rows,
                     uint64_t ld, uint32_t box_cols, uint32_t box_rows);
cudaError_t launch_gemv_l1(const Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                           int splits, cudaStream_t s);
cudaError_t launch_umma_l1(const Ctx &c, int n, int bn, int splits, cudaStream_t s);
cudaError_t launch_head(const Ctx &c, int n, int splits, const uint32_t *ids,
                        const uint8_t *is_prefill, const float *prior_override,
                        float *post, float *L, cudaStream_t s);
cudaError_t launch_pack(const Ctx &c, const uint32_t *ids, const uint32_t *arrival,
                        const int32_t *kv, const uint8_t *running, int n, Record *out,
                        int n_pad_to, cudaStream_t s);
cudaError_t launch_select(const Ctx &c, const Record *rec, int n, int64_t budget, int max_run,
                          uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                          cudaStream_t s);
cudaError_t launch_time_update(const Ctx &c, const uint32_t *ids, int n, int steps, float *post,
                               float *L, cudaStream_t s);
constexpr int kMaxLayers = 8;
struct MixArgs {                  // multi-layer weighted embeddings (k_mix.cu, reading D-28)
  const void *emb[kMaxLayers];
  double a[kMaxLayers];           // normalised weights (fp64, host)
  int L;
};
cudaError_t launch_layer_mix(Ctx &c, const MixArgs &ma, int64_t ld, const int32_t *off, int n,
                             cudaStream_t s);
cudaError_t launch_prefill_chunk(Ctx &c, const void *emb, int64_t ld, const int32_t *off,
                                 const uint32_t *ids, const uint8_t *is_final, int n,
                                 void *pooled, int64_t pld, cudaStream_t s);
cudaError_t launch_release(const Ctx &c, const uint32_t *ids, int n, cudaStream_t s);
cudaError_t launch_read_state(const Ctx &c, const uint32_t *ids, int n, float *L, uint32_t *age,
                              uint32_t *thr, uint8_t *seen, float *post, cudaStream_t s);
cudaError_t umma_prepare(Ctx &c);
// K2t (k_tf32.cu): 3xTF32 tcgen05 layer 1 for fp32 handles
bool encode_rows_f32_sw128(CUtensorMap *m, const void *base, uint64_t cols, uint64_t rows,
                           uint64_t ld, uint32_t box_cols, uint32_t box_rows);
cudaError_t tf32_prepare(Ctx &c);
bool tf32_supported(const Ctx &c);
int tf32_splits(const Ctx &c);
cudaError_t launch_tf32_l1(Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                           cudaStream_t s);
bool encode_rows_bf16(CUtensorMap *m, const void *base, uint64_t cols, uint64_t rows, uint64_t ld,
                      uint32_t box_cols, uint32_t box_rows);                // encode tensor maps, set smem attributes
int umma_max_bn(const Ctx &c);
cudaError_t fused_prepare(Ctx &c);
int fused_splits(const Ctx &c, int n);
cudaError_t launch_fused_predict(Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                                 int splits, const uint32_t *ids,
                                 const uint8_t *is_prefill, const float *prior_override,
                                 float *post, float *L, cudaStream_t s);
bool ensure_emb_tmaps(Ctx &c, const void *emb, int64_t ld);
bool wide_supported(const Ctx &c);
int wide_min_n();
cudaError_t wide_prepare(Ctx &c);
cudaError_t launch_wide_predict(Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                                const uint32_t *ids, const uint8_t *is_prefill,
                                const float *prior_override, float *post, float *L,
                                cudaStream_t s, int decode_only = 0);
cudaError_t select_prepare(Ctx &c);
// K4 selection: one thread-block cluster (k_csort.cu).  rec_in != nullptr: select over given
// records; else build the local records (fused K5 pack) from (ids, arrival, kv, running)
// into rec_out and select over them.
cudaError_t select_cluster_prepare();
int select_cluster_capacity();
cudaError_t launch_select_cluster(const Ctx &c, const Record *rec_in, Record *rec_out,
                                  const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                                  const uint8_t *running, int m, int64_t budget, int max_run,
                                  uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                                  cudaStream_t s);
// default dispatch: rank-counting kernel (k_rank.cu) up to kRankMaxRecords records, the
// bucketed kernels (k_bucket.cu) above; the cluster kernel for first-fit filling and as
// TRAIL_SELECT=cluster
int select_impl();
int select_local_capacity();
cudaError_t launch_select_any(const Ctx &c, const Record *rec_in, Record *rec_out,
                              const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                              const uint8_t *running, int n, int64_t budget, int max_run,
                              uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                              cudaStream_t s);
cudaError_t launch_select_local(const Ctx &c, const uint32_t *ids, const uint32_t *arrival,
                                const int32_t *kv, const uint8_t *running, int n, int64_t budget,
                                int max_run, uint32_t *run, uint32_t *pre, uint32_t *adm,
                                int32_t *counts, cudaStream_t s);
cudaError_t select_rank_prepare();
cudaError_t select_bucket_prepare();
size_t bucket_workspace_bytes(int m_max);
cudaError_t launch_select_bucket(const Ctx &c, const Record *rec_in, Record *rec_out,
                                 const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                                 const uint8_t *running, int m, int64_t budget,
                                 int max_run, uint32_t *run, uint32_t *pre, uint32_t *adm,
                                 int32_t *counts, cudaStream_t s);
constexpr int kRankMaxRecords = 2048;
cudaError_t launch_select_rank(const Ctx &c, const Record *rec_in, Record *rec_out,
                               const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                               const uint8_t *running, int n, int64_t budget, int max_run,
                               uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                               cudaStream_t s);
cudaError_t head_prepare(Ctx &c);

// ---------------------------------------------------------------- launch helper
// Programmatic dependent launch (PDL): consecutive kernels of a step overlap the next
// kernel's launch + prologue with the previous kernel's tail.  Every kernel executes
// griddep_wait() before touching data produced by an earlier kernel and
// griddep_launch() once all its CTAs are resident (so a waiting dependent can never
// starve it of SM resources).
bool pdl_enabled();

// L2-persisting W1 (optional; trail_set_w1_l2_persist): while a layer-1 kernel
// is launched, this points at the access-policy window over W1 and every launch made through
// launch_k / add_l1_window carries it (set and cleared by predict_body, one host thread per
// handle).
extern thread_local const cudaAccessPolicyWindow *tl_l1_window;
inline int add_l1_window(cudaLaunchAttribute *attr, int na) {
  if (tl_l1_window) {
    attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[na].val.accessPolicyWindow = *tl_l1_window;
    ++na;
  }
  return na;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  na = add_l1_window(attr, na);
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace trail
