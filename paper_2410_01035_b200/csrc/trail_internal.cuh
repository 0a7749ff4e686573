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
  float *pool_head = nullptr;       // [pool_grid][d] K1 partial sums (request began earlier)
  float *pool_tail = nullptr;       // [pool_grid][d] K1 partial sums (request continues)
  uint32_t *pool_cnt = nullptr;     // [max_requests] K1 per-request chunk arrival counters
  void *bk_ws = nullptr;            // bucketed selection workspace (k_bucket.cu)
  int bk_cap = 0;                   // records it holds
  Record *rank_sorted = nullptr;    // [max_sched * world] rank-select scatter target
  uint32_t *rank_cnt = nullptr;     // rank-select CTA completion counter  // fused kernel: resident clusters of size s (occupancy)
  Record *rec_local = nullptr; // [max_sched]
  Record *rec_all = nullptr;   // [max_sched * world]
  void *sel_scratch = nullptr; // global scratch for large selections
  size_t sel_scratch_bytes = 0;
  // TMA descriptors (bf16 path)
  CUtensorMap tmap_x, tmap_w128, tmap_w256;
  CUtensorMap tmap_w_gemv;                       // W1, 16-byte x 64-row boxes (K2a)
  bool have_tmap_gemv = false;
  CUtensorMap tmap_xs1, tmap_xs4, tmap_xs32;     // xs rows, boxes 64 x {1, 4, 32} (fused gather)
  CUtensorMap tmap_emb, tmap_emb4, tmap_emb32;   // caller's embeddings, same boxes; re-encoded
                                                 // whenever emb / ld change
  const void *tmap_emb_ptr = nullptr;
  int64_t tmap_emb_ld = 0;
  bool have_tmaps = false;
  int num_sms = 148;
  int64_t rows_hint = 0;        // trail_set_rows_hint: embedding rows of the next predict steps
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
                        int write_singles, cudaStream_t s);
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
cudaError_t launch_prefill_chunk(Ctx &c, const void *emb, int64_t ld, const int32_t *off,
                                 const uint32_t *ids, const uint8_t *is_final, int n,
                                 void *pooled, int64_t pld, cudaStream_t s);
cudaError_t launch_release(const Ctx &c, const uint32_t *ids, int n, cudaStream_t s);
cudaError_t launch_read_state(const Ctx &c, const uint32_t *ids, int n, float *L, uint32_t *age,
                              uint32_t *thr, uint8_t *seen, float *post, cudaStream_t s);
cudaError_t umma_prepare(Ctx &c);
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
                                cudaStream_t s);
cudaError_t select_prepare(Ctx &c);
cudaError_t select_radix_prepare();
int select_radix_capacity();
cudaError_t launch_select_radix(const Ctx &c, const Record *rec_in, Record *rec_out,
                                const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                                const uint8_t *running, int n, int64_t budget, int max_run,
                                uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                                cudaStream_t s);
bool use_bitonic_select();
int select_impl();
int select_local_capacity();
cudaError_t launch_select_local(const Ctx &c, const uint32_t *ids, const uint32_t *arrival,
                                const int32_t *kv, const uint8_t *running, int n, int64_t budget,
                                int max_run, uint32_t *run, uint32_t *pre, uint32_t *adm,
                                int32_t *counts, cudaStream_t s);
cudaError_t select_rank_prepare();
cudaError_t select_bucket_prepare();
size_t bucket_workspace_bytes(int m_max);
cudaError_t launch_select_bucket(const Ctx &c, const Record *rec, int m, int64_t budget,
                                 int max_run, uint32_t *run, uint32_t *pre, uint32_t *adm,
                                 int32_t *counts, cudaStream_t s);
constexpr int kRankMaxRecords = 2048;   // rank-counting kernel below, bucketed kernels above
int select_rank_capacity();
cudaError_t launch_select_rank(const Ctx &c, const Record *rec_in, Record *rec_out,
                               const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                               const uint8_t *running, int n, int64_t budget, int max_run,
                               uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                               cudaStream_t s);
cudaError_t select_fast_prepare();
int select_fast_capacity();
// rec_in != nullptr: select over given records; else build local records (fused pack)
// from (ids, arrival, kv, running) into rec_out and select over them.
cudaError_t launch_select_fast(const Ctx &c, const Record *rec_in, Record *rec_out,
                               const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                               const uint8_t *running, int n, int64_t budget, int max_run,
                               uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                               cudaStream_t s);
cudaError_t head_prepare(Ctx &c);
size_t select_scratch_bytes(int n_max);
int select_smem_capacity();

// ---------------------------------------------------------------- launch helper
// Programmatic dependent launch (PDL): consecutive kernels of a step overlap the next
// kernel's launch + prologue with the previous kernel's tail.  Every kernel executes
// griddep_wait() before touching data produced by an earlier kernel and
// griddep_launch() once all its CTAs are resident (so a waiting dependent can never
// starve it of SM resources).
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
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
