/* trail.h — C ABI of libtrail.so: TRAIL's per-iteration predict+schedule hot path on
 * B200 (sm_100a).  arXiv 2410.01035; citations P:<line> refer to PAPER.md.
 *
 * Conventions (apply to every entry point)
 *   - Every data pointer is a DEVICE pointer unless marked (host).  Device buffers are
 *     owned by the caller; the library never frees or retains them past the call.
 *   - Every call enqueues work on `stream` (a cudaStream_t; NULL = legacy default stream)
 *     and returns without synchronising, unless documented as synchronising.  Outputs are
 *     valid once the stream reaches that point.  Calls are CUDA-graph capturable (no
 *     allocation, no host synchronisation, no host reads of device data).
 *   - A handle is not thread-safe: one host thread (and one stream at a time) per handle.
 *   - Return value: TRAIL_OK, or a negative trail_status.  A negative status means the
 *     call was rejected on the host before any work was enqueued and no state changed.
 *     Errors that can only be seen on the device (an id >= max_slots, an empty row range,
 *     a negative KV count, a non-finite length) set sticky bits readable with
 *     trail_device_errors(); the offending request is skipped or clamped as documented.
 *   - No exceptions cross the ABI.
 */
#ifndef TRAIL_H_
#define TRAIL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TRAIL_ABI_VERSION 1

#if defined(__GNUC__)
#define TRAIL_API __attribute__((visibility("default")))
#else
#define TRAIL_API
#endif

typedef struct trail_ctx *trail_handle;
typedef struct CUstream_st *trail_stream; /* == cudaStream_t */

typedef enum {
  TRAIL_OK = 0,
  TRAIL_WARN_OVER_BUDGET = 1,  /* forced (non-preemptible) set alone exceeds budget/cap */
  TRAIL_ERR_INVALID = -1,      /* bad argument (shape, pointer, alignment, value)       */
  TRAIL_ERR_CUDA = -2,         /* a CUDA runtime/driver call failed                      */
  TRAIL_ERR_NOMEM = -3,        /* device or host allocation failed                       */
  TRAIL_ERR_CAPACITY = -4,     /* n exceeds the capacity fixed at trail_create            */
  TRAIL_ERR_NCCL = -5,         /* NCCL unavailable or a collective failed                */
  TRAIL_ERR_STATE = -6,        /* call not valid in the handle's current state            */
  TRAIL_ERR_UNSUPPORTED = -7   /* configuration outside what this build implements       */
} trail_status;

typedef enum { TRAIL_F32 = 0, TRAIL_BF16 = 1 } trail_dtype;

/* Layer-1 kernel selection (row a2). */
typedef enum {
  TRAIL_L1_AUTO = 0,   /* GEMV for fp32 or small n, fused tcgen05 kernel (K2c) for moderate n,
                          wide CTA-pair kernel (K2d) for large n */
  TRAIL_L1_GEMV = 1,   /* K2a: warp-per-output-slice split-K GEMV (CUDA cores) + head K3 */
  TRAIL_L1_UMMA = 2,   /* K2c: fused TMA + tcgen05/TMEM layer 1, cluster split-K reduction,
                          layer 2 and head in the epilogue (bf16 only) */
  TRAIL_L1_UMMA_UNFUSED = 3, /* K2b + K3: tcgen05 layer 1 with split-K partials in global
                                memory, then the separate head kernel (bf16 only) */
  TRAIL_L1_WIDE = 4,   /* K2d: CTA-pair (cta_group::2) tcgen05 layer 1 over the whole hidden
                          width (H = 512) in TMEM, layer 2 and head in the epilogue; AUTO picks
                          it for large n (bf16, H = 512 only) */
  TRAIL_L1_TF32 = 5    /* K2t + K3: fp32 handles — tcgen05 kind::tf32 layer 1 with an exact
                          hi/lo operand split (3 MMAs per product, fp32-level accuracy), split-K
                          partials, then the head kernel (fp32 only; H % 128 == 0, d % 4 == 0;
                          AUTO keeps K2a) */
} trail_l1_mode;

/* Sticky device-side error bits (trail_device_errors). */
#define TRAIL_DEV_BAD_ID   0x1u   /* request id >= max_slots: request skipped            */
#define TRAIL_DEV_BAD_ROWS 0x2u   /* row range empty or reversed: treated as a zero row   */
#define TRAIL_DEV_NEG_KV   0x4u   /* kv_blocks < 0: treated as 0                          */
#define TRAIL_DEV_NONFIN   0x8u   /* non-finite expected length: key encoded as +inf      */
#define TRAIL_DEV_BAD_HINT 0x10u  /* trail_set_prefill_start broken: a multi-row request
                                     before the hinted start (its outputs are undefined)  */

typedef struct {
  /* Classifier (Linear(d, 512) - ReLU - Linear(512, k); P:362 ~2.1M params). */
  int32_t d;               /* embedding width; multiple of 64 (bf16) or 8 (fp32)          */
  int32_t hidden;          /* probe width H; multiple of 128, <= 512 (paper: 512)         */
  int32_t k;               /* number of bins, 1..32 (paper: 10)                           */
  int32_t dtype;           /* trail_dtype of W1 and of the embeddings                     */
  const void *w1;          /* (host) [hidden][d] row-major (nn.Linear [out][in]), dtype   */
  const float *b1;         /* (host) [hidden]                                             */
  const float *w2;         /* (host) [k][hidden] row-major                                */
  const float *b2;         /* (host) [k]                                                  */
  /* Bins: B_i = [b_i, b_{i+1}), last bin closed; widths >= 1 token.  */
  const double *bin_edges; /* (host) [k+1] strictly increasing, b_0 >= 0                 */
  const double *prior;     /* (host) [k] prior pi on the simplex, or NULL = uniform       */
  double c;                /* limited preemption: preemptible while a < floor(c*r);
                              c >= 0; INFINITY = unlimited (reading D-14)                  */
  /* Capacities (fixed for the handle's lifetime). */
  int32_t max_slots;       /* request ids are slot indices in [0, max_slots)              */
  int32_t max_requests;    /* max n per trail_predict_step, <= 262144                      */
  int32_t max_sched;       /* max records per trail_schedule_step on THIS rank            */
  int32_t world_size;      /* ranks sharing one selection (1 = single GPU)                */
  uint32_t id_base;        /* added to slot ids in the returned lists (e.g. rank*max_slots) */
  int32_t device;          /* CUDA device ordinal the handle lives on                     */
  int32_t l1_mode;         /* trail_l1_mode                                               */
} trail_config;

/* Library ABI version (TRAIL_ABI_VERSION). */
TRAIL_API int32_t trail_abi_version(void);

/* Validates cfg, copies weights and constants to library-owned device memory and
 * precomputes in fp64 on the host: bin midpoints m_i, the transition
 * coefficients log(1-1/w_i) and log(1/w_{i+1}) of T (reading D-1), the
 * threshold table floor(c*m_j) (D-10) and E_pi[L] (D-24).  Allocates per-slot
 * state (all slots unobserved) and step workspaces.  Synchronising.
 * Errors: TRAIL_ERR_INVALID (shapes, non-increasing edges, width < 1, prior not on the
 * simplex, c < 0 or NaN), TRAIL_ERR_NOMEM, TRAIL_ERR_CUDA. */
TRAIL_API trail_status trail_create(const trail_config *cfg, trail_handle *out);

/* Frees everything the handle owns (and its NCCL communicator).  Synchronising. */
TRAIL_API trail_status trail_destroy(trail_handle h);

/* One prediction iteration for the n requests that just ran.
 *   emb            [rows][emb_ld] in cfg.dtype: the layer-l hidden states of the flat
 *                  token batch, 16-byte aligned, emb_ld a multiple of 8 (bf16) /
 *                  4 (fp32) elements, emb_ld >= d.
 *   row_offsets    [n+1] int32 CSR: request j owns rows [row_offsets[j], row_offsets[j+1]).
 *                  A decode observation has 1 row (its new token); a prefill
 *                  observation has its prompt rows, which are mean-pooled (D-12).
 *   request_ids    [n] slot ids, unique within the call.
 *   is_prefill     [n] 1 = first observation of the request: q^(0) = normalise(pi * p)
 *                  (P:219), r = m[argmax q^(0)], threshold = floor(c r), age a = 0.
 *                  0 = decode: q = normalise((T q_prev) * p) (D-2), a += 1.
 *                  A decode on a never-observed slot is treated as a prefill (D-23).
 *   prior_override [n][k] fp32 per-request prior pi for prefill rows, or NULL.
 *   posteriors     [n][k] fp32 out (may be NULL): q^(t) of each request.
 *   expected_remaining [n] fp32 out (may be NULL): L_t = sum_i q(i) m_i.
 * Updates the per-slot state (log q in fp32, reading D-22; a; threshold; L_t). */
TRAIL_API trail_status trail_predict_step(trail_handle h, const void *emb, int64_t emb_ld,
                                const int32_t *row_offsets, const uint32_t *request_ids,
                                const uint8_t *is_prefill, const float *prior_override,
                                int32_t n, float *posteriors, float *expected_remaining,
                                trail_stream stream);

/* Multi-layer weighted embeddings ("estimate the prediction using
 * ... a weighted average of their outputs", "leveraging multiple-layer embeddings
 * through weighted averaging"; reading D-28).  The probe input of request j is
 *   u_j = sum_l a_l u_{l,j},   a = layer_weights / sum(layer_weights),
 * u_{l,j} = layer l's embedding of request j: the mean of its prompt rows at prefill,
 * its row at decode.  Every layer buffer uses the same row_offsets and emb_ld.  The weighted
 * mean is accumulated in fp32 (layer order, rows in order), divided by the row count
 * (correctly rounded), rounded to bf16 (RNE) once for bf16 handles (D-12), written to a
 * library buffer [max_requests][d] (allocated on first use: synchronising, so make the
 * first call outside CUDA-graph capture), and the rest of the step is trail_predict_step
 * on it (one row per request; is_prefill keeps its meaning).
 *   embs           (host) array of n_layers DEVICE pointers, [rows][emb_ld] cfg.dtype each
 *   layer_weights  (host) n_layers finite non-negative fp32 with a positive sum
 *   n_layers       1 .. 8
 * Other arguments, outputs and errors as trail_predict_step; TRAIL_ERR_INVALID for bad
 * weights or n_layers. */
TRAIL_API trail_status trail_predict_step_layers(trail_handle h, const void *const *embs,
                                const float *layer_weights, int32_t n_layers, int64_t emb_ld,
                                const int32_t *row_offsets, const uint32_t *request_ids,
                                const uint8_t *is_prefill, const float *prior_override,
                                int32_t n, float *posteriors, float *expected_remaining,
                                trail_stream stream);

/* Chunked prefill (P:432 vLLM chunked prefill, reading D-27).  A prompt's
 * rows may arrive over several iterations; the pooled input is still the mean of ALL its
 * rows.  For each of the n requests, adds its chunk's rows
 * [row_offsets[j], row_offsets[j+1]) of emb ([rows][emb_ld], cfg.dtype) to the slot's
 * running fp32 sum and row count; where is_final[j] != 0 writes the mean of every row
 * seen — rounded to bf16 (RNE) for bf16 handles, reading D-12 — to row j of `pooled`
 * ([n][pooled_ld], cfg.dtype, device, caller-owned) and clears the slot's accumulator.
 * The caller then passes `pooled` rows to trail_predict_step as one-row prefill
 * observations.  Non-final rows of `pooled` are not written.  Request ids unique within a
 * call.  The [max_slots][d] fp32 accumulator is allocated on first use (synchronising).
 * Errors: TRAIL_ERR_INVALID (NULL pointers, ld < d, 16-byte alignment);
 * TRAIL_DEV_BAD_ID / TRAIL_DEV_BAD_ROWS device bits for bad ids / reversed ranges. */
TRAIL_API trail_status trail_prefill_chunk(trail_handle h, const void *emb, int64_t emb_ld,
                                           const int32_t *row_offsets,
                                           const uint32_t *request_ids, const uint8_t *is_final,
                                           int32_t n, void *pooled, int64_t pooled_ld,
                                           trail_stream stream);

/* Iterations without an observation — the "predict every K iterations" variant (P:717,
 * SURVEY §8(f)3).  For each listed slot that has been observed: the transition alone acts,
 * q <- normalise(T q) (readings D-1/D-4, log domain D-22), `steps` times; the
 * age a advances by `steps` (the request kept generating, D-11) and L_t is refreshed, so
 * the next trail_predict_step / trail_schedule_step see the propagated state (reading
 * D-25).  Never-observed slots are untouched and report the prior pi and E_pi[L] (D-24).
 *   request_ids [n] device slot ids;  steps >= 0 (0 = only report the state);
 *   posteriors [n][k] / expected_remaining [n] fp32 device outputs, may be NULL.
 * Enqueued on `stream`.  Errors: TRAIL_ERR_INVALID (n < 0, steps < 0, NULL ids with n > 0);
 * a slot id >= max_slots sets TRAIL_DEV_BAD_ID and NaN outputs for that request. */
TRAIL_API trail_status trail_time_update(trail_handle h, const uint32_t *request_ids, int32_t n,
                                         int32_t steps, float *posteriors,
                                         float *expected_remaining, trail_stream stream);

/* Next-batch selection: limited-preemption SPRPT under a KV-block budget (P:171, P:394,
 * P:570).  Inputs are THIS rank's live requests (running + waiting):
 *   request_ids  [n] slot ids;  arrival_seq [n] arrival order (FCFS tie-break),
 *                globally unique across ranks;  kv_blocks [n] >= 0 blocks the request needs
 *                resident to run the next iteration;  is_running [n] 1 = in the batch that
 *                just ran.
 *   kv_budget    blocks available to the run set;  max_run  cap on the run-set size (0 =
 *                no cap).
 * Key = L_t of the slot (E_pi[L] if never observed, D-24).  A request is forced
 * (non-preemptible, rank -inf) iff running, observed and a >= floor(c r).
 * Order: forced first, then ascending key, then arrival_seq.  Run set = all forced +
 * the longest prefix of the rest that keeps the cumulative KV within the budget and the
 * count within max_run (strict prefix, D-15).  If the forced set alone violates either
 * limit, run = forced and status TRAIL_WARN_OVER_BUDGET (D-16).
 * With world_size > 1 (after trail_comm_init) the 16-byte records of all ranks are
 * all-gathered over NCCL and every rank computes the identical global selection.
 * Outputs (ids are id_base + slot of the owning rank, in priority order):
 *   run_ids, preempt_ids, admit_ids  capacity max_sched * world_size each;
 *   counts[4] = {n_run, n_preempt (running, not in run), n_admit (waiting, in run), status}.
 * The returned status reports host-side validation only; the selection's own status
 * (TRAIL_OK / TRAIL_WARN_OVER_BUDGET) is counts[3] on the device. */
TRAIL_API trail_status trail_schedule_step(trail_handle h, const uint32_t *request_ids,
                                 const uint32_t *arrival_seq, const int32_t *kv_blocks,
                                 const uint8_t *is_running, int32_t n, int64_t kv_budget,
                                 int32_t max_run, uint32_t *run_ids, uint32_t *preempt_ids,
                                 uint32_t *admit_ids, int32_t *counts, trail_stream stream);

/* The two halves of trail_schedule_step, for callers that run their own collective
 * (SURVEY §8(b) prose alternative: pack -> caller's all-gather -> select).
 * pack writes `capacity` (>= n) 16-byte records {u32 keybits, u32 arrival_seq,
 * u32 kv_blocks, u32 (id_base+slot) | running<<31} where keybits = (!forced)<<31 | fp32 bits
 * of the key (P:394 forced = rank -inf, P:570 key = predicted remaining length); records
 * [n, capacity) are padding (keybits = arrival = id word = 0xFFFFFFFF, kv = 0) so that every rank sends the same byte
 * count — this is the same kernel, with capacity = max_sched, that trail_schedule_step
 * runs before its NCCL all-gather.  `records` is device memory of capacity * 16 bytes.
 * select consumes n_records such records (from any number of ranks, any order; records
 * with keybits == 0xFFFFFFFF are padding and ignored); n_records <= max_sched * world_size.
 * Errors: TRAIL_ERR_INVALID for capacity < n or NULL pointers. */
TRAIL_API trail_status trail_schedule_pack(trail_handle h, const uint32_t *request_ids,
                                 const uint32_t *arrival_seq, const int32_t *kv_blocks,
                                 const uint8_t *is_running, int32_t n, int32_t capacity,
                                 void *records, trail_stream stream);
TRAIL_API trail_status trail_schedule_select(trail_handle h, const void *records, int32_t n_records,
                                   int64_t kv_budget, int32_t max_run, uint32_t *run_ids,
                                   uint32_t *preempt_ids, uint32_t *admit_ids,
                                   int32_t *counts, trail_stream stream);

/* Marks n slots as never observed (finished requests). */
TRAIL_API trail_status trail_release(trail_handle h, const uint32_t *request_ids, int32_t n,
                           trail_stream stream);

/* Reads per-slot state for n ids (any output may be NULL): L_t, age a, threshold
 * floor(c r), seen flag, and the posterior q (fp32 [n][k], = exp of the log state). */
TRAIL_API trail_status trail_read_state(trail_handle h, const uint32_t *request_ids, int32_t n,
                              float *L, uint32_t *age, uint32_t *threshold, uint8_t *seen,
                              float *posterior, trail_stream stream);

/* Multi-GPU: NCCL unique id (128 bytes, host) generated on rank 0 and broadcast by the
 * caller; then every rank calls trail_comm_init.  NCCL is loaded at run time
 * (libnccl.so.2); TRAIL_ERR_NCCL if it is unavailable.  Synchronising. */
TRAIL_API trail_status trail_nccl_unique_id(void *id_out /* (host) 128 bytes */);
TRAIL_API trail_status trail_comm_init(trail_handle h, const void *id /* (host) 128 bytes */,
                             int32_t rank, int32_t world_size);

/* Sticky device error bits (TRAIL_DEV_*); synchronising; clear != 0 resets them. */
TRAIL_API trail_status trail_device_errors(trail_handle h, uint32_t *bits_out, int32_t clear);

/* Per-kernel timing with CUDA events on the launch stream.  enable: 0 = off;
 * 1 = accumulate: trail_profile_read returns, for kernel id `kid` (TRAIL_K_*), the summed
 *     device time in ms and the number of launches since the last reset;
 * 2 = last launch (CUDA-graph friendly: one event pair per kernel id, re-recorded on
 *     every launch, including by event-record nodes of a graph captured in this mode):
 *     trail_profile_read returns the duration of the most recent launch of `kid`.
 * trail_profile_read is synchronising. */
#define TRAIL_K_POOL 0
#define TRAIL_K_GEMV 1
#define TRAIL_K_UMMA 2
#define TRAIL_K_HEAD 3
#define TRAIL_K_PACK 4
#define TRAIL_K_SELECT 5
#define TRAIL_K_GATHER 6
#define TRAIL_K_COUNT 7
TRAIL_API trail_status trail_profile_enable(trail_handle h, int32_t enable);
TRAIL_API trail_status trail_profile_read(trail_handle h, int32_t kid, double *total_ms,
                                int64_t *launches, int32_t reset);

/* Diagnostics: per-CTA phase timestamps of the fused tcgen05 predict kernel (16 u64 per CTA:
 * globaltimer ns at entry, after the prologue, first stage landed, mainloop done, tile
 * staged, cluster barrier passed, reduction done, second barrier passed, exit; [14] = ran the
 * head, [15] = SM id).  enable allocates room for max_ctas CTAs (0 = off); a launch whose
 * grid exceeds it is not traced.  trail_trace_read synchronises and copies max_ctas entries
 * to host memory. */
TRAIL_API trail_status trail_trace_enable(trail_handle h, int32_t max_ctas);
TRAIL_API trail_status trail_trace_read(trail_handle h, uint64_t *host_out, int32_t max_ctas);

/* Overrides cfg.l1_mode for subsequent calls (the tcgen05 modes require bf16). */
TRAIL_API trail_status trail_set_l1_mode(trail_handle h, int32_t l1_mode);

/* Preemption-threshold rule (row a4).  0 (default): the paper's static rule, preemptible
 * while a < floor(c r) with r the initial prediction (D-9, D-10).  1: the dynamic
 * variant of SURVEY §8(f)3 (reading D-26): preemptible while a < c (a + L_t), i.e. forced
 * once a >= c L_t / (1 - c) (never for c >= 1), re-evaluated whenever L_t changes
 * (predict step or time update) and stored as the slot threshold.  Synchronising; CUDA
 * graphs captured earlier keep the old rule.  Errors: TRAIL_ERR_INVALID (mode not 0/1). */
TRAIL_API trail_status trail_set_threshold_mode(trail_handle h, int32_t mode);

/* Budget fill rule of the selection (row a6; P:171 is silent, reading D-15).  0 (default):
 * strict prefix — stop at the first request in priority order whose KV blocks do not fit.
 * 1: first-fit — skip it and keep taking every later request that still
 * fits the remaining budget and run cap; the lists stay in priority order.  Applies to
 * trail_schedule_step / trail_schedule_select calls enqueued afterwards (CUDA graphs captured
 * earlier keep the old rule).  Errors: TRAIL_ERR_INVALID (mode not 0/1). */
TRAIL_API trail_status trail_set_fill_mode(trail_handle h, int32_t mode);

/* Batch-layout hint (host knowledge of the flat batch, like trail_set_rows_hint): every
 * request with index < first_prefill in the next predict steps is a single-row (decode)
 * observation — vLLM-style schedulers put running decodes first and new prefills last
 * (P:432).  With it (opt-in), the large-batch path splits the step: the CTA-pair kernel runs
 * the decode tiles [0, t) (t = first_prefill rounded down to a 256-request tile) on most SMs
 * at once, while on a library side stream the pooling kernel (on the remaining SMs) and the
 * split-K kernel handle the tail [t, n) that contains the prompts — the prompt pooling no
 * longer sits in front of the whole layer-1 contraction.  The streams re-join before the
 * call returns (capturable in a CUDA graph).  Measured at configs[3] (≈100 MB of prompt rows
 * per step) the side path is the longer one (239 -> 250 us per step), so it pays only with
 * fewer prompt rows per step.  -1 (default) disables it.  A multi-row request
 * before the hinted start breaks the contract: TRAIL_DEV_BAD_HINT is raised and that tile's
 * outputs are undefined.  Errors: TRAIL_ERR_INVALID (first_prefill < -1). */
TRAIL_API trail_status trail_set_prefill_start(trail_handle h, int32_t first_prefill);

/* L2-persisting W1 (optional; W1 is 99.7 % of the probe's parameters).
 * 1: sets the device's persisting-L2 set-aside to cover W1 (cudaLimitPersistingL2CacheSize —
 * a DEVICE-WIDE limit) and attaches an access-policy window (persisting hits, streaming misses)
 * over the library's W1 copy to every layer-1 launch, so W1 survives the LLM layers that run
 * between two predict steps.  0 (default): normal caching; resets the persisting lines and
 * the set-aside.  Launches enqueued afterwards follow the setting (graphs captured earlier
 * keep theirs).  Errors: TRAIL_ERR_UNSUPPORTED if the device has no persisting L2,
 * TRAIL_ERR_CUDA. */
TRAIL_API trail_status trail_set_w1_l2_persist(trail_handle h, int32_t enable);

/* Optional host-side hint: the number of embedding rows (the flat batch's token count,
 * row_offsets[n] - row_offsets[0]) of the next trail_predict_step calls; 0 = unknown (the
 * default).  It only selects the pooling kernel variant and grid (bulk-copy streaming for
 * prefill-heavy batches, P:570 burst shape; more row chunks for large mixed batches).  The
 * fp32 prompt sums are combined over row chunks in a fixed order, so results are
 * deterministic for a given hint; between hints the pooled means of prompts that cross a
 * chunk boundary may differ in the last bit (fp32 summation grouping).  Kept until
 * changed.  Errors: TRAIL_ERR_INVALID (rows < 0). */
TRAIL_API trail_status trail_set_rows_hint(trail_handle h, int64_t rows);

/* Which layer-1 kernel trail_predict_step uses for n requests, and its split-K factor. */
TRAIL_API trail_status trail_plan_l1(trail_handle h, int32_t n, int32_t *l1_mode_out,
                           int32_t *splits_out);

/* Human-readable message for a status. */
TRAIL_API const char *trail_status_string(trail_status s);

#ifdef __cplusplus
}
#endif
#endif /* TRAIL_H_ */
