// K5 record pack (row a4), K4 selection (row a6), slot release / state read.
//
// Record (16 B): keybits = (!forced) << 31 | fp32 bits of the key.  The key is L_t of the
// slot (E_pi[L] if never observed, D-24); forced = running & observed & a >= floor(c r)
// ("we only allow preemption for the first floor(C r) iterations"; rank -inf,
// P:830-831).  L_t >= m_0 > 0, so its fp32 bits order like the values and a forced record
// (bit 31 clear) sorts before every non-forced one.
//
// Selection ("prioritizing those with the shortest predicted remaining time ... limited
// by the available GPU memory"; "ranks all requests (running and waiting)"): sort the
// 64-bit composite (keybits << 32 | arrival_seq) ascending — ties FCFS, then input
// position (stable) — then take every forced record plus the longest prefix of the rest whose
// cumulative KV blocks fit the budget (and the run cap): strict prefix (D-15).  The sort and
// the cut run in one thread-block cluster (k_csort.cu).  Every rank runs it on identical
// bytes -> identical lists.
#include "trail_internal.cuh"

namespace trail {

thread_local const cudaAccessPolicyWindow *tl_l1_window = nullptr;   // see trail_internal.cuh

// ------------------------------------------------------------------ K5 pack
__global__ void trail_pack_kernel(const uint32_t *__restrict__ ids,
                                  const uint32_t *__restrict__ arrival,
                                  const int32_t *__restrict__ kv,
                                  const uint8_t *__restrict__ running,
                                  const SlotMeta *__restrict__ meta,
                                  const HeadConsts *__restrict__ cst, int n, int n_pad_to,
                                  int max_slots, uint32_t id_base, Record *__restrict__ out,
                                  uint32_t *__restrict__ err) {
  griddep_wait();
  griddep_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pad_to) return;
  Record r;
  if (i >= n) {
    r.keybits = kPadKey; r.arrival = 0xFFFFFFFFu; r.kv = 0; r.gid = 0xFFFFFFFFu;
    out[i] = r;
    return;
  }
  const uint32_t slot = __ldg(ids + i);
  const bool run = __ldg(running + i) != 0;
  int32_t kvb = __ldg(kv + i);
  if (kvb < 0) { atomicOr(err, TRAIL_DEV_NEG_KV); kvb = 0; }
  float key = cst->prior_L;
  bool forced = false;
  if (slot < (uint32_t)max_slots) {
    const SlotMeta m = meta[slot];
    if (m.flags & 1u) {
      key = m.L;
      forced = run && (m.age >= m.thr);
    }
  } else {
    atomicOr(err, TRAIL_DEV_BAD_ID);
    key = INFINITY;   // sorts last among non-forced; never displaces a valid request
  }
  uint32_t kb;
  if (isfinite(key) && key >= 0.f) {
    kb = __float_as_uint(key) & 0x7FFFFFFFu;
  } else {
    if (slot < (uint32_t)max_slots) atomicOr(err, TRAIL_DEV_NONFIN);
    kb = 0x7F800000u;
  }
  r.keybits = (forced ? 0u : 0x80000000u) | kb;
  r.arrival = __ldg(arrival + i);
  r.kv = (uint32_t)kvb;
  r.gid = ((id_base + slot) & 0x7FFFFFFFu) | (run ? 0x80000000u : 0u);
  out[i] = r;
}

cudaError_t launch_pack(const Ctx &c, const uint32_t *ids, const uint32_t *arrival,
                        const int32_t *kv, const uint8_t *running, int n, Record *out,
                        int n_pad_to, cudaStream_t s) {
  if (n_pad_to <= 0) return cudaSuccess;
  return launch_k(trail_pack_kernel, dim3((n_pad_to + 255) / 256), dim3(256), 0, s, ids, arrival,
                  kv, running, (const SlotMeta *)c.meta, (const HeadConsts *)c.consts, n, n_pad_to,
                  c.cfg.max_slots, c.cfg.id_base, out, c.dev_err);
}

// ------------------------------------------------------------------ K4 select
cudaError_t select_prepare(Ctx &c) {
  (void)c;
  cudaError_t e = select_cluster_prepare();
  if (e == cudaSuccess) e = select_rank_prepare();
  if (e == cudaSuccess) e = select_bucket_prepare();
  return e;
}

// Which K4 kernel: the multi-CTA rank-counting kernel (<= 2048 records) or the bucketed
// three-kernel pipeline above it — both spread the O(m^2) / O(sum b^2) comparisons over every
// SM, which is what a latency-bound selection needs (one cluster's serial phases cost more:
// measured 38 us for 640 records in the radix form, 45 us in the bitonic form) — and the
// single-cluster kernel for first-fit filling (a sequential rule) or TRAIL_SELECT=cluster.
cudaError_t launch_select_any(const Ctx &c, const Record *rec_in, Record *rec_out,
                              const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                              const uint8_t *running, int n, int64_t budget, int max_run,
                              uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                              cudaStream_t s) {
  const bool cluster = c.fill_mode != 0 || select_impl() == 2;
  if (!cluster && n <= kRankMaxRecords && c.rank_cnt)
    return launch_select_rank(c, rec_in, rec_out, ids, arrival, kv, running, n, budget, max_run,
                              run, pre, adm, counts, s);
  if (!cluster && n <= c.bk_cap)
    return launch_select_bucket(c, rec_in, rec_out, ids, arrival, kv, running, n, budget,
                                max_run, run, pre, adm, counts, s);
  return launch_select_cluster(c, rec_in, rec_out, ids, arrival, kv, running, n, budget, max_run,
                               run, pre, adm, counts, s);
}

cudaError_t launch_select(const Ctx &c, const Record *rec, int n, int64_t budget, int max_run,
                          uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                          cudaStream_t s) {
  return launch_select_any(c, rec, nullptr, nullptr, nullptr, nullptr, nullptr, n, budget,
                           max_run, run, pre, adm, counts, s);
}

// ------------------------------------------------------------------ release / read state
__global__ void trail_release_kernel(const uint32_t *__restrict__ ids, int n, int max_slots,
                                     SlotMeta *__restrict__ meta, uint32_t *__restrict__ err) {
  griddep_wait();
  griddep_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t slot = ids[i];
  if (slot >= (uint32_t)max_slots) { atomicOr(err, TRAIL_DEV_BAD_ID); return; }
  SlotMeta m;
  m.L = 0.f; m.age = 0; m.thr = 0; m.flags = 0;
  meta[slot] = m;
}

// a released slot also drops any partial chunked-prefill sum (K1c, reading D-27): a request
// aborted between two chunks must not leak its rows into the slot's next prompt.  A CTA per
// id, one thread per float4 of the row.
__global__ void trail_release_chunks_kernel(const uint32_t *__restrict__ ids, int n, int d,
                                            int max_slots, float *__restrict__ acc,
                                            uint32_t *__restrict__ cnt) {
  griddep_wait();
  griddep_launch();
  const uint32_t slot = ids[blockIdx.x];
  if (slot >= (uint32_t)max_slots) return;
  float4 *row = reinterpret_cast<float4 *>(acc + (int64_t)slot * d);
  for (int v = threadIdx.x; v < d / 4; v += blockDim.x) row[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) cnt[slot] = 0u;
}

cudaError_t launch_release(const Ctx &c, const uint32_t *ids, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  trail_release_kernel<<<(n + 255) / 256, 256, 0, s>>>(ids, n, c.cfg.max_slots, c.meta,
                                                       c.dev_err);
  if (c.chunk_acc)
    trail_release_chunks_kernel<<<n, 256, 0, s>>>(ids, n, c.d, c.cfg.max_slots, c.chunk_acc,
                                                  c.chunk_cnt);
  return cudaGetLastError();
}

__global__ void trail_read_state_kernel(const uint32_t *__restrict__ ids, int n, int k,
                                        int max_slots, const SlotMeta *__restrict__ meta,
                                        const float *__restrict__ lq, float *L, uint32_t *age,
                                        uint32_t *thr, uint8_t *seen, float *post) {
  griddep_wait();
  griddep_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t slot = ids[i];
  if (slot >= (uint32_t)max_slots) return;
  const SlotMeta m = meta[slot];
  if (L) L[i] = m.L;
  if (age) age[i] = m.age;
  if (thr) thr[i] = m.thr;
  if (seen) seen[i] = (uint8_t)(m.flags & 1u);
  if (post)
    for (int b = 0; b < k; ++b) post[(int64_t)i * k + b] = (m.flags & 1u) ? expf(lq[(int64_t)slot * k + b]) : 0.f;
}

cudaError_t launch_read_state(const Ctx &c, const uint32_t *ids, int n, float *L, uint32_t *age,
                              uint32_t *thr, uint8_t *seen, float *post, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  trail_read_state_kernel<<<(n + 255) / 256, 256, 0, s>>>(ids, n, c.k, c.cfg.max_slots, c.meta,
                                                          c.lq, L, age, thr, seen, post);
  return cudaGetLastError();
}

}  // namespace trail
