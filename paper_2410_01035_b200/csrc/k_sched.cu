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
// cumulative KV blocks fit the budget (and the run cap): strict prefix (D-15).  One CTA of
// 1024 threads: a bitonic sort of (key, index) pairs in shared memory (global scratch beyond
// 16384 records), then block-wide scans for the cumulative KV and for compacting the
// preempt / admit lists.  Every rank runs it on identical bytes -> identical lists.
#include "trail_internal.cuh"

namespace trail {

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
namespace {
constexpr int kSelThreads = 1024;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSmemCapRecords = 16384;   // 16384 * (8 + 4) B = 192 KB of shared memory

struct SelShared {
  long long wsum[kSelWarps];
  int wcnt[kSelWarps];
  int wcnt2[kSelWarps];
  long long total;
  int cnt_total, cnt2_total;
};

// Block-wide exclusive scan of a 64-bit value and two int counters (one per thread).
__device__ __forceinline__ void block_scan3(SelShared &sh, long long v, int c1, int c2,
                                            long long &ex_v, int &ex_c1, int &ex_c2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long iv = v;
  int i1 = c1, i2 = c2;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long tv = __shfl_up_sync(0xffffffffu, iv, o);
    const int t1 = __shfl_up_sync(0xffffffffu, i1, o);
    const int t2 = __shfl_up_sync(0xffffffffu, i2, o);
    if (lane >= o) { iv += tv; i1 += t1; i2 += t2; }
  }
  if (lane == 31) { sh.wsum[warp] = iv; sh.wcnt[warp] = i1; sh.wcnt2[warp] = i2; }
  __syncthreads();
  if (warp == 0) {
    long long wv = sh.wsum[lane];
    int w1 = sh.wcnt[lane], w2 = sh.wcnt2[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long tv = __shfl_up_sync(0xffffffffu, wv, o);
      const int t1 = __shfl_up_sync(0xffffffffu, w1, o);
      const int t2 = __shfl_up_sync(0xffffffffu, w2, o);
      if (lane >= o) { wv += tv; w1 += t1; w2 += t2; }
    }
    sh.wsum[lane] = wv - sh.wsum[lane];   // exclusive warp offsets
    const int e1 = w1 - sh.wcnt[lane], e2 = w2 - sh.wcnt2[lane];
    sh.wcnt[lane] = e1;
    sh.wcnt2[lane] = e2;
    if (lane == 31) { sh.total = wv; sh.cnt_total = w1; sh.cnt2_total = w2; }
  }
  __syncthreads();
  ex_v = sh.wsum[warp] + iv - v;
  ex_c1 = sh.wcnt[warp] + i1 - c1;
  ex_c2 = sh.wcnt2[warp] + i2 - c2;
  __syncthreads();
}
}  // namespace

__global__ void __launch_bounds__(kSelThreads, 1)
trail_select_large_kernel(const Record *__restrict__ rec, int n, int npow2, long long budget,
                    int max_run, unsigned long long *gkeys, uint32_t *gidx,
                    uint32_t *__restrict__ run_ids, uint32_t *__restrict__ pre_ids,
                    uint32_t *__restrict__ adm_ids, int32_t *__restrict__ counts) {
  griddep_wait();
  griddep_launch();
  extern __shared__ __align__(16) uint8_t sel_smem[];
  __shared__ SelShared sh;
  __shared__ int s_valid;
  unsigned long long *keys = gkeys ? gkeys : reinterpret_cast<unsigned long long *>(sel_smem);
  uint32_t *idx = gidx ? gidx : reinterpret_cast<uint32_t *>(sel_smem + (size_t)npow2 * 8);
  const int tid = threadIdx.x;
  if (tid == 0) s_valid = 0;
  __syncthreads();
  // 1. load composite keys; padding and out-of-range slots sort last
  int my_valid = 0;
  for (int i = tid; i < npow2; i += kSelThreads) {
    unsigned long long kk = ~0ull;
    uint32_t ii = 0xFFFFFFFFu;
    if (i < n) {
      const Record r = rec[i];
      if (r.keybits != kPadKey) {
        kk = ((unsigned long long)r.keybits << 32) | r.arrival;
        ii = (uint32_t)i;
        ++my_valid;
      }
    }
    keys[i] = kk;
    idx[i] = ii;
  }
  atomicAdd(&s_valid, my_valid);
  __syncthreads();
  const int nv = s_valid;
  // 2. bitonic sort of (key, index) ascending; index breaks ties -> stable order
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int p = tid; p < (npow2 >> 1); p += kSelThreads) {
        const int lo = 2 * p - (p & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const unsigned long long ka = keys[lo], kb = keys[hi];
        const uint32_t ia = idx[lo], ib = idx[hi];
        const bool gt = (ka > kb) || (ka == kb && ia > ib);
        if (gt == asc) {
          keys[lo] = kb; keys[hi] = ka;
          idx[lo] = ib; idx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  // 3. contiguous chunk per thread over the nv sorted valid records
  const int ipt = (nv + kSelThreads - 1) / kSelThreads;
  const int b0 = min(nv, tid * ipt), b1 = min(nv, b0 + ipt);
  long long kv_sum = 0;
  int n_forced = 0;
  for (int p = b0; p < b1; ++p) {
    const Record r = rec[idx[p]];
    kv_sum += (long long)r.kv;
    n_forced += (r.keybits >> 31) == 0u ? 1 : 0;
  }
  long long kv_off;
  int f_off, dummy;
  block_scan3(sh, kv_sum, n_forced, 0, kv_off, f_off, dummy);
  const long long kv_total = sh.total;
  const int nf = sh.cnt_total;
  // forced records are the sorted prefix [0, nf): S_f = cumulative kv at nf - 1
  __shared__ long long s_Sf;
  __shared__ int s_fit;
  if (tid == 0) { s_Sf = 0; s_fit = 0; }
  __syncthreads();
  int my_fit = 0;
  {
    long long cum = kv_off;
    for (int p = b0; p < b1; ++p) {
      cum += (long long)rec[idx[p]].kv;
      if (p == nf - 1) s_Sf = cum;
      if (cum <= budget) ++my_fit;   // cum is non-decreasing: fitting positions are a prefix
    }
  }
  atomicAdd(&s_fit, my_fit);
  __syncthreads();
  const long long Sf = nf > 0 ? s_Sf : 0;
  const int cap = max_run > 0 ? max_run : nv;
  int n_run, status;
  if (Sf > budget || nf > cap) {
    n_run = nf;
    status = TRAIL_WARN_OVER_BUDGET;
  } else {
    n_run = min(s_fit, cap);
    status = TRAIL_OK;
  }
  (void)kv_total;
  // 4. lists in priority order
  int my_pre = 0, my_adm = 0;
  for (int p = b0; p < b1; ++p) {
    const Record r = rec[idx[p]];
    const bool running = (r.gid >> 31) != 0u;
    const uint32_t gid = r.gid & 0x7FFFFFFFu;
    if (p < n_run) {
      run_ids[p] = gid;
      if (!running) ++my_adm;
    } else if (running) {
      ++my_pre;
    }
  }
  long long unused;
  int pre_off, adm_off;
  block_scan3(sh, 0, my_pre, my_adm, unused, pre_off, adm_off);
  const int n_pre = sh.cnt_total, n_adm = sh.cnt2_total;
  for (int p = b0; p < b1; ++p) {
    const Record r = rec[idx[p]];
    const bool running = (r.gid >> 31) != 0u;
    const uint32_t gid = r.gid & 0x7FFFFFFFu;
    if (p < n_run) {
      if (!running) adm_ids[adm_off++] = gid;
    } else if (running) {
      pre_ids[pre_off++] = gid;
    }
  }
  if (tid == 0) {
    counts[0] = n_run;
    counts[1] = n_pre;
    counts[2] = n_adm;
    counts[3] = status;
  }
}

int select_smem_capacity() { return kSmemCapRecords; }

size_t select_scratch_bytes(int n_max) {
  int p = 1;
  while (p < n_max) p <<= 1;
  if (p <= kSmemCapRecords) return 0;
  return (size_t)p * (8 + 4);
}

cudaError_t select_prepare(Ctx &c) {
  (void)c;
  cudaError_t e = select_fast_prepare();
  if (e == cudaSuccess) e = select_radix_prepare();
  if (e == cudaSuccess) e = select_rank_prepare();
  if (e == cudaSuccess) e = select_bucket_prepare();
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(trail_select_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kSmemCapRecords * 12);
}

cudaError_t launch_select(const Ctx &c, const Record *rec, int n, int64_t budget, int max_run,
                          uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                          cudaStream_t s) {
  if (select_impl() == 0 && n <= kRankMaxRecords)
    return launch_select_rank(c, rec, nullptr, nullptr, nullptr, nullptr, nullptr, n, budget,
                              max_run, run, pre, adm, counts, s);
  if (select_impl() == 0 && n <= c.bk_cap)
    return launch_select_bucket(c, rec, n, budget, max_run, run, pre, adm, counts, s);
  if (select_impl() != 2 && n <= select_radix_capacity())
    return launch_select_radix(c, rec, nullptr, nullptr, nullptr, nullptr, nullptr, n, budget,
                               max_run, run, pre, adm, counts, s);
  if (n <= select_fast_capacity())
    return launch_select_fast(c, rec, nullptr, nullptr, nullptr, nullptr, nullptr, n, budget,
                              max_run, run, pre, adm, counts, s);
  int p = 1;
  while (p < n) p <<= 1;
  if (p < 2) p = 2;
  unsigned long long *gk = nullptr;
  uint32_t *gi = nullptr;
  size_t smem = (size_t)p * 12;
  if (p > kSmemCapRecords) {
    if (!c.sel_scratch || c.sel_scratch_bytes < (size_t)p * 12) return cudaErrorInvalidValue;
    gk = reinterpret_cast<unsigned long long *>(c.sel_scratch);
    gi = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(c.sel_scratch) + (size_t)p * 8);
    smem = 0;
  }
  trail_select_large_kernel<<<1, kSelThreads, smem, s>>>(rec, n, p, (long long)budget, max_run, gk, gi,
                                                   run, pre, adm, counts);
  return cudaGetLastError();
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
