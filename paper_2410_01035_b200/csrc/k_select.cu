// K4 — selection (row a6), register/shuffle bitonic variant for up to 16384 records, with
// the record build of K5 (row a4) fused in when the selection is local (one rank).
//
// P:171 "prioritizing those with the shortest predicted remaining time ... the number of
// requests that can be scheduled simultaneously is limited by the available GPU memory";
// P:394 preemption only for the first floor(C r) iterations (rank -inf afterwards,
// P:830-831); "ranks all requests (running and waiting)"; ties FCFS.
//
// One CTA of 1024 threads.  Element i = e*1024 + t lives in register slot e of thread t
// (E = N/1024 slots).  Bitonic compare-exchange stages with stride >= 1024 are in-thread
// register swaps, 32 <= stride < 1024 go through shared memory, stride < 32 are warp
// shuffles; the 64-bit composite (keybits << 32 | arrival_seq) is tie-broken by input
// position, so the order equals a stable sort.  Then per 1024-slab block scans give the
// cumulative KV blocks in priority order, the strict-prefix cut under the budget / run cap
// (D-15, D-16), and the compaction offsets of the preempt / admit lists.
#include <algorithm>

#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int kT = 1024;
constexpr int kW = kT / 32;

struct Scan3 {
  long long v[kW];
  int a[kW], b[kW];
  long long tv;
  int ta, tb;
};

// records written earlier in this kernel by other threads: read coherently through L2
__device__ __forceinline__ Record load_rec(const Record *p) {
  const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(p));
  Record r;
  r.keybits = v.x; r.arrival = v.y; r.kv = v.z; r.gid = v.w;
  return r;
}

__device__ __forceinline__ bool key_less(unsigned long long ka, uint32_t xa,
                                         unsigned long long kb, uint32_t xb) {
  return ka < kb || (ka == kb && xa < xb);
}

// exclusive block scan of (v, a, b); totals in sh.tv/ta/tb
__device__ __forceinline__ void scan3(Scan3 &sh, long long v, int a, int b, long long &ev,
                                      int &ea, int &eb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long iv = v;
  int ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long tv = __shfl_up_sync(0xffffffffu, iv, o);
    const int ta = __shfl_up_sync(0xffffffffu, ia, o);
    const int tb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { iv += tv; ia += ta; ib += tb; }
  }
  if (lane == 31) { sh.v[w] = iv; sh.a[w] = ia; sh.b[w] = ib; }
  __syncthreads();
  if (w == 0) {
    const long long wv0 = sh.v[lane];
    const int wa0 = sh.a[lane], wb0 = sh.b[lane];
    long long wv = wv0;
    int wa = wa0, wb = wb0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long tv = __shfl_up_sync(0xffffffffu, wv, o);
      const int ta = __shfl_up_sync(0xffffffffu, wa, o);
      const int tb = __shfl_up_sync(0xffffffffu, wb, o);
      if (lane >= o) { wv += tv; wa += ta; wb += tb; }
    }
    sh.v[lane] = wv - wv0;
    sh.a[lane] = wa - wa0;
    sh.b[lane] = wb - wb0;
    if (lane == 31) { sh.tv = wv; sh.ta = wa; sh.tb = wb; }
  }
  __syncthreads();
  ev = sh.v[w] + iv - v;
  ea = sh.a[w] + ia - a;
  eb = sh.b[w] + ib - b;
  __syncthreads();
}

template <int E, int ES>
__device__ __forceinline__ void stage_regs(unsigned long long (&k)[E], uint32_t (&x)[E], int t,
                                           int size) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if ((e & ES) == 0) {
      const int e2 = e | ES;
      const int i = e * kT + t;
      const bool asc = (i & size) == 0;
      const bool sw = key_less(k[e2], x[e2], k[e], x[e]) == asc;
      if (sw) {
        const unsigned long long tk = k[e]; k[e] = k[e2]; k[e2] = tk;
        const uint32_t tx = x[e]; x[e] = x[e2]; x[e2] = tx;
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void stage_in_thread(unsigned long long (&k)[E], uint32_t (&x)[E],
                                                int t, int size, int es) {
  if constexpr (E >= 2) { if (es == 1) { stage_regs<E, 1>(k, x, t, size); return; } }
  if constexpr (E >= 4) { if (es == 2) { stage_regs<E, 2>(k, x, t, size); return; } }
  if constexpr (E >= 8) { if (es == 4) { stage_regs<E, 4>(k, x, t, size); return; } }
  if constexpr (E >= 16) { if (es == 8) { stage_regs<E, 8>(k, x, t, size); return; } }
}

// Build the record of local request i (fused K5; same encoding as trail_pack_kernel).
__device__ __forceinline__ Record make_record(int i, const uint32_t *ids, const uint32_t *arrival,
                                              const int32_t *kv, const uint8_t *running,
                                              const SlotMeta *meta, const HeadConsts *cst,
                                              int max_slots, uint32_t id_base, uint32_t *err) {
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
  r.arrival = __ldg(arrival + i);
  r.kv = (uint32_t)kvb;
  r.gid = ((id_base + slot) & 0x7FFFFFFFu) | (run ? 0x80000000u : 0u);
  return r;
}
}  // namespace

// rec_in != nullptr: select over n given records.  rec_in == nullptr: build the n local
// records from (ids, arrival, kv, running) and the slot state, writing them to rec_out.
template <int E>
__global__ void __launch_bounds__(kT, 1)
trail_select_kernel(const Record *rec_in, Record *rec_out,
                    const uint32_t *__restrict__ ids, const uint32_t *__restrict__ arrival,
                    const int32_t *__restrict__ kv, const uint8_t *__restrict__ running,
                    const SlotMeta *__restrict__ meta, const HeadConsts *__restrict__ cst,
                    int max_slots, uint32_t id_base, uint32_t *__restrict__ err, int n,
                    long long budget, int max_run, uint32_t *__restrict__ run_ids,
                    uint32_t *__restrict__ pre_ids, uint32_t *__restrict__ adm_ids,
                    int32_t *__restrict__ counts) {
  constexpr int N = E * kT;
  extern __shared__ __align__(16) uint8_t smem[];
  unsigned long long *sk = reinterpret_cast<unsigned long long *>(smem);
  uint32_t *sx = reinterpret_cast<uint32_t *>(smem + (size_t)N * 8);
  __shared__ Scan3 sh;
  const int t = threadIdx.x;
  const int lane = t & 31;
  const Record *rec = rec_in ? rec_in : rec_out;
  griddep_wait();      // slot state written by the head kernel
  griddep_launch();

  // 1. load / build records; composite keys; padding sorts last
  unsigned long long k[E];
  uint32_t x[E];
  int my_valid = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * kT + t;
    k[e] = ~0ull;
    x[e] = 0xFFFFFFFFu;
    if (i < n) {
      Record r;
      if (rec_in) {
        r = rec_in[i];
      } else {
        r = make_record(i, ids, arrival, kv, running, meta, cst, max_slots, id_base, err);
        rec_out[i] = r;
      }
      if (r.keybits != kPadKey) {
        k[e] = ((unsigned long long)r.keybits << 32) | r.arrival;
        x[e] = (uint32_t)i;
        ++my_valid;
      }
    }
  }
  long long d0;
  int vo, d1;
  scan3(sh, 0, my_valid, 0, d0, vo, d1);
  const int nv = sh.ta;

  // 2. bitonic sort (ascending (key, position))
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= kT) {
        stage_in_thread<E>(k, x, t, size, stride / kT);
      } else if (stride >= 32) {
#pragma unroll
        for (int e = 0; e < E; ++e) { sk[e * kT + t] = k[e]; sx[e * kT + t] = x[e]; }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = e * kT + t;
          const int j = i ^ stride;
          const unsigned long long kj = sk[j];
          const uint32_t xj = sx[j];
          const bool asc = (i & size) == 0;
          const bool take_min = ((i & stride) == 0) == asc;
          const bool pl = key_less(kj, xj, k[e], x[e]);
          if (take_min == pl) { k[e] = kj; x[e] = xj; }
        }
        __syncthreads();
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = e * kT + t;
          const unsigned long long kj = __shfl_xor_sync(0xffffffffu, k[e], stride);
          const uint32_t xj = __shfl_xor_sync(0xffffffffu, x[e], stride);
          const bool asc = (i & size) == 0;
          const bool take_min = ((lane & stride) == 0) == asc;
          const bool pl = key_less(kj, xj, k[e], x[e]);
          if (take_min == pl) { k[e] = kj; x[e] = xj; }
        }
      }
    }
  }

  // 3. forced prefix, KV totals, strict-prefix cut
  Record rs[E];
  long long f_kv = 0;
  int f_cnt = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * kT + t;
    if (i < nv) {
      rs[e] = load_rec(rec + x[e]);
      if ((rs[e].keybits >> 31) == 0u) { f_kv += rs[e].kv; ++f_cnt; }
    } else {
      rs[e].keybits = kPadKey; rs[e].kv = 0; rs[e].gid = 0; rs[e].arrival = 0;
    }
  }
  scan3(sh, f_kv, f_cnt, 0, d0, vo, d1);
  const long long Sf = sh.tv;
  const int nf = sh.ta;
  long long carry = 0;
  int fit = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * kT + t;
    const long long v = i < nv ? (long long)rs[e].kv : 0;
    long long ex;
    scan3(sh, v, 0, 0, ex, vo, d1);
    const long long cum = carry + ex + v;      // inclusive cumulative KV in priority order
    if (i < nv && cum <= budget) ++fit;        // cum is non-decreasing: a prefix
    carry += sh.tv;
  }
  scan3(sh, 0, fit, 0, d0, vo, d1);
  const int n_fit = sh.ta;
  const int cap = max_run > 0 ? max_run : nv;
  int n_run, status;
  if (Sf > budget || nf > cap) { n_run = nf; status = TRAIL_WARN_OVER_BUDGET; }
  else { n_run = min(n_fit, cap); status = TRAIL_OK; }

  // 4. lists in priority order
  int pre_carry = 0, adm_carry = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * kT + t;
    const bool valid = i < nv;
    const bool runn = valid && (rs[e].gid >> 31) != 0u;
    const uint32_t gid = rs[e].gid & 0x7FFFFFFFu;
    const bool in_run = valid && i < n_run;
    const int is_pre = (valid && !in_run && runn) ? 1 : 0;
    const int is_adm = (in_run && !runn) ? 1 : 0;
    if (in_run) run_ids[i] = gid;
    long long dd;
    int po, ao;
    scan3(sh, 0, is_pre, is_adm, dd, po, ao);
    if (is_pre) pre_ids[pre_carry + po] = gid;
    if (is_adm) adm_ids[adm_carry + ao] = gid;
    pre_carry += sh.ta;
    adm_carry += sh.tb;
  }
  if (t == 0) {
    counts[0] = n_run;
    counts[1] = pre_carry;
    counts[2] = adm_carry;
    counts[3] = status;
  }
}

// ------------------------------------------------------------------ host
static int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

cudaError_t select_fast_prepare() {
  cudaError_t e = cudaSuccess;
#define TRAIL_SEL_ATTR(E)                                                                      \
  if (e == cudaSuccess)                                                                        \
    e = cudaFuncSetAttribute(trail_select_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             E * kT * 12);
  TRAIL_SEL_ATTR(1) TRAIL_SEL_ATTR(2) TRAIL_SEL_ATTR(4) TRAIL_SEL_ATTR(8) TRAIL_SEL_ATTR(16)
#undef TRAIL_SEL_ATTR
  return e;
}

int select_fast_capacity() { return 16 * kT; }

cudaError_t launch_select_fast(const Ctx &c, const Record *rec_in, Record *rec_out,
                               const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                               const uint8_t *running, int n, int64_t budget, int max_run,
                               uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                               cudaStream_t s) {
  const int N = std::max(kT, pow2_at_least(std::max(n, 1)));
  const int E = N / kT;
  const size_t smem = (size_t)N * 12;
#define TRAIL_SEL_LAUNCH(EE)                                                                  \
  return launch_k(trail_select_kernel<EE>, dim3(1), dim3(kT), smem, s, rec_in, rec_out, ids,   \
                  arrival, kv, running, (const SlotMeta *)c.meta, (const HeadConsts *)c.consts, \
                  c.cfg.max_slots, c.cfg.id_base, c.dev_err, n, (long long)budget, max_run, run, \
                  pre, adm, counts)
  switch (E) {
    case 1: TRAIL_SEL_LAUNCH(1);
    case 2: TRAIL_SEL_LAUNCH(2);
    case 4: TRAIL_SEL_LAUNCH(4);
    case 8: TRAIL_SEL_LAUNCH(8);
    case 16: TRAIL_SEL_LAUNCH(16);
    default: return cudaErrorInvalidValue;
  }
#undef TRAIL_SEL_LAUNCH
}

}  // namespace trail
