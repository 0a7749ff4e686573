// K4 (row a6) with K5 (row a4) fused — multi-CTA selection by rank counting.
//
// Same contract as the other selection kernels: order = composite 64-bit key
// (keybits << 32 | arrival_seq) ascending — forced first (rank -inf), then the
// shortest predicted remaining length, ties FCFS, then input position
// (stable) — run set = every forced record + the longest prefix of the rest within the KV
// budget and the run cap (strict prefix, D-15; forced overflow -> D-16).
//
// Instead of one CTA sorting (a chain of ~60 block barriers), every CTA of a small grid
// stages all n composite keys in shared memory and computes the exact rank of 64 records
// by counting smaller keys (8 threads per record, keys broadcast from shared memory), then
// scatters each record to its rank in a global array: all 148 SMs count in parallel, and
// no barrier chain is on the critical path.  The last CTA to finish (release/acquire
// counter) runs the linear part — one block scan over the sorted records gives the
// cumulative KV, forced and running counts from which the cut and the run / preempt / admit
// list positions follow directly.
//
// Local selection (rec_in == nullptr): every CTA builds the keys from the slot state
// (row a4: key = L_t, or E_pi[L] if never observed; forced = running and a >= floor(c r))
// and the owner of a record writes it (16 B) to `rec_out` for trail_schedule_pack parity.
#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int kT = 512;               // threads per CTA
constexpr int kItems = kT / 8;        // records ranked per CTA
constexpr int kRankCap = 8192;        // keys staged in shared memory (64 KB)

struct RkShared {
  long long v0[kT / 32], v1[kT / 32];
  int c0[kT / 32], c1[kT / 32], c2[kT / 32];
  long long tv0, tv1;
  int tc0, tc1, tc2;
  int last, nv;
};

// exclusive block scan over (int64 a, int64 b, int x, int y, int z); totals in sh.t*
__device__ __forceinline__ void rk_scan(RkShared &sh, long long &a, long long &b, int &x, int &y,
                                        int &z) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long ia = a, ib = b;
  int ix = x, iy = y, iz = z;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long ta = __shfl_up_sync(0xffffffffu, ia, o);
    const long long tb = __shfl_up_sync(0xffffffffu, ib, o);
    const int tx = __shfl_up_sync(0xffffffffu, ix, o);
    const int ty = __shfl_up_sync(0xffffffffu, iy, o);
    const int tz = __shfl_up_sync(0xffffffffu, iz, o);
    if (lane >= o) { ia += ta; ib += tb; ix += tx; iy += ty; iz += tz; }
  }
  if (lane == 31) { sh.v0[w] = ia; sh.v1[w] = ib; sh.c0[w] = ix; sh.c1[w] = iy; sh.c2[w] = iz; }
  __syncthreads();
  if (w == 0) {
    constexpr int W = kT / 32;
    long long wa = lane < W ? sh.v0[lane] : 0, wb = lane < W ? sh.v1[lane] : 0;
    int wx = lane < W ? sh.c0[lane] : 0, wy = lane < W ? sh.c1[lane] : 0;
    int wz = lane < W ? sh.c2[lane] : 0;
    const long long a0 = wa, b0 = wb;
    const int x0 = wx, y0 = wy, z0 = wz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long ta = __shfl_up_sync(0xffffffffu, wa, o);
      const long long tb = __shfl_up_sync(0xffffffffu, wb, o);
      const int tx = __shfl_up_sync(0xffffffffu, wx, o);
      const int ty = __shfl_up_sync(0xffffffffu, wy, o);
      const int tz = __shfl_up_sync(0xffffffffu, wz, o);
      if (lane >= o) { wa += ta; wb += tb; wx += tx; wy += ty; wz += tz; }
    }
    if (lane < W) {
      sh.v0[lane] = wa - a0; sh.v1[lane] = wb - b0;
      sh.c0[lane] = wx - x0; sh.c1[lane] = wy - y0; sh.c2[lane] = wz - z0;
    }
    if (lane == W - 1) { sh.tv0 = wa; sh.tv1 = wb; sh.tc0 = wx; sh.tc1 = wy; sh.tc2 = wz; }
  }
  __syncthreads();
  a = sh.v0[w] + ia - a; b = sh.v1[w] + ib - b;
  x = sh.c0[w] + ix - x; y = sh.c1[w] + iy - y; z = sh.c2[w] + iz - z;
  __syncthreads();
}

// Row a4: the 16-byte record of request i (key L_t or E_pi[L]; forced = running, observed,
// a >= floor(c r)).  err bits are idempotent (every CTA may set them).
__device__ __forceinline__ Record rk_make_record(int i, const uint32_t *ids, const uint32_t *arrival,
                                                 const int32_t *kv, const uint8_t *running,
                                                 const SlotMeta *meta, const HeadConsts *cst,
                                                 int max_slots, uint32_t id_base, uint32_t *err,
                                                 bool flag_errors) {
  const uint32_t slot = __ldg(ids + i);
  const bool run = __ldg(running + i) != 0;
  int32_t kvb = __ldg(kv + i);
  if (kvb < 0) {
    if (flag_errors) atomicOr(err, TRAIL_DEV_NEG_KV);
    kvb = 0;
  }
  float key = cst->prior_L;
  bool forced = false;
  if (slot < (uint32_t)max_slots) {
    const SlotMeta m = meta[slot];
    if (m.flags & 1u) {
      key = m.L;
      forced = run && (m.age >= m.thr);
    }
  } else {
    if (flag_errors) atomicOr(err, TRAIL_DEV_BAD_ID);
    key = INFINITY;
  }
  uint32_t kb;
  if (isfinite(key) && key >= 0.f) {
    kb = __float_as_uint(key) & 0x7FFFFFFFu;
  } else {
    if (flag_errors && slot < (uint32_t)max_slots) atomicOr(err, TRAIL_DEV_NONFIN);
    kb = 0x7F800000u;
  }
  Record r;
  r.keybits = (forced ? 0u : 0x80000000u) | kb;
  r.arrival = __ldg(arrival + i);
  r.kv = (uint32_t)kvb;
  r.gid = ((id_base + slot) & 0x7FFFFFFFu) | (run ? 0x80000000u : 0u);
  return r;
}

__device__ __forceinline__ unsigned long long rk_key(const Record &r) {
  return r.keybits == kPadKey ? ~0ull : ((unsigned long long)r.keybits << 32) | r.arrival;
}
}  // namespace

template <int E>
__global__ void __launch_bounds__(kT)
trail_select_rank_kernel(const Record *__restrict__ rec_in, Record *__restrict__ rec_out,
                         const uint32_t *__restrict__ ids, const uint32_t *__restrict__ arrival,
                         const int32_t *__restrict__ kv, const uint8_t *__restrict__ running,
                         const SlotMeta *__restrict__ meta, const HeadConsts *__restrict__ cst,
                         int max_slots, uint32_t id_base, uint32_t *__restrict__ err, int n,
                         long long budget, int max_run, Record *__restrict__ sorted,
                         uint32_t *__restrict__ done_cnt, uint32_t *__restrict__ run_ids,
                         uint32_t *__restrict__ pre_ids, uint32_t *__restrict__ adm_ids,
                         int32_t *__restrict__ counts) {
  extern __shared__ unsigned long long skey[];   // [n]
  __shared__ RkShared sh;
  const int tid = threadIdx.x, lane = tid & 31;
  griddep_wait();     // slot state from the predict kernels
  griddep_launch();

  // 1. all n composite keys -> shared memory; count the valid (non-padding) records
  int my_valid = 0;
  for (int j = tid; j < n; j += kT) {
    Record r = rec_in ? rec_in[j]
                      : rk_make_record(j, ids, arrival, kv, running, meta, cst, max_slots,
                                       id_base, err, blockIdx.x == 0);
    const unsigned long long kk = rk_key(r);
    skey[j] = kk;
    my_valid += kk != ~0ull ? 1 : 0;
  }
  {
    long long a = 0, b = 0;
    int x = my_valid, y = 0, z = 0;
    rk_scan(sh, a, b, x, y, z);     // (also the barrier that publishes skey)
  }
  const int nv = sh.tc0;

  // 2. exact rank of my records: 8 threads per record, each counting 1/8 of the keys
  {
    const int a = blockIdx.x * kItems + (tid >> 3), part = tid & 7;
    const bool have = a < n;
    const unsigned long long ka = have ? skey[a] : ~0ull;
    int cnt = 0;
    if (have && ka != ~0ull) {
      int j = part;
      for (; j + 24 < n; j += 32) {
        const unsigned long long k0 = skey[j], k1 = skey[j + 8], k2 = skey[j + 16],
                                 k3 = skey[j + 24];
        cnt += (k0 < ka || (k0 == ka && j < a)) ? 1 : 0;
        cnt += (k1 < ka || (k1 == ka && j + 8 < a)) ? 1 : 0;
        cnt += (k2 < ka || (k2 == ka && j + 16 < a)) ? 1 : 0;
        cnt += (k3 < ka || (k3 == ka && j + 24 < a)) ? 1 : 0;
      }
      for (; j < n; j += 8) {
        const unsigned long long k0 = skey[j];
        cnt += (k0 < ka || (k0 == ka && j < a)) ? 1 : 0;
      }
    }
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, 4);
    if (have && part == 0 && ka != ~0ull) {
      const Record r = rec_in ? rec_in[a]
                              : rk_make_record(a, ids, arrival, kv, running, meta, cst,
                                               max_slots, id_base, err, false);
      sorted[cnt] = r;
      if (!rec_in && rec_out) rec_out[a] = r;
    }
  }

  // 3. the last CTA to finish runs the linear part
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const uint32_t old = atomicAdd(done_cnt, 1u);
    const bool last = old == gridDim.x - 1;
    if (last) *done_cnt = 0u;       // re-arm for the next launch
    sh.last = last ? 1 : 0;
  }
  __syncthreads();
  if (!sh.last) return;
  __threadfence();

  // blocked arrangement: thread t owns sorted positions [t*E, t*E + E)
  uint32_t kvv[E], gidv[E];
  unsigned fmask = 0u, rmask = 0u;
  long long kv_t = 0, fkv_t = 0;
  int f_t = 0, r_t = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int p = tid * E + e;
    kvv[e] = 0u;
    gidv[e] = 0u;
    if (p < nv) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(sorted + p));
      kvv[e] = v.z;
      gidv[e] = v.w;
      const bool forced = (v.x >> 31) == 0u;
      const bool runn = (v.w >> 31) != 0u;
      fmask |= forced ? 1u << e : 0u;
      rmask |= runn ? 1u << e : 0u;
      kv_t += v.z;
      fkv_t += forced ? v.z : 0u;
      f_t += forced ? 1 : 0;
      r_t += runn ? 1 : 0;
    }
  }
  long long kv_off = kv_t, fkv_dummy = fkv_t;
  int f_off = f_t, r_off = r_t, z_dummy = 0;
  rk_scan(sh, kv_off, fkv_dummy, f_off, r_off, z_dummy);
  const long long Sf = sh.tv1;       // KV of the forced set (the sorted prefix [0, nf))
  const int nf = sh.tc0;
  const int R_total = sh.tc1;        // running requests among the valid records
  // non-forced positions whose cumulative KV fits: a prefix (cumulative KV is monotone)
  int fit_t = 0;
  {
    long long cum = kv_off;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int p = tid * E + e;
      if (p < nv) {
        cum += kvv[e];
        if (!(fmask >> e & 1u) && cum <= budget) ++fit_t;
      }
    }
  }
  const int cap = max_run > 0 ? max_run : nv;
  int n_run, status;
  {
    long long a = 0, b = 0;
    int x = fit_t, y = 0, z = 0;
    rk_scan(sh, a, b, x, y, z);
    const int n_fit = sh.tc0;
    if (Sf > budget || nf > cap) { n_run = nf; status = TRAIL_WARN_OVER_BUDGET; }
    else { n_run = min(nf + n_fit, cap); status = TRAIL_OK; }
  }
  // running requests before the cut, R(n_run)
  int R_cut;
  {
    int rb_t = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int p = tid * E + e;
      if (p < nv && p < n_run && (rmask >> e & 1u)) ++rb_t;
    }
    long long a = 0, b = 0;
    int x = rb_t, y = 0, z = 0;
    rk_scan(sh, a, b, x, y, z);
    R_cut = sh.tc0;
  }
  {
    int rp = r_off;                  // running requests at sorted positions < p
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int p = tid * E + e;
      if (p < nv) {
        const bool runn = (rmask >> e & 1u) != 0u;
        const uint32_t gid = gidv[e] & 0x7FFFFFFFu;
        if (p < n_run) {
          run_ids[p] = gid;
          if (!runn) adm_ids[p - rp] = gid;     // waiting requests before p: p - rp
        } else if (runn) {
          pre_ids[rp - R_cut] = gid;
        }
        rp += runn ? 1 : 0;
      }
    }
  }
  if (tid == 0) {
    counts[0] = n_run;
    counts[1] = R_total - R_cut;
    counts[2] = n_run - R_cut;
    counts[3] = status;
  }
  (void)lane;
  (void)fkv_dummy;
  (void)z_dummy;
}

// ------------------------------------------------------------------ host
int select_rank_capacity() { return kRankCap; }

cudaError_t select_rank_prepare() {
  cudaError_t e = cudaSuccess;
#define RK_ATTR(EE)                                                                     \
  if (e == cudaSuccess)                                                                 \
    e = cudaFuncSetAttribute(trail_select_rank_kernel<EE>,                              \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kRankCap * 8);
  RK_ATTR(1) RK_ATTR(2) RK_ATTR(4) RK_ATTR(8) RK_ATTR(16)
#undef RK_ATTR
  return e;
}

cudaError_t launch_select_rank(const Ctx &c, const Record *rec_in, Record *rec_out,
                               const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                               const uint8_t *running, int n, int64_t budget, int max_run,
                               uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                               cudaStream_t s) {
  if (n > kRankCap || !c.rank_sorted || !c.rank_cnt) return cudaErrorInvalidValue;
  const int grid = n > 0 ? (n + kItems - 1) / kItems : 1;
  const size_t smem = (size_t)n * 8;
#define RK_LAUNCH(EE)                                                                         \
  return launch_k(trail_select_rank_kernel<EE>, dim3(grid), dim3(kT), smem, s, rec_in, rec_out, \
                  ids, arrival, kv, running, (const SlotMeta *)c.meta,                        \
                  (const HeadConsts *)c.consts, c.cfg.max_slots, c.cfg.id_base, c.dev_err, n, \
                  (long long)budget, max_run, c.rank_sorted, c.rank_cnt, run, pre, adm, counts)
  if (n <= kT) RK_LAUNCH(1);
  if (n <= 2 * kT) RK_LAUNCH(2);
  if (n <= 4 * kT) RK_LAUNCH(4);
  if (n <= 8 * kT) RK_LAUNCH(8);
  RK_LAUNCH(16);
#undef RK_LAUNCH
}

}  // namespace trail
