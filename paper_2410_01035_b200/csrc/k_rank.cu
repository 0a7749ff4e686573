// K4 (row a6) with K5 (row a4) fused — multi-CTA selection by rank counting.
//
// Same contract as the other selection kernels: order = composite 64-bit key
// (keybits << 32 | arrival_seq) ascending — forced first (rank -inf), then the
// shortest predicted remaining length, ties FCFS, then input position
// (stable) — run set = every forced record + the longest prefix of the rest within the KV
// budget and the run cap (strict prefix, D-15; forced overflow -> D-16).
//
// Instead of one CTA sorting (a chain of ~60 block barriers), every CTA of a grid sized to
// about one wave stages all n records (key, KV, flags; 16 B each) in shared memory, and for
// each of its own records computes, in ONE pass over all keys (TPI threads per record),
//   pos  = #records ordered before it       (its exact rank: run-list position),
//   cum  = KV of the records before it       (+ its own KV: the cumulative KV at pos),
//   rb   = #running records before it.
// Because forced records sort first, cum includes the forced KV S_f, and the run set is
//   in_run = forced  or  (not over-budget and cum_incl <= budget and pos < cap)
// (the non-forced cumulative KV is monotone, so this is exactly the strict prefix), while
// the list positions follow directly: run_ids[pos], admit_ids[pos - rb] (waiting records
// before pos), and preempt_ids[rb - R(cut)] with R(cut) = running records in the run set —
// the one global quantity, summed with atomics; the last CTA to finish writes the preempt
// list from the (pos -> gid, rb) scratch array.  All SMs work in parallel; the only
// serial part is one pass over the records past the cut.
//
// Local selection (rec_in == nullptr): every CTA builds the records from the slot state
// (row a4: key = L_t, or E_pi[L] if never observed; forced = running and a >= floor(c r))
// and the owner of a record writes it (16 B) to `rec_out` for trail_schedule_pack parity.
#include <stdlib.h>

#include <algorithm>

#include "sm100_ptx.cuh"
#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int kT = 512;               // threads per CTA
constexpr int kRankCap = kRankMaxRecords;   // records staged in shared memory (32 KB)

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

__device__ __forceinline__ unsigned long long rk_key(const Record &r) {
  return r.keybits == kPadKey ? ~0ull : ((unsigned long long)r.keybits << 32) | r.arrival;
}
}  // namespace

// Per-record state kept in shared memory by every CTA (16 B): composite key (forced <=>
// bit 63 clear), KV blocks, (id_base + slot) | running << 31.
struct RkItem {
  unsigned long long key;
  uint32_t kv;
  uint32_t gid;
};

__global__ void __launch_bounds__(kT)
trail_select_rank_kernel(const Record *__restrict__ rec_in, Record *__restrict__ rec_out,
                         const uint32_t *__restrict__ ids, const uint32_t *__restrict__ arrival,
                         const int32_t *__restrict__ kv, const uint8_t *__restrict__ running,
                         const SlotMeta *__restrict__ meta, const HeadConsts *__restrict__ cst,
                         int max_slots, uint32_t id_base, uint32_t *__restrict__ err, int n,
                         int ipc_log2, long long budget, int max_run,
                         uint2 *__restrict__ scratch, uint32_t *__restrict__ gcnt,
                         uint32_t *__restrict__ run_ids, uint32_t *__restrict__ pre_ids,
                         uint32_t *__restrict__ adm_ids, int32_t *__restrict__ counts,
                         uint64_t *__restrict__ trace) {
  extern __shared__ RkItem sitem[];   // [n]
  __shared__ RkShared sh;
  __shared__ unsigned long long s_part[kT / 32][3];
  __shared__ uint32_t s_cta_run, s_cta_rcut;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t *tr = trace ? trace + 16 * (2048 + (int64_t)blockIdx.x) : nullptr;   // diagnostics
  if (tr && tid == 0) tr[0] = ptx::gtimer();
  if (tid == 0) { s_cta_run = 0u; s_cta_rcut = 0u; }
  // inputs of the local path are the caller's (not produced by the predict kernels): stage
  // them before waiting on the previous kernel, so only the slot-state loads follow the wait
  if (!rec_in) {
    for (int j = tid; j < n; j += kT) {
      RkItem it;
      const uint32_t slot = __ldg(ids + j);
      it.key = __ldg(arrival + j);                       // arrival (low word) for now
      it.kv = (uint32_t)__ldg(kv + j);
      it.gid = slot | (__ldg(running + j) ? 0x80000000u : 0u);
      sitem[j] = it;
    }
  }
  griddep_wait();     // slot state from the predict kernels
  griddep_launch();
  if (tr && tid == 0) tr[1] = ptx::gtimer();

  // 1. every record's key, kv and flags -> shared memory; forced count / KV, running count
  long long fkv_t = 0;
  int f_t = 0, r_t = 0, v_t = 0;
  // every dependent load of a thread (slot state / given records) issued before any is used:
  // one L2 round trip after the wait instead of one per 512 records
  constexpr int kPer = kRankCap / kT;
  SlotMeta mt[kPer];
  Record rin[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int j = tid + u * kT;
    if (j < n) {
      if (rec_in) {
        rin[u] = rec_in[j];
      } else {
        const uint32_t slot = sitem[j].gid & 0x7FFFFFFFu;
        if (slot < (uint32_t)max_slots) mt[u] = meta[slot];
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int j = tid + u * kT;
    if (j >= n) break;
    Record r;
    if (rec_in) {
      r = rin[u];
    } else {   // row a4 from the staged inputs + the slot state
      const RkItem in = sitem[j];
      const uint32_t slot = in.gid & 0x7FFFFFFFu;
      const bool run = (in.gid >> 31) != 0u;
      int32_t kvb = (int32_t)in.kv;
      if (kvb < 0) {
        if (blockIdx.x == 0) atomicOr(err, TRAIL_DEV_NEG_KV);
        kvb = 0;
      }
      float key = cst->prior_L;
      bool forced = false;
      if (slot < (uint32_t)max_slots) {
        const SlotMeta m = mt[u];
        if (m.flags & 1u) {
          key = m.L;
          forced = run && (m.age >= m.thr);
        }
      } else {
        if (blockIdx.x == 0) atomicOr(err, TRAIL_DEV_BAD_ID);
        key = INFINITY;
      }
      uint32_t kb;
      if (isfinite(key) && key >= 0.f) {
        kb = __float_as_uint(key) & 0x7FFFFFFFu;
      } else {
        if (blockIdx.x == 0 && slot < (uint32_t)max_slots) atomicOr(err, TRAIL_DEV_NONFIN);
        kb = 0x7F800000u;
      }
      r.keybits = (forced ? 0u : 0x80000000u) | kb;
      r.arrival = (uint32_t)in.key;
      r.kv = (uint32_t)kvb;
      r.gid = ((id_base + slot) & 0x7FFFFFFFu) | (run ? 0x80000000u : 0u);
    }
    RkItem it;
    it.key = rk_key(r);
    const bool valid = it.key != ~0ull;
    const bool forced = valid && (r.keybits >> 31) == 0u;
    const bool runn = valid && (r.gid >> 31) != 0u;
    it.kv = valid ? r.kv : 0u;
    it.gid = valid ? r.gid : 0u;
    sitem[j] = it;
    v_t += valid ? 1 : 0;
    f_t += forced ? 1 : 0;
    r_t += runn ? 1 : 0;
    fkv_t += forced ? (long long)r.kv : 0;
  }
  {
    long long a = fkv_t, b = 0;
    int x = v_t, y = f_t, z = r_t;
    rk_scan(sh, a, b, x, y, z);     // totals only (also publishes sitem)
  }
  const int nv = sh.tc0, nf = sh.tc1, R_total = sh.tc2;
  const long long Sf = sh.tv0;
  const int cap = max_run > 0 ? max_run : nv;
  const bool over = Sf > budget || nf > cap;   // D-16: run = forced only
  if (tr && tid == 0) tr[2] = ptx::gtimer();

  // 2. for each of my records: position in the order, cumulative KV through it, running
  //    records before it — one pass over all keys, TPI threads per record
  const int ipc = 1 << ipc_log2, tpi = kT >> ipc_log2;
  const int li = tid / tpi, part = tid % tpi;
  const int i = blockIdx.x * ipc + li;
  const bool have = i < n;
  const RkItem me = have ? sitem[i] : RkItem{~0ull, 0u, 0u};
  const bool mine = have && me.key != ~0ull;
  unsigned long long cnt = 0, cum = 0, rb = 0;
  if (mine) {
    const unsigned long long ki = me.key;
    for (int j = part; j < n; j += tpi) {
      const RkItem o = sitem[j];
      const bool less = o.key < ki || (o.key == ki && j < i);
      if (less) {
        cnt += 1;
        cum += o.kv;
        rb += o.gid >> 31;
      }
    }
  }
  // reduce over the tpi threads of a record (consecutive threads)
  const int wl = tpi < 32 ? tpi : 32;
  for (int o = 1; o < wl; o <<= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    cum += __shfl_xor_sync(0xffffffffu, cum, o);
    rb += __shfl_xor_sync(0xffffffffu, rb, o);
  }
  if (tpi > 32) {
    if (lane == 0) { s_part[warp][0] = cnt; s_part[warp][1] = cum; s_part[warp][2] = rb; }
    __syncthreads();
    if (part == 0) {
      const int w0 = tid >> 5, nw = tpi >> 5;
      cnt = 0; cum = 0; rb = 0;
      for (int q = 0; q < nw; ++q) {
        cnt += s_part[w0 + q][0]; cum += s_part[w0 + q][1]; rb += s_part[w0 + q][2];
      }
    }
  }
  if (mine && part == 0) {
    const int pos = (int)cnt;
    const bool forced = (me.key >> 63) == 0ull;
    const bool runn = (me.gid >> 31) != 0u;
    const long long cum_incl = (long long)cum + me.kv;
    const bool in_run = forced ? true : (!over && cum_incl <= budget && pos < cap);
    const uint32_t gid = me.gid & 0x7FFFFFFFu;
    if (in_run) {
      run_ids[pos] = gid;
      if (!runn) adm_ids[pos - (int)rb] = gid;   // waiting records before pos: pos - rb
      atomicAdd(&s_cta_run, 1u);
      if (runn) atomicAdd(&s_cta_rcut, 1u);
    }
    scratch[pos] = make_uint2(me.gid, (uint32_t)rb);
    if (!rec_in && rec_out) {
      Record r;
      r.keybits = (uint32_t)(me.key >> 32);
      r.arrival = (uint32_t)me.key;
      r.kv = me.kv;
      r.gid = me.gid;
      rec_out[i] = r;
    }
  }
  __syncthreads();
  if (tr && tid == 0) tr[3] = ptx::gtimer();

  // 3. per-CTA totals in ONE 64-bit acq_rel atomic (done:16 | run-set size:24 | running in
  //    the run set:24): the last CTA gets every total from the returned value
  __shared__ unsigned long long s_tot;
  if (tid == 0) {
    const unsigned long long inc = (1ull << 48) | ((unsigned long long)s_cta_run << 24) |
                                   (unsigned long long)s_cta_rcut;
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;"
                 : "=l"(old) : "l"(gcnt), "l"(inc) : "memory");
    const unsigned long long tot = old + inc;
    sh.last = (int)(tot >> 48) == (int)gridDim.x ? 1 : 0;
    if (sh.last) *reinterpret_cast<unsigned long long *>(gcnt) = 0ull;   // re-arm
    s_tot = tot;
  }
  __syncthreads();
  if (tr && tid == 0) { tr[4] = ptx::gtimer(); tr[14] = sh.last; }
  if (!sh.last) return;
  const int n_run = (int)((s_tot >> 24) & 0xFFFFFFull);
  const int R_cut = (int)(s_tot & 0xFFFFFFull);
  if (tr && tid == 0) tr[5] = ptx::gtimer();
  // positions past the cut: all loads of a thread in flight before its stores
  for (int p0 = n_run; p0 < nv; p0 += 4 * kT) {
    uint2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u * kT + tid;
      v[u] = p < nv ? __ldcg(scratch + p) : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v[u].x >> 31) pre_ids[(int)v[u].y - R_cut] = v[u].x & 0x7FFFFFFFu;
  }
  if (tr && tid == 0) tr[6] = ptx::gtimer();
  __syncthreads();
  if (tid == 0) {
    counts[0] = n_run;
    counts[1] = R_total - R_cut;
    counts[2] = n_run - R_cut;
    counts[3] = over ? TRAIL_WARN_OVER_BUDGET : TRAIL_OK;
  }
  if (tr && tid == 0) tr[7] = ptx::gtimer();
  (void)lane;
}

// ------------------------------------------------------------------ host
cudaError_t select_rank_prepare() {
  cudaError_t e = cudaFuncSetAttribute(trail_select_rank_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kRankCap * (int)sizeof(RkItem));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(trail_select_rank_kernel,
                              cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

cudaError_t launch_select_rank(const Ctx &c, const Record *rec_in, Record *rec_out,
                               const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                               const uint8_t *running, int n, int64_t budget, int max_run,
                               uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                               cudaStream_t s) {
  if (n > kRankCap || !c.rank_sorted || !c.rank_cnt) return cudaErrorInvalidValue;
  // records per CTA: a power of two spreading the n records over about one wave of SMs,
  // with at least 8 threads per record
  int ipc_log2 = 0;
  while ((1 << ipc_log2) * c.num_sms < n && ipc_log2 < 6) ++ipc_log2;
  const int ipc = 1 << ipc_log2;
  const int grid = n > 0 ? (n + ipc - 1) / ipc : 1;
  const size_t smem = (size_t)std::max(n, 1) * sizeof(RkItem);
  return launch_k(trail_select_rank_kernel, dim3(grid), dim3(kT), smem, s, rec_in, rec_out, ids,
                  arrival, kv, running, (const SlotMeta *)c.meta, (const HeadConsts *)c.consts,
                  c.cfg.max_slots, c.cfg.id_base, c.dev_err, n, ipc_log2, (long long)budget,
                  max_run, reinterpret_cast<uint2 *>(c.rank_sorted), c.rank_cnt, run, pre, adm,
                  counts,
                  (c.trace && 2048 + grid <= c.trace_cap) ? c.trace
                                                                                   : nullptr);
}

}  // namespace trail
