// K4 (row a6) for large record counts (multi-rank all-gathers, configs 3-5): a bucketed
// exact ranking in four PDL-chained kernels over the 16-byte records (row a4/a5).
//
// Same contract as every selection kernel: order = (keybits << 32 | arrival, input position)
// ascending — forced first (rank -inf), then shortest predicted remaining length
// (P:171), FCFS ties, then input position (D-18) — run set = all forced + the
// longest prefix of the rest within the KV budget and run cap (strict prefix D-15, overflow
// D-16).
//
// The key of a record is L_t, a convex combination of the bin midpoints, so it lies in
// [m_0, m_{k-1}] (create-time constants): buckets are equal-width L intervals (1024 for the
// forced class, 1024 for the rest), a monotone map of the key.  One exact tie is systematic:
// every never-observed request is keyed E_pi[L] (D-24), and a burst of arrivals puts thousands
// of them on one key; their order is FCFS (arrival), so that key gets its own range of 1024
// arrival sub-buckets between the lower and the upper part of its L interval.
//   B0  (local path) the records (row a4, fused pack); arrival range of the E_pi[L] tie group
//   B1  histogram of (count, KV, running) per bucket (warp-aggregated global atomics)
//   B2  scatter of the records into bucket order (prefix of the counts, atomic cursors)
//   B3  each record counts the records of its own bucket ordered before it (the bucket range
//       is staged in shared memory; 16 threads per record), adds the bucket prefixes
//       -> position, cumulative KV, running-before, and the lists follow as in k_rank.cu
//       (one packed acq_rel atomic; the last CTA writes the preempt list and re-arms).
// Cost is O(m + sum over buckets of size^2 / 16).
#include <string.h>

#include <algorithm>

#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int kBH = 1024;               // L buckets per class (forced / not forced)
constexpr int kTie = 1024;              // arrival sub-buckets of the E_pi[L] tie group
constexpr int kBUsed = 2 * kBH + 1 + kTie;
constexpr int kB = 4096;                // bucket slots (kBUsed rounded up; 4 per scan thread)
static_assert(kBUsed <= kB, "bucket layout exceeds the scanned slots");
constexpr int kB3Threads = 1024;
constexpr int kB3Tpi = 16;              // threads per record in B3
constexpr int kB3Items = kB3Threads / kB3Tpi;
constexpr int kStageCap = 8192;         // bucket entries staged in shared memory (128 KB)

struct BkEntry {                        // bucket-sorted record (16 B)
  unsigned long long key;               // keybits << 32 | arrival
  uint32_t kvr;                         // kv | running << 31  (kv_blocks >= 0 fits 31 bits)
  uint32_t idx;                         // input position (final tie-break, D-18)
};

struct BkParams {
  float m0, scale;                      // L interval of bucket 0, buckets per unit of L
  uint32_t tie_bits;                    // keybits of an unobserved request: !forced | E_pi[L]
  int ustar;                            // L bucket of E_pi[L]
};

__device__ __forceinline__ int bk_lbucket(uint32_t keybits, const BkParams &bp) {
  const float L = __uint_as_float(keybits & 0x7FFFFFFFu);
  const float u = (L - bp.m0) * bp.scale;  // NaN/inf keys -> last bucket of the class
  int b = (u >= 0.f) ? (u < (float)kBH ? (int)u : kBH - 1) : 0;
  if (!(L == L) || L == INFINITY) b = kBH - 1;
  return b;
}

// bucket of a (non-padding) record; tie = (~amin, amax) of the tie group's arrivals
__device__ __forceinline__ int bk_bucket(uint32_t keybits, uint32_t arrival, const BkParams &bp,
                                         uint32_t amin, uint32_t amax) {
  const int u = bk_lbucket(keybits, bp);
  if ((keybits >> 31) == 0u) return u;                                   // forced class
  if (keybits == bp.tie_bits) {
    const unsigned long long span = (unsigned long long)(amax - amin) + 1ull;
    const unsigned long long sub = ((unsigned long long)(arrival - amin) * kTie) / span;
    return kBH + bp.ustar + 1 + (int)(sub < (unsigned long long)kTie ? sub : kTie - 1);
  }
  if (u < bp.ustar) return kBH + u;
  if (u > bp.ustar) return kBH + u + 1 + kTie;
  return keybits < bp.tie_bits ? kBH + bp.ustar : kBH + bp.ustar + 1 + kTie;
}

__device__ __forceinline__ bool bk_less(const BkEntry &a, const BkEntry &b) {
  return a.key < b.key || (a.key == b.key && a.idx < b.idx);
}

// exclusive scan of kB (u32 count, u32 run, u64 kv) bucket totals by a 1024-thread CTA
struct BkScan {
  uint32_t cnt[kB], run[kB];
  unsigned long long kv[kB];
  uint32_t wc[32], wr[32];
  unsigned long long wk[32];
};

__device__ void bk_scan_buckets(BkScan &sh, const uint32_t *hcnt, const uint32_t *hrun,
                                const unsigned long long *hkv) {
  constexpr int PT = kB / kB3Threads;   // consecutive buckets per thread
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t c[PT], r[PT];
  unsigned long long k[PT];
  uint32_t ic = 0, ir = 0;
  unsigned long long ik = 0;
#pragma unroll
  for (int q = 0; q < PT; ++q) {
    c[q] = __ldcg(hcnt + PT * t + q);
    r[q] = __ldcg(hrun + PT * t + q);
    k[q] = __ldcg(hkv + PT * t + q);
    ic += c[q]; ir += r[q]; ik += k[q];
  }
  const uint32_t tc0 = ic, tr0 = ir;
  const unsigned long long tk0 = ik;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t tc = __shfl_up_sync(0xffffffffu, ic, o), tr = __shfl_up_sync(0xffffffffu, ir, o);
    const unsigned long long tk = __shfl_up_sync(0xffffffffu, ik, o);
    if (lane >= o) { ic += tc; ir += tr; ik += tk; }
  }
  if (lane == 31) { sh.wc[w] = ic; sh.wr[w] = ir; sh.wk[w] = ik; }
  __syncthreads();
  if (w == 0) {
    uint32_t a = sh.wc[lane], b = sh.wr[lane];
    unsigned long long cc = sh.wk[lane];
    const uint32_t a0 = a, b0 = b;
    const unsigned long long cc0 = cc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ta = __shfl_up_sync(0xffffffffu, a, o), tb = __shfl_up_sync(0xffffffffu, b, o);
      const unsigned long long tk = __shfl_up_sync(0xffffffffu, cc, o);
      if (lane >= o) { a += ta; b += tb; cc += tk; }
    }
    sh.wc[lane] = a - a0; sh.wr[lane] = b - b0; sh.wk[lane] = cc - cc0;
  }
  __syncthreads();
  uint32_t ec = sh.wc[w] + ic - tc0, er = sh.wr[w] + ir - tr0;
  unsigned long long ek = sh.wk[w] + ik - tk0;
#pragma unroll
  for (int q = 0; q < PT; ++q) {
    sh.cnt[PT * t + q] = ec; sh.run[PT * t + q] = er; sh.kv[PT * t + q] = ek;
    ec += c[q]; er += r[q]; ek += k[q];
  }
  __syncthreads();
}
}  // namespace

// B0: records (local path) and the arrival range of the E_pi[L] tie group
__global__ void __launch_bounds__(256)
trail_bucket_prep_kernel(const Record *__restrict__ rec, Record *__restrict__ rec_out,
                         const uint32_t *__restrict__ ids, const uint32_t *__restrict__ arrival,
                         const int32_t *__restrict__ kvin, const uint8_t *__restrict__ running,
                         const SlotMeta *__restrict__ meta, const HeadConsts *__restrict__ cst,
                         int max_slots, uint32_t id_base, uint32_t *__restrict__ err, int m,
                         uint32_t tie_bits, uint32_t *__restrict__ tie) {
  griddep_wait();     // records from the pack kernel / the all-gather, or the slot state
  griddep_launch();
  for (int i0 = blockIdx.x * blockDim.x; i0 < m; i0 += gridDim.x * blockDim.x) {
    const int i = i0 + threadIdx.x;
    uint32_t kb = kPadKey, arr = 0u;
    if (i < m) {
      if (rec) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(rec + i));
        kb = v.x;
        arr = v.y;
      } else {        // local path: row a4 fused (the record build of trail_schedule_pack)
        const Record r = build_record(__ldg(ids + i), __ldg(arrival + i), __ldg(kvin + i),
                                      __ldg(running + i) != 0, meta, cst, max_slots, id_base, err);
        rec_out[i] = r;
        kb = r.keybits;
        arr = r.arrival;
      }
    }
    const bool t = kb == tie_bits;
    const uint32_t mx = __reduce_max_sync(0xffffffffu, t ? arr : 0u);
    const uint32_t nmn = __reduce_max_sync(0xffffffffu, t ? ~arr : 0u);
    const bool any = __any_sync(0xffffffffu, t);          // every lane votes
    if ((threadIdx.x & 31) == 0 && any) {
      atomicMax(tie, nmn);          // ~min arrival
      atomicMax(tie + 1, mx);       // max arrival
    }
  }
}

// B1: per-bucket totals
__global__ void __launch_bounds__(256)
trail_bucket_hist_kernel(const Record *__restrict__ rec, int m, BkParams bp,
                         const uint32_t *__restrict__ tie, uint32_t *__restrict__ hcnt,
                         uint32_t *__restrict__ hrun, unsigned long long *__restrict__ hkv) {
  griddep_wait();     // records and the tie range from B0
  griddep_launch();
  const uint32_t amin = ~__ldcg(tie), amax = __ldcg(tie + 1);
  const int lane = threadIdx.x & 31;
  for (int i0 = blockIdx.x * blockDim.x; i0 < m; i0 += gridDim.x * blockDim.x) {
    const int i = i0 + threadIdx.x;
    int b = -1;
    uint32_t kvv = 0, runn = 0;
    if (i < m) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(rec + i));
      if (v.x != kPadKey) {
        b = bk_bucket(v.x, v.y, bp, amin, amax);
        kvv = v.z;
        runn = v.w >> 31;
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    const uint32_t c = __popc(peers);
    const uint32_t r = __reduce_add_sync(peers, runn);
    const uint32_t klo = __reduce_add_sync(peers, kvv & 0xFFFFu);
    const uint32_t khi = __reduce_add_sync(peers, kvv >> 16);
    if (b >= 0 && lane == __ffs(peers) - 1) {
      atomicAdd(hcnt + b, c);
      if (r) atomicAdd(hrun + b, r);
      atomicAdd(hkv + b, ((unsigned long long)khi << 16) + klo);
    }
  }
}

// B2: scatter into bucket order
__global__ void __launch_bounds__(kB3Threads)
trail_bucket_scatter_kernel(const Record *__restrict__ rec, int m, BkParams bp,
                            const uint32_t *__restrict__ tie,
                            const uint32_t *__restrict__ hcnt, const uint32_t *__restrict__ hrun,
                            const unsigned long long *__restrict__ hkv,
                            uint32_t *__restrict__ cursor, BkEntry *__restrict__ sorted) {
  extern __shared__ __align__(16) uint8_t bsm[];
  BkScan &sh = *reinterpret_cast<BkScan *>(bsm);
  griddep_wait();
  griddep_launch();
  bk_scan_buckets(sh, hcnt, hrun, hkv);
  const uint32_t amin = ~__ldcg(tie), amax = __ldcg(tie + 1);
  const int lane = threadIdx.x & 31;
  for (int i0 = blockIdx.x * blockDim.x; i0 < m; i0 += gridDim.x * blockDim.x) {
    const int i = i0 + threadIdx.x;
    int b = -1;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (i < m) {
      v = __ldcg(reinterpret_cast<const uint4 *>(rec + i));
      if (v.x != kPadKey) b = bk_bucket(v.x, v.y, bp, amin, amax);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (b >= 0 && lane == leader) base = atomicAdd(cursor + b, (uint32_t)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (b >= 0) {
      const uint32_t slot = sh.cnt[b] + base + __popc(peers & ((1u << lane) - 1u));
      BkEntry e;
      e.key = ((unsigned long long)v.x << 32) | v.y;
      e.kvr = (v.z & 0x7FFFFFFFu) | (v.w & 0x80000000u);
      e.idx = (uint32_t)i;
      sorted[slot] = e;
    }
  }
}

// B3: exact positions, cumulative KV, running-before; lists
__global__ void __launch_bounds__(kB3Threads)
trail_bucket_rank_kernel(const Record *__restrict__ rec, int m, uint32_t *__restrict__ tie,
                         uint32_t *__restrict__ hcnt,
                         uint32_t *__restrict__ hrun, unsigned long long *__restrict__ hkv,
                         uint32_t *__restrict__ cursor, const BkEntry *__restrict__ sorted,
                         long long budget, int max_run, unsigned long long *__restrict__ gcnt,
                         uint2 *__restrict__ scratch, uint32_t *__restrict__ run_ids,
                         uint32_t *__restrict__ pre_ids, uint32_t *__restrict__ adm_ids,
                         int32_t *__restrict__ counts) {
  extern __shared__ __align__(16) uint8_t bsm[];
  BkScan &sh = *reinterpret_cast<BkScan *>(bsm);
  BkEntry *stage = reinterpret_cast<BkEntry *>(bsm + sizeof(BkScan));
  __shared__ int s_lo, s_hi, s_last;
  __shared__ uint32_t s_run, s_rcut;
  __shared__ unsigned long long s_tot;
  griddep_wait();
  griddep_launch();
  const int t = threadIdx.x;
  bk_scan_buckets(sh, hcnt, hrun, hkv);
  const int nv = (int)(sh.cnt[kB - 1] + __ldcg(hcnt + kB - 1));
  const int nf = (int)sh.cnt[kBH];                 // forced records = the first class
  const unsigned long long Sf = sh.kv[kBH];
  const int R_total = (int)(sh.run[kB - 1] + __ldcg(hrun + kB - 1));
  const int cap = max_run > 0 ? max_run : nv;
  const bool over = (long long)Sf > budget || nf > cap;
  // my positions in the bucket-sorted array, and the bucket range they span
  const int p0 = blockIdx.x * kB3Items, p1 = min(nv, p0 + kB3Items);
  if (t == 0) {
    s_run = 0u;
    s_rcut = 0u;
    int lo = 0, hi = 0;
    if (p0 < p1) {
      // buckets of the first and last of my positions (binary search over the prefix)
      int a = 0, z = kB - 1;
      while (a < z) { const int mid = (a + z + 1) >> 1; if ((int)sh.cnt[mid] <= p0) a = mid; else z = mid - 1; }
      lo = (int)sh.cnt[a];
      a = 0; z = kB - 1;
      while (a < z) { const int mid = (a + z + 1) >> 1; if ((int)sh.cnt[mid] <= p1 - 1) a = mid; else z = mid - 1; }
      hi = a + 1 < kB ? (int)sh.cnt[a + 1] : nv;
    }
    s_lo = lo;
    s_hi = hi;
  }
  __syncthreads();
  const int lo = s_lo, hi = s_hi;
  const bool staged = hi - lo <= kStageCap;
  if (staged)
    for (int q = lo + t; q < hi; q += kB3Threads) stage[q - lo] = sorted[q];
  __syncthreads();
  // kB3Tpi threads per record
  const int li = t / kB3Tpi, part = t % kB3Tpi;
  const int p = p0 + li;
  const bool have = p < p1;
  BkEntry me;
  int bs = 0, be = 0, b = 0;
  if (have) {
    me = staged ? stage[p - lo] : sorted[p];
    int a = 0, z = kB - 1;           // my bucket: the last prefix <= p
    while (a < z) { const int mid = (a + z + 1) >> 1; if ((int)sh.cnt[mid] <= p) a = mid; else z = mid - 1; }
    b = a;
    bs = (int)sh.cnt[b];
    be = b + 1 < kB ? (int)sh.cnt[b + 1] : nv;
  }
  uint32_t cnt = 0, rb = 0;
  unsigned long long cum = 0;
  if (have) {
    for (int q = bs + part; q < be; q += kB3Tpi) {
      const BkEntry o = staged ? stage[q - lo] : sorted[q];
      if (bk_less(o, me)) { ++cnt; cum += o.kvr & 0x7FFFFFFFu; rb += o.kvr >> 31; }
    }
  }
#pragma unroll
  for (int o = 1; o < kB3Tpi; o <<= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    rb += __shfl_xor_sync(0xffffffffu, rb, o);
    cum += __shfl_xor_sync(0xffffffffu, cum, o);
  }
  if (have && part == 0) {
    const int pos = (int)(sh.cnt[b] + cnt);
    const unsigned long long cum_incl = sh.kv[b] + cum + (me.kvr & 0x7FFFFFFFu);
    const uint32_t rbefore = sh.run[b] + rb;
    const bool forced = (me.key >> 63) == 0ull;
    const bool runn = (me.kvr >> 31) != 0u;
    const bool in_run = forced ? true : (!over && (long long)cum_incl <= budget && pos < cap);
    const uint32_t gidw = __ldg(&rec[me.idx].gid);
    const uint32_t gid = gidw & 0x7FFFFFFFu;
    if (in_run) {
      run_ids[pos] = gid;
      if (!runn) adm_ids[pos - (int)rbefore] = gid;
      atomicAdd(&s_run, 1u);
      if (runn) atomicAdd(&s_rcut, 1u);
    }
    scratch[pos] = make_uint2(gidw, rbefore);
  }
  __syncthreads();
  if (t == 0) {
    const unsigned long long inc = (1ull << 48) | ((unsigned long long)s_run << 24) | s_rcut;
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], %2;" : "=l"(old) : "l"(gcnt), "l"(inc) : "memory");
    const unsigned long long tot = old + inc;
    s_last = (int)(tot >> 48) == (int)gridDim.x ? 1 : 0;
    if (s_last) *gcnt = 0ull;
    s_tot = tot;
  }
  __syncthreads();
  if (!s_last) return;
  const int n_run = (int)((s_tot >> 24) & 0xFFFFFFull);
  const int R_cut = (int)(s_tot & 0xFFFFFFull);
  for (int q = n_run + t; q < nv; q += kB3Threads) {
    const uint2 v = __ldcg(scratch + q);
    if (v.x >> 31) pre_ids[(int)v.y - R_cut] = v.x & 0x7FFFFFFFu;
  }
  // re-arm the histogram and cursors for the next call (every CTA has finished with them)
  for (int q = t; q < kB; q += kB3Threads) { hcnt[q] = 0u; hrun[q] = 0u; hkv[q] = 0ull; cursor[q] = 0u; }
  if (t == 0) {
    tie[0] = 0u;
    tie[1] = 0u;
    counts[0] = n_run;
    counts[1] = R_total - R_cut;
    counts[2] = n_run - R_cut;
    counts[3] = over ? TRAIL_WARN_OVER_BUDGET : TRAIL_OK;
  }
}

// ------------------------------------------------------------------ host
size_t bucket_workspace_bytes(int m_max) {
  return (size_t)kB * (4 + 4 + 8 + 4) + 16 + 16 + (size_t)m_max * (sizeof(BkEntry) + sizeof(uint2));
}

cudaError_t select_bucket_prepare() {
  cudaError_t e = cudaFuncSetAttribute(trail_bucket_scatter_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BkScan));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(trail_bucket_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(sizeof(BkScan) + kStageCap * sizeof(BkEntry)));
}

cudaError_t launch_select_bucket(const Ctx &c, const Record *rec_in, Record *rec_out,
                                 const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                                 const uint8_t *running, int m, int64_t budget,
                                 int max_run, uint32_t *run, uint32_t *pre, uint32_t *adm,
                                 int32_t *counts, cudaStream_t s) {
  const Record *rec = rec_in ? rec_in : rec_out;
  if (!c.bk_ws) return cudaErrorInvalidValue;
  uint8_t *ws = reinterpret_cast<uint8_t *>(c.bk_ws);
  unsigned long long *hkv = reinterpret_cast<unsigned long long *>(ws);
  uint32_t *hcnt = reinterpret_cast<uint32_t *>(ws + (size_t)kB * 8);
  uint32_t *hrun = hcnt + kB;
  uint32_t *cursor = hrun + kB;
  unsigned long long *gcnt = reinterpret_cast<unsigned long long *>(cursor + kB);
  uint32_t *tie = reinterpret_cast<uint32_t *>(gcnt + 2);       // ~min, max arrival of the group
  BkEntry *sorted = reinterpret_cast<BkEntry *>(reinterpret_cast<uint8_t *>(gcnt) + 32);
  uint2 *scratch = reinterpret_cast<uint2 *>(sorted + c.bk_cap);
  const HeadConsts &hc = c.host_consts;
  BkParams bp;
  bp.m0 = hc.m[0];
  const float mk = hc.m[c.k - 1];
  bp.scale = mk > bp.m0 ? (float)kBH / (mk - bp.m0) : 0.f;
  float pl = hc.prior_L;
  uint32_t plb;
  memcpy(&plb, &pl, 4);
  bp.tie_bits = 0x80000000u | (plb & 0x7FFFFFFFu);
  {
    const float u = (pl - bp.m0) * bp.scale;
    bp.ustar = (u >= 0.f) ? (u < (float)kBH ? (int)u : kBH - 1) : 0;
  }
  const int g1 = std::max(1, std::min(2 * c.num_sms, (m + 255) / 256));
  cudaError_t e = launch_k(trail_bucket_prep_kernel, dim3(g1), dim3(256), 0, s, rec_in, rec_out,
                           ids, arrival, kv, running, (const SlotMeta *)c.meta,
                           (const HeadConsts *)c.consts, c.cfg.max_slots, c.cfg.id_base,
                           c.dev_err, m, bp.tie_bits, tie);
  if (e != cudaSuccess) return e;
  e = launch_k(trail_bucket_hist_kernel, dim3(g1), dim3(256), 0, s, rec, m, bp,
               (const uint32_t *)tie, hcnt, hrun, hkv);
  if (e != cudaSuccess) return e;
  const int g2 = std::max(1, std::min(c.num_sms, (m + kB3Threads - 1) / kB3Threads));
  e = launch_k(trail_bucket_scatter_kernel, dim3(g2), dim3(kB3Threads), sizeof(BkScan), s, rec, m,
               bp, (const uint32_t *)tie, (const uint32_t *)hcnt, (const uint32_t *)hrun,
               (const unsigned long long *)hkv, cursor, sorted);
  if (e != cudaSuccess) return e;
  const int g3 = std::max(1, (m + kB3Items - 1) / kB3Items);
  return launch_k(trail_bucket_rank_kernel, dim3(g3), dim3(kB3Threads),
                  sizeof(BkScan) + kStageCap * sizeof(BkEntry), s, rec, m, tie, hcnt, hrun, hkv,
                  cursor, (const BkEntry *)sorted, (long long)budget, max_run, gcnt, scratch, run,
                  pre, adm, counts);
}

}  // namespace trail
