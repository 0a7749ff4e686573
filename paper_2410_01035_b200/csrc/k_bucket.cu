// K4 (row a6) for large record counts (multi-rank all-gathers, configs 3-5): a sample sort
// in four PDL-chained kernels over the 16-byte records (row a4/a5).
//
// Same contract as every selection kernel: order = (keybits << 32 | arrival, input position)
// ascending — forced first (rank -inf), then shortest predicted remaining length
// (P:171), FCFS ties, then input position (D-18) — run set = all forced + the
// longest prefix of the rest within the KV budget and run cap (strict prefix D-15, overflow
// D-16).  (key, input position) pairs are unique, so the order is a strict total order.
//
// Bucket boundaries come from the data, not from the key range: the keys cluster — every
// never-observed request is keyed E_pi[L] exactly (D-24), thousands of them in a burst of
// arrivals, and posteriors that have collapsed onto one bin put their L at that bin's middle
// to within ~1e-6 — so equal-width L buckets leave a few buckets with thousands of records
// and an O(b^2) in-bucket ranking (measured: 49 us of a 65 us selection at configs[3] with
// L buckets; 4.7 ms for an 81 920-record unseen burst).
//   B0  1024 samples of (composite key, input position) on a jittered stride are ranked by
//       counting (32 samples per CTA, one per lane, each warp against a 32-key slice of the
//       staged sample set, partial counts summed in shared memory); sample of rank r becomes
//       splitter r - 1, so the 1023 splitters cut the records into 1024 buckets of about
//       m / 1024 whatever the key distribution (a tie cluster is split by arrival like any
//       other run of keys).  On the local path B0 also builds every record (row a4).
//   B1  bucket of each record = binary search over the splitters (shared memory); histogram
//       of (count, KV, running) per bucket in shared memory, added to the global histogram
//       one bucket per thread; forced totals
//   B2  scatter of the records into bucket order (prefix of the counts, atomic cursors; the
//       bucket ids B1 found are reused)
//   B3  each record counts the records of its own bucket ordered before it (the bucket range
//       is staged in shared memory; 8 threads per record), adds the bucket prefixes
//       -> position, cumulative KV, running-before, and the lists follow as in k_rank.cu
//       (one packed acq_rel atomic; the last CTA writes the preempt list and re-arms).
// Cost is O(m log m + sum over buckets of size^2 / 8) with bucket sizes ~ m / 1024.
#include <algorithm>

#include "sm100_ptx.cuh"
#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int kB = 1024;                // buckets (= samples: every sample but the smallest
constexpr int kS = kB;                  //  is a splitter)
constexpr int kB0Threads = 1024;
constexpr int kB1Threads = 1024;
constexpr int kB3Threads = 1024;
constexpr int kB3Tpi = 4;               // threads per record in B3 (256 records per CTA)
constexpr int kB3Items = kB3Threads / kB3Tpi;
constexpr int kStageCap = 4096;         // bucket entries staged in shared memory (64 KB)
// per-CTA phase traces (trail_trace_*, diagnostics): trace rows of B3, B0, B1, B2
constexpr int kTrB3 = 2048, kTrB0 = 3072, kTrB1 = 3136, kTrB2 = 3584;

struct BkEntry {                        // bucket-sorted record (16 B)
  unsigned long long key;               // keybits << 32 | arrival
  uint32_t kvr;                         // kv | running << 31  (kv_blocks >= 0 fits 31 bits)
  uint32_t idx;                         // input position (final tie-break, D-18)
};

struct __align__(16) BkKey {            // splitter / sample: (composite key, input position)
  unsigned long long key;
  uint32_t idx, pad;
};

__device__ __forceinline__ bool bk_lt(unsigned long long ka, uint32_t ia, unsigned long long kb,
                                      uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__device__ __forceinline__ bool bk_less(const BkEntry &a, const BkEntry &b) {
  return bk_lt(a.key, a.idx, b.key, b.idx);
}

__device__ __forceinline__ unsigned long long rec_key(uint32_t keybits, uint32_t arrival) {
  return keybits == kPadKey ? ~0ull : (((unsigned long long)keybits << 32) | arrival);
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

// sample j of kS: a jittered stride over the input positions
__device__ __forceinline__ int bk_sample_pos(int j, int m) {
  const long long lo = (long long)j * m / kS, hi = (long long)(j + 1) * m / kS;
  const uint32_t h = (uint32_t)j * 2654435761u;
  return (int)(lo + (hi > lo ? (long long)(h % (uint32_t)(hi - lo)) : 0));
}
}  // namespace

// B0: records (local path) + sample ranking -> splitters
__global__ void __launch_bounds__(kB0Threads)
trail_bucket_sample_kernel(const Record *__restrict__ rec, Record *__restrict__ rec_out,
                           const uint32_t *__restrict__ ids, const uint32_t *__restrict__ arrival,
                           const int32_t *__restrict__ kvin, const uint8_t *__restrict__ running,
                           const SlotMeta *__restrict__ meta, const HeadConsts *__restrict__ cst,
                           int max_slots, uint32_t id_base, uint32_t *__restrict__ err, int m,
                           BkKey *__restrict__ spl, uint64_t *__restrict__ trace) {
  __shared__ BkKey smp[kS];                                   // 32 KB
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint64_t *tr = trace ? trace + 16 * (kTrB0 + (int64_t)blockIdx.x) : nullptr;   // diagnostics
  if (tr && t == 0) tr[0] = ptx::gtimer();
  griddep_wait();     // records from the pack kernel / the all-gather, or the slot state
  griddep_launch();
  if (tr && t == 0) tr[1] = ptx::gtimer();
  // local path: every record, grid-stride (row a4, the record build of trail_schedule_pack)
  if (!rec)
    for (int i = blockIdx.x * kB0Threads + t; i < m; i += gridDim.x * kB0Threads)
      rec_out[i] = build_record(__ldg(ids + i), __ldg(arrival + i), __ldg(kvin + i),
                                __ldg(running + i) != 0, meta, cst, max_slots, id_base, err);
  // the kS sample keys (built from the inputs on the local path: no dependency on other CTAs)
  for (int j = t; j < kS; j += kB0Threads) {
    const int i = bk_sample_pos(j, m);
    uint32_t kb, ar;
    if (rec) {
      const uint2 v = __ldg(reinterpret_cast<const uint2 *>(rec + i));
      kb = v.x;
      ar = v.y;
    } else {
      const Record r = build_record(__ldg(ids + i), __ldg(arrival + i), __ldg(kvin + i),
                                    __ldg(running + i) != 0, meta, cst, max_slots, id_base, err);
      kb = r.keybits;
      ar = r.arrival;
    }
    BkKey k;
    k.key = rec_key(kb, ar);
    k.idx = (uint32_t)i;
    k.pad = 0u;
    smp[j] = k;
  }
  __syncthreads();
  if (tr && t == 0) tr[2] = ptx::gtimer();
  // ranks of this CTA's 32 samples (lane l of every warp: sample 32c + l) by counting, warp w
  // against the key slice [32w, 32w + 32) (broadcast reads), partial counts added in shared
  // memory; rank r >= 1 makes the sample splitter r - 1
  __shared__ uint32_t s_rank[32];
  if (t < 32) s_rank[t] = 0u;
  __syncthreads();
  for (int j0 = blockIdx.x * 32; j0 < kS; j0 += gridDim.x * 32) {
    const BkKey me = smp[j0 + lane];
    uint32_t cnt = 0;
#pragma unroll 8
    for (int q = 32 * warp; q < 32 * warp + 32; ++q) {
      const BkKey o = smp[q];
      cnt += bk_lt(o.key, o.idx, me.key, me.idx) ? 1u : 0u;
    }
    atomicAdd(&s_rank[lane], cnt);
    __syncthreads();
    if (t < 32) {
      const uint32_t r = s_rank[t];
      if (r > 0) spl[r - 1] = smp[j0 + t];
      s_rank[t] = 0u;
    }
    __syncthreads();
  }
  if (tr && t == 0) tr[3] = ptx::gtimer();
}

// B1: per-bucket totals (+ forced count / KV): a shared-memory histogram per CTA, added to the
// global one bucket per thread (the warp-aggregated global atomics it replaces serialised on
// match_any groups: 8 us at configs[3])
__global__ void __launch_bounds__(kB1Threads)
trail_bucket_hist_kernel(const Record *__restrict__ rec, int m, const BkKey *__restrict__ spl_g,
                         uint32_t *__restrict__ hcnt, uint32_t *__restrict__ hrun,
                         unsigned long long *__restrict__ hkv,
                         unsigned long long *__restrict__ forced_tot,
                         uint16_t *__restrict__ bkid, uint64_t *__restrict__ trace) {
  // splitters as separate key / index arrays: the search's (divergent) loads are 8 + 4 bytes
  __shared__ unsigned long long spl_k[kB];
  __shared__ uint32_t spl_i[kB];
  // KV per bucket as two 32-bit halves (native shared-memory atomics; a 64-bit shared atomic
  // add is a CAS loop on this part)
  __shared__ uint32_t h_cnt[kB], h_run[kB], h_klo[kB], h_khi[kB];
  uint64_t *tr = trace ? trace + 16 * (kTrB1 + (int64_t)blockIdx.x) : nullptr;   // diagnostics
  if (tr && threadIdx.x == 0) tr[0] = ptx::gtimer();
  for (int q = threadIdx.x; q < kB; q += kB1Threads) {
    h_cnt[q] = 0u; h_run[q] = 0u; h_klo[q] = 0u; h_khi[q] = 0u;
  }
  griddep_wait();     // splitters (and local records) from B0
  griddep_launch();
  if (tr && threadIdx.x == 0) tr[1] = ptx::gtimer();
  for (int q = threadIdx.x; q < kB - 1; q += kB1Threads) {
    const BkKey sp = spl_g[q];
    spl_k[q] = sp.key;
    spl_i[q] = sp.idx;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int i0 = blockIdx.x * kB1Threads; i0 < m; i0 += gridDim.x * kB1Threads) {
    const int i = i0 + threadIdx.x;
    uint32_t kvv = 0, frc = 0;
    if (i < m) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(rec + i));
      int b = -1;
      if (v.x != kPadKey) {
        {   // bucket = number of splitters <= (key, i)
          const unsigned long long key = rec_key(v.x, v.y);
          int lo = 0, hi = kB - 1;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const unsigned long long sk = spl_k[mid];
            if (sk < key || (sk == key && spl_i[mid] <= (uint32_t)i)) lo = mid + 1;
            else hi = mid;
          }
          b = lo;
        }
        kvv = v.z;
        frc = (v.x >> 31) == 0u ? 1u : 0u;
        atomicAdd(&h_cnt[b], 1u);
        if (v.w >> 31) atomicAdd(&h_run[b], 1u);
        atomicAdd(&h_klo[b], kvv & 0xFFFFu);
        if (kvv >> 16) atomicAdd(&h_khi[b], kvv >> 16);
      }
      bkid[i] = (uint16_t)(b < 0 ? 0xFFFF : b);   // reused by B2 (no second search)
    }
    // forced totals: count in the high 24 bits, KV in the low 40 (both far below the caps)
    const uint32_t fc = __reduce_add_sync(0xffffffffu, frc);
    const uint32_t flo = __reduce_add_sync(0xffffffffu, frc ? (kvv & 0xFFFFu) : 0u);
    const uint32_t fhi = __reduce_add_sync(0xffffffffu, frc ? (kvv >> 16) : 0u);
    if (lane == 0 && fc)
      atomicAdd(forced_tot, ((unsigned long long)fc << 40) + ((unsigned long long)fhi << 16) + flo);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kB; q += kB1Threads)
    if (h_cnt[q]) {
      atomicAdd(hcnt + q, h_cnt[q]);
      if (h_run[q]) atomicAdd(hrun + q, h_run[q]);
      atomicAdd(hkv + q, ((unsigned long long)h_khi[q] << 16) + h_klo[q]);
    }
  if (tr && threadIdx.x == 0) tr[2] = ptx::gtimer();
}

// B2: scatter into bucket order
__global__ void __launch_bounds__(kB3Threads)
trail_bucket_scatter_kernel(const Record *__restrict__ rec, int m,
                            const uint16_t *__restrict__ bkid,
                            const uint32_t *__restrict__ hcnt, const uint32_t *__restrict__ hrun,
                            const unsigned long long *__restrict__ hkv,
                            uint32_t *__restrict__ cursor, BkEntry *__restrict__ sorted,
                            uint64_t *__restrict__ trace) {
  extern __shared__ __align__(16) uint8_t bsm[];
  BkScan &sh = *reinterpret_cast<BkScan *>(bsm);
  uint64_t *tr = trace ? trace + 16 * (kTrB2 + (int64_t)blockIdx.x) : nullptr;   // diagnostics
  if (tr && threadIdx.x == 0) tr[0] = ptx::gtimer();
  griddep_wait();
  griddep_launch();
  if (tr && threadIdx.x == 0) tr[1] = ptx::gtimer();
  bk_scan_buckets(sh, hcnt, hrun, hkv);       // (synchronises)
  if (tr && threadIdx.x == 0) tr[2] = ptx::gtimer();
  const int lane = threadIdx.x & 31;
  for (int i0 = blockIdx.x * blockDim.x; i0 < m; i0 += gridDim.x * blockDim.x) {
    const int i = i0 + threadIdx.x;
    int b = -1;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (i < m) {
      v = __ldcg(reinterpret_cast<const uint4 *>(rec + i));
      const uint16_t bb = __ldcg(bkid + i);
      b = bb == 0xFFFF ? -1 : (int)bb;
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
  if (tr && threadIdx.x == 0) tr[3] = ptx::gtimer();
}

// B3: exact positions, cumulative KV, running-before; lists
__global__ void __launch_bounds__(kB3Threads)
trail_bucket_rank_kernel(const Record *__restrict__ rec, int m, uint32_t *__restrict__ hcnt,
                         uint32_t *__restrict__ hrun, unsigned long long *__restrict__ hkv,
                         unsigned long long *__restrict__ forced_tot,
                         uint32_t *__restrict__ cursor, const BkEntry *__restrict__ sorted,
                         long long budget, int max_run, unsigned long long *__restrict__ gcnt,
                         uint2 *__restrict__ scratch, uint32_t *__restrict__ run_ids,
                         uint32_t *__restrict__ pre_ids, uint32_t *__restrict__ adm_ids,
                         int32_t *__restrict__ counts, uint64_t *__restrict__ trace) {
  extern __shared__ __align__(16) uint8_t bsm[];
  BkScan &sh = *reinterpret_cast<BkScan *>(bsm);
  BkEntry *stage = reinterpret_cast<BkEntry *>(bsm + sizeof(BkScan));
  __shared__ int s_lo, s_hi, s_last;
  __shared__ uint32_t s_run, s_rcut;
  __shared__ unsigned long long s_tot;
  uint64_t *tr = trace ? trace + 16 * (kTrB3 + (int64_t)blockIdx.x) : nullptr;   // diagnostics
  if (tr && threadIdx.x == 0) tr[0] = ptx::gtimer();
  griddep_wait();
  griddep_launch();
  const int t = threadIdx.x;
  if (tr && t == 0) tr[1] = ptx::gtimer();
  bk_scan_buckets(sh, hcnt, hrun, hkv);
  if (tr && t == 0) tr[2] = ptx::gtimer();
  const int nv = (int)(sh.cnt[kB - 1] + __ldcg(hcnt + kB - 1));
  const unsigned long long ft = __ldcg(forced_tot);
  const int nf = (int)(ft >> 40);
  const unsigned long long Sf = ft & ((1ull << 40) - 1);
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
  if (tr && t == 0) tr[3] = ptx::gtimer();
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
  if (tr && t == 0) tr[4] = ptx::gtimer();
  if (t == 0) {
    const unsigned long long inc = (1ull << 48) | ((unsigned long long)s_run << 24) | s_rcut;
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(gcnt), "l"(inc) : "memory");
    const unsigned long long tot = old + inc;
    s_last = (int)(tot >> 48) == (int)gridDim.x ? 1 : 0;
    if (s_last) *gcnt = 0ull;
    s_tot = tot;
  }
  __syncthreads();
  if (tr && t == 0) { tr[5] = ptx::gtimer(); tr[14] = (uint64_t)s_last; }
  if (!s_last) return;
  const int n_run = (int)((s_tot >> 24) & 0xFFFFFFull);
  const int R_cut = (int)(s_tot & 0xFFFFFFull);
  // positions past the cut: 8 independent loads per thread in flight per round (a plain
  // load -> store loop is one L2 round trip per 1024 records)
  for (int q0 = n_run; q0 < nv; q0 += 8 * kB3Threads) {
    uint2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = q0 + u * kB3Threads + t;
      v[u] = q < nv ? __ldcg(scratch + q) : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (v[u].x >> 31) pre_ids[(int)v[u].y - R_cut] = v[u].x & 0x7FFFFFFFu;
  }
  // re-arm the histogram and cursors for the next call (every CTA has finished with them)
  for (int q = t; q < kB; q += kB3Threads) { hcnt[q] = 0u; hrun[q] = 0u; hkv[q] = 0ull; cursor[q] = 0u; }
  if (t == 0) {
    *forced_tot = 0ull;
    counts[0] = n_run;
    counts[1] = R_total - R_cut;
    counts[2] = n_run - R_cut;
    counts[3] = over ? TRAIL_WARN_OVER_BUDGET : TRAIL_OK;
  }
  if (tr && t == 0) tr[6] = ptx::gtimer();
}

// ------------------------------------------------------------------ host
size_t bucket_workspace_bytes(int m_max) {
  return (size_t)kB * (4 + 4 + 8 + 4) + 16 + 16 + (size_t)kB * sizeof(BkKey) +
         (size_t)m_max * (sizeof(BkEntry) + sizeof(uint2) + sizeof(uint16_t)) + 16;
}

cudaError_t select_bucket_prepare() {
  cudaError_t e = cudaFuncSetAttribute(trail_bucket_scatter_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(BkScan));
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
  if (!c.bk_ws || m < kS) return cudaErrorInvalidValue;
  uint8_t *ws = reinterpret_cast<uint8_t *>(c.bk_ws);
  unsigned long long *hkv = reinterpret_cast<unsigned long long *>(ws);
  uint32_t *hcnt = reinterpret_cast<uint32_t *>(ws + (size_t)kB * 8);
  uint32_t *hrun = hcnt + kB;
  uint32_t *cursor = hrun + kB;
  unsigned long long *gcnt = reinterpret_cast<unsigned long long *>(cursor + kB);
  unsigned long long *forced_tot = gcnt + 2;
  BkKey *spl = reinterpret_cast<BkKey *>(forced_tot + 2);
  BkEntry *sorted = reinterpret_cast<BkEntry *>(spl + kB);
  uint2 *scratch = reinterpret_cast<uint2 *>(sorted + c.bk_cap);
  uint16_t *bkid = reinterpret_cast<uint16_t *>(scratch + c.bk_cap);
  // B0: enough CTAs to build the records (local path) and a warp per sample
  const int g0 = std::max(kS / 32, rec_in ? 0 : std::min(c.num_sms, (m + kB0Threads - 1) / kB0Threads));
  cudaError_t e = launch_k(trail_bucket_sample_kernel, dim3(g0), dim3(kB0Threads), 0, s, rec_in,
                           rec_out, ids, arrival, kv, running, (const SlotMeta *)c.meta,
                           (const HeadConsts *)c.consts, c.cfg.max_slots, c.cfg.id_base,
                           c.dev_err, m, spl, (c.trace && kTrB0 + g0 <= c.trace_cap) ? c.trace : nullptr);
  if (e != cudaSuccess) return e;
  const int g1 = std::max(1, std::min(c.num_sms, (m + kB1Threads - 1) / kB1Threads));
  e = launch_k(trail_bucket_hist_kernel, dim3(g1), dim3(kB1Threads), 0, s, rec, m, (const BkKey *)spl,
               hcnt, hrun, hkv, forced_tot, bkid,
               (c.trace && kTrB1 + g1 <= c.trace_cap && g1 <= kTrB2 - kTrB1) ? c.trace : nullptr);
  if (e != cudaSuccess) return e;
  const int g2 = std::max(1, std::min(c.num_sms, (m + kB3Threads - 1) / kB3Threads));
  e = launch_k(trail_bucket_scatter_kernel, dim3(g2), dim3(kB3Threads), sizeof(BkScan), s, rec, m,
               (const uint16_t *)bkid, (const uint32_t *)hcnt, (const uint32_t *)hrun,
               (const unsigned long long *)hkv, cursor, sorted,
               (c.trace && kTrB2 + g2 <= c.trace_cap) ? c.trace : nullptr);
  if (e != cudaSuccess) return e;
  const int g3 = std::max(1, (m + kB3Items - 1) / kB3Items);
  return launch_k(trail_bucket_rank_kernel, dim3(g3), dim3(kB3Threads),
                  sizeof(BkScan) + kStageCap * sizeof(BkEntry), s, rec, m, hcnt, hrun, hkv,
                  forced_tot, cursor, (const BkEntry *)sorted, (long long)budget, max_run, gcnt,
                  scratch, run, pre, adm, counts,
                  (c.trace && g3 <= kTrB0 - kTrB3) ? c.trace : nullptr);
}

}  // namespace trail
