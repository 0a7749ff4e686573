// K4 — selection, with the record build of row a4 fused on the local
// path: ONE thread-block cluster sorts the records by their composite key and cuts the
// KV-budget prefix, writing the run / preempt / admit lists.
//
// Order (the oracle's `select` contract): composite key (keybits << 32 | arrival_seq)
// ascending — forced first (keybits bit 31 clear: rank -inf), then the shortest
// predicted remaining length, ties FCFS (D-18), then input position.
// Run set = every forced record + the longest prefix of the rest whose cumulative KV stays
// within the budget and whose size stays within the run cap (strict prefix, D-15; fill = 1:
// first-fit); a forced set over the limits gives run = forced,
// TRAIL_WARN_OVER_BUDGET (D-16).  preempt = running records outside the run set, admit =
// waiting records inside it, both in priority order.
//
// Layout: C CTAs (one cluster, C = 1..16), 512 threads each; CTA r owns input range
// [r P, r P + P) and, after the sort, sorted positions [r P, r P + P).  Elements are 16 bytes
// (u64 composite key, u32 input index): (key, index) pairs are unique, so comparisons are
// strict and the order is the oracle's stable order.  Padding records (keybits 0xFFFFFFFF,
// multi-rank blocks) get key ~0 and sort after every valid record.
//  phase 0  build (local path: caller inputs + slot state, row a4) or load the records of the
//           input range; count the valid ones.
//  sort     bitonic network over the CTA's pow2-padded elements in shared memory: stages whose
//           partner distance is below 64 stay inside a warp (__syncwarp only); the few
//           longer ones use __syncthreads (c2: 15 of 55 stages).
//  rank     (C > 1) cluster barrier; every element's global position = its local position +
//           the number of elements that precede it in each other CTA's sorted chunk, found by
//           binary searches over DSMEM run side by side for all chunks (one round of
//           independent loads per step); the input index is stored at that position in the
//           owning CTA (st.shared::cluster); cluster barrier.
//  final    records of the sorted items (16 B, L2), cluster-wide exclusive scan of KV and
//           running counts, forced totals -> over-budget flag and the cut; run / admit lists;
//           one more exchange of the run-set size places the preempt list.
// No global atomics, no second kernel: the selection is one launch of one cluster.
#include "sm100_ptx.cuh"
#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int kCsT = 512;
constexpr int kCsW = kCsT / 32;
constexpr int kCsCap = 8192;               // elements per CTA
constexpr int kCsMaxK = kCsCap / kCsT;     // 16 items per thread
constexpr int kCsMaxC = 16;                // CTAs per cluster (non-portable above 8)

struct CsXchg {                            // per-CTA values read by the cluster (DSMEM)
  long long kv, fkv, inkv;
  int nvalid, run, forced, inrun, rcut, rx, wx, pad_;
};

struct CsShared {
  CsXchg x;                                // published values
  CsXchg peer[kCsMaxC];                    // copies of every CTA's published values
  long long sv[kCsW];
  int sc[kCsW], sd[kCsW];
  long long tot_a;
  int tot_b, tot_c;
  // first-fit continuation (fill = 1): per-iteration candidate, double-buffered by parity
  int ffmin;
  int ffpos[2];
  uint32_t ffkv[2];
  int pffpos[kCsMaxC];
  uint32_t pffkv[kCsMaxC];
};

struct __align__(16) CsElem {
  unsigned long long key;
  uint32_t idx, pad;
};

__device__ __forceinline__ bool cs_less(const CsElem &a, const CsElem &b) {
  return a.key < b.key || (a.key == b.key && a.idx < b.idx);
}

__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_cluster_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ CsElem ld_cluster_elem(uint32_t addr) {
  CsElem e;
  asm volatile("ld.shared::cluster.v2.u64 {%0, %1}, [%2];"
               : "=l"(e.key), "=l"(*reinterpret_cast<unsigned long long *>(&e.idx))
               : "r"(addr)
               : "memory");
  return e;
}
__device__ __forceinline__ void ld_cluster_bytes(void *dst, uint32_t addr, int words) {
  uint32_t *d = reinterpret_cast<uint32_t *>(dst);
  for (int i = 0; i < words; ++i) d[i] = ld_cluster_u32(addr + 4 * i);
}

// every thread of every CTA of the cluster (a CTA barrier when C == 1)
__device__ __forceinline__ void cs_sync(int C) {
  if (C > 1) {
    ptx::cluster_arrive();
    ptx::cluster_wait();
  } else {
    __syncthreads();
  }
}

// exclusive block scan of (a, b, c) over the CTA's threads; totals in s.tot_*
__device__ __forceinline__ void cs_scan(CsShared &s, long long &a, int &b, int &c) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long ia = a;
  int ib = b, ic = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long ta = __shfl_up_sync(0xffffffffu, ia, o);
    const int tb = __shfl_up_sync(0xffffffffu, ib, o);
    const int tc = __shfl_up_sync(0xffffffffu, ic, o);
    if (lane >= o) { ia += ta; ib += tb; ic += tc; }
  }
  if (lane == 31) { s.sv[w] = ia; s.sc[w] = ib; s.sd[w] = ic; }
  __syncthreads();
  if (w == 0) {
    long long va = lane < kCsW ? s.sv[lane] : 0;
    int vb = lane < kCsW ? s.sc[lane] : 0, vc = lane < kCsW ? s.sd[lane] : 0;
    const long long a0 = va;
    const int b0 = vb, c0 = vc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long ta = __shfl_up_sync(0xffffffffu, va, o);
      const int tb = __shfl_up_sync(0xffffffffu, vb, o);
      const int tc = __shfl_up_sync(0xffffffffu, vc, o);
      if (lane >= o) { va += ta; vb += tb; vc += tc; }
    }
    if (lane < kCsW) { s.sv[lane] = va - a0; s.sc[lane] = vb - b0; s.sd[lane] = vc - c0; }
    if (lane == kCsW - 1) { s.tot_a = va; s.tot_b = vb; s.tot_c = vc; }
  }
  __syncthreads();
  a = s.sv[w] + ia - a;
  b = s.sc[w] + ib - b;
  c = s.sd[w] + ic - c;
  __syncthreads();
}

// threads < C copy every CTA's published values into s.peer
__device__ __forceinline__ void cs_gather_peers(CsShared &s, int C, int r) {
  const int t = threadIdx.x;
  if (t < C) {
    if (t == r) s.peer[t] = s.x;
    else ld_cluster_bytes(&s.peer[t], ptx::mapa(ptx::smem_u32(&s.x), t), sizeof(CsXchg) / 4);
  }
  __syncthreads();
}
}  // namespace

__global__ void __launch_bounds__(kCsT, 1)
trail_select_cluster_kernel(const Record *__restrict__ rec_in, Record *__restrict__ rec_out,
                            const uint32_t *__restrict__ ids, const uint32_t *__restrict__ arrival,
                            const int32_t *__restrict__ kv, const uint8_t *__restrict__ running,
                            const SlotMeta *__restrict__ meta, const HeadConsts *__restrict__ cst,
                            int max_slots, uint32_t id_base, uint32_t *__restrict__ err, int m,
                            int P, int NP, long long budget, int max_run, int fill,
                            uint32_t *__restrict__ run_ids,
                            uint32_t *__restrict__ pre_ids, uint32_t *__restrict__ adm_ids,
                            int32_t *__restrict__ counts) {
  extern __shared__ __align__(16) unsigned char cs_dyn[];
  __shared__ CsShared s;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int C = 1, r = 0;
  {
    uint32_t nc;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nc));
    C = (int)nc;
    r = C > 1 ? (int)ptx::cluster_rank() : 0;
  }
  CsElem *el = reinterpret_cast<CsElem *>(cs_dyn);                 // [NP] sorted in place
  uint32_t *sidx = reinterpret_cast<uint32_t *>(el + NP);          // [P] input index by position

  // ---- phase 0: this CTA's input range [i0, i1), K0 contiguous items per thread
  const int i0 = min(m, r * P), i1 = min(m, i0 + P);
  const int n_in = i1 - i0;
  const int K0 = (P + kCsT - 1) / kCsT;
  const int q0 = tid * K0;
  uint32_t in_slot[kCsMaxK], in_arr[kCsMaxK], in_run = 0u;
  int32_t in_kv[kCsMaxK];
  if (!rec_in) {          // caller inputs (not produced by the predict kernels): before the wait
#pragma unroll
    for (int k = 0; k < kCsMaxK; ++k) {
      const int i = i0 + q0 + k;
      if (k < K0 && i < i1) {
        in_slot[k] = __ldg(ids + i);
        in_arr[k] = __ldg(arrival + i);
        in_kv[k] = __ldg(kv + i);
        in_run |= __ldg(running + i) ? (1u << k) : 0u;
      }
    }
  }
  griddep_wait();         // slot state (local path) / packed records
  griddep_launch();
  int nval = 0;
#pragma unroll
  for (int k = 0; k < kCsMaxK; ++k) {
    const int q = q0 + k;
    if (k >= K0 || q >= NP) continue;
    const int i = i0 + q;
    CsElem e;
    e.key = ~0ull;
    e.idx = 0xFFFFFFFFu;                         // sentinel past the range: sorts last
    e.pad = 0u;
    if (i < i1) {
      Record rc;
      if (rec_in) {
        rc = rec_in[i];
      } else {            // row a4: key = L_t (E_pi[L] if never observed), forced flag
        const uint32_t slot = in_slot[k];
        const bool run = (in_run >> k) & 1u;
        int32_t kvb = in_kv[k];
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
          key = INFINITY;   // sorts last among non-forced; never displaces a valid request
        }
        uint32_t kb;
        if (isfinite(key) && key >= 0.f) {
          kb = __float_as_uint(key) & 0x7FFFFFFFu;
        } else {
          if (slot < (uint32_t)max_slots) atomicOr(err, TRAIL_DEV_NONFIN);
          kb = 0x7F800000u;
        }
        rc.keybits = (forced ? 0u : 0x80000000u) | kb;
        rc.arrival = in_arr[k];
        rc.kv = (uint32_t)kvb;
        rc.gid = ((id_base + slot) & 0x7FFFFFFFu) | (run ? 0x80000000u : 0u);
        if (rec_out) rec_out[i] = rc;
      }
      e.idx = (uint32_t)i;
      if (rc.keybits != kPadKey) {
        e.key = ((unsigned long long)rc.keybits << 32) | rc.arrival;
        ++nval;
      }
    }
    el[q] = e;
  }
  // sentinels beyond the threads' item ranges (NP may exceed K0 * threads' coverage of P)
  for (int q = kCsT * K0 + tid; q < NP; q += kCsT) {
    CsElem e;
    e.key = ~0ull;
    e.idx = 0xFFFFFFFFu;
    e.pad = 0u;
    el[q] = e;
  }
  for (int o = 16; o > 0; o >>= 1) nval += __shfl_xor_sync(0xffffffffu, nval, o);
  if (lane == 0) s.sc[w] = nval;
  __syncthreads();

  // ---- local bitonic sort of el[0, NP): pair p -> (i, i + j), i = 2p - (p & (j - 1)); a
  // warp's 32 pairs of one round cover 64 consecutive elements, so stages with j <= 32 only
  // need __syncwarp
  {
    const int npairs = NP >> 1;
    for (int kk = 2; kk <= NP; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int p = tid; p < npairs; p += kCsT) {
          const int i = 2 * p - (p & (j - 1));
          const CsElem a = el[i], b = el[i + j];
          const bool up = (i & kk) == 0;
          if (cs_less(b, a) == up) {
            el[i] = b;
            el[i + j] = a;
          }
        }
        if (j > 32) __syncthreads();
        else __syncwarp();
      }
      if (kk >= 64) __syncthreads();   // the next merge's first stage crosses warps
    }
    __syncthreads();
  }
  if (tid == 0) {
    int t = 0;
    for (int q = 0; q < kCsW; ++q) t += s.sc[q];
    s.x.nvalid = t;
  }

  // ---- global positions (C > 1): local position + elements of each other chunk ahead of it
  if (C > 1) {
    cs_sync(C);                                     // (1) chunks sorted, valid counts published
    const uint32_t el_base = ptx::smem_u32(el);
    const uint32_t idx_base = ptx::smem_u32(sidx);
    int lg = 0;
    while ((1 << lg) < P) ++lg;
    for (int q = tid; q < n_in; q += kCsT) {
      const CsElem me = el[q];
      int pos[kCsMaxC];
      uint32_t base[kCsMaxC];
      int len[kCsMaxC];
#pragma unroll
      for (int c = 0; c < kCsMaxC; ++c) {
        pos[c] = 0;
        len[c] = 0;
        base[c] = 0u;
        if (c < C && c != r) {
          len[c] = max(0, min(P, m - c * P));
          base[c] = ptx::mapa(el_base, (uint32_t)c);
        }
      }
      // branchless lower bound, all chunks side by side: pos_c = #elements of chunk c < me
      for (int st = 1 << lg; st > 0; st >>= 1) {
        CsElem probe[kCsMaxC];
#pragma unroll
        for (int c = 0; c < kCsMaxC; ++c)
          if (pos[c] + st <= len[c])
            probe[c] = ld_cluster_elem(base[c] + (uint32_t)(pos[c] + st - 1) * 16u);
#pragma unroll
        for (int c = 0; c < kCsMaxC; ++c)
          if (pos[c] + st <= len[c] && cs_less(probe[c], me)) pos[c] += st;
      }
      // elements ahead of me: q in my own chunk + pos_c in every other chunk
      int g = q;
#pragma unroll
      for (int c = 0; c < kCsMaxC; ++c) g += pos[c];
      const int tc = g / P, off = g - tc * P;
      if (tc == r) sidx[off] = me.idx;
      else st_cluster_u32(ptx::mapa(idx_base + (uint32_t)off * 4u, (uint32_t)tc), me.idx);
    }
    cs_sync(C);                                     // (2) every position has its index
  } else {
    for (int q = tid; q < n_in; q += kCsT) sidx[q] = el[q].idx;
    __syncthreads();
  }
  cs_gather_peers(s, C, r);
  int nv = 0;
  for (int c = 0; c < C; ++c) nv += s.peer[c].nvalid;
  // this CTA's valid sorted positions: [r P, r P + n_c)
  const int n_c = max(0, min(n_in, nv - r * P));
  const int Pv = P;
  const int K = (P + kCsT - 1) / kCsT;

  // ---- final: cut and lists.  Thread t holds sorted local positions [t Kf, t Kf + Kf).
  const Record *src = rec_in ? rec_in : rec_out;
  const int Kf = K;
  const int f0 = tid * Kf;
  uint32_t fgid[kCsMaxK];
  uint32_t fkv[kCsMaxK];
  uint32_t fflag[kCsMaxK];   // bit0 forced, bit1 running, bit2 have
  long long kv_t = 0, fkv_t = 0;
  int run_t = 0, forced_t = 0;
#pragma unroll
  for (int k = 0; k < kCsMaxK; ++k) {
    fflag[k] = 0u;
    const int q = f0 + k;
    if (k < Kf && q < n_c) {
      const Record rc = src[sidx[q]];
      const bool forced = (rc.keybits >> 31) == 0u;
      const bool runn = (rc.gid >> 31) != 0u;
      fgid[k] = rc.gid & 0x7FFFFFFFu;
      fkv[k] = rc.kv;
      fflag[k] = (forced ? 1u : 0u) | (runn ? 2u : 0u) | 4u;
      kv_t += rc.kv;
      run_t += runn ? 1 : 0;
      forced_t += forced ? 1 : 0;
      fkv_t += forced ? (long long)rc.kv : 0;
    }
  }
  long long kv_x = kv_t;
  int run_x = run_t, forced_x = forced_t;
  cs_scan(s, kv_x, run_x, forced_x);
  const long long cta_kv = s.tot_a;
  const int cta_run = s.tot_b, cta_forced = s.tot_c;
  // forced KV of the CTA: forced items are the sorted prefix, so a block reduction suffices
  long long fkv_red = fkv_t;
  for (int o = 16; o > 0; o >>= 1) fkv_red += __shfl_xor_sync(0xffffffffu, fkv_red, o);
  if (lane == 0) s.sv[w] = fkv_red;
  __syncthreads();
  if (tid == 0) {
    long long t = 0;
    for (int q = 0; q < kCsW; ++q) t += s.sv[q];
    s.x.kv = cta_kv;
    s.x.fkv = t;
    s.x.run = cta_run;
    s.x.forced = cta_forced;
  }
  cs_sync(C);                                       // (5) KV / running / forced totals
  cs_gather_peers(s, C, r);
  long long kv_pre = 0, Sf = 0;
  int run_pre = 0, nf = 0, R_total = 0;
  for (int c = 0; c < C; ++c) {
    if (c < r) { kv_pre += s.peer[c].kv; run_pre += s.peer[c].run; }
    Sf += s.peer[c].fkv;
    nf += s.peer[c].forced;
    R_total += s.peer[c].run;
  }
  const int cap = max_run > 0 ? max_run : nv;
  const bool over = Sf > budget || nf > cap;
  long long cum = kv_pre + kv_x;
  int rb = run_pre + run_x;
  int in_t = 0, rcut_t = 0;
  long long inkv_t = 0;
  uint32_t inrun_mask = 0u;
#pragma unroll
  for (int k = 0; k < kCsMaxK; ++k) {
    if (fflag[k] & 4u) {
      const int pos = r * Pv + f0 + k;
      cum += fkv[k];
      const bool forced = fflag[k] & 1u, runn = (fflag[k] & 2u) != 0u;
      const bool in_run = forced || (!over && cum <= budget && pos < cap);
      if (in_run) {
        inrun_mask |= 1u << k;
        run_ids[pos] = fgid[k];
        if (!runn) adm_ids[pos - rb] = fgid[k];
        ++in_t;
        rcut_t += runn ? 1 : 0;
        inkv_t += fkv[k];
      }
      rb += runn ? 1 : 0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    in_t += __shfl_xor_sync(0xffffffffu, in_t, o);
    rcut_t += __shfl_xor_sync(0xffffffffu, rcut_t, o);
    inkv_t += __shfl_xor_sync(0xffffffffu, inkv_t, o);
  }
  if (lane == 0) { s.sc[w] = in_t; s.sd[w] = rcut_t; s.sv[w] = inkv_t; }
  __syncthreads();
  if (tid == 0) {
    int a = 0, b = 0;
    long long kvs = 0;
    for (int q = 0; q < kCsW; ++q) { a += s.sc[q]; b += s.sd[q]; kvs += s.sv[q]; }
    s.x.inrun = a;
    s.x.rcut = b;
    s.x.inkv = kvs;
  }
  cs_sync(C);                                       // (6) run-set size and its running count
  cs_gather_peers(s, C, r);
  int n_run = 0, R_cut = 0;
  long long run_kv = 0;
  for (int c = 0; c < C; ++c) {
    n_run += s.peer[c].inrun;
    R_cut += s.peer[c].rcut;
    run_kv += s.peer[c].inkv;
  }

  // ---- first-fit continuation (fill = 1, the D-15 alternative): past the
  // strict prefix, repeatedly take the earliest request that still fits the remaining budget
  // (and run cap).  The remaining budget only shrinks, so a request passed over never fits
  // later and "earliest fitting" reproduces the sequential first-fit walk.  One cluster-wide
  // min per taken request; taken requests get fflag bit 3.
  int n_ext = 0;
  if (fill && !over) {
    long long rem = budget - run_kv;
    int capl = cap - n_run;
    for (int it = 0; capl > 0; ++it) {
      const int par = it & 1;
      if (tid == 0) s.ffmin = 0x7FFFFFFF;
      __syncthreads();
      int myp = 0x7FFFFFFF;
#pragma unroll
      for (int k = kCsMaxK - 1; k >= 0; --k) {
        const int pos = r * Pv + f0 + k;
        if ((fflag[k] & 4u) && !(fflag[k] & 8u) && pos >= n_run && (long long)fkv[k] <= rem)
          myp = pos;
      }
      for (int o = 16; o > 0; o >>= 1) myp = min(myp, __shfl_xor_sync(0xffffffffu, myp, o));
      if (lane == 0 && myp != 0x7FFFFFFF) atomicMin(&s.ffmin, myp);
      __syncthreads();
      const int cmin = s.ffmin;
      if (tid == 0 && cmin == 0x7FFFFFFF) { s.ffpos[par] = cmin; s.ffkv[par] = 0u; }
#pragma unroll
      for (int k = 0; k < kCsMaxK; ++k)
        if ((fflag[k] & 4u) && r * Pv + f0 + k == cmin) {
          s.ffpos[par] = cmin;
          s.ffkv[par] = fkv[k];
        }
      cs_sync(C);                                   // (7.it) every CTA's earliest candidate
      if (tid < C) {
        if (tid == r) {
          s.pffpos[tid] = s.ffpos[par];
          s.pffkv[tid] = s.ffkv[par];
        } else {
          s.pffpos[tid] = (int)ld_cluster_u32(ptx::mapa(ptx::smem_u32(&s.ffpos[par]), tid));
          s.pffkv[tid] = ld_cluster_u32(ptx::mapa(ptx::smem_u32(&s.ffkv[par]), tid));
        }
      }
      __syncthreads();
      int gpos = 0x7FFFFFFF;
      uint32_t gkv = 0u;
      for (int c = 0; c < C; ++c)
        if (s.pffpos[c] < gpos) { gpos = s.pffpos[c]; gkv = s.pffkv[c]; }
      if (gpos == 0x7FFFFFFF) break;                // nothing else fits
#pragma unroll
      for (int k = 0; k < kCsMaxK; ++k)
        if ((fflag[k] & 4u) && r * Pv + f0 + k == gpos) fflag[k] |= 8u;
      rem -= gkv;
      --capl;
      ++n_ext;
    }
  }
  int rx_x = 0, wx_x = 0, RX = 0;
  if (n_ext > 0) {                                  // list positions of the extra requests
    int rx_t = 0, wx_t = 0;
#pragma unroll
    for (int k = 0; k < kCsMaxK; ++k)
      if (fflag[k] & 8u) {
        if (fflag[k] & 2u) ++rx_t;
        else ++wx_t;
      }
    long long dz = 0;
    rx_x = rx_t;
    wx_x = wx_t;
    cs_scan(s, dz, rx_x, wx_x);
    if (tid == 0) { s.x.rx = s.tot_b; s.x.wx = s.tot_c; }
    cs_sync(C);                                     // (8) extras per CTA
    cs_gather_peers(s, C, r);
    for (int c = 0; c < C; ++c) {
      if (c < r) { rx_x += s.peer[c].rx; wx_x += s.peer[c].wx; }
      RX += s.peer[c].rx;
    }
    int e_r = rx_x, e_w = wx_x;
#pragma unroll
    for (int k = 0; k < kCsMaxK; ++k)
      if (fflag[k] & 8u) {
        run_ids[n_run + e_r + e_w] = fgid[k];
        if (fflag[k] & 2u) {
          ++e_r;
        } else {
          adm_ids[(n_run - R_cut) + e_w] = fgid[k];
          ++e_w;
        }
      }
  }
  rb = run_pre + run_x;
  int rxb = rx_x;                                   // running extras before this item
#pragma unroll
  for (int k = 0; k < kCsMaxK; ++k) {
    if (fflag[k] & 4u) {
      const bool runn = (fflag[k] & 2u) != 0u;
      const bool ext = (fflag[k] & 8u) != 0u;
      if (runn && !ext && !(inrun_mask & (1u << k))) pre_ids[rb - R_cut - rxb] = fgid[k];
      rb += runn ? 1 : 0;
      rxb += (runn && ext) ? 1 : 0;
    }
  }
  if (r == 0 && tid == 0) {
    const int n_tot = n_run + n_ext;
    counts[0] = n_tot;
    counts[1] = R_total - R_cut - RX;
    counts[2] = n_tot - R_cut - RX;
    counts[3] = over ? TRAIL_WARN_OVER_BUDGET : TRAIL_OK;
  }
  if (C > 1) cs_sync(C);                            // peers may still read this CTA's values
}

// ------------------------------------------------------------------ host
namespace {
int g_cs_maxc = 0;   // largest cluster size that can be resident (queried once)
}

int select_cluster_capacity() { return (g_cs_maxc > 0 ? g_cs_maxc : 8) * kCsCap; }

cudaError_t select_cluster_prepare() {
  const size_t smem = (size_t)kCsCap * (sizeof(CsElem) + 4);
  cudaError_t e = cudaFuncSetAttribute(trail_select_cluster_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(trail_select_cluster_kernel,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  if (g_cs_maxc == 0) {
    g_cs_maxc = 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kCsMaxC);
    cfg.blockDim = dim3(kCsT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = kCsMaxC;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, trail_select_cluster_kernel, &cfg) ==
            cudaSuccess && nclusters > 0)
      g_cs_maxc = kCsMaxC;
    cudaGetLastError();
  }
  return cudaSuccess;
}

// cluster size: the smallest power of two giving <= `target` items per CTA (env
// TRAIL_CSORT_ITEMS overrides the target; default 2048)
static int cs_cluster_size(int m) {
  static int target = -1;
  if (target < 0) {
    const char *e = getenv("TRAIL_CSORT_ITEMS");
    target = e ? atoi(e) : 2048;
    if (target < 256) target = 256;
    if (target > kCsCap) target = kCsCap;
  }
  const int maxc = g_cs_maxc > 0 ? g_cs_maxc : 8;
  int C = 1;
  while (C < maxc && (m + C - 1) / C > target) C <<= 1;
  while (C < maxc && (m + C - 1) / C > kCsCap) C <<= 1;
  return C;
}

cudaError_t launch_select_cluster(const Ctx &c, const Record *rec_in, Record *rec_out,
                                  const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                                  const uint8_t *running, int m, int64_t budget, int max_run,
                                  uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                                  cudaStream_t s) {
  if (m > select_cluster_capacity()) return cudaErrorInvalidValue;
  const int C = cs_cluster_size(m);
  const int P = std::max(1, (m + C - 1) / C);
  int NP = 2;
  while (NP < P) NP <<= 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kCsT);
  cfg.dynamicSmemBytes = (size_t)NP * sizeof(CsElem) + (size_t)P * 4;
  cfg.stream = s;
  cudaLaunchAttribute a[2];
  int na = 0;
  if (C > 1) {
    a[na].id = cudaLaunchAttributeClusterDimension;
    a[na].val.clusterDim.x = C;
    a[na].val.clusterDim.y = 1;
    a[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    a[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = a;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, trail_select_cluster_kernel, rec_in, rec_out, ids, arrival, kv,
                            running, (const SlotMeta *)c.meta, (const HeadConsts *)c.consts,
                            c.cfg.max_slots, c.cfg.id_base, c.dev_err, m, P, NP,
                            (long long)budget, max_run, c.fill_mode, run, pre, adm, counts);
}

}  // namespace trail
