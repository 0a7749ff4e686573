// K4 — selection (row a6) with a single-CTA LSD radix sort (up to 16384 records), the
// record build of K5 (row a4) fused in for the local (one-rank) selection.
//
// Same contract as trail_select_kernel (k_select.cu): sort the 64-bit composite
// (keybits << 32 | arrival_seq) ascending — forced first (rank -inf), then the
// shortest predicted remaining length, ties FCFS, then input
// position (the sort is stable) — and take every forced record plus the longest prefix of
// the rest within the KV budget and run cap (D-15, D-16).
//
// Radix sort, 8-bit digits, least significant first; digits that are constant over all
// valid records are skipped (block OR/AND of the keys), so a step with a few thousand
// arrivals and keys in [25.6, 486.4] takes ~6 passes.  Per pass each warp ranks its items
// with __match_any_sync (rank within the warp = popcount of lower peers + a per-warp digit
// counter), one block scan over (digit, warp) counters gives the scatter offsets, and the
// keys are scattered to shared memory and re-read.  Items are held warp-striped
// (element i = warp*32E + e*32 + lane) so that ranks follow input order: stable.
#include <algorithm>

#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int kBins = 257;          // 256 digits + one bucket for empty slots (sorted last)
constexpr int kHistLd = 257;        // per-warp histogram row (odd stride: no bank conflicts)

__device__ __forceinline__ Record rx_load_rec(const Record *p) {
  const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(p));
  Record r;
  r.keybits = v.x; r.arrival = v.y; r.kv = v.z; r.gid = v.w;
  return r;
}

// exclusive block scan of an int and an int64 (one value per thread) + totals
template <int T>
struct RxScan {
  long long v[T / 32];
  int a[T / 32];
  long long tv;
  int ta;
};

template <int T>
__device__ __forceinline__ void rx_scan(RxScan<T> &sh, long long v, int a, long long &ev, int &ea) {
  constexpr int W = T / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long iv = v;
  int ia = a;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long tv = __shfl_up_sync(0xffffffffu, iv, o);
    const int ta = __shfl_up_sync(0xffffffffu, ia, o);
    if (lane >= o) { iv += tv; ia += ta; }
  }
  if (lane == 31) { sh.v[w] = iv; sh.a[w] = ia; }
  __syncthreads();
  if (w == 0) {
    long long wv = lane < W ? sh.v[lane] : 0;
    int wa = lane < W ? sh.a[lane] : 0;
    const long long wv0 = wv;
    const int wa0 = wa;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long tv = __shfl_up_sync(0xffffffffu, wv, o);
      const int ta = __shfl_up_sync(0xffffffffu, wa, o);
      if (lane >= o) { wv += tv; wa += ta; }
    }
    if (lane < W) { sh.v[lane] = wv - wv0; sh.a[lane] = wa - wa0; }
    if (lane == W - 1) { sh.tv = wv; sh.ta = wa; }
  }
  __syncthreads();
  ev = sh.v[w] + iv - v;
  ea = sh.a[w] + ia - a;
  __syncthreads();
}

__device__ __forceinline__ Record rx_make_record(int i, const uint32_t *ids, const uint32_t *arrival,
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

template <int T, int E>
__global__ void __launch_bounds__(T, 1)
trail_select_radix_kernel(const Record *rec_in, Record *rec_out, const uint32_t *__restrict__ ids,
                          const uint32_t *__restrict__ arrival, const int32_t *__restrict__ kv,
                          const uint8_t *__restrict__ running, const SlotMeta *__restrict__ meta,
                          const HeadConsts *__restrict__ cst, int max_slots, uint32_t id_base,
                          uint32_t *__restrict__ err, int n, long long budget, int max_run,
                          uint32_t *__restrict__ run_ids, uint32_t *__restrict__ pre_ids,
                          uint32_t *__restrict__ adm_ids, int32_t *__restrict__ counts) {
  constexpr int W = T / 32;
  constexpr int N = T * E;
  constexpr int G = T / 256 > 0 ? T / 256 : 1;   // threads per digit in the offset scan
  constexpr int WPG = W / G;                      // warps per scan thread
  extern __shared__ __align__(16) uint8_t smem[];
  unsigned long long *skey = reinterpret_cast<unsigned long long *>(smem);     // [N]
  uint32_t *sidx = reinterpret_cast<uint32_t *>(smem + (size_t)N * 8);          // [N]
  uint32_t *hist = reinterpret_cast<uint32_t *>(smem + (size_t)N * 12);         // [W][kHistLd]
  // (kv | forced<<31, gid) by input position, when they fit next to the keys
  constexpr bool kSmemRec = N <= 8192;
  uint32_t *skv = hist + W * kHistLd;                                            // [N]
  uint32_t *sgid = skv + N;                                                      // [N]
  __shared__ RxScan<T> sh;
  __shared__ unsigned long long s_or, s_and;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const Record *rec = rec_in ? rec_in : rec_out;
  griddep_wait();     // slot state from the predict kernels
  griddep_launch();

  // 1. load / build records (blocked: record t*E + e), compact the valid ones
  uint32_t valid_mask = 0u;
  unsigned long long kk_e[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = t * E + e;
    kk_e[e] = ~0ull;
    if (i < n) {
      Record r;
      if (rec_in) {
        r = rec_in[i];
      } else {
        r = rx_make_record(i, ids, arrival, kv, running, meta, cst, max_slots, id_base, err);
        rec_out[i] = r;
      }
      if (r.keybits != kPadKey) {
        valid_mask |= 1u << e;
        kk_e[e] = ((unsigned long long)r.keybits << 32) | r.arrival;
        if (kSmemRec) {
          skv[i] = (r.kv & 0x7FFFFFFFu) | ((r.keybits >> 31) == 0u ? 0x80000000u : 0u);
          sgid[i] = r.gid;
        }
      }
    }
  }
  if (t == 0) { s_or = 0ull; s_and = ~0ull; }
  long long d0;
  int voff;
  rx_scan<T>(sh, 0, __popc(valid_mask), d0, voff);   // (also orders rec_out writes)
  const int nv = sh.ta;
  // compacted valid items -> shared memory (position order = input order)
  unsigned long long my_or = 0ull, my_and = ~0ull;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (valid_mask & (1u << e)) {
      const unsigned long long kk = kk_e[e];
      skey[voff] = kk;
      sidx[voff] = (uint32_t)(t * E + e);
      my_or |= kk;
      my_and &= kk;
      ++voff;
    }
  }
  // OR / AND over valid keys (digits constant over all of them are skipped)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    my_or |= __shfl_xor_sync(0xffffffffu, my_or, o);
    my_and &= __shfl_xor_sync(0xffffffffu, my_and, o);
  }
  __syncthreads();
  if (lane == 0) {
    atomicOr(&s_or, my_or);
    atomicAnd(&s_and, my_and);
  }
  __syncthreads();
  const unsigned long long vary = nv > 0 ? (s_or ^ s_and) : 0ull;

  // 2. warp-striped items: element i = w*32E + e*32 + lane
  unsigned long long key[E];
  uint32_t idx[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = w * 32 * E + e * 32 + lane;
    key[e] = i < nv ? skey[i] : ~0ull;
    idx[e] = i < nv ? sidx[i] : 0xFFFFFFFFu;
  }
  uint32_t *whist = hist + w * kHistLd;
  for (int pass = 0; pass < 8; ++pass) {
    const int sh8 = pass * 8;
    if (((vary >> sh8) & 0xFFull) == 0ull) continue;     // uniform across the block
    __syncthreads();                                     // skey/sidx reads of the last pass done
    for (int b = lane; b < kBins; b += 32) whist[b] = 0u;
    __syncwarp();
    int local[E];
    int dig[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = w * 32 * E + e * 32 + lane;
      const int d = i < nv ? (int)((key[e] >> sh8) & 0xFFull) : 256;
      dig[e] = d;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int leader = __ffs(peers) - 1;
      const int below = __popc(peers & ((1u << lane) - 1u));
      uint32_t base = 0;
      if (lane == leader) {
        base = whist[d];
        whist[d] = base + (uint32_t)__popc(peers);
      }
      base = __shfl_sync(0xffffffffu, base, leader);
      local[e] = (int)base + below;
      __syncwarp();
    }
    __syncthreads();
    // offsets: digit-major, warp-minor exclusive scan over the W x 257 counters
    {
      int run_sum = 0;
      uint32_t tmp[WPG > 0 ? WPG : 1];
      int dd = -1, g = 0;
      if (t < 256 * G) {
        dd = t / G;
        g = t % G;
#pragma unroll
        for (int q = 0; q < WPG; ++q) {
          tmp[q] = hist[(g * WPG + q) * kHistLd + dd];
          run_sum += (int)tmp[q];
        }
      }
      // the empty-slot bucket (256) goes last: handled by thread T-1 below
      long long dz;
      int ex;
      rx_scan<T>(sh, 0, run_sum, dz, ex);
      if (dd >= 0) {
#pragma unroll
        for (int q = 0; q < WPG; ++q) {
          hist[(g * WPG + q) * kHistLd + dd] = (uint32_t)ex;
          ex += (int)tmp[q];
        }
      }
      __syncthreads();
      if (t == 0) {   // bucket 256 (empty slots): after every real digit, in warp order
        int off = sh.ta;
        for (int q = 0; q < W; ++q) {
          const uint32_t c = hist[q * kHistLd + 256];
          hist[q * kHistLd + 256] = (uint32_t)off;
          off += (int)c;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int pos = (int)whist[dig[e]] + local[e];
      skey[pos] = key[e];
      sidx[pos] = idx[e];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = w * 32 * E + e * 32 + lane;
      key[e] = skey[i];
      idx[e] = sidx[i];
    }
  }
  // make the sorted order visible in shared memory (also when no pass ran)
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = w * 32 * E + e * 32 + lane;
    skey[i] = key[e];
    sidx[i] = idx[e];
  }
  __syncthreads();

  // 3. blocked arrangement over the sorted valid items: positions [t*E, t*E+E); records
  //    are re-read (L1/L2) instead of being held in registers
  uint32_t kvv[E], gidv[E];
  long long kv_t = 0, fkv_t = 0;
  int f_t = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int p = t * E + e;
    kvv[e] = 0u;
    gidv[e] = 0u;
    if (p < nv) {
      bool forced;
      if (kSmemRec) {
        const uint32_t src = sidx[p];
        kvv[e] = skv[src] & 0x7FFFFFFFu;
        forced = (skv[src] >> 31) != 0u;
        gidv[e] = sgid[src];
      } else {
        const Record r = rx_load_rec(rec + sidx[p]);
        kvv[e] = r.kv;
        gidv[e] = r.gid;
        forced = (r.keybits >> 31) == 0u;
      }
      kv_t += kvv[e];
      if (forced) { fkv_t += kvv[e]; ++f_t; }
    }
  }
  long long kv_off;
  int f_off;
  rx_scan<T>(sh, fkv_t, f_t, kv_off, f_off);
  const long long Sf = sh.tv;
  const int nf = sh.ta;
  rx_scan<T>(sh, kv_t, 0, kv_off, f_off);
  int fit_t = 0;
  {
    long long cum = kv_off;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int p = t * E + e;
      if (p < nv) {
        cum += kvv[e];
        fit_t += cum <= budget ? 1 : 0;      // non-decreasing: the fitting set is a prefix
      }
    }
  }
  rx_scan<T>(sh, 0, fit_t, kv_off, f_off);
  const int n_fit = sh.ta;
  const int cap = max_run > 0 ? max_run : nv;
  int n_run, status;
  if (Sf > budget || nf > cap) { n_run = nf; status = TRAIL_WARN_OVER_BUDGET; }
  else { n_run = min(n_fit, cap); status = TRAIL_OK; }

  // 4. lists in priority order
  int pre_t = 0, adm_t = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int p = t * E + e;
    if (p < nv) {
      const bool runn = (gidv[e] >> 31) != 0u;
      if (p < n_run) {
        run_ids[p] = gidv[e] & 0x7FFFFFFFu;
        adm_t += runn ? 0 : 1;
      } else {
        pre_t += runn ? 1 : 0;
      }
    }
  }
  long long pre_off64;
  int pre_off;
  rx_scan<T>(sh, (long long)pre_t, adm_t, pre_off64, pre_off);
  const int n_pre = (int)sh.tv, n_adm = sh.ta;
  int po = (int)pre_off64, ao = pre_off;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int p = t * E + e;
    if (p < nv) {
      const bool runn = (gidv[e] >> 31) != 0u;
      const uint32_t gid = gidv[e] & 0x7FFFFFFFu;
      if (p < n_run) {
        if (!runn) adm_ids[ao++] = gid;
      } else if (runn) {
        pre_ids[po++] = gid;
      }
    }
  }
  if (t == 0) {
    counts[0] = n_run;
    counts[1] = n_pre;
    counts[2] = n_adm;
    counts[3] = status;
  }
}

// ------------------------------------------------------------------ host
template <int T, int E>
static size_t rx_smem() {
  const size_t N = (size_t)T * E;
  return N * 12 + (size_t)(T / 32) * kHistLd * 4 + (N <= 8192 ? N * 8 : 0);
}

cudaError_t select_radix_prepare() {
  cudaError_t e = cudaSuccess;
#define RX_ATTR(TT, EE)                                                                      \
  if (e == cudaSuccess)                                                                      \
    e = cudaFuncSetAttribute(trail_select_radix_kernel<TT, EE>,                               \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rx_smem<TT, EE>());
  RX_ATTR(256, 1) RX_ATTR(256, 2) RX_ATTR(256, 4) RX_ATTR(256, 8)
  RX_ATTR(1024, 4) RX_ATTR(1024, 8) RX_ATTR(1024, 16)
#undef RX_ATTR
  return e;
}

int select_radix_capacity() { return 1024 * 16; }

cudaError_t launch_select_radix(const Ctx &c, const Record *rec_in, Record *rec_out,
                                const uint32_t *ids, const uint32_t *arrival, const int32_t *kv,
                                const uint8_t *running, int n, int64_t budget, int max_run,
                                uint32_t *run, uint32_t *pre, uint32_t *adm, int32_t *counts,
                                cudaStream_t s) {
#define RX_LAUNCH(TT, EE)                                                                     \
  return launch_k(trail_select_radix_kernel<TT, EE>, dim3(1), dim3(TT), rx_smem<TT, EE>(), s,  \
                  rec_in, rec_out, ids, arrival, kv, running, (const SlotMeta *)c.meta,        \
                  (const HeadConsts *)c.consts, c.cfg.max_slots, c.cfg.id_base, c.dev_err, n,  \
                  (long long)budget, max_run, run, pre, adm, counts)
  if (n <= 256) RX_LAUNCH(256, 1);
  if (n <= 512) RX_LAUNCH(256, 2);
  if (n <= 1024) RX_LAUNCH(256, 4);
  if (n <= 2048) RX_LAUNCH(256, 8);
  if (n <= 4096) RX_LAUNCH(1024, 4);
  if (n <= 8192) RX_LAUNCH(1024, 8);
  if (n <= 16384) RX_LAUNCH(1024, 16);
#undef RX_LAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace trail
