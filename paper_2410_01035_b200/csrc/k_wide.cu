// K2d — the wide predict kernel for large batches (rows a2 + a3): layer 1 on a CTA PAIR
// (tcgen05.mma.cta_group::2, M = 256) with the whole hidden width H = 512 in TMEM, so
// every request's h, layer 2 and head stay inside its own CTA — no split-K, no cross-CTA
// reduction, no arrival counters, any number of waves.
//
//   P:201  h = ReLU(W1 x + b1) (d -> 512), z = W2 h + b2 (512 -> k)
//   P:204/P:219-226  softmax, Bayesian refinement (log domain, D-22), L_t   (head_dev.cuh)
//
// Why: at configs[3] (16 384 x 8192) the split-K kernel K2c runs 512 tiles of 128 x 128 in
// four waves and reads X four times (once per column tile) — 363 µs, L2/HBM-bound.  Here the
// pair p owns requests [256p, 256p + 256): CTA r of the pair loads its 128 rows of X and the
// W1 rows {128r .. 128r+127} and {256 + 128r .. 256 + 128r + 127} (its halves of the two
// N = 256 MMAs) — 48 KB per 64-wide K block — and the even CTA issues two M = 256, N = 256,
// K = 16 MMAs per 16 columns of K for both.  X is read from HBM exactly once.
//   warp 0        : X producer (row gather shared with K2c, xgather.cuh) into the X ring
//                   (XS x 16 KB) — cta_group::2 loads completing on the LEADER's barrier
//   warp 2        : W1 producer (2 x 128 x 64 per K block) into the W1 ring (WS x 32 KB)
//   warp 1, even  : MMA issuer; tcgen05.commit multicast frees both rings' stages in both CTAs
//   warps 3-7     : stage b1, head constants and the slot state of the CTA's 128 rows
// Separate rings because the two operands behave differently (scripts/wide_probe.py,
// configs[3], L2 flushed): the MMAs alone take 136 us, + the L2-resident W1 loads 138 us,
// + the cold X rows from HBM 183 us with one shared 4 x 48 KB ring — X needs the deeper
// buffer (7 x 16 KB: 191 -> 179 us per launch).  Deeper or batched X requests (8 stages,
// 4 K blocks per request group) and L2 prefetch of the X rows ahead of the ring were
// measured slower.
//   all 8 warps   : epilogue — TMEM (lane = row) -> +b1, ReLU -> layer 2 on the tensor cores
//                   (3xTF32 pair MMA, M = 256, N = 16/32 bins, 16 chunks of 32 hidden units,
//                   4 A buffers) -> head, one lane per bin (head_dev.cuh)
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "head_dev.cuh"
#include "sm100_ptx.cuh"
#include "trail_internal.cuh"
#include "xgather.cuh"

namespace trail {

using namespace ptx;

namespace {
constexpr int WT = 256;
constexpr int WBM = 128;                       // rows per CTA (256 per pair)
constexpr int WBK = 64;
constexpr int WH = 512;                        // hidden width held in TMEM (fp32 columns)
constexpr int WA = WBM * WBK * 2;              // 16 KB: my 128 rows of X
constexpr int WBH = 128 * WBK * 2;             // 16 KB: my 128 rows of one N half of W1
constexpr int WS = 3;                          // W1 ring stages (2 x 16 KB each; L2-resident)

template <int KB>
struct WCfg {
  static constexpr int KBP = (KB + 3) & ~3;    // layer-2 bins padded to float4
  static constexpr int XS = KB <= 20 ? 7 : 6;  // X ring stages (16 KB each)
  static constexpr int PIPE = XS * WA + WS * 2 * WBH;
  static constexpr int BAR_OFF = PIPE;         // xfull, xempty, wfull, wempty, done, tmem slot
  static constexpr int B1_OFF = BAR_OFF + 256;
  static constexpr int SLOT_OFF = B1_OFF + WH * 4;
  static constexpr int META_OFF = SLOT_OFF + WBM * 4;
  static constexpr int LQ_OFF = META_OFF + WBM * 16;
  static constexpr int HC_OFF = LQ_OFF + WBM * KB * 4;
  static constexpr int SMEM_USED = HC_OFF + (int)sizeof(HeadSmem);
  static constexpr int SMEM_TOTAL = SMEM_USED + 1024;
  // after the mainloop the pipeline buffers hold W2 hi / lo (2 x 32 KB), the layer-2 A tiles
  // (2 x 32 KB) and z [128][KBP]
  static_assert(2 * 16 * 2048 + 4 * 32768 <= PIPE, "epilogue staging must fit");
  static_assert(8 * (2 * XS + 2 * WS + 1) + 8 <= 176, "barrier block");
  static_assert(SMEM_TOTAL <= 232448, "shared memory budget");
};
}  // namespace

template <int KB>
__global__ void __launch_bounds__(WT, 1)
trail_wide_predict_kernel(const __grid_constant__ CUtensorMap tmap_emb,
                          const __grid_constant__ CUtensorMap tmap_emb4,
                          const __grid_constant__ CUtensorMap tmap_emb32,
                          const __grid_constant__ CUtensorMap tmap_xs,
                          const __grid_constant__ CUtensorMap tmap_xs4,
                          const __grid_constant__ CUtensorMap tmap_xs32,
                          const __grid_constant__ CUtensorMap tmap_w,
                          const int32_t *__restrict__ off, int n, int kblocks,
                          const float *__restrict__ b1, const float *__restrict__ w2,
                          const float *__restrict__ b2, const __grid_constant__ HeadConsts cst,
                          const uint32_t *__restrict__ ids, const uint8_t *__restrict__ is_prefill,
                          const float *__restrict__ prior_override, int max_slots,
                          float *__restrict__ lq_state, SlotMeta *__restrict__ meta,
                          float *__restrict__ post, float *__restrict__ Lout,
                          uint32_t *__restrict__ err, int decode_only, int wflags,
                          uint64_t *__restrict__ trace) {
  using C = WCfg<KB>;
  constexpr int KBP = C::KBP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t s0 = smem_u32(smem);
  constexpr int XS = C::XS;
  const uint32_t xfull0 = s0 + C::BAR_OFF, xempty0 = xfull0 + 8 * XS;
  const uint32_t wfull0 = xempty0 + 8 * XS, wempty0 = wfull0 + 8 * WS, done = wempty0 + 8 * WS;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::BAR_OFF + 8 * (2 * XS + 2 * WS + 1));
  // wflags bits 8/9: diagnostics that skip the X / W1 loads (wrong results; probes only)
  const bool skip_x = (wflags & 0x100) != 0, skip_w = (wflags & 0x200) != 0;
  float *b1s = reinterpret_cast<float *>(smem + C::B1_OFF);
  uint32_t *s_slot = reinterpret_cast<uint32_t *>(smem + C::SLOT_OFF);
  SlotMeta *s_meta = reinterpret_cast<SlotMeta *>(smem + C::META_OFF);
  float *s_lq = reinterpret_cast<float *>(smem + C::LQ_OFF);
  HeadSmem &hs = *reinterpret_cast<HeadSmem *>(smem + C::HC_OFF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const uint32_t r = cluster_rank();
  uint64_t *tr = trace ? trace + 16 * (int64_t)blockIdx.x : nullptr;   // diagnostics (trail_trace_*)
  if (tr && tid == 0) tr[0] = gtimer();
  const int m0 = (int)(blockIdx.x >> 1) * 2 * WBM + (int)r * WBM;
  const int k = cst.k;

  if (tid == 0) {
    for (int i = 0; i < XS; ++i) {
      mbar_init(xfull0 + 8 * i, 1);
      mbar_init(xempty0 + 8 * i, 1);
    }
    for (int i = 0; i < WS; ++i) {
      mbar_init(wfull0 + 8 * i, 1);
      mbar_init(wempty0 + 8 * i, 1);
    }
    // layer-2 barriers (epilogue): afull[4] (4 producer warps x 2 CTAs), afree[4], zdone
    for (int i = 0; i < 4; ++i) {
      mbar_init(s0 + C::BAR_OFF + 176 + 8 * i, 8);
      mbar_init(s0 + C::BAR_OFF + 208 + 8 * i, 1);
    }
    mbar_init(s0 + C::BAR_OFF + 240, 1);
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_w)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_emb)) : "memory");
  }
  if (warp == 0) tmem_alloc_pair(smem_u32(tmem_slot), (uint32_t)WH);
  tc_fence_before();
  cluster_sync();                    // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_launch();
  if (tr && tid == 0) tr[1] = gtimer();

  if (warp == 0) {
    // ---- X producer (all lanes: the row gather of xgather.cuh) into the X ring.  X streams
    // from HBM once (cold rows), W1 from L2 (shared by every pair): measured alone, the MMAs
    // take 136 us at configs[3], + W1 loads 138, + X loads 183 — the X stream needs the
    // deeper buffer, so X and W1 have separate rings (XS x 16 KB, WS x 32 KB per CTA).
    const XPlan xp = xplan_make(off, n, m0, lane);
    const uint32_t lead_xfull0 = mapa(xfull0, 0u);
    const uint32_t x_tx = skip_x ? 0u : (uint32_t)(2 * WA);
    if (xp.tile_xs) {
      // decode/prefill split: this launch was promised decode-only tiles (trail_set_prefill_start)
      if (decode_only) {
        if (lane == 0) atomicOr(err, TRAIL_DEV_BAD_HINT);
      } else {
        griddep_wait();
      }
    }
    __syncwarp();
    for (int i = 0; i < kblocks; ++i) {
      const int st = i % XS;
      if (lane == 0) {
        if (i >= XS) mbar_wait(xempty0 + 8 * st, ((uint32_t)(i / XS) & 1u) ^ 1u);
        if (r == 0) mbar_expect_tx(xfull0 + 8 * st, x_tx);
      }
      __syncwarp();
      if (!skip_x)
        xplan_issue<true>(xp, lane, s0 + st * WA, lead_xfull0 + 8 * st, i * WBK, &tmap_emb,
                          &tmap_emb4, &tmap_emb32, &tmap_xs, &tmap_xs4, &tmap_xs32);
    }
  } else if (warp == 2) {
    // ---- W1 producer (the converged warp, one elected lane issues): my halves of the two
    // N = 256 column blocks into the W1 ring; W1 does not depend on an earlier kernel, so the
    // first stages overlap its tail (PDL)
    const uint32_t lead_wfull0 = mapa(wfull0, 0u);
    const uint32_t w_tx = skip_w ? 0u : (uint32_t)(4 * WBH);
    for (int i = 0; i < kblocks; ++i) {
      const int st = i % WS;
      if (i >= WS) mbar_wait(wempty0 + 8 * st, ((uint32_t)(i / WS) & 1u) ^ 1u);
      const uint32_t sb = s0 + XS * WA + st * 2 * WBH;
      if (elect_one()) {
        if (r == 0) mbar_expect_tx(wfull0 + 8 * st, w_tx);
        if (!skip_w) {
          tma_load_2d_pair(sb, &tmap_w, lead_wfull0 + 8 * st, i * WBK, (int)r * 128);
          tma_load_2d_pair(sb + WBH, &tmap_w, lead_wfull0 + 8 * st, i * WBK, 256 + (int)r * 128);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---- MMA issue (leader CTA): the whole warp walks the K loop (waits, descriptors: all
    // warp-uniform), one elected lane issues the MMAs and commits
    if (r == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(2 * WBM, 256);
      for (int i = 0; i < kblocks; ++i) {
        const int sx = i % XS, sw = i % WS;
        mbar_wait(xfull0 + 8 * sx, (uint32_t)(i / XS) & 1u);
        mbar_wait(wfull0 + 8 * sw, (uint32_t)(i / WS) & 1u);
        tc_fence_after();
        const uint64_t da = sw128_kmajor_desc(s0 + sx * WA);
        const uint32_t sb = s0 + XS * WA + sw * 2 * WBH;
        if (elect_one()) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint64_t db = sw128_kmajor_desc(sb + h * WBH);
#pragma unroll
            for (int kk = 0; kk < WBK / 16; ++kk)
              umma_bf16_pair(tmem + 256 * h, da + 2 * kk, db + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit_pair(xempty0 + 8 * sx);
          umma_commit_pair(wempty0 + 8 * sw);
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit_pair(done);
      __syncwarp();
    }
  } else {
    // warps 3-7: b1, head constants and this CTA's slot state (weights and state written by
    // kernels that completed before the pool kernel passed its own griddep_wait: PDL chain)
    const int t = tid - 96;
    for (int v = t; v < WH / 4; v += WT - 96)
      reinterpret_cast<float4 *>(b1s)[v] = __ldg(reinterpret_cast<const float4 *>(b1) + v);
    if (t < kMaxBins) {
      hs.m[t] = cst.m[t];
      hs.log_stay[t] = cst.log_stay[t];
      hs.log_move[t] = cst.log_move[t];
      hs.log_prior[t] = cst.log_prior[t];
      hs.thr[t] = cst.thr_tab[t];
    }
    if (t < WBM) {
      const int j = m0 + t;
      uint32_t sl = 0xFFFFFFFFu;
      if (j < n) {
        sl = __ldg(ids + j);
        const bool pref = __ldg(is_prefill + j) != 0;
        if (sl < (uint32_t)max_slots) {
          s_meta[t] = meta[sl];
#pragma unroll
          for (int b = 0; b < KB; ++b)
            if (b < k) s_lq[t * KB + b] = lq_state[(int64_t)sl * k + b];
          sl |= pref ? 0x80000000u : 0u;
        } else {
          sl = 0xFFFFFFFFu;
        }
      }
      s_slot[t] = sl;
    }
  }

  // ---- epilogue: the pipeline is idle once `done` completes (all MMAs of the pair retired)
  constexpr int NB = KB <= 16 ? 16 : 32;           // layer-2 MMA N (bins padded)
  constexpr int BH = NB / 2;                       // bins held by this CTA (B split of the pair)
  constexpr int W2PER = BH * WH / WT;              // W2 values per thread
  // this CTA's W2 rows into registers while the last MMAs run (L2 latency off the tail)
  float w2r[W2PER];
#pragma unroll
  for (int u = 0; u < W2PER; ++u) {
    const int v = tid + u * WT, bl = v / WH, x = v - bl * WH, bin = (int)r * BH + bl;
    w2r[u] = bin < k ? __ldg(w2 + (int64_t)bin * WH + x) : 0.f;
  }
  mbar_wait(done, 0);
  __syncwarp();
  tc_fence_after();
  if (tr && tid == 0) tr[2] = gtimer();
  // ---- layer 2 on the tensor cores (3xTF32, exact hi/lo split): z[256 x NB] = h W2^T over the
  // pair (M = 256, N = NB bins padded, K = 512 hidden in 16 chunks of 32).  The FFMA version
  // (128 x 512 x 20 FMAs per CTA on the CUDA cores) cost ~18 us of the kernel (probe).
  //   W2 -> this CTA's NB/2 bins of every chunk, split into TF32 hi / fp32 lo, K-major SW128
  //   producers: warps w and w + 4 own TMEM lanes 32 (w & 3) ..; warps 0-3 build the even
  //   chunks, 4-7 the odd ones: h = ReLU(acc + b1) from TMEM -> hi / lo A tiles (4 buffers)
  //   MMA issue: warp 0 of the leader (converged, one elected lane), in chunk order, 3 MMAs
  //   per 8 columns of K
  //   (hi.hi + hi.lo + lo.hi); the accumulator takes TMEM columns [0, NB) once chunk 0 (those
  //   columns of h) has been read by every producer.
  constexpr int W2T = 2048;                        // bytes per chunk of B (hi or lo)
  constexpr int NA = 4;                            // A buffers (32 KB each: hi + lo)
  const uint32_t w2hi = s0, w2lo = s0 + 16 * W2T, abuf = s0 + 32 * W2T;
  const uint32_t ebar = s0 + C::BAR_OFF + 176;     // afull[NA] (8 arrivals), afree[NA], zdone
  const uint32_t afull0 = ebar, afree0 = ebar + 8 * NA, zdone = ebar + 16 * NA;
#pragma unroll
  for (int u = 0; u < W2PER; ++u) {
    const int v = tid + u * WT, bl = v / WH, x = v - bl * WH;
    const float val = w2r[u];
    const float hi = tf32_hi(val);
    const int kk = x & 31;
    const uint32_t off = (uint32_t)((x >> 5) * W2T + (bl >> 3) * 1024 + (bl & 7) * 128 +
                                    (((kk >> 2) ^ (bl & 7)) << 4) + (kk & 3) * 4);
    *reinterpret_cast<float *>(smem + off) = hi;
    *reinterpret_cast<float *>(smem + 16 * W2T + off) = val - hi;
  }
  fence_proxy_async_smem();
  __syncthreads();
  {
    constexpr uint32_t idesc2 = idesc_tf32_f32(2 * WBM, NB);
    auto issue = [&](int cc) {                     // leader CTA, warp 0 converged, one lane issues
      const int bf = cc % NA;
      mbar_wait(afull0 + 8 * bf, (uint32_t)(cc / NA) & 1u);
      tc_fence_after();
      const uint64_t ah = sw128_kmajor_desc(abuf + bf * 32768), al = sw128_kmajor_desc(abuf + bf * 32768 + 16384);
      const uint64_t bh = sw128_kmajor_desc(w2hi + cc * W2T), bl = sw128_kmajor_desc(w2lo + cc * W2T);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {           // +32 bytes along K per 8 fp32
          umma_tf32_pair(tmem, ah + 2 * kk, bh + 2 * kk, idesc2, (cc > 0 || kk > 0) ? 1u : 0u);
          umma_tf32_pair(tmem, ah + 2 * kk, bl + 2 * kk, idesc2, 1u);
          umma_tf32_pair(tmem, al + 2 * kk, bh + 2 * kk, idesc2, 1u);
        }
        umma_commit_pair(afree0 + 8 * bf);
      }
      __syncwarp();
    };
    const int g = warp & 3, par = warp >> 2, row = 32 * g + lane;
    const int rb = (row >> 3) * 1024 + (row & 7) * 128;
    for (int c = par; c < WH / 32; c += 2) {
      const int bf = c % NA;
      // TMEM -> registers and the split before waiting for the buffer (only the stores need it)
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(32 * g) << 16) + (uint32_t)(32 * c), v);
      float hh[32], hl[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const float h = fmaxf(__uint_as_float(v[q]) + b1s[32 * c + q], 0.f);
        hh[q] = tf32_hi(h);
        hl[q] = h - hh[q];
      }
      if (c >= NA) mbar_wait(afree0 + 8 * bf, (uint32_t)(c / NA - 1) & 1u);
      uint8_t *ahi = smem + 32 * W2T + bf * 32768, *alo = ahi + 16384;
#pragma unroll
      for (int q4 = 0; q4 < 8; ++q4) {
        const int off = rb + ((q4 ^ (row & 7)) << 4);
        *reinterpret_cast<float4 *>(ahi + off) =
            make_float4(hh[4 * q4], hh[4 * q4 + 1], hh[4 * q4 + 2], hh[4 * q4 + 3]);
        *reinterpret_cast<float4 *>(alo + off) =
            make_float4(hl[4 * q4], hl[4 * q4 + 1], hl[4 * q4 + 2], hl[4 * q4 + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa(afull0 + 8 * bf, 0u));
      __syncwarp();
      if (r == 0 && warp == 0)
        for (int cc = c > 0 ? c - 1 : 0; cc <= c; ++cc) issue(cc);
    }
    if (r == 0 && warp == 0) {
      issue(WH / 32 - 1);
      if (elect_one()) umma_commit_pair(zdone);
      __syncwarp();
    }
  }
  mbar_wait(zdone, 0);
  tc_fence_after();
  if (tr && tid == 0) tr[3] = gtimer();
  float *zs2 = reinterpret_cast<float *>(smem + 32 * W2T);   // [WBM][KBP] over A buffer 0
  if (warp < 4) {
    uint32_t v[32];
    tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16), v);
#pragma unroll
    for (int b = 0; b < KBP; ++b) zs2[(32 * warp + lane) * KBP + b] = __uint_as_float(v[b]);
  }
  __syncthreads();
  // ---- head (row a3): one thread per row, all k bins in registers (head_row)
  if (tid < WBM) {
    const int rr = tid, j = m0 + rr;
    if (j < n) {
      float z[KB];
#pragma unroll
      for (int b = 0; b < KB; ++b) z[b] = b < k ? __ldg(b2 + b) + zs2[rr * KBP + b] : 0.f;
      head_row<KB>(j, k, z, hs, cst.dyn_c, s_slot[rr], s_meta[rr], s_lq + rr * KB, prior_override,
                   lq_state, meta, post, Lout, err);
    }
  }
  if (tr && tid == 0) tr[4] = gtimer();
  tc_fence_before();
  cluster_sync();                    // both CTAs done with TMEM
  if (warp == 0) tmem_dealloc_pair(tmem, (uint32_t)WH);
  if (tr && tid == 0) tr[5] = gtimer();
}

// ------------------------------------------------------------------ host
static int wide_kb(int k) { return k <= 10 ? 10 : k <= 16 ? 16 : k <= 20 ? 20 : 32; }

bool wide_supported(const Ctx &c) {
  return c.dtype == TRAIL_BF16 && c.H == WH && c.k <= 32 && c.d % WBK == 0;
}

// AUTO uses the wide kernel from this many requests on (TRAIL_WIDE_MIN overrides; measured
// crossover against K2c)
int wide_min_n() {
  static const int v = [] {
    const char *e = getenv("TRAIL_WIDE_MIN");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? x : 4608;
  }();
  return v;
}

// TRAIL_WIDE_DIAG: 1 = skip the X loads, 2 = skip the W1 loads, 3 = both (timing probes of
// the MMA / load paths, scripts/wide_probe.py — wrong results)
static int wide_flags() {
  static const int v = [] {
    const char *g = getenv("TRAIL_WIDE_DIAG");
    return (g ? atoi(g) & 3 : 0) << 8;
  }();
  return v;
}

template <int KB>
static cudaError_t wide_attr() {
  return cudaFuncSetAttribute(trail_wide_predict_kernel<KB>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, WCfg<KB>::SMEM_TOTAL);
}

cudaError_t wide_prepare(Ctx &c) {
  if (!wide_supported(c)) return cudaSuccess;
  switch (wide_kb(c.k)) {
    case 10: return wide_attr<10>();
    case 16: return wide_attr<16>();
    case 20: return wide_attr<20>();
    default: return wide_attr<32>();
  }
}

cudaError_t launch_wide_predict(Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                                const uint32_t *ids, const uint8_t *is_prefill,
                                const float *prior_override, float *post, float *L,
                                cudaStream_t s, int decode_only) {
  if (!c.have_tmaps || !wide_supported(c)) return cudaErrorInvalidValue;
  if (!ensure_emb_tmaps(c, emb, ld)) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * ((n + 2 * WBM - 1) / (2 * WBM)));
  cfg.blockDim = dim3(WT);
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = 2;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  na = add_l1_window(attr, na);
  cfg.attrs = attr;
  cfg.numAttrs = na;
#define TRAIL_WIDE(KB)                                                                            \
  cfg.dynamicSmemBytes = WCfg<KB>::SMEM_TOTAL;                                                    \
  return cudaLaunchKernelEx(&cfg, trail_wide_predict_kernel<KB>, c.tmap_emb, c.tmap_emb4,        \
                            c.tmap_emb32, c.tmap_xs1, c.tmap_xs4, c.tmap_xs32, c.tmap_w128, off, \
                            n, c.d / WBK, (const float *)c.b1, (const float *)c.w2,              \
                            (const float *)c.b2, c.host_consts, ids, is_prefill, prior_override, \
                            c.cfg.max_slots, c.lq, c.meta, post, L, c.dev_err, decode_only,     \
                            wide_flags(),                                                         \
                            (c.trace && (int)cfg.gridDim.x <= c.trace_cap) ? c.trace : nullptr)
  switch (wide_kb(c.k)) {
    case 10: TRAIL_WIDE(10);
    case 16: TRAIL_WIDE(16);
    case 20: TRAIL_WIDE(20);
    default: TRAIL_WIDE(32);
  }
#undef TRAIL_WIDE
}

}  // namespace trail
