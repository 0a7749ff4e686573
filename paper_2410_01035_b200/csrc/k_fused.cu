// K2c — the fused predict kernel (rows a2 + a3): layer 1 on tcgen05 with a cluster split-K
// reduction through distributed shared memory, bias + ReLU + layer-2 partial logits in the
// epilogue, and the head (softmax, Bayesian refinement, expected length, state update) run
// by the last of the H/128 column-tile CTAs to finish each row group.
//
//   P:201  h = ReLU(W1 x + b1) (d -> 512), z = W2 h + b2 (512 -> k)
//   P:204  p = softmax(z) (CrossEntropy-trained logits, reading D-6)
//   P:219  q^(0) = normalise(pi * p^(0)); r = m[argmax q^(0)], thr = floor(c r)
//   P:220-222 (D-1, D-2)  q^(t) = normalise((T q^(t-1)) * p^(t)), in the log domain (D-22)
//   P:226  L_t = sum_i q(i) m_i
//
// Grid (m_tiles, H/128, S) with cluster dims (1, 1, S), S in [1, 16] chosen on the host so
// that every cluster is resident in one wave (cudaOccupancyMaxActiveClusters).  The S CTAs of
// a cluster compute the same 128-request x 128-hidden tile over disjoint K ranges.
//   warp 0 / lane 0 : TMA producer (X tile 128x64 + W1 tile 128x64 per stage, SW128)
//   warp 1 / lane 0 : tcgen05.mma.cta_group::1.kind::f16 issuer, accumulator in TMEM
//   warps 2-7       : stage the W2 / b1 slices of this column tile (overlaps the mainloop)
//   all 8 warps     : epilogue
//     1. TMEM -> registers -> own shared memory (fp32 128x128 partial tile, padded rows)
//     2. cluster barrier; CTA r owns rows [r*128/S, (r+1)*128/S) and reads those rows of
//        every peer's partial tile straight from the peer's shared memory
//        (ld.shared::cluster, all S loads of an item in flight) — or, with
//        TRAIL_FUSED_PULL=0, each CTA PUSHES row group r to CTA r with one bulk
//        shared::cta -> shared::cluster copy per peer (completion on the receiver's mbarrier);
//     3. CTA r sums its rows over the S partials in fixed rank order (deterministic), adds
//        b1, ReLU, and contracts its 128 hidden units with W2[:, n0:n0+128] -> z_part;
//     4. release fence + atomic arrival counter per (m_tile, r); the CTA that completes the
//        H/128 column tiles of that row group runs the head, one thread per request.
// No fp32 h round trip through HBM and no separate head launch.  KB (template) bounds the
// bin count; W2 rows >= k are zero-padded in shared memory so the layer-2 loops have a
// compile-time trip count.
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "head_dev.cuh"
#include "xgather.cuh"
#include "sm100_ptx.cuh"
#include "trail_internal.cuh"

namespace trail {

using namespace ptx;

namespace {
constexpr int THREADS = 256;
constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 64;
constexpr int MAXS = 16;                              // max cluster size along K
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TILE_LD = BN + 4;                       // padded fp32 row stride (528 B)
constexpr int ROW_BYTES = TILE_LD * 4;
constexpr int TILE_BYTES = BM * ROW_BYTES;            // 67584
constexpr int LAND_OFF = TILE_BYTES;                  // landing slots for peers' row groups

// Shared-memory plan (KB = bin bound): pipeline stages (reused by the partial tile and the
// landing slots after the mainloop), barriers, W2 / b1 slices, and the per-row slot state
// of the rows this CTA may run the head for (prefetched during the mainloop).
template <int KB>
struct FCfg {
  static constexpr int STAGES = KB <= 20 ? 6 : 5;
  static constexpr int PIPE_BYTES = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFF = PIPE_BYTES;
  static constexpr int W2_OFF = BAR_OFF + 256;
  static constexpr int B1_OFF = W2_OFF + KB * BN * 4;
  static constexpr int SLOT_OFF = B1_OFF + BN * 4;     // u32 [BM]: slot id | prefill << 31
  static constexpr int META_OFF = SLOT_OFF + BM * 4;   // SlotMeta [BM]
  static constexpr int LQ_OFF = META_OFF + BM * 16;    // float [BM][KB] previous log q
  static constexpr int HC_OFF = LQ_OFF + BM * KB * 4;   // HeadSmem (per-bin constants)
  static constexpr int SMEM_USED = HC_OFF + 5 * kMaxBins * 4;
  static constexpr int SMEM_TOTAL = SMEM_USED + 1024;  // + slack for 1024-byte alignment
  static_assert(LAND_OFF + (BM + MAXS) * ROW_BYTES <= PIPE_BYTES, "tile + landing must fit");
  static_assert(SMEM_TOTAL <= 232448, "shared memory budget");
};

__host__ __device__ __forceinline__ int row_lo(int r, int S) { return (r * BM) / S; }
}  // namespace

template <int KB>
__global__ void __launch_bounds__(THREADS, 1)
trail_fused_predict_kernel(const __grid_constant__ CUtensorMap tmap_emb,
                           const __grid_constant__ CUtensorMap tmap_emb4,
                           const __grid_constant__ CUtensorMap tmap_emb32,
                           const __grid_constant__ CUtensorMap tmap_xs,
                           const __grid_constant__ CUtensorMap tmap_xs4,
                           const __grid_constant__ CUtensorMap tmap_xs32,
                           const __grid_constant__ CUtensorMap tmap_w,
                           const int32_t *__restrict__ off, int n, int H, int kblocks,
                           int splits, const float *__restrict__ b1, const float *__restrict__ w2,
                           const float *__restrict__ b2, const __grid_constant__ HeadConsts cst,
                           float *__restrict__ zpart, uint32_t *__restrict__ arrive_cnt,
                           const uint32_t *__restrict__ ids, const uint8_t *__restrict__ is_prefill,
                           const float *__restrict__ prior_override, int max_slots,
                           float *__restrict__ lq_state, SlotMeta *__restrict__ meta,
                           float *__restrict__ post, float *__restrict__ Lout,
                           uint32_t *__restrict__ err, uint64_t *__restrict__ trace, int spin,
                           int pull) {
  using C = FCfg<KB>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the SW128 operand tiles; offsetting the __shared__ array (not
  // casting through an integer) keeps every epilogue access an LDS/STS, not a generic LD/ST
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::BAR_OFF);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::BAR_OFF + 8 * (2 * STAGES + 2));
  uint32_t *flag = tmem_slot + 1;
  float *w2s = reinterpret_cast<float *>(smem + C::W2_OFF);   // float4 [BN/4][KB], b >= k zero
  float *b1s = reinterpret_cast<float *>(smem + C::B1_OFF);   // [BN]
  uint32_t *s_slot = reinterpret_cast<uint32_t *>(smem + C::SLOT_OFF);
  SlotMeta *s_meta = reinterpret_cast<SlotMeta *>(smem + C::META_OFF);
  float *s_lq = reinterpret_cast<float *>(smem + C::LQ_OFF);
  float *tile = reinterpret_cast<float *>(smem);           // [BM][TILE_LD] after the mainloop
  const uint32_t sA0 = smem_u32(smem), sB0 = sA0 + STAGES * A_BYTES;
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * STAGES;
  const uint32_t done = full0 + 16 * STAGES, land = done + 8;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  // diagnostics (trail_trace_*): per-CTA phase timestamps, globaltimer ns
  uint64_t *tr = trace ? trace + 16 * (int64_t)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) : nullptr;
  if (tr && tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[0] = gtimer();
    tr[15] = smid;
  }
  const int m0 = blockIdx.x * BM, nt = blockIdx.y, n0 = nt * BN, NT = gridDim.y;
  const int S = splits;
  const int crank = S > 1 ? (int)cluster_rank() : 0;
  const int k = cst.k;
  const int kb0 = (int)((int64_t)crank * kblocks / S);
  const int kb1 = (int)((int64_t)(crank + 1) * kblocks / S);
  const int nkb = kb1 - kb0;
  const int r0 = row_lo(crank, S), rows = row_lo(crank + 1, S) - r0;
  const int slot_rows = (BM + S - 1) / S;                  // landing slot size (rows)

  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, 1);
    }
    mbar_init(done, 1);
    mbar_init(land, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_emb)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_emb32)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_xs32)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_w)) : "memory");
  }
  if (warp == 0) tmem_alloc(smem_u32(tmem_slot), (uint32_t)BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // the landing barrier's single arrival, carrying the bytes the S-1 peers will push
  if (tid == 0 && S > 1 && !pull) mbar_expect_tx(land, (uint32_t)((S - 1) * rows * ROW_BYTES));
  griddep_launch();
  if (tr && tid == 0) tr[1] = gtimer();

  // roles: lane 0 of warp 0 = TMA producer, lane 0 of warp 1 = MMA issuer; the other lanes
  // of those warps park at __syncwarp; warps 2-7 stage the epilogue weights meanwhile.
  // PDL: only the producer's X loads depend on the previous kernel (the pool kernel writes
  // X), so the W1 tiles of the first STAGES stages are requested before griddep_wait and
  // the prologue + first weight fetches overlap the previous kernel's tail.  Every other
  // thread waits before the epilogue, which reads the slot state.
  if (warp == 0) {
    // A operand = the n x d embedding matrix X, gathered row by row (row a1): request j's row
    // is emb row off[j] when it has exactly one row (decode: bit-exact), else the
    // pooled prompt mean the pool kernel wrote to xs row j (prefill).  Lane l owns rows
    // 4l..4l+3 of the tile: one TMA tile::gather4 per k-block when all four come from emb,
    // else four single-row loads.  Only xs rows depend on the previous kernel (PDL): decode
    // tiles never wait for the pool kernel.
    const XPlan xp = xplan_make(off, n, m0, lane);
    const bool tile_xs = xp.tile_xs;
    const int pre = nkb < STAGES ? nkb : STAGES;
    if (lane == 0)
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(full0 + 8 * i, STAGE_BYTES);
        tma_load_2d(sB0 + i * B_BYTES, &tmap_w, full0 + 8 * i, (kb0 + i) * BK, n0);
      }
    if (tile_xs) griddep_wait();
    __syncwarp();
    for (int i = 0; i < nkb; ++i) {
      const int st = i % STAGES;
      const int kc = (kb0 + i) * BK;
      if (i >= STAGES) {
        if (lane == 0) {
          const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
          mbar_wait(empty0 + 8 * st, ph ^ 1u);
          mbar_expect_tx(full0 + 8 * st, STAGE_BYTES);
          tma_load_2d(sB0 + st * B_BYTES, &tmap_w, full0 + 8 * st, kc, n0);
        }
        __syncwarp();
      }
      xplan_issue<false>(xp, lane, sA0 + st * A_BYTES, full0 + 8 * st, kc, &tmap_emb, &tmap_emb4,
                         &tmap_emb32, &tmap_xs, &tmap_xs4, &tmap_xs32);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      for (int i = 0; i < nkb; ++i) {
        const int st = i % STAGES;
        const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
        mbar_wait(full0 + 8 * st, ph);
        if (tr && i == 0) tr[2] = gtimer();
        tc_fence_after();
        const uint64_t da = sw128_kmajor_desc(sA0 + st * A_BYTES);
        const uint64_t db = sw128_kmajor_desc(sB0 + st * B_BYTES);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          umma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : 0u);
        umma_commit(empty0 + 8 * st);
      }
      umma_commit(done);
    }
    __syncwarp();
  } else {
    // W2[:, n0:n0+BN] (zero rows for b >= k) and b1[n0:n0+BN]: weights, not produced by an
    // earlier kernel; 192 threads, float4 loads all in flight
    const int t = tid - 64;
    constexpr int NV = KB * (BN / 4);
#pragma unroll
    for (int v0 = 0; v0 < NV; v0 += THREADS - 64) {
      const int v = v0 + t;
      if (v < NV) {
        const int b = v / (BN / 4), c = (v % (BN / 4)) * 4;
        float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
        if (b < k) w = __ldg(reinterpret_cast<const float4 *>(w2 + (int64_t)b * H + n0 + c));
        reinterpret_cast<float4 *>(w2s)[(c >> 2) * KB + b] = w;   // w2q[c/4][b] = W2[b][c..c+3]
      }
    }
    if (t < BN / 4)
      *reinterpret_cast<float4 *>(b1s + 4 * t) =
          __ldg(reinterpret_cast<const float4 *>(b1 + n0 + 4 * t));
    if (t < kMaxBins) {
      HeadSmem &hs = *reinterpret_cast<HeadSmem *>(smem + C::HC_OFF);
      hs.m[t] = cst.m[t];
      hs.log_stay[t] = cst.log_stay[t];
      hs.log_move[t] = cst.log_move[t];
      hs.log_prior[t] = cst.log_prior[t];
      hs.thr[t] = cst.thr_tab[t];
    }
    // slot state of the rows this CTA may run the head for (no other CTA of this launch
    // touches those slots; earlier writers completed — PDL chain): off the critical path
    if (t < rows) {
      const int j = m0 + r0 + t;
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

  // No griddep_wait for the epilogue: it reads only inputs, weights and slot state written by
  // kernels that completed before the pool kernel passed its own griddep_wait (PDL chain).
  // ---- 1. partial tile: TMEM -> own shared memory (pipeline buffers are idle now)
  mbar_wait(done, 0);
  __syncwarp();
  if (tr && tid == 0) tr[3] = gtimer();
  tc_fence_after();
  {
    const int g = warp & 3, half = warp >> 2;
    const int row = 32 * g + lane;
#pragma unroll
    for (int cc = 0; cc < 64; cc += 32) {
      const int c = 64 * half + cc;
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)(32 * g) << 16) + (uint32_t)c, r);
      float4 *dst = reinterpret_cast<float4 *>(tile + row * TILE_LD + c);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                             __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
    }
  }
  tc_fence_before();
  fence_proxy_async_smem();          // the tile is read by the bulk-copy (async) proxy
  if (tr && tid == 0) tr[4] = gtimer();
  if (S > 1) cluster_sync(); else __syncthreads();
  if (tr && tid == 0) tr[5] = gtimer();

  // ---- 2. push row group p of my partial tile to CTA p (one bulk copy per peer)
  const uint32_t land_base = smem_u32(smem + LAND_OFF);
  if (S > 1 && !pull) {
    if (tid == 0) {
      for (int q = 1; q < S; ++q) {
        const int p = (crank + q) % S;
        const int pr0 = row_lo(p, S), prows = row_lo(p + 1, S) - pr0;
        const uint32_t src = smem_u32(tile + pr0 * TILE_LD);
        const uint32_t dst = mapa(land_base + (uint32_t)(crank * slot_rows * ROW_BYTES), (uint32_t)p);
        bulk_s2cluster(dst, src, (uint32_t)(prows * ROW_BYTES), mapa(land, (uint32_t)p));
      }
    }
    mbar_wait(land, 0);
    cluster_arrive();                // "my slices have landed" (waited on before exit)
  }
  if (tr && tid == 0) tr[6] = gtimer();

  // ---- 3a. h = ReLU(sum of the S partials in rank order + b1) for my rows, in place
  //           (compact loops: these kernels run once per step, so instruction fetch from
  //           L2 is on the critical path and straight-line unrolled code costs more than
  //           it saves)
  if (pull && S > 1) {
    // pull variant: read the peers' partial rows straight from their shared memory
    // (ld.shared::cluster, all S loads of an item in flight), no landing copies
    const uint32_t tile_s = smem_u32(tile);
    for (int i = tid; i < rows * (BN / 4); i += THREADS) {
      const int r = i >> 5, c = (i & 31) * 4;
      const uint32_t off = (uint32_t)(((r0 + r) * TILE_LD + c) * 4);
      float4 v[MAXS];
#pragma unroll
      for (int p = 0; p < MAXS; ++p)
        if (p < S) v[p] = ld_cluster_f4(mapa(tile_s + off, (uint32_t)p));
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int p = 0; p < MAXS; ++p)
        if (p < S) { acc.x += v[p].x; acc.y += v[p].y; acc.z += v[p].z; acc.w += v[p].w; }
      const float4 bb = *reinterpret_cast<const float4 *>(b1s + c);
      *reinterpret_cast<float4 *>(tile + (r0 + r) * TILE_LD + c) =
          make_float4(fmaxf(acc.x + bb.x, 0.f), fmaxf(acc.y + bb.y, 0.f),
                      fmaxf(acc.z + bb.z, 0.f), fmaxf(acc.w + bb.w, 0.f));
    }
    cluster_arrive();                // done reading the peers (waited on before exit)
  } else {
    const float *land_f = reinterpret_cast<const float *>(smem + LAND_OFF);
    for (int i = tid; i < rows * (BN / 4); i += THREADS) {
      const int r = i >> 5, c = (i & 31) * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int p = 0; p < S; ++p) {
        const float *src = p == crank ? tile + (r0 + r) * TILE_LD + c
                                      : land_f + (p * slot_rows + r) * TILE_LD + c;
        const float4 v = *reinterpret_cast<const float4 *>(src);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      const float4 bb = *reinterpret_cast<const float4 *>(b1s + c);
      *reinterpret_cast<float4 *>(tile + (r0 + r) * TILE_LD + c) =
          make_float4(fmaxf(acc.x + bb.x, 0.f), fmaxf(acc.y + bb.y, 0.f),
                      fmaxf(acc.z + bb.z, 0.f), fmaxf(acc.w + bb.w, 0.f));
    }
  }
  __syncthreads();
  // ---- 3b. layer-2 partial logits of this column tile, one thread per (row, bin)
  for (int i = tid; i < rows * KB; i += THREADS) {
    const int r = i / KB, b = i - r * KB;
    const int j = m0 + r0 + r;
    if (b < k && j < n) {
      const float4 *hr = reinterpret_cast<const float4 *>(tile + (r0 + r) * TILE_LD);
      const float4 *wq = reinterpret_cast<const float4 *>(w2s) + b;
      float z0 = 0.f, z1 = 0.f;
#pragma unroll 4
      for (int c4 = 0; c4 < BN / 4; c4 += 2) {
        const float4 h0 = hr[c4], w0 = wq[c4 * KB];
        const float4 h1 = hr[c4 + 1], w1 = wq[(c4 + 1) * KB];
        z0 = fmaf(h0.x, w0.x, fmaf(h0.y, w0.y, fmaf(h0.z, w0.z, fmaf(h0.w, w0.w, z0))));
        z1 = fmaf(h1.x, w1.x, fmaf(h1.y, w1.y, fmaf(h1.z, w1.z, fmaf(h1.w, w1.w, z1))));
      }
      zpart[((int64_t)j * NT + nt) * k + b] = z0 + z1;
    }
  }
  if (tr && tid == 0) tr[7] = gtimer();

  // ---- 4. head (row a3) once the NT column tiles of this row group have their z_part.
  //    spin mode (the whole grid is one wave, so the NT CTAs are co-resident): every column
  //    tile waits for the group's epoch counter and runs the head for rows r = nt (mod NT);
  //    otherwise the last CTA to arrive runs the head for all rows of the group.
  __syncthreads();
  if (tid == 0) {
    uint32_t *cnt = arrive_cnt + (int64_t)blockIdx.x * MAXS + crank;
    uint32_t old;
    // release: this CTA's z_part stores (ordered before it by the barrier)
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    if (spin) {
      const uint32_t target = (old / (uint32_t)NT + 1u) * (uint32_t)NT;   // monotone epochs
      uint32_t cur = old + 1u;
      while ((int)(cur - target) < 0) {
        __nanosleep(32);
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(cnt) : "memory");
      }
      *flag = 1u;
    } else {
      const bool last = old % (uint32_t)NT == (uint32_t)(NT - 1);
      *flag = last ? 1u : 0u;
    }
  }
  __syncthreads();
  if (tr && tid == 0) tr[9] = gtimer();
  if (*flag) {
    // one lane per bin, SEG-lane segments (2 requests per warp for k <= 16)
    const int SEG = k <= 16 ? 16 : 32;
    const int per_warp = 32 / SEG, seg = lane / SEG, b = lane % SEG;
    const int rstep = spin ? NT : 1, rfirst = spin ? nt : 0;
    const int my_rows = rows > rfirst ? (rows - rfirst + rstep - 1) / rstep : 0;
    const HeadSmem &hc = *reinterpret_cast<const HeadSmem *>(smem + C::HC_OFF);
    for (int base = warp * per_warp; base < my_rows; base += (THREADS / 32) * per_warp) {
      const int q = base + seg;
      const int r = rfirst + q * rstep;
      const bool rv = q < my_rows;
      const int j = rv ? m0 + r0 + r : n;
      float z = 0.f;
      if (j < n && b < k) {
        z = __ldg(b2 + b);
        for (int t = 0; t < NT; ++t) z += __ldcg(zpart + ((int64_t)j * NT + t) * k + b);
      }
      const int rr = rv ? r : 0;
      head_seg(j, n, k, SEG, b, z, hc, cst.dyn_c, rv ? s_slot[r] : 0xFFFFFFFFu, s_meta[rr],
               b < KB ? s_lq[rr * KB + (b < KB ? b : 0)] : -INFINITY, prior_override, lq_state,
               meta, post, Lout, err);
    }
  }
  if (tr && tid == 0) tr[11] = gtimer();
  if (S > 1) cluster_wait();         // every CTA's incoming slices landed: my copies are done
  __syncthreads();
  if (tr && tid == 0) { tr[8] = gtimer(); tr[14] = *flag; }
  if (warp == 0) tmem_dealloc(tmem, (uint32_t)BN);
}

// ------------------------------------------------------------------ host
template <int KB>
static cudaError_t fused_attr() {
  cudaError_t e = cudaFuncSetAttribute(trail_fused_predict_kernel<KB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, FCfg<KB>::SMEM_TOTAL);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(trail_fused_predict_kernel<KB>,
                              cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

template <int KB>
static cudaError_t fused_occupancy(Ctx &c) {
  for (int s = 1; s <= MAXS; ++s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, 1, s);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = FCfg<KB>::SMEM_TOTAL;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, trail_fused_predict_kernel<KB>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      nc = 0;
    }
    c.fused_max_clusters[s] = nc;
  }
  return cudaSuccess;
}

// Split-K reduction by direct DSMEM loads (default; measured 0.9 µs shorter than the bulk
// push + landing wait at c2); TRAIL_FUSED_PULL=0 selects the push variant for comparison
static int fused_pull() {
  static const int v = [] {
    const char *e = getenv("TRAIL_FUSED_PULL");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}

static int fused_kb(int k) { return k <= 10 ? 10 : k <= 16 ? 16 : k <= 20 ? 20 : 32; }

cudaError_t fused_prepare(Ctx &c) {
  if (c.dtype != TRAIL_BF16) return cudaSuccess;
  cudaError_t e = fused_attr<10>();
  if (e == cudaSuccess) e = fused_attr<16>();
  if (e == cudaSuccess) e = fused_attr<20>();
  if (e == cudaSuccess) e = fused_attr<32>();
  if (e != cudaSuccess) return e;
  switch (fused_kb(c.k)) {
    case 10: return fused_occupancy<10>(c);
    case 16: return fused_occupancy<16>(c);
    case 20: return fused_occupancy<20>(c);
    default: return fused_occupancy<32>(c);
  }
}

// Split-K factor: the largest SM coverage (tiles x S) for which every cluster of S CTAs is
// resident at once (one wave; the cluster barrier requires co-residency anyway), S <= 16
// and S <= the number of 64-wide K blocks.  Ties go to the smaller S (less exchange).
int fused_splits(const Ctx &c, int n) {
  const int tiles = ((n + BM - 1) / BM) * (c.H / BN);
  const int kblocks = c.d / BK;
  if (const char *e = getenv("TRAIL_FUSED_SPLITS")) {
    const int v = atoi(e);
    if (v >= 1 && v <= MAXS) return std::min(v, kblocks);
  }
  int best = 1, best_cov = 0;
  for (int s = 1; s <= std::min(MAXS, kblocks); ++s) {
    const int maxc = c.fused_max_clusters[s];
    if (maxc <= 0 || tiles > maxc) continue;
    if (tiles * s > best_cov) { best_cov = tiles * s; best = s; }
  }
  return best;
}

// row-gather tensor maps over the caller's embeddings (boxes 64 x {1, 4, 32}, SW128),
// re-encoded only when the pointer or the row stride changes
bool ensure_emb_tmaps(Ctx &c, const void *emb, int64_t ld) {
  if (emb == c.tmap_emb_ptr && ld == c.tmap_emb_ld) return true;
  const uint64_t rows = 0x7FFFFFFF;     // rows are addressed through off[] only
  if (!encode_rows_bf16(&c.tmap_emb, emb, (uint64_t)c.d, rows, (uint64_t)ld, BK, 1) ||
      !encode_rows_bf16(&c.tmap_emb4, emb, (uint64_t)c.d, rows, (uint64_t)ld, BK, 4) ||
      !encode_rows_bf16(&c.tmap_emb32, emb, (uint64_t)c.d, rows, (uint64_t)ld, BK, 32))
    return false;
  c.tmap_emb_ptr = emb;
  c.tmap_emb_ld = ld;
  return true;
}

cudaError_t launch_fused_predict(Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                                 int splits, const uint32_t *ids,
                                 const uint8_t *is_prefill, const float *prior_override,
                                 float *post, float *L, cudaStream_t s) {
  if (!c.have_tmaps) return cudaErrorInvalidValue;
  if (!ensure_emb_tmaps(c, emb, ld)) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((n + BM - 1) / BM, c.H / BN, splits);
  cfg.blockDim = dim3(THREADS);
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = 1;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = splits;
  ++na;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  na = add_l1_window(attr, na);
  cfg.attrs = attr;
  cfg.numAttrs = na;
  uint64_t *trace =
      (c.trace && (int)(cfg.gridDim.x * cfg.gridDim.y * cfg.gridDim.z) <= c.trace_cap) ? c.trace
                                                                                       : nullptr;
  // the spin-wait head needs every cluster resident at once.  Occupancy on an idle GPU says
  // one wave fits, but nothing guarantees it under MPS / green contexts / a concurrent
  // persistent kernel (the side-stream overlap use case), where a spinning CTA could wait on
  // a peer that never gets an SM.  So the default is the last-arriver head (no inter-CTA
  // wait); TRAIL_HEAD_SPIN=1 opts into the spin head for a GPU the caller owns exclusively.
  const int tiles = (int)(cfg.gridDim.x * cfg.gridDim.y);
  static const bool spin_opt_in = [] {
    const char *e = getenv("TRAIL_HEAD_SPIN");
    return e && e[0] == '1';
  }();
  const int spin =
      (spin_opt_in && splits <= MAXS && tiles <= c.fused_max_clusters[splits]) ? 1 : 0;
#define TRAIL_FUSED(KB)                                                                          \
  cfg.dynamicSmemBytes = FCfg<KB>::SMEM_TOTAL;                                                     \
  return cudaLaunchKernelEx(&cfg, trail_fused_predict_kernel<KB>, c.tmap_emb, c.tmap_emb4,       \
                            c.tmap_emb32, c.tmap_xs1, c.tmap_xs4, c.tmap_xs32,                    \
                            c.tmap_w128, off, n, c.H,                                             \
                            c.d / BK, splits, (const float *)c.b1, (const float *)c.w2,           \
                            (const float *)c.b2, c.host_consts, c.zpart,                                  \
                            c.arrive_cnt, ids, is_prefill, prior_override, c.cfg.max_slots, c.lq, \
                            c.meta, post, L, c.dev_err, trace, spin, fused_pull())
  switch (fused_kb(c.k)) {
    case 10: TRAIL_FUSED(10);
    case 16: TRAIL_FUSED(16);
    case 20: TRAIL_FUSED(20);
    default: TRAIL_FUSED(32);
  }
#undef TRAIL_FUSED
}

}  // namespace trail
