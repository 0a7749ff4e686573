// K2c — the fused predict kernel (rows a2 + a3): layer 1 on tcgen05 with a cluster split-K
// reduction through distributed shared memory, bias + ReLU + layer-2 partial logits in the
// epilogue, and the head (softmax, Bayesian refinement, expected length, state update) run
// by the last of the H/128 column-tile clusters to finish each row group.
//
//   P:201  h = ReLU(W1 x + b1) (d -> 512), z = W2 h + b2 (512 -> k)
//   P:204  p = softmax(z) (CrossEntropy-trained logits, reading D-6)
//   P:219  q^(0) = normalise(pi * p^(0)); r = m[argmax q^(0)], thr = floor(c r)
//   P:220-222 (D-1, D-2)  q^(t) = normalise((T q^(t-1)) * p^(t)), in the log domain (D-22)
//   P:226  L_t = sum_i q(i) m_i
//
// Grid (m_tiles, H/128, S) with cluster dims (1, 1, S): the S CTAs of a cluster compute the
// same 128-request x 128-hidden tile over disjoint K ranges.
//   warp 0 / lane 0 : TMA producer (X tile 128x64 + W1 tile 128x64 per stage, SW128)
//   warp 1 / lane 0 : tcgen05.mma.cta_group::1.kind::f16 issuer, accumulator in TMEM
//   all 4 warps     : epilogue
//     1. TMEM -> registers -> own shared memory (fp32 128x128 partial tile)
//     2. cluster barrier; CTA r of the cluster sums rows [r*128/S, (r+1)*128/S) over the S
//        partial tiles (ld.shared::cluster, fixed order -> deterministic), adds b1, ReLU,
//        and contracts its 128 hidden units with W2[:, n0:n0+128] -> z_part[row][tile][k]
//     3. release fence + atomic arrival counter per (m_tile, r); the CTA that completes
//        the H/128 column tiles of that row group runs the head, one thread per request.
// No fp32 h round trip through HBM and no separate head launch.  KB (template) bounds the
// bin count so that per-bin loops unroll into registers without code bloat.
#include <math.h>

#include <algorithm>

#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 64;
constexpr int STAGES = 6;
constexpr int MAXS = 16;                              // max cluster size along K
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TILE_LD = BN + 4;                       // padded fp32 row stride
constexpr int PIPE_BYTES = STAGES * STAGE_BYTES;      // 192 KB, reused for the tile
constexpr int BAR_OFF = PIPE_BYTES;
constexpr int W2_OFF = PIPE_BYTES + 256;
constexpr int W2_FLOATS = kMaxBins * BN;
constexpr int SMEM_TOTAL = W2_OFF + (W2_FLOATS + BN) * 4;
static_assert(BM * TILE_LD * 4 <= PIPE_BYTES, "tile must fit in the pipeline buffers");

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of `local_addr` in the shared memory of cluster CTA `rank` (volatile: it must not
// be hoisted above the cluster barrier; the loads that use it may then be batched freely)
__device__ __forceinline__ uint32_t mapa(uint32_t local_addr, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
  return remote;
}
__device__ __forceinline__ float4 ld_cluster_f4(uint32_t addr) {
  float4 v;
  asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(addr));
  return v;
}
__device__ __forceinline__ float logaddexp_f(float a, float b) {
  const float mx = fmaxf(a, b), mn = fminf(a, b);
  if (mx == -INFINITY) return -INFINITY;
  return mx + log1pf(expf(mn - mx));
}
}  // namespace

// One request's head in one thread (all bins in registers, KB >= k compile-time bound).
template <int KB>
__device__ __forceinline__ void head_one(int j, const float (&z)[KB] /* incl. b2 */, int k,
                                         const HeadConsts *__restrict__ cst,
                                         const uint32_t *__restrict__ ids,
                                         const uint8_t *__restrict__ is_prefill,
                                         const float *__restrict__ prior_override, int max_slots,
                                         float *__restrict__ lq_state,
                                         SlotMeta *__restrict__ meta, float *__restrict__ post,
                                         float *__restrict__ Lout, uint32_t *__restrict__ err) {
  const uint32_t slot = __ldg(ids + j);
  if (slot >= (uint32_t)max_slots) {
    atomicOr(err, TRAIL_DEV_BAD_ID);
    if (post)
      for (int b = 0; b < k; ++b) post[(int64_t)j * k + b] = NAN;
    if (Lout) Lout[j] = NAN;
    return;
  }
  // log p = z - logsumexp(z)
  float zmax = -INFINITY;
#pragma unroll
  for (int b = 0; b < KB; ++b)
    if (b < k) zmax = fmaxf(zmax, z[b]);
  float se = 0.f;
#pragma unroll
  for (int b = 0; b < KB; ++b)
    if (b < k) se += expf(z[b] - zmax);
  const float lse = zmax + logf(se);
  SlotMeta mt = meta[slot];
  const bool first = (__ldg(is_prefill + j) != 0) || !(mt.flags & 1u);
  float lq[KB];
  if (first) {
#pragma unroll
    for (int b = 0; b < KB; ++b)
      if (b < k)
        lq[b] = (z[b] - lse) + (prior_override ? logf(__ldg(prior_override + (int64_t)j * k + b))
                                               : cst->log_prior[b]);
  } else {
    float prev[KB];
#pragma unroll
    for (int b = 0; b < KB; ++b)
      if (b < k) prev[b] = lq_state[(int64_t)slot * k + b];
#pragma unroll
    for (int b = 0; b < KB; ++b) {
      if (b < k) {
        // prior(b) = (1 - 1/w_b) q(b) + (1/w_{b+1}) q(b+1): T applied to the posterior
        const float stay = cst->log_stay[b] + prev[b];
        const float move = (b + 1 < k) ? cst->log_move[b] + prev[(b + 1) % KB] : -INFINITY;
        lq[b] = logaddexp_f(stay, move) + (z[b] - lse);
      }
    }
  }
  float qmax = -INFINITY;
#pragma unroll
  for (int b = 0; b < KB; ++b)
    if (b < k) qmax = fmaxf(qmax, lq[b]);
  if (qmax == -INFINITY) {          // all-zero product: fall back to p (D-5)
#pragma unroll
    for (int b = 0; b < KB; ++b)
      if (b < k) {
        lq[b] = z[b] - lse;
        qmax = fmaxf(qmax, lq[b]);
      }
  }
  float qs = 0.f;
#pragma unroll
  for (int b = 0; b < KB; ++b)
    if (b < k) qs += expf(lq[b] - qmax);
  const float lnorm = qmax + logf(qs);
  float L = 0.f;
  int amax = 0;
  float best = -INFINITY;
#pragma unroll
  for (int b = 0; b < KB; ++b) {
    if (b < k) {
      lq[b] -= lnorm;
      const float q = expf(lq[b]);
      L = fmaf(q, cst->m[b], L);
      if (lq[b] > best) { best = lq[b]; amax = b; }    // lowest index on ties
      lq_state[(int64_t)slot * k + b] = lq[b];
      if (post) post[(int64_t)j * k + b] = q;
    }
  }
  if (first) {
    mt.thr = cst->thr_tab[amax];
    mt.age = 0;
    mt.flags = 1u;
  } else {
    mt.age += 1;
  }
  mt.L = L;
  meta[slot] = mt;
  if (Lout) Lout[j] = L;
}

template <int KB>
__global__ void __launch_bounds__(128, 1)
trail_fused_predict_kernel(const __grid_constant__ CUtensorMap tmap_x,
                           const __grid_constant__ CUtensorMap tmap_w, int n, int H, int kblocks,
                           int splits, const float *__restrict__ b1, const float *__restrict__ w2,
                           const float *__restrict__ b2, const HeadConsts *__restrict__ cst,
                           float *__restrict__ zpart, uint32_t *__restrict__ arrive_cnt,
                           const uint32_t *__restrict__ ids, const uint8_t *__restrict__ is_prefill,
                           const float *__restrict__ prior_override, int max_slots,
                           float *__restrict__ lq_state, SlotMeta *__restrict__ meta,
                           float *__restrict__ post, float *__restrict__ Lout,
                           uint32_t *__restrict__ err) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + BAR_OFF);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + BAR_OFF + 8 * (2 * STAGES + 1));
  uint32_t *flag = tmem_slot + 1;
  float *w2s = reinterpret_cast<float *>(smem + W2_OFF);   // [k][BN]
  float *b1s = w2s + W2_FLOATS;                            // [BN]
  float *tile = reinterpret_cast<float *>(smem);           // [BM][TILE_LD] after the mainloop
  const uint32_t sA0 = smem_u32(smem), sB0 = sA0 + STAGES * A_BYTES;
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * STAGES, done = full0 + 16 * STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int m0 = blockIdx.x * BM, nt = blockIdx.y, n0 = nt * BN, NT = gridDim.y;
  const int s = blockIdx.z;
  const uint32_t crank = splits > 1 ? cluster_rank() : 0u;
  const int k = cst->k;
  const int kb0 = (int)((int64_t)s * kblocks / splits);
  const int kb1 = (int)((int64_t)(s + 1) * kblocks / splits);
  const int nkb = kb1 - kb0;

  // constant operands of the epilogue (weights: not produced by an earlier kernel)
  for (int b = 0; b < k; ++b) w2s[b * BN + tid] = __ldg(w2 + (int64_t)b * H + n0 + tid);
  b1s[tid] = __ldg(b1 + n0 + tid);
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_w)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"((uint32_t)BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  griddep_wait();     // X from the pool kernel, slot state from the previous step
  griddep_launch();

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < nkb; ++i) {
      const int st = i % STAGES;
      const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
      mbar_wait(empty0 + 8 * st, ph ^ 1u);
      mbar_expect_tx(full0 + 8 * st, STAGE_BYTES);
      const int kc = (kb0 + i) * BK;
      tma_load_2d(sA0 + st * A_BYTES, &tmap_x, full0 + 8 * st, kc, m0);
      tma_load_2d(sB0 + st * B_BYTES, &tmap_w, full0 + 8 * st, kc, n0);
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
    for (int i = 0; i < nkb; ++i) {
      const int st = i % STAGES;
      const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
      mbar_wait(full0 + 8 * st, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t da = sw128_kmajor_desc(sA0 + st * A_BYTES);
      const uint64_t db = sw128_kmajor_desc(sB0 + st * B_BYTES);
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk)
        umma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : 0u);
      umma_commit(empty0 + 8 * st);
    }
    umma_commit(done);
  }

  // ---- 1. partial tile: TMEM -> own shared memory (pipeline buffers are idle now)
  mbar_wait(done, 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, r);
    float4 *dst = reinterpret_cast<float4 *>(tile + (warp * 32 + lane) * TILE_LD + c);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                           __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (splits > 1) cluster_sync(); else __syncthreads();

  // ---- 2. reduce my row group over the cluster, bias + ReLU, layer-2 partial logits
  const int rows = BM / splits;                 // rows reduced by this CTA (16 for S = 8)
  const int r0 = (int)crank * rows;
  const int tpr = 128 / rows;                   // threads per row (8 for S = 8)
  const int cols = BN / tpr;                    // columns per thread (16 for S = 8)
  const int rr = tid / tpr, cg = tid % tpr;
  const int grow = m0 + r0 + rr;                // request index
  float zp[KB];
#pragma unroll
  for (int b = 0; b < KB; ++b) zp[b] = 0.f;
  {
    const uint32_t base = smem_u32(tile + (r0 + rr) * TILE_LD + cg * cols);
    uint32_t rbase[MAXS];
#pragma unroll
    for (int p = 0; p < MAXS; ++p) rbase[p] = (splits > 1 && p < splits) ? mapa(base, p) : base;
    for (int c4 = 0; c4 < cols / 4; ++c4) {
      float4 v[MAXS];
#pragma unroll
      for (int p = 0; p < MAXS; ++p)             // all S loads in flight, then a fixed-order sum
        if (p < splits) v[p] = ld_cluster_f4(rbase[p] + 16 * c4);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int p = 0; p < MAXS; ++p)
        if (p < splits) { acc.x += v[p].x; acc.y += v[p].y; acc.z += v[p].z; acc.w += v[p].w; }
      const int col = cg * cols + 4 * c4;
      const float h0 = fmaxf(acc.x + b1s[col], 0.f), h1 = fmaxf(acc.y + b1s[col + 1], 0.f);
      const float h2 = fmaxf(acc.z + b1s[col + 2], 0.f), h3 = fmaxf(acc.w + b1s[col + 3], 0.f);
#pragma unroll
      for (int b = 0; b < KB; ++b) {
        if (b < k) {
          const float4 w = *reinterpret_cast<const float4 *>(w2s + b * BN + col);
          zp[b] = fmaf(w.x, h0, fmaf(w.y, h1, fmaf(w.z, h2, fmaf(w.w, h3, zp[b]))));
        }
      }
    }
  }
  // reduce over the tpr threads of a row (consecutive lanes)
  for (int o = 1; o < tpr; o <<= 1) {
#pragma unroll
    for (int b = 0; b < KB; ++b)
      if (b < k) zp[b] += __shfl_xor_sync(0xffffffffu, zp[b], o);
  }
  if (cg == 0 && grow < n) {
    float *zo = zpart + ((int64_t)grow * NT + nt) * k;
#pragma unroll
    for (int b = 0; b < KB; ++b)
      if (b < k) zo[b] = zp[b];
  }
  // peers must finish reading my tile before this CTA exits
  if (splits > 1) cluster_sync();

  // ---- 3. last column tile of this row group runs the head
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    uint32_t *cnt = arrive_cnt + (int64_t)blockIdx.x * splits + crank;
    const uint32_t old = atomicAdd(cnt, 1u);
    const bool last = old == (uint32_t)(NT - 1);
    if (last) *cnt = 0u;                        // re-arm for the next launch
    *flag = last ? 1u : 0u;
  }
  __syncthreads();
  if (*flag) {
    __threadfence();
    if (tid < rows) {
      const int j = m0 + r0 + tid;
      if (j < n) {
        float z[KB];
#pragma unroll
        for (int b = 0; b < KB; ++b) z[b] = 0.f;
        for (int t2 = 0; t2 < NT; ++t2) {       // fixed column-tile order
          const float *zi = zpart + ((int64_t)j * NT + t2) * k;
#pragma unroll
          for (int b = 0; b < KB; ++b)
            if (b < k) z[b] += __ldcg(zi + b);
        }
#pragma unroll
        for (int b = 0; b < KB; ++b)
          if (b < k) z[b] += __ldg(b2 + b);
        head_one<KB>(j, z, k, cst, ids, is_prefill, prior_override, max_slots, lq_state, meta,
                     post, Lout, err);
      }
    }
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"((uint32_t)BN)
                 : "memory");
}

// ------------------------------------------------------------------ host
template <int KB>
static cudaError_t fused_attr() {
  cudaError_t e = cudaFuncSetAttribute(trail_fused_predict_kernel<KB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(trail_fused_predict_kernel<KB>,
                              cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

cudaError_t fused_prepare(Ctx &c) {
  if (c.dtype != TRAIL_BF16) return cudaSuccess;
  cudaError_t e = fused_attr<10>();
  if (e == cudaSuccess) e = fused_attr<16>();
  if (e == cudaSuccess) e = fused_attr<20>();
  if (e == cudaSuccess) e = fused_attr<32>();
  return e;
}

int fused_splits(const Ctx &c, int n) {
  const int tiles = ((n + BM - 1) / BM) * (c.H / BN);
  const int kblocks = c.d / BK;
  int s = std::max(1, c.num_sms / std::max(1, tiles));
  int p = 1;
  while (p * 2 <= std::min(std::min(s, MAXS), kblocks)) p *= 2;   // power of two <= 16
  return p;
}

cudaError_t launch_fused_predict(const Ctx &c, int n, int splits, const uint32_t *ids,
                                 const uint8_t *is_prefill, const float *prior_override,
                                 float *post, float *L, cudaStream_t s) {
  if (!c.have_tmaps) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((n + BM - 1) / BM, c.H / BN, splits);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = SMEM_TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
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
  cfg.attrs = attr;
  cfg.numAttrs = na;
#define TRAIL_FUSED(KB)                                                                          \
  return cudaLaunchKernelEx(&cfg, trail_fused_predict_kernel<KB>, c.tmap_x, c.tmap_w128, n, c.H,  \
                            c.d / BK, splits, (const float *)c.b1, (const float *)c.w2,           \
                            (const float *)c.b2, (const HeadConsts *)c.consts, c.zpart,           \
                            c.arrive_cnt, ids, is_prefill, prior_override, c.cfg.max_slots, c.lq, \
                            c.meta, post, L, c.dev_err)
  if (c.k <= 10) TRAIL_FUSED(10);
  if (c.k <= 16) TRAIL_FUSED(16);
  if (c.k <= 20) TRAIL_FUSED(20);
  TRAIL_FUSED(32);
#undef TRAIL_FUSED
}

}  // namespace trail
