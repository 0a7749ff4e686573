// K2t — classifier layer 1 of an fp32 handle (configs[0]) on the 5th-generation tensor cores,
// with fp32-level accuracy from a 3xTF32 split (row a2).
//
// P:201 "The first layer maps the input embedding to a 512-dimensional space": the split-K
// pre-activation partial sums
//     partial[s][j][o] = sum_{k in split s} W1[o][k] * X[j][k]
// in the same layout as K2a (k_gemv.cu), so bias, ReLU, the fixed-order reduction over the S
// splits, layer 2 and the head stay in K3 (k_head.cu).
//
// Why: fp32 W1 (8 MB at d = 4096) with n = 64 requests is 268 MFLOP; on the CUDA cores K2a is
// FFMA-bound at ~15 TFLOP/s (0.2 of the FFMA peak).  tcgen05.mma kind::tf32 reads fp32 words
// but uses only 10 mantissa bits, which would put ~1e-3 relative error into h.  So every
// operand is split exactly, x = hi + lo with hi = x with its 13 low mantissa bits cleared
// (a TF32 value) and lo = x - hi (exact in fp32), and the product is accumulated as
//     hi_W hi_X + hi_W lo_X + lo_W hi_X          (fp32 accumulator in TMEM)
// — the dropped lo_W lo_X term and lo's own truncation leave ~2^-20 relative error per
// product, the same order as fp32 FFMA accumulation (the BASELINE bound is 2e-3 on q).
//
// Grid (H / 128, S), S = ceil(d / 128): a CTA owns 128 hidden rows x 128 columns of K.
//   thread 0 : W1 slices by TMA (4 boxes of 128 rows x 32 fp32, SW128) before the PDL wait
//   warp 0   : X rows by TMA from the caller's embeddings (decode: bit-exact row) or
//              xs (prompt mean from K1), planned as in the bf16 kernels (xgather.cuh)
//   all      : hi / lo split in shared memory (position-wise, so the swizzle is irrelevant)
//   thread 0 : 4 slices x 4 K-steps x 3 MMAs (M = 128, N = 64, K = 8) into 64 TMEM columns
//   warps 0-3: TMEM lane = hidden row -> partial[s][j][o] (coalesced over o)
// Requests are processed in blocks of 64 (N); W1's split tiles are reused across blocks.
#include "sm100_ptx.cuh"
#include "trail_internal.cuh"
#include "xgather.cuh"

namespace trail {

using namespace ptx;

namespace {
constexpr int TT = 256;                     // threads
constexpr int TBM = 128;                    // hidden rows per CTA (MMA M)
constexpr int TBN = 64;                     // requests per block (MMA N)
constexpr int TSL = 32;                     // fp32 per 128-byte swizzle atom = one K slice
constexpr int TNS = 4;                      // slices per CTA
constexpr int TKC = TNS * TSL;              // K columns per CTA (128)
constexpr int W_SLICE = TBM * 128;          // 16 KB
constexpr int X_SLICE = TBN * 128;          // 8 KB
constexpr int W_BYTES = TNS * W_SLICE;      // 64 KB
constexpr int X_BYTES = TNS * X_SLICE;      // 32 KB
constexpr int OFF_WLO = W_BYTES;
constexpr int OFF_XHI = 2 * W_BYTES;
constexpr int OFF_XLO = 2 * W_BYTES + X_BYTES;
constexpr int OFF_BAR = 2 * W_BYTES + 2 * X_BYTES;
constexpr int TSMEM = OFF_BAR + 64 + 1024;  // + slack for 1024-byte alignment

// x -> (hi, lo) in place: hi over x, lo into the twin tile at the same offset
__device__ __forceinline__ void split_tf32(uint8_t *hi, uint8_t *lo, int bytes) {
  for (int v = threadIdx.x; v < bytes / 16; v += TT) {
    const float4 x = reinterpret_cast<const float4 *>(hi)[v];
    float4 h;
    h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
    h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
    h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
    h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
    reinterpret_cast<float4 *>(hi)[v] = h;
    reinterpret_cast<float4 *>(lo)[v] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
  }
}
}  // namespace

__global__ void __launch_bounds__(TT, 1)
trail_tf32_l1_kernel(const __grid_constant__ CUtensorMap tmap_w,
                     const __grid_constant__ CUtensorMap tmap_e1,
                     const __grid_constant__ CUtensorMap tmap_e4,
                     const __grid_constant__ CUtensorMap tmap_e32,
                     const __grid_constant__ CUtensorMap tmap_x1,
                     const __grid_constant__ CUtensorMap tmap_x4,
                     const __grid_constant__ CUtensorMap tmap_x32, const int32_t *__restrict__ off,
                     int n, int H, float *__restrict__ partial) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t s0 = smem_u32(smem);
  const uint32_t wbar = s0 + OFF_BAR, xbar = wbar + 8, mbar = wbar + 16;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + OFF_BAR + 24);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int o0 = blockIdx.x * TBM, s = blockIdx.y, k0 = s * TKC;

  if (tid == 0) {
    mbar_init(wbar, 1);
    mbar_init(xbar, 1);
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // W1 is a weight (independent of earlier kernels): in flight before the PDL wait
    mbar_expect_tx(wbar, W_BYTES);
#pragma unroll
    for (int sl = 0; sl < TNS; ++sl) tma_load_2d(s0 + sl * W_SLICE, &tmap_w, wbar, k0 + sl * TSL, o0);
  }
  if (warp == 0) tmem_alloc(smem_u32(tmem_slot), (uint32_t)TBN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // prompt means (xs) come from K1: wait for it only when some request has several rows
  bool pooled = false;
  for (int j = tid; j < n; j += TT) pooled |= __ldg(off + j + 1) - __ldg(off + j) != 1;
  if (__syncthreads_or(pooled)) griddep_wait();
  griddep_launch();

  constexpr uint32_t idesc = idesc_tf32_f32(TBM, TBN);
  for (int j0 = 0, blk = 0; j0 < n; j0 += TBN, ++blk) {
    const int nb = min(TBN, n - j0);
    const uint32_t ph = (uint32_t)(blk & 1);
    if (warp == 0) {
      // the block's 64 rows planned like the bf16 kernels' A tiles (xgather.cuh): runs of
      // consecutive decode rows become 32- or 4-row boxes, scattered rows tile::gather4 —
      // lanes 0-15 own rows 4 lane .. 4 lane + 3 (rows past n are zero-filled / unused)
      const XPlan xp = xplan_make(off, n, j0, lane);
      if (lane == 0) mbar_expect_tx(xbar, (uint32_t)(TBN * TNS * 128));
      __syncwarp();
      if (lane < TBN / 4)
#pragma unroll
        for (int sl = 0; sl < TNS; ++sl)
          xplan_issue<false>(xp, lane, s0 + OFF_XHI + sl * X_SLICE, xbar, k0 + sl * TSL, &tmap_e1,
                             &tmap_e4, &tmap_e32, &tmap_x1, &tmap_x4, &tmap_x32);
    }
    if (blk == 0) {
      mbar_wait(wbar, 0);
      split_tf32(smem, smem + OFF_WLO, W_BYTES);
    }
    mbar_wait(xbar, ph);
    split_tf32(smem + OFF_XHI, smem + OFF_XLO, X_BYTES);
    fence_proxy_async_smem();         // generic-proxy writes -> tensor-core (async proxy) reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
#pragma unroll
      for (int sl = 0; sl < TNS; ++sl) {
        const uint64_t wh = sw128_kmajor_desc(s0 + sl * W_SLICE);
        const uint64_t wl = sw128_kmajor_desc(s0 + OFF_WLO + sl * W_SLICE);
        const uint64_t xh = sw128_kmajor_desc(s0 + OFF_XHI + sl * X_SLICE);
        const uint64_t xl = sw128_kmajor_desc(s0 + OFF_XLO + sl * X_SLICE);
#pragma unroll
        for (int kk = 0; kk < TSL / 8; ++kk) {   // +32 bytes along K per 8 fp32
          umma_tf32(tmem, wh + 2 * kk, xh + 2 * kk, idesc, (sl > 0 || kk > 0) ? 1u : 0u);
          umma_tf32(tmem, wh + 2 * kk, xl + 2 * kk, idesc, 1u);
          umma_tf32(tmem, wl + 2 * kk, xh + 2 * kk, idesc, 1u);
        }
      }
      umma_commit(mbar);
    }
    __syncwarp();
    mbar_wait(mbar, ph);
    tc_fence_after();
    if (warp < 4) {                   // TMEM lane = hidden row o0 + 32 warp + lane
      const int o = o0 + 32 * warp + lane;
#pragma unroll
      for (int cb = 0; cb < TBN; cb += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)cb, r);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int j = j0 + cb + q;
          if (j < n) partial[((int64_t)s * n + j) * H + o] = __uint_as_float(r[q]);
        }
      }
    }
    tc_fence_before();
    __syncthreads();                  // TMEM and the X tiles are reused by the next block
    tc_fence_after();
  }
  if (warp == 0) tmem_dealloc(tmem, (uint32_t)TBN);
}

// ------------------------------------------------------------------ host
int tf32_splits(const Ctx &c) { return (c.d + TKC - 1) / TKC; }

bool tf32_supported(const Ctx &c) {
  return c.dtype == TRAIL_F32 && c.H % TBM == 0 && c.d % 4 == 0 && c.have_tmap_tf32;
}

cudaError_t tf32_prepare(Ctx &c) {
  if (c.dtype != TRAIL_F32 || c.H % TBM != 0 || c.d % 4 != 0) return cudaSuccess;
  const uint64_t xr = (uint64_t)c.cfg.max_requests, dd = (uint64_t)c.d;
  c.have_tmap_tf32 = encode_rows_f32_sw128(&c.tmap_w_tf32, c.w1, dd, (uint64_t)c.H, dd, TSL, TBM) &&
                     encode_rows_f32_sw128(&c.tmap_xs_tf32[0], c.xs, dd, xr, dd, TSL, 1) &&
                     encode_rows_f32_sw128(&c.tmap_xs_tf32[1], c.xs, dd, xr, dd, TSL, 4) &&
                     encode_rows_f32_sw128(&c.tmap_xs_tf32[2], c.xs, dd, xr, dd, TSL, 32);
  if (!c.have_tmap_tf32) return cudaSuccess;   // K2a serves the handle
  return cudaFuncSetAttribute(trail_tf32_l1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              TSMEM);
}

cudaError_t launch_tf32_l1(Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                           cudaStream_t s) {
  if (!tf32_supported(c)) return cudaErrorInvalidValue;
  if (emb != c.tmap_e_tf32_ptr || ld != c.tmap_e_tf32_ld) {   // rows addressed through off[]
    const uint64_t dd = (uint64_t)c.d, rows = 0x7FFFFFFF, l = (uint64_t)ld;
    if (!encode_rows_f32_sw128(&c.tmap_e_tf32[0], emb, dd, rows, l, TSL, 1) ||
        !encode_rows_f32_sw128(&c.tmap_e_tf32[1], emb, dd, rows, l, TSL, 4) ||
        !encode_rows_f32_sw128(&c.tmap_e_tf32[2], emb, dd, rows, l, TSL, 32))
      return cudaErrorInvalidValue;
    c.tmap_e_tf32_ptr = emb;
    c.tmap_e_tf32_ld = ld;
  }
  return launch_k(trail_tf32_l1_kernel, dim3(c.H / TBM, tf32_splits(c)), dim3(TT), (size_t)TSMEM, s,
                  c.tmap_w_tf32, c.tmap_e_tf32[0], c.tmap_e_tf32[1], c.tmap_e_tf32[2],
                  c.tmap_xs_tf32[0], c.tmap_xs_tf32[1], c.tmap_xs_tf32[2], off, n, c.H, c.partial);
}

}  // namespace trail
