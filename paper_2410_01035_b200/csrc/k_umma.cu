// K2b — classifier layer 1 on the 5th-generation tensor cores (row a2, bf16, large n).
//
// P:201 "The first layer maps the input embedding to a 512-dimensional space": with n
// requests this is the dense contraction D[n][H] = X[n][d] . W1[H][d]^T (a "TN" GEMM, both
// operands K-major).  One CTA computes a 128 x BN tile (BN = 128 or 256 hidden units) over
// the K range of its split s (grid = m_tiles x H/BN x S, sized to one wave of the 148 SMs):
//   warp 0 / lane 0 : TMA producer — cp.async.bulk.tensor 2-D loads of a 128x64 X tile and a
//                     BNx64 W1 tile per stage into 128-byte-swizzled shared memory, arriving
//                     on the stage's mbarrier with complete_tx;
//   warp 1 / lane 0 : MMA issuer — tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32,
//                     M=128, N=BN, K=16) x 4 per stage into a TMEM accumulator of BN columns;
//                     tcgen05.commit frees the stage, and a final commit signals the epilogue;
//   warps 0-3       : epilogue — tcgen05.ld 32x32b.x32 (warp w owns TMEM lanes 32w..32w+31 =
//                     tile rows), fp32 partial sums written to partial[s][row][n0 + col].
// Bias, ReLU and the fixed-order reduction over splits are fused into the head kernel K3,
// which keeps h in fp32 (D-22 note: rounding h to bf16 breaks the 2e-3 posterior bound).
#include <stdio.h>

#include "sm100_ptx.cuh"
#include "trail_internal.cuh"

namespace trail {

using namespace ptx;   // mbarrier / TMA / tcgen05 wrappers shared with K2c and K2d

namespace {
constexpr int BM = 128;
constexpr int BK = 64;   // one 128-byte swizzle atom of bf16 per row

template <int BN>
struct UCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_BYTES = 256;
  static constexpr int SMEM = STAGES * STAGE_BYTES + BAR_BYTES + 1024;
};

}  // namespace

template <int BN>
__global__ void __launch_bounds__(128, 1)
trail_umma_l1_kernel(const __grid_constant__ CUtensorMap tmap_x,
                     const __grid_constant__ CUtensorMap tmap_w, int n, int H, int kblocks,
                     int splits, float *__restrict__ partial) {
  using C = UCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::STAGES * C::A_BYTES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + C::STAGES * C::B_BYTES);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * C::STAGES + 1);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + C::STAGES),
                 done = smem_u32(bars + 2 * C::STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN, s = blockIdx.z;
  const int kb0 = (int)((int64_t)s * kblocks / splits);
  const int kb1 = (int)((int64_t)(s + 1) * kblocks / splits);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_w)) : "memory");
  }
  if (warp == 0) {  // whole warp: allocate BN fp32 columns of tensor memory
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
  griddep_wait();      // X is produced by the pool kernel
  griddep_launch();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int i = 0; i < nkb; ++i) {
      const int st = i % C::STAGES;
      const uint32_t ph = (uint32_t)(i / C::STAGES) & 1u;
      mbar_wait(empty0 + 8 * st, ph ^ 1u);
      mbar_expect_tx(full0 + 8 * st, C::STAGE_BYTES);
      const int kc = (kb0 + i) * BK;
      tma_load_2d(smem_u32(sA + st * C::A_BYTES), &tmap_x, full0 + 8 * st, kc, m0);
      tma_load_2d(smem_u32(sB + st * C::B_BYTES), &tmap_w, full0 + 8 * st, kc, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread)
    constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
    for (int i = 0; i < nkb; ++i) {
      const int st = i % C::STAGES;
      const uint32_t ph = (uint32_t)(i / C::STAGES) & 1u;
      mbar_wait(full0 + 8 * st, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t da = sw128_kmajor_desc(smem_u32(sA + st * C::A_BYTES));
      const uint64_t db = sw128_kmajor_desc(smem_u32(sB + st * C::B_BYTES));
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk)   // +32 bytes along K inside the swizzle atom
        umma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : 0u);
      umma_commit(empty0 + 8 * st);
    }
    umma_commit(done);
  }
  // ---------------- epilogue: TMEM -> registers -> fp32 partials
  mbar_wait(done, 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // Stage each warp's 32 rows through (now idle) pipeline shared memory, then write them
  // out row by row: one 16-byte vector per lane, BN*4 contiguous bytes per row (coalesced).
  constexpr int LD = BN + 4;                       // padded row stride (floats)
  float *stile = reinterpret_cast<float *>(smem) + warp * 32 * LD;
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, r);
    float4 *srow = reinterpret_cast<float4 *>(stile + lane * LD + c);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      srow[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                            __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
  }
  __syncwarp();
  const int row0 = m0 + warp * 32;
#pragma unroll 4
  for (int rr = 0; rr < 32; ++rr) {
    if (row0 + rr >= n) break;
    float *dst = partial + ((int64_t)s * n + row0 + rr) * H + n0;
    const float *src = stile + rr * LD;
#pragma unroll
    for (int c = lane * 4; c < BN; c += 128)
      *reinterpret_cast<float4 *>(dst + c) = *reinterpret_cast<const float4 *>(src + c);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"((uint32_t)BN)
                 : "memory");
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

// bf16 row-major [rows][ld] (cols used), SWIZZLE_128B boxes of box_cols x box_rows
bool encode_rows_bf16(CUtensorMap *m, const void *base, uint64_t cols, uint64_t rows, uint64_t ld,
                      uint32_t box_cols, uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// fp32 row-major [rows][ld] (cols used), SWIZZLE_128B boxes of box_cols (<= 32) x box_rows (K2t)
bool encode_rows_f32_sw128(CUtensorMap *m, const void *base, uint64_t cols, uint64_t rows,
                           uint64_t ld, uint32_t box_cols, uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// plain (no swizzle) 2-D map of a row-major [rows][ld] fp32/bf16 matrix, boxes box_cols x box_rows
bool encode_plain_2d(CUtensorMap *m, const void *base, bool bf16, uint64_t cols, uint64_t rows,
                     uint64_t ld, uint32_t box_cols, uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  const uint64_t es = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * es};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t el[2] = {1, 1};
  CUresult r = enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void *>(base), dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static bool encode_2d_bf16(CUtensorMap *m, const void *base, uint64_t inner, uint64_t outer,
                           uint32_t box_inner, uint32_t box_outer) {
  return encode_rows_bf16(m, base, inner, outer, inner, box_inner, box_outer);
}

cudaError_t umma_prepare(Ctx &c) {
  if (c.dtype != TRAIL_BF16) return cudaSuccess;
  if (!encode_2d_bf16(&c.tmap_x, c.xs, (uint64_t)c.d, (uint64_t)c.cfg.max_requests, BK, BM) ||
      !encode_2d_bf16(&c.tmap_w128, c.w1, (uint64_t)c.d, (uint64_t)c.H, BK, 128) ||
      (c.H % 256 == 0 &&
       !encode_2d_bf16(&c.tmap_w256, c.w1, (uint64_t)c.d, (uint64_t)c.H, BK, 256)))
    return cudaErrorInvalidValue;
  const uint64_t xr = (uint64_t)c.cfg.max_requests;
  if (!encode_rows_bf16(&c.tmap_xs1, c.xs, (uint64_t)c.d, xr, (uint64_t)c.d, BK, 1) ||
      !encode_rows_bf16(&c.tmap_xs4, c.xs, (uint64_t)c.d, xr, (uint64_t)c.d, BK, 4) ||
      !encode_rows_bf16(&c.tmap_xs32, c.xs, (uint64_t)c.d, xr, (uint64_t)c.d, BK, 32))
    return cudaErrorInvalidValue;
  c.have_tmaps = true;
  cudaError_t e = cudaFuncSetAttribute(trail_umma_l1_kernel<128>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, UCfg<128>::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(trail_umma_l1_kernel<256>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, UCfg<256>::SMEM);
}

int umma_max_bn(const Ctx &c) { return c.H % 256 == 0 ? 256 : 128; }

cudaError_t launch_umma_l1(const Ctx &c, int n, int bn, int splits, cudaStream_t s) {
  if (!c.have_tmaps) return cudaErrorInvalidValue;
  const int kblocks = c.d / BK;
  dim3 grid((n + BM - 1) / BM, c.H / bn, splits);
  if (bn == 256)
    return launch_k(trail_umma_l1_kernel<256>, grid, dim3(128), UCfg<256>::SMEM, s, c.tmap_x,
                    c.tmap_w256, n, c.H, kblocks, splits, c.partial);
  return launch_k(trail_umma_l1_kernel<128>, grid, dim3(128), UCfg<128>::SMEM, s, c.tmap_x,
                  c.tmap_w128, n, c.H, kblocks, splits, c.partial);
}

}  // namespace trail
