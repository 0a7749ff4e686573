// K2a — classifier layer 1 as a warp-per-output-slice split-K GEMV (row a2, small n and
// the fp32 configuration).
//
// P:201 "The first layer maps the input embedding to a 512-dimensional space, followed by
// a ReLU".  This kernel computes the pre-activation partial sums
//     partial[s][j][o] = sum_{k in split s} W1[o][k] * X[j][k]
// for every hidden unit o and request j; bias, ReLU and the deterministic (fixed-order)
// reduction over the S splits happen in the head kernel (K3).
//
// Layout: grid = (H / 64, S), ~one CTA per SM.  CUDA cores, fp32 FFMA throughout (exact
// fp32 products for the fp32 configuration; bf16 inputs are widened exactly).  In this
// regime (configs[0]: n = 64, fp32 W1 of 8 MB) the contraction is FFMA-bound, not HBM-bound:
// 2 n d H = 268 MFLOP against ~74 TFLOP/s of fp32 FMA.
#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int kWarps = 8;
constexpr int kGemvSmemMax = 200 * 1024;   // W1 + X slices staged in shared memory
}  // namespace

// Broadcast GEMV (the kernel K2a launches): no cross-lane reduction at all.  A CTA owns 64
// hidden rows x the K range of its split and stages both operand slices in shared memory with
// cp.async; lane = request, warp = (request group of 32, 16 rows).  Shared memory is K4-major
// — [K/4][64 rows][4 elements] for W1 and [K/4][64 requests][4 elements] for X — so for each
// group of 4 K columns a lane reads its X vector (lanes consecutive: conflict-free) and the 16
// W1 vectors its warp shares (broadcast) at compile-time offsets from one moving pointer,
// then issues 64 FFMAs: 17 LDS per 64 FFMA and no address arithmetic in the loop.
constexpr int kGbRows = 64, kGbReq = 64, kGbRpw = 16;

template <typename T>
struct Q4;   // 4 consecutive elements
template <>
struct Q4<float> {
  using V = uint4;
  static __device__ __forceinline__ void widen(const V &u, float (&f)[4]) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
};
template <>
struct Q4<__nv_bfloat16> {
  using V = uint2;
  static __device__ __forceinline__ void widen(const V &u, float (&f)[4]) {
    f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xFFFF0000u);
    f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xFFFF0000u);
  }
};

// copy 4 consecutive elements (16 B fp32 / 8 B bf16) global -> shared, asynchronously
template <typename T>
__device__ __forceinline__ void cp4(void *dst, const T *src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  if (sizeof(T) == 4)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(kWarps * 32, 1)
trail_gemv_l1_kernel(const T *__restrict__ w1, const T *__restrict__ emb, int64_t ld,
                     const int32_t *__restrict__ off, const T *__restrict__ xs, int n, int d, int H,
                     int kchunk, float *__restrict__ partial) {
  using V = typename Q4<T>::V;
  constexpr int QB = 4 * (int)sizeof(T);                 // bytes of one 4-element group
  extern __shared__ __align__(16) uint8_t gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int o0 = blockIdx.x * kGbRows;
  const int s = blockIdx.y;
  const int kb = s * kchunk;
  const int kc = max(0, min(d, kb + kchunk) - kb);
  const int nq = kc / 4;                                 // 4-element groups of the K range
  uint8_t *wsm = gsm;                                    // [nq][64][QB]
  uint8_t *xsm = gsm + (size_t)nq * kGbRows * QB;        // [nq][64][QB]
  int64_t *src = reinterpret_cast<int64_t *>(xsm + (size_t)nq * kGbReq * QB);   // [64]
  // W1 slice: a weight, independent of earlier kernels — in flight before the PDL wait
  for (int r = warp; r < kGbRows; r += kWarps)          // a warp per row: coalesced reads
    for (int q = lane; q < nq; q += 32)
      cp4<T>(wsm + ((size_t)q * kGbRows + r) * QB, w1 + (int64_t)(o0 + r) * d + kb + 4 * q);
  asm volatile("cp.async.commit_group;" ::: "memory");
  // X row of request j (row a1): a decode request's single row straight from the caller's
  // embeddings (bit-exact), a prompt's mean from xs (K1).  Only the latter
  // depends on the previous kernel: decode-only steps start without waiting for K1 (PDL).
  bool pooled = false;
  for (int j = tid; j < n; j += blockDim.x) pooled |= __ldg(off + j + 1) - __ldg(off + j) != 1;
  if (__syncthreads_or(pooled)) griddep_wait();
  griddep_launch();
  float *out = partial + (int64_t)s * n * H;
  const int rg = warp >> 1;                              // 16-row group of this warp
  for (int j0 = 0; j0 < n; j0 += kGbReq) {
    const int nb = min(kGbReq, n - j0);
    __syncthreads();                                     // previous block's X reads done
    for (int t = tid; t < nb; t += blockDim.x) {
      const int j = j0 + t;
      const int a = __ldg(off + j), b = __ldg(off + j + 1);
      src[t] = b - a == 1 ? (int64_t)a * ld : -1 - (int64_t)j * d;
    }
    __syncthreads();
    for (int t = warp; t < nb; t += kWarps) {
      const int64_t sj = src[t];
      const T *p = (sj >= 0 ? emb + sj : xs + (-1 - sj)) + kb;
      for (int q = lane; q < nq; q += 32) cp4<T>(xsm + ((size_t)q * kGbReq + t) * QB, p + 4 * q);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int t = (warp & 1) * 32 + lane;                // my request in the block
    const uint8_t *xp = xsm + (size_t)min(t, nb - 1) * QB;
    const uint8_t *wp = wsm + (size_t)rg * kGbRpw * QB;
    float acc[kGbRpw];
#pragma unroll
    for (int r = 0; r < kGbRpw; ++r) acc[r] = 0.f;
    // software pipeline: group q + 1's 17 vectors are loaded while group q's 64 FFMAs issue
    V xv = *reinterpret_cast<const V *>(xp), wv[kGbRpw];
#pragma unroll
    for (int r = 0; r < kGbRpw; ++r) wv[r] = *reinterpret_cast<const V *>(wp + r * QB);
    for (int q = 0; q < nq; ++q) {
      const int qn = q + 1 < nq ? q + 1 : q;
      const V xn = *reinterpret_cast<const V *>(xp + (size_t)qn * kGbReq * QB);
      V wn[kGbRpw];
      const uint8_t *wq = wp + (size_t)qn * kGbRows * QB;
#pragma unroll
      for (int r = 0; r < kGbRpw; ++r) wn[r] = *reinterpret_cast<const V *>(wq + r * QB);
      float x[4];
      Q4<T>::widen(xv, x);
#pragma unroll
      for (int r = 0; r < kGbRpw; ++r) {
        float w[4];
        Q4<T>::widen(wv[r], w);
        acc[r] = fmaf(w[0], x[0], acc[r]);
        acc[r] = fmaf(w[1], x[1], acc[r]);
        acc[r] = fmaf(w[2], x[2], acc[r]);
        acc[r] = fmaf(w[3], x[3], acc[r]);
      }
      xv = xn;
#pragma unroll
      for (int r = 0; r < kGbRpw; ++r) wv[r] = wn[r];
    }
    if (t < nb) {
      float4 *dst = reinterpret_cast<float4 *>(out + (int64_t)(j0 + t) * H + o0 + rg * kGbRpw);
#pragma unroll
      for (int q = 0; q < kGbRpw / 4; ++q)
        dst[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
    }
  }
}

cudaError_t launch_gemv_l1(const Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                           int splits, cudaStream_t s) {
  // split length: a multiple of 8 elements (16-byte copies for bf16 and fp32)
  const int kchunk = ((c.d + splits - 1) / splits + 7) / 8 * 8;
  dim3 grid(c.H / kGbRows, splits);
  const size_t smem = (size_t)(kGbRows + kGbReq) * kchunk * c.esize + kGbReq * 8;
  if (smem > (size_t)kGemvSmemMax) return cudaErrorInvalidValue;
  if (c.dtype == TRAIL_BF16)
    return launch_k(trail_gemv_l1_kernel<__nv_bfloat16>, grid, dim3(kWarps * 32), smem, s,
                    (const __nv_bfloat16 *)c.w1, (const __nv_bfloat16 *)emb, ld, off,
                    (const __nv_bfloat16 *)c.xs, n, c.d, c.H, kchunk, c.partial);
  return launch_k(trail_gemv_l1_kernel<float>, grid, dim3(kWarps * 32), smem, s, (const float *)c.w1,
                  (const float *)emb, ld, off, (const float *)c.xs, n, c.d, c.H, kchunk, c.partial);
}

cudaError_t gemv_prepare() {
  cudaError_t e = cudaFuncSetAttribute(trail_gemv_l1_kernel<float>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvSmemMax);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(trail_gemv_l1_kernel<__nv_bfloat16>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvSmemMax);
}

}  // namespace trail
