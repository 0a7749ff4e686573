// K2a — classifier layer 1 as a warp-per-output-slice split-K GEMV (row a2, small n and
// the fp32 configuration).
//
// P:201 "The first layer maps the input embedding to a 512-dimensional space, followed by
// a ReLU".  This kernel computes the pre-activation partial sums
//     partial[s][j][o] = sum_{k in split s} W1[o][k] * X[j][k]
// for every hidden unit o and request j; bias, ReLU and the deterministic (fixed-order)
// reduction over the S splits happen in the head kernel (K3).
//
// Layout: grid = (H / 16, S).  A CTA is 8 warps; warp w owns hidden rows
// o = 16*blockIdx.x + 2w, +1 and the K range of split s.  Lanes stride that range with
// 16-byte vectors of W1 (8 bf16 or 4 fp32), so each warp streams 512 contiguous bytes of
// each of its two W1 rows per iteration — W1 is read exactly once from HBM per step.
// The staged embeddings X (tiny in this regime) are re-read from L1/L2 per request tile of
// NT = 8 requests; each lane keeps 2 x 8 fp32 accumulators, reduced across the warp with
// shuffles at the end of the tile.  fp32 FFMA throughout (exact fp32 products for the
// fp32 configuration; bf16 inputs are widened exactly).
#include "trail_internal.cuh"

namespace trail {

namespace {
constexpr int kRowsPerWarp = 2;
constexpr int kWarps = 8;
constexpr int kRowsPerCta = kRowsPerWarp * kWarps;
constexpr int kNT = 8;

template <typename T>
struct V16;
template <>
struct V16<__nv_bfloat16> {
  static constexpr int N = 8;
  static __device__ __forceinline__ void ld(const __nv_bfloat16 *p, float f[8]) {
    uint4 u = __ldg(reinterpret_cast<const uint4 *>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};
template <>
struct V16<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void ld(const float *p, float f[4]) {
    float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  }
};
}  // namespace

template <typename T>
__global__ void __launch_bounds__(kWarps * 32)
trail_gemv_l1_kernel(const T *__restrict__ w1, const T *__restrict__ xs, int n, int d, int H,
                     int kchunk, float *__restrict__ partial) {
  constexpr int VEC = V16<T>::N;
  griddep_wait();
  griddep_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int o0 = blockIdx.x * kRowsPerCta + warp * kRowsPerWarp;
  const int s = blockIdx.y;
  const int kb = s * kchunk;
  const int ke = min(d, kb + kchunk);
  const T *wr0 = w1 + (int64_t)o0 * d;
  const T *wr1 = wr0 + d;
  float *out = partial + (int64_t)s * n * H;
  for (int j0 = 0; j0 < n; j0 += kNT) {
    float acc0[kNT], acc1[kNT];
#pragma unroll
    for (int t = 0; t < kNT; ++t) acc0[t] = acc1[t] = 0.f;
    for (int k = kb + lane * VEC; k < ke; k += 32 * VEC) {
      float a[VEC], b[VEC];
      V16<T>::ld(wr0 + k, a);
      V16<T>::ld(wr1 + k, b);
#pragma unroll
      for (int t = 0; t < kNT; ++t) {
        if (j0 + t < n) {
          float x[VEC];
          V16<T>::ld(xs + (int64_t)(j0 + t) * d + k, x);
#pragma unroll
          for (int i = 0; i < VEC; ++i) {
            acc0[t] = fmaf(a[i], x[i], acc0[t]);
            acc1[t] = fmaf(b[i], x[i], acc1[t]);
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kNT; ++t) {
      acc0[t] = warp_sum(acc0[t]);
      acc1[t] = warp_sum(acc1[t]);
    }
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < kNT; ++t) {
        if (j0 + t < n) {
          float2 v = make_float2(acc0[t], acc1[t]);
          *reinterpret_cast<float2 *>(out + (int64_t)(j0 + t) * H + o0) = v;
        }
      }
    }
  }
}

cudaError_t launch_gemv_l1(const Ctx &c, int n, int splits, cudaStream_t s) {
  const int vec = c.dtype == TRAIL_BF16 ? 8 : 4;
  // split length: multiple of one warp-iteration (32 vectors) where possible
  int kchunk = (c.d + splits - 1) / splits;
  kchunk = (kchunk + vec - 1) / vec * vec;
  dim3 grid(c.H / kRowsPerCta, splits);
  if (c.dtype == TRAIL_BF16)
    return launch_k(trail_gemv_l1_kernel<__nv_bfloat16>, grid, dim3(kWarps * 32), 0, s,
                    (const __nv_bfloat16 *)c.w1, (const __nv_bfloat16 *)c.xs, n, c.d, c.H, kchunk,
                    c.partial);
  return launch_k(trail_gemv_l1_kernel<float>, grid, dim3(kWarps * 32), 0, s, (const float *)c.w1,
                  (const float *)c.xs, n, c.d, c.H, kchunk, c.partial);
}

}  // namespace trail
