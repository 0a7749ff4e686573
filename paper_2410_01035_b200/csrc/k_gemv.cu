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

// Register-tiled GEMV (the kernel K2a launches).  A CTA owns 64 hidden rows x the K range of
// its split; W1 is staged in shared memory "group-major": [K/G][64][G] with G = 16 B of
// elements (4 fp32 / 8 bf16) — by TMA (one 64-row x 16-byte box per
// group, issued by warp 0 before the PDL wait); X rows by 1-D bulk copies (one per request,
// from emb or xs) into a row-major layout whose row stride is an odd number of 16-byte units.
// 8 warps = 2 K halves x 4 warp tiles of 32 requests x 32 rows; lane = 4 requests x 8 rows
// (requests lq, lq+8, lq+16, lq+24 of its tile: the 8 lanes of a quarter-warp read 8
// consecutive X vectors, conflict-free; its 8 rows are a shared broadcast per quarter-warp).
// Per group a lane loads 4 X + 8 W1 vectors (12 LDS.128) for 32 G FFMAs — 2.8x fewer
// shared-memory wavefronts per FFMA than the 1-request-per-lane broadcast form — and the two
// K halves are added in a fixed order (deterministic).
constexpr int kGbRows = 64, kGbReq = 64;

template <typename T>
struct G16;   // one 16-byte group of elements
template <>
struct G16<float> {
  static constexpr int G = 4;
  static __device__ __forceinline__ void widen(const uint4 &u, float (&f)[4]) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
};
template <>
struct G16<__nv_bfloat16> {
  static constexpr int G = 8;
  static __device__ __forceinline__ void widen(const uint4 &u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};

template <typename T>
__global__ void __launch_bounds__(kWarps * 32, 1)
trail_gemv_l1_kernel(const __grid_constant__ CUtensorMap tmap_w, const T *__restrict__ emb,
                     int64_t ld, const int32_t *__restrict__ off, const T *__restrict__ xs, int n,
                     int d, int H, int kchunk, float *__restrict__ partial,
                     uint64_t *__restrict__ trace) {
  constexpr int G = G16<T>::G;
  // diagnostics (trail_trace_*): per-CTA phase timestamps, globaltimer ns
  uint64_t *tr = trace ? trace + 16 * (int64_t)(blockIdx.x + gridDim.x * blockIdx.y) : nullptr;
  auto stamp = [&](int i) {
    if (tr && threadIdx.x == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tr[i] = t;
    }
  };
  stamp(0);
  extern __shared__ __align__(128) uint8_t gsm[];
  __shared__ __align__(8) uint64_t s_bar, s_xbar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int o0 = blockIdx.x * kGbRows;
  const int s = blockIdx.y;
  const int kb = s * kchunk;
  const int kc = max(0, min(d, kb + kchunk) - kb);
  const int ng = kc / G;                                 // 16-byte groups of the K range
  uint8_t *wsm = gsm;                                    // [ng][64 rows][16 B]
  uint8_t *xsm = gsm + (size_t)ng * kGbRows * 16;        // [64 requests][XS]
  int64_t *src = reinterpret_cast<int64_t *>(xsm + (size_t)kGbReq * (((kchunk * (int)sizeof(T) / 16) | 1) * 16));
  float *red = reinterpret_cast<float *>(src + kGbReq);  // [4 tiles][32 acc][32 lanes]
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
  const uint32_t xbar = (uint32_t)__cvta_generic_to_shared(&s_xbar);
  // X is row-major [64 requests][XS bytes], XS an odd number of 16-byte units (the 8 lanes of
  // a quarter-warp read 8 consecutive requests at the same K: conflict-free)
  const int XS = ((kc * (int)sizeof(T) / 16) | 1) * 16;
  // W1 slice: a weight, independent of earlier kernels — TMA boxes in flight before the PDL wait
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(xbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((uint32_t)(ng * kGbRows * 16))
                 : "memory");
  }
  __syncwarp();
  if (warp == 0) {   // the TMA boxes issued by the 32 lanes of warp 0
    for (int g = lane; g < ng; g += 32)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"((uint32_t)__cvta_generic_to_shared(wsm + (size_t)g * kGbRows * 16)),
          "l"(reinterpret_cast<uint64_t>(&tmap_w)), "r"(bar), "r"(kb + g * G), "r"(o0)
          : "memory");
  }
  // X row of request j (row a1): a decode request's single row straight from the caller's
  // embeddings (bit-exact), a prompt's mean from xs (K1).  Only the latter
  // depends on the previous kernel: decode-only steps start without waiting for K1 (PDL).
  bool pooled = false;
  for (int j = tid; j < n; j += blockDim.x) pooled |= __ldg(off + j + 1) - __ldg(off + j) != 1;
  stamp(1);
  if (__syncthreads_or(pooled)) griddep_wait();
  griddep_launch();
  stamp(2);
  float *out = partial + (int64_t)s * n * H;
  const int kh = warp >> 2, tw = warp & 3;               // K half, warp tile
  const int rq = tw & 1, rr = tw >> 1;                    // 32-request group, 32-row group
  const int lq = lane & 7, lr = lane >> 3;
  const int ga = kh ? ng / 2 : 0, gb = kh ? ng : ng / 2;
  bool w_ready = false;
  for (int j0 = 0; j0 < n; j0 += kGbReq) {
    const int nb = min(kGbReq, n - j0);
    __syncthreads();                                     // previous block's X reads done
    for (int t = tid; t < nb; t += blockDim.x) {
      const int j = j0 + t;
      const int a = __ldg(off + j), b = __ldg(off + j + 1);
      src[t] = b - a == 1 ? (int64_t)a * ld : -1 - (int64_t)j * d;
    }
    __syncthreads();
    // X rows: one 1-D bulk copy per request (kc elements), issued by warp 0's lanes
    if (tid == 0 && kc > 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(xbar),
                   "r"((uint32_t)(nb * kc * (int)sizeof(T)))
                   : "memory");
    else if (tid == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(xbar) : "memory");
    __syncwarp();
    if (warp == 0 && kc > 0)
      for (int t = lane; t < nb; t += 32) {
        const int64_t sj = src[t];
        const T *p = (sj >= 0 ? emb + sj : xs + (-1 - sj)) + kb;
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(xsm + (size_t)t * XS)), "l"(p),
                     "r"((uint32_t)(kc * (int)sizeof(T))), "r"(xbar)
                     : "memory");
      }
    stamp(3);
    {
      const uint32_t xph = (uint32_t)((j0 / kGbReq) & 1);
      uint32_t ok = 0;
      do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(xbar), "r"(xph) : "memory");
      } while (!ok);
    }
    if (!w_ready) {
      uint32_t ok = 0;
      do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(bar) : "memory");
      } while (!ok);
      w_ready = true;
    }
    __syncthreads();
    stamp(4);
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[i][r] = 0.f;
    const uint8_t *xp = xsm + (size_t)(rq * 32 + lq) * XS;
    const uint8_t *wp = wsm + (size_t)(rr * 32 + lr * 8) * 16;
#pragma unroll 2
    for (int g = ga; g < gb; ++g) {
      float x[4][G], w[8][G];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        G16<T>::widen(*reinterpret_cast<const uint4 *>(xp + (size_t)(8 * i) * XS + (size_t)g * 16), x[i]);
#pragma unroll
      for (int r = 0; r < 8; ++r)
        G16<T>::widen(*reinterpret_cast<const uint4 *>(wp + ((size_t)g * kGbRows + r) * 16), w[r]);
#pragma unroll
      for (int e = 0; e < G; ++e)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int r = 0; r < 8; ++r) acc[i][r] = fmaf(w[r][e], x[i][e], acc[i][r]);
    }
    if (kh) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int r = 0; r < 8; ++r) red[((tw * 4 + i) * 8 + r) * 32 + lane] = acc[i][r];
    }
    __syncthreads();
    if (!kh) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int t = rq * 32 + 8 * i + lq;
        if (t < nb) {
          float v[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) v[r] = acc[i][r] + red[((tw * 4 + i) * 8 + r) * 32 + lane];
          float4 *dst = reinterpret_cast<float4 *>(out + (int64_t)(j0 + t) * H + o0 + rr * 32 + lr * 8);
          dst[0] = make_float4(v[0], v[1], v[2], v[3]);
          dst[1] = make_float4(v[4], v[5], v[6], v[7]);
        }
      }
    }
  }
  __syncthreads();
  stamp(5);
}

cudaError_t launch_gemv_l1(const Ctx &c, const void *emb, int64_t ld, const int32_t *off, int n,
                           int splits, cudaStream_t s) {
  if (!c.have_tmap_gemv) return cudaErrorInvalidValue;
  const int G = c.dtype == TRAIL_BF16 ? 8 : 4;
  // split length: a multiple of one 16-byte group
  const int kchunk = ((c.d + splits - 1) / splits + G - 1) / G * G;
  dim3 grid(c.H / kGbRows, splits);
  const size_t smem = (size_t)kGbRows * kchunk * c.esize +
                      (size_t)kGbReq * (((kchunk * c.esize / 16) | 1) * 16) + kGbReq * 8 +
                      (size_t)4 * 32 * 32 * sizeof(float);
  if (smem > (size_t)kGemvSmemMax) return cudaErrorInvalidValue;
  uint64_t *tr = (c.trace && (int)(grid.x * grid.y) <= c.trace_cap) ? c.trace : nullptr;
  if (c.dtype == TRAIL_BF16)
    return launch_k(trail_gemv_l1_kernel<__nv_bfloat16>, grid, dim3(kWarps * 32), smem, s,
                    c.tmap_w_gemv, (const __nv_bfloat16 *)emb, ld, off,
                    (const __nv_bfloat16 *)c.xs, n, c.d, c.H, kchunk, c.partial, tr);
  return launch_k(trail_gemv_l1_kernel<float>, grid, dim3(kWarps * 32), smem, s, c.tmap_w_gemv,
                  (const float *)emb, ld, off, (const float *)c.xs, n, c.d, c.H, kchunk, c.partial,
                  tr);
}

cudaError_t gemv_prepare(Ctx &c) {
  const uint32_t G = c.dtype == TRAIL_BF16 ? 8 : 4;
  c.have_tmap_gemv = encode_plain_2d(&c.tmap_w_gemv, c.w1, c.dtype == TRAIL_BF16, (uint64_t)c.d,
                                     (uint64_t)c.H, (uint64_t)c.d, G, kGbRows);
  if (!c.have_tmap_gemv) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(trail_gemv_l1_kernel<float>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvSmemMax);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(trail_gemv_l1_kernel<__nv_bfloat16>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, kGemvSmemMax);
}

}  // namespace trail
