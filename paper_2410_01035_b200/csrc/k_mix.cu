// K1m — multi-layer weighted embeddings ("a weighted average of their
// outputs", "leveraging multiple-layer embeddings through weighted averaging"; reading
// D-28).  u_j = sum_l a_l u_{l,j} with a = w / sum(w), u_{l,j} = the mean of request j's rows
// of layer l (its prompt at prefill; its single row at decode).  One thread per 16-byte
// column vector of a request: fp64 sums over the rows of each layer in row order (exact for
// bf16 inputs), divided by the row count, scaled by a_l and added in layer order in fp64, then
// rounded ONCE to bf16 (RNE) for bf16 handles (D-12) — every decode row is such a rounded
// mix, so an fp32 intermediate would flip an occasional bf16 ulp against the fp64 definition
// (measured: 1.1e-3 relative in L on a 4-layer case); fp64 arithmetic is free here.
// HBM-bound: reads L x rows x d elements, writes n x d.
#include "trail_internal.cuh"

namespace trail {

namespace {
template <typename T>
struct MxIO;
template <>
struct MxIO<__nv_bfloat16> {
  static constexpr int V = 8;
  static __device__ __forceinline__ void add(const void *p, double (&f)[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4 *>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] += (double)__uint_as_float(w[i] << 16);
      f[2 * i + 1] += (double)__uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
  static __device__ __forceinline__ void store(void *p, const double (&f)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {     // fp64 -> bf16 in one rounding (RNE)
      const __nv_bfloat16 lo = __double2bfloat16(f[2 * i]), hi = __double2bfloat16(f[2 * i + 1]);
      w[i] = (uint32_t)*reinterpret_cast<const uint16_t *>(&lo) |
             ((uint32_t)*reinterpret_cast<const uint16_t *>(&hi) << 16);
    }
    *reinterpret_cast<uint4 *>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct MxIO<float> {
  static constexpr int V = 4;
  static __device__ __forceinline__ void add(const void *p, double (&f)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    f[0] += v.x; f[1] += v.y; f[2] += v.z; f[3] += v.w;
  }
  static __device__ __forceinline__ void store(void *p, const double (&f)[4]) {
    *reinterpret_cast<float4 *>(p) =
        make_float4(__double2float_rn(f[0]), __double2float_rn(f[1]), __double2float_rn(f[2]),
                    __double2float_rn(f[3]));
  }
};
}  // namespace

template <typename T>
__global__ void __launch_bounds__(256)
trail_layer_mix_kernel(MixArgs ma, int64_t ld, const int32_t *__restrict__ off, int n, int d,
                       T *__restrict__ out, uint32_t *__restrict__ err) {
  using IO = MxIO<T>;
  constexpr int V = IO::V;
  griddep_wait();
  griddep_launch();
  const int j = blockIdx.x;
  const int v = blockIdx.y * blockDim.x + threadIdx.x;   // 16-byte column vector
  if (j >= n || v * V >= d) return;
  const int r0 = __ldg(off + j), r1 = __ldg(off + j + 1);
  double acc[V];
#pragma unroll
  for (int q = 0; q < V; ++q) acc[q] = 0.0;
  if (r1 <= r0) {
    if (threadIdx.x == 0 && blockIdx.y == 0) atomicOr(err, TRAIL_DEV_BAD_ROWS);
    IO::store(out + (int64_t)j * d + v * V, acc);
    return;
  }
  const double cnt = (double)(r1 - r0);
  for (int l = 0; l < ma.L; ++l) {
    const T *e = reinterpret_cast<const T *>(ma.emb[l]);
    double s[V];
#pragma unroll
    for (int q = 0; q < V; ++q) s[q] = 0.0;
    for (int r = r0; r < r1; ++r) IO::add(e + (int64_t)r * ld + v * V, s);
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] += ma.a[l] * (s[q] / cnt);   // a_l * mean_l (oracle order)
  }
  IO::store(out + (int64_t)j * d + v * V, acc);
}

cudaError_t launch_layer_mix(Ctx &c, const MixArgs &ma, int64_t ld, const int32_t *off, int n,
                             cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int vec = c.dtype == TRAIL_BF16 ? 8 : 4;
  dim3 grid(n, (c.d / vec + 255) / 256);
  if (c.dtype == TRAIL_BF16)
    return launch_k(trail_layer_mix_kernel<__nv_bfloat16>, grid, dim3(256), 0, s, ma, ld, off, n,
                    c.d, (__nv_bfloat16 *)c.xmix, c.dev_err);
  return launch_k(trail_layer_mix_kernel<float>, grid, dim3(256), 0, s, ma, ld, off, n, c.d,
                  (float *)c.xmix, c.dev_err);
}

}  // namespace trail
