// K1c — chunked prefill (reading D-27).  With vLLM-style chunked prefill
// a prompt's rows arrive over several iterations; the pooled input is still the mean
// of ALL prompt rows ("averaging the embeddings of all the input tokens").  Each
// call adds a chunk's rows (fp32, row order) to a per-slot running sum + row count; for
// requests whose chunk is the last, the mean is written — rounded to bf16 (RNE) for bf16
// handles, reading D-12 — to the caller's `pooled` row j, which then enters
// trail_predict_step as a one-row prefill observation (gathered bit-exactly), and the slot's
// accumulator is cleared.  One thread per 16-byte column vector of a request: every
// (slot, column) has a single owner, so the accumulation order is the call order.
#include "trail_internal.cuh"

namespace trail {

namespace {
template <typename T>
struct CkIO;
template <>
struct CkIO<__nv_bfloat16> {
  static constexpr int V = 8;
  static __device__ __forceinline__ void add(const void *p, float (&f)[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4 *>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] += __uint_as_float(w[i] << 16);
      f[2 * i + 1] += __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
  static __device__ __forceinline__ void store(void *p, const float (&f)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t *>(&b);
    }
    *reinterpret_cast<uint4 *>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct CkIO<float> {
  static constexpr int V = 4;
  static __device__ __forceinline__ void add(const void *p, float (&f)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    f[0] += v.x; f[1] += v.y; f[2] += v.z; f[3] += v.w;
  }
  static __device__ __forceinline__ void store(void *p, const float (&f)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(f[0], f[1], f[2], f[3]);
  }
};
}  // namespace

template <typename T>
__global__ void __launch_bounds__(256)
trail_prefill_chunk_kernel(const T *__restrict__ emb, int64_t ld, const int32_t *__restrict__ off,
                           const uint32_t *__restrict__ ids, const uint8_t *__restrict__ is_final,
                           int n, int d, int max_slots, float *__restrict__ acc,
                           uint32_t *__restrict__ cnt, T *__restrict__ pooled, int64_t pld,
                           uint32_t *__restrict__ err) {
  using IO = CkIO<T>;
  constexpr int V = IO::V;
  griddep_wait();
  griddep_launch();
  const int j = blockIdx.x;
  const int v = blockIdx.y * blockDim.x + threadIdx.x;   // 16-byte column vector
  if (j >= n || v * V >= d) return;
  const uint32_t slot = __ldg(ids + j);
  const int r0 = __ldg(off + j), r1 = __ldg(off + j + 1);
  const bool fin = __ldg(is_final + j) != 0;
  if (slot >= (uint32_t)max_slots || r1 < r0) {
    if (threadIdx.x == 0 && blockIdx.y == 0)
      atomicOr(err, slot >= (uint32_t)max_slots ? TRAIL_DEV_BAD_ID : TRAIL_DEV_BAD_ROWS);
    return;
  }
  float s[V];
  float *a = acc + (int64_t)slot * d + v * V;
#pragma unroll
  for (int q = 0; q < V; ++q) s[q] = a[q];                // running sum of earlier chunks
  int r = r0;
  for (; r + 4 <= r1; r += 4) {                            // row order, 4 rows in flight
    float t0[V] = {}, t1[V] = {}, t2[V] = {}, t3[V] = {};
    IO::add(emb + (int64_t)r * ld + v * V, t0);
    IO::add(emb + (int64_t)(r + 1) * ld + v * V, t1);
    IO::add(emb + (int64_t)(r + 2) * ld + v * V, t2);
    IO::add(emb + (int64_t)(r + 3) * ld + v * V, t3);
#pragma unroll
    for (int q = 0; q < V; ++q) s[q] = (((s[q] + t0[q]) + t1[q]) + t2[q]) + t3[q];
  }
  for (; r < r1; ++r) IO::add(emb + (int64_t)r * ld + v * V, s);
  const uint32_t total = cnt[slot] + (uint32_t)(r1 - r0);
  if (fin) {
    float m[V];
    const float fc = (float)total;
#pragma unroll
    for (int q = 0; q < V; ++q) { m[q] = total ? __fdiv_rn(s[q], fc) : 0.f; a[q] = 0.f; }
    IO::store(pooled + (int64_t)j * pld + v * V, m);
  } else {
#pragma unroll
    for (int q = 0; q < V; ++q) a[q] = s[q];
  }
  // (the slot's row count is updated by the next, PDL-chained kernel, after every column
  // thread of this call has read the old count)
}

// the count update runs after every column of the call has read the old count
__global__ void trail_prefill_chunk_count_kernel(const int32_t *__restrict__ off,
                                                 const uint32_t *__restrict__ ids,
                                                 const uint8_t *__restrict__ is_final, int n,
                                                 int max_slots, uint32_t *__restrict__ cnt) {
  griddep_wait();
  griddep_launch();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t slot = __ldg(ids + j);
  const int r0 = __ldg(off + j), r1 = __ldg(off + j + 1);
  if (slot >= (uint32_t)max_slots || r1 < r0) return;
  cnt[slot] = __ldg(is_final + j) ? 0u : cnt[slot] + (uint32_t)(r1 - r0);
}

cudaError_t launch_prefill_chunk(Ctx &c, const void *emb, int64_t ld, const int32_t *off,
                                 const uint32_t *ids, const uint8_t *is_final, int n,
                                 void *pooled, int64_t pld, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (!c.chunk_acc) {   // lazily: [max_slots][d] fp32 sums + counts (synchronous, first use)
    if (cudaMalloc(&c.chunk_acc, (size_t)c.cfg.max_slots * c.d * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&c.chunk_cnt, (size_t)c.cfg.max_slots * sizeof(uint32_t)) != cudaSuccess)
      return cudaErrorMemoryAllocation;
    if (cudaMemset(c.chunk_acc, 0, (size_t)c.cfg.max_slots * c.d * sizeof(float)) != cudaSuccess ||
        cudaMemset(c.chunk_cnt, 0, (size_t)c.cfg.max_slots * sizeof(uint32_t)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
      return cudaErrorUnknown;
  }
  const int vec = c.dtype == TRAIL_BF16 ? 8 : 4;
  const int nv = c.d / vec;
  dim3 grid(n, (nv + 255) / 256);
  cudaError_t e;
  if (c.dtype == TRAIL_BF16)
    e = launch_k(trail_prefill_chunk_kernel<__nv_bfloat16>, grid, dim3(256), 0, s,
                 (const __nv_bfloat16 *)emb, ld, off, ids, is_final, n, c.d, c.cfg.max_slots,
                 c.chunk_acc, c.chunk_cnt, (__nv_bfloat16 *)pooled, pld, c.dev_err);
  else
    e = launch_k(trail_prefill_chunk_kernel<float>, grid, dim3(256), 0, s, (const float *)emb, ld,
                 off, ids, is_final, n, c.d, c.cfg.max_slots, c.chunk_acc, c.chunk_cnt,
                 (float *)pooled, pld, c.dev_err);
  if (e != cudaSuccess) return e;
  return launch_k(trail_prefill_chunk_count_kernel, dim3((n + 255) / 256), dim3(256), 0, s, off,
                  ids, is_final, n, c.cfg.max_slots, c.chunk_cnt);
}

}  // namespace trail
