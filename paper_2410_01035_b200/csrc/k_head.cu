// K3 — warp-per-request head (row a3): split-K reduction + bias + ReLU (end of layer 1),
// layer 2, softmax, Bayesian refinement, renormalisation, expected length, state update.
//
//   h      = max(0, sum_s partial[s][j] + b1)                     P:201 (ReLU), fp32
//   z      = W2 h + b2 ;  log p = z - logsumexp(z)                 P:201, P:204 (D-6)
//   first observation (prefill, or an unseen slot, D-23):
//     log q = log p + log pi - logsumexp(.)                        P:219 (uniform pi: q = p)
//     r = m[argmax q] (lowest index on ties), thr = floor(c r), a = 0       P:394, D-9, D-10
//   decode:
//     log prior(i) = logaddexp(log(1-1/w_i) + lq(i), log(1/w_{i+1}) + lq(i+1))  P:216, D-1/D-2
//     log q = log prior + log p - logsumexp(.)
//     a = a + 1                                                    D-11
//   L = sum_i exp(lq(i)) m_i
//
// The state is the LOG posterior in fp32 (reading D-22): the same real-number recursion as
// P:220-222 without the underflow of a linear fp32 filter under confident, contradictory
// observations.  Lane i of the warp owns bin i (k <= 32); the 512 hidden values are spread
// 16 per lane as 4 float4 chunks (coalesced 512-byte rows of the partials).  W2 is staged
// in shared memory once per CTA; the reduction over splits runs in a fixed order, so
// results are bit-reproducible.
#include <math.h>

#include "trail_internal.cuh"

namespace trail {

namespace {
__device__ __forceinline__ float logaddexp_f(float a, float b) {
  const float mx = fmaxf(a, b), mn = fminf(a, b);
  if (mx == -INFINITY) return -INFINITY;
  return mx + log1pf(expf(mn - mx));
}
}  // namespace

template <int HC>  // hidden = 128 * HC
__global__ void __launch_bounds__(256)
trail_head_kernel(const float *__restrict__ partial, int splits, int n,
                  const float *__restrict__ b1, const float *__restrict__ w2,
                  const float *__restrict__ b2, const HeadConsts *__restrict__ cst,
                  const uint32_t *__restrict__ ids, const uint8_t *__restrict__ is_prefill,
                  const float *__restrict__ prior_override, int max_slots,
                  float *__restrict__ lq_state, SlotMeta *__restrict__ meta,
                  float *__restrict__ post, float *__restrict__ Lout, uint32_t *__restrict__ err) {
  constexpr int H = 128 * HC;
  extern __shared__ float w2s[];  // [k][H]
  const int k = cst->k;
  for (int i = threadIdx.x; i < k * H / 4; i += blockDim.x)
    reinterpret_cast<float4 *>(w2s)[i] = __ldg(reinterpret_cast<const float4 *>(w2) + i);
  __syncthreads();
  griddep_wait();      // partials from layer 1, slot state from the previous step
  griddep_launch();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool active = lane < k;
  const float m_i = active ? cst->m[lane] : 0.f;
  const float lstay = active ? cst->log_stay[lane] : -INFINITY;
  const float lmove = active ? cst->log_move[lane] : -INFINITY;
  const float lpi = active ? cst->log_prior[lane] : -INFINITY;
  const float bias2 = active ? __ldg(b2 + lane) : 0.f;
  float4 bias1[HC];
#pragma unroll
  for (int c = 0; c < HC; ++c)
    bias1[c] = __ldg(reinterpret_cast<const float4 *>(b1 + c * 128) + lane);

  const int warps_total = gridDim.x * (blockDim.x >> 5);
  for (int j = blockIdx.x * (blockDim.x >> 5) + warp; j < n; j += warps_total) {
    const uint32_t slot = __ldg(ids + j);
    if (slot >= (uint32_t)max_slots) {
      if (lane == 0) atomicOr(err, TRAIL_DEV_BAD_ID);
      if (active && post) post[(int64_t)j * k + lane] = NAN;
      if (lane == 0 && Lout) Lout[j] = NAN;
      continue;
    }
    // ---- h = ReLU(sum_s partial + b1), fixed split order
    float4 h[HC];
#pragma unroll
    for (int c = 0; c < HC; ++c) h[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < splits; ++s) {
      const float4 *src = reinterpret_cast<const float4 *>(partial + ((int64_t)s * n + j) * H);
#pragma unroll
      for (int c = 0; c < HC; ++c) {
        const float4 v = __ldcs(src + c * 32 + lane);
        h[c].x += v.x; h[c].y += v.y; h[c].z += v.z; h[c].w += v.w;
      }
    }
#pragma unroll
    for (int c = 0; c < HC; ++c) {
      h[c].x = fmaxf(h[c].x + bias1[c].x, 0.f);
      h[c].y = fmaxf(h[c].y + bias1[c].y, 0.f);
      h[c].z = fmaxf(h[c].z + bias1[c].z, 0.f);
      h[c].w = fmaxf(h[c].w + bias1[c].w, 0.f);
    }
    // ---- z = W2 h + b2 ; lane b keeps z_b
    float z = -INFINITY;
    for (int b = 0; b < k; ++b) {
      const float4 *wr = reinterpret_cast<const float4 *>(w2s + b * H);
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < HC; ++c) {
        const float4 w = wr[c * 32 + lane];
        acc = fmaf(w.x, h[c].x, acc);
        acc = fmaf(w.y, h[c].y, acc);
        acc = fmaf(w.z, h[c].z, acc);
        acc = fmaf(w.w, h[c].w, acc);
      }
      acc = warp_sum(acc);
      if (lane == b) z = acc + bias2;
    }
    // ---- log-softmax over the k lanes
    const float zmax = warp_max(z);
    const float se = warp_sum(active ? expf(z - zmax) : 0.f);
    const float logp = active ? z - zmax - logf(se) : -INFINITY;

    SlotMeta mt = meta[slot];
    const bool seen = (mt.flags & 1u) != 0u;
    const bool first = (__ldg(is_prefill + j) != 0) || !seen;
    float lq;
    if (first) {
      float lp = lpi;
      if (prior_override) lp = active ? logf(__ldg(prior_override + (int64_t)j * k + lane)) : -INFINITY;
      lq = logp + lp;
    } else {
      const float prev = active ? lq_state[(int64_t)slot * k + lane] : -INFINITY;
      const float next = __shfl_down_sync(0xffffffffu, prev, 1);
      const float lprior = logaddexp_f(lstay + prev, (lane + 1 < k) ? lmove + next : -INFINITY);
      lq = active ? lprior + logp : -INFINITY;
    }
    // normalise: lq -= logsumexp(lq); an all-zero product falls back to p (D-5)
    if (warp_max(lq) == -INFINITY) lq = logp;
    const float qmax = warp_max(lq);
    const float qs = warp_sum(active ? expf(lq - qmax) : 0.f);
    lq = active ? lq - (qmax + logf(qs)) : -INFINITY;
    const float q = active ? expf(lq) : 0.f;
    const float L = warp_sum(q * m_i);

    if (first) {
      // argmax of q (lowest index on ties): smallest lane holding the max
      const float best = warp_max(lq);
      const unsigned ball = __ballot_sync(0xffffffffu, active && lq == best);
      const int amax = __ffs(ball) - 1;
      mt.thr = cst->thr_tab[amax];
      mt.age = 0;
      mt.flags = 1u;
    } else {
      mt.age += 1;
    }
    mt.L = L;
    if (active) {
      lq_state[(int64_t)slot * k + lane] = lq;
      if (post) post[(int64_t)j * k + lane] = q;
    }
    if (lane == 0) {
      meta[slot] = mt;
      if (Lout) Lout[j] = L;
    }
  }
}

cudaError_t launch_head(const Ctx &c, int n, int splits, const uint32_t *ids,
                        const uint8_t *is_prefill, const float *prior_override, float *post,
                        float *L, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  // 4 requests per CTA: >= one CTA per SM already at n = 512 (latency-bound kernel)
  const int warps = 4;
  int blocks = (n + warps - 1) / warps;
  const int cap = c.num_sms * 8;
  if (blocks > cap) blocks = cap;
  const size_t smem = (size_t)c.k * c.H * sizeof(float);
#define TRAIL_HEAD(HC)                                                                        \
  return launch_k(trail_head_kernel<HC>, dim3(blocks), dim3(warps * 32), smem, s, c.partial,  \
                  splits, n, c.b1, c.w2, c.b2, c.consts, ids, is_prefill, prior_override,     \
                  c.cfg.max_slots, c.lq, c.meta, post, L, c.dev_err)
  switch (c.H / 128) {
    case 1: TRAIL_HEAD(1);
    case 2: TRAIL_HEAD(2);
    case 3: TRAIL_HEAD(3);
    default: TRAIL_HEAD(4);
  }
#undef TRAIL_HEAD
}

cudaError_t head_prepare(Ctx &c) {
  const int smem = c.k * c.H * (int)sizeof(float);
  cudaError_t e = cudaSuccess;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(trail_head_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(trail_head_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(trail_head_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(trail_head_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  return e;
}

}  // namespace trail
