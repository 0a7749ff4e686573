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
// over the warps of the request's CTA, 4 per lane (coalesced 512-byte rows of the partials);
// layer 2 per warp + a fixed-order sum of the warps' bin partials; the reduction over splits
// runs in a fixed order, so results are bit-reproducible.
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
__global__ void __launch_bounds__(128)
trail_head_kernel(const float *__restrict__ partial, int splits, int n,
                  const float *__restrict__ b1, const float *__restrict__ w2,
                  const float *__restrict__ b2, const HeadConsts *__restrict__ cst,
                  const uint32_t *__restrict__ ids, const uint8_t *__restrict__ is_prefill,
                  const float *__restrict__ prior_override, int max_slots,
                  float *__restrict__ lq_state, SlotMeta *__restrict__ meta,
                  float *__restrict__ post, float *__restrict__ Lout, uint32_t *__restrict__ err) {
  constexpr int H = 128 * HC;
  __shared__ float zs[HC][32];
  const int k = cst->k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // one CTA per request, warp c owns hidden units [128 c, 128 c + 128) (4 per lane): the
  // split-K sum of those units has all `splits` loads of a lane in flight at once
  const int c = warp;
  const float4 bias1 = c < HC ? __ldg(reinterpret_cast<const float4 *>(b1 + c * 128) + lane)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
  griddep_wait();      // partials from layer 1, slot state from the previous step
  griddep_launch();
  const bool active = lane < k;
  for (int j = blockIdx.x; j < n; j += gridDim.x) {
    // ---- h = ReLU(sum_s partial + b1) for my 4 hidden units, fixed split order
    if (c < HC) {
      float4 h = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 *src = reinterpret_cast<const float4 *>(partial + (int64_t)j * H + c * 128) + lane;
      const int64_t sstride = (int64_t)n * H / 4;
      int sp = 0;
      for (; sp + 8 <= splits; sp += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + (sp + u) * sstride);
#pragma unroll
        for (int u = 0; u < 8; ++u) { h.x += v[u].x; h.y += v[u].y; h.z += v[u].z; h.w += v[u].w; }
      }
      for (; sp < splits; ++sp) {
        const float4 v = __ldcs(src + sp * sstride);
        h.x += v.x; h.y += v.y; h.z += v.z; h.w += v.w;
      }
      h.x = fmaxf(h.x + bias1.x, 0.f);
      h.y = fmaxf(h.y + bias1.y, 0.f);
      h.z = fmaxf(h.z + bias1.z, 0.f);
      h.w = fmaxf(h.w + bias1.w, 0.f);
      // ---- layer 2 over my units: every lane forms its 32 per-bin partial dots (bins >= k
      //      zero), one warp reduce-scatter (31 shuffles) leaves bin b's chunk sum on lane b
      float zp[32];
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        float acc = 0.f;
        if (b < k) {
          const float4 w = __ldg(reinterpret_cast<const float4 *>(w2 + (int64_t)b * H + c * 128) + lane);
          acc = fmaf(w.x, h.x, fmaf(w.y, h.y, fmaf(w.z, h.z, w.w * h.w)));
        }
        zp[b] = acc;
      }
#pragma unroll
      for (int step = 0; step < 5; ++step) {
        const int half = 16 >> step;
        const bool upper = (lane & half) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
          const float a = zp[i], b = zp[i + half];
          zp[i] = (upper ? b : a) + __shfl_xor_sync(0xffffffffu, upper ? a : b, half);
        }
      }
      zs[c][lane] = zp[0];    // lane l holds bin 16 b4 + 8 b3 + 4 b2 + 2 b1 + b0 = l
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t slot = __ldg(ids + j);
      if (slot >= (uint32_t)max_slots) {
        if (lane == 0) atomicOr(err, TRAIL_DEV_BAD_ID);
        if (active && post) post[(int64_t)j * k + lane] = NAN;
        if (lane == 0 && Lout) Lout[j] = NAN;
      } else {
        const float m_i = active ? cst->m[lane] : 0.f;
        const float lstay = active ? cst->log_stay[lane] : -INFINITY;
        const float lmove = active ? cst->log_move[lane] : -INFINITY;
        const float lpi = active ? cst->log_prior[lane] : -INFINITY;
        float z = active ? __ldg(b2 + lane) : 0.f;
#pragma unroll
        for (int cc = 0; cc < HC; ++cc) z += zs[cc][lane];
        if (!active) z = -INFINITY;
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
    if (cst->dyn_c >= 0.f) mt.thr = dynamic_threshold(cst->dyn_c, L);
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
    __syncthreads();   // zs reused by the next request of this CTA
  }
}

cudaError_t launch_head(const Ctx &c, int n, int splits, const uint32_t *ids,
                        const uint8_t *is_prefill, const float *prior_override, float *post,
                        float *L, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  // one CTA per request (a warp per 128 hidden units), up to 8 CTAs per SM
  const int warps = 4;
  int blocks = n;
  const int cap = c.num_sms * 8;
  if (blocks > cap) blocks = cap;
  const size_t smem = 0;
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

cudaError_t head_prepare(Ctx &) { return cudaSuccess; }   // no dynamic shared memory

}  // namespace trail
