// K6 — time update between observations (the "predict every K iterations"
// variant): for requests that ran but were not observed this iteration, only the
// transition acts on the posterior,
//     log q <- logaddexp(log T_bb + lq(b), log T_b,b+1 + lq(b+1)) - logsumexp(.)   (P:215-216,
//                                                     readings D-1, D-4, D-22, D-25)
// applied `steps` times, then age a += steps (D-11) and L_t = sum_b q(b) m_b.  One warp
// per request, lane b = bin b (k <= 32), like the head K3.  Unobserved slots are untouched
// and report the prior pi and E_pi[L] (D-24).
#include <math.h>

#include "trail_internal.cuh"

namespace trail {

__global__ void __launch_bounds__(128)
trail_time_update_kernel(const uint32_t *__restrict__ ids, int n, int steps,
                         const HeadConsts *__restrict__ cst, int max_slots,
                         float *__restrict__ lq_state, SlotMeta *__restrict__ meta,
                         float *__restrict__ post, float *__restrict__ Lout,
                         uint32_t *__restrict__ err) {
  griddep_wait();      // slot state written by earlier kernels of the stream
  griddep_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + warp;
  if (j >= n) return;
  const int k = cst->k;
  const bool active = lane < k;
  const uint32_t slot = __ldg(ids + j);
  if (slot >= (uint32_t)max_slots) {
    if (lane == 0) atomicOr(err, TRAIL_DEV_BAD_ID);
    if (active && post) post[(int64_t)j * k + lane] = NAN;
    if (lane == 0 && Lout) Lout[j] = NAN;
    return;
  }
  SlotMeta mt = meta[slot];
  const float m_i = active ? cst->m[lane] : 0.f;
  if (!(mt.flags & 1u)) {            // never observed: nothing to propagate (D-24)
    if (active && post) post[(int64_t)j * k + lane] = __expf(cst->log_prior[lane]);
    if (lane == 0 && Lout) Lout[j] = cst->prior_L;
    return;
  }
  const float lstay = active ? cst->log_stay[lane] : -INFINITY;
  const float lmove = active ? cst->log_move[lane] : -INFINITY;
  float lq = active ? lq_state[(int64_t)slot * k + lane] : -INFINITY;
  for (int s = 0; s < steps; ++s) {
    const float next = __shfl_down_sync(0xffffffffu, lq, 1);
    const float a = lstay + lq, b = (lane + 1 < k) ? lmove + next : -INFINITY;
    const float mx = fmaxf(a, b), mn = fminf(a, b);
    float lp = mx == -INFINITY ? -INFINITY : mx + log1pf(__expf(mn - mx));
    if (!active) lp = -INFINITY;
    const float qmax = warp_max(lp);
    const float qs = warp_sum(active ? __expf(lp - qmax) : 0.f);
    lq = active ? lp - (qmax + __logf(qs)) : -INFINITY;
  }
  const float q = active ? __expf(lq) : 0.f;
  const float L = warp_sum(q * m_i);
  if (active) {
    lq_state[(int64_t)slot * k + lane] = lq;
    if (post) post[(int64_t)j * k + lane] = q;
  }
  if (lane == 0) {
    mt.age += (uint32_t)steps;
    mt.L = L;
    if (cst->dyn_c >= 0.f) mt.thr = dynamic_threshold(cst->dyn_c, L);
    meta[slot] = mt;
    if (Lout) Lout[j] = L;
  }
}

cudaError_t launch_time_update(const Ctx &c, const uint32_t *ids, int n, int steps, float *post,
                               float *L, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_k(trail_time_update_kernel, dim3((n + 3) / 4), dim3(128), 0, s, ids, n, steps,
                  (const HeadConsts *)c.consts, c.cfg.max_slots, c.lq, c.meta, post, L, c.dev_err);
}

}  // namespace trail
