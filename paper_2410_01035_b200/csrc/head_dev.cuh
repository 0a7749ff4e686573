// head_dev.cuh — row a3 head shared by the fused (K2c) and wide (K2d) tcgen05 kernels:
// layer-2 logits -> softmax -> Bayesian refinement in the log domain -> expected length ->
// slot-state update, one lane per bin.  CUDA path only.
#pragma once

#include <math.h>

#include "trail_internal.cuh"

namespace trail {

// Per-bin constants of the head, staged in shared memory (lane b reads entry b).
struct HeadSmem {
  float m[kMaxBins], log_stay[kMaxBins], log_move[kMaxBins], log_prior[kMaxBins];
  uint32_t thr[kMaxBins];
};

__device__ __forceinline__ float seg_max(float v, int seg) {
  for (int o = seg >> 1; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o, seg));
  return v;
}
__device__ __forceinline__ float seg_sum(float v, int seg) {
  for (int o = seg >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, seg);
  return v;
}

// Row a3 head for request j, one lane per bin (b) in a SEG-lane segment; every lane of the
// warp calls it (j >= n: inactive segment, shuffles only).  Log-domain recursion (D-22) with
// fast-math exp/log (MUFU, ~2 ulp: errors ~1e-7, far inside the 2e-3 posterior bound).
//   log p = z - logsumexp(z)                                   (softmax)
//   prefill: log q = log pi + log p                            (D-9 threshold)
//   decode:  log q = logaddexp(log T_bb + lq(b), log T_b,b+1 + lq(b+1)) + log p
//   normalise; L = sum_b q(b) m_b
// Five segment reductions: max z, sum exp, (max, argmax) of the unnormalised log q, sum exp,
// sum q m.  The D-5 fallback (all-zero product) redoes the (max, argmax) over log p.
__device__ __forceinline__ void head_seg(int j, int n, int k, int SEG, int b, float z,
                                         const HeadSmem &hc, float hc_dyn_c, uint32_t sl,
                                         const SlotMeta &mt,
                                         float lq_prev, const float *__restrict__ prior_override,
                                         float *__restrict__ lq_state, SlotMeta *__restrict__ meta,
                                         float *__restrict__ post, float *__restrict__ Lout,
                                         uint32_t *__restrict__ err) {
  const bool act = j < n && b < k;
  const bool bad = sl == 0xFFFFFFFFu;
  const uint32_t slot = sl & 0x7FFFFFFFu;
  if (!act) z = -INFINITY;
  const float zmax = seg_max(z, SEG);
  const float lse = zmax + __logf(seg_sum(act ? __expf(z - zmax) : 0.f, SEG));
  const float lp = act ? z - lse : -INFINITY;
  const bool first = (sl >> 31) != 0u || !(mt.flags & 1u);
  const float prev = (act && !first && !bad) ? lq_prev : -INFINITY;
  float prev1 = __shfl_down_sync(0xffffffffu, prev, 1, SEG);
  if (b + 1 >= k) prev1 = -INFINITY;
  float lq = -INFINITY;
  if (act) {
    float lpr;
    if (first) {
      lpr = prior_override ? __logf(__ldg(prior_override + (int64_t)j * k + b)) : hc.log_prior[b];
    } else {
      // prior(b) = (1 - 1/w_b) q(b) + (1/w_{b+1}) q(b+1): T applied to the posterior (D-1, D-2)
      const float stay = hc.log_stay[b] + prev, move = hc.log_move[b] + prev1;
      const float mx = fmaxf(stay, move), mn = fminf(stay, move);
      lpr = mx == -INFINITY ? -INFINITY : mx + __logf(1.f + __expf(mn - mx));
    }
    lq = lpr + lp;
  }
  // (max, argmax) of the unnormalised log q, lowest index on ties (argmax of q^(0), D-9), and
  // of log p for the D-5 fallback — reduced together by every lane (no divergent shuffles:
  // inactive segments also have an all -inf q)
  float qmax = lq, pmax = act ? lp : -INFINITY;
  int bi = act ? b : 0x7FFFFFFF, pi = bi;
  for (int o = SEG >> 1; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, qmax, o, SEG);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o, SEG);
    const float pv = __shfl_xor_sync(0xffffffffu, pmax, o, SEG);
    const int pj = __shfl_xor_sync(0xffffffffu, pi, o, SEG);
    if (ov > qmax || (ov == qmax && oi < bi)) { qmax = ov; bi = oi; }
    if (pv > pmax || (pv == pmax && pj < pi)) { pmax = pv; pi = pj; }
  }
  if (qmax == -INFINITY) {          // all-zero product: fall back to p (D-5); only reachable
    lq = lp;                        // for a prior that is zero on every bin; the threshold
    qmax = pmax;                    // comes from argmax p, as in K3 and the oracle
    bi = pi;
  }
  const float qs = seg_sum(act ? __expf(lq - qmax) : 0.f, SEG);   // every lane shuffles
  lq = act ? lq - (qmax + __logf(qs)) : -INFINITY;
  const float q = act ? __expf(lq) : 0.f;
  const float L = seg_sum(act ? q * hc.m[b] : 0.f, SEG);
  if (j >= n) return;
  if (bad) {
    if (b == 0) atomicOr(err, TRAIL_DEV_BAD_ID);
    if (b < k && post) post[(int64_t)j * k + b] = NAN;
    if (b == 0 && Lout) Lout[j] = NAN;
    return;
  }
  if (b < k) {
    lq_state[(int64_t)slot * k + b] = lq;
    if (post) post[(int64_t)j * k + b] = q;
  }
  if (b == 0) {
    SlotMeta o = mt;
    if (first) {
      o.thr = hc.thr[bi];
      o.age = 0;
      o.flags = 1u;
    } else {
      o.age += 1;
    }
    o.L = L;
    if (hc_dyn_c >= 0.f) o.thr = dynamic_threshold(hc_dyn_c, L);
    meta[slot] = o;
    if (Lout) Lout[j] = L;
  }
}


// Row a3 head for request j by ONE thread over all k bins (same recursion as head_seg, the
// reductions sequential in bin order instead of shuffle trees): no cross-lane dependency
// chains, so 128 rows run as 128 independent threads.  K2d's epilogue (128 rows per CTA)
// measured 23 us with head_seg (one warp per row: five dependent shuffle reductions per
// row, 16 rows per warp in sequence).
template <int KB>
__device__ __forceinline__ void head_row(int j, int k, const float (&z)[KB], const HeadSmem &hc,
                                         float hc_dyn_c, uint32_t sl, const SlotMeta &mt,
                                         const float *__restrict__ lq_prev,
                                         const float *__restrict__ prior_override,
                                         float *__restrict__ lq_state, SlotMeta *__restrict__ meta,
                                         float *__restrict__ post, float *__restrict__ Lout,
                                         uint32_t *__restrict__ err) {
  if (sl == 0xFFFFFFFFu) {
    atomicOr(err, TRAIL_DEV_BAD_ID);
    if (post)
      for (int b = 0; b < k; ++b) post[(int64_t)j * k + b] = NAN;
    if (Lout) Lout[j] = NAN;
    return;
  }
  const uint32_t slot = sl & 0x7FFFFFFFu;
  const bool first = (sl >> 31) != 0u || !(mt.flags & 1u);
  float zmax = -INFINITY;
#pragma unroll
  for (int b = 0; b < KB; ++b) if (b < k) zmax = fmaxf(zmax, z[b]);
  float se = 0.f;
#pragma unroll
  for (int b = 0; b < KB; ++b) if (b < k) se += __expf(z[b] - zmax);
  const float lse = zmax + __logf(se);
  float lp[KB], lq[KB];
#pragma unroll
  for (int b = 0; b < KB; ++b) {
    lp[b] = b < k ? z[b] - lse : -INFINITY;
    float lpr = -INFINITY;
    if (b < k) {
      if (first) {
        lpr = prior_override ? __logf(__ldg(prior_override + (int64_t)j * k + b)) : hc.log_prior[b];
      } else {
        // prior(b) = (1 - 1/w_b) q(b) + (1/w_{b+1}) q(b+1): T applied to the posterior (D-1, D-2)
        const float stay = hc.log_stay[b] + lq_prev[b];
        const float move = b + 1 < k ? hc.log_move[b] + lq_prev[b + 1 < KB ? b + 1 : b] : -INFINITY;
        const float mx = fmaxf(stay, move), mn = fminf(stay, move);
        lpr = mx == -INFINITY ? -INFINITY : mx + __logf(1.f + __expf(mn - mx));
      }
    }
    lq[b] = lpr + lp[b];
  }
  // (max, argmax) of the unnormalised log q and of log p (D-5 fallback), lowest index on ties
  float qmax = -INFINITY, pmax = -INFINITY;
  int bi = 0, pi = 0;
#pragma unroll
  for (int b = 0; b < KB; ++b)
    if (b < k) {
      if (lq[b] > qmax) { qmax = lq[b]; bi = b; }
      if (lp[b] > pmax) { pmax = lp[b]; pi = b; }
    }
  if (qmax == -INFINITY) {          // all-zero product: fall back to p (D-5)
#pragma unroll
    for (int b = 0; b < KB; ++b) lq[b] = lp[b];
    qmax = pmax;
    bi = pi;
  }
  float qs = 0.f;
#pragma unroll
  for (int b = 0; b < KB; ++b) if (b < k) qs += __expf(lq[b] - qmax);
  const float lnorm = qmax + __logf(qs);
  float L = 0.f;
#pragma unroll
  for (int b = 0; b < KB; ++b)
    if (b < k) {
      const float l = lq[b] - lnorm;
      const float q = __expf(l);
      L += q * hc.m[b];
      lq_state[(int64_t)slot * k + b] = l;
      if (post) post[(int64_t)j * k + b] = q;
    }
  SlotMeta o = mt;
  if (first) {
    o.thr = hc.thr[bi];
    o.age = 0;
    o.flags = 1u;
  } else {
    o.age += 1;
  }
  o.L = L;
  if (hc_dyn_c >= 0.f) o.thr = dynamic_threshold(hc_dyn_c, L);
  meta[slot] = o;
  if (Lout) Lout[j] = L;
}

}  // namespace trail
