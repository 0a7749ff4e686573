// xgather.cuh — the A-operand (X) row gather shared by the fused (K2c) and wide (K2d)
// tcgen05 kernels (row a1 at decode): request j's row is emb row off[j] when it
// has exactly one row (decode: bit-exact), else the pooled prompt mean K1 wrote to xs row j
// (prefill).  One warp plans a 128-row tile: lane l owns rows 4l..4l+3; runs of
// consecutive source rows become one TMA box (32 rows per 8-lane block, else 4 rows),
// scattered single rows one tile::gather4, mixed groups four 1-row loads.  Only xs rows
// depend on the previous kernel (PDL).  CUDA path only.
#pragma once

#include "sm100_ptx.cuh"

namespace trail {

struct XPlan {
  int src[4];
  unsigned emask;   // bit q: row 4*lane+q comes from emb
  int mode;         // 0 none (covered by the block op), 1 block emb32, 2 block xs32, 3 emb4,
                    // 4 xs4, 5 gather4 (emb), 6 four single rows
  bool tile_xs;     // some row of the tile reads xs (must wait for K1)
};

// warp-collective (all 32 lanes)
__device__ __forceinline__ XPlan xplan_make(const int32_t *__restrict__ off, int n, int m0, int lane) {
  XPlan p;
  p.emask = 0u;
  bool any_xs = false;
  const int j4 = m0 + 4 * lane;
  int o[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) o[q] = (j4 + q <= n) ? __ldg(off + j4 + q) : 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = j4 + q;
    const bool single = j < n && o[q + 1] - o[q] == 1;
    p.src[q] = single ? o[q] : j;            // emb row, or xs row (padding rows: xs, unused)
    p.emask |= single ? 1u << q : 0u;
    any_xs |= !single && j < n;
  }
  const bool g_emb = p.emask == 0xFu, g_xs = p.emask == 0u;
  const bool g_contig = p.src[1] == p.src[0] + 1 && p.src[2] == p.src[0] + 2 && p.src[3] == p.src[0] + 3;
  const int prev_src0 = __shfl_up_sync(0xffffffffu, p.src[0], 1);
  const bool link = (lane & 7) == 0 || prev_src0 + 4 == p.src[0];
  const unsigned blk = 0xFFu << (lane & 24);
  const bool b_emb = (__ballot_sync(0xffffffffu, g_emb && g_contig && link) & blk) == blk;
  const bool b_xs = (__ballot_sync(0xffffffffu, g_xs && g_contig && link) & blk) == blk;
  if (b_emb || b_xs) p.mode = (lane & 7) == 0 ? (b_emb ? 1 : 2) : 0;
  else if (g_contig && g_emb) p.mode = 3;
  else if (g_contig && g_xs) p.mode = 4;
  else if (g_emb) p.mode = 5;
  else p.mode = 6;
  p.tile_xs = __any_sync(0xffffffffu, any_xs);
  return p;
}

// this lane's loads of k-block column kc into the tile at a_base (lane's 4 rows at +512*lane);
// PAIR: cta_group::2 loads completing on the leader's barrier fb (shared::cluster address)
template <bool PAIR>
__device__ __forceinline__ void xplan_issue(const XPlan &p, int lane, uint32_t a_base, uint32_t fb,
                                            int kc, const CUtensorMap *emb1, const CUtensorMap *emb4,
                                            const CUtensorMap *emb32, const CUtensorMap *xs1,
                                            const CUtensorMap *xs4, const CUtensorMap *xs32) {
  using namespace ptx;
  const uint32_t dst = a_base + (uint32_t)(lane * 4 * 128);
  auto ld = [&](uint32_t d, const CUtensorMap *m, int row) {
    if (PAIR) tma_load_2d_pair(d, m, fb, kc, row);
    else tma_load_2d(d, m, fb, kc, row);
  };
  switch (p.mode) {
    case 1: ld(dst, emb32, p.src[0]); break;
    case 2: ld(dst, xs32, p.src[0]); break;
    case 3: ld(dst, emb4, p.src[0]); break;
    case 4: ld(dst, xs4, p.src[0]); break;
    case 5:
      if (PAIR) tma_gather4_pair(dst, emb1, fb, kc, p.src[0], p.src[1], p.src[2], p.src[3]);
      else tma_gather4(dst, emb1, fb, kc, p.src[0], p.src[1], p.src[2], p.src[3]);
      break;
    case 6:
#pragma unroll
      for (int q = 0; q < 4; ++q) ld(dst + q * 128, ((p.emask >> q) & 1u) ? emb1 : xs1, p.src[q]);
      break;
    default: break;
  }
}

}  // namespace trail
