// 2-CTA (cta_group::2) tcgen05 GEMM probe (diagnostic, not product code): D[M][512] =
// X[M][K] . W[512][K]^T in bf16 -> fp32, one CTA pair per 256 rows, full N = 512 in TMEM
// (two N = 256 MMAs per K step).  Checks the operand split (A by rows, B by N halves), the
// peer-signalled TMA, the multicast commit and the 2-CTA TMEM allocation against a host
// reference, then times it at the configs[3] size.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 umma2.cu -o umma2 -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int BM = 128, BK = 64, H = 512;
constexpr int A_BYTES = BM * BK * 2;           // 16 KB: my 128 rows
constexpr int BH_BYTES = 128 * BK * 2;         // 16 KB: my 128 rows of one N half
constexpr int STAGE_BYTES = A_BYTES + 2 * BH_BYTES;
constexpr int STAGES = 4;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(ok) : "r"(b), "r"(ph) : "memory");
  } while (!ok);
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
// TMA 2-D load into MY smem, completion on the barrier `bar` (a shared::cluster address: the leader's)
__device__ __forceinline__ void tma2_load(uint32_t dst, const CUtensorMap *m, uint32_t bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ uint64_t sw128(uint32_t a) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(bar), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t t, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(256, 1) gemm2(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tw,
                                                int M, int kblocks, float *D) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  const uint32_t s0 = su32(sm);
  const uint32_t bar0 = s0 + STAGES * STAGE_BYTES;
  const uint32_t full0 = bar0, empty0 = bar0 + 8 * STAGES, done = bar0 + 16 * STAGES;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(sm + STAGES * STAGE_BYTES + 16 * STAGES + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r = crank();
  const int pair = blockIdx.x >> 1;
  const int m0 = pair * 256 + (int)r * BM;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(full0 + 8 * i, 1); mbar_init(empty0 + 8 * i, 1); }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  csync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0) {
    const uint32_t lead_full0 = mapa(full0, 0);
    for (int i = 0; i < kblocks; ++i) {
      const int st = i % STAGES;
      if (i >= STAGES) mbar_wait(empty0 + 8 * st, ((i / STAGES) & 1) ^ 1);
      if (r == 0) mbar_expect_tx(full0 + 8 * st, 2 * STAGE_BYTES);
      const uint32_t sa = s0 + st * STAGE_BYTES;
      const uint32_t fb = lead_full0 + 8 * st;
      tma2_load(sa, &tx, fb, i * BK, m0);
      tma2_load(sa + A_BYTES, &tw, fb, i * BK, 0 * 256 + (int)r * 128);
      tma2_load(sa + A_BYTES + BH_BYTES, &tw, fb, i * BK, 1 * 256 + (int)r * 128);
    }
  } else if (warp == 1 && lane == 0 && r == 0) {
    constexpr uint32_t id = idesc(256, 256);
    for (int i = 0; i < kblocks; ++i) {
      const int st = i % STAGES;
      mbar_wait(full0 + 8 * st, (i / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = s0 + st * STAGE_BYTES;
      const uint64_t da = sw128(sa);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint64_t db = sw128(sa + A_BYTES + h * BH_BYTES);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          umma2(tmem + 256 * h, da + 2 * kk, db + 2 * kk, id, (i > 0 || kk > 0) ? 1u : 0u);
      }
      commit2(empty0 + 8 * st);
    }
    commit2(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int g = warp & 3, half = warp >> 2;
    const int row = m0 + 32 * g + lane;
    for (int c = 256 * half; c < 256 * half + 256; c += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(32 * g) << 16) + (uint32_t)c, v);
      if (row < M)
        for (int q = 0; q < 32; ++q) D[(int64_t)row * H + c + q] = __uint_as_float(v[q]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  csync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

typedef CUresult (*PFN_enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool enc(CUtensorMap *m, void *p, uint64_t cols, uint64_t rows, uint32_t bc, uint32_t br) {
  static PFN_enc fn = nullptr;
  if (!fn) {
    void *q = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &qr);
    fn = (PFN_enc)q;
  }
  cuuint64_t dims[2] = {cols, rows}, str[1] = {cols * 2};
  cuuint32_t box[2] = {bc, br}, es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static float bf(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }

int run(int M, int K, bool check, int reps) {
  std::vector<uint16_t> hx((size_t)M * K), hw((size_t)H * K);
  uint32_t s = 12345;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return (uint16_t)(((s >> 9) & 0x7F) | 0x3F00 | ((s >> 20) & 1 ? 0x8000 : 0)); };
  for (auto &v : hx) v = rnd();
  for (auto &v : hw) v = rnd();
  void *dx, *dw;
  float *dd;
  CK(cudaMalloc(&dx, hx.size() * 2));
  CK(cudaMalloc(&dw, hw.size() * 2));
  CK(cudaMalloc(&dd, (size_t)M * H * 4));
  CK(cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(dd, 0xFF, (size_t)M * H * 4));
  CUtensorMap tx, tw;
  if (!enc(&tx, dx, K, M, BK, 128) || !enc(&tw, dw, K, H, BK, 128)) { printf("encode failed\n"); return 1; }
  CK(cudaFuncSetAttribute(gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * ((M + 255) / 256));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, gemm2, tx, tw, M, K / BK, dd));
  CK(cudaDeviceSynchronize());
  if (check) {
    std::vector<float> hd((size_t)M * H);
    CK(cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost));
    double worst = 0;
    int bad = 0;
    for (int m = 0; m < M; m += (M > 1024 ? 37 : 1))
      for (int n = 0; n < H; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)bf(hx[(size_t)m * K + k]) * bf(hw[(size_t)n * K + k]);
        const double e = fabs(ref - hd[(size_t)m * H + n]) / (1.0 + fabs(ref));
        if (e > worst) worst = e;
        if (!(e < 1e-3) && bad++ < 5) printf("  mismatch m=%d n=%d ref=%f got=%f\n", m, n, ref, hd[(size_t)m * H + n]);
      }
    printf("check M=%d K=%d: worst rel err %.3e  %s\n", M, K, worst, bad ? "FAIL" : "ok");
  }
  if (reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    void *fl; CK(cudaMalloc(&fl, 256 << 20));
    float best = 1e9;
    for (int i = 0; i < reps; ++i) {
      cudaMemsetAsync(fl, i, 256 << 20);
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, gemm2, tx, tw, M, K / BK, dd);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double fl_ = 2.0 * M * (double)K * H;
    printf("time M=%d K=%d: %.2f us  %.1f TFLOP/s  (X %.1f MB)\n", M, K, best * 1e3, fl_ / (best * 1e-3) / 1e12, (double)M * K * 2 / 1e6);
    cudaFree(fl);
  }
  cudaFree(dx); cudaFree(dw); cudaFree(dd);
  return 0;
}

int main() {
  run(512, 1024, true, 0);
  run(768, 4096, true, 0);
  run(16384, 8192, true, 10);
  run(16384, 4096, false, 10);
  run(8192, 4096, false, 10);
  CK(cudaGetLastError());
  return 0;
}
