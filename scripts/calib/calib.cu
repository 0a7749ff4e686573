// Latency calibration on the B200 box (diagnostic, not product code): pointer-chase
// latency for L2- and HBM-resident data, __syncthreads cost, global atomic round trip,
// back-to-back kernel start gaps (plain and PDL).  nvcc -arch=sm_100a calib.cu -o calib
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void chase(const uint32_t *nxt, int hops, uint64_t *out) {
  uint32_t p = 0;
  uint64_t t0 = gt();
  for (int i = 0; i < hops; ++i) p = __ldcg(nxt + p);
  uint64_t t1 = gt();
  out[0] = t1 - t0; out[1] = p;
}
__global__ void syncs(int iters, uint64_t *out) {
  __shared__ int x;
  uint64_t t0 = gt();
  for (int i = 0; i < iters; ++i) { if (threadIdx.x == i % blockDim.x) x = i; __syncthreads(); }
  uint64_t t1 = gt();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = x; }
}
__global__ void atomics(uint32_t *c, int iters, uint64_t *out) {
  uint32_t v = 0;
  uint64_t t0 = gt();
  for (int i = 0; i < iters; ++i) v += atomicAdd(c, v & 1);
  uint64_t t1 = gt();
  out[0] = t1 - t0; out[1] = v;
}
__global__ void stamp(uint64_t *out, int idx, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) out[2 * idx] = gt();
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[2 * idx + 1] = gt();
}

// straight-line code: N independent FMAs on 8 registers, executed once by one warp
template <int N>
__global__ void straight(float *out, uint64_t *t) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
        a6 = a0 + 6, a7 = a0 + 7;
  uint64_t t0 = gt();
  a0 += (float)(t0 & 1);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    a0 = fmaf(a0, 1.0001f, 0.5f); a1 = fmaf(a1, 1.0001f, 0.5f); a2 = fmaf(a2, 1.0001f, 0.5f);
    a3 = fmaf(a3, 1.0001f, 0.5f); a4 = fmaf(a4, 1.0001f, 0.5f); a5 = fmaf(a5, 1.0001f, 0.5f);
    a6 = fmaf(a6, 1.0001f, 0.5f); a7 = fmaf(a7, 1.0001f, 0.5f);
  }
  const float sum = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  uint64_t t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1) : "f"(sum));
  if (threadIdx.x == 0) { t[0] = t1 - t0; }
  out[threadIdx.x] = sum;
}
__global__ void evict(float *buf, int n) {   // big unrelated kernel + L2 traffic
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) buf[i] += 1.f;
}

int main() {
  uint64_t *d_out; cudaMalloc(&d_out, 1024 * 8);
  uint64_t h[256];
  // pointer chase: random cycle over N elements
  for (size_t N : {size_t(1) << 16, size_t(1) << 26}) {
    std::vector<uint32_t> perm(N), nxt(N);
    for (size_t i = 0; i < N; ++i) perm[i] = i;
    uint64_t s = 88172645463325252ull;
    for (size_t i = N - 1; i > 0; --i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; size_t j = s % (i + 1); std::swap(perm[i], perm[j]); }
    for (size_t i = 0; i < N; ++i) nxt[perm[i]] = perm[(i + 1) % N];
    uint32_t *d; cudaMalloc(&d, N * 4); cudaMemcpy(d, nxt.data(), N * 4, cudaMemcpyHostToDevice);
    chase<<<1, 1>>>(d, 1000, d_out); cudaDeviceSynchronize();
    chase<<<1, 1>>>(d, 2000, d_out); cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
    printf("chase N=%zu (%zu KB): %.1f ns/hop\n", N, N * 4 / 1024, h[0] / 2000.0);
    cudaFree(d);
  }
  for (int t : {128, 256, 512, 1024}) {
    syncs<<<1, t>>>(1000, d_out); cudaDeviceSynchronize();
    syncs<<<1, t>>>(1000, d_out); cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
    printf("__syncthreads %d threads: %.1f ns\n", t, h[0] / 1000.0);
  }
  uint32_t *c; cudaMalloc(&c, 4); cudaMemset(c, 0, 4);
  atomics<<<1, 1>>>(c, 200, d_out); cudaDeviceSynchronize();
  atomics<<<1, 1>>>(c, 200, d_out); cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
  printf("atomicAdd round trip: %.1f ns\n", h[0] / 200.0);
  // back-to-back kernels in a stream: gap between end of k and start of k+1
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaStream_t st; cudaStreamCreate(&st);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.stream = st;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = pdl;
    for (int rep = 0; rep < 2; ++rep) {
      // graph of 8 kernels
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < 8; ++i) cudaLaunchKernelEx(&cfg, stamp, d_out, i, pdl);
      cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
      cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
      cudaMemcpy(h, d_out, 16 * 8, cudaMemcpyDeviceToHost);
      printf("graph pdl=%d: kernel start-to-start gaps (ns):", pdl);
      for (int i = 1; i < 8; ++i) printf(" %lld", (long long)(h[2 * i] - h[2 * i - 2]));
      printf("  | first kernel body %lld\n", (long long)(h[1] - h[0]));
    }
  }
  {
    float *o; cudaMalloc(&o, 4096); float *big; size_t nb = size_t(64) << 20; cudaMalloc(&big, nb * 4);
    for (int rep = 0; rep < 3; ++rep) {
      evict<<<592, 256>>>(big, (int)nb); cudaDeviceSynchronize();
      straight<512><<<1, 32>>>(o, d_out); cudaDeviceSynchronize();
      cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost); uint64_t cold = h[0];
      straight<512><<<1, 32>>>(o, d_out); cudaDeviceSynchronize();
      cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
      printf("straight-line 4096 FMAs (+overhead): cold %llu ns, warm %llu ns\n",
             (unsigned long long)cold, (unsigned long long)h[0]);
    }
  }
  return 0;
}
