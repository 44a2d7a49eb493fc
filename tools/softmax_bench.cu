// Forward softmax microbenchmark: the per-tile softmax work of fwd_kernel's
// softmax warps in isolation (no MMA): tcgen05.ld of a 128-column S row per
// thread, row max, 128 exponentials (1 of every EMU pairs through the FMA-pipe
// cubic), row sum, bf16 pack, tcgen05.st of P.  Cycles per 128-element row per
// warp with 1 or 2 such warps per SMSP — i.e. how long a tile's softmax takes
// alone and how two tiles' softmax share an SMSP; optionally with a spare warp
// streaming M=128 N=128 SS MMAs into other TMEM columns (the tensor core busy).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_10377_b200/csrc -o tools/softmax_bench tools/softmax_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "sm100_ptx.cuh"

using namespace sppo::ptx;

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

template <int EMU, int SUMS>
__device__ __forceinline__ void exps64(const float* s, int j0, float negm, float sl2, uint32_t* out, float2& lsum) {
  const float2 nm2 = make_float2(negm, negm);
  const float2 sl22 = make_float2(sl2, sl2);
  float2 l2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = j0; j < j0 + 64; j += 2) {
    const float2 x = ffma2(make_float2(s[j], s[j + 1]), sl22, nm2);
    float2 e;
    if (EMU > 0 && (j >> 1) % EMU == EMU - 1) e = ex2_poly2(x);
    else e = make_float2(ex2(x.x), ex2(x.y));
    if (SUMS == 2 && ((j >> 1) & 1)) l2 = fadd2(l2, e);
    else lsum = fadd2(lsum, e);
    out[(j - j0) >> 1] = pack_bf16(e.x, e.y);
  }
  if (SUMS == 2) lsum = fadd2(lsum, l2);
}

// -DSTAMPS=1: clock64 stamps per phase of warp 0 of CTA 0 (ld, exps 1, max, exps 2 +
// stores).  The stamps themselves change the schedule: 1762 vs 1197 cycles per row —
// which is how the kernels' (untaken) trace points were found to cost the forward 6 %.
#ifndef STAMPS
#define STAMPS 0
#endif
__device__ long long g_phase[4];

template <int EMU, int SUMS>
__global__ void __launch_bounds__(288, 1) softmax_kernel(int iters, long long* cyc, float* sink, int nsoft, int mma) {
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t mbar;
  __shared__ volatile int done;
  extern __shared__ __align__(1024) uint8_t dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == nsoft) {  // MMA warp: S-like MMAs into columns 256..383 until the softmax warps finish
    if (mma) {
      const uint64_t da = sdesc_kmajor(smem_u32(dsm)), db = sdesc_kmajor(smem_u32(dsm + 16384));
      constexpr uint32_t idesc = idesc_bf16(128, 128, 0, 0);
      uint32_t ph = 0;
      while (!done) {
        for (int k = 0; k < 8; ++k) mma_ss_w(tmem_base + 256, da + 2 * k, db + 2 * k, idesc, k > 0);
        mma_commit_w(&mbar);
        mbar_wait(&mbar, ph);
        ph ^= 1;
      }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem_base);
    return;
  }
  // warps w and w+4 share TMEM lane quarter (w & 3) (= SMSP); each owns 128 columns
  const uint32_t t = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  {
    uint32_t init[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) init[i] = __float_as_uint(0.01f * (float)((lane * 7 + i * 13) % 97) - 0.5f);
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_st32(t + c * 32, init);
    tmem_wait_st();
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nsoft * 32));  // the softmax warps only (the MMA warp is looping)
  const float sl2 = 0.08838834764831845f * 1.4426950408889634f;
  float m_used = 0.f, l = 0.f;
  const long long t0 = clock64();
  long long ph[4] = {0, 0, 0, 0};
  const bool stamp = STAMPS && blockIdx.x == 0 && warp == 0;
  for (int it = 0; it < iters; ++it) {
    long long c0 = stamp ? clock64() : 0;
    uint32_t r[128];
    auto R32 = [&](int c) -> uint32_t(&)[32] { return *reinterpret_cast<uint32_t(*)[32]>(&r[c]); };
    tmem_ld32(t + 0, R32(0));
    tmem_ld32(t + 32, R32(32));
    tmem_wait_ld_regs(R32(0));
    tmem_wait_ld_regs(R32(32));
    tmem_ld32(t + 64, R32(64));
    tmem_ld32(t + 96, R32(96));
    float* s = reinterpret_cast<float*>(r);
    uint32_t pk0[32];
    float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
    long long c1 = stamp ? clock64() : 0;
    exps64<EMU, SUMS>(s, 0, -m_used, sl2, pk0, ls0);
    long long c2 = stamp ? clock64() : 0;
    tmem_wait_ld_regs(R32(64));
    tmem_wait_ld_regs(R32(96));
    float mx0 = s[0], mx1 = s[1];
#pragma unroll
    for (int j = 2; j < 126; j += 4) {
      mx0 = fmax3(mx0, s[j], s[j + 1]);
      mx1 = fmax3(mx1, s[j + 2], s[j + 3]);
    }
    const float mx = fmax3(mx0, mx1, fmaxf(s[126], s[127])) * sl2;
    if (__any_sync(0xffffffffu, mx > m_used + 8.f)) m_used = mx;  // (never: data in [-0.5, 0.5])
    long long c3 = stamp ? clock64() : 0;
    tmem_st32(t + 0, pk0);
    tmem_wait_st();
    exps64<EMU, SUMS>(s, 64, -m_used, sl2, &r[32], ls1);
    tmem_st32(t + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
    tmem_wait_st();
    l += ls0.x + ls0.y + ls1.x + ls1.y;
    if (stamp) {
      const long long c4 = clock64();
      ph[0] += c1 - c0;
      ph[1] += c2 - c1;
      ph[2] += c3 - c2;
      ph[3] += c4 - c3;
    }
  }
  const long long t1 = clock64();
  if (stamp && lane == 0)
    for (int k = 0; k < 4; ++k) g_phase[k] = ph[k] / iters;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = l;
  if (lane == 0) cyc[blockIdx.x * 8 + warp] = t1 - t0;
  asm volatile("bar.sync 1, %0;" ::"r"(nsoft * 32));
  if (threadIdx.x == 0) done = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem_base);
}

template <int EMU, int SUMS>
void run(const char* name, int warps_per_smsp, long long* dcyc, float* sink, int mma = 0) {
  const int iters = 2000, nsoft = 4 * warps_per_smsp, threads = 32 * (nsoft + 1);
  cudaFuncSetAttribute(softmax_kernel<EMU, SUMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  softmax_kernel<EMU, SUMS><<<148, threads, 32768 + 1024>>>(iters, dcyc, sink, nsoft, mma);
  softmax_kernel<EMU, SUMS><<<148, threads, 32768 + 1024>>>(iters, dcyc, sink, nsoft, mma);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 8];
  cudaMemcpy(h, dcyc, sizeof h, cudaMemcpyDeviceToHost);
  double sum = 0;
  int n = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < 4 * warps_per_smsp; ++w) sum += h[b * 8 + w], ++n;
  long long ph[4];
  cudaMemcpyFromSymbol(ph, g_phase, sizeof ph);
  printf("{\"case\": \"%s\", \"warps_per_smsp\": %d, \"mma_warp\": %d, \"cycles_per_row_per_warp\": %.0f, "
         "\"phases_warp0\": {\"ld\": %lld, \"exps1\": %lld, \"max\": %lld, \"exps2_st\": %lld}, \"err\": \"%s\"}\n",
         name, warps_per_smsp, mma, sum / n / iters, ph[0], ph[1], ph[2], ph[3], cudaGetErrorString(e));
}

int main() {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 8 * sizeof(long long));
  cudaMalloc(&sink, 148 * 512 * sizeof(float));
  for (int w : {1, 2}) {
    run<4, 1>("emu1of4 (kernel) + MMA stream", w, cyc, sink, 1);
    run<4, 1>("emu1of4 (kernel)", w, cyc, sink);
    run<0, 1>("all MUFU", w, cyc, sink);
    run<2, 1>("emu1of2", w, cyc, sink);
    run<3, 1>("emu1of3", w, cyc, sink);
    run<4, 2>("emu1of4 two sums", w, cyc, sink);
  }
  return 0;
}
