// MUFU.EX2 throughput per SM: ex2.approx.ftz.f32 vs ex2.approx.f16x2 (2 results
// per lane per instruction) vs ex2.approx.ftz.bf16x2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_bench.cu -o tools/mufu_bench
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
template <int MODE>
__global__ void ex2_kernel(float* out, int iters, long long* cyc) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) {
    float f = -(threadIdx.x * 1e-3f + i * 0.1f);
    if (MODE == 0) a[i] = __float_as_uint(f);
    else if (MODE == 1) { __half2 h = __floats2half2_rn(f, f * 0.5f); a[i] = *reinterpret_cast<uint32_t*>(&h); }
    else { __nv_bfloat162 h = __floats2bfloat162_rn(f, f * 0.5f); a[i] = *reinterpret_cast<uint32_t*>(&h); }
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(a[i]));
      else if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
      else asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
    }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char* name, float* o, long long* c) {
  for (int warps : {8, 16}) {
    int iters = 4096;
    ex2_kernel<MODE><<<148, warps * 32>>>(o, iters, c);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double lanes = warps * 32.0 * 8 * iters;
    printf("%-8s warps/SM=%2d: %.2f instr/clk/SM -> %.2f exp2 results/clk/SM\n", name, warps, lanes / h,
           lanes / h * (MODE == 0 ? 1 : 2));
  }
}
int main() {
  float* o;
  long long* c;
  cudaMalloc(&o, 1 << 24);
  cudaMalloc(&c, 8 * 1024);
  run<0>("f32", o, c);
  run<1>("f16x2", o, c);
  run<2>("bf16x2", o, c);
  return 0;
}
