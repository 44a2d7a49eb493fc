// MUFU.EX2 / FFMA2 throughput per SM (cycles per warp-instruction per SMSP)
#include <cstdio>
__global__ void ex2_kernel(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 0.1f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 8 * 1024);
  for (int warps : {4, 8, 16, 32}) {
    int iters = 4096;
    ex2_kernel<<<148, warps * 32>>>(o, iters, c);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double per_warp_instr = (double)h / (iters * 8.0);  // cycles per instruction-slot of one warp
    printf("warps/SM=%2d: %.2f cycles per (8 ex2 per thread) iter -> %.2f ex2/clk/SM\n", warps, (double)h / iters,
           warps * 32.0 * 8 * iters / h);
  }
  return 0;
}
