// TMA ingress microbenchmark: how many bytes per cycle can one SM pull through
// cp.async.bulk.tensor from L2-resident data, as a function of box size and ring
// depth, with one CTA per SM on all SMs (the attention kernels' K/V streams).
// The tensor is a [rows, heads, 128] bf16 token-major buffer (K-like: the rows of
// one head are heads*256 B apart), boxes of {64 cols, 1 head, box_rows}.
// Each CTA streams `iters` boxes of its head through a `stages`-deep ring; a
// consumer warp waits each fill and releases it at once (no compute).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench tools/tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                 : "=r"(ok)
                 : "r"(smem_u32(b)), "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__global__ void tma_stream(const __grid_constant__ CUtensorMap map, int heads, int rows, int box_rows, int boxes_per_fill,
                           int stages, int iters, int producers, int prefetch, int no_wait, int distinct, int two_d, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t box_bytes = box_rows * 128;
  const uint32_t fill = box_bytes * boxes_per_fill;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int head = blockIdx.x % heads;
  const int nrow_tiles = rows / box_rows;
  unsigned long long t0 = clock64();
  if (prefetch && lane == 0 && warp < producers)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
  // producers > 0: that many warps (lane 0 each); producers < 0: -producers lanes of warp 0
  const bool is_prod = producers > 0 ? (warp < producers && lane == 0) : (warp == 0 && lane < -producers);
  const int pid = producers > 0 ? warp : lane, np = producers > 0 ? producers : -producers;
  if (is_prod) {
    for (int it = pid; it < iters; it += np) {
      const int s = it % stages;
      if (!no_wait) mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      mbar_expect(&full[s], fill);
      // distinct > 0: CTAs sharing a head start `distinct` row tiles apart (no two SMs on the same lines)
      const int rt = (it / boxes_per_fill * boxes_per_fill + distinct * (blockIdx.x / heads)) % nrow_tiles;
      for (int b = 0; b < boxes_per_fill; ++b) {
        const int r = ((rt + b / 2 + it) % nrow_tiles) * box_rows;
        if (two_d)  // 2-D view of one head: [rows, 128] with a heads*256-byte row pitch
          tma2(smem + s * fill + b * box_bytes, &map, &full[s], (b & 1) * 64, r);
        else
          tma3(smem + s * fill + b * box_bytes, &map, &full[s], (b & 1) * 64, head, r);
      }
    }
  } else if (warp == (producers > 0 ? producers : 1) && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      mbar_arrive(&empty[s]);
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
}

int main(int argc, char** argv) {
  const int heads = 32, rows = argc > 1 ? atoi(argv[1]) : 8192;  // 8192 x 32 heads x 256 B = 64 MB: L2-resident
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void* buf = nullptr;
  cudaMalloc(&buf, (size_t)rows * heads * 256);
  cudaMemset(buf, 1, (size_t)rows * heads * 256);
  unsigned long long* cyc = nullptr;
  cudaMalloc(&cyc, sizeof(unsigned long long) * 4096);
  printf("box_rows boxes/fill stages producers ctas  bytes/cycle/SM\n");
  for (int box_rows : {64, 128}) {
   for (int mk : {0}) {  // 0: 3-D SW128 L2_256B, 1: 3-D SW128 no L2 promotion, 2: 2-D SW128, 3: 3-D no swizzle
    CUtensorMap m;
    CUresult rr;
    if (mk == 2) {
      cuuint64_t dims[2] = {128, (cuuint64_t)rows};
      cuuint64_t str[1] = {(cuuint64_t)heads * 256};
      cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      rr = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[3] = {128, (cuuint64_t)heads, (cuuint64_t)rows};
      cuuint64_t str[2] = {256, (cuuint64_t)heads * 256};
      cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
      cuuint32_t es[3] = {1, 1, 1};
      rr = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  mk == 3 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                                  mk == 1 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (rr != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)rr);
      return 1;
    }
    for (int bpf : {2}) {
     for (int prod : {1, 2, -2, 4, -4}) {
      for (int variant : {0}) {
       const int stages = 8;
        const int fill = box_rows * 128 * bpf;
        const int smem = fill * stages;
        if (smem > 200 * 1024) continue;
        cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int ctas : {sms}) {
          const int iters = 4000;
          // variant 0: plain; 1: prefetch.tensormap; 2: no empty wait (issue rate only; iters = stages)
          const int it_n = (variant == 2 || variant == 4) ? stages : iters;
          // 3: distinct rows per CTA (streaming); 4: distinct + issue only
          const int dist = (variant >= 3) ? 37 : 0;
          const bool nw = variant == 2 || variant == 4;
          const int it_m = nw ? stages : iters;
          tma_stream<<<ctas, 192, smem>>>(m, heads, rows, box_rows, bpf, stages, nw ? stages : 200, prod,
                                         variant == 1, nw, dist, mk == 2, cyc);
          tma_stream<<<ctas, 192, smem>>>(m, heads, rows, box_rows, bpf, stages, it_m, prod, variant == 1, nw, dist,
                                         mk == 2, cyc);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          unsigned long long h[4096];
          cudaMemcpy(h, cyc, sizeof(unsigned long long) * ctas, cudaMemcpyDeviceToHost);
          unsigned long long mx = 0;
          for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
          const double per_sm = (double)fill * it_n * ((double)ctas / sms) / (double)mx;
          printf("%8d %10d %6d %9d %5d  %8.1f   map %d variant %d (cycles %llu)\n", box_rows, bpf, stages, prod, ctas,
                 per_sm, mk, variant, mx);
        }
      }
     }
    }
   }
  }
  return 0;
}
