// Reduction egress microbenchmark: how many bytes per cycle can one SM push into
// fp32 accumulators in global memory (the backward's dQ TMA reduce-add and dK/dV
// red.global.add), alone and with every SM doing it at once, versus plain bulk
// stores and a bulk shared::cta -> shared::cluster copy to the peer CTA (DSMEM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_bench tools/red_bench.cu
//   tools/red_bench            (prints one JSON line per case)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kBuf = 32768;  // bytes per operation (one dQ piece pair / one dS half is 16-32 KB)

// mode 0: bulk reduce-add f32 smem -> global; 1: bulk store smem -> global;
// 2: red.global.add.v4.f32 from registers, one 512 B row per thread (32 rows per warp
// instruction, the dK/dV epilogue pattern); 3: same, coalesced (a warp covers one row);
// 4: bulk copy smem -> peer CTA smem (cluster of 2), completing on the peer's mbarrier
template <int MODE>
__global__ void __launch_bounds__(256, 1) red_kernel(float* dst, size_t region_floats, int iters, int shared_dst,
                                                      long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* buf = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < kBuf / 4; i += blockDim.x) buf[i] = 1.0f;
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (MODE == 4) {
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0 && rank == 1)  // all of the sender's bytes complete one phase
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(iters * kBuf)
                   : "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  }
  float* my = dst + (shared_dst ? 0 : (size_t)blockIdx.x * region_floats);
  const long long t0 = clock64();
  if (MODE <= 1) {
    if (threadIdx.x == 0) {
      for (int it = 0; it < iters; ++it) {
        float* d = my + (size_t)(it % 8) * (kBuf / 4);
        if (MODE == 0)
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(d),
                       "r"(smem_u32(buf)), "r"(kBuf)
                       : "memory");
        else
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(smem_u32(buf)),
                       "r"(kBuf)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else if (MODE <= 3) {
    // 256 threads; kBuf bytes per iteration = 64 rows of 512 B (128 floats)
    for (int it = 0; it < iters; ++it) {
      float* d = my + (size_t)(it % 8) * (kBuf / 4);
      for (int k = 0; k < kBuf / 16 / 256; ++k) {
        int row, col4;
        if (MODE == 2) {  // thread = row (64 rows: threads 0..63), k-th float4 of it; 4 thread groups
          row = threadIdx.x & 63;
          col4 = (threadIdx.x >> 6) * (kBuf / 16 / 256) + k;
        } else {  // warp covers 512 B of one row
          const int idx = k * 256 + threadIdx.x;
          row = idx >> 5;
          col4 = idx & 31;
        }
        asm volatile("red.global.add.v4.f32 [%0], {%1, %1, %1, %1};" ::"l"(d + row * 128 + col4 * 4), "f"(1.0f)
                     : "memory");
      }
    }
  } else {
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0 && rank == 0) {
      uint32_t peer_buf, peer_bar;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(peer_buf) : "r"(smem_u32(buf + kBuf / 4)));
      asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(peer_bar) : "r"(smem_u32(&bar)));
      for (int it = 0; it < iters; ++it) {
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         peer_buf),
                     "r"(smem_u32(buf)), "r"(kBuf), "r"(peer_bar)
                     : "memory");
      }
    }
    if (threadIdx.x == 0 && rank == 1) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}"
                     : "=r"(ok)
                     : "r"(smem_u32(&bar))
                     : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

template <int MODE>
void run(const char* name, int grid, int shared_dst, float* dst, long long* dcyc, int cluster) {
  const int iters = MODE == 4 ? 16 : 64;
  const size_t region = (size_t)8 * kBuf / 4;
  const int smem = 2 * kBuf + 1024;
  cudaFuncSetAttribute(red_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = 256;
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, red_kernel<MODE>, dst, region, iters, shared_dst, dcyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, dcyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double mx = 0, sum = 0;
  for (int i = 0; i < grid; ++i) {
    sum += h[i];
    mx = h[i] > mx ? h[i] : mx;
  }
  const double bytes = (double)iters * kBuf;
  printf("{\"case\": \"%s\", \"ctas\": %d, \"cluster\": %d, \"same_dst\": %d, \"B_per_clk_per_sm_mean\": %.2f, "
         "\"B_per_clk_per_sm_slowest\": %.2f, \"err\": \"%s\"}\n",
         name, grid, cluster, shared_dst, bytes / (sum / grid), bytes / mx, cudaGetErrorString(e));
}

int main() {
  float* dst;
  long long* cyc;
  const int sms = 148;
  cudaMalloc(&dst, (size_t)sms * 8 * kBuf + 4096);
  cudaMemset(dst, 0, (size_t)sms * 8 * kBuf);
  cudaMalloc(&cyc, 512 * sizeof(long long));
  for (int g : {1, sms}) {
    run<0>("bulk_reduce_add_f32", g, 0, dst, cyc, 1);
    run<1>("bulk_store", g, 0, dst, cyc, 1);
    run<2>("red_v4_row_per_thread", g, 0, dst, cyc, 1);
    run<3>("red_v4_coalesced", g, 0, dst, cyc, 1);
  }
  run<0>("bulk_reduce_add_f32", sms, 1, dst, cyc, 1);  // every SM into the same 256 KB
  run<4>("bulk_copy_to_peer_smem", 2, 0, dst, cyc, 2);
  run<4>("bulk_copy_to_peer_smem", sms, 0, dst, cyc, 2);
  return 0;
}
