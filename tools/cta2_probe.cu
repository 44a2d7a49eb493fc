// Standalone probe of the cta_group::2 (CTA pair) tcgen05 path on sm_100a,
// ahead of a paired backward kernel.  Not linked into the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2503_10377_b200/csrc \
//        tools/cta2_probe.cu -o tools/cta2_probe -lcuda && tools/cta2_probe
// Modes (cluster of 2 CTAs, 128 threads each; D = A B^T, A [256][128], B [128][128], K = 128):
//   0  cta_group::2 SS, M=256 N=128: CTA c holds A rows [128c,+128) and B rows [64c,+64)
//   1  cta_group::2 TS, M=256 N=128: A rows of CTA c from its own TMEM
//   2  cta_group::2 SS, M=128 N=128: CTA c holds A rows [64c,+64), B rows [64c,+64); D layout dump
//   3  cta_group::1 SS in each CTA of the pair (TMEM allocated with cta_group::2): D_c = A_c B^T
//   4  cta_group::2 SS, M=256 N=128, B MN-major (B stored [k][n], CTA c holds columns [64c,+64))
// Timing (mode+10): thread 0 of the leader issues reps x 8 MMAs; cycles per 8.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100_ptx.cuh"

using namespace sppo::ptx;

__device__ __forceinline__ uint32_t sw128(int r, int c) {  // element (r, c) of a [rows][64] bf16 SW128 sub-tile
  const uint32_t lin = r * 128 + c * 2;
  return lin ^ (((lin >> 7) & 7u) << 4);
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe2(int mode, int reps, int N, const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;          // [128 rows][128 k] K-major: 2 x 16 KB sub-tiles (64-row variant uses 8 KB each)
  uint8_t* sB = smem + 32768;  // B half: [64 rows][128 k] K-major: 2 x 8 KB, or MN-major [128 k][64 n]: 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const bool timing = mode >= 10;
  mode %= 10;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  // ---- stage this CTA's operand slices
  const int a_rows = (mode == 2) ? 64 : 128;
  const int a_row0 = (mode == 2) ? 64 * rank : 128 * rank;
  for (int e = tid; e < a_rows * 128; e += 128) {
    const int r = e / 128, c = e % 128;
    *(__nv_bfloat16*)(sA + (c / 64) * (a_rows * 128) + sw128(r, c % 64)) =
        A[(mode == 3 ? 128 * rank + r : a_row0 + r) * 128 + c];
  }
  if (mode == 3) {  // full B in each CTA
    for (int e = tid; e < 128 * 128; e += 128) {
      const int r = e / 128, c = e % 128;
      *(__nv_bfloat16*)(sB + (c / 64) * 16384 + sw128(r, c % 64)) = B[r * 128 + c];
    }
  } else if (mode == 4) {  // B^T stored [k][n] MN-major: this CTA's 64 n columns
    for (int e = tid; e < 128 * 64; e += 128) {
      const int k = e / 64, n = e % 64;
      *(__nv_bfloat16*)(sB + sw128(k, n)) = B[(64 * rank + n) * 128 + k];
    }
  } else {
    for (int e = tid; e < 64 * 128; e += 128) {
      const int r = e / 128, c = e % 128;
      *(__nv_bfloat16*)(sB + (c / 64) * 8192 + sw128(r, c % 64)) = B[(64 * rank + r) * 128 + c];
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  if (mode == 1) {  // A rows of this CTA into TMEM columns [128, 192) as bf16 pairs
    const int row = warp * 32 + lane;
#pragma unroll
    for (int blk = 0; blk < 4; ++blk) {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = blk * 16 + j;
        const __nv_bfloat16* ap = A + (128 * rank + row) * 128 + 2 * c;
        r[j] = pack_bf16(__bfloat162float(ap[0]), __bfloat162float(ap[1]));
      }
      tmem_st16(tb + ((uint32_t)(warp * 32) << 16) + 128 + blk * 16, r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();

  if (tid == 0 && (rank == 0 || mode == 3)) {
    const int M = (mode == 2) ? 128 : 256;
    const uint32_t idesc = (mode == 3) ? idesc_bf16(128, N, 0, 0) : idesc_bf16(M, N, 0, mode == 4 ? 1 : 0);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      ad[k] = sdesc_kmajor(smem_u32(sA) + (k / 4) * (a_rows * 128) + (k % 4) * 32);
      if (mode == 3)
        bd[k] = sdesc_kmajor(smem_u32(sB) + (k / 4) * 16384 + (k % 4) * 32);
      else if (mode == 4)
        bd[k] = sdesc_mnmajor(smem_u32(sB) + k * 2048, 16384);
      else
        bd[k] = sdesc_kmajor(smem_u32(sB) + (k / 4) * 8192 + (k % 4) * 32);
    }
    const int R = timing ? reps : 1;
    const long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t acc = timing ? 1u : (k > 0 ? 1u : 0u);
        if (mode == 3)
          mma_ss(tb, ad[k], bd[k], idesc, acc);
        else if (mode == 1)
          mma2_ts(tb, tb + 128 + k * 8, bd[k], idesc, acc);
        else
          mma2_ss(tb, ad[k], bd[k], idesc, acc);
      }
    }
    if (mode == 3)
      mma_commit(&bar);
    else
      commit2(&bar);
    mbar_wait(&bar, 0);
    if (timing) cyc[rank] = (clock64() - t0) / R;
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // ---- dump TMEM lanes 0..127, columns 0..127 of this CTA
  const int row = warp * 32 + lane;
  for (int cb = 0; cb < 4; ++cb) {
    uint32_t r[32];
    tmem_ld32(tb + ((uint32_t)(warp * 32) << 16) + cb * 32, r);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) D[(rank * 128 + row) * 128 + cb * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tb) : "memory");
}


// Clean timing: compile-time mode/N, descriptors precomputed, fully unrolled issue.
// K2=1: cta_group::2 (leader issues), else cta_group::1 (both CTAs issue).  TS=1: A from TMEM.
template <int K2, int M, int N, int TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) tbench(int reps, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    if (K2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc<512>(&tmem_base);
    }
  }
  for (int i = tid; i < 131072 / 2; i += 128) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    reinterpret_cast<__nv_bfloat16*>(smem)[i] = __float2bfloat16(((h & 0xFFFF) / 65536.f - 0.5f) * 4.f);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  if (tid == 0 && (rank == 0 || !K2)) {
    constexpr uint32_t idesc = idesc_bf16(M, N, 0, 0);
    const uint32_t sA = smem_u32(smem), sB = smem_u32(smem + 65536);
    constexpr uint32_t a_atom = (K2 ? M / 2 : M) * 128, b_atom = (K2 ? N / 2 : N) * 128;
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      ad[k] = sdesc_kmajor(sA + (k / 4) * a_atom + (k % 4) * 32);
      bd[k] = sdesc_kmajor(sB + (k / 4) * b_atom + (k % 4) * 32);
    }
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (K2) {
          if (TS) mma2_ts(tb, tb + 256 + k * 8, bd[k], idesc, 1); else mma2_ss(tb, ad[k], bd[k], idesc, 1);
        } else {
          if (TS) mma_ts(tb, tb + 256 + k * 8, bd[k], idesc, 1); else mma_ss(tb, ad[k], bd[k], idesc, 1);
        }
      }
    }
    if (K2) commit2(&bar); else mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[rank] = (clock64() - t0) / reps;
  }
  if (K2) mbar_wait(&bar, 0);
  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    if (K2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
    else tmem_dealloc<512>(tb);
  }
}

template <int K2, int M, int N, int TS>
static void run_t(const char* name) {
  long long* dC;
  cudaMalloc(&dC, 16);
  cudaMemset(dC, 0, 16);
  const int smem = 131072 + 1024;
  cudaFuncSetAttribute(tbench<K2, M, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tbench<K2, M, N, TS><<<2, 128, smem>>>(4000, dC);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, dC, 16, cudaMemcpyDeviceToHost);
  const double ideal = 64.0 * (K2 ? M / 2 : M) / 128.0 * N / 128.0 * 8;  // per-SM cycles for 8 x (M x N x 16)
  printf("%-34s %6lld cycles / 8 MMAs  (ideal per SM %4.0f) %s\n", name, h[0], ideal, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(dC);
}

static float bf(float x) {  // round to bf16 and back
  __nv_bfloat16 b = __float2bfloat16(x);
  return __bfloat162float(b);
}

int main(int argc, char** argv) {
  std::vector<__nv_bfloat16> hA(256 * 128), hB(128 * 128);
  std::vector<float> fA(256 * 128), fB(128 * 128);
  srand(1);
  for (int i = 0; i < 256 * 128; ++i) fA[i] = bf((rand() % 17 - 8) / 4.f), hA[i] = __float2bfloat16(fA[i]);
  for (int i = 0; i < 128 * 128; ++i) fB[i] = bf((rand() % 17 - 8) / 4.f), hB[i] = __float2bfloat16(fB[i]);
  std::vector<float> ref(256 * 128);
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < 128; ++n) {
      double s = 0;
      for (int k = 0; k < 128; ++k) s += (double)fA[m * 128 + k] * fB[n * 128 + k];
      ref[m * 128 + n] = (float)s;
    }
  __nv_bfloat16 *dA, *dB;
  float* dD;
  long long* dC;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dD, 256 * 128 * 4);
  cudaMalloc(&dC, 16);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<float> hD(256 * 128);
  for (int mode = 0; mode <= 4; ++mode) {
    cudaMemset(dD, 0, 256 * 128 * 4);
    probe2<<<2, 128, smem>>>(mode, 1, 128, dA, dB, dD, dC);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
    if (mode != 2) {
      double err = 0;
      for (int i = 0; i < 256 * 128; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
      printf("mode %d: max |D - ref| = %g  (D[0]=%g ref=%g, D[128*128]=%g ref=%g)\n", mode, err, hD[0], ref[0],
             hD[128 * 128], ref[128 * 128]);
    } else {
      // where did ref rows 0..127 (M = 128) land?  match each (cta, lane) row against ref rows
      int found = 0;
      for (int c = 0; c < 2; ++c)
        for (int l = 0; l < 128; ++l) {
          int match = -1;
          for (int m = 0; m < 128 && match < 0; ++m) {
            bool ok = true;
            for (int n = 0; n < 128 && ok; ++n) ok = hD[(c * 128 + l) * 128 + n] == ref[m * 128 + n];
            if (ok) match = m;
          }
          if (match >= 0) {
            ++found;
            if (l % 16 == 0 || l % 32 == 31) printf("  mode 2: cta %d lane %3d <- row %3d\n", c, l, match);
          }
        }
      printf("mode 2: %d (cta,lane) rows hold a full ref row\n", found);
    }
  }
  run_t<0, 128, 64, 0>("1cta SS M128 N64");
  run_t<0, 128, 128, 0>("1cta SS M128 N128");
  run_t<0, 128, 256, 0>("1cta SS M128 N256");
  run_t<0, 128, 128, 1>("1cta TS M128 N128");
  run_t<1, 256, 64, 0>("2cta SS M256 N64");
  run_t<1, 256, 128, 0>("2cta SS M256 N128");
  run_t<1, 256, 256, 0>("2cta SS M256 N256");
  run_t<1, 256, 128, 1>("2cta TS M256 N128");
  run_t<1, 128, 128, 0>("2cta SS M128 N128");
  run_t<1, 128, 256, 0>("2cta SS M128 N256");
  // M=128 cta_group::2 layout: run a (D = m + 1), run b (D = n + 1)
  for (int run = 0; run < 2; ++run) {
    std::vector<__nv_bfloat16> pA(256 * 128, __float2bfloat16(0.f)), pB(128 * 128, __float2bfloat16(0.f));
    for (int m = 0; m < 128; ++m) pA[m * 128] = __float2bfloat16(run == 0 ? (float)(m + 1) : 1.f);
    for (int n = 0; n < 128; ++n) pB[n * 128] = __float2bfloat16(run == 0 ? 1.f : (float)(n + 1));
    cudaMemcpy(dA, pA.data(), pA.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, pB.data(), pB.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 256 * 128 * 4);
    probe2<<<2, 128, smem>>>(2, 1, 128, dA, dB, dD, dC);
    cudaDeviceSynchronize();
    cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
    printf("M=128 pair layout, run %s:\n", run == 0 ? "a (value = row+1)" : "b (value = col+1)");
    for (int c = 0; c < 2; ++c)
      for (int l : {0, 1, 15, 16, 31, 32, 33, 63, 64, 65, 95, 96, 127}) {
        printf("  cta %d lane %3d:", c, l);
        for (int col : {0, 1, 31, 32, 63, 64, 65, 127}) printf(" %5g", hD[(c * 128 + l) * 128 + col]);
        printf("\n");
      }
  }
  return 0;
}
