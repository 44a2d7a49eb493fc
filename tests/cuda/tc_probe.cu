// Test-only probe of the sm_100a building blocks used by the attention kernels:
// UMMA smem descriptors (K-major and MN-major, SWIZZLE_128B), the BF16
// instruction descriptor, A-operand from TMEM (packed bf16 pairs), tcgen05
// ld/st 32x32b, tcgen05.commit -> mbarrier, and TMA SW128 tile loads.
// One CTA computes a single 128 x N x 128 product; tests/test_gpu_probe.py
// compares it with torch.  Not linked into the product library.
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../paper_2503_10377_b200/csrc/sm100_ptx.cuh"

using namespace sppo::ptx;

namespace {

// byte offset of element (r, c) of a [rows][64] bf16 SW128 sub-tile
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  const uint32_t lin = r * 128 + c * 2;
  return lin ^ (((lin >> 7) & 7u) << 4);
}

// mode 0: D = A * B^T, A [128][128] K-major (row = m), B [N][128] K-major (row = n)
// mode 1: D = A * B,   A K-major, B stored [128 (k)][N] (MN-major)
// mode 2: D = A * B,   A from TMEM (bf16 pairs), B stored [128][N] (MN-major)
// mode 3: D = At^T * B, A stored transposed At [128 (k)][128 (m)] (MN-major), B stored [128][N] MN-major
template <int N>
__global__ void __launch_bounds__(128, 1) probe_kernel(int mode, const __nv_bfloat16* A, const __nv_bfloat16* B,
                                                       float* D, const CUtensorMap* tmA, const CUtensorMap* tmB) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;              // 2 sub-tiles of 16 KB
  uint8_t* sB = smem + 32768;      // up to 2 sub-tiles of 16 KB
  __shared__ uint64_t bar_mma, bar_tma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    mbar_init(&bar_mma, 1);
    mbar_init(&bar_tma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;

  // ---- stage operands
  if (tmA) {
    if (tid == 0) {
      // A: [128 rows][128 cols] as two boxes of 64 columns (rows = m for K-major, k for MN-major)
      // B: rows = n (K-major, N rows) or k (MN-major, 128 rows); boxes of 64 columns.
      const int b_rows = (mode == 0) ? N : 128;
      const int b_boxes = (mode == 0) ? 2 : N / 64;
      const uint32_t bytes = 2 * 16384 + b_boxes * b_rows * 128;
      mbar_arrive_expect_tx(&bar_tma, bytes);
      tma_load_3d(sA, tmA, &bar_tma, 0, 0, 0);
      tma_load_3d(sA + 16384, tmA, &bar_tma, 64, 0, 0);
      for (int bx = 0; bx < b_boxes; ++bx) tma_load_3d(sB + bx * b_rows * 128, tmB, &bar_tma, 64 * bx, 0, 0);
    }
    mbar_wait(&bar_tma, 0);
  } else {
    // manual SW128 staging: element (r, c) of a [rows][128|N] matrix goes to
    // sub-tile c/64 at sw128(r, c%64)
    for (int e = tid; e < 128 * 128; e += 128) {
      const int r = e / 128, c = e % 128;
      *(__nv_bfloat16*)(sA + (c / 64) * 16384 + sw128(r, c % 64)) = A[e];
    }
    const int b_rows = (mode == 0) ? N : 128, b_cols = (mode == 0) ? 128 : N;
    for (int e = tid; e < b_rows * b_cols; e += 128) {
      const int r = e / b_cols, c = e % b_cols;
      *(__nv_bfloat16*)(sB + (c / 64) * (b_rows * 128) + sw128(r, c % 64)) = B[e];
    }
    fence_proxy_async_smem();
  }
  if (mode == 2) {
    // A into TMEM columns [128, 192): thread owns row 32*warp + lane, col c = (A[2c], A[2c+1])
    const int row = warp * 32 + lane;
#pragma unroll
    for (int blk = 0; blk < 4; ++blk) {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = blk * 16 + j;
        r[j] = pack_bf16(__bfloat162float(A[row * 128 + 2 * c]), __bfloat162float(A[row * 128 + 2 * c + 1]));
      }
      tmem_st16(tbase + ((uint32_t)(warp * 32) << 16) + 128 + blk * 16, r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // ---- MMA
  if (tid == 0) {
    const uint32_t a_mn = (mode == 3) ? 1 : 0;
    const uint32_t b_mn = (mode == 0) ? 0 : 1;
    const uint32_t idesc = idesc_bf16(128, N, a_mn, b_mn);
    const int b_rows = (mode == 0) ? N : 128;
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
      uint64_t bdesc;
      if (b_mn)
        bdesc = sdesc_mnmajor(smem_u32(sB) + k * 2048, b_rows * 128);
      else
        bdesc = sdesc_kmajor(smem_u32(sB) + (k / 4) * (b_rows * 128) + (k % 4) * 32);
      if (mode == 2) {
        mma_ts(tbase, tbase + 128 + k * 8, bdesc, idesc, k > 0);
      } else {
        uint64_t adesc = a_mn ? sdesc_mnmajor(smem_u32(sA) + k * 2048, 16384)
                              : sdesc_kmajor(smem_u32(sA) + (k / 4) * 16384 + (k % 4) * 32);
        mma_ss(tbase, adesc, bdesc, idesc, k > 0);
      }
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  // ---- D rows -> global
  const int row = warp * 32 + lane;
#pragma unroll
  for (int cb = 0; cb < N / 32; ++cb) {
    uint32_t r[32];
    tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + cb * 32, r);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) D[row * N + cb * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

// MMA throughput microbenchmark: thread 0 issues `reps` x 8 MMAs (128 x N x 16
// each, K = 128 per group) of one operand mode back to back, commit, wait; the
// clock64 delta per 128x N x 128 group is written to out[0].  Operands are
// uninitialised smem (values irrelevant for timing).
template <int N>
__global__ void __launch_bounds__(128, 1) mma_bench_kernel(int mode, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  // operand contents: mode >= 10 -> zeros, else N(0,1)-like bf16 from a hash (data can affect TC power/speed)
  const int fill = mode >= 10 ? 0 : 1;
  mode %= 10;
  for (int i = threadIdx.x; i < 65536 / 2; i += 128) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 15;
    const float u = ((h & 0xFFFF) / 65536.f + ((h >> 16) & 0xFFFF) / 65536.f + ((h * 7u) & 0xFFFF) / 65536.f - 1.5f) * 2.f;
    reinterpret_cast<__nv_bfloat16*>(smem)[i] = __float2bfloat16(fill ? u : 0.f);
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t sA = smem_u32(smem), sB = smem_u32(smem + 32768);
    // mode 4: SS with A MN-major, B K-major
    const uint32_t a_mn = (mode == 3 || mode == 4) ? 1 : 0, b_mn = (mode == 0 || mode == 4) ? 0 : 1;
    const uint32_t idesc = idesc_bf16(128, N, a_mn, b_mn);
    uint64_t ad[8], bd[8];  // descriptors precomputed: the timed loop only issues
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      bd[k] = b_mn ? sdesc_mnmajor(sB + k * 2048, 16384) : sdesc_kmajor(sB + (k / 4) * 16384 + (k % 4) * 32);
      ad[k] = a_mn ? sdesc_mnmajor(sA + k * 2048, 16384) : sdesc_kmajor(sA + (k / 4) * 16384 + (k % 4) * 32);
    }
    const long long t0 = clock64();
    if (mode == 2) {
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ts(tb, tb + 128 + k * 8, bd[k], idesc, 1);
      }
    } else {
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int k = 0; k < 8; ++k) mma_ss(tb, ad[k], bd[k], idesc, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[0] = (t1 - t0) / reps;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tb);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int encode(CUtensorMap* m, const void* p, int rows, int cols, int box_rows) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return -1;
  // 3-D view {cols, 1, rows} to exercise the same rank as the product kernels
  cuuint64_t dims[3] = {(cuuint64_t)cols, 1, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)cols * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = ((EncodeTiledFn)fn)(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(p), dims, strides, box,
                                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

}  // namespace

extern "C" long long tc_mma_bench(int mode, int N, int reps) {
  long long* d = nullptr;
  long long h = -1;
  if (cudaMalloc(&d, sizeof(long long)) != cudaSuccess) return -1;
  const int smem = 65536 + 1024;
  if (N == 128) {
    cudaFuncSetAttribute(mma_bench_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_bench_kernel<128><<<1, 128, smem>>>(mode, reps, d);
  } else {
    cudaFuncSetAttribute(mma_bench_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_bench_kernel<64><<<1, 128, smem>>>(mode, reps, d);
  }
  if (cudaDeviceSynchronize() == cudaSuccess) cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}

extern "C" int tc_probe_run(int mode, int N, int use_tma, const void* A, const void* B, float* D) {
  CUtensorMap* maps = nullptr;
  if (use_tma) {
    CUtensorMap h[2];
    const int b_rows = (mode == 0) ? N : 128, b_cols = (mode == 0) ? 128 : N;
    if (encode(&h[0], A, 128, 128, 128) || encode(&h[1], B, b_rows, b_cols, b_rows)) return -10;
    if (cudaMalloc(&maps, sizeof h) != cudaSuccess) return -11;
    cudaMemcpy(maps, h, sizeof h, cudaMemcpyHostToDevice);
  }
  const int smem = 65536 + 1024;
  cudaError_t e;
  if (N == 128) {
    cudaFuncSetAttribute(probe_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe_kernel<128><<<1, 128, smem>>>(mode, (const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D,
                                        maps ? maps : nullptr, maps ? maps + 1 : nullptr);
  } else if (N == 64) {
    cudaFuncSetAttribute(probe_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe_kernel<64><<<1, 128, smem>>>(mode, (const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D,
                                       maps ? maps : nullptr, maps ? maps + 1 : nullptr);
  } else {
    return -1;
  }
  e = cudaDeviceSynchronize();
  if (maps) cudaFree(maps);
  return e == cudaSuccess ? 0 : (int)e;
}
