// Persistent tcgen05 GEMM for the per-chunk transformer layer (
// include/sppo_layer.h): D[M][N] = sum_k A(m,k) B(k,n), bf16 operands staged by
// TMA (SWIZZLE_128B) through a kStages-deep shared-memory ring, fp32
// accumulators in TMEM (two buffers, so the epilogue of tile t overlaps the
// main loop of tile t+1), fused epilogues (bias, residual add, GELU with the
// pre-activation saved, GELU backward, fp32 weight-gradient accumulation).
//
// CTA = 192 threads, one per SM (grid = min(tiles, #SMs), static round-robin
// tile schedule in grouped raster order, tile_coords()):
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM alloc + MMA issuer (converged warp, one elected lane issues)
//   warps 2..5  epilogue: warp w reads TMEM lanes 32*(w%4).. (tcgen05.ld 32x32b),
//               thread = one output row, 32 columns per tcgen05.ld
// Operand orientation (a_mn / b_mn) selects K-major or MN-major UMMA smem
// descriptors; the same smem ring serves both (K-major: one box of 64 K x rows;
// MN-major: boxes of 64 MN x 64 K, 8 KB apart = the descriptor's LBO).
#include <cuda.h>
#include <cuda_bf16.h>

#include "../../include/sppo_layer.h"
#include "internal.h"
#include "sm100_ptx.cuh"

namespace sppo {
namespace {

using namespace ptx;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;
constexpr uint32_t kMnBox = 64 * BK * 2;  // 8 KB: one MN-major box (64 MN x 64 K)

template <int BN>
struct Cfg {
  static constexpr uint32_t kABytes = BM * BK * 2;
  static constexpr uint32_t kBBytes = BN * BK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kSmem = kStages * kStageBytes + 1024;
  static constexpr uint32_t kTmemCols = 2 * BN;
};

struct GemmBars {
  uint64_t full[8], empty[8];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

// Tile t -> (m block, n block), grouped raster: kGroupM consecutive m blocks sweep
// the n blocks together, so the CTAs running at one time share a few A row panels
// and B column panels (L2 reuse) instead of all of A.
#ifndef SPPO_GEMM_ACC_RED
#define SPPO_GEMM_ACC_RED 0  // red.global.add for fp32 +=: measured 1246 / 1057 vs 1239 / 1147 TF/s (fc1 / o wgrad)
#endif
#ifndef SPPO_GEMM_GROUP
#define SPPO_GEMM_GROUP 8
#endif
constexpr int kGroupM = SPPO_GEMM_GROUP;
__device__ __forceinline__ void tile_coords(int t, int Mt, int Nt, int& mb, int& nb) {
  const int per_group = kGroupM * Nt;
  const int g = t / per_group, r = t - g * per_group;
  const int m_first = g * kGroupM;
  const int gm = min(Mt - m_first, kGroupM);
  mb = m_first + r % gm;
  nb = r / gm;
}

__device__ __forceinline__ float gelu_f(float u) { return 0.5f * u * (1.f + erff(u * 0.7071067811865476f)); }
__device__ __forceinline__ float gelu_grad_f(float u) {
  return 0.5f * (1.f + erff(u * 0.7071067811865476f)) + u * 0.3989422804014327f * __expf(-0.5f * u * u);
}

__device__ __forceinline__ void load_bf16x32(const void* src, float (&v)[32]) {
  const uint4* p = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 w = __ldg(p + q);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ws[e]));
      v[8 * q + 2 * e] = f.x;
      v[8 * q + 2 * e + 1] = f.y;
    }
  }
}

__device__ __forceinline__ void store_bf16x32(void* dst, const float (&v)[32]) {
  uint4* p = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    p[q] = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                      pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
}

// Epilogue of 32 consecutive columns [n, n+32) of output row `row`.
__device__ __forceinline__ void epilogue32(const GemmParams& p, int row, int n, const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  const int part = n / p.c_part_w;
  const int col = n - part * p.c_part_w;
  if (p.epi == SPPO_EPI_ACC_F32) {
    float* c = static_cast<float*>(p.c[part]) + (size_t)row * p.c_part_w + col;
#if SPPO_GEMM_ACC_RED
    // one writer per element (each tile has one owner): red.add performs the same
    // single fp32 addition as load-add-store, without the load round trip
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(c + 4 * q), "f"(v[4 * q]),
                   "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                   : "memory");
#else
    float4* c4 = reinterpret_cast<float4*>(c);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 t = c4[q];
      t.x += v[4 * q];
      t.y += v[4 * q + 1];
      t.z += v[4 * q + 2];
      t.w += v[4 * q + 3];
      c4[q] = t;
    }
#endif
    return;
  }
  if (p.bias) {
    float b[32];
    load_bf16x32(static_cast<const __nv_bfloat16*>(p.bias) + n, b);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += b[i];
  }
  const size_t idx = (size_t)row * p.N + n;
  if (p.epi == SPPO_EPI_STORE) {
    if (p.residual) {
      float x[32];
      load_bf16x32(static_cast<const __nv_bfloat16*>(p.residual) + idx, x);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += x[i];
    }
  } else if (p.epi == SPPO_EPI_GELU) {
    store_bf16x32(static_cast<__nv_bfloat16*>(p.aux_out) + idx, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = gelu_f(v[i]);
  } else {  // SPPO_EPI_DGELU
    float u[32];
    load_bf16x32(static_cast<const __nv_bfloat16*>(p.aux_in) + idx, u);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_f(u[i]);
  }
  store_bf16x32(static_cast<__nv_bfloat16*>(p.c[part]) + (size_t)row * p.c_part_w + col, v);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
                const __grid_constant__ CUtensorMap ta2, const __grid_constant__ CUtensorMap tb,
                const __grid_constant__ GemmParams p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ GemmBars bars;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id(), lane = lane_id();
  const int Mt = (p.M + BM - 1) / BM, Nt = p.N / BN, Kt = (p.K + BK - 1) / BK;
  const int tiles = Mt * Nt;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.acc_full[b], 1);
      mbar_init(&bars.acc_empty[b], 128);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&ta0);
    prefetch_tmap(&tb);
    if (p.a_parts > 1) prefetch_tmap(&ta1);
    if (p.a_parts > 2) prefetch_tmap(&ta2);
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(&bars.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, Mt, Nt, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        for (int kb = 0; kb < Kt; ++kb) {
          mbar_wait(&bars.empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * C::kStageBytes;
          uint8_t* sB = sA + C::kABytes;
          mbar_arrive_expect_tx(&bars.full[stage], C::kStageBytes);
          const int k0 = kb * BK;
          if (!p.a_mn) {  // A [M][K], split along K
            const int part = k0 / p.a_part_w;
            const CUtensorMap* m = part == 0 ? &ta0 : (part == 1 ? &ta1 : &ta2);
            tma_load_2d(sA, m, &bars.full[stage], k0 - part * p.a_part_w, m0);
          } else {  // A [K][M], split along M
            const int part = m0 / p.a_part_w;
            const CUtensorMap* m = part == 0 ? &ta0 : (part == 1 ? &ta1 : &ta2);
            const int mc = m0 - part * p.a_part_w;
#pragma unroll
            for (int b = 0; b < BM / 64; ++b) tma_load_2d(sA + b * kMnBox, m, &bars.full[stage], mc + 64 * b, k0);
          }
          if (!p.b_mn) {
            tma_load_2d(sB, &tb, &bars.full[stage], k0, n0);
          } else {
#pragma unroll
            for (int b = 0; b < BN / 64; ++b) tma_load_2d(sB + b * kMnBox, &tb, &bars.full[stage], n0 + 64 * b, k0);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t idesc = idesc_bf16(BM, BN, p.a_mn, p.b_mn);
    const uint32_t sbase = smem_u32(smem);
    // base descriptors once; a stage / K=16 step adds (byte offset >> 4) to the
    // start-address field (smem addresses < 2^18: no carry out of the field)
    const uint64_t a0 = p.a_mn ? sdesc_mnmajor(sbase, kMnBox) : sdesc_kmajor(sbase);
    const uint64_t b0 = p.b_mn ? sdesc_mnmajor(sbase + C::kABytes, kMnBox) : sdesc_kmajor(sbase + C::kABytes);
    const uint32_t a_k = (p.a_mn ? 2048u : 32u) >> 4, b_k = (p.b_mn ? 2048u : 32u) >> 4;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(&bars.acc_empty[buf], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + buf * BN;
      for (int kb = 0; kb < Kt; ++kb) {
        mbar_wait(&bars.full[stage], phase);
        tc_fence_after();
        const uint64_t so = (uint64_t)((stage * C::kStageBytes) >> 4);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          mma_ss_w(d, a0 + so + k * a_k, b0 + so + k * b_k, idesc, (kb | k) != 0);
        mma_commit_w(&bars.empty[stage]);
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      mma_commit_w(&bars.acc_full[buf]);
    }
  } else {
    // ===================== epilogue =====================
    const int lane_base = (warp & 3) * 32;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int buf = it & 1;
      int mb, nb;
      tile_coords(t, Mt, Nt, mb, nb);
      const int m0 = mb * BM, n0 = nb * BN;
      mbar_wait(&bars.acc_full[buf], (it >> 1) & 1);
      tc_fence_after();
      const int row = m0 + lane_base + lane;
      const uint32_t taddr = tmem + ((uint32_t)lane_base << 16) + buf * BN;
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        uint32_t r[32];
        tmem_ld32(taddr + cc * 32, r);
        tmem_wait_ld_regs(r);
        if (cc == BN / 32 - 1) {  // every column of this buffer is in registers: release it
          tc_fence_before();
          mbar_arrive(&bars.acc_empty[buf]);
        }
        if (row < p.M) epilogue32(p, row, n0 + cc * 32, r);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------- CTA-pair variant
// Cluster of 2 CTAs shares one 256 x 256 tile: tcgen05.mma.cta_group::2 M=256
// N=256 issued by the leader; CTA r holds A rows [128r, 128r+128) and B columns
// [128r, 128r+128) of the tile in its own smem (half of B per SM: 32 KB of
// operands per 64-deep K block instead of 48 KB), its TMEM receives its 128 D
// rows x 256 columns.  Both CTAs' TMA loads complete on the leader's full
// barrier; MMA commits multicast to both CTAs; both CTAs' epilogue threads
// release an accumulator buffer on the leader's acc_empty barrier.
#ifndef SPPO_GEMM_PAIR_BK
#define SPPO_GEMM_PAIR_BK 128  // measured: 128 vs 64 -> x W^T 1444-1519 vs 1330-1373 TF/s, dy W 1471 vs 1162-1249
#endif
// K depth of one pipeline stage (64 | 128).  The MMA issuer waits on one barrier
// and commits once per stage, so a deeper stage (8 MMAs instead of 4) halves that
// per-stage overhead on the issue path, which runs nearly synchronously with the
// tensor pipe; 3 stages x 64 KB still fill the 192 KB ring.
constexpr int PBK = SPPO_GEMM_PAIR_BK;
constexpr int kPairStages = PBK == 64 ? 6 : 3;
constexpr uint32_t kPairA = 128 * PBK * 2, kPairB = 128 * PBK * 2, kPairStage = kPairA + kPairB;
constexpr uint32_t kPairMnBlock = 64 * PBK * 2;  // one 64-wide MN block over the stage's K depth
constexpr int kPairSmem = kPairStages * kPairStage + 1024;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
                 const __grid_constant__ CUtensorMap ta2, const __grid_constant__ CUtensorMap tb,
                 const __grid_constant__ GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ GemmBars bars;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int Mt = (p.M + 255) / 256, Nt = p.N / 256, Kt = (p.K + PBK - 1) / PBK;
  const int tiles = Mt * Nt;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPairStages; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.acc_full[b], 1);
      mbar_init(&bars.acc_empty[b], 256);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&ta0);
    prefetch_tmap(&tb);
    if (p.a_parts > 1) prefetch_tmap(&ta1);
    if (p.a_parts > 2) prefetch_tmap(&ta2);
  }
  if (warp == 1) tmem_alloc_pair<512>(&bars.tmem_base);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < tiles; t += ncl) {
        int mb, nb;
        tile_coords(t, Mt, Nt, mb, nb);
        const int m0 = mb * 256 + 128 * (int)rank, n0 = nb * 256 + 128 * (int)rank;
        for (int kb = 0; kb < Kt; ++kb) {
          mbar_wait(&bars.empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * kPairStage;
          uint8_t* sB = sA + kPairA;
          if (leader) mbar_arrive_expect_tx(&bars.full[stage], 2 * kPairStage);
          const uint32_t Lf = mapa(smem_u32(&bars.full[stage]), 0);
          const int k0 = kb * PBK;
#pragma unroll
          for (int h = 0; h < PBK / 64; ++h) {  // 64-deep K halves of the stage
            const int kh = k0 + 64 * h;
            if (!p.a_mn) {  // K-major: box h at +16 KB * h
              const int part = kh / p.a_part_w;
              const CUtensorMap* m = part == 0 ? &ta0 : (part == 1 ? &ta1 : &ta2);
              tma_load_2d_pair(sA + h * 16384, m, Lf, kh - part * p.a_part_w, m0);
            } else {  // MN-major: block b (64 MN) holds all PBK K rows, half h at +8 KB * h
              const int part = m0 / p.a_part_w;
              const CUtensorMap* m = part == 0 ? &ta0 : (part == 1 ? &ta1 : &ta2);
              const int mc = m0 - part * p.a_part_w;
              tma_load_2d_pair(sA + h * kMnBox, m, Lf, mc, kh);
              tma_load_2d_pair(sA + kPairMnBlock + h * kMnBox, m, Lf, mc + 64, kh);
            }
            if (!p.b_mn) {
              tma_load_2d_pair(sB + h * 16384, &tb, Lf, kh, n0);
            } else {
              tma_load_2d_pair(sB + h * kMnBox, &tb, Lf, n0, kh);
              tma_load_2d_pair(sB + kPairMnBlock + h * kMnBox, &tb, Lf, n0 + 64, kh);
            }
          }
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      const uint32_t idesc = idesc_bf16(256, 256, p.a_mn, p.b_mn);
      const uint32_t sbase = smem_u32(smem);
      const uint64_t a0 = p.a_mn ? sdesc_mnmajor(sbase, kPairMnBlock) : sdesc_kmajor(sbase);
      const uint64_t b0 = p.b_mn ? sdesc_mnmajor(sbase + kPairA, kPairMnBlock) : sdesc_kmajor(sbase + kPairA);
      // K=16 step k: MN-major +2 KB * k (the K halves of a block are contiguous);
      // K-major +32 B * (k % 4) within a 64-deep box, +16 KB per box
      auto koff = [](int k, int mn) -> uint64_t {
        return (uint64_t)((mn ? 2048u * k : 16384u * (k >> 2) + 32u * (k & 3)) >> 4);
      };
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cid; t < tiles; t += ncl, ++it) {
        const int buf = it & 1;
        mbar_wait(&bars.acc_empty[buf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * 256;
        for (int kb = 0; kb < Kt; ++kb) {
          mbar_wait(&bars.full[stage], phase);
          tc_fence_after();
          const uint64_t so = (uint64_t)((stage * kPairStage) >> 4);
#pragma unroll
          for (int k = 0; k < PBK / 16; ++k)
            mma2_ss_w(d, a0 + so + koff(k, p.a_mn), b0 + so + koff(k, p.b_mn), idesc, (kb | k) != 0);
          mma2_commit_w(&bars.empty[stage]);
          if (++stage == kPairStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma2_commit_w(&bars.acc_full[buf]);
      }
    }
  } else {
    const int lane_base = (warp & 3) * 32;
    int it = 0;
    for (int t = cid; t < tiles; t += ncl, ++it) {
      const int buf = it & 1;
      int mb, nb;
      tile_coords(t, Mt, Nt, mb, nb);
      const int m0 = mb * 256 + 128 * (int)rank, n0 = nb * 256;
      mbar_wait(&bars.acc_full[buf], (it >> 1) & 1);
      tc_fence_after();
      const int row = m0 + lane_base + lane;
      const uint32_t taddr = tmem + ((uint32_t)lane_base << 16) + buf * 256;
      const uint32_t Le = mapa(smem_u32(&bars.acc_empty[buf]), 0);
#pragma unroll 1
      for (int cc = 0; cc < 8; ++cc) {
        uint32_t r[32];
        tmem_ld32(taddr + cc * 32, r);
        tmem_wait_ld_regs(r);
        if (cc == 7) {
          tc_fence_before();
          mbar_arrive_cluster(Le);
        }
        if (row < p.M) epilogue32(p, row, n0 + cc * 32, r);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
}

cudaError_t launch_pair(const CUtensorMap* ta, const CUtensorMap* tb, const GemmParams& p, int num_sms,
                        cudaStream_t s) {
  cudaError_t e = ensure_smem_attr((const void*)gemm2_kernel, kPairSmem);
  if (e != cudaSuccess) return e;
  const int tiles = ((p.M + 255) / 256) * (p.N / 256);
  const int clusters = tiles < num_sms / 2 ? tiles : num_sms / 2;
  gemm2_kernel<<<2 * clusters, kThreads, kPairSmem, s>>>(ta[0], ta[1], ta[2], *tb, p);
  return cudaGetLastError();
}

template <int BN>
cudaError_t launch_bn(const CUtensorMap* ta, const CUtensorMap* tb, const GemmParams& p, int num_sms,
                      cudaStream_t s) {
  using C = Cfg<BN>;
  cudaError_t e = ensure_smem_attr((const void*)gemm_kernel<BN>, C::kSmem);
  if (e != cudaSuccess) return e;
  const int tiles = ((p.M + BM - 1) / BM) * (p.N / BN);
  const int grid = tiles < num_sms ? tiles : num_sms;
  gemm_kernel<BN><<<grid, kThreads, C::kSmem, s>>>(ta[0], ta[1], ta[2], *tb, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm_sm100(const void* tmap_a3, const void* tmap_b, const GemmParams& p, int bn, bool pair,
                              int num_sms, cudaStream_t s) {
  const CUtensorMap* ta = static_cast<const CUtensorMap*>(tmap_a3);
  const CUtensorMap* tb = static_cast<const CUtensorMap*>(tmap_b);
  if (pair) return launch_pair(ta, tb, p, num_sms, s);
  return bn == 256 ? launch_bn<256>(ta, tb, p, num_sms, s) : launch_bn<128>(ta, tb, p, num_sms, s);
}

}  // namespace sppo
