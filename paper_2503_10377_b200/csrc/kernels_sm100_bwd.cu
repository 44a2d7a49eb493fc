// sm_100a tensor-core backward of chunked causal attention.
//
// Method (P:356 [§5.1]; oracle/attention.py chunked_attention_bwd): for chunk
// i and every prior chunk j in the window,
//   P = exp(tau Q_i K_j^T - LSE_i),  dV_j += P^T dO_i,  dP = dO_i V_j^T,
//   dS = P (dP - Delta_i),  dQ_i += tau dS K_j,  dK_j += tau dS^T Q_i.
//
// B200 design: KV-stationary.  CTA = one 128-key tile of
// chunk j (one head), looping over the causally relevant 128-row Q tiles of
// chunk i.  512 threads, 1 CTA / SM:
//   warps 0-3   dQ reducer: tcgen05.ld dQ -> swizzled smem -> TMA reduce-add
//               (cp.reduce.async.bulk.tensor .add.f32) into the fp32 dQ_i acc.
//   warps 4-11  compute: P (exp2) and dS; WG A owns q columns 0-63, WG B 64-127
//               of every TMEM lane (= key row).
//   warp 12     MMA issuer (one thread), warp 13 TMA producer, warp 14 TMEM alloc.
// TMEM (512 cols): S/P [0,128) | dV [128,256) | dP/dS/dQ [256,384) | dK [384,512)
// 5 MMAs per Q tile (M=N=128, K=128):  S = K Q^T, dP = V dO^T (both K-major),
// dV += P^T dO and dK += dS^T Q (A = P / dS straight from TMEM, B MN-major),
// dQ = dS K (A = dS from smem, MN-major).  tau is folded into dS.
#include <cuda.h>
#include <math.h>

#include "internal.h"
#include "sm100_ptx.cuh"

namespace sppo {
namespace {
using namespace ptx;

constexpr int BQ = 128, BKV = 128, HD = 128;
constexpr int kThreads = 512;
constexpr uint32_t kTile = BQ * HD * 2;  // 32 KB bf16 tile (two 16 KB SW128 boxes)
constexpr uint32_t kHalf = kTile / 2;
// dynamic smem map (bytes); the base is 1024-aligned (no static smem is used)
constexpr uint32_t kOffK = 0;
constexpr uint32_t kOffV = kOffK + kTile;
constexpr uint32_t kOffQ = kOffV + kTile;         // 2 stages
constexpr uint32_t kOffDO = kOffQ + 2 * kTile;    // 1 stage
constexpr uint32_t kOffDS = kOffDO + kTile;       // dS, MN-major A of dQ = dS K
constexpr uint32_t kOffDQ = kOffDS + kTile;       // 2 x 16 KB fp32 reduce staging
constexpr uint32_t kOffLSE = kOffDQ + 2 * 16384;  // 2 x 128 fp32 (LSE * log2 e)
constexpr uint32_t kOffDelta = kOffLSE + 1024;    // 2 x 128 fp32
constexpr uint32_t kOffBars = kOffDelta + 1024;
constexpr uint32_t kSmemBytes = kOffBars + 256;
static_assert(kSmemBytes <= 232448, "smem budget");

constexpr uint32_t kIdescSS = idesc_bf16(128, 128, 0, 0);   // K-major x K-major
constexpr uint32_t kIdescTS = idesc_bf16(128, 128, 0, 1);   // TMEM A x MN-major B
constexpr uint32_t kIdescDQ = idesc_bf16(128, 128, 1, 1);   // MN-major A x MN-major B
constexpr float kLog2e = 1.4426950408889634f;
#ifndef SPPO_DQ_DIRECT_RED
#define SPPO_DQ_DIRECT_RED 0  // measured: direct REDG doubles the tile period (L2/LSU bound)
#endif
constexpr bool kDqDirectRed = SPPO_DQ_DIRECT_RED;  // dQ: red.global from registers (1) or TMA reduce (0)

struct Bars {
  uint64_t kv_full;
  uint64_t q_full[2], q_empty[2];
  uint64_t do_full, do_empty;
  uint64_t s_full, dp_full, p_full, ds_full;
  uint64_t dq_full, dq_free;
  uint64_t dkdv_done;
  uint32_t tmem_base;
};

__device__ __forceinline__ const CUtensorMap* tmap(const Sm100Bwd& a, int slot) {
  return reinterpret_cast<const CUtensorMap*>(a.desc_table) + slot;
}

__device__ __forceinline__ uint32_t sw128(int r, int byte_in_row) {
  const uint32_t lin = r * 128 + byte_in_row;
  return lin ^ (((lin >> 7) & 7u) << 4);
}

__global__ void __launch_bounds__(kThreads, 1) bwd_kernel(const __grid_constant__ Sm100Bwd a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars& bars = *reinterpret_cast<Bars*>(smem + kOffBars);
  float* sLSE = reinterpret_cast<float*>(smem + kOffLSE);
  float* sDelta = reinterpret_cast<float*>(smem + kOffDelta);
  const BwdParams& p = a.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;

  // ---- which key tile: window chunk c, tile kt within it
  int c = 0;
  while (c + 1 < a.n && a.tile_base[c + 1] <= (int)blockIdx.x) ++c;
  const int kt = blockIdx.x - a.tile_base[c];
  const int kv_row0 = kt * BKV;                    // row within chunk j
  const int kv_len = min(BKV, a.len[c] - kv_row0);  // valid keys in this tile
  const int kvp0 = a.start[c] + kv_row0;           // absolute position of key row 0
  // Q tiles of chunk i with some row at position >= kvp0
  const int q_tiles = (p.q_len + BQ - 1) / BQ;
  const int qt_first = max(0, (kvp0 - p.q_start) / BQ);
  const int M = q_tiles - qt_first;
  const int rot = (int)((blockIdx.x * 7u + blockIdx.y * 13u) % (uint32_t)M);  // spread dQ reduce traffic
  auto qtile = [&](int m) { return qt_first + (m + rot) % M; };

  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 atoms need 1024 B alignment
    mbar_init(&bars.kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars.q_full[s], 33);
      mbar_init(&bars.q_empty[s], 1);
    }
    mbar_init(&bars.do_full, 33);
    mbar_init(&bars.do_empty, 1);
    mbar_init(&bars.s_full, 1);
    mbar_init(&bars.dp_full, 1);
    mbar_init(&bars.p_full, 256);
    mbar_init(&bars.ds_full, 256);
    mbar_init(&bars.dq_full, 1);
    mbar_init(&bars.dq_free, 128);
    mbar_init(&bars.dkdv_done, 1);
    fence_mbar_init();
  }
  if (warp == 14) tmem_alloc<512>(&bars.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const uint32_t tS = tmem, tdV = tmem + 128, tdP = tmem + 256, tdK = tmem + 384;
  // debug trace of CTA (0,0): clock64 per pipeline event (SPPO_TRACE)
  unsigned long long* tr = (p.trace && blockIdx.x == 0 && blockIdx.y == 0) ? p.trace : nullptr;
#define TR(slot, it)                                                              \
  do {                                                                            \
    if (tr && (it) < kTraceIters) tr[(it) * kTraceSlots + (slot)] = clock64();   \
  } while (0)

  if (warp >= 12) {
    setmaxnreg_dec<104>();
    if (warp == 13) {
      // ===================== TMA producer (+ LSE / Delta vectors) =====================
      const CUtensorMap* mq = tmap(a, a.q_slot);
      const CUtensorMap* mdo = tmap(a, a.do_slot);
      if (lane == 0) {
        const CUtensorMap* mk = tmap(a, a.slots.k[c]);
        const CUtensorMap* mv = tmap(a, a.slots.v[c]);
        mbar_arrive_expect_tx(&bars.kv_full, 2 * kTile);
        tma_load_3d(smem + kOffK, mk, &bars.kv_full, 0, head, kv_row0);
        tma_load_3d(smem + kOffK + kHalf, mk, &bars.kv_full, 64, head, kv_row0);
        tma_load_3d(smem + kOffV, mv, &bars.kv_full, 0, head, kv_row0);
        tma_load_3d(smem + kOffV + kHalf, mv, &bars.kv_full, 64, head, kv_row0);
      }
      const float* lse_h = p.lse + (size_t)head * p.q_len;
      const float* delta_h = p.delta + (size_t)head * p.q_len;
      for (int m = 0; m < M; ++m) {
        const int s = m & 1;
        const int q0 = qtile(m) * BQ;
        mbar_wait(&bars.q_empty[s], ((m >> 1) & 1) ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&bars.q_full[s], kTile);
          tma_load_3d(smem + kOffQ + s * kTile, mq, &bars.q_full[s], 0, head, q0);
          tma_load_3d(smem + kOffQ + s * kTile + kHalf, mq, &bars.q_full[s], 64, head, q0);
        }
        {
          float4 w;
          float* wp = reinterpret_cast<float*>(&w);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = q0 + lane * 4 + k;
            wp[k] = r < p.q_len ? lse_h[r] * kLog2e : INFINITY;  // OOB row -> P = 0
          }
          *reinterpret_cast<float4*>(sLSE + s * 128 + lane * 4) = w;  // one conflict-free STS.128
        }
        if (lane == 0) TR(15, m);
        mbar_arrive(&bars.q_full[s]);
        mbar_wait(&bars.do_empty, (m & 1) ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&bars.do_full, kTile);
          tma_load_3d(smem + kOffDO, mdo, &bars.do_full, 0, head, q0);
          tma_load_3d(smem + kOffDO + kHalf, mdo, &bars.do_full, 64, head, q0);
        }
        {
          float4 w;
          float* wp = reinterpret_cast<float*>(&w);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = q0 + lane * 4 + k;
            wp[k] = r < p.q_len ? delta_h[r] : 0.f;
          }
          *reinterpret_cast<float4*>(sDelta + s * 128 + lane * 4) = w;
        }
        mbar_arrive(&bars.do_full);
      }
    } else if (warp == 12) {
      // ===================== MMA issuer (whole warp, converged; one elected lane issues) =====================
      // Base descriptors computed once; a k-step only adds (byte offset >> 4) to the
      // 14-bit start-address field (smem < 256 KB, so no carry leaves the field).
      const uint64_t dK_k = sdesc_kmajor(smem_u32(smem + kOffK)), dV_k = sdesc_kmajor(smem_u32(smem + kOffV));
      const uint64_t dDO_k = sdesc_kmajor(smem_u32(smem + kOffDO));
      const uint64_t dDO_mn = sdesc_mnmajor(smem_u32(smem + kOffDO), kHalf);
      const uint64_t dDS_mn = sdesc_mnmajor(smem_u32(smem + kOffDS), kHalf);
      const uint64_t dK_mn = sdesc_mnmajor(smem_u32(smem + kOffK), kHalf);
      const uint64_t dQ_k0 = sdesc_kmajor(smem_u32(smem + kOffQ));
      const uint64_t dQ_mn0 = sdesc_mnmajor(smem_u32(smem + kOffQ), kHalf);
      constexpr uint64_t kStageStep = kTile >> 4;
      auto koff = [](int k) { return (uint64_t)(((k >> 2) * kHalf + (k & 3) * 32) >> 4); };  // K-major k-step
      auto moff = [](int k) { return (uint64_t)((k * 2048) >> 4); };                         // MN-major k-step
      auto mma_kmajor = [&](uint32_t d, uint64_t A, uint64_t B) {  // D = A B^T, both [128][128] K-major
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) mma_ss_w(d, A + koff(k), B + koff(k), kIdescSS, k > 0);
      };
      // D (+)= A[tmem] B (B MN-major).  A (P or dS, bf16 pairs) of q columns 64g..64g+63
      // sits in TMEM columns [64g, 64g+32) of its region (each WG writes its own half).
      auto mma_tmemA = [&](uint32_t d, uint32_t tA, uint64_t B, bool acc) {
#pragma unroll
        for (int k = 0; k < BQ / 16; ++k)
          mma_ts_w(d, tA + (k >> 2) * 64 + (k & 3) * 8, B + moff(k), kIdescTS, (acc || k > 0) ? 1u : 0u);
      };
      auto q_k = [&](int m) { return dQ_k0 + (m & 1) * kStageStep; };
      auto q_mn = [&](int m) { return dQ_mn0 + (m & 1) * kStageStep; };
      mbar_wait(&bars.kv_full, 0);
      mbar_wait(&bars.q_full[0], 0);
      tc_fence_after();
      mma_kmajor(tS, dK_k, q_k(0));  // S(0) = K Q^T
      mma_commit_w(&bars.s_full);
      for (int m = 0; m < M; ++m) {
        TR(0, m);
        mbar_wait(&bars.do_full, m & 1);
        if (m > 0) mbar_wait(&bars.dq_free, (m - 1) & 1);  // reducer has read dQ(m-1) out of TMEM
        tc_fence_after();
        TR(1, m);
        mma_kmajor(tdP, dV_k, dDO_k);  // dP = V dO^T
        mma_commit_w(&bars.dp_full);
        mbar_wait(&bars.p_full, m & 1);
        tc_fence_after();
        TR(2, m);
        mma_tmemA(tdV, tS, dDO_mn, m > 0);  // dV += P^T dO
        mma_commit_w(&bars.do_empty);
        if (m + 1 < M) {
          mbar_wait(&bars.q_full[(m + 1) & 1], ((m + 1) >> 1) & 1);
          tc_fence_after();
          TR(3, m);
          mma_kmajor(tS, dK_k, q_k(m + 1));  // S(m+1): P(m) already consumed (in-order pipe)
          mma_commit_w(&bars.s_full);
        }
        mbar_wait(&bars.ds_full, m & 1);
        tc_fence_after();
        TR(4, m);
        mma_tmemA(tdK, tdP, q_mn(m), m > 0);  // dK += dS^T Q
        mma_commit_w(&bars.q_empty[m & 1]);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)  // dQ = dS K  (A = dS MN-major in smem, B = K MN-major)
          mma_ss_w(tdP, dDS_mn + moff(k), dK_mn + moff(k), kIdescDQ, k > 0);
        mma_commit_w(&bars.dq_full);
        TR(5, m);
      }
      mma_commit_w(&bars.dkdv_done);
    }
  } else if (warp < 4) {
    setmaxnreg_inc<136>();
    // ===================== dQ reducer (TMEM lane = q row) =====================
    const CUtensorMap* mdq = tmap(a, a.dq_slot);
    const float tau = p.scale;
    const int row = warp * 32 + lane;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    int piece_ctr = 0;
    for (int m = 0; m < M; ++m) {
      const int q0 = qtile(m) * BQ;
      mbar_wait(&bars.dq_full, m & 1);
      if (threadIdx.x == 0) TR(12, m);
      tc_fence_after();
      uint32_t v[128];
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) tmem_ld32(tdP + lane_off + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[cb * 32]));
      tmem_wait_ld();
      tc_fence_before();
      if (threadIdx.x == 0) TR(13, m);
      mbar_arrive(&bars.dq_free);
      if constexpr (kDqDirectRed) {
        // fp32 vector reductions straight from registers: keeps the 128 KB / tile of
        // staging traffic off shared memory (the bwd is smem-bandwidth bound)
        if (q0 + row < p.q_len) {
          float* dst = p.dq_acc + ((size_t)(q0 + row) * p.heads + head) * HD;
#pragma unroll
          for (int c4 = 0; c4 < 32; ++c4)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * c4),
                         "f"(__uint_as_float(v[4 * c4 + 0]) * tau), "f"(__uint_as_float(v[4 * c4 + 1]) * tau),
                         "f"(__uint_as_float(v[4 * c4 + 2]) * tau), "f"(__uint_as_float(v[4 * c4 + 3]) * tau)
                         : "memory");
        }
        continue;
      }
#pragma unroll
      for (int pc = 0; pc < 4; ++pc, ++piece_ctr) {
        const int buf = piece_ctr & 1;
        uint8_t* stg = smem + kOffDQ + buf * 16384;
        if (threadIdx.x == 0) bulk_wait_read<1>();  // the reduce that last read `buf` is done
        named_bar_sync(5, 128);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {  // dQ = tau (dS K): tau applied here (dS is unscaled)
          const float2 x0 = fmul2(make_float2(__uint_as_float(v[pc * 32 + ch * 4 + 0]),
                                              __uint_as_float(v[pc * 32 + ch * 4 + 1])), make_float2(tau, tau));
          const float2 x1 = fmul2(make_float2(__uint_as_float(v[pc * 32 + ch * 4 + 2]),
                                              __uint_as_float(v[pc * 32 + ch * 4 + 3])), make_float2(tau, tau));
          *reinterpret_cast<float4*>(stg + sw128(row, ch * 16)) = make_float4(x0.x, x0.y, x1.x, x1.y);
        }
        fence_proxy_async_smem();
        named_bar_sync(5, 128);
        if (threadIdx.x == 0) {
          tma_reduce_add_3d(mdq, stg, pc * 32, head, q0);
          bulk_commit();
        }
      }
    }
    if (threadIdx.x == 0) bulk_wait<0>();
  } else {
    setmaxnreg_inc<136>();
    // ===================== compute: P and dS (TMEM lane = key row) =====================
    const int g = (warp - 4) >> 2;  // column half: q in [64g, 64g+64)
    const int wq = warp & 3;
    const int row = wq * 32 + lane;  // key row in tile
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int kv_pos = kvp0 + row;
    const bool kv_ok = row < kv_len;
    const float sl2 = p.scale * kLog2e;
    const float tau = p.scale;
    uint8_t* sDS = smem + kOffDS + g * kHalf;
    for (int m = 0; m < M; ++m) {
      const int s = m & 1;
      const int q0 = qtile(m) * BQ;
      const int qpos0 = p.q_start + q0 + g * 64;  // absolute position of this half's column 0
      mbar_wait(&bars.q_full[s], (m >> 1) & 1);
      mbar_wait(&bars.do_full, m & 1);
      mbar_wait(&bars.s_full, m & 1);
      if (lane == 0 && wq == 0) TR(6 + 4 * g, m);
      tc_fence_after();
      // ---- P = exp2(S tau log2e - LSE log2e) for q columns [64g, 64g+64); two 32-column
      //      halves so the second TMEM load overlaps the first half's math
      const uint32_t tSg = tS + lane_off + g * 64;
      const float* lse2 = sLSE + s * 128 + g * 64;
      // column j visible iff q position >= key position and the key row exists
      const int first_vis = kv_ok ? (kv_pos - qpos0) : 1 << 30;  // columns j >= first_vis are visible
      const bool masked = __any_sync(0xffffffffu, first_vis > 0);
      float2 pr[32];
      uint32_t pk[32];
      tmem_ld32(tSg, *reinterpret_cast<uint32_t(*)[32]>(&pr[0]));
      tmem_wait_ld();
      tmem_ld32(tSg + 32, *reinterpret_cast<uint32_t(*)[32]>(&pr[16]));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1) tmem_wait_ld();
#pragma unroll
        for (int c = 16 * h; c < 16 * h + 16; c += 2) {
          const float4 l4 = *reinterpret_cast<const float4*>(lse2 + 2 * c);
          float2 x0 = ffma2(pr[c], make_float2(sl2, sl2), make_float2(-l4.x, -l4.y));
          float2 x1 = ffma2(pr[c + 1], make_float2(sl2, sl2), make_float2(-l4.z, -l4.w));
          if (masked) {
            const int j = 2 * c;
            x0.x = (j + 0 >= first_vis) ? x0.x : -INFINITY;
            x0.y = (j + 1 >= first_vis) ? x0.y : -INFINITY;
            x1.x = (j + 2 >= first_vis) ? x1.x : -INFINITY;
            x1.y = (j + 3 >= first_vis) ? x1.y : -INFINITY;
          }
          pr[c] = make_float2(ex2(x0.x), ex2(x0.y));
          pr[c + 1] = make_float2(ex2(x1.x), ex2(x1.y));
          pk[c] = pack_bf16(pr[c].x, pr[c].y);
          pk[c + 1] = pack_bf16(pr[c + 1].x, pr[c + 1].y);
        }
        // P^T bf16 pairs into this WG's own S columns: A operand of dV += P^T dO
        tmem_st16(tSg + 16 * h, *reinterpret_cast<uint32_t(*)[16]>(&pk[16 * h]));
      }
      tmem_wait_st();
      tc_fence_before();
      if (lane == 0 && wq == 0 && g == 0) TR(7, m);
      mbar_arrive(&bars.p_full);

      // ---- dS = P (dP - Delta)   (tau is applied to dK / dQ at their write-out)
      mbar_wait(&bars.dp_full, m & 1);
      if (lane == 0 && wq == 0 && g == 0) TR(8, m);
      tc_fence_after();
      const uint32_t tPg = tdP + lane_off + g * 64;
      const float* dl = sDelta + s * 128 + g * 64;
      float2 dp[32];
      tmem_ld32(tPg, *reinterpret_cast<uint32_t(*)[32]>(&dp[0]));
      tmem_wait_ld();
      tmem_ld32(tPg + 32, *reinterpret_cast<uint32_t(*)[32]>(&dp[16]));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1) tmem_wait_ld();
#pragma unroll
        for (int c = 16 * h; c < 16 * h + 16; c += 2) {
          const float4 d4 = *reinterpret_cast<const float4*>(dl + 2 * c);
          const float2 t0 = fadd2(dp[c], make_float2(-d4.x, -d4.y));
          const float2 t1 = fadd2(dp[c + 1], make_float2(-d4.z, -d4.w));
          const float2 a0 = fmul2(pr[c], t0);
          const float2 a1 = fmul2(pr[c + 1], t1);
          pk[c] = pack_bf16(a0.x, a0.y);
          pk[c + 1] = pack_bf16(a1.x, a1.y);
        }
        tmem_st16(tPg + 16 * h, *reinterpret_cast<uint32_t(*)[16]>(&pk[16 * h]));  // dS^T: A of dK += dS^T Q
#pragma unroll
        for (int ch = 4 * h; ch < 4 * h + 4; ++ch)  // dS as MN-major A of dQ = dS K: row = key, 64 q per half
          *reinterpret_cast<uint4*>(sDS + sw128(row, ch * 16)) =
              make_uint4(pk[ch * 4 + 0], pk[ch * 4 + 1], pk[ch * 4 + 2], pk[ch * 4 + 3]);
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      if (lane == 0 && wq == 0) TR(9 + 2 * g, m);
      mbar_arrive(&bars.ds_full);
    }
    // ---- epilogue: dK_j, dV_j of this key tile (+= into the fp32 accumulators)
    mbar_wait(&bars.dkdv_done, 0);
    tc_fence_after();
    const bool final_out = (c == p.final_slot);
    const size_t base = ((size_t)(kv_row0 + row) * p.heads + head) * HD + g * 64;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t tsrc = (which == 0 ? tdV : tdK) + lane_off + g * 64;
      float* acc = (which == 0 ? a.dv[c] : a.dk[c]) + base;
      __nv_bfloat16* out = final_out ? reinterpret_cast<__nv_bfloat16*>(which == 0 ? p.dv_out : p.dk_out) + base
                                     : nullptr;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t v[32];
        tmem_ld32(tsrc + half * 32, v);
        tmem_wait_ld();
        if (kv_ok) {
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            float4* ap = reinterpret_cast<float4*>(acc + half * 32 + q4 * 4);
            float4 o = *ap;
            const float f = which == 0 ? 1.f : tau;  // dK = tau dS^T Q
            o.x += __uint_as_float(v[q4 * 4 + 0]) * f;
            o.y += __uint_as_float(v[q4 * 4 + 1]) * f;
            o.z += __uint_as_float(v[q4 * 4 + 2]) * f;
            o.w += __uint_as_float(v[q4 * 4 + 3]) * f;
            if (final_out) {
              uint2 b;
              b.x = pack_bf16(o.x, o.y);
              b.y = pack_bf16(o.z, o.w);
              *reinterpret_cast<uint2*>(out + half * 32 + q4 * 4) = b;
            } else {
              *ap = o;
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 14) tmem_dealloc<512>(tmem);
}

}  // namespace

cudaError_t launch_bwd_sm100(const Sm100Bwd& a, cudaStream_t s) {
  if (a.p.d != HD) return cudaErrorNotSupported;
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    init = true;
  }
  dim3 grid(a.tile_base[a.n], a.p.heads);
  bwd_kernel<<<grid, kThreads, kSmemBytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sppo
