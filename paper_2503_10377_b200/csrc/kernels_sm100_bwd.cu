// sm_100a tensor-core backward of chunked causal attention.
//
// Method (P:356 [§5.1]; oracle/attention.py chunked_attention_bwd): for chunk
// i and every prior chunk j in the window,
//   P = exp(tau Q_i K_j^T - LSE_i),  dV_j += P^T dO_i,  dP = dO_i V_j^T,
//   dS = P (dP - Delta_i),  dQ_i += tau dS K_j,  dK_j += tau dS^T Q_i.
//
// B200 design: KV-stationary on a CTA PAIR (cluster of 2,
// tcgen05 cta_group::2).  The pair owns 256 keys of chunk j (rank r: keys
// [128r, 128r+128)) of one head and loops over the causally relevant 128-row Q
// tiles of chunk i.  Four of the five MMAs per Q tile are pair instructions
// issued by the leader, each CTA supplying its own A rows and half of B:
//   S^T  = K Q^T      M=256 N=128 K=128  A = own K (smem), B = Q rows [64r,+64)
//   dP^T = V dO^T     M=256 N=128 K=128  A = own V,        B = dO rows [64r,+64)
//   dV  += P^T dO     M=256 N=128 K=128  A = P^T (TMEM),   B = dO cols [64r,+64)
//   dK  += dS^T Q     M=256 N=128 K=128  A = dS^T (smem, K-major), B = Q cols [64r,+64)
// and dQ = dS K (M=N=K=128, A = dS, B = own K, both MN-major smem) is a
// cta_group::1 MMA each CTA issues for its own keys.  dS lives only in smem
// ([keys][q]: K-major A of dK and MN-major A of dQ), so dQ(m) is issued before
// dK(m) and its TMEM readout overlaps dK(m): the per-tile critical chain is
// dP -> dS -> dQ -> readout -> next dP (all share TMEM region 2).
// (Pairing dQ too, M=128 over 256 keys, needs half of dS from the peer over
// DSMEM at ~20 B/clk: measured 3000 cycles per tile slower; not used.)
// 512 threads per CTA:
//   warps 0-3   dQ reducer: tcgen05.ld dQ -> swizzled smem -> TMA reduce-add
//   warps 4-11  compute: P (exp2) and dS; WG A owns q columns 0-63, WG B 64-127
//               of every TMEM lane (= key row)
//   warp 12     MMA issuer: pair MMAs + own dQ (leader), own dQ (peer)
//   warp 13     TMA: K, V once; Q rows half + LSE per tile
//   warp 14     TMEM alloc/dealloc; TMA dO columns half + Q columns half per tile
//   warp 15     TMA: dO rows half + Delta per tile
// TMEM (512 cols per CTA): S/P [0,128) | dV [128,256) | dP/dQ [256,384) | dK [384,512)
// Operand TMA loads of both CTAs complete on the leader's barriers; MMA commits
// multicast to both CTAs; compute/reducer warps arrive on the leader's barriers
// remotely.  tau is folded into dK / dQ at their write-out.
#include <cuda.h>
#include <math.h>

#include "internal.h"
#include "sm100_ptx.cuh"

namespace sppo {
namespace {
using namespace ptx;

constexpr int BQ = 128, BKV = 128, HD = 128;
constexpr int kThreads = 512;
constexpr uint32_t kTile = 32768;  // [128 rows][128 d] bf16 = two [128][64] SW128 boxes
constexpr uint32_t kBox = 16384;   // [128 rows][64 d] bf16
constexpr uint32_t kHBox = 8192;   // [64 rows][64 d] bf16
// dynamic smem map (bytes); the base is 1024-aligned (no static smem is used)
constexpr uint32_t kOffK = 0;                     // own K, K-major: A of S^T = K Q^T
constexpr uint32_t kOffV = kOffK + kTile;         // own V, K-major: A of dP^T = V dO^T
constexpr uint32_t kStageA = 2 * kHBox;           // one [64 rows][128 d] K-major stage
constexpr int kStagesA = 1;  // single-stage Q/dO row halves: 2 stages measured slower (TMA-reduce contention)
constexpr uint32_t kOffQA = kOffV + kTile;        // Q rows [64r,+64), all d, K-major: B of S^T
constexpr uint32_t kOffQB = kOffQA + kStagesA * kStageA;  // Q all rows, d cols [64r,+64), MN-major: B of dK
constexpr uint32_t kOffOA = kOffQB + kBox;        // dO rows half: B of dP^T
constexpr uint32_t kOffOB = kOffOA + kStagesA * kStageA;  // dO cols half: B of dV
constexpr uint32_t kOffDS = kOffOB + kBox;        // dS [128 keys][128 q] (two q halves): A of dQ and dK
#ifndef SPPO_DQ_RED_PIECES
#define SPPO_DQ_RED_PIECES 0  // measured: 1 piece -> bwd 841, 2 -> 775 vs 1017 TF/s (L2/LSU bound)
#endif
constexpr int kDqRedPieces = SPPO_DQ_RED_PIECES;  // of the 4 dQ pieces, sent by red.global.add.v4.f32
// Two staging buffers, one issuing thread.  Measured alternatives (profiles/r02):
// 4 buffers with each reducer warp issuing its own piece -> bwd 950-955 vs 1037-1039
// TF/s; the 4 pieces as ONE 4-D reduce (box {32, 128, 4, 1}) -> 937 vs 1049: a 64 KB
// reduce-add takes ~3600 cycles to drain from shared memory (~18 B/clk per SM), i.e.
// the dQ path is bound by the L2 reduction rate, not by TMA issue.  Summing the
// pair's two partials first (CTA r keeps d-columns [64r, +64) and stores the other
// 64 into the peer's smem over DSMEM, halving the L2 reduce bytes) measured bwd
// 612-627 (row-swizzled remote stores) / 720 (coalesced [chunk][row] layout) vs
// 1032-1036 TF/s: thread stores to the peer's shared memory moved ~4-5 B/clk.
constexpr int kDqBufs = 2;
#ifndef SPPO_EPI_RED
#define SPPO_EPI_RED 1  // measured: bwd +3 % at C2, +9 % at 2K chunks vs load-add-store
#endif
#ifndef SPPO_BWD_EMU_EVERY
#define SPPO_BWD_EMU_EVERY 0  // 1 of every N exp2 pairs of P on the FMA pipe (cubic, as the forward); 0 = off
#endif
constexpr int kBwdEmu = SPPO_BWD_EMU_EVERY;
constexpr bool kEpiRed = SPPO_EPI_RED;  // dK/dV accumulator epilogue: red.global.add (1) or load-add-store (0)  // 4 buffers measured slower: the reduces queue ahead of Q/dO loads on the TMA unit
constexpr uint32_t kOffDQ = kOffDS + kTile;       // kDqBufs x [128 rows][32 fp32] reduce staging
constexpr uint32_t kOffLSE = kOffDQ + kDqBufs * 16384;  // 2 x 128 fp32 (LSE * log2 e)
constexpr uint32_t kOffDelta = kOffLSE + 1024;    // 2 x 128 fp32
#ifndef SPPO_DQ_HINT
#define SPPO_DQ_HINT 0  // evict_last L2 hint on the dQ reduce-add: measured bwd 1051.7-1052.8 vs 1053.4-1055.3 TF/s, off
#endif
#ifndef SPPO_BWD_FOLD
#define SPPO_BWD_FOLD 0
#endif
// SPPO_BWD_FOLD: -LSE/tau and -Delta enter S^T and dP^T through one extra K=16
// MMA step (A: a constant [keys][16] block with ones in k = 0, 1; B: per-tile
// [q][16] blocks holding a bf16 hi/lo split of the statistic), so the compute
// warps read no LSE / Delta from shared memory (their broadcast LDS.128 were
// ~40 % of the kernel's LSU shared-memory wavefronts).  No-swizzle K-major core
// matrices: element (row, k) at (row/8)*256 + (k/8)*128 + (row%8)*16 + (k%8)*2.
constexpr bool kFold = SPPO_BWD_FOLD;
#ifndef SPPO_WARP_ARRIVE
#define SPPO_WARP_ARRIVE 1  // consumer releases (LSE / Delta / dS-local) as one arrival per warp after __syncwarp
#endif
constexpr bool kWarpArrive = SPPO_WARP_ARRIVE;
constexpr uint32_t kComputeArrivals = kWarpArrive ? 8 : 256;  // 8 compute warps x (1 or 32 lanes)
constexpr uint32_t kOffXK = kOffDelta + 1024;   // [128 keys][16]: ones at k = 0, 1 (A of the extra step)
constexpr uint32_t kOffXQ = kOffXK + 4096;      // [64 q][16]: -LSE/tau hi, lo (B of S^T's extra step)
constexpr uint32_t kOffXO = kOffXQ + 2048;      // [64 q][16]: -Delta hi, lo (B of dP^T's extra step)
constexpr uint32_t kOffBars = kFold ? kOffXO + 2048 : kOffDelta + 1024;
constexpr uint32_t kSmemBytes = kOffBars + 256;
static_assert(kSmemBytes <= 232448, "smem budget");

constexpr uint32_t kIdescS = idesc_bf16(256, 128, 0, 0);  // pair, K-major x K-major
constexpr uint32_t kIdescT = idesc_bf16(256, 128, 0, 1);  // pair, TMEM or K-major A x MN-major B
constexpr uint32_t kIdescQ = idesc_bf16(128, 128, 1, 1);  // one CTA, MN-major x MN-major
constexpr float kLog2e = 1.4426950408889634f;

struct Bars {
  uint64_t kv_full;                   // leader: K, V of both CTAs (tx)
  uint64_t qa_full[2], qb_full;       // leader (tx of both CTAs)
  uint64_t oa_full[2], ob_full;       // leader (tx of both CTAs)
  uint64_t qa_empty[2], qb_empty;     // both (MMA commit multicast)
  uint64_t oa_empty[2], ob_empty;     // both
  uint64_t lse_full[2], delta_full[2];    // local: producer lanes (32)
  uint64_t lse_empty[2], delta_empty[2];  // local: compute threads (256)
  uint64_t s_full, dp_full, dq_full;  // both (MMA commit multicast)
  uint64_t p_full, ds_full;           // leader: compute warps of both CTAs (16)
  uint64_t ds_local;                  // peer only: compute threads (256), dS in smem, dP read
  uint64_t dq_free;                   // leader: reducer warps of both CTAs (8)
  uint64_t dkdv_done;                 // both
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

__device__ __forceinline__ const CUtensorMap* tmap(const Sm100Bwd& a, int slot) {
  return reinterpret_cast<const CUtensorMap*>(a.desc_table) + slot;
}

// UMMA smem descriptor of a no-swizzle K-major operand (core matrices of 8 rows x 16 B)
__device__ __forceinline__ uint64_t sdesc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return make_sdesc(saddr, lbo, sbo) & ~((uint64_t)7 << 61);
}

__device__ __forceinline__ uint32_t sw128(int r, int byte_in_row) {
  const uint32_t lin = r * 128 + byte_in_row;
  return lin ^ (((lin >> 7) & 7u) << 4);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    bwd_kernel(const __grid_constant__ Sm100Bwd a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars& bars = *reinterpret_cast<Bars*>(smem + kOffBars);
  float* sLSE = reinterpret_cast<float*>(smem + kOffLSE);
  float* sDelta = reinterpret_cast<float*>(smem + kOffDelta);
  const BwdParams& p = a.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;

  // ---- which 256-key pair tile: window chunk c, pair pt within it
  int c = 0;
  while (c + 1 < a.n && a.pair_base[c + 1] <= pair) ++c;
  const int pair_row0 = (pair - a.pair_base[c]) * 2 * BKV;  // first key row of the pair within chunk j
  const int kv_row0 = pair_row0 + (int)rank * BKV;          // this CTA's key rows
  const int kv_len = min(BKV, a.len[c] - kv_row0);          // valid keys (<= 0: rank 1 of a ragged pair)
  const int kvp0 = a.start[c] + kv_row0;                    // absolute position of key row 0
  // Q tiles of chunk i with some row at position >= the pair's first key
  const int q_tiles = (p.q_len + BQ - 1) / BQ;
  const int qt_first = max(0, (a.start[c] + pair_row0 - p.q_start) / BQ);
  const int M = q_tiles - qt_first;
#ifndef SPPO_BWD_ROT
#define SPPO_BWD_ROT 1  // measured: without the rotation bwd 985.6-986.0 vs 1042.0-1049.1 TF/s
#endif
  // start Q tile rotated per pair: concurrent pairs reduce dQ into different rows
#ifndef SPPO_BWD_ROT_SHIFT
#define SPPO_BWD_ROT_SHIFT 0  // 2^shift consecutive pairs share a start tile (reduce the same dQ lines together)
#endif
  const int rot = SPPO_BWD_ROT ? (int)((((uint32_t)pair >> SPPO_BWD_ROT_SHIFT) * 7u + blockIdx.y * 13u) % (uint32_t)M)
                               : 0;
  auto qtile = [&](int m) { return qt_first + (m + rot) % M; };

  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 atoms need 1024 B alignment
    mbar_init(&bars.kv_full, 1);
    mbar_init(&bars.qb_full, 1);
    mbar_init(&bars.ob_full, 1);
    mbar_init(&bars.qb_empty, 1);
    mbar_init(&bars.ob_empty, 1);
    for (int s = 0; s < 2; ++s) {
      // fold: + one remote arrival per CTA once its extra B block is written
      mbar_init(&bars.qa_full[s], kFold ? 3 : 1);
      mbar_init(&bars.oa_full[s], kFold ? 3 : 1);
      mbar_init(&bars.qa_empty[s], 1);
      mbar_init(&bars.oa_empty[s], 1);
      mbar_init(&bars.lse_full[s], 32);
      mbar_init(&bars.delta_full[s], 32);
      mbar_init(&bars.lse_empty[s], kComputeArrivals);
      mbar_init(&bars.delta_empty[s], kComputeArrivals);
    }
    mbar_init(&bars.s_full, 1);
    mbar_init(&bars.dp_full, 1);
    mbar_init(&bars.dq_full, 1);
    mbar_init(&bars.p_full, 16);
    mbar_init(&bars.ds_full, 16);
    mbar_init(&bars.ds_local, kComputeArrivals);
    mbar_init(&bars.dq_free, 8);
    mbar_init(&bars.dkdv_done, 1);
    fence_mbar_init();
  }
  if (warp == 14) tmem_alloc_pair<512>(&bars.tmem_base);
  if (kFold) {
    // constant parts of the extra K=16 operand blocks: ones block (A) and the
    // all-zero k = 8..15 core matrices of the per-tile B blocks
    const uint32_t one2 = 0x3F803F80u;  // bf16 (1, 1)
    for (int r = threadIdx.x; r < 128; r += kThreads) {
      *reinterpret_cast<uint4*>(smem + kOffXK + (r >> 3) * 256 + (r & 7) * 16) = make_uint4(one2, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(smem + kOffXK + (r >> 3) * 256 + 128 + (r & 7) * 16) = make_uint4(0u, 0u, 0u, 0u);
      if (r < 64) {
        *reinterpret_cast<uint4*>(smem + kOffXQ + (r >> 3) * 256 + 128 + (r & 7) * 16) = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(smem + kOffXO + (r >> 3) * 256 + 128 + (r & 7) * 16) = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const uint32_t tS = tmem, tdV = tmem + 128, tdP = tmem + 256, tdK = tmem + 384;
  // leader-side barriers as shared::cluster addresses
  const uint32_t L_kv = mapa(smem_u32(&bars.kv_full), 0);
  const uint32_t L_qb = mapa(smem_u32(&bars.qb_full), 0), L_ob = mapa(smem_u32(&bars.ob_full), 0);
  // debug trace of CTA (0,0): clock64 per pipeline event (SPPO_TRACE)
  unsigned long long* tr = (p.trace && blockIdx.x == 0 && blockIdx.y == 0) ? p.trace : nullptr;
#define TR(slot, it)                                                              \
  do {                                                                            \
    if (tr && (it) < kTraceIters) tr[(it) * kTraceSlots + (slot)] = clock64();   \
  } while (0)

  if (warp >= 12) {
    setmaxnreg_dec<104>();
    if (warp == 13) {
      // ===================== TMA: K, V once; Q rows half + LSE per tile =====================
      const CUtensorMap* mq64 = tmap(a, a.q64_slot);
      if (lane == 0) {
        const CUtensorMap* mk = tmap(a, a.slots.k[c]);
        const CUtensorMap* mv = tmap(a, a.slots.v[c]);
        if (leader) mbar_arrive_expect_tx(&bars.kv_full, 2 * 2 * kTile);
        tma_load_3d_pair(smem + kOffK, mk, L_kv, 0, head, kv_row0);
        tma_load_3d_pair(smem + kOffK + kBox, mk, L_kv, 64, head, kv_row0);
        tma_load_3d_pair(smem + kOffV, mv, L_kv, 0, head, kv_row0);
        tma_load_3d_pair(smem + kOffV + kBox, mv, L_kv, 64, head, kv_row0);
      }
      const float* lse_h = p.lse + (size_t)head * p.q_len;
      for (int m = 0; m < M; ++m) {
        const int s = m & 1;
        const int q0 = qtile(m) * BQ;
        const int sa = m % kStagesA, ua = m / kStagesA;  // stage and its use count
        if (ua > 0) mbar_wait(&bars.qa_empty[sa], (ua - 1) & 1);
        if (kFold) {  // this CTA's 64 q rows of the tile: -LSE/tau as bf16 hi + lo at k = 0, 1
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = lane + 32 * e;
            const int r = q0 + 64 * (int)rank + i;
            const float cv = r < p.q_len ? -lse_h[r] / p.scale : -INFINITY;
            const __nv_bfloat16 hi = __float2bfloat16_rn(cv);
            const float lo = r < p.q_len ? cv - __bfloat162float(hi) : 0.f;
            const __nv_bfloat162 hl = __halves2bfloat162(hi, __float2bfloat16_rn(lo));
            *reinterpret_cast<uint4*>(smem + kOffXQ + (i >> 3) * 256 + (i & 7) * 16) =
                make_uint4(*reinterpret_cast<const uint32_t*>(&hl), 0u, 0u, 0u);
          }
          fence_proxy_async_smem();
          __syncwarp();
        }
        if (lane == 0) {
          const uint32_t L_qa = mapa(smem_u32(&bars.qa_full[sa]), 0);
          if (leader) mbar_arrive_expect_tx(&bars.qa_full[sa], 2 * kStageA);
          tma_load_3d_pair(smem + kOffQA + sa * kStageA, mq64, L_qa, 0, head, q0 + 64 * (int)rank);
          tma_load_3d_pair(smem + kOffQA + sa * kStageA + kHBox, mq64, L_qa, 64, head, q0 + 64 * (int)rank);
          if (kFold) mbar_arrive_cluster(L_qa);
        }
        if (kFold) continue;
        if (m >= 2) mbar_wait(&bars.lse_empty[s], ((m >> 1) - 1) & 1);
        float4 w;
        float* wp = reinterpret_cast<float*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = q0 + lane * 4 + k;
          wp[k] = r < p.q_len ? lse_h[r] * kLog2e : INFINITY;  // OOB row -> P = 0
        }
        *reinterpret_cast<float4*>(sLSE + s * 128 + lane * 4) = w;  // one conflict-free STS.128
        if (lane == 0) TR(15, m);
        mbar_arrive(&bars.lse_full[s]);
      }
      if (!kFold)
        for (int m = max(M - 2, 0); m < M; ++m) mbar_wait(&bars.lse_empty[m & 1], (m >> 1) & 1);
    } else if (warp == 15) {
      // ===================== TMA: dO rows half + Delta per tile =====================
      const CUtensorMap* mdo64 = tmap(a, a.do64_slot);
      const float* delta_h = p.delta + (size_t)head * p.q_len;
      for (int m = 0; m < M; ++m) {
        const int s = m & 1;
        const int q0 = qtile(m) * BQ;
        const int sa = m % kStagesA, ua = m / kStagesA;
        if (ua > 0) mbar_wait(&bars.oa_empty[sa], (ua - 1) & 1);
        if (kFold) {  // this CTA's 64 q rows: -Delta as bf16 hi + lo at k = 0, 1
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = lane + 32 * e;
            const int r = q0 + 64 * (int)rank + i;
            const float cv = r < p.q_len ? -delta_h[r] : 0.f;
            const __nv_bfloat16 hi = __float2bfloat16_rn(cv);
            const __nv_bfloat162 hl = __halves2bfloat162(hi, __float2bfloat16_rn(cv - __bfloat162float(hi)));
            *reinterpret_cast<uint4*>(smem + kOffXO + (i >> 3) * 256 + (i & 7) * 16) =
                make_uint4(*reinterpret_cast<const uint32_t*>(&hl), 0u, 0u, 0u);
          }
          fence_proxy_async_smem();
          __syncwarp();
        }
        if (lane == 0) {
          const uint32_t L_oa = mapa(smem_u32(&bars.oa_full[sa]), 0);
          if (leader) mbar_arrive_expect_tx(&bars.oa_full[sa], 2 * kStageA);
          tma_load_3d_pair(smem + kOffOA + sa * kStageA, mdo64, L_oa, 0, head, q0 + 64 * (int)rank);
          tma_load_3d_pair(smem + kOffOA + sa * kStageA + kHBox, mdo64, L_oa, 64, head, q0 + 64 * (int)rank);
          if (kFold) mbar_arrive_cluster(L_oa);
        }
        if (kFold) continue;
        if (m >= 2) mbar_wait(&bars.delta_empty[s], ((m >> 1) - 1) & 1);
        float4 w;
        float* wp = reinterpret_cast<float*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = q0 + lane * 4 + k;
          wp[k] = r < p.q_len ? delta_h[r] : 0.f;
        }
        *reinterpret_cast<float4*>(sDelta + s * 128 + lane * 4) = w;
        mbar_arrive(&bars.delta_full[s]);
      }
      if (!kFold)
        for (int m = max(M - 2, 0); m < M; ++m) mbar_wait(&bars.delta_empty[m & 1], (m >> 1) & 1);
    } else if (warp == 14) {
      // ===================== TMA: dO columns half, Q columns half per tile =====================
      const CUtensorMap* mq = tmap(a, a.q_slot);
      const CUtensorMap* mdo = tmap(a, a.do_slot);
      for (int m = 0; m < M; ++m) {
        const int q0 = qtile(m) * BQ;
        if (m > 0) mbar_wait(&bars.ob_empty, (m - 1) & 1);
        if (lane == 0) {
          if (leader) mbar_arrive_expect_tx(&bars.ob_full, 2 * kBox);
          tma_load_3d_pair(smem + kOffOB, mdo, L_ob, 64 * rank, head, q0);
        }
        if (m > 0) mbar_wait(&bars.qb_empty, (m - 1) & 1);
        if (lane == 0) {
          if (leader) mbar_arrive_expect_tx(&bars.qb_full, 2 * kBox);
          tma_load_3d_pair(smem + kOffQB, mq, L_qb, 64 * rank, head, q0);
        }
      }
    } else if (warp == 12) {
      // ===================== MMA issuer (warp 12, converged; one elected lane issues) =====================
      // Base descriptors computed once; a k-step only adds (byte offset >> 4) to the
      // 14-bit start-address field (smem < 256 KB, so no carry leaves the field).
      const uint64_t dK_k = sdesc_kmajor(smem_u32(smem + kOffK)), dV_k = sdesc_kmajor(smem_u32(smem + kOffV));
      const uint64_t dQA_k = sdesc_kmajor(smem_u32(smem + kOffQA)), dOA_k = sdesc_kmajor(smem_u32(smem + kOffOA));
      const uint64_t dQB_mn = sdesc_mnmajor(smem_u32(smem + kOffQB), kBox);
      const uint64_t dOB_mn = sdesc_mnmajor(smem_u32(smem + kOffOB), kBox);
      const uint64_t dDS_mn = sdesc_mnmajor(smem_u32(smem + kOffDS), kBox);
      const uint64_t dDS_k = sdesc_kmajor(smem_u32(smem + kOffDS));
      const uint64_t dK_mn = sdesc_mnmajor(smem_u32(smem + kOffK), kBox);
      auto koff = [](int k) { return (uint64_t)(((k >> 2) * kBox + (k & 3) * 32) >> 4); };    // 128-row K-major
      auto koffh = [](int k) { return (uint64_t)(((k >> 2) * kHBox + (k & 3) * 32) >> 4); };  // 64-row K-major
      auto moff = [](int k) { return (uint64_t)((k * 2048) >> 4); };                          // MN-major k-step
      // dQ = dS K for this CTA's 128 keys (cta_group::1; D lanes = q rows)
      auto mma_dq = [&]() {
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) mma_ss_w(tdP, dDS_mn + moff(k), dK_mn + moff(k), kIdescQ, k > 0);
        mma_commit_w(&bars.dq_full);
      };
      if (!leader) {
        for (int m = 0; m < M; ++m) {
          mbar_wait(&bars.ds_local, m & 1);  // dS(m) in this CTA's smem, dP(m) read out of tdP
          tc_fence_after();
          mma_dq();
        }
      } else {
        // D = A B^T, A = own 128 keys (K-major), B = this CTA's 64 q rows (K-major)
        auto mma_kk = [&](uint32_t d, uint64_t A, uint64_t B) {
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) mma2_ss_w(d, A + koff(k), B + koffh(k), kIdescS, k > 0);
        };
        // D (+)= A[tmem] B, B = this CTA's 64 d columns (MN-major).  A (P or dS, bf16 pairs)
        // of q columns 64g..64g+63 sits in TMEM columns [64g, 64g+32) of its region.
        auto mma_tmemA = [&](uint32_t d, uint32_t tA, uint64_t B, bool acc) {
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)
            mma2_ts_w(d, tA + (k >> 2) * 64 + (k & 3) * 8, B + moff(k), kIdescT, (acc || k > 0) ? 1u : 0u);
        };
        mbar_wait(&bars.kv_full, 0);
        constexpr uint64_t kStageStep = kStageA >> 4;
        mbar_wait(&bars.qa_full[0], 0);
        tc_fence_after();
        const uint64_t dXK = sdesc_noswz(smem_u32(smem + kOffXK), 128, 256);
        const uint64_t dXQ = sdesc_noswz(smem_u32(smem + kOffXQ), 128, 256);
        const uint64_t dXO = sdesc_noswz(smem_u32(smem + kOffXO), 128, 256);
        mma_kk(tS, dK_k, dQA_k);  // S^T(0) = K Q^T
        if (kFold) mma2_ss_w(tS, dXK, dXQ, kIdescS, 1u);  // - LSE / tau
        mma2_commit_w(&bars.s_full);
        mma2_commit_w(&bars.qa_empty[0]);
        for (int m = 0; m < M; ++m) {
          TR(0, m);
          mbar_wait(&bars.oa_full[m % kStagesA], (m / kStagesA) & 1);
          if (m > 0) mbar_wait(&bars.dq_free, (m - 1) & 1);  // both CTAs' reducers have read dQ(m-1)
          tc_fence_after();
          TR(1, m);
          mma_kk(tdP, dV_k, dOA_k + (m % kStagesA) * kStageStep);  // dP^T = V dO^T
          if (kFold) mma2_ss_w(tdP, dXK, dXO, kIdescS, 1u);  // - Delta
          mma2_commit_w(&bars.dp_full);
          mma2_commit_w(&bars.oa_empty[m % kStagesA]);
          mbar_wait(&bars.p_full, m & 1);
          mbar_wait(&bars.ob_full, m & 1);
          tc_fence_after();
          TR(2, m);
          mma_tmemA(tdV, tS, dOB_mn, m > 0);  // dV += P^T dO
          mma2_commit_w(&bars.ob_empty);
          if (m + 1 < M) {
            const int n1 = m + 1;
            mbar_wait(&bars.qa_full[n1 % kStagesA], (n1 / kStagesA) & 1);
            tc_fence_after();
            TR(3, m);
            mma_kk(tS, dK_k, dQA_k + (n1 % kStagesA) * kStageStep);  // S^T(m+1): P(m) consumed (in-order pipe)
            if (kFold) mma2_ss_w(tS, dXK, dXQ, kIdescS, 1u);
            mma2_commit_w(&bars.s_full);
            mma2_commit_w(&bars.qa_empty[n1 % kStagesA]);
          }
          mbar_wait(&bars.ds_full, m & 1);  // both CTAs: dS(m) in smem (implies own ds_local(m))
          tc_fence_after();
          TR(4, m);
          mma_dq();  // own dQ first: its readout overlaps the pair dK below
          mbar_wait(&bars.qb_full, m & 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < BQ / 16; ++k)  // dK += dS^T Q  (A = dS^T: rows = keys, K-major over q)
            mma2_ss_w(tdK, dDS_k + koff(k), dQB_mn + moff(k), kIdescT, (m > 0 || k > 0) ? 1u : 0u);
          mma2_commit_w(&bars.qb_empty);
          TR(5, m);
        }
        mma2_commit_w(&bars.dkdv_done);
      }
    }
  } else if (warp < 4) {
    setmaxnreg_inc<136>();
    // ===================== dQ reducer (TMEM lane = q row) =====================
    const CUtensorMap* mdq = tmap(a, a.dq_slot);
#if SPPO_DQ_HINT
    const uint64_t dq_policy = policy_evict_last();  // keep the dQ accumulator lines in L2
#endif
    const float tau = p.scale;
    const int row = warp * 32 + lane;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t L_dq_free = mapa(smem_u32(&bars.dq_free), 0);
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
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(L_dq_free);
      if (threadIdx.x == 0) TR(13, m);
      // the last kDqRedPieces 32-column pieces go straight from registers as vector
      // reductions (LSU path), in parallel with the TMA reduces of the others
#pragma unroll
      for (int pc = 4 - kDqRedPieces; pc < 4; ++pc) {
        if (q0 + row < p.q_len) {
          float* dst = p.dq_acc + ((size_t)(q0 + row) * p.heads + head) * HD + pc * 32;
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * c4),
                         "f"(__uint_as_float(v[pc * 32 + 4 * c4 + 0]) * tau),
                         "f"(__uint_as_float(v[pc * 32 + 4 * c4 + 1]) * tau),
                         "f"(__uint_as_float(v[pc * 32 + 4 * c4 + 2]) * tau),
                         "f"(__uint_as_float(v[pc * 32 + 4 * c4 + 3]) * tau)
                         : "memory");
        }
      }
#pragma unroll
      for (int pc = 0; pc < 4 - kDqRedPieces; ++pc, ++piece_ctr) {
        const int buf = piece_ctr % kDqBufs;
        uint8_t* stg = smem + kOffDQ + buf * 16384;
        if (threadIdx.x == 0) bulk_wait_read<kDqBufs - 1>();  // the reduce that last read `buf` is done
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
#if SPPO_DQ_HINT
          tma_reduce_add_3d_hint(mdq, stg, pc * 32, head, q0, dq_policy);
#else
          tma_reduce_add_3d(mdq, stg, pc * 32, head, q0);
#endif
          bulk_commit();
        }
      }
      if (threadIdx.x == 0) TR(14, m);
    }
    if (threadIdx.x == 0) bulk_wait<0>();
  } else {
    setmaxnreg_inc<136>();
    // ===================== compute: P and dS (TMEM lane = key row) =====================
    const int g = (warp - 4) >> 2;  // column half: q in [64g, 64g+64)
    const int wq = warp & 3;
    const int row = wq * 32 + lane;  // key row in this CTA's tile
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int kv_pos = kvp0 + row;
    const bool kv_ok = row < kv_len;
    const float sl2 = p.scale * kLog2e;
    const float tau = p.scale;
    const uint32_t L_p_full = mapa(smem_u32(&bars.p_full), 0), L_ds_full = mapa(smem_u32(&bars.ds_full), 0);
    uint8_t* sDS = smem + kOffDS + g * kBox;
    for (int m = 0; m < M; ++m) {
      const int s = m & 1;
      const int q0 = qtile(m) * BQ;
      const int qpos0 = p.q_start + q0 + g * 64;  // absolute position of this half's column 0
      if (!kFold) mbar_wait(&bars.lse_full[s], (m >> 1) & 1);
      mbar_wait(&bars.s_full, m & 1);
#ifndef SPPO_TRACE_DS
      if (lane == 0 && wq == 0) TR(6 + 4 * g, m);
#endif
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
        for (int c2 = 16 * h; c2 < 16 * h + 16; c2 += 2) {
          float2 x0, x1;
          if (kFold) {  // S already holds s - LSE / tau
            x0 = fmul2(pr[c2], make_float2(sl2, sl2));
            x1 = fmul2(pr[c2 + 1], make_float2(sl2, sl2));
          } else {
            const float4 l4 = *reinterpret_cast<const float4*>(lse2 + 2 * c2);
            x0 = ffma2(pr[c2], make_float2(sl2, sl2), make_float2(-l4.x, -l4.y));
            x1 = ffma2(pr[c2 + 1], make_float2(sl2, sl2), make_float2(-l4.z, -l4.w));
          }
          if (masked) {
            const int j = 2 * c2;
            x0.x = (j + 0 >= first_vis) ? x0.x : -INFINITY;
            x0.y = (j + 1 >= first_vis) ? x0.y : -INFINITY;
            x1.x = (j + 2 >= first_vis) ? x1.x : -INFINITY;
            x1.y = (j + 3 >= first_vis) ? x1.y : -INFINITY;
          }
          if (kBwdEmu > 0 && c2 % kBwdEmu == kBwdEmu - 1)
            pr[c2] = ex2_poly2(x0);
          else
            pr[c2] = make_float2(ex2(x0.x), ex2(x0.y));
          if (kBwdEmu > 0 && (c2 + 1) % kBwdEmu == kBwdEmu - 1)
            pr[c2 + 1] = ex2_poly2(x1);
          else
            pr[c2 + 1] = make_float2(ex2(x1.x), ex2(x1.y));
          pk[c2] = pack_bf16(pr[c2].x, pr[c2].y);
          pk[c2 + 1] = pack_bf16(pr[c2 + 1].x, pr[c2 + 1].y);
        }
        // P^T bf16 pairs into this WG's own S columns: A operand of dV += P^T dO
        tmem_st16(tSg + 16 * h, *reinterpret_cast<uint32_t(*)[16]>(&pk[16 * h]));
      }
      tmem_wait_st();
      tc_fence_before();
      if (!kFold && !kWarpArrive) mbar_arrive(&bars.lse_empty[s]);  // every thread: its LSE reads are done
      __syncwarp();
      if (lane == 0) {
        if (!kFold && kWarpArrive) mbar_arrive(&bars.lse_empty[s]);  // the warp's LSE reads are done
        mbar_arrive_cluster(L_p_full);
      }
      if (lane == 0 && wq == 0 && g == 0) TR(7, m);

      // ---- dS = P (dP - Delta)   (tau is applied to dK / dQ at their write-out)
      if (!kFold) mbar_wait(&bars.delta_full[s], (m >> 1) & 1);
      mbar_wait(&bars.dp_full, m & 1);
      if (lane == 0 && wq == 0 && g == 0) TR(8, m);
      tc_fence_after();
      const uint32_t tPg = tdP + lane_off + g * 64;
      const float* dl = sDelta + s * 128 + g * 64;
      float2 dp[32];
      tmem_ld32(tPg, *reinterpret_cast<uint32_t(*)[32]>(&dp[0]));
      tmem_wait_ld();
#ifdef SPPO_TRACE_DS
      if (lane == 0 && wq == 0 && g == 1) TR(10, m);  // WG1: first dP half in registers
#endif
      tmem_ld32(tPg + 32, *reinterpret_cast<uint32_t(*)[32]>(&dp[16]));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1) tmem_wait_ld();
#pragma unroll
        for (int c2 = 16 * h; c2 < 16 * h + 16; c2 += 2) {
          float2 t0 = dp[c2], t1 = dp[c2 + 1];  // fold: dP already holds dP - Delta
          if (!kFold) {
            const float4 d4 = *reinterpret_cast<const float4*>(dl + 2 * c2);
            t0 = fadd2(t0, make_float2(-d4.x, -d4.y));
            t1 = fadd2(t1, make_float2(-d4.z, -d4.w));
          }
          const float2 a0 = fmul2(pr[c2], t0);
          const float2 a1 = fmul2(pr[c2 + 1], t1);
          pk[c2] = pack_bf16(a0.x, a0.y);
          pk[c2 + 1] = pack_bf16(a1.x, a1.y);
        }
#pragma unroll
        for (int ch = 4 * h; ch < 4 * h + 4; ++ch)  // dS: row = key, 64 q per half (A of dQ and of dK)
          *reinterpret_cast<uint4*>(sDS + sw128(row, ch * 16)) =
              make_uint4(pk[ch * 4 + 0], pk[ch * 4 + 1], pk[ch * 4 + 2], pk[ch * 4 + 3]);
      }
#ifdef SPPO_TRACE_DS
      if (lane == 0 && wq == 0 && g == 1) TR(11, m);  // WG1: dS math + stores issued
#endif
      fence_proxy_async_smem();
      tc_fence_before();
      if (!kWarpArrive) {
        if (!kFold) mbar_arrive(&bars.delta_empty[s]);  // every thread: its Delta reads are done
        if (!leader) mbar_arrive(&bars.ds_local);  // the peer's own dQ MMA waits on this
      }
      __syncwarp();
      if (lane == 0) {
        if (kWarpArrive) {
          if (!kFold) mbar_arrive(&bars.delta_empty[s]);  // the warp's Delta reads are done
          if (!leader) mbar_arrive(&bars.ds_local);  // its dS stores fenced: the peer's own dQ MMA waits on this
        }
        mbar_arrive_cluster(L_ds_full);
      }
#ifdef SPPO_TRACE_DS
      if (lane == 0 && wq == 0 && g == 0) TR(9, m);
#else
      if (lane == 0 && wq == 0) TR(9 + 2 * g, m);
#endif
    }
    // ---- epilogue: dK_j, dV_j of this key tile (+= into the fp32 accumulators).
    // One key row per thread, so a warp's vector reduction touches 32 different
    // rows.  Staging the tile in shared memory and reducing whole 512-byte rows per
    // warp (coalesced) measured bwd -6 % (profiles/r02): reductions to the same L2
    // line serialise, spread ones proceed in parallel.
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
            const float f = which == 0 ? 1.f : tau;  // dK = tau dS^T Q
            if (kEpiRed && !final_out) {  // += as a fire-and-forget vector reduction (L2 does the RMW)
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(ap),
                           "f"(__uint_as_float(v[q4 * 4 + 0]) * f), "f"(__uint_as_float(v[q4 * 4 + 1]) * f),
                           "f"(__uint_as_float(v[q4 * 4 + 2]) * f), "f"(__uint_as_float(v[q4 * 4 + 3]) * f)
                           : "memory");
              continue;
            }
            float4 o = *ap;
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
  cluster_sync();  // the peer's smem / TMEM / barriers stay live until both CTAs are done
  if (warp == 14) tmem_dealloc_pair<512>(tmem);
}

}  // namespace

cudaError_t launch_bwd_sm100(const Sm100Bwd& a, cudaStream_t s) {
  if (a.p.d != HD) return cudaErrorNotSupported;
  cudaError_t e = ensure_smem_attr((const void*)bwd_kernel, kSmemBytes);
  if (e != cudaSuccess) return e;
  dim3 grid(2 * a.pair_base[a.n], a.p.heads);
  bwd_kernel<<<grid, kThreads, kSmemBytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sppo
