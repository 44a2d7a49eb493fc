// sm_100a tensor-core forward of chunked causal attention.
//
// Method: P:356 [§5.1] — chunk i's queries attend causally to K_j, V_j of the
// chunks j <= i in the window; online softmax across KV tiles (FlashAttention,
// P:134); O = softmax * V, LSE = m + ln l (readings L1, L2, L5).
//
// B200 design:
//   CTA = 2 Q tiles x 128 rows of one head, 384 threads, 1 CTA / SM.
//   warp 0      : TMA producer (Q once; K, V tiles through 2-stage rings)
//   warp 1      : MMA issuer (one thread): S_t = Q_t K^T and O_t += P_t V,
//                 tcgen05.mma kind::f16, M=128 N=128 K=16, fp32 accum in TMEM
//   warp 2      : TMEM allocator (512 columns: S0, S1, O0, O1)
//   warps 4-7   : softmax + epilogue of Q tile 0 (one TMEM lane = one row)
//   warps 8-11  : softmax + epilogue of Q tile 1
// P (bf16) overwrites the first 64 columns of its S tile and feeds the PV MMA
// straight from TMEM (A operand); the two Q tiles ping-pong so the tensor core
// computes one tile's MMAs while the other tile's softmax runs.  O is rescaled
// lazily (only when a row max grows by > 8 in log2 units; exact because O and
// l share the stale max).
#include <cuda.h>
#include <math.h>

#include "internal.h"
#include "sm100_ptx.cuh"

namespace sppo {
namespace {
using namespace ptx;

constexpr int BM = 128;                          // rows per Q tile
constexpr int BN = 128;                          // keys per KV tile
constexpr int HD = 128;                          // head dim
constexpr int kThreads = 384;
constexpr uint32_t kTileBytes = BM * HD * 2;     // 32 KB (two 16 KB SW128 boxes)
constexpr uint32_t kHalf = kTileBytes / 2;       // one box: 128 rows x 64 cols
constexpr int kSmemBytes = 6 * kTileBytes + 1024;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;        // log2 units
#ifndef SPPO_EMU_EVERY
#define SPPO_EMU_EVERY 4  // measured best among 2, 3, 4, 6 (tools/gpu_abn.sh)
#endif
constexpr int kEmuEvery = SPPO_EMU_EVERY;        // 1 of every kEmuEvery exp2 pairs on the FMA pipe
#ifndef SPPO_WARP_ARRIVE
#define SPPO_WARP_ARRIVE 1  // P-ready signals as one arrival per warp after __syncwarp
#endif
constexpr bool kWarpArrive = SPPO_WARP_ARRIVE;
#ifndef SPPO_FWD_SPEC
#define SPPO_FWD_SPEC 0  // 1: first 64 exponentials against the stale row max, redone on a rescale (fwd -1 %)
#endif
constexpr bool kSpec = SPPO_FWD_SPEC;
#ifndef SPPO_FWD_TOKEN
#define SPPO_FWD_TOKEN 0
#endif
// Option (off): the two tiles' softmax alternate — tile t runs its exponentials only
// while holding its token (taken once its S is in TMEM, passed to the other tile once
// its P is stored).  tools/softmax_bench.cu puts a lone softmax row at ~1200 cycles
// per SMSP vs ~2000 when both tiles' softmax overlap, and the tiles drift into near
// lockstep (period ~= 2000 + the ~900-cycle S(n+1) chain).  Measured: in the kernel a
// lone row block still takes ~1740 cycles (first LD 140, first 64 exponentials 753,
// row max 244, rest 601) + ~130 for the hand-over, so the period grows to ~3580-3830
// (fwd 987 vs 1084-1090 TF/s): the overlap of the two tiles is worth more.
constexpr bool kToken = SPPO_FWD_TOKEN;

constexpr uint32_t kIdescS = idesc_bf16(128, 128, 0, 0);   // Q (K-major) x K (K-major)
constexpr uint32_t kIdescPV = idesc_bf16(128, 128, 0, 1);  // P (TMEM) x V (MN-major)

struct Bars {
  uint64_t q_full;
  uint64_t k_full[2], k_empty[2];
  uint64_t v_full[2], v_empty[2];
  uint64_t s_full[2];   // S_t ready in TMEM (per Q tile)
  uint64_t p_full[2][2];  // P_t keys [64h, 64h+64) written to TMEM (128 softmax threads arrive)
  uint64_t o_full[2];   // PV_t complete
  uint64_t tok[2];      // softmax token of tile t (4 warps of the other tile arrive)
  uint32_t tmem_base;
};

__device__ __forceinline__ const CUtensorMap* tmap(const Sm100Fwd& a, int slot) {
  return reinterpret_cast<const CUtensorMap*>(a.desc_table) + slot;
}

// KV tile cursor over the window: chunks in order, 128-key tiles within each.
struct TileCursor {
  int c, tt;
  __device__ TileCursor() : c(0), tt(0) {}
  __device__ void next(const Sm100Fwd& a) {
    if ((tt + 1) * BN < a.len[c]) {
      ++tt;
    } else {
      ++c;
      tt = 0;
    }
  }
};

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}


__global__ void __launch_bounds__(kThreads, 1) fwd_kernel(const __grid_constant__ Sm100Fwd a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                       // Q0, Q1
  uint8_t* sK = smem + 2 * kTileBytes;      // 2 stages
  uint8_t* sV = smem + 4 * kTileBytes;      // 2 stages
  __shared__ Bars bars;

  const FwdParams& p = a.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  // ---- this CTA's Q chunk: the call's chunk, or (multi-chunk launch) the chunk whose
  // block range holds blockIdx.x — longest chunks first, so the last wave is short
  int q_start = p.q_start, q_len = p.q_len, q_slot = a.q_slot, o_slot = a.o_slot, win_n = a.n;
  float* lse_out = p.lse;
  int r0 = blockIdx.x * (2 * BM);  // first local row of Q tile 0
  if (a.nq > 0) {
    int k = 0;
    while (k + 1 < a.nq && a.block_base[k + 1] <= (int)blockIdx.x) ++k;
    const int c = a.q0 + a.nq - 1 - k;  // chunk id = its window index
    q_start = a.start[c];
    q_len = a.len[c];
    q_slot = a.qslots[c - a.q0];
    o_slot = a.oslots[c - a.q0];
    lse_out = a.lses[c - a.q0];
    win_n = c + 1;  // later chunks of the window are invisible to these rows
    r0 = ((int)blockIdx.x - a.block_base[k]) * (2 * BM);
  }

  // ---- per-CTA tile counts (the diagonal chunk is last in the window)
  int T[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int first_row = r0 + t * BM;
    if (first_row >= q_len) {
      T[t] = 0;
      continue;
    }
    const int last_pos = q_start + min(first_row + BM, q_len) - 1;
    int n = 0;
    for (int c = 0; c < win_n; ++c) {
      const int st = a.start[c], ln = a.len[c];
      const int hi = min(st + ln - 1, last_pos);  // last visible key of this chunk
      if (hi >= st) n += (hi - st) / BN + 1;
    }
    T[t] = n;
  }
  const int Tn = max(T[0], T[1]);

  if (threadIdx.x == 0) {
    mbar_init(&bars.q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars.k_full[s], 1);
      mbar_init(&bars.k_empty[s], 1);
      mbar_init(&bars.v_full[s], 1);
      mbar_init(&bars.v_empty[s], 1);
      mbar_init(&bars.s_full[s], 1);
      mbar_init(&bars.p_full[s][0], kWarpArrive ? 4 : 128);
      mbar_init(&bars.p_full[s][1], kWarpArrive ? 4 : 128);
      mbar_init(&bars.o_full[s], 1);
      mbar_init(&bars.tok[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&bars.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const uint32_t tS[2] = {tmem + 0, tmem + 128};
  const uint32_t tO[2] = {tmem + 256, tmem + 384};
  unsigned long long* tr = (p.trace && blockIdx.x == 0 && blockIdx.y == 0) ? p.trace : nullptr;
#define TR(slot, it)                                                            \
  do {                                                                          \
    if (SPPO_TRACE_BUILD && tr && (it) < kTraceIters) tr[(it) * kTraceSlots + (slot)] = clock64(); \
  } while (0)

  // register budget per warpgroup: control WG 56, softmax WGs 224 (no merge of the
  // role branches before the teardown, so ptxas allocates per branch)
  if (warp < 4) {
  setmaxnreg_dec<56>();
  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const CUtensorMap* mq = tmap(a, q_slot);
      prefetch_tmap(mq);
      mbar_arrive_expect_tx(&bars.q_full, 2 * kTileBytes);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        tma_load_3d(sQ + t * kTileBytes, mq, &bars.q_full, 0, head, r0 + t * BM);
        tma_load_3d(sQ + t * kTileBytes + kHalf, mq, &bars.q_full, 64, head, r0 + t * BM);
      }
      TileCursor cur;
      for (int n = 0; n < Tn; ++n, cur.next(a)) {
        const int s = n & 1;
        const uint32_t ph = (n >> 1) & 1;
        const CUtensorMap* mk = tmap(a, a.slots.k[cur.c]);
        const CUtensorMap* mv = tmap(a, a.slots.v[cur.c]);
        const int row = cur.tt * BN;
        mbar_wait(&bars.k_empty[s], ph ^ 1);
        TR(11, n);
        mbar_arrive_expect_tx(&bars.k_full[s], kTileBytes);
        tma_load_3d(sK + s * kTileBytes, mk, &bars.k_full[s], 0, head, row);
        tma_load_3d(sK + s * kTileBytes + kHalf, mk, &bars.k_full[s], 64, head, row);
        mbar_wait(&bars.v_empty[s], ph ^ 1);
        TR(12, n);
        mbar_arrive_expect_tx(&bars.v_full[s], kTileBytes);
        tma_load_3d(sV + s * kTileBytes, mv, &bars.v_full[s], 0, head, row);
        tma_load_3d(sV + s * kTileBytes + kHalf, mv, &bars.v_full[s], 64, head, row);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (Tn > 0) {  // whole warp, converged; one elected lane issues (mma_*_w)
      // base descriptors once; a k-step adds (byte offset >> 4) to the start-address field
      const uint64_t dQ0 = sdesc_kmajor(smem_u32(sQ)), dK0 = sdesc_kmajor(smem_u32(sK));
      const uint64_t dV0 = sdesc_mnmajor(smem_u32(sV), kHalf);
      constexpr uint64_t kStep = kTileBytes >> 4;
      auto issue_s = [&](int t, int stage) {
        const uint64_t qa = dQ0 + t * kStep, ka = dK0 + stage * kStep;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint64_t off = ((k >> 2) * kHalf + (k & 3) * 32) >> 4;
          mma_ss_w(tS[t], qa + off, ka + off, kIdescS, k > 0);
        }
        mma_commit_w(&bars.s_full[t]);
      };
      // O_t += P_t V in two K-halves: the first 64 keys go as soon as the softmax has
      // written them, overlapping the exponentials of the second half
      auto issue_pv = [&](int t, int stage, int n) {
        const uint64_t va = dV0 + stage * kStep;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&bars.p_full[t][h], n & 1);
          tc_fence_after();
#pragma unroll
          for (int k = 4 * h; k < 4 * h + 4; ++k)
            mma_ts_w(tO[t], tS[t] + k * 8, va + ((k * 2048) >> 4), kIdescPV,
                     (n > 0 || k > 0 || !p.first) ? 1u : 0u);  // !first: O holds the carried-in state
        }
        mma_commit_w(&bars.o_full[t]);
      };
      mbar_wait(&bars.q_full, 0);
      mbar_wait(&bars.k_full[0], 0);
      tc_fence_after();
      if (T[0] > 0) issue_s(0, 0);
      if (T[1] > 0) issue_s(1, 0);
      mma_commit_w(&bars.k_empty[0]);
      for (int n = 0; n < Tn; ++n) {
        const int vs = n & 1;
        const int nx = n + 1, ks = nx & 1;
        const uint32_t kph = (nx >> 1) & 1;
        mbar_wait(&bars.v_full[vs], (n >> 1) & 1);
        TR(0, n);
        tc_fence_after();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (n < T[t]) {

            TR(1 + 2 * t, n);
            issue_pv(t, vs, n);
            if (nx < T[t]) {
              mbar_wait(&bars.k_full[ks], kph);
              tc_fence_after();
              TR(2 + 2 * t, n);
              issue_s(t, ks);
            }
          }
        }
        if (nx < Tn) mma_commit_w(&bars.k_empty[ks]);
        mma_commit_w(&bars.v_empty[vs]);
      }
    }
  }
  } else {
    setmaxnreg_inc<224>();
    // ===================== softmax + epilogue =====================
    const int t = (warp - 4) >> 2;                 // Q tile of this warpgroup
    const int wq = warp & 3;                       // TMEM lane quarter
    const int row_in_tile = wq * 32 + lane;
    const int row = r0 + t * BM + row_in_tile;     // local row in chunk i
    const int pos = q_start + row;               // absolute position
    const float sl2 = p.scale * kLog2e;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t sS = tS[t] + lane_off, sO = tO[t] + lane_off;
    float m_used = -INFINITY, l = 0.f;
    if (!p.first && T[t] > 0) {
      // carry-in of an earlier window: natural-log m, l and the
      // unnormalised o_acc row go straight into O / the running state; the first
      // tile then proceeds like any later one (speculative exps + rescale check)
      const bool ok = row < q_len;
      const size_t vi = (size_t)head * q_len + row;
      const float m_in = ok ? p.m[vi] * kLog2e : -INFINITY;
      m_used = (m_in == -INFINITY) ? 0.f : m_in;
      l = ok ? p.l[vi] : 0.f;
      const float4* src = reinterpret_cast<const float4*>(p.o_acc + ((size_t)row * p.heads + head) * HD);
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        uint32_t o[32];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float4 x = ok ? src[cb * 8 + v] : make_float4(0.f, 0.f, 0.f, 0.f);
          o[4 * v + 0] = __float_as_uint(x.x);
          o[4 * v + 1] = __float_as_uint(x.y);
          o[4 * v + 2] = __float_as_uint(x.z);
          o[4 * v + 3] = __float_as_uint(x.w);
        }
        tmem_st32(sO + cb * 32, o);
      }
      tmem_wait_st();
    }
    const int Tt = T[t];
    TileCursor cur;
    for (int n = 0; n < Tt; ++n, cur.next(a)) {
      const int kpos0 = a.start[cur.c] + cur.tt * BN;
      const int valid = min(BN, a.len[cur.c] - cur.tt * BN);
      const int limit = min(valid, pos - kpos0 + 1);  // columns >= limit are masked
      mbar_wait(&bars.s_full[t], n & 1);
      // PV(n-1) completed before S(n) (same issuing thread, in-order pipe): consuming its
      // o_full phase here is free and keeps every mbarrier phase waited on (synccheck-clean)
      if (n > 0) mbar_wait(&bars.o_full[t], (n - 1) & 1);
      // softmax token: tile 0 waits from its second row block on (phase n-1, passed by
      // tile 1's softmax n-1), tile 1 from its first (phase n, passed by tile 0's n) —
      // only while the other tile still has that row block (ragged diagonal CTAs).  A
      // tile can pass at most one phase ahead of the other's wait (its next pass needs
      // the other's), so the parity waits never alias.
      if (kToken && (t == 1 ? n < T[0] : (n > 0 && n - 1 < T[1])))
        mbar_wait(&bars.tok[t], (t == 1 ? n : n - 1) & 1);
      if (lane == 0 && wq == 0) TR(5 + 3 * t, n);
      tc_fence_after();
      uint32_t r[128];
      auto R32 = [&](int c) -> uint32_t(&)[32] { return *reinterpret_cast<uint32_t(*)[32]>(&r[c]); };
      // keys 0..63 first; on unmasked later tiles keys 64..127 keep loading while the
      // first 64 exponentials run (split load), otherwise everything is loaded up front
      const bool split = !(n == 0 && p.first) && __all_sync(0xffffffffu, limit >= BN);
      tmem_ld32(sS + 0, R32(0));
      tmem_ld32(sS + 32, R32(32));
      tmem_wait_ld_regs(R32(0));
      tmem_wait_ld_regs(R32(32));
      if (lane == 0 && wq == 0 && t == 0) TR(13, n);  // (trace: first S half in registers)
      tmem_ld32(sS + 64, R32(64));
      tmem_ld32(sS + 96, R32(96));
      if (!split) {
        tmem_wait_ld_regs(R32(64));
        tmem_wait_ld_regs(R32(96));
      }
      float* s = reinterpret_cast<float*>(r);
      if (limit < BN) {
#pragma unroll
        for (int j = 0; j < BN; ++j) s[j] = (j < limit) ? s[j] : -INFINITY;
      }
      auto row_max = [&]() {
        float mx0 = s[0], mx1 = s[1];
#pragma unroll
        for (int j = 2; j < BN - 2; j += 4) {  // two chains of 3-input max (FMNMX3)
          mx0 = fmax3(mx0, s[j], s[j + 1]);
          mx1 = fmax3(mx1, s[j + 2], s[j + 3]);
        }
        return fmax3(mx0, mx1, fmaxf(s[BN - 2], s[BN - 1])) * sl2;
      };
      // P = exp2(s tau log2e - m) for 64 keys from j0, bf16 pairs into out[]; packed
      // FP32x2 math, 1 of every kEmuEvery pairs through a cubic on the FMA pipe
      auto exps = [&](int j0, float negm, uint32_t* out, float2& lsum) {
        const float2 nm2 = make_float2(negm, negm);
        const float2 sl22 = make_float2(sl2, sl2);
#pragma unroll
        for (int j = j0; j < j0 + 64; j += 2) {
          const float2 x = ffma2(make_float2(s[j], s[j + 1]), sl22, nm2);
          float2 e;
          if ((j >> 1) % kEmuEvery == kEmuEvery - 1) {
            e = ex2_poly2(x);
          } else {
            e = make_float2(ex2(x.x), ex2(x.y));
          }
          lsum = fadd2(lsum, e);
          out[(j - j0) >> 1] = pack_bf16(e.x, e.y);
        }
      };
      uint32_t pk0[32];
      float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
      if (n == 0 && p.first) {
        const float mx = row_max();
        m_used = (mx == -INFINITY) ? 0.f : mx;
        exps(0, -m_used, pk0, ls0);
      } else if (!kSpec) {
        // max first (all 128 columns loaded), then the exponentials once.  Measured
        // against the speculative order below (interleaved, trace points out): fwd
        // 1127-1154 vs 1109-1137 TF/s — one exponential path schedules better.
        if (split) {
          tmem_wait_ld_regs(R32(64));
          tmem_wait_ld_regs(R32(96));
        }
        const float mx = row_max();
        const bool need = mx > m_used + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float f = need ? ex2(m_used - mx) : 1.f;
          if (need) {
            m_used = mx;
            l *= f;
          }
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) {
            uint32_t o[32];
            tmem_ld32(sO + cb * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * f);
            tmem_st32(sO + cb * 32, o);
          }
          tmem_wait_st();
        }
        exps(0, -m_used, pk0, ls0);
      } else {
        // speculative: the first 64 exponentials run against the stale max m_used
        // while the row max is computed alongside; only a (rare) rescale redoes them
        exps(0, -m_used, pk0, ls0);
        if (lane == 0 && wq == 0 && t == 0) TR(14, n);  // (trace: first 64 exponentials done)
        if (split) {
          tmem_wait_ld_regs(R32(64));
          tmem_wait_ld_regs(R32(96));
        }
        const float mx = row_max();
        const bool need = mx > m_used + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float f = need ? ex2(m_used - mx) : 1.f;
          if (need) {
            m_used = mx;
            l *= f;
          }
          // PV(n-1) finished writing O (waited above)
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) {
            uint32_t o[32];
            tmem_ld32(sO + cb * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * f);
            tmem_st32(sO + cb * 32, o);
          }
          tmem_wait_st();
          ls0 = make_float2(0.f, 0.f);
          exps(0, -m_used, pk0, ls0);
        }
      }
      if (lane == 0 && wq == 0) TR(6 + 3 * t, n);
      tmem_st32(sS + 0, pk0);  // P keys 0..63 -> the MMA warp starts PV's first half
      tmem_wait_st();
      tc_fence_before();
      if (kWarpArrive) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.p_full[t][0]);
      } else {
        mbar_arrive(&bars.p_full[t][0]);
      }
      exps(64, -m_used, &r[32], ls1);  // keys 64..127 packed over r[32..63] (already consumed)
      tmem_st32(sS + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
      tmem_wait_st();
      tc_fence_before();
      if (lane == 0 && wq == 0) TR(7 + 3 * t, n);
      if (kWarpArrive) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.p_full[t][1]);
      } else {
        mbar_arrive(&bars.p_full[t][1]);
      }
      if (kToken) {  // pass the token (P stored: this tile's MUFU work of row block n is done)
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.tok[t ^ 1]);
      }
      l += ls0.x + ls0.y + ls1.x + ls1.y;
    }
    if (Tt > 0) {
      mbar_wait(&bars.o_full[t], (Tt - 1) & 1);
      tc_fence_after();
      const bool ok = row < q_len;
      if (!p.last) {
        // carry-out for the next window: unnormalised O, natural-log m, l
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
          uint32_t o[32];
          tmem_ld32(sO + cb * 32, o);
          tmem_wait_ld();
          if (ok) {
            float4* dst = reinterpret_cast<float4*>(p.o_acc + ((size_t)row * p.heads + head) * HD + cb * 32);
#pragma unroll
            for (int v = 0; v < 8; ++v)
              dst[v] = make_float4(__uint_as_float(o[4 * v]), __uint_as_float(o[4 * v + 1]),
                                   __uint_as_float(o[4 * v + 2]), __uint_as_float(o[4 * v + 3]));
          }
        }
        if (ok) {
          p.m[(size_t)head * q_len + row] = m_used * 0.6931471805599453f;
          p.l[(size_t)head * q_len + row] = l;
        }
      }
      if (p.last) {
        // O = acc / l in bf16 into the tile's Q buffer (free: its last S MMA completed
        // before the last softmax), SW128 layout, then two TMA stores (coalesced;
        // rows >= q_len clipped by the tensor map)
        const float inv = 1.f / l;
        uint8_t* qb = sQ + t * kTileBytes;
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
          uint32_t o[32];
          tmem_ld32(sO + cb * 32, o);
          tmem_wait_ld();
          uint8_t* box = qb + (cb >> 1) * kHalf;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(o[8 * v + 0]) * inv, __uint_as_float(o[8 * v + 1]) * inv);
            w.y = pack_bf16(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv);
            w.z = pack_bf16(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv);
            w.w = pack_bf16(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv);
            const int chunk16 = (cb & 1) * 4 + v;  // 16-byte chunk within the 128-byte box row
            *reinterpret_cast<uint4*>(box + row_in_tile * 128 + ((chunk16 ^ (row_in_tile & 7)) << 4)) = w;
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(9 + t, 128);  // the tile's four softmax warps staged their rows
        if (wq == 0 && lane == 0) {
          const CUtensorMap* mo = tmap(a, o_slot);
          tma_store_3d(mo, qb, 0, head, r0 + t * BM);
          tma_store_3d(mo, qb + kHalf, 64, head, r0 + t * BM);
          bulk_commit();
          bulk_wait_read<0>();
        }
      }
      if (ok && p.last) lse_out[(size_t)head * q_len + row] = (m_used + __log2f(l)) * 0.6931471805599453f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}



}  // namespace

cudaError_t launch_fwd_sm100(const Sm100Fwd& a, cudaStream_t s) {
  if (a.p.d != HD) return cudaErrorNotSupported;
  dim3 grid(a.nq > 0 ? a.block_base[a.nq] : (a.p.q_len + 2 * BM - 1) / (2 * BM), a.p.heads);
  cudaError_t e = ensure_smem_attr((const void*)fwd_kernel, kSmemBytes);
  if (e != cudaSuccess) return e;
  fwd_kernel<<<grid, kThreads, kSmemBytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sppo
