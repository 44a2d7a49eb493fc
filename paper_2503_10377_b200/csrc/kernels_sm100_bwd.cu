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
// Persistent: the grid is one CTA pair per two SMs; a pair takes work items (256
// keys x one head; head-major, longest first within a head) from a per-launch
// counter as it becomes free, and the item boundaries overlap: the next item's V
// loads as soon as the last dP^T has read V (v_free), its K once the last dQ has
// read K (k_free), its first S^T/dP^T/P run
// while the reducer warps drain the last item's dV/dK out of TMEM (acc_free gates
// only the next dV MMA), and the dK/dV accumulator += goes through the reducers'
// TMA reduce-add ring like dQ.  Per-CTA
// lifetime traces of the one-launch-per-item kernel (tools/life_stats.py) showed
// ~25K cycles per CTA outside the Q-tile loop (setup, K/V fill, epilogue,
// teardown, launch gap): 8.5 % of SM time at 8K chunks, 28 % at 2K chunks.
// 512 threads per CTA:
//   warps 0-3   dQ reducer: tcgen05.ld dQ -> swizzled smem -> TMA reduce-add;
//               item epilogue: dV/dK TMEM -> TMA reduce-add (or final bf16 rows)
//   warps 4-11  compute: P (exp2) and dS; WG A owns q columns 0-63, WG B 64-127
//               of every TMEM lane (= key row)
//   warp 12     MMA issuer: pair MMAs + own dQ (leader), own dQ (peer)
//   warp 13     TMA: K, V once per item; Q rows half + LSE per tile
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
// Reduce staging ring: [128 rows][32 fp32] SW128 pieces (dQ pieces; dK/dV pieces of the
// item epilogue).  Measured alternatives for dQ (profiles/r02): 4 buffers with each
// reducer warp issuing its own piece -> bwd 950-955 vs 1037-1039 TF/s; the 4 pieces as
// ONE 4-D reduce -> 937 vs 1049; pair-summed partials over DSMEM stores -> 612-720.
// tools/red_bench.cu: an SM pushes ~24 B/clk of fp32 bulk reduce-add into L2 (~32 B/clk
// of plain bulk stores, ~13 B/clk of red.global.add.v4 with one row per thread).
constexpr int kDqBufs = 2;
constexpr uint32_t kStageA = 2 * kHBox;  // one [64 rows][128 d] K-major stage
// dynamic smem map (bytes); the base is 1024-aligned (no static smem is used)
constexpr uint32_t kOffK = 0;                  // own K, K-major: A of S^T = K Q^T (MN-major B of dQ)
constexpr uint32_t kOffV = kOffK + kTile;      // own V, K-major: A of dP^T = V dO^T
constexpr uint32_t kOffQA = kOffV + kTile;     // Q rows [64r,+64), all d, K-major: B of S^T
constexpr uint32_t kOffQB = kOffQA + kStageA;  // Q all rows, d cols [64r,+64), MN-major: B of dK
constexpr uint32_t kOffOA = kOffQB + kBox;     // dO rows half: B of dP^T
constexpr uint32_t kOffOB = kOffOA + kStageA;  // dO cols half: B of dV
constexpr uint32_t kOffDS = kOffOB + kBox;     // dS [128 keys][128 q] (two q halves): A of dQ and dK
constexpr uint32_t kOffDQ = kOffDS + kTile;    // reduce staging ring
constexpr uint32_t kOffLSE = kOffDQ + kDqBufs * 16384;  // 2 x 128 fp32 (LSE * log2 e)
constexpr uint32_t kOffDelta = kOffLSE + 1024;          // 2 x 128 fp32
constexpr uint32_t kOffBars = kOffDelta + 1024;
constexpr uint32_t kSmemBytes = kOffBars + 512;
static_assert(kSmemBytes <= 232448, "smem budget");
// A second K buffer (the next item's K prefetched during the item's first tiles, in the
// 32 KB still free) measured slower: the items whose K sat in the second buffer ran
// ~800 cycles per Q tile slower (trace: 4200-4300 vs 3450), at either free position and
// with every SS MMA's operands in different 128 KB halves (bwd 1003-1013 vs 1040-1053
// TF/s without it).  K of the next item loads after k_free instead (~3.5K cycles).
#ifndef SPPO_BWD_EMU_EVERY
#define SPPO_BWD_EMU_EVERY 0  // 1 of every N exp2 pairs of P on the FMA pipe (cubic, as the forward); 0 = off
#endif
constexpr int kBwdEmu = SPPO_BWD_EMU_EVERY;
constexpr int kEmuDiv = kBwdEmu > 0 ? kBwdEmu : 1;  // (no modulo by zero when off)
// register budget per role (the launch gives 128 per thread: 512 x 128 = 65536).
// Measured: compute 160 / control 56 -> bwd 1022-1027, compute 152 / control 72 ->
// 1075-1080 vs 1103 TF/s (the MMA / producer warps spill).
#ifndef SPPO_BWD_REGS_COMP
#define SPPO_BWD_REGS_COMP 136  // compute warps 4-11
#endif
#ifndef SPPO_BWD_REGS_RED
#define SPPO_BWD_REGS_RED 136   // dQ reducer warps 0-3
#endif
#ifndef SPPO_BWD_REGS_CTRL
#define SPPO_BWD_REGS_CTRL 104  // MMA issuer + TMA producers, warps 12-15
#endif
static_assert(256 * SPPO_BWD_REGS_COMP + 128 * SPPO_BWD_REGS_RED + 128 * SPPO_BWD_REGS_CTRL <= 512 * 128,
              "setmaxnreg budget exceeds the launch's register allocation (the increase would never complete)");
#ifndef SPPO_BWD_ROT
#define SPPO_BWD_ROT 1  // measured: without the rotation bwd 985.6-986.0 vs 1042.0-1049.1 TF/s
#endif

constexpr uint32_t kIdescS = idesc_bf16(256, 128, 0, 0);  // pair, K-major x K-major
constexpr uint32_t kIdescT = idesc_bf16(256, 128, 0, 1);  // pair, TMEM or K-major A x MN-major B
constexpr uint32_t kIdescQ = idesc_bf16(128, 128, 1, 1);  // one CTA, MN-major x MN-major
constexpr float kLog2e = 1.4426950408889634f;

#ifndef SPPO_BWD_KV_LANES
#define SPPO_BWD_KV_LANES 1  // K / V loads issued by lanes 1 / 2 of warp 13, Q rows by lane 0: bwd +1.9 % (1094 vs 1075 TF/s)
#endif
constexpr int kKLane = SPPO_BWD_KV_LANES ? 1 : 0, kVLane = SPPO_BWD_KV_LANES ? 2 : 0;
// (Measured without gain: the Q column half issued by a second lane of warp 14, and
// each staging buffer's reduces issued by its own reducer warp: bwd within +-0.5 %.)
// Item ring depth: the scheduler runs at most ~4 items ahead of the slowest consumer
// (the reducers): publishing item j+4 (during item j+3) needs item j+3's K loaded ->
// k_free(j+2) -> the MMA finished item j+2 -> acc_free(j+1) -> the reducers read
// out item j+1 (so entries j+2 .. j+4 may be live).
constexpr int kItemRing = 8;
struct Bars {
  uint64_t k_full, v_full;            // leader: K (alternating buffers) / V of both CTAs (tx), once per item
  uint64_t qa_full, qb_full;          // leader (tx of both CTAs)
  uint64_t oa_full, ob_full;          // leader (tx of both CTAs)
  uint64_t qa_empty, qb_empty;        // both (MMA commit multicast)
  uint64_t oa_empty, ob_empty;        // both
  uint64_t lse_full[2], delta_full[2];    // local: producer lanes (32)
  uint64_t lse_empty[2], delta_empty[2];  // local: compute warps (8)
  uint64_t s_full, dp_full, dq_full;  // both (MMA commit multicast)
  uint64_t p_full, ds_full;           // leader: compute warps of both CTAs (16)
  uint64_t ds_local;                  // peer only: compute warps (8), dS in smem, dP read
  uint64_t dq_free;                   // leader: reducer warps of both CTAs (8)
  uint64_t dkdv_done;                 // both: the item's last dK MMA (multicast), per item
  uint64_t k_free;                    // both: K of the item no longer read (multicast after dK + own dQ commit)
  uint64_t v_free;                    // both: V of the item no longer read (multicast after the last dP^T)
  uint64_t acc_free;                  // leader: dV/dK TMEM read out by the reducers of both CTAs (8)
  // item schedule: the leader's warp 13 takes items from a global counter and
  // publishes each one (and a final k >= n_items) to both CTAs through this ring
  uint64_t item_full[kItemRing];      // both: one (local or remote) arrival per entry
  int32_t item[kItemRing];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 512, "barrier block");

__device__ __forceinline__ const CUtensorMap* tmap(const Sm100Bwd& a, int slot) {
  return reinterpret_cast<const CUtensorMap*>(a.desc_table) + slot;
}

__device__ __forceinline__ uint32_t sw128(int r, int byte_in_row) {
  const uint32_t lin = r * 128 + byte_in_row;
  return lin ^ (((lin >> 7) & 7u) << 4);
}

// One work item: 256 keys (a CTA pair: rank r owns keys [128r, 128r+128)) of window
// chunk c, one head, against the causally relevant Q tiles of chunk i.  Items are
// numbered head-major (k = head * pairs + pair): the ~74 items in flight at a time
// then belong to one or two heads, so their Q / dO tiles and dQ accumulator rows
// (4 + 4 MB per head at C2) stay in L2 — pair-major numbering (all 32 heads in
// flight, 256 MB) measured bwd 878 vs 1031 TF/s with the SM clock 20 % lower.
// Within a head a later pair never has more Q tiles (longest first).
struct Item {
  int head, c, pair, pair_row0, kv_row0, kv_len, kvp0, qt_first, M, rot;
};
__device__ __forceinline__ Item get_item(const Sm100Bwd& a, int k, uint32_t rank) {
  Item I;
  const int pairs = a.pair_base[a.n];
  I.head = k / pairs;
  I.pair = k - I.head * pairs;
  int lo = 0, hi = a.n - 1;  // last window chunk with pair_base[c] <= pair
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.pair_base[mid] <= I.pair) lo = mid;
    else hi = mid - 1;
  }
  I.c = lo;
  I.pair_row0 = (I.pair - a.pair_base[lo]) * 2 * BKV;  // first key row of the pair within chunk j
  I.kv_row0 = I.pair_row0 + (int)rank * BKV;           // this CTA's key rows
  I.kv_len = min(BKV, a.len[lo] - I.kv_row0);          // valid keys (<= 0: rank 1 of a ragged pair)
  I.kvp0 = a.start[lo] + I.kv_row0;                    // absolute position of key row 0
  // Q tiles of chunk i with some row at position >= the pair's first key
  const int q_tiles = (a.p.q_len + BQ - 1) / BQ;
  I.qt_first = max(0, (a.start[lo] + I.pair_row0 - a.p.q_start) / BQ);
  I.M = q_tiles - I.qt_first;
  // start Q tile rotated per pair: concurrent pairs reduce dQ into different rows
  I.rot = SPPO_BWD_ROT ? (int)(((uint32_t)I.pair * 7u + (uint32_t)I.head * 13u) % (uint32_t)max(I.M, 1)) : 0;
  return I;
}
__device__ __forceinline__ int qtile(const Item& I, int m) { return I.qt_first + (m + I.rot) % I.M; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    bwd_kernel(const __grid_constant__ Sm100Bwd a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars& bars = *reinterpret_cast<Bars*>(smem + kOffBars);
  float* sLSE = reinterpret_cast<float*>(smem + kOffLSE);
  float* sDelta = reinterpret_cast<float*>(smem + kOffDelta);
  const BwdParams& p = a.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  // persistent: cluster g0 of G starts with item g0, then takes items G, G+1, ... from
  // the launch's counter in the order the pairs become free (both CTAs the same ones)
  const int g0 = blockIdx.x >> 1, G = gridDim.x >> 1;
  const int n_items = a.pair_base[a.n] * p.heads;

  // lifetime trace (SPPO_TRACE_LIFE, in a -DSPPO_BWD_LIFE=1 build; tools/life_stats.py)
#ifndef SPPO_BWD_LIFE
#define SPPO_BWD_LIFE 0
#endif
  unsigned long long* life =
      !SPPO_BWD_LIFE ? nullptr : (p.trace && p.trace_life) ? p.trace + (size_t)blockIdx.x * kLifeSlots : nullptr;
  if (life && (size_t)(blockIdx.x + 1) * kLifeSlots > kLifeWords) life = nullptr;
#define LIFE(k)                    \
  do {                             \
    if (life) life[k] = clock64(); \
  } while (0)
  if (threadIdx.x == 0) LIFE(0);

  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023u) != 0) __trap();  // SW128 atoms need 1024 B alignment
    mbar_init(&bars.k_full, 1);
    mbar_init(&bars.v_full, 1);
    mbar_init(&bars.qa_full, 1);
    mbar_init(&bars.qb_full, 1);
    mbar_init(&bars.oa_full, 1);
    mbar_init(&bars.ob_full, 1);
    mbar_init(&bars.qa_empty, 1);
    mbar_init(&bars.qb_empty, 1);
    mbar_init(&bars.oa_empty, 1);
    mbar_init(&bars.ob_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars.lse_full[s], 32);
      mbar_init(&bars.delta_full[s], 32);
      mbar_init(&bars.lse_empty[s], 8);
      mbar_init(&bars.delta_empty[s], 8);
    }
    mbar_init(&bars.s_full, 1);
    mbar_init(&bars.dp_full, 1);
    mbar_init(&bars.dq_full, 1);
    mbar_init(&bars.p_full, 16);
    mbar_init(&bars.ds_full, 16);
    mbar_init(&bars.ds_local, 8);
    mbar_init(&bars.dq_free, 8);
    mbar_init(&bars.dkdv_done, 1);
    mbar_init(&bars.k_free, 2);
    mbar_init(&bars.v_free, 1);
    mbar_init(&bars.acc_free, 8);
    for (int r = 0; r < kItemRing; ++r) mbar_init(&bars.item_full[r], 1);
    fence_mbar_init();
  }
  if (warp == 14) tmem_alloc_pair<512>(&bars.tmem_base);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const uint32_t tS = tmem, tdV = tmem + 128, tdP = tmem + 256, tdK = tmem + 384;
  // leader-side barriers as shared::cluster addresses
  const uint32_t L_k = mapa(smem_u32(&bars.k_full), 0), L_v = mapa(smem_u32(&bars.v_full), 0);
  const uint32_t L_qa = mapa(smem_u32(&bars.qa_full), 0), L_oa = mapa(smem_u32(&bars.oa_full), 0);
  const uint32_t L_qb = mapa(smem_u32(&bars.qb_full), 0), L_ob = mapa(smem_u32(&bars.ob_full), 0);
  // debug trace of CTA 0: clock64 per pipeline event of its first kTraceIters tiles (SPPO_TRACE)
  unsigned long long* tr = (p.trace && !p.trace_life && blockIdx.x == 0) ? p.trace : nullptr;
#define TR(slot, it)                                                              \
  do {                                                                            \
    if (SPPO_TRACE_BUILD && tr && (it) < kTraceIters) tr[(it) * kTraceSlots + (slot)] = clock64();   \
  } while (0)
  if (threadIdx.x == 0) LIFE(1);
  int red_tiles = 0;  // Q tiles this CTA processed (lifetime trace)
  // the j-th item of this pair (k >= n_items: no more)
  auto item_at = [&](int j) -> int {
    const int r = j % kItemRing;
    mbar_wait_cluster(&bars.item_full[r], (j / kItemRing) & 1);
    return *reinterpret_cast<volatile int32_t*>(&bars.item[r]);
  };

  if (warp >= 12) {
    setmaxnreg_dec<SPPO_BWD_REGS_CTRL>();
    if (warp == 13) {
      // ===================== TMA: K, V once per item; Q rows half + LSE per tile =====================
      const CUtensorMap* mq64 = tmap(a, a.q64_slot);
      int gt = 0;
      auto publish = [&](int j, int k) {  // leader lane 0: item j to both CTAs
        const int r = j % kItemRing;
        bars.item[r] = k;
        mbar_arrive(&bars.item_full[r]);
        st_cluster_u32(mapa(smem_u32(&bars.item[r]), 1), (uint32_t)k);
        mbar_arrive_cluster_release(mapa(smem_u32(&bars.item_full[r]), 1));
      };
      // K of the pair's j-th item, once item j-1's MMAs have read the buffer
      auto load_k = [&](int j, const Item& I) {
        if (j >= 1) mbar_wait(&bars.k_free, (j - 1) & 1);
        if (lane == kKLane) {
          const CUtensorMap* mk = tmap(a, a.slots.k[I.c]);
          if (leader) mbar_arrive_expect_tx(&bars.k_full, 2 * kTile);
          tma_load_3d_pair(smem + kOffK, mk, L_k, 0, I.head, I.kv_row0);
          tma_load_3d_pair(smem + kOffK + kBox, mk, L_k, 64, I.head, I.kv_row0);
        }
      };
      if (leader && lane == 0) publish(0, g0);
      int k = leader ? g0 : item_at(0);
      if (k < n_items) load_k(0, get_item(a, k, rank));
      for (int j = 0; k < n_items; ++j) {
        const Item I = get_item(a, k, rank);
        int knext = 0;
        if (leader && lane == 0) knext = G + atomicAdd(a.sched, 1);  // the next item, fetched early
        int kn = n_items;
        const int pf_m = min(1, I.M - 1);  // where the next item is published
        const float* lse_h = p.lse + (size_t)I.head * p.q_len;
        for (int m = 0; m < I.M; ++m, ++gt) {
          const int s = gt & 1;
          const int q0 = qtile(I, m) * BQ;
          if (gt > 0) mbar_wait(&bars.qa_empty, (gt - 1) & 1);
          if (lane == 0) {
            if (leader) mbar_arrive_expect_tx(&bars.qa_full, 2 * kStageA);
            tma_load_3d_pair(smem + kOffQA, mq64, L_qa, 0, I.head, q0 + 64 * (int)rank);
            tma_load_3d_pair(smem + kOffQA + kHBox, mq64, L_qa, 64, I.head, q0 + 64 * (int)rank);
          }
          if (m == 0) {  // this item's V once the previous item's last dP^T has read the buffer
            if (j > 0) mbar_wait(&bars.v_free, (j - 1) & 1);
            if (lane == kVLane) {
              const CUtensorMap* mv = tmap(a, a.slots.v[I.c]);
              if (leader) mbar_arrive_expect_tx(&bars.v_full, 2 * kTile);
              tma_load_3d_pair(smem + kOffV, mv, L_v, 0, I.head, I.kv_row0);
              tma_load_3d_pair(smem + kOffV + kBox, mv, L_v, 64, I.head, I.kv_row0);
            }
          }
          if (m == pf_m) {  // publish the next item
            if (leader) {
              kn = __shfl_sync(0xffffffffu, knext, 0);
              if (lane == 0) publish(j + 1, kn);
            } else {
              kn = item_at(j + 1);
            }
          }
          if (gt >= 2) mbar_wait(&bars.lse_empty[s], ((gt >> 1) - 1) & 1);
          float4 w;
          float* wp = reinterpret_cast<float*>(&w);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = q0 + lane * 4 + e;
            wp[e] = r < p.q_len ? lse_h[r] * kLog2e : INFINITY;  // OOB row -> P = 0
          }
          *reinterpret_cast<float4*>(sLSE + s * 128 + lane * 4) = w;  // one conflict-free STS.128
          if (lane == 0) TR(15, gt);
          mbar_arrive(&bars.lse_full[s]);
        }
        k = kn;
        if (k < n_items) load_k(j + 1, get_item(a, k, rank));  // after this item's MMAs have read K
      }
      for (int t = max(gt - 2, 0); t < gt; ++t) mbar_wait(&bars.lse_empty[t & 1], (t >> 1) & 1);
    } else if (warp == 15) {
      // ===================== TMA: dO rows half + Delta per tile =====================
      const CUtensorMap* mdo64 = tmap(a, a.do64_slot);
      int gt = 0;
      for (int j = 0;; ++j) {
        const int k = item_at(j);
        if (k >= n_items) break;
        const Item I = get_item(a, k, rank);
        const float* delta_h = p.delta + (size_t)I.head * p.q_len;
        for (int m = 0; m < I.M; ++m, ++gt) {
          const int s = gt & 1;
          const int q0 = qtile(I, m) * BQ;
          if (gt > 0) mbar_wait(&bars.oa_empty, (gt - 1) & 1);
          if (lane == 0) {
            if (leader) mbar_arrive_expect_tx(&bars.oa_full, 2 * kStageA);
            tma_load_3d_pair(smem + kOffOA, mdo64, L_oa, 0, I.head, q0 + 64 * (int)rank);
            tma_load_3d_pair(smem + kOffOA + kHBox, mdo64, L_oa, 64, I.head, q0 + 64 * (int)rank);
          }
          if (gt >= 2) mbar_wait(&bars.delta_empty[s], ((gt >> 1) - 1) & 1);
          float4 w;
          float* wp = reinterpret_cast<float*>(&w);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = q0 + lane * 4 + e;
            wp[e] = r < p.q_len ? delta_h[r] : 0.f;
          }
          *reinterpret_cast<float4*>(sDelta + s * 128 + lane * 4) = w;
          mbar_arrive(&bars.delta_full[s]);
        }
      }
      for (int t = max(gt - 2, 0); t < gt; ++t) mbar_wait(&bars.delta_empty[t & 1], (t >> 1) & 1);
    } else if (warp == 14) {
      // ===================== TMA: dO columns half, Q columns half per tile =====================
      const CUtensorMap* mq = tmap(a, a.q_slot);
      const CUtensorMap* mdo = tmap(a, a.do_slot);
      int gt = 0;
      for (int j = 0;; ++j) {
        const int k = item_at(j);
        if (k >= n_items) break;
        const Item I = get_item(a, k, rank);
        for (int m = 0; m < I.M; ++m, ++gt) {
          const int q0 = qtile(I, m) * BQ;
          if (gt > 0) mbar_wait(&bars.ob_empty, (gt - 1) & 1);
          if (lane == 0) {
            if (leader) mbar_arrive_expect_tx(&bars.ob_full, 2 * kBox);
            tma_load_3d_pair(smem + kOffOB, mdo, L_ob, 64 * rank, I.head, q0);
          }
          if (gt > 0) mbar_wait(&bars.qb_empty, (gt - 1) & 1);
          if (lane == 0) {
            if (leader) mbar_arrive_expect_tx(&bars.qb_full, 2 * kBox);
            tma_load_3d_pair(smem + kOffQB, mq, L_qb, 64 * rank, I.head, q0);
          }
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
        int gt = 0;
        for (int j = 0;; ++j) {
          const int k = item_at(j);
          if (k >= n_items) break;
          const int M = get_item(a, k, rank).M;
          for (int m = 0; m < M; ++m, ++gt) {
            mbar_wait(&bars.ds_local, gt & 1);  // dS in this CTA's smem, dP read out of tdP
            tc_fence_after();
            mma_dq();
          }
          mma_commit_w(&bars.k_free);  // own K no longer read by this item's dQ MMAs
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
        auto issue_s = [&](int t) {  // S^T(t) = K Q^T
          mbar_wait(&bars.qa_full, t & 1);
          tc_fence_after();
          mma_kk(tS, dK_k, dQA_k);
          mma2_commit_w(&bars.s_full);
          mma2_commit_w(&bars.qa_empty);
        };
        int gt = 0;
        for (int j = 0;; ++j) {
          const int k = item_at(j);
          if (k >= n_items) break;
          const int M = get_item(a, k, rank).M;
          mbar_wait(&bars.k_full, j & 1);  // this item's K (both CTAs)
          if (gt > 0) TR(3, gt - 1);       // (trace: slot 3 of an item's last tile = next K arrived)
          issue_s(gt);  // S^T of the item's first tile: P of the previous tile consumed (in-order pipe)
          for (int m = 0; m < M; ++m, ++gt) {
            TR(0, gt);
            mbar_wait(&bars.oa_full, gt & 1);
            if (gt > 0) mbar_wait(&bars.dq_free, (gt - 1) & 1);  // both CTAs' reducers have read dQ(gt-1)
            if (m == 0) mbar_wait(&bars.v_full, j & 1);          // this item's V (both CTAs)
            tc_fence_after();
            TR(1, gt);
            mma_kk(tdP, dV_k, dOA_k);  // dP^T = V dO^T
            mma2_commit_w(&bars.dp_full);
            mma2_commit_w(&bars.oa_empty);
            if (m + 1 == M) mma2_commit_w(&bars.v_free);  // both CTAs: V no longer read
            mbar_wait(&bars.p_full, gt & 1);
            mbar_wait(&bars.ob_full, gt & 1);
            if (m == 0 && j > 0) mbar_wait(&bars.acc_free, (j - 1) & 1);  // dV/dK of the last item read out
            tc_fence_after();
            TR(2, gt);
            mma_tmemA(tdV, tS, dOB_mn, m > 0);  // dV += P^T dO
            mma2_commit_w(&bars.ob_empty);
            if (m + 1 < M) {
              TR(3, gt);
              issue_s(gt + 1);  // S^T(m+1): P(m) consumed (in-order pipe)
            }
            mbar_wait(&bars.ds_full, gt & 1);  // both CTAs: dS(m) in smem (implies own ds_local(m))
            tc_fence_after();
            TR(4, gt);
            mma_dq();  // own dQ first: its readout overlaps the pair dK below
            if (m + 1 == M) {            // K no longer read once the last S^T / dQ are done
              mma2_commit_w(&bars.k_free);  // both CTAs: the pair MMAs (the last S^T)
              mma_commit_w(&bars.k_free);   // the leader's own dQ (same count as the peer)
            }
            mbar_wait(&bars.qb_full, gt & 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < BQ / 16; ++kk)  // dK += dS^T Q  (A = dS^T: rows = keys, K-major over q)
              mma2_ss_w(tdK, dDS_k + koff(kk), dQB_mn + moff(kk), kIdescT, (m > 0 || kk > 0) ? 1u : 0u);
            mma2_commit_w(&bars.qb_empty);
            TR(5, gt);
          }
          mma2_commit_w(&bars.dkdv_done);
        }
      }
    }
  } else if (warp < 4) {
    setmaxnreg_inc<SPPO_BWD_REGS_RED>();
    // ===================== dQ reducer + item epilogue (TMEM lane = q row / key row) =====================
    const CUtensorMap* mdq = tmap(a, a.dq_slot);
    const float tau = p.scale;
    const int row = warp * 32 + lane;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t L_dq_free = mapa(smem_u32(&bars.dq_free), 0);
    const uint32_t L_acc_free = mapa(smem_u32(&bars.acc_free), 0);
    int piece_ctr = 0;
    uint32_t v[128];
    // stage v[32 pc .. 32 pc + 31] * f as one [128 rows][32 fp32] SW128 piece and reduce-add it
    auto reduce_piece = [&](const CUtensorMap* map, int pc, float f, int c0, int c1, int c2) {
      const int buf = piece_ctr % kDqBufs;
      ++piece_ctr;
      uint8_t* stg = smem + kOffDQ + buf * 16384;
      if (threadIdx.x == 0) bulk_wait_read<kDqBufs - 1>();  // the reduce that last read `buf` is done
      named_bar_sync(5, 128);
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const float2 x0 = fmul2(make_float2(__uint_as_float(v[pc * 32 + ch * 4 + 0]),
                                            __uint_as_float(v[pc * 32 + ch * 4 + 1])), make_float2(f, f));
        const float2 x1 = fmul2(make_float2(__uint_as_float(v[pc * 32 + ch * 4 + 2]),
                                            __uint_as_float(v[pc * 32 + ch * 4 + 3])), make_float2(f, f));
        *reinterpret_cast<float4*>(stg + sw128(row, ch * 16)) = make_float4(x0.x, x0.y, x1.x, x1.y);
      }
      fence_proxy_async_smem();
      named_bar_sync(5, 128);
      if (threadIdx.x == 0) {
        tma_reduce_add_3d(map, stg, c0, c1, c2);
        bulk_commit();
      }
    };
    int gt = 0;
    for (int j = 0;; ++j) {
      const int k = item_at(j);
      if (k >= n_items) break;
      const Item I = get_item(a, k, rank);
      for (int m = 0; m < I.M; ++m, ++gt) {
        const int q0 = qtile(I, m) * BQ;
        mbar_wait(&bars.dq_full, gt & 1);
        if (threadIdx.x == 0) TR(12, gt);
        tc_fence_after();
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) tmem_ld32(tdP + lane_off + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[cb * 32]));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(L_dq_free);
        if (threadIdx.x == 0) TR(13, gt);
#pragma unroll
        for (int pc = 0; pc < 4; ++pc) reduce_piece(mdq, pc, tau, pc * 32, I.head, q0);  // dQ = tau (dS K)
        if (threadIdx.x == 0) TR(14, gt);
      }
      // ---- item epilogue: dV_j, dK_j of these 128 keys += into the fp32 accumulators
      // (TMA reduce-add through the same staging ring), or load-add and written final
      // in bf16 for chunk i's own keys.  The TMEM regions are released (acc_free) as
      // soon as both are in registers / staged, so the next item's dV MMA can start.
      mbar_wait(&bars.dkdv_done, j & 1);
      tc_fence_after();
      const bool final_out = (I.c == p.final_slot);
      const bool kv_ok = row < I.kv_len;
#pragma unroll 1
      for (int which = 0; which < 2; ++which) {
        const uint32_t tsrc = (which == 0 ? tdV : tdK) + lane_off;
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) tmem_ld32(tsrc + cb * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[cb * 32]));
        tmem_wait_ld();
        if (which == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(L_acc_free);
        }
        const float f = which == 0 ? 1.f : tau;  // dK = tau dS^T Q
        if (!final_out) {
          const CUtensorMap* macc = tmap(a, which == 0 ? a.acc.v[I.c] : a.acc.k[I.c]);
#pragma unroll
          for (int pc = 0; pc < 4; ++pc) reduce_piece(macc, pc, f, pc * 32, I.head, I.kv_row0);
        } else if (kv_ok) {
          const size_t base = ((size_t)(I.kv_row0 + row) * p.heads + I.head) * HD;
          const float* acc = (which == 0 ? a.dv[I.c] : a.dk[I.c]) + base;
          __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(which == 0 ? p.dv_out : p.dk_out) + base;
#pragma unroll
          for (int q4 = 0; q4 < 32; ++q4) {
            float4 o = *reinterpret_cast<const float4*>(acc + q4 * 4);
            o.x += __uint_as_float(v[q4 * 4 + 0]) * f;
            o.y += __uint_as_float(v[q4 * 4 + 1]) * f;
            o.z += __uint_as_float(v[q4 * 4 + 2]) * f;
            o.w += __uint_as_float(v[q4 * 4 + 3]) * f;
            uint2 b;
            b.x = pack_bf16(o.x, o.y);
            b.y = pack_bf16(o.z, o.w);
            *reinterpret_cast<uint2*>(out + q4 * 4) = b;
          }
        }
      }
    }
    if (threadIdx.x == 0) bulk_wait<0>();
    red_tiles = gt;
  } else {
    setmaxnreg_inc<SPPO_BWD_REGS_COMP>();
    // ===================== compute: P and dS (TMEM lane = key row) =====================
    const int g = (warp - 4) >> 2;  // column half: q in [64g, 64g+64)
    const int wq = warp & 3;
    const int row = wq * 32 + lane;  // key row in this CTA's tile
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const float sl2 = p.scale * kLog2e;
    const uint32_t L_p_full = mapa(smem_u32(&bars.p_full), 0), L_ds_full = mapa(smem_u32(&bars.ds_full), 0);
    uint8_t* sDS = smem + kOffDS + g * kBox;
    int gt = 0;
    for (int j = 0;; ++j) {
      const int k = item_at(j);
      if (k >= n_items) break;
      const Item I = get_item(a, k, rank);
      const int kv_pos = I.kvp0 + row;
      const bool kv_ok = row < I.kv_len;
      for (int m = 0; m < I.M; ++m, ++gt) {
        const int s = gt & 1;
        const int q0 = qtile(I, m) * BQ;
        const int qpos0 = p.q_start + q0 + g * 64;  // absolute position of this half's column 0
        mbar_wait(&bars.lse_full[s], (gt >> 1) & 1);
        mbar_wait(&bars.s_full, gt & 1);
        if (gt == 0 && warp == 4 && lane == 0) LIFE(2);
        if (lane == 0 && wq == 0) TR(6 + 4 * g, gt);
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
            const float4 l4 = *reinterpret_cast<const float4*>(lse2 + 2 * c2);
            float2 x0 = ffma2(pr[c2], make_float2(sl2, sl2), make_float2(-l4.x, -l4.y));
            float2 x1 = ffma2(pr[c2 + 1], make_float2(sl2, sl2), make_float2(-l4.z, -l4.w));
            if (masked) {
              const int jj = 2 * c2;
              x0.x = (jj + 0 >= first_vis) ? x0.x : -INFINITY;
              x0.y = (jj + 1 >= first_vis) ? x0.y : -INFINITY;
              x1.x = (jj + 2 >= first_vis) ? x1.x : -INFINITY;
              x1.y = (jj + 3 >= first_vis) ? x1.y : -INFINITY;
            }
            if (kBwdEmu > 0 && c2 % kEmuDiv == kEmuDiv - 1)
              pr[c2] = ex2_poly2(x0);
            else
              pr[c2] = make_float2(ex2(x0.x), ex2(x0.y));
            if (kBwdEmu > 0 && (c2 + 1) % kEmuDiv == kEmuDiv - 1)
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
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars.lse_empty[s]);  // the warp's LSE reads are done
          mbar_arrive_cluster(L_p_full);
        }
        if (lane == 0 && wq == 0 && g == 0) TR(7, gt);

        // ---- dS = P (dP - Delta)   (tau is applied to dK / dQ at their write-out)
        mbar_wait(&bars.delta_full[s], (gt >> 1) & 1);
        mbar_wait(&bars.dp_full, gt & 1);
        if (lane == 0 && wq == 0 && g == 0) TR(8, gt);
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
          for (int c2 = 16 * h; c2 < 16 * h + 16; c2 += 2) {
            const float4 d4 = *reinterpret_cast<const float4*>(dl + 2 * c2);
            const float2 t0 = fadd2(dp[c2], make_float2(-d4.x, -d4.y));
            const float2 t1 = fadd2(dp[c2 + 1], make_float2(-d4.z, -d4.w));
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
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars.delta_empty[s]);        // the warp's Delta reads are done
          if (!leader) mbar_arrive(&bars.ds_local);  // its dS stores fenced: the peer's own dQ MMA waits on this
          mbar_arrive_cluster(L_ds_full);
        }
        if (lane == 0 && wq == 0) TR(9 + 2 * g, gt);
      }
    }
    if (warp == 4 && lane == 0) LIFE(3);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's smem / TMEM / barriers stay live until both CTAs are done
  if (life && threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    life[7] = smid | ((unsigned long long)red_tiles << 32);
    LIFE(6);
  }
  if (warp == 14) tmem_dealloc_pair<512>(tmem);
}

}  // namespace

cudaError_t launch_bwd_sm100(const Sm100Bwd& a, cudaStream_t s) {
  if (a.p.d != HD) return cudaErrorNotSupported;
  cudaError_t e = ensure_smem_attr((const void*)bwd_kernel, kSmemBytes);
  if (e != cudaSuccess) return e;
  // persistent: one CTA pair per two SMs (or fewer when there are fewer items)
  const int items = a.pair_base[a.n] * a.p.heads;
  const int clusters = items < num_sms() / 2 ? items : num_sms() / 2;
  if (clusters <= 0) return cudaSuccess;
  bwd_kernel<<<dim3(2 * clusters), kThreads, kSmemBytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sppo
