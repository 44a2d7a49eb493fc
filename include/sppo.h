/*
 * sppo.h — C ABI of the SPPO hot path on B200 (sm_100a):
 * subsequence-chunked causal attention forward/backward with per-chunk
 * offload/prefetch of activations and KV to pinned host memory.
 *
 * What is computed (PAPER.md = /root/reference/PAPER.md):
 *   P:356 [§5.1 Two-Level Activation Management]: "due to the casual mask, after
 *   attention computation, Q_i will not be used in the forward pass anymore,
 *   while K_i and V_i need to participate in the following Q_N computation,
 *   where i<N" — chunk i's queries attend causally to the K/V of chunks 0..i.
 *   P:369 [§5.2]: "overlapping data transfer operations for the (i-1)-th
 *   subsequence with the computation of the i-th subsequence".
 *   offloaded activations "just need to reside in GPU memory at least
 *   before the backward propagation of the subsequence begins".
 *   P:371-377 [§5.2]: offload ratio alpha_i with alpha_i * A_i = M_threshold.
 *
 * Conventions (readings):
 *   - tau = 1/sqrt(d) unless layout.scale != 0                      (L1)
 *   - row p (absolute position) sees keys t <= p                    (L2)
 *   - chunks 0..N-1, offsets c_0 = 0 < c_1 < ... < c_N = S          (L3, L4)
 *   - LSE is natural-log, fp32, head-major [heads, s_i]             (L5)
 *   - bf16 path: bf16 in, fp32 accumulate, P and dS rounded to bf16
 *     before their MMAs; fp32 path: FP32 FMA only (no TF32)        (L6)
 *
 * Tensor layout: every per-chunk activation is token-major [s_j, heads, d]
 * (contiguous, row stride heads*d elements), so one chunk is one allocation
 * and one offload is one cudaMemcpyAsync.  [s, heads, d] device pointers must
 * be 16-byte aligned, [heads, s] fp32 vectors (lse, delta, m, l) 4-byte
 * aligned (SPPO_E_ALIGN otherwise).  dtype: SPPO_BF16 (tensor-core path, d = 128) or SPPO_FP32 (SIMT
 * FP32 reference path, d <= 128).
 *
 * Ownership: the caller owns every device and host tensor passed in.  The
 * library owns only the ctx (copy streams, events, TMA descriptor table,
 * window-coverage state) and host buffers returned by sppo_host_alloc.
 * No call frees caller memory.
 *
 * Errors: every call returns sppo_status and never throws.  Arguments are
 * validated on the host before anything is enqueued; on any non-OK status
 * nothing has been enqueued (except SPPO_E_CUDA from a launch, reported via
 * cudaGetLastError).  sppo_last_error() returns thread-local text for the last
 * non-OK status.  There is no CPU fallback and no alternative backend.
 *
 * Streams/events are passed as void* holding a cudaStream_t / cudaEvent_t
 * (NULL stream = legacy default stream).  No call synchronises the device
 * unless its name says so.  Descriptor table: the TMA tensor maps of every
 * (pointer, shape) a call reads live in one persistent device table of the ctx
 * (16384 maps), uploaded once, on first use, on the launch stream; a later call
 * on another stream waits on that upload's event.  When a call's new maps do
 * not fit, the table is recycled first: sppo_attn_fwd / sppo_attn_bwd then wait
 * on the host until every stream that launched from the ctx since the last
 * recycle has drained (rare: thousands of distinct buffers or chunk views).
 */
#ifndef SPPO_H_
#define SPPO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPPO_OK = 0,
  SPPO_E_ARG = 1,          /* null pointer / bad scalar argument              */
  SPPO_E_SHAPE = 2,        /* heads/head_dim/offsets/chunk id inconsistent    */
  SPPO_E_ALIGN = 3,        /* pointer not 16-byte aligned                     */
  SPPO_E_STATE = 4,        /* FIRST/LAST window coverage violated             */
  SPPO_E_NOT_RESIDENT = 5, /* reserved                                        */
  SPPO_E_OOM = 6,          /* host/device allocation failed                   */
  SPPO_E_CUDA = 7,         /* CUDA runtime/driver error (launch or async)     */
  SPPO_E_UNSUPPORTED = 8   /* valid request this build does not implement     */
} sppo_status;

enum { SPPO_BF16 = 0, SPPO_FP32 = 1 };

/* flags of sppo_attn_fwd / sppo_attn_bwd */
enum {
  SPPO_FIRST = 1, /* first window of chunk i: start a fresh state            */
  SPPO_LAST = 2   /* last window of chunk i: finalise outputs                */
};

typedef struct sppo_ctx_s* sppo_ctx;

/* One ctx per (device, host thread).  Creates two copy streams (D2H, H2D). */
sppo_status sppo_ctx_create(int device, sppo_ctx* out);
sppo_status sppo_ctx_destroy(sppo_ctx ctx);
/* Synchronises the device; surfaces asynchronous CUDA faults as SPPO_E_CUDA. */
sppo_status sppo_ctx_sync(sppo_ctx ctx);
const char* sppo_last_error(void);
int32_t sppo_version(void);

/* Problem layout shared by every call of one sequence (per device). */
typedef struct {
  int32_t heads;          /* heads on this device (h_dev = h / G, §8(e))         */
  int32_t head_dim;       /* d                                                   */
  int32_t dtype;          /* SPPO_BF16 | SPPO_FP32                               */
  int32_t num_chunks;     /* N                                                   */
  const int64_t* offsets; /* HOST array, N+1 entries, 0 = c_0 < ... < c_N = S    */
  float scale;            /* softmax scale tau; 0 => 1/sqrt(d)                   */
} sppo_layout;

/* Prior-KV set of one call: chunk ids (ascending or not, each <= chunk i,
 * no duplicates) and their device buffers K_j, V_j, each [s_j, heads, d]. */
typedef struct {
  int32_t n;
  const int32_t* ids;    /* HOST array of n chunk ids                    */
  const void* const* k;  /* HOST array of n DEVICE pointers              */
  const void* const* v;  /* HOST array of n DEVICE pointers              */
} sppo_kv_set;

/* Online-softmax carry between windows of one chunk.
 * fp32 DEVICE scratch owned by the caller: o_acc [s_i, heads, d]
 * (unnormalised), m and l [heads, s_i].  Needed unless flags == FIRST|LAST. */
typedef struct {
  float* o_acc;
  float* m;
  float* l;
} sppo_fwd_state;

/*
 * sppo_attn_fwd — forward of chunk i over one window of its prior-KV set.
 *   P:356 (chunk i attends to K_j, V_j, j <= i).  For every row p of chunk i
 *   and key t <= p in the window: s = tau <q_p, k_t>; online softmax over the
 *   window; on LAST: O_p = sum softmax * v_t and LSE_p = m + ln l.
 *   q   : DEVICE [s_i, heads, d] (dtype)
 *   kv  : window; over FIRST..LAST calls of chunk i the ids must cover 0..i
 *         exactly once (SPPO_E_STATE otherwise)
 *   st  : carry state (may be NULL when flags == FIRST|LAST)
 *   o   : DEVICE [s_i, heads, d] (dtype), written on LAST
 *   lse : DEVICE [heads, s_i] fp32, written on LAST
 * Enqueued on `stream`; returns after enqueue.
 */
sppo_status sppo_attn_fwd(sppo_ctx ctx, const sppo_layout* layout, int32_t chunk,
                          const void* q, const sppo_kv_set* kv, int32_t flags,
                          const sppo_fwd_state* st, void* o, float* lse, void* stream);

/*
 * sppo_attn_fwd_chunks — forward of chunks i0..i1-1 in ONE launch, each over its
 *   whole prior-KV set (one window, FIRST|LAST; same results as sppo_attn_fwd
 *   per chunk).  The Q tiles of all the chunks form one grid ordered longest
 *   chunk first (the last wave holds the shortest work), and their CTAs sweep
 *   the shared K/V from position 0 upward together — the per-chunk launches'
 *   wave tails and launch gaps disappear (SURVEY §8(e) "persistent scheduler").
 *   Chunk i's queries still see only keys t <= p.  bf16 only
 *   (SPPO_E_UNSUPPORTED for fp32: use sppo_attn_fwd per chunk).
 *   q, o : HOST arrays of i1 - i0 DEVICE pointers, chunk i0 + k at [k], each [s_i, heads, d]
 *   lse  : HOST array of i1 - i0 DEVICE pointers, each [heads, s_i] fp32
 *   kv   : ids exactly 0..i1-1 in ascending order (SPPO_E_ARG otherwise)
 * Enqueued on `stream`; returns after enqueue.
 */
sppo_status sppo_attn_fwd_chunks(sppo_ctx ctx, const sppo_layout* layout, int32_t i0, int32_t i1,
                                 const void* const* q, const sppo_kv_set* kv, void* const* o, float* const* lse,
                                 void* stream);

/* Backward tensors of chunk i.  All DEVICE pointers. */
typedef struct {
  const void* o;          /* [s_i, heads, d] dtype: forward output O_i              */
  const float* lse;       /* [heads, s_i] fp32: forward LSE_i                       */
  const void* dout;       /* [s_i, heads, d] dtype: upstream gradient dO_i          */
  float* delta;           /* [heads, s_i] fp32 scratch: Delta_i, written on FIRST   */
  float* dq_acc;          /* [s_i, heads, d] fp32 scratch: zeroed on FIRST, += each */
  float* const* dk_acc;   /* HOST array aligned with kv->ids: DEVICE [s_j,heads,d]  */
  float* const* dv_acc;   /*   fp32 accumulators, += (caller zeroes before bwd(N-1)) */
  void* dq;               /* [s_i, heads, d] dtype: dQ_i, written on LAST           */
  void* dk;               /* optional [s_i, heads, d] dtype: final dK_i, written by  */
  void* dv;               /*   the call whose window holds chunk i (else NULL)      */
} sppo_bwd_args;

/*
 * sppo_attn_bwd — backward of chunk i over one window (chunks in strictly
 * descending order N-1..0, reading L11; dK_j/dV_j final after bwd(j)).
 *   Delta_p = <dO_p, O_p>;  P = exp(tau q.k - LSE);  dV_j += P^T dO_i;
 *   dP = dO_i V_j^T;  dS = P (dP - Delta);  dQ_i += tau dS K_j;
 *   dK_j += tau dS^T Q_i   for every j in the window.
 * Enqueued on `stream`: Delta (FIRST), a 4-byte reset of the launch's work counter,
 * the backward kernel (bf16: persistent CTA pairs taking 256-key x head items from
 * that counter), the dQ cast (LAST).  dK_j/dV_j accumulate by TMA reduce-add, so
 * the order of the fp32 additions into dk_acc/dv_acc is not fixed.
 */
sppo_status sppo_attn_bwd(sppo_ctx ctx, const sppo_layout* layout, int32_t chunk,
                          const void* q, const sppo_kv_set* kv, const sppo_bwd_args* a,
                          int32_t flags, void* stream);

/*
 * sppo_finalize — a7 as a standalone call: dst(dtype) = src(fp32), n elements,
 * RNE for SPPO_BF16, a copy for SPPO_FP32.  For gradient accumulators that were
 * completed outside the descending chunk order (e.g. rotated around a ring of
 * GPUs, context parallelism): sppo_attn_bwd writes the final dK_i / dV_i itself
 * only when its window holds chunk i and it is the last contributor.
 *   src : DEVICE fp32, 16-byte aligned;  dst : DEVICE dtype, 16-byte aligned
 *   n   : multiple of 4 (SPPO_E_SHAPE otherwise)
 * Enqueued on `stream`.
 */
sppo_status sppo_finalize(sppo_ctx ctx, const float* src, void* dst, size_t n, int32_t dtype, void* stream);

/* ---- two-level activation management: pinned host arena + copies ------- */

/* Pinned (page-locked) host memory, NUMA-local to the ctx's GPU (P:472 [§7]:
 * "bind the NUMA node ... page-locked memory"): the GPU's node is read from
 * sysfs at sppo_ctx_create; the pages are bound to it (mbind, preferred) before
 * first touch and page-locked with cudaHostRegister.  When the node is unknown
 * or the placement is refused, a portable cudaHostAlloc is used instead.
 * Returns SPPO_E_OOM if neither succeeds.  Free with sppo_host_free (same ctx);
 * sppo_ctx_destroy frees what is left. */
sppo_status sppo_host_alloc(sppo_ctx ctx, size_t bytes, void** host);
sppo_status sppo_host_free(sppo_ctx ctx, void* host);
/* NUMA node of the ctx's GPU as seen by sppo_host_alloc (-1 = unknown). */
sppo_status sppo_ctx_numa_node(sppo_ctx ctx, int32_t* node);

/*
 * sppo_kv_offload — D2H copy of chunk `chunk`'s buffer prefix to host, on the
 * ctx's D2H copy stream, after all work already enqueued on `producer`
 * (P:369 overlap; P:371 offload ratio).  Copies
 *   n = min(bytes, round_up(alpha * bytes, granule))   bytes, granule = 64 KiB,
 * i.e. the alpha-prefix of the token-major buffer (reading L8).  alpha in
 * [0,1]; alpha = 0 copies nothing.  If `done` (cudaEvent_t) is non-NULL it is
 * recorded on the D2H stream after the copy: the caller must not overwrite or
 * free `dev` before `done` completes.  `*copied` (optional) receives n.
 */
sppo_status sppo_kv_offload(sppo_ctx ctx, int32_t chunk, const void* dev, void* host,
                            size_t bytes, double alpha, void* producer, void* done,
                            size_t* copied);

/* flags of sppo_kv_prefetch */
enum {
  SPPO_COPY_NO_ORDER = 1,   /* do not order the copy after `consumer`'s enqueued work */
  SPPO_COPY_DEFER_WAIT = 2  /* do not make `consumer` wait; the caller waits on `done` */
};

/*
 * sppo_kv_prefetch — H2D copy of `bytes` from host back to `dev` on the ctx's
 * H2D copy stream (offloaded activations must be resident "before the
 * backward propagation of the subsequence begins").  By default (flags = 0)
 * the copy starts after all work already enqueued on `consumer` (so `dev` is
 * free) and `consumer` waits for the copy before any later work.
 * SPPO_COPY_NO_ORDER drops the first ordering (dev known to be free);
 * SPPO_COPY_DEFER_WAIT drops the second: the caller must make its stream wait
 * on `done` (required then) before reading `dev` — this is how a copy is
 * overlapped with compute enqueued after the call.  `done` (cudaEvent_t,
 * optional otherwise) is recorded on the H2D stream after the copy.
 */
sppo_status sppo_kv_prefetch(sppo_ctx ctx, int32_t chunk, const void* host, void* dev,
                             size_t bytes, void* consumer, void* done, int32_t flags);

/* The ctx's copy streams (cudaStream_t) that sppo_kv_offload (D2H) and
 * sppo_kv_prefetch (H2D) enqueue on, for callers that order or time work
 * against them (e.g. events recorded around copies for an overlap timeline).
 * The ctx keeps ownership; either output may be NULL. */
sppo_status sppo_ctx_streams(sppo_ctx ctx, void** d2h, void** h2d);

/* ---- host-side plan helpers ----------------------- */

/* Equal partition: N+1 offsets, first S mod N chunks longer. */
sppo_status sppo_partition_equal(int64_t S, int32_t N, int64_t* offsets_out);
/* FLOPs-balanced partition (P:253, P:256, P:327 [§3.2, §4]): the N
 * chunks minimising the largest per-chunk causal pair count (attention FLOPs),
 * ties broken toward longer leading chunks (lengths come out non-increasing).
 * Writes N+1 offsets.  O(N log^2 S). */
sppo_status sppo_partition_balanced(int64_t S, int32_t N, int64_t* offsets_out);
/* Same with a per-token linear term (S:46 [forward_flops] c_lin H^2 s_len; the
 * token-wise GEMM / LayerNorm work of a full layer): minimises
 * max_i (pairs_i + lin * s_i), lin in pair units (e.g. a GPT layer, fwd+bwd:
 * 72 h^2 s + 14 h pairs FLOPs -> lin = 36 h / 7).  lin = 0 is the call above. */
sppo_status sppo_partition_balanced_lin(int64_t S, int32_t N, int64_t lin, int64_t* offsets_out);
/* Causal (q,k) pairs of all chunks: sum_i s_i c_i + s_i (s_i + 1) / 2. */
sppo_status sppo_causal_pairs(const int64_t* offsets, int32_t N, int64_t* pairs_out);
/* Sequence-aware offload ratio (P:371-377 [§5.2]; reading L9):
 * alpha_i = min(1, M_i / A_i) for i < N-1 with M_i = m_threshold[i] (the bytes
 * the D2H link moves during the compute that the offload of chunk i overlaps,
 * BW_D2H * T_comp(i+1); the paper's single M_threshold is the constant case),
 * alpha_{N-1} = last, A_i <= 0 => alpha_i = 1.  m_threshold has N entries. */
sppo_status sppo_offload_alpha(const double* A, const double* m_threshold, int32_t N, double last,
                               double* alpha_out);

#ifdef __cplusplus
}
#endif
#endif /* SPPO_H_ */
