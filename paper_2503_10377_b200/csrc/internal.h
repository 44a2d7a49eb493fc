// Internal launch interfaces between the C-ABI runtime (sppo_api.cu) and the
// kernels.  Not part of the public ABI (include/sppo.h is).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sppo {

// Maximum number of prior-KV chunks in one window (one launch).  A caller
// with more chunks splits the prior set into several FIRST..LAST windows.
constexpr int kMaxWindow = 256;

// Window description carried in the kernel parameter block (by value).
struct KvWindow {
  int32_t n;                  // chunks in this window
  int32_t start[kMaxWindow];  // absolute position c_j of the chunk's first key
  int32_t len[kMaxWindow];    // s_j
  const void* k[kMaxWindow];  // [s_j, heads, d]
  const void* v[kMaxWindow];
};

struct KvGradWindow {
  float* dk[kMaxWindow];  // fp32 accumulators [s_j, heads, d], +=
  float* dv[kMaxWindow];
};

struct FwdParams {
  int32_t heads, d;
  int32_t q_start, q_len;  // c_i, s_i
  float scale;             // tau
  int32_t first, last;
  const void* q;
  void* o;
  float* lse;
  float* o_acc;  // carry (unnormalised), may be null when first&&last
  float* m;
  float* l;
  unsigned long long* trace;  // debug: per-event clock64 stamps of CTA (0, 0), or null
};

struct BwdParams {
  int32_t heads, d;
  int32_t q_start, q_len;
  float scale;
  int32_t first, last;
  const void* q;
  const void* o;
  const float* lse;
  const void* dout;
  float* delta;
  float* dq_acc;
  void* dq;
  int32_t final_slot;  // window slot holding chunk i when dk/dv outputs are requested, else -1
  void* dk_out;
  void* dv_out;
  unsigned long long* trace;  // debug: per-event clock64 stamps of CTA (0, 0), or null
  int32_t trace_life;         // debug: trace holds kLifeSlots stamps per CTA of the launch instead
};

// Debug tracing (env SPPO_TRACE=<file>): slot layout trace[iter * kTraceSlots + event].
// The clock64 stamps are compiled in only with -DSPPO_TRACE_BUILD=1 (tools/make_variant.sh):
// even untaken, the stamp points constrain the instruction schedule of the hot loops.
#ifndef SPPO_TRACE_BUILD
#define SPPO_TRACE_BUILD 0  // measured: with the stamp points compiled in, fwd 1066 vs 1130-1136 TF/s
#endif
constexpr int kTraceSlots = 16;
constexpr int kTraceIters = 512;
// Lifetime mode (env SPPO_TRACE_LIFE=1, bwd only): trace[cta * kLifeSlots + k], cta =
// blockIdx.y * gridDim.x + blockIdx.x; stamps (clock64): 0 entry, 1 setup done,
// 2 first S seen, 3 loop done, 4 dK/dV done seen, 5 epilogue issued, 6 exit, 7 smid | M << 32
constexpr int kLifeSlots = 8;
constexpr size_t kLifeWords = (size_t)1 << 22;

// ---- SIMT kernels (fp32 path; exact FP32 FMA, no tensor cores) ----------
cudaError_t launch_fwd_simt_f32(const FwdParams& p, const KvWindow& w, cudaStream_t s);
cudaError_t launch_bwd_simt_f32(const BwdParams& p, const KvWindow& w, const KvGradWindow& g,
                                cudaStream_t s);

// ---- sm_100a tensor-core kernels (bf16, d = 128) -------------------------
// Descriptor tables (CUtensorMap, 128 B each) live in device memory owned by
// the ctx; kernels receive slot indices.
struct TmaSlots {
  uint16_t k[kMaxWindow];
  uint16_t v[kMaxWindow];
};

struct Sm100Fwd {
  FwdParams p;
  const void* desc_table;  // device array of CUtensorMap
  int32_t q_slot;          // descriptor slot of Q_i
  int32_t o_slot;          // descriptor slot of O_i (bf16, 128-row boxes; TMA store on LAST), -1 if none
  int32_t n;               // window size
  int32_t start[kMaxWindow];
  int32_t len[kMaxWindow];
  TmaSlots slots;
  // multi-chunk launch (nq > 0, sppo_attn_fwd_chunks): Q chunks q0..q0+nq-1 (window
  // index = chunk id, window = chunks 0..q0+nq-1, FIRST|LAST), blocks ordered longest
  // chunk first: block_base[k] = first block of chunk q0+nq-1-k
  int32_t nq, q0;
  int32_t block_base[kMaxWindow + 1];
  uint16_t qslots[kMaxWindow], oslots[kMaxWindow];  // by chunk - q0
  float* lses[kMaxWindow];
};

struct Sm100Bwd {
  BwdParams p;
  const void* desc_table;
  // bf16 Q_i / dO_i maps with 128-row and 64-row boxes; fp32 dQ-accumulator map
  // (TMA reduce-add of dQ partial sums)
  int32_t q_slot, do_slot, q64_slot, do64_slot, dq_slot;
  int32_t n;
  int32_t start[kMaxWindow];
  int32_t len[kMaxWindow];
  int32_t pair_base[kMaxWindow + 1];  // prefix count of 256-key CTA-pair tiles per window chunk
  TmaSlots slots;
  TmaSlots acc;  // fp32 dK (acc.k) / dV (acc.v) accumulator maps (TMA reduce-add of the item epilogue)
  int* sched;    // item counter of this launch (zeroed on the stream before it): dynamic item schedule
  float* dk[kMaxWindow];
  float* dv[kMaxWindow];
};

cudaError_t launch_fwd_sm100(const Sm100Fwd& a, cudaStream_t s);
cudaError_t launch_bwd_sm100(const Sm100Bwd& a, cudaStream_t s);

// ---- elementwise helpers (bwd pre/post-processing, memory-bound) ---------
// delta[h, r] = sum_d dO[r,h,d] * O[r,h,d]; optionally zero dq_acc.
cudaError_t launch_bwd_preprocess(const BwdParams& p, bool bf16, cudaStream_t s);
// dst(dtype) = src(fp32), n elements (n % 4 == 0 fast path).
cudaError_t launch_cast_f32(const float* src, void* dst, size_t n, bool bf16, cudaStream_t s);

// ---- per-chunk transformer layer (include/sppo_layer.h) ---------------------
// tcgen05 GEMM: the TMA tensor maps are built on the host (2-D, SWIZZLE_128B):
// K-major operand [rows][K]: box {64, 128 (A) | BN (B)};  MN-major operand
// [K][MN]: box {64, 64}.  Epilogue pointers are raw bf16 / fp32.
struct GemmParams {
  int32_t M, N, K;
  int32_t a_mn, b_mn;
  int32_t a_parts, a_part_w;  // A split along its contiguous dim: width of one part
  int32_t epi;                // SPPO_EPI_*
  const void* bias;           // bf16 [N] or null
  const void* residual;       // bf16 [M][N] or null
  const void* aux_in;         // bf16 [M][N] (DGELU)
  void* aux_out;              // bf16 [M][N] (GELU)
  int32_t c_parts, c_part_w;
  void* c[3];
};
// maps: a[0..a_parts-1], b.  bn = 128 | 256 (single CTA); pair: the cluster-of-2
// 256 x 256 kernel (b's K-major box then spans 128 rows).
cudaError_t launch_gemm_sm100(const void* tmap_a3, const void* tmap_b, const GemmParams& p, int bn, bool pair,
                              int num_sms, cudaStream_t s);
cudaError_t launch_layernorm_fwd(const void* x, const void* gamma, const void* beta, int64_t rows, int cols,
                                 float eps, void* y, float* mean, float* rstd, cudaStream_t s);
cudaError_t launch_layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean,
                                 const float* rstd, const void* dres, int64_t rows, int cols, void* dx,
                                 cudaStream_t s);
cudaError_t launch_col_reduce(int parts, const void* const* dy, const void* x, const float* mean, const float* rstd,
                              int64_t rows, int cols, float* sum_acc, float* prod_acc, int num_sms,
                              cudaStream_t s);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, current device).
cudaError_t ensure_smem_attr(const void* fn, int bytes);
// SM count of the current device.
int num_sms();

// error text for the ABI (thread-local; defined in sppo_api.cu)
int api_fail(int status, const char* fmt, ...);

}  // namespace sppo

