// C-ABI entry points of the per-chunk transformer layer (include/sppo_layer.h):
// argument validation, 2-D TMA tensor maps for the GEMM operands (passed to
// the kernel by value as __grid_constant__ parameters), dispatch.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "../../include/sppo_layer.h"
#include "internal.h"

using namespace sppo;

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

#define err(status, ...) ((sppo_status)api_fail((status), __VA_ARGS__))

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// bf16 row-major matrix [rows][cols] (cols contiguous), box {64 cols, box_rows}, SWIZZLE_128B
sppo_status encode2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  EncodeTiledFn enc = encoder();
  if (!enc) return err(SPPO_E_CUDA, "%s", "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return err(SPPO_E_CUDA, "cuTensorMapEncodeTiled failed (%lld)", (long long)r);
  return SPPO_OK;
}

}  // namespace

extern "C" {

sppo_status sppo_gemm(sppo_ctx ctx, const sppo_gemm_args* g, void* stream) {
  if (!ctx || !g) return err(SPPO_E_ARG, "ctx or args is NULL");
  if (g->M < 1 || g->N < 1 || g->K < 1) return err(SPPO_E_SHAPE, "gemm: M, N, K must be >= 1");
  if (g->M > INT32_MAX || g->N > INT32_MAX || g->K > INT32_MAX) return err(SPPO_E_SHAPE, "gemm: dims exceed 2^31");
  if (g->N % 128) return err(SPPO_E_SHAPE, "gemm: N = %lld not a multiple of 128", (long long)g->N);
  if ((!g->a_mn || !g->b_mn) && g->K % 8) return err(SPPO_E_SHAPE, "gemm: K = %lld not a multiple of 8", (long long)g->K);
  if ((g->a_mn != 0 && g->a_mn != 1) || (g->b_mn != 0 && g->b_mn != 1)) return err(SPPO_E_ARG, "gemm: a_mn/b_mn must be 0|1");
  if (g->a_parts < 1 || g->a_parts > 3 || g->c_parts < 1 || g->c_parts > 3)
    return err(SPPO_E_ARG, "gemm: a_parts / c_parts must be in 1..3");
  if (g->epilogue < SPPO_EPI_STORE || g->epilogue > SPPO_EPI_ACC_F32) return err(SPPO_E_ARG, "gemm: bad epilogue");
  if (!g->b) return err(SPPO_E_ARG, "gemm: b is NULL");
  if (!al16(g->b)) return err(SPPO_E_ALIGN, "gemm: b not 16-byte aligned");
  for (int i = 0; i < g->a_parts; ++i) {
    if (!g->a[i]) return err(SPPO_E_ARG, "gemm: a[%d] is NULL", i);
    if (!al16(g->a[i])) return err(SPPO_E_ALIGN, "gemm: a[%d] not 16-byte aligned", i);
  }
  for (int i = 0; i < g->c_parts; ++i) {
    if (!g->c[i]) return err(SPPO_E_ARG, "gemm: c[%d] is NULL", i);
    if (!al16(g->c[i])) return err(SPPO_E_ALIGN, "gemm: c[%d] not 16-byte aligned", i);
  }
  const int64_t a_cont = g->a_mn ? g->M : g->K;  // contiguous extent of A's storage
  if (a_cont % g->a_parts) return err(SPPO_E_SHAPE, "gemm: A's contiguous dim not divisible by a_parts");
  const int64_t apw = a_cont / g->a_parts;
  if (g->a_parts > 1 && apw % (g->a_mn ? 128 : 64))
    return err(SPPO_E_SHAPE, "gemm: A part width %lld must be a multiple of %d", (long long)apw, g->a_mn ? 128 : 64);
  if (g->a_mn && g->M % 64) return err(SPPO_E_SHAPE, "gemm: M-major A needs M %% 64 == 0");
  if (g->N % g->c_parts || (g->N / g->c_parts) % 128)
    return err(SPPO_E_SHAPE, "gemm: C part width must be a multiple of 128");
  if (g->epilogue == SPPO_EPI_GELU && !g->aux_out) return err(SPPO_E_ARG, "gemm: GELU needs aux_out");
  if (g->epilogue == SPPO_EPI_DGELU && !g->aux_in) return err(SPPO_E_ARG, "gemm: DGELU needs aux_in");
  if (g->epilogue == SPPO_EPI_ACC_F32 && (g->bias || g->residual))
    return err(SPPO_E_ARG, "gemm: ACC_F32 takes no bias/residual");
  for (const void* q : {g->bias, g->residual, g->aux_in, (const void*)g->aux_out})
    if (q && !al16(q)) return err(SPPO_E_ALIGN, "gemm: epilogue operand not 16-byte aligned");

  const int64_t cpw = g->N / g->c_parts;
  int bn = (cpw % 256 == 0) ? 256 : 128;
  // CTA pair (cluster of 2, 256 x 256 tiles, 128-deep K stages) whenever N tiles
  // are 256 wide and M spans more than one 128-row tile, every operand
  // orientation (measured at the GPT-7B chunk shapes, tools/gemm_bench.py, vs the
  // single-CTA kernel: x W^T 1444-1519 vs 1330-1373 TF/s, dy W 1471-1473 vs
  // 1162-1266, dy^T x 1180-1218 vs 1049-1152).  SPPO_GEMM_PAIR=0 selects the
  // single-CTA kernel, =1 the pair only for K-major x K-major.
  static const int pair_env = [] {
    const char* e = getenv("SPPO_GEMM_PAIR");
    return e ? atoi(e) : 2;
  }();
  const bool pair = bn == 256 && g->M > 128 && (pair_env == 2 || (pair_env == 1 && !g->a_mn && !g->b_mn));
  CUtensorMap ta[3], tb;
  memset(ta, 0, sizeof ta);
  for (int i = 0; i < g->a_parts; ++i) {
    sppo_status s = g->a_mn ? encode2d(&ta[i], g->a[i], g->K, apw, 64) : encode2d(&ta[i], g->a[i], g->M, apw, 128);
    if (s != SPPO_OK) return s;
  }
  for (int i = g->a_parts; i < 3; ++i) ta[i] = ta[0];
  {
    sppo_status s = g->b_mn ? encode2d(&tb, g->b, g->K, g->N, 64) : encode2d(&tb, g->b, g->N, g->K, pair ? 128 : bn);
    if (s != SPPO_OK) return s;
  }
  GemmParams p{};
  p.M = (int32_t)g->M;
  p.N = (int32_t)g->N;
  p.K = (int32_t)g->K;
  p.a_mn = g->a_mn;
  p.b_mn = g->b_mn;
  p.a_parts = g->a_parts;
  p.a_part_w = (int32_t)apw;
  p.epi = g->epilogue;
  p.bias = g->bias;
  p.residual = g->residual;
  p.aux_in = g->aux_in;
  p.aux_out = g->aux_out;
  p.c_parts = g->c_parts;
  p.c_part_w = (int32_t)cpw;
  for (int i = 0; i < 3; ++i) p.c[i] = i < g->c_parts ? g->c[i] : g->c[0];
  cudaError_t e = launch_gemm_sm100(ta, &tb, p, bn, pair, sm_count(), (cudaStream_t)stream);
  if (e != cudaSuccess) return err(SPPO_E_CUDA, "gemm launch: %s", cudaGetErrorString(e));
  return SPPO_OK;
}

sppo_status sppo_layernorm_fwd(sppo_ctx ctx, const void* x, const void* gamma, const void* beta, int64_t rows,
                               int32_t cols, float eps, void* y, float* mean, float* rstd, void* stream) {
  if (!ctx || !x || !gamma || !beta || !y || !mean || !rstd) return err(SPPO_E_ARG, "layernorm_fwd: NULL argument");
  if (rows < 0 || cols < 256 || cols % 256 || cols > 16384)
    return err(SPPO_E_SHAPE, "layernorm_fwd: cols %d must be a multiple of 256 in [256, 16384]", cols);
  if (!(eps > 0.f)) return err(SPPO_E_ARG, "layernorm_fwd: eps must be > 0");
  for (const void* q : {x, gamma, beta, (const void*)y})
    if (!al16(q)) return err(SPPO_E_ALIGN, "layernorm_fwd: pointer not 16-byte aligned");
  cudaError_t e = launch_layernorm_fwd(x, gamma, beta, rows, cols, eps, y, mean, rstd, (cudaStream_t)stream);
  if (e != cudaSuccess) return err(SPPO_E_CUDA, "layernorm_fwd launch: %s", cudaGetErrorString(e));
  return SPPO_OK;
}

sppo_status sppo_layernorm_bwd(sppo_ctx ctx, const void* dy, const void* x, const void* gamma, const float* mean,
                               const float* rstd, const void* dres, int64_t rows, int32_t cols, void* dx,
                               void* stream) {
  if (!ctx || !dy || !x || !gamma || !mean || !rstd || !dx) return err(SPPO_E_ARG, "layernorm_bwd: NULL argument");
  if (rows < 0 || cols < 256 || cols % 256 || cols > 16384)
    return err(SPPO_E_SHAPE, "layernorm_bwd: cols %d must be a multiple of 256 in [256, 16384]", cols);
  for (const void* q : {dy, x, gamma, dres, (const void*)dx})
    if (q && !al16(q)) return err(SPPO_E_ALIGN, "layernorm_bwd: pointer not 16-byte aligned");
  cudaError_t e = launch_layernorm_bwd(dy, x, gamma, mean, rstd, dres, rows, cols, dx, (cudaStream_t)stream);
  if (e != cudaSuccess) return err(SPPO_E_CUDA, "layernorm_bwd launch: %s", cudaGetErrorString(e));
  return SPPO_OK;
}

sppo_status sppo_col_reduce(sppo_ctx ctx, int32_t parts, const void* const* dy, const void* x, const float* mean,
                            const float* rstd, int64_t rows, int32_t cols, float* sum_acc, float* prod_acc,
                            void* stream) {
  if (!ctx || !dy || !sum_acc) return err(SPPO_E_ARG, "col_reduce: NULL argument");
  if (parts < 1 || parts > 3) return err(SPPO_E_ARG, "col_reduce: parts must be in 1..3");
  if (rows < 0 || cols < 8 || cols % parts || (cols / parts) % 8)
    return err(SPPO_E_SHAPE, "col_reduce: cols / parts must be a multiple of 8 (cols = %d)", cols);
  if (x && (!mean || !rstd || !prod_acc)) return err(SPPO_E_ARG, "col_reduce: x needs mean, rstd, prod_acc");
  for (int i = 0; i < parts; ++i)
    if (!dy[i] || !al16(dy[i])) return err(SPPO_E_ALIGN, "col_reduce: dy part NULL or not 16-byte aligned");
  if (x && !al16(x)) return err(SPPO_E_ALIGN, "col_reduce: x not 16-byte aligned");
  cudaError_t e =
      launch_col_reduce(parts, dy, x, mean, rstd, rows, cols, sum_acc, prod_acc, sm_count(), (cudaStream_t)stream);
  if (e != cudaSuccess) return err(SPPO_E_CUDA, "col_reduce launch: %s", cudaGetErrorString(e));
  return SPPO_OK;
}

}  // extern "C"
