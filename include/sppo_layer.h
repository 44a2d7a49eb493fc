/*
 * sppo_layer.h — C ABI of the per-chunk GPT transformer layer around the
 * chunked attention of sppo.h ("QKV/out-proj/MLP tcgen05
 * GEMMs plus offload of the remaining Type-1 tensors with alpha").
 *
 * What is computed (PAPER.md = /root/reference/PAPER.md):
 *   P:356 [§5.1, Fig. "computation of s_N in a Transformer-based model and the
 *   skeletal tensors with its sizes"]: the forward of subsequence i runs the
 *   whole layer on the chunk's tokens; K_i/V_i are kept on the GPU (Type-0),
 *   the remaining activations (Type-1) are offloaded with ratio alpha_i and
 *   must be back "before the backward propagation of the subsequence begins".
 *   The layer is the Megatron GPT layer (P:472 [§7]; reading L16):
 *     a = LN1(x); [q k v] = a W_qkv^T + b_qkv; o = attention (sppo.h);
 *     y = x + o W_o^T + b_o; b = LN2(y); u = b W_1^T + b_1; g = GELU(u);
 *     z = y + g W_2^T + b_2            (GELU exact: u * Phi(u))
 *   Every op here except attention is token-wise, so the chunk loop of
 *   sppo.h's ordering contract (forward ascending, backward descending)
 *   applies unchanged.
 *
 * Conventions: matrices are row-major with an explicit "stored" orientation
 * (below); bf16 storage, fp32 accumulation (tensor cores: tcgen05.mma
 * kind::f16, accumulators in TMEM); LayerNorm statistics fp32 [rows];
 * weight / bias / LayerNorm-parameter gradients accumulate in caller-owned
 * fp32 buffers (+=).  All pointers are DEVICE pointers, 16-byte aligned
 * (SPPO_E_ALIGN); the caller owns every buffer.  Errors: validated on the
 * host before anything is enqueued; a non-OK status enqueues nothing;
 * sppo_last_error() has the text.  Calls enqueue on `stream` and return.
 */
#ifndef SPPO_LAYER_H_
#define SPPO_LAYER_H_

#include <stdint.h>

#include "sppo.h"

#ifdef __cplusplus
extern "C" {
#endif

/* epilogues of sppo_gemm (applied to the fp32 accumulator D[m][n]) */
enum {
  SPPO_EPI_STORE = 0,   /* C = bf16(D + bias[n] + residual[m][n])  (bias/residual optional)   */
  SPPO_EPI_GELU = 1,    /* u = D + bias[n]; aux_out = bf16(u); C = bf16(GELU(u))  (fp32 u)     */
  SPPO_EPI_DGELU = 2,   /* C = bf16(D * GELU'(aux_in[m][n]))  (backward through the GELU)       */
  SPPO_EPI_ACC_F32 = 3  /* C (fp32) += D   (weight gradients accumulated over chunks)           */
};

/*
 * One GEMM  D[M][N] = sum_k A(m,k) B(k,n)  on the tensor cores, plus epilogue.
 *   a_mn = 0: A stored [M][K] (K contiguous);  a_mn = 1: A stored [K][M].
 *   b_mn = 0: B stored [N][K] (nn.Linear weight [out][in]);  b_mn = 1: B stored [K][N].
 *   A may be split along its CONTIGUOUS dimension into a_parts (1..3) equal
 *   buffers a[0..a_parts-1] (e.g. dQ|dK|dV as three [s, H] buffers = one
 *   [s, 3H] operand); C likewise into c_parts buffers along N (Q|K|V outputs).
 *   Forward y = x W^T: a_mn = 0, b_mn = 0.  Data gradient dx = dy W: a_mn = 0,
 *   b_mn = 1.  Weight gradient dW += dy^T x: a_mn = 1, b_mn = 1, SPPO_EPI_ACC_F32.
 * Shapes: N % 128 == 0, K % 8 == 0 when K is a contiguous dim (a_mn = 0 or
 * b_mn = 0), M >= 1 (row tail masked, K tail zero-
 * filled by TMA); a part's width (contiguous elements) % 64 == 0 for a_mn = 0
 * and % 128 == 0 for a_mn = 1; C part width % 128 == 0 (else SPPO_E_SHAPE).
 * bias bf16 [N]; residual, aux_in, aux_out bf16 [M][N] (single buffers).
 */
typedef struct {
  int64_t M, N, K;
  int32_t a_mn, b_mn;
  int32_t a_parts;
  const void* a[3];
  const void* b;
  int32_t epilogue;
  const void* bias;
  const void* residual;
  const void* aux_in;
  void* aux_out;
  int32_t c_parts;
  void* c[3];
} sppo_gemm_args;

sppo_status sppo_gemm(sppo_ctx ctx, const sppo_gemm_args* g, void* stream);

/*
 * LayerNorm forward over the last dimension (P:356 Fig. skeletal tensors; L16):
 *   mean_r = avg_c x[r][c], rstd_r = 1/sqrt(var_r + eps),
 *   y[r][c] = (x[r][c] - mean_r) rstd_r gamma[c] + beta[c].
 *   x, y bf16 [rows][cols]; gamma, beta bf16 [cols]; mean, rstd fp32 [rows].
 *   cols % 256 == 0, cols <= 16384.
 */
sppo_status sppo_layernorm_fwd(sppo_ctx ctx, const void* x, const void* gamma, const void* beta, int64_t rows,
                               int32_t cols, float eps, void* y, float* mean, float* rstd, void* stream);

/*
 * LayerNorm backward, data part:  xhat = (x - mean) rstd,  g = dy gamma,
 *   dx[r][c] = dres[r][c] + rstd_r (g - avg_c g - xhat avg_c(g xhat))
 *   (dres = the residual-stream gradient added in, optional, bf16 [rows][cols]).
 *   dx bf16 [rows][cols].  Parameter gradients: sppo_col_reduce with x/mean/rstd.
 */
sppo_status sppo_layernorm_bwd(sppo_ctx ctx, const void* dy, const void* x, const void* gamma, const float* mean,
                               const float* rstd, const void* dres, int64_t rows, int32_t cols, void* dx,
                               void* stream);

/*
 * Column reductions over rows (bias and LayerNorm-parameter gradients):
 *   sum_acc[c]  += sum_r dy[r][c]                               (always)
 *   prod_acc[c] += sum_r dy[r][c] (x[r][c] - mean_r) rstd_r      (if x != NULL)
 *   dy is split along columns into `parts` equal bf16 buffers dy[0..parts-1]
 *   (total width cols); x bf16 [rows][cols]; sum_acc, prod_acc fp32 [cols].
 *   cols / parts % 8 == 0.  Accumulation order across rows is not fixed
 *   (fp32 atomics): results are reproducible to fp32 rounding only.
 */
sppo_status sppo_col_reduce(sppo_ctx ctx, int32_t parts, const void* const* dy, const void* x, const float* mean,
                            const float* rstd, int64_t rows, int32_t cols, float* sum_acc, float* prod_acc,
                            void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPPO_LAYER_H_ */
