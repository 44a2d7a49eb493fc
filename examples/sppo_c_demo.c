/*
 * sppo_c_demo.c — one SPPO training step of attention driven from plain C
 * through the C ABI (include/sppo.h), no Python and no torch:
 *
 *   1. FLOPs-balanced partition of S tokens into N chunks (sppo_partition_balanced)
 *   2. forward of chunk i = 0..N-1 over the K/V of chunks 0..i (sppo_attn_fwd),
 *      O_i offloaded to pinned host memory right after fwd(i) (sppo_kv_offload)
 *   3. backward of chunk i = N-1..0 (sppo_attn_bwd) after O_i was prefetched
 *      back from the host (sppo_kv_prefetch) into a device buffer that was
 *      overwritten with garbage in between
 *
 * It prints properties that hold for causal softmax attention independently of
 * any reference implementation (they are not the parity tests — those live in
 * tests/ and compare with oracle/):
 *   - O row 0 == V row 0 (row 0 attends only to itself),
 *   - dQ row 0 == 0      (dS = P (dP - Delta) = 1 * (dO.v0 - dO.O0) = 0),
 *   - sum_t dV_t == sum_p dO_p per head and column (every softmax row sums to 1).
 *
 * Build (after `python -m paper_2503_10377_b200.build`):
 *   gcc -O2 -std=c11 examples/sppo_c_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2503_10377_b200 -lsppo -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2503_10377_b200:/usr/local/cuda/lib64 -lm -o examples/sppo_c_demo
 * Run on a B200:  examples/sppo_c_demo [S] [N] [heads]     (exit 0 = all checks pass)
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "sppo.h"

#define D 128

#define CK(x)                                                                      \
  do {                                                                             \
    sppo_status s_ = (x);                                                          \
    if (s_ != SPPO_OK) {                                                           \
      fprintf(stderr, "%s:%d %s -> %d: %s\n", __FILE__, __LINE__, #x, (int)s_,     \
              sppo_last_error());                                                  \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)
#define CU(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

static uint16_t to_bf16(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint64_t rng = 0x9E3779B97F4A7C15ull;
static float uniform(void) { /* splitmix64 -> [-1, 1) */
  uint64_t z = (rng += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (float)((double)(z >> 11) / 9007199254740992.0 * 2.0 - 1.0);
}

int main(int argc, char** argv) {
  const int64_t S = argc > 1 ? atoll(argv[1]) : 5000;
  const int32_t N = argc > 2 ? atoi(argv[2]) : 4;
  const int32_t H = argc > 3 ? atoi(argv[3]) : 2;
  const size_t row = (size_t)H * D;          /* elements per token */
  const size_t nel = (size_t)S * row;

  sppo_ctx ctx;
  CK(sppo_ctx_create(0, &ctx));
  printf("libsppo version %d, S=%lld N=%d heads=%d d=%d bf16\n", sppo_version(), (long long)S, N, H, D);

  int64_t* off = malloc(sizeof(int64_t) * (N + 1));
  CK(sppo_partition_balanced(S, N, off));
  int64_t smax = 0;
  for (int i = 0; i < N; ++i) {
    int64_t s = off[i + 1] - off[i];
    if (s > smax) smax = s;
    printf("  chunk %d: [%lld, %lld)\n", i, (long long)off[i], (long long)off[i + 1]);
  }
  sppo_layout L = {H, D, SPPO_BF16, N, off, 0.0f};

  /* host inputs: Q, K, V, dO ~ U[-1,1) (bf16) */
  uint16_t* h_in[4];
  for (int t = 0; t < 4; ++t) {
    h_in[t] = malloc(nel * 2);
    for (size_t e = 0; e < nel; ++e) h_in[t][e] = to_bf16(uniform() * (t == 3 ? 0.1f : 1.0f));
  }
  /* device tensors, all token-major [S, H, D] */
  void *q, *k, *v, *dout, *o, *dq, *dk, *dv;
  float *lse, *delta, *dq_acc, *dk_acc, *dv_acc;
  void** dev_in[4] = {&q, &k, &v, &dout};
  for (int t = 0; t < 4; ++t) {
    CU(cudaMalloc(dev_in[t], nel * 2));
    CU(cudaMemcpy(*dev_in[t], h_in[t], nel * 2, cudaMemcpyHostToDevice));
  }
  CU(cudaMalloc(&o, nel * 2));
  CU(cudaMalloc(&dq, nel * 2));
  CU(cudaMalloc(&dk, nel * 2));
  CU(cudaMalloc(&dv, nel * 2));
  CU(cudaMalloc((void**)&lse, (size_t)S * H * 4));       /* chunk i: [H, s_i] at H*c_i */
  CU(cudaMalloc((void**)&delta, (size_t)smax * H * 4));
  CU(cudaMalloc((void**)&dq_acc, (size_t)smax * row * 4));
  CU(cudaMalloc((void**)&dk_acc, nel * 4));
  CU(cudaMalloc((void**)&dv_acc, nel * 4));
  void* h_o;
  CK(sppo_host_alloc(ctx, nel * 2, &h_o));

  cudaStream_t st;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t* o_home = malloc(sizeof(cudaEvent_t) * N);
  for (int i = 0; i < N; ++i) CU(cudaEventCreateWithFlags(&o_home[i], cudaEventDisableTiming));

  int32_t* ids = malloc(sizeof(int32_t) * N);
  const void** kp = malloc(sizeof(void*) * N);
  const void** vp = malloc(sizeof(void*) * N);
  float** dkp = malloc(sizeof(float*) * N);
  float** dvp = malloc(sizeof(float*) * N);
  for (int j = 0; j < N; ++j) {
    ids[j] = j;
    kp[j] = (const uint16_t*)k + off[j] * row;
    vp[j] = (const uint16_t*)v + off[j] * row;
    dkp[j] = dk_acc + off[j] * row;
    dvp[j] = dv_acc + off[j] * row;
  }

  /* ---- forward: chunk i attends to chunks 0..i (one window), O_i -> host */
  for (int i = 0; i < N; ++i) {
    sppo_kv_set kv = {i + 1, ids, kp, vp};
    uint16_t* oi = (uint16_t*)o + off[i] * row;
    CK(sppo_attn_fwd(ctx, &L, i, (const uint16_t*)q + off[i] * row, &kv, SPPO_FIRST | SPPO_LAST, NULL, oi,
                     lse + off[i] * H, st));
    size_t nb = (size_t)(off[i + 1] - off[i]) * row * 2;
    CK(sppo_kv_offload(ctx, i, oi, (uint8_t*)h_o + off[i] * row * 2, nb, 1.0, st, o_home[i], NULL));
  }
  /* the device O may now be reused: overwrite it (0xFF bytes = bf16 NaN) once every copy landed */
  for (int i = 0; i < N; ++i) CU(cudaStreamWaitEvent(st, o_home[i], 0));
  CU(cudaMemsetAsync(o, 0xFF, nel * 2, st));

  /* ---- backward: chunk i = N-1..0, O_i prefetched back first */
  CU(cudaMemsetAsync(dk_acc, 0, nel * 4, st));
  CU(cudaMemsetAsync(dv_acc, 0, nel * 4, st));
  for (int i = N - 1; i >= 0; --i) {
    size_t nb = (size_t)(off[i + 1] - off[i]) * row * 2;
    uint16_t* oi = (uint16_t*)o + off[i] * row;
    CK(sppo_kv_prefetch(ctx, i, (const uint8_t*)h_o + off[i] * row * 2, oi, nb, st, NULL, 0));
    sppo_kv_set kv = {i + 1, ids, kp, vp};
    sppo_bwd_args a = {oi, lse + off[i] * H, (const uint16_t*)dout + off[i] * row, delta, dq_acc, dkp, dvp,
                       (uint16_t*)dq + off[i] * row, (uint16_t*)dk + off[i] * row, (uint16_t*)dv + off[i] * row};
    CK(sppo_attn_bwd(ctx, &L, i, (const uint16_t*)q + off[i] * row, &kv, &a, SPPO_FIRST | SPPO_LAST, st));
  }
  CU(cudaStreamSynchronize(st));
  CK(sppo_ctx_sync(ctx));

  /* ---- properties */
  uint16_t* h_o2 = malloc(nel * 2);
  uint16_t* h_dq = malloc(nel * 2);
  uint16_t* h_dv = malloc(nel * 2);
  CU(cudaMemcpy(h_o2, o, nel * 2, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(h_dq, dq, nel * 2, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(h_dv, dv, nel * 2, cudaMemcpyDeviceToHost));
  double e_o0 = 0, e_dq0 = 0, e_sum = 0, e_rt = 0;
  for (size_t c = 0; c < row; ++c) {
    e_o0 = fmax(e_o0, fabs(from_bf16(h_o2[c]) - from_bf16(h_in[2][c])));
    e_dq0 = fmax(e_dq0, fabs(from_bf16(h_dq[c])));
    double sdv = 0, sdo = 0;
    for (int64_t p = 0; p < S; ++p) {
      sdv += from_bf16(h_dv[p * row + c]);
      sdo += from_bf16(h_in[3][p * row + c]);
    }
    e_sum = fmax(e_sum, fabs(sdv - sdo) / (1.0 + fabs(sdo)));
  }
  e_rt = memcmp(h_o2, h_o, nel * 2) == 0 ? 0.0 : 1.0;
  const int ok = e_o0 <= 1e-2 && e_dq0 <= 1e-3 && e_sum <= 2e-2 && e_rt == 0.0;
  printf("max |O_0 - V_0|            = %.3g\n", e_o0);
  printf("max |dQ_0|                 = %.3g\n", e_dq0);
  printf("max rel |sum dV - sum dO|  = %.3g\n", e_sum);
  printf("O host round trip bitwise  = %s\n", e_rt == 0.0 ? "yes" : "NO");
  printf("%s\n", ok ? "PASS" : "FAIL");

  CK(sppo_host_free(ctx, h_o));
  CK(sppo_ctx_destroy(ctx));
  return ok ? 0 : 1;
}
