// Memory-bound kernels of the per-chunk transformer layer (include/sppo_layer.h):
// LayerNorm forward / backward (one warp per row, 16-B coalesced accesses, fp32
// statistics) and column reductions for bias and LayerNorm-parameter gradients
// (a warp covers 256 consecutive columns of a row, 8 warps per CTA stride the
// rows of one row split, CTA partials combined in shared memory then one fp32
// atomic per column).  Each kernel reads its inputs once from HBM (the row
// re-reads of the LayerNorm passes hit L1).
#include <cuda_bf16.h>

#include "internal.h"

namespace sppo {
namespace {

constexpr int kRowsPerCta = 8;  // warps per CTA, one row each

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 w = *reinterpret_cast<const uint4*>(p);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ws[e]));
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
}

__device__ __forceinline__ void st8(__nv_bfloat16* p, const float (&v)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
    w[e] = *reinterpret_cast<uint32_t*>(&b);
  }
  *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__global__ void __launch_bounds__(32 * kRowsPerCta) layernorm_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                                        const __nv_bfloat16* __restrict__ gamma,
                                                                        const __nv_bfloat16* __restrict__ beta,
                                                                        int64_t rows, int cols, float eps,
                                                                        __nv_bfloat16* __restrict__ y,
                                                                        float* __restrict__ mean,
                                                                        float* __restrict__ rstd) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kRowsPerCta + (threadIdx.x >> 5);
  if (r >= rows) return;
  const __nv_bfloat16* xr = x + r * cols;
  float s = 0.f;
  for (int c = lane * 8; c < cols; c += 256) {
    float v[8];
    ld8(xr + c, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) s += v[e];
  }
  const float mu = warp_sum(s) / cols;
  float q = 0.f;
  for (int c = lane * 8; c < cols; c += 256) {
    float v[8];
    ld8(xr + c, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) q += (v[e] - mu) * (v[e] - mu);
  }
  const float rs = rsqrtf(warp_sum(q) / cols + eps);
  for (int c = lane * 8; c < cols; c += 256) {
    float v[8], g[8], b[8];
    ld8(xr + c, v);
    ld8(gamma + c, g);
    ld8(beta + c, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = (v[e] - mu) * rs * g[e] + b[e];
    st8(y + r * cols + c, v);
  }
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

__global__ void __launch_bounds__(32 * kRowsPerCta) layernorm_bwd_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const __nv_bfloat16* __restrict__ gamma, const float* __restrict__ mean, const float* __restrict__ rstd,
    const __nv_bfloat16* __restrict__ dres, int64_t rows, int cols, __nv_bfloat16* __restrict__ dx) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kRowsPerCta + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float mu = mean[r], rs = rstd[r];
  const __nv_bfloat16* dyr = dy + r * cols;
  const __nv_bfloat16* xr = x + r * cols;
  float sg = 0.f, sgx = 0.f;
  for (int c = lane * 8; c < cols; c += 256) {
    float d[8], v[8], g[8];
    ld8(dyr + c, d);
    ld8(xr + c, v);
    ld8(gamma + c, g);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float gg = d[e] * g[e];
      sg += gg;
      sgx += gg * (v[e] - mu) * rs;
    }
  }
  const float mg = warp_sum(sg) / cols, mgx = warp_sum(sgx) / cols;
  for (int c = lane * 8; c < cols; c += 256) {
    float d[8], v[8], g[8], o[8];
    ld8(dyr + c, d);
    ld8(xr + c, v);
    ld8(gamma + c, g);
    if (dres) {
      ld8(dres + r * cols + c, o);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] += rs * (d[e] * g[e] - mg - (v[e] - mu) * rs * mgx);
    st8(dx + r * cols + c, o);
  }
}

struct ColParts {
  const __nv_bfloat16* p[3];
};

// grid (ceil(cols / 256), splits): CTA (cb, s) reduces columns [256 cb, 256 cb + 256)
// (clipped to cols) over rows [s * rows_per, (s + 1) * rows_per); a lane owns 8
// consecutive columns, which lie in one part (part widths are multiples of 8).
__global__ void __launch_bounds__(256) col_reduce_kernel(ColParts dy, int part_w, const __nv_bfloat16* __restrict__ x,
                                                         const float* __restrict__ mean,
                                                         const float* __restrict__ rstd, int64_t rows, int cols,
                                                         int64_t rows_per, float* __restrict__ sum_acc,
                                                         float* __restrict__ prod_acc) {
  __shared__ float red[2][kRowsPerCta][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c0 = blockIdx.x * 256;
  const int col = c0 + lane * 8;          // this lane's 8 columns (parts are multiples of 8 wide)
  const bool live = col < cols;
  const int part = live ? col / part_w : 0;
  const int pc = col - part * part_w;
  const __nv_bfloat16* src = dy.p[part];
  const int64_t r0 = (int64_t)blockIdx.y * rows_per;
  const int64_t r1 = r0 + rows_per < rows ? r0 + rows_per : rows;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float q[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int64_t r = r0 + w; live && r < r1; r += kRowsPerCta) {
    float d[8];
    ld8(src + r * part_w + pc, d);
#pragma unroll
    for (int e = 0; e < 8; ++e) s[e] += d[e];
    if (x) {
      float v[8];
      ld8(x + r * cols + col, v);
      const float mu = mean[r], rs = rstd[r];
#pragma unroll
      for (int e = 0; e < 8; ++e) q[e] += d[e] * (v[e] - mu) * rs;
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red[0][w][lane * 8 + e] = s[e];
    red[1][w][lane * 8 + e] = q[e];
  }
  __syncthreads();
  const int c = threadIdx.x;
  float ts = 0.f, tq = 0.f;
#pragma unroll
  for (int k = 0; k < kRowsPerCta; ++k) {
    ts += red[0][k][c];
    tq += red[1][k][c];
  }
  if (c0 + c < cols) {
    atomicAdd(sum_acc + c0 + c, ts);
    if (x) atomicAdd(prod_acc + c0 + c, tq);
  }
}

}  // namespace

cudaError_t launch_layernorm_fwd(const void* x, const void* gamma, const void* beta, int64_t rows, int cols,
                                 float eps, void* y, float* mean, float* rstd, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((rows + kRowsPerCta - 1) / kRowsPerCta);
  layernorm_fwd_kernel<<<grid, 32 * kRowsPerCta, 0, s>>>(
      static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(gamma),
      static_cast<const __nv_bfloat16*>(beta), rows, cols, eps, static_cast<__nv_bfloat16*>(y), mean, rstd);
  return cudaGetLastError();
}

cudaError_t launch_layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean,
                                 const float* rstd, const void* dres, int64_t rows, int cols, void* dx,
                                 cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((rows + kRowsPerCta - 1) / kRowsPerCta);
  layernorm_bwd_kernel<<<grid, 32 * kRowsPerCta, 0, s>>>(
      static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x),
      static_cast<const __nv_bfloat16*>(gamma), mean, rstd, static_cast<const __nv_bfloat16*>(dres), rows, cols,
      static_cast<__nv_bfloat16*>(dx));
  return cudaGetLastError();
}

cudaError_t launch_col_reduce(int parts, const void* const* dy, const void* x, const float* mean, const float* rstd,
                              int64_t rows, int cols, float* sum_acc, float* prod_acc, int num_sms,
                              cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  ColParts cp{};
  for (int i = 0; i < parts; ++i) cp.p[i] = static_cast<const __nv_bfloat16*>(dy[i]);
  const int cblocks = (cols + 255) / 256;
  int64_t splits = (4LL * num_sms + cblocks - 1) / cblocks;
  const int64_t max_splits = (rows + 4 * kRowsPerCta - 1) / (4 * kRowsPerCta);  // >= 4 rows per warp
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  const int64_t rows_per = (rows + splits - 1) / splits;
  splits = (rows + rows_per - 1) / rows_per;
  col_reduce_kernel<<<dim3(cblocks, (unsigned)splits), 256, 0, s>>>(
      cp, cols / parts, static_cast<const __nv_bfloat16*>(x), mean, rstd, rows, cols, rows_per, sum_acc, prod_acc);
  return cudaGetLastError();
}

}  // namespace sppo
