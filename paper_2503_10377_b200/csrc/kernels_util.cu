// Memory-bound helpers of the backward:
//   Delta_p = <dO_p, O_p> (FlashAttention convention; O is the STORED forward
//   output in its storage dtype, reading L6), zeroing of the fp32 dQ
//   accumulator, and fp32 -> dtype casts of finished gradients.
// Coalesced 16-byte vector accesses; grid sized in multiples of the SM count.
#include <cuda_bf16.h>

#include <mutex>
#include <set>
#include <utility>

#include "internal.h"

namespace sppo {
namespace {

// One warp per (row, head): d elements of O and dO, d/32 per lane.
template <typename T, int D>
__global__ void __launch_bounds__(256) preprocess_kernel(const BwdParams p, int zero_dq) {
  const int warps_per_block = blockDim.x >> 5;
  const long long gw = (long long)blockIdx.x * warps_per_block + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const long long total = (long long)p.q_len * p.heads;
  if (gw >= total) return;
  const int r = (int)(gw / p.heads), h = (int)(gw % p.heads);
  const size_t base = ((size_t)r * p.heads + h) * D;
  const T* o = (const T*)p.o + base;
  const T* dout = (const T*)p.dout + base;
  float acc = 0.f;
#pragma unroll
  for (int c = lane; c < D; c += 32) acc = fmaf((float)o[c], (float)dout[c], acc);
#pragma unroll
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) p.delta[(size_t)h * p.q_len + r] = acc;
  if (zero_dq) {
    float* dq = p.dq_acc + base;
#pragma unroll
    for (int c = lane; c < D; c += 32) dq[c] = 0.f;
  }
}

// bf16 fast path for D = 128: each lane reads 4 consecutive bf16 of O and dO.
__global__ void __launch_bounds__(256) preprocess_bf16_d128_kernel(const BwdParams p, int zero_dq) {
  const long long gw = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const long long total = (long long)p.q_len * p.heads;
  if (gw >= total) return;
  const int r = (int)(gw / p.heads), h = (int)(gw % p.heads);
  const size_t base = ((size_t)r * p.heads + h) * 128;
  const uint2 ov = *reinterpret_cast<const uint2*>((const __nv_bfloat16*)p.o + base + lane * 4);
  const uint2 dv = *reinterpret_cast<const uint2*>((const __nv_bfloat16*)p.dout + base + lane * 4);
  const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
  const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float2 a = __bfloat1622float2(o2[k]);
    const float2 b = __bfloat1622float2(d2[k]);
    acc = fmaf(a.x, b.x, acc);
    acc = fmaf(a.y, b.y, acc);
  }
#pragma unroll
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) p.delta[(size_t)h * p.q_len + r] = acc;
  if (zero_dq) *reinterpret_cast<float4*>(p.dq_acc + base + lane * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void cast_f32_bf16_kernel(const float4* __restrict__ src, uint2* __restrict__ dst, size_t n4) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y);
    __nv_bfloat162 b = __floats2bfloat162_rn(v.z, v.w);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&a);
    o.y = *reinterpret_cast<uint32_t*>(&b);
    dst[i] = o;
  }
}

__global__ void cast_f32_f32_kernel(const float4* __restrict__ src, float4* __restrict__ dst, size_t n4) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace

// Attributes are per device: remember (kernel, device) pairs, not a process-wide flag.
cudaError_t ensure_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({fn, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({fn, dev});
  return e;
}

int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

cudaError_t launch_bwd_preprocess(const BwdParams& p, bool bf16, cudaStream_t s) {
  const long long warps = (long long)p.q_len * p.heads;
  const unsigned blocks = (unsigned)((warps + 7) / 8);
  const int zero = p.first ? 1 : 0;
  if (bf16 && p.d == 128)
    preprocess_bf16_d128_kernel<<<blocks, 256, 0, s>>>(p, zero);
  else if (!bf16 && p.d == 128)
    preprocess_kernel<float, 128><<<blocks, 256, 0, s>>>(p, zero);
  else if (!bf16 && p.d == 64)
    preprocess_kernel<float, 64><<<blocks, 256, 0, s>>>(p, zero);
  else if (!bf16 && p.d == 32)
    preprocess_kernel<float, 32><<<blocks, 256, 0, s>>>(p, zero);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_cast_f32(const float* src, void* dst, size_t n, bool bf16, cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  const size_t n4 = n / 4;
  size_t nb = (n4 + 255) / 256;
  if (nb > (size_t)num_sms() * 16) nb = (size_t)num_sms() * 16;
  const unsigned blocks = (unsigned)nb;
  if (!blocks) return cudaSuccess;
  if (bf16)
    cast_f32_bf16_kernel<<<blocks, 256, 0, s>>>((const float4*)src, (uint2*)dst, n4);
  else
    cast_f32_f32_kernel<<<blocks, 256, 0, s>>>((const float4*)src, (float4*)dst, n4);
  return cudaGetLastError();
}

}  // namespace sppo
