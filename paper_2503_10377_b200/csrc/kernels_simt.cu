// FP32 SIMT path of chunked causal attention: exact FP32 FMA,
// no tensor cores (TF32 would miss the 1e-4 tolerance of the fp32 path, reading
// L6).  It serves configs[0] (h=1, d=64, S=1024).  The bf16 production path is
// the sm_100a tensor-core kernels in kernels_sm100_*.cu.
//
// Method (P:356 [§5.1]): chunk i's queries attend causally to K_j, V_j, j <= i,
// with online softmax carried across the window's key tiles (FlashAttention,
// P:134) and across windows through the (o_acc, m, l) state.
#include <math.h>

#include "internal.h"

namespace sppo {
namespace {

constexpr int kWarps = 4;   // rows (fwd/dQ) or keys (dK/dV) per block, one warp each
constexpr int kTile = 32;   // keys (or query rows) per smem tile: one per lane

__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// ---------------------------------------------------------------- forward
// block = kWarps query rows of chunk i (one warp per row), head blockIdx.y.
// Key tiles of 32 are staged in smem; lane j scores key j, then every lane
// accumulates its d/32 output dims with the 32 probabilities (shuffle bcast).
template <int D>
__global__ void __launch_bounds__(kWarps * 32) fwd_simt_kernel(const FwdParams p, const KvWindow w) {
  constexpr int DPL = D / 32;  // dims per lane
  __shared__ float sk[kTile][D + 1];
  __shared__ float sv[kTile][D];
  __shared__ float sq[kWarps][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int r0 = blockIdx.x * kWarps;
  const int r = r0 + warp;
  const bool row_ok = r < p.q_len;
  const int pos = p.q_start + r;                              // absolute position of this row
  const int pos_max = p.q_start + min(r0 + kWarps, p.q_len) - 1;  // last row of the block
  const size_t rs = (size_t)p.heads * D;                     // token row stride
  const float* q = (const float*)p.q;

  for (int c = lane; c < D; c += 32) sq[warp][c] = row_ok ? q[(size_t)r * rs + (size_t)head * D + c] : 0.f;

  float m, l, acc[DPL];
  if (p.first || !row_ok) {
    m = -INFINITY; l = 0.f;
#pragma unroll
    for (int t = 0; t < DPL; ++t) acc[t] = 0.f;
  } else {
    m = p.m[(size_t)head * p.q_len + r];
    l = p.l[(size_t)head * p.q_len + r];
#pragma unroll
    for (int t = 0; t < DPL; ++t) acc[t] = p.o_acc[(size_t)r * rs + (size_t)head * D + lane + 32 * t];
  }

  for (int c = 0; c < w.n; ++c) {
    const int kstart = w.start[c];
    const int klen = w.len[c];
    const float* K = (const float*)w.k[c];
    const float* V = (const float*)w.v[c];
    const int kend = min(kstart + klen, pos_max + 1);  // keys beyond the block's last row are masked for all
    for (int t0 = kstart; t0 < kend; t0 += kTile) {
      __syncthreads();
      for (int e = threadIdx.x; e < kTile * D; e += blockDim.x) {
        const int j = e / D, cc = e % D;
        const int t = t0 + j;
        const bool ok = t < kstart + klen;
        const size_t off = (size_t)(t - kstart) * rs + (size_t)head * D + cc;
        sk[j][cc] = ok ? K[off] : 0.f;
        sv[j][cc] = ok ? V[off] : 0.f;
      }
      __syncthreads();
      if (!row_ok) continue;
      const int t = t0 + lane;
      float s = 0.f;
#pragma unroll 8
      for (int cc = 0; cc < D; ++cc) s = fmaf(sq[warp][cc], sk[lane][cc], s);
      s *= p.scale;
      const bool vis = (t < kstart + klen) && (t <= pos);  // causal mask on absolute positions (L2)
      s = vis ? s : -INFINITY;
      const float tmax = warp_max(s);
      const float m_new = fmaxf(m, tmax);
      if (m_new == -INFINITY) continue;  // nothing visible yet in this row
      const float corr = (m == -INFINITY) ? 0.f : expf(m - m_new);
      const float pj = vis ? expf(s - m_new) : 0.f;
      l = l * corr + warp_sum(pj);
#pragma unroll
      for (int tt = 0; tt < DPL; ++tt) acc[tt] *= corr;
      for (int j = 0; j < kTile; ++j) {
        const float pb = __shfl_sync(0xffffffffu, pj, j);
#pragma unroll
        for (int tt = 0; tt < DPL; ++tt) acc[tt] = fmaf(pb, sv[j][lane + 32 * tt], acc[tt]);
      }
      m = m_new;
    }
  }
  if (!row_ok) return;
  if (p.last) {
    const float inv = 1.f / l;
    float* o = (float*)p.o;
#pragma unroll
    for (int tt = 0; tt < DPL; ++tt) o[(size_t)r * rs + (size_t)head * D + lane + 32 * tt] = acc[tt] * inv;
    if (lane == 0) p.lse[(size_t)head * p.q_len + r] = m + logf(l);
  } else {
#pragma unroll
    for (int tt = 0; tt < DPL; ++tt) p.o_acc[(size_t)r * rs + (size_t)head * D + lane + 32 * tt] = acc[tt];
    if (lane == 0) {
      p.m[(size_t)head * p.q_len + r] = m;
      p.l[(size_t)head * p.q_len + r] = l;
    }
  }
}

// ---------------------------------------------------------------- backward
// dQ: one warp per query row p; keys staged in tiles of 32 (lane j = key j).
//   P_pj = exp(s - LSE_p), dP = <dO_p, v_j>, dS = P (dP - Delta_p),
//   dQ_p += tau sum_j dS_pj k_j
template <int D>
__global__ void __launch_bounds__(kWarps * 32) bwd_dq_simt_kernel(const BwdParams p, const KvWindow w) {
  constexpr int DPL = D / 32;
  __shared__ float sk[kTile][D + 1];
  __shared__ float sv[kTile][D + 1];
  __shared__ float sq[kWarps][D];
  __shared__ float sdo[kWarps][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int r0 = blockIdx.x * kWarps;
  const int r = r0 + warp;
  const bool row_ok = r < p.q_len;
  const int pos = p.q_start + r;
  const int pos_max = p.q_start + min(r0 + kWarps, p.q_len) - 1;
  const size_t rs = (size_t)p.heads * D;
  const float* q = (const float*)p.q;
  const float* dout = (const float*)p.dout;
  for (int c = lane; c < D; c += 32) {
    sq[warp][c] = row_ok ? q[(size_t)r * rs + (size_t)head * D + c] : 0.f;
    sdo[warp][c] = row_ok ? dout[(size_t)r * rs + (size_t)head * D + c] : 0.f;
  }
  const float lse = row_ok ? p.lse[(size_t)head * p.q_len + r] : 0.f;
  const float delta = row_ok ? p.delta[(size_t)head * p.q_len + r] : 0.f;
  float dq[DPL];
#pragma unroll
  for (int t = 0; t < DPL; ++t) dq[t] = 0.f;

  for (int c = 0; c < w.n; ++c) {
    const int kstart = w.start[c], klen = w.len[c];
    const float* K = (const float*)w.k[c];
    const float* V = (const float*)w.v[c];
    const int kend = min(kstart + klen, pos_max + 1);
    for (int t0 = kstart; t0 < kend; t0 += kTile) {
      __syncthreads();
      for (int e = threadIdx.x; e < kTile * D; e += blockDim.x) {
        const int j = e / D, cc = e % D;
        const int t = t0 + j;
        const bool ok = t < kstart + klen;
        const size_t off = (size_t)(t - kstart) * rs + (size_t)head * D + cc;
        sk[j][cc] = ok ? K[off] : 0.f;
        sv[j][cc] = ok ? V[off] : 0.f;
      }
      __syncthreads();
      if (!row_ok) continue;
      const int t = t0 + lane;
      float s = 0.f, dp = 0.f;
#pragma unroll 8
      for (int cc = 0; cc < D; ++cc) {
        s = fmaf(sq[warp][cc], sk[lane][cc], s);
        dp = fmaf(sdo[warp][cc], sv[lane][cc], dp);
      }
      const bool vis = (t < kstart + klen) && (t <= pos);
      const float pr = vis ? expf(s * p.scale - lse) : 0.f;
      const float ds = pr * (dp - delta);
      for (int j = 0; j < kTile; ++j) {
        const float db = __shfl_sync(0xffffffffu, ds, j);
#pragma unroll
        for (int tt = 0; tt < DPL; ++tt) dq[tt] = fmaf(db, sk[j][lane + 32 * tt], dq[tt]);
      }
    }
  }
  if (!row_ok) return;
#pragma unroll
  for (int tt = 0; tt < DPL; ++tt) p.dq_acc[(size_t)r * rs + (size_t)head * D + lane + 32 * tt] += p.scale * dq[tt];
}

// dK/dV: one warp per key t of window chunk blockIdx.z; query rows of chunk i
// staged in tiles of 32 (lane r = row r).
//   dV_t += sum_p P_pt dO_p,  dK_t += tau sum_p dS_pt q_p   (p >= t)
template <int D>
__global__ void __launch_bounds__(kWarps * 32) bwd_dkdv_simt_kernel(const BwdParams p, const KvWindow w,
                                                                   const KvGradWindow g) {
  constexpr int DPL = D / 32;
  __shared__ float sq[kTile][D + 1];
  __shared__ float sdo[kTile][D + 1];
  __shared__ float slse[kTile], sdelta[kTile];
  __shared__ float sk[kWarps][D];
  __shared__ float sv[kWarps][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int c = blockIdx.z;
  const int kstart = w.start[c], klen = w.len[c];
  const int j0 = blockIdx.x * kWarps;
  if (j0 >= klen) return;
  const int j = j0 + warp;
  const bool key_ok = j < klen;
  const int t = kstart + j;
  const int t_min = kstart + j0;  // first key of the block
  const size_t rs = (size_t)p.heads * D;
  const float* K = (const float*)w.k[c];
  const float* V = (const float*)w.v[c];
  for (int cc = lane; cc < D; cc += 32) {
    sk[warp][cc] = key_ok ? K[(size_t)j * rs + (size_t)head * D + cc] : 0.f;
    sv[warp][cc] = key_ok ? V[(size_t)j * rs + (size_t)head * D + cc] : 0.f;
  }
  float dk[DPL], dv[DPL];
#pragma unroll
  for (int tt = 0; tt < DPL; ++tt) dk[tt] = dv[tt] = 0.f;
  const float* q = (const float*)p.q;
  const float* dout = (const float*)p.dout;
  // rows p >= t_min only
  const int rstart = max(0, t_min - p.q_start);
  for (int r0 = (rstart / kTile) * kTile; r0 < p.q_len; r0 += kTile) {
    __syncthreads();
    for (int e = threadIdx.x; e < kTile * D; e += blockDim.x) {
      const int rr = e / D, cc = e % D;
      const int row = r0 + rr;
      const bool ok = row < p.q_len;
      const size_t off = (size_t)row * rs + (size_t)head * D + cc;
      sq[rr][cc] = ok ? q[off] : 0.f;
      sdo[rr][cc] = ok ? dout[off] : 0.f;
    }
    if (threadIdx.x < kTile) {
      const int row = r0 + threadIdx.x;
      const bool ok = row < p.q_len;
      slse[threadIdx.x] = ok ? p.lse[(size_t)head * p.q_len + row] : 0.f;
      sdelta[threadIdx.x] = ok ? p.delta[(size_t)head * p.q_len + row] : 0.f;
    }
    __syncthreads();
    if (!key_ok) continue;
    const int row = r0 + lane;
    float s = 0.f, dp = 0.f;
#pragma unroll 8
    for (int cc = 0; cc < D; ++cc) {
      s = fmaf(sq[lane][cc], sk[warp][cc], s);
      dp = fmaf(sdo[lane][cc], sv[warp][cc], dp);
    }
    const bool vis = (row < p.q_len) && (p.q_start + row >= t);
    const float pr = vis ? expf(s * p.scale - slse[lane]) : 0.f;
    const float ds = pr * (dp - sdelta[lane]);
    for (int rr = 0; rr < kTile; ++rr) {
      const float pb = __shfl_sync(0xffffffffu, pr, rr);
      const float db = __shfl_sync(0xffffffffu, ds, rr);
#pragma unroll
      for (int tt = 0; tt < DPL; ++tt) {
        dv[tt] = fmaf(pb, sdo[rr][lane + 32 * tt], dv[tt]);
        dk[tt] = fmaf(db, sq[rr][lane + 32 * tt], dk[tt]);
      }
    }
  }
  if (!key_ok) return;
  float* dka = g.dk[c];
  float* dva = g.dv[c];
  const bool final_out = (c == p.final_slot);
#pragma unroll
  for (int tt = 0; tt < DPL; ++tt) {
    const size_t off = (size_t)j * rs + (size_t)head * D + lane + 32 * tt;
    const float nk = dka[off] + p.scale * dk[tt];
    const float nv = dva[off] + dv[tt];
    dka[off] = nk;
    dva[off] = nv;
    if (final_out) {
      ((float*)p.dk_out)[off] = nk;
      ((float*)p.dv_out)[off] = nv;
    }
  }
}

}  // namespace

cudaError_t launch_fwd_simt_f32(const FwdParams& p, const KvWindow& w, cudaStream_t s) {
  dim3 grid((p.q_len + kWarps - 1) / kWarps, p.heads);
  if (p.d == 64)
    fwd_simt_kernel<64><<<grid, kWarps * 32, 0, s>>>(p, w);
  else if (p.d == 128)
    fwd_simt_kernel<128><<<grid, kWarps * 32, 0, s>>>(p, w);
  else if (p.d == 32)
    fwd_simt_kernel<32><<<grid, kWarps * 32, 0, s>>>(p, w);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_bwd_simt_f32(const BwdParams& p, const KvWindow& w, const KvGradWindow& g,
                                cudaStream_t s) {
  dim3 gq((p.q_len + kWarps - 1) / kWarps, p.heads);
  int maxlen = 0;
  for (int c = 0; c < w.n; ++c) maxlen = w.len[c] > maxlen ? w.len[c] : maxlen;
  dim3 gk((maxlen + kWarps - 1) / kWarps, p.heads, w.n);
  switch (p.d) {
    case 32:
      bwd_dq_simt_kernel<32><<<gq, kWarps * 32, 0, s>>>(p, w);
      bwd_dkdv_simt_kernel<32><<<gk, kWarps * 32, 0, s>>>(p, w, g);
      break;
    case 64:
      bwd_dq_simt_kernel<64><<<gq, kWarps * 32, 0, s>>>(p, w);
      bwd_dkdv_simt_kernel<64><<<gk, kWarps * 32, 0, s>>>(p, w, g);
      break;
    case 128:
      bwd_dq_simt_kernel<128><<<gq, kWarps * 32, 0, s>>>(p, w);
      bwd_dkdv_simt_kernel<128><<<gk, kWarps * 32, 0, s>>>(p, w, g);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace sppo
