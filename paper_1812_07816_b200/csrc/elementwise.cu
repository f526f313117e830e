// HBM-bound kernels of the U-Net step: input layout conversion, BatchNorm
// statistics / apply / backward, ReLU backward, 2x2x2 max-pool forward and
// backward (fused with the concat-shortcut gradient), channel concat, the
// 1x1x1 head + softmax + soft-Dice loss and its gradient, and Adam.
//
// Activations are NDHWC, stored as fp32 (check mode) or bf16; all arithmetic
// and reductions are fp32 (partials) / fp64 (cross-block finalisation).
// Op semantics follow the reference graph's node kinds (pkg/src/swapsim/
// models.py:91-153): norm -> BatchNorm3d (batch statistics; = InstanceNorm at
// batch 1), activation -> ReLU, pool -> MaxPool3d(2), concat -> [shortcut,
// upsampled], loss -> 1x1x1 head + softmax + soft Dice.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>

#include "kernels.h"
#include "sm100.cuh"

namespace us {
namespace {

constexpr int kT = 256;

__device__ __forceinline__ float ld(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ld(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}
__device__ __forceinline__ void st(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void st(__nv_bfloat16* p, int64_t i, float v) {
  p[i] = __float2bfloat16(v);
}

// 8 consecutive elements (16 B of bf16 / 32 B of fp32) <-> 8 floats.
__device__ __forceinline__ void ld8(const float* p, int64_t i, float (&o)[8]) {
  float4 a = *reinterpret_cast<const float4*>(p + i);
  float4 b = *reinterpret_cast<const float4*>(p + i + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
__device__ __forceinline__ void ld8(const __nv_bfloat16* p, int64_t i, float (&o)[8]) {
  uint4 u = *reinterpret_cast<const uint4*>(p + i);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 f = __bfloat1622float2(h[j]);
    o[2 * j] = f.x;
    o[2 * j + 1] = f.y;
  }
}
__device__ __forceinline__ void st8(float* p, int64_t i, const float (&o)[8]) {
  *reinterpret_cast<float4*>(p + i) = make_float4(o[0], o[1], o[2], o[3]);
  *reinterpret_cast<float4*>(p + i + 4) = make_float4(o[4], o[5], o[6], o[7]);
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, int64_t i, const float (&o)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(o[2 * j], o[2 * j + 1]);
  *reinterpret_cast<uint4*>(p + i) = u;
}

inline int grid_for(int64_t work, int per = kT, int cap = 148 * 16) {
  int64_t b = (work + per - 1) / per;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

#define DISPATCH_T(dtype, ...)                  \
  do {                                          \
    if ((dtype) == 2) {                         \
      using T = __nv_bfloat16;                  \
      __VA_ARGS__;                              \
    } else {                                    \
      using T = float;                          \
      __VA_ARGS__;                              \
    }                                           \
  } while (0)

// ------------------------------------------------------------------ layout
// Augmentation (paper: random axis flips and permutations before every iteration,
// PAPER.md:90) folded into the input conversion: output voxel (z, y, x) reads the input
// voxel whose axis perm[i] coordinate is output coordinate i, flipped if bit i of the mask
// is set (bit 0 = x, 1 = y, 2 = z).  aug = {flip mask, permutation index} or null.
__constant__ int8_t c_aug_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                        {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

__device__ __forceinline__ int64_t aug_source(const int* aug, int64_t s, int D, int H, int W) {
  if (!aug) return s;
  const int dims[3] = {D, H, W};
  int o[3];
  o[2] = (int)(s % W);
  int64_t r = s / W;
  o[1] = (int)(r % H);
  o[0] = (int)(r / H);
  const int flips = aug[0], perm = aug[1];
  int in[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    int v = o[i];
    if (flips & (1 << (2 - i))) v = dims[i] - 1 - v;
    in[c_aug_perm[perm][i]] = v;
  }
  // input dims along axis perm[i] equal the output dims (only shape-preserving perms)
  return ((int64_t)in[0] * H + in[1]) * W + in[2];
}

template <class T>
__global__ void k_input_ncdhw(const float* __restrict__ src, T* __restrict__ dst, int N, int C,
                              int D, int H, int W, int Cdst, const int* __restrict__ aug) {
  int64_t vox = (int64_t)D * H * W;
  int64_t total = (int64_t)N * vox;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = v / vox, s = aug_source(aug, v % vox, D, H, W);
    for (int c = 0; c < Cdst; ++c)
      st(dst, v * Cdst + c, c < C ? src[(n * C + c) * vox + s] : 0.f);
  }
}

__global__ void k_labels_aug(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int N,
                             int D, int H, int W, const int* __restrict__ aug) {
  int64_t vox = (int64_t)D * H * W;
  int64_t total = (int64_t)N * vox;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = v / vox;
    dst[v] = src[n * vox + aug_source(aug, v % vox, D, H, W)];
  }
}

// One thread per (voxel, 8-channel group of the destination): 16/32-byte stores.
template <class T>
__global__ void k_pad_v8(const T* __restrict__ src, T* __restrict__ dst, int64_t vox, int C,
                         int Cdst) {
  int gv = Cdst / 8;
  int64_t total = vox * gv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = i / gv;
    int c0 = (int)(i % gv) * 8;
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (c0 + j < C) ? ld(src, v * C + c0 + j) : 0.f;
    st8(dst, i * 8, o);
  }
}

template <class T>
__global__ void k_pad(const T* __restrict__ src, T* __restrict__ dst, int64_t vox, int C,
                      int Cdst) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < vox;
       v += (int64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < Cdst; ++c) st(dst, v * Cdst + c, c < C ? ld(src, v * C + c) : 0.f);
}

// ------------------------------------------------------------------ channel reductions
// Per-channel sums over voxels of an NDHWC tensor.  Thread layout: lane group
// g handles channels [g*CV, g*CV+CV) for a strided set of voxels; each block
// writes one partial row part[block][2][C].
//   mode 0: (sum x, sum x^2)             -- BatchNorm forward statistics
//   mode 1: (sum dy, sum dy*xhat)        -- BatchNorm backward reductions
template <class T, int CV>
__global__ void k_chan_sums(const T* __restrict__ x, const T* __restrict__ dy,
                            const float* __restrict__ stat, float* __restrict__ part,
                            int64_t vox, int C, int mode) {
  extern __shared__ float sh[];  // [blockDim][2*CV]
  int groups = C / CV;
  int lanes = blockDim.x / groups;     // voxel lanes per block
  int t = threadIdx.x;
  int g = t % groups, vl = t / groups;
  float a[CV], b[CV], mean[CV], rstd[CV];
#pragma unroll
  for (int j = 0; j < CV; ++j) {
    a[j] = b[j] = 0.f;
    if (mode == 1) {
      mean[j] = stat[g * CV + j];
      rstd[j] = stat[C + g * CV + j];
    }
  }
  if (vl < lanes) {
    for (int64_t v = (int64_t)blockIdx.x * lanes + vl; v < vox; v += (int64_t)gridDim.x * lanes) {
      int64_t base = v * C + g * CV;
      float xv[CV], dv[CV];
      if constexpr (CV == 8) {
        ld8(x, base, xv);
        if (mode == 1) ld8(dy, base, dv);
      } else {
#pragma unroll
        for (int j = 0; j < CV; ++j) {
          xv[j] = ld(x, base + j);
          dv[j] = mode == 1 ? ld(dy, base + j) : 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < CV; ++j) {
        if (mode == 0) {
          a[j] += xv[j];
          b[j] += xv[j] * xv[j];
        } else {
          a[j] += dv[j];
          b[j] += dv[j] * ((xv[j] - mean[j]) * rstd[j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < CV; ++j) {
    sh[t * 2 * CV + j] = (vl < lanes) ? a[j] : 0.f;
    sh[t * 2 * CV + CV + j] = (vl < lanes) ? b[j] : 0.f;
  }
  __syncthreads();
  // reduce over voxel lanes sharing the same channel group
  for (int idx = t; idx < groups * 2 * CV; idx += blockDim.x) {
    int gg = idx / (2 * CV), r = idx % (2 * CV);
    float s = 0.f;
    for (int l = 0; l < lanes; ++l) s += sh[(l * groups + gg) * 2 * CV + r];
    int c = gg * CV + (r % CV);
    part[(int64_t)blockIdx.x * 2 * C + (r < CV ? 0 : C) + c] = s;
  }
}

int chan_vec(int C) { return (C % 8 == 0) ? 8 : (C % 4 == 0 ? 4 : 1); }

int chan_sum_blocks(int64_t vox, int C) {
  int cv = chan_vec(C);
  int groups = C / cv;
  int lanes = kT / groups;
  if (lanes < 1) lanes = 1;
  int64_t b = (vox + lanes * 8 - 1) / ((int64_t)lanes * 8);
  if (b < 1) b = 1;
  if (b > 148 * 4) b = 148 * 4;
  return (int)b;
}

template <class T>
cudaError_t launch_chan_sums(cudaStream_t s, const T* x, const T* dy, const float* stat,
                             float* part, int64_t vox, int C, int mode, int blocks) {
  int cv = chan_vec(C);
  int groups = C / cv;
  int threads = groups > kT ? groups : (kT / groups) * groups;
  if (threads > 1024) return cudaErrorInvalidValue;
  size_t smem = (size_t)threads * 2 * cv * sizeof(float);
  if (cv == 8)
    k_chan_sums<T, 8><<<blocks, threads, smem, s>>>(x, dy, stat, part, vox, C, mode);
  else if (cv == 4)
    k_chan_sums<T, 4><<<blocks, threads, smem, s>>>(x, dy, stat, part, vox, C, mode);
  else
    k_chan_sums<T, 1><<<blocks, threads, smem, s>>>(x, dy, stat, part, vox, C, mode);
  return cudaGetLastError();
}

// Sum of the per-block partials part[p][2][C] for 32 channels per block: 32 part
// lanes x 32 channel lanes (1024 threads), then a fixed-order combination of the 32
// lanes (deterministic).  nparts is ~1000 at full resolution: 32 lanes keep the
// per-thread dependent-load chain short.
constexpr int kFinLanes = 32;
__device__ __forceinline__ void sum_parts_2c(const float* __restrict__ part, int nparts, int C,
                                             int c, double& s, double& q) {
  __shared__ double rs[kFinLanes][32], rq[kFinLanes][32];
  int lc = threadIdx.x & 31, pl = threadIdx.x >> 5;
  double a = 0, b = 0;
  if (c < C)
    for (int p = pl; p < nparts; p += kFinLanes) {
      a += part[(int64_t)p * 2 * C + c];
      b += part[(int64_t)p * 2 * C + C + c];
    }
  rs[pl][lc] = a;
  rq[pl][lc] = b;
  __syncthreads();
  s = q = 0;
  for (int k = 0; k < kFinLanes; ++k) {
    s += rs[k][lc];
    q += rq[k][lc];
  }
}

__global__ void __launch_bounds__(32 * kFinLanes) k_bn_finalize(const float* __restrict__ part, int nparts, int C, double count,
                              float* __restrict__ stat, double eps) {
  int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double s, q;
  sum_parts_2c(part, nparts, C, c, s, q);
  if (threadIdx.x >= 32 || c >= C) return;
  double mean = s / count;
  double var = q / count - mean * mean;
  if (var < 0) var = 0;
  stat[c] = (float)mean;
  stat[C + c] = (float)(1.0 / sqrt(var + eps));
}

template <class T>
__global__ void k_norm_act(const T* __restrict__ x, const float* __restrict__ stat,
                           const float* __restrict__ gamma, const float* __restrict__ beta,
                           T* __restrict__ norm, T* __restrict__ act, int64_t n, int C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    float y = (ld(x, i) - stat[c]) * stat[C + c] * gamma[c] + beta[c];
    if (norm) st(norm, i, y);
    if (act) st(act, i, y > 0.f ? y : 0.f);
  }
}

// bf16 vectorised variant: 8 channels (16 bytes) per thread step.
__global__ void k_norm_act_v8(const uint4* __restrict__ x, const float* __restrict__ stat,
                              const float* __restrict__ gamma, const float* __restrict__ beta,
                              uint4* __restrict__ norm, uint4* __restrict__ act, int64_t nvec,
                              int C) {
  // y = x * a[c] + b[c] with a = rstd * gamma, b = beta - mean * a, staged in smem
  extern __shared__ float ab[];   // [2][C]
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float a = stat[C + c] * gamma[c];
    ab[c] = a;
    ab[C + c] = beta[c] - stat[c] * a;
  }
  __syncthreads();
  const int cvec = C / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // 4 independent 16-byte loads in flight per thread (the loop is otherwise one HBM
  // round trip per vector)
  constexpr int kU = 4;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < nvec;
       i0 += kU * stride) {
    uint4 in[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * stride;
      in[u] = i < nvec ? __ldg(x + i) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= nvec) break;
      int c0 = (int)(i % cvec) * 8;
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&in[u]);
      float4 a0 = *reinterpret_cast<const float4*>(ab + c0);
      float4 a1 = *reinterpret_cast<const float4*>(ab + c0 + 4);
      float4 b0 = *reinterpret_cast<const float4*>(ab + C + c0);
      float4 b1 = *reinterpret_cast<const float4*>(ab + C + c0 + 4);
      float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      uint4 on, oa;
      __nv_bfloat162* hn = reinterpret_cast<__nv_bfloat162*>(&on);
      __nv_bfloat162* ha = reinterpret_cast<__nv_bfloat162*>(&oa);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        float y0 = f.x * av[2 * j] + bv[2 * j];
        float y1 = f.y * av[2 * j + 1] + bv[2 * j + 1];
        hn[j] = __floats2bfloat162_rn(y0, y1);
        ha[j] = __floats2bfloat162_rn(y0 > 0.f ? y0 : 0.f, y1 > 0.f ? y1 : 0.f);
      }
      if (norm) norm[i] = on;
      if (act) act[i] = oa;
    }
  }
}

template <class T>
__global__ void k_relu_bwd(const T* __restrict__ dy, const T* __restrict__ y, T* __restrict__ dx,
                           int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    st(dx, i, ld(y, i) > 0.f ? ld(dy, i) : 0.f);
}

// BN backward finalisation: grads of gamma/beta and the apply coefficients
// coef[c] = (gamma*rstd, mean(dy), mean(dy*xhat)).
__global__ void __launch_bounds__(32 * kFinLanes) k_bn_bwd_finalize(const float* __restrict__ part, int nparts, int C, double count,
                                  const float* __restrict__ stat, const float* __restrict__ gamma,
                                  float* __restrict__ ggamma, float* __restrict__ gbeta,
                                  float* __restrict__ coef) {
  int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double s, q;
  sum_parts_2c(part, nparts, C, c, s, q);
  if (threadIdx.x >= 32 || c >= C) return;
  ggamma[c] = (float)q;
  gbeta[c] = (float)s;
  coef[c] = gamma[c] * stat[C + c];
  coef[C + c] = (float)(s / count);
  coef[2 * C + c] = (float)(q / count);
}

template <class T>
__global__ void k_bn_bwd_apply(const T* __restrict__ x, const T* __restrict__ dy,
                               const float* __restrict__ stat, const float* __restrict__ coef,
                               T* __restrict__ dx, int64_t n, int C) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    float xh = (ld(x, i) - stat[c]) * stat[C + c];
    st(dx, i, coef[c] * (ld(dy, i) - coef[C + c] - xh * coef[2 * C + c]));
  }
}

// ------------------------------------------------------------------ pooling
template <class T>
__global__ void k_pool_fwd(const T* __restrict__ x, T* __restrict__ y, int N, int D, int H, int W,
                           int C) {
  int Do = D / 2, Ho = H / 2, Wo = W / 2;
  int64_t total = (int64_t)N * Do * Ho * Wo * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    int64_t r = i / C;
    int xo = (int)(r % Wo); r /= Wo;
    int yo = (int)(r % Ho); r /= Ho;
    int zo = (int)(r % Do);
    int n = (int)(r / Do);
    float m = -INFINITY;
    for (int dz = 0; dz < 2; ++dz)
      for (int dyy = 0; dyy < 2; ++dyy)
        for (int dx = 0; dx < 2; ++dx) {
          int64_t idx = ((((int64_t)n * D + 2 * zo + dz) * H + 2 * yo + dyy) * W + 2 * xo + dx) * C + c;
          float v = ld(x, idx);
          if (v > m || v != v) m = v;
        }
    st(y, i, m);
  }
}

// dx = route(dy to the first max of each window) + dcat[..., dcat_co + c]
template <class T>
__global__ void k_pool_bwd(const T* __restrict__ x, const T* __restrict__ dy,
                           const T* __restrict__ dcat, int dcat_cs, int dcat_co,
                           T* __restrict__ dx, int N, int D, int H, int W, int C, int relu) {
  int Do = D / 2, Ho = H / 2, Wo = W / 2;
  int64_t total = (int64_t)N * Do * Ho * Wo * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    int64_t r = i / C;
    int xo = (int)(r % Wo); r /= Wo;
    int yo = (int)(r % Ho); r /= Ho;
    int zo = (int)(r % Do);
    int n = (int)(r / Do);
    float m = -INFINITY;
    int best = 0, pos = 0;
    int64_t vidx[8];
    int k = 0;
    for (int dz = 0; dz < 2; ++dz)
      for (int dyy = 0; dyy < 2; ++dyy)
        for (int dxx = 0; dxx < 2; ++dxx, ++k) {
          vidx[k] = (((int64_t)n * D + 2 * zo + dz) * H + 2 * yo + dyy) * W + 2 * xo + dxx;
          float v = ld(x, vidx[k] * C + c);
          if (v > 0.f) pos |= 1 << k;
          if (v > m || v != v) {
            m = v;
            best = k;
          }
        }
    float g = ld(dy, i);
    for (k = 0; k < 8; ++k) {
      float o = (k == best) ? g : 0.f;
      if (dcat) o += ld(dcat, vidx[k] * dcat_cs + dcat_co + c);
      if (relu && !((pos >> k) & 1)) o = 0.f;   // fused ReLU backward (x is the ReLU output)
      st(dx, vidx[k] * C + c, o);
    }
  }
}

template <class T>
__global__ void k_concat(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ y,
                         int64_t vox, int Ca, int Cb) {
  int Cy = Ca + Cb;
  int64_t total = vox * Cy;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = i / Cy;
    int c = (int)(i % Cy);
    st(y, i, c < Ca ? ld(a, v * Ca + c) : ld(b, v * Cb + (c - Ca)));
  }
}

// ------------------------------------------------------------------ 8-wide variants
// (C % 8 == 0: every 8-channel group is 16/32-byte aligned in NDHWC)
template <class T>
__global__ void k_relu_fwd(const T* __restrict__ x, T* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = ld(x, i);
    st(y, i, v > 0.f ? v : 0.f);
  }
}

template <class T>
__global__ void k_relu_fwd_v8(const T* __restrict__ x, T* __restrict__ y, int64_t nvec) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v[8];
    ld8(x, i * 8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = v[j] > 0.f ? v[j] : 0.f;
    st8(y, i * 8, v);
  }
}

template <class T>
__global__ void k_relu_bwd_v8(const T* __restrict__ dy, const T* __restrict__ y,
                              T* __restrict__ dx, int64_t nvec) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    float d[8], m[8];
    ld8(dy, i * 8, d);
    ld8(y, i * 8, m);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = m[j] > 0.f ? d[j] : 0.f;
    st8(dx, i * 8, d);
  }
}

template <class T>
__global__ void k_bn_bwd_apply_v8(const T* __restrict__ x, const T* __restrict__ dy,
                                  const float* __restrict__ stat, const float* __restrict__ coef,
                                  T* __restrict__ dx, int64_t nvec, int C) {
  // dx = k1*(dy - mdy - xhat*mdyx), xhat = (x - mean)*rstd  ==  A*dy + B*x + K
  extern __shared__ float cf[];   // [3][C]
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float k1 = coef[c], mdy = coef[C + c], mdyx = coef[2 * C + c];
    float r = stat[C + c], m = stat[c];
    cf[c] = k1;
    cf[C + c] = -k1 * r * mdyx;
    cf[2 * C + c] = -k1 * mdy + k1 * r * mdyx * m;
  }
  __syncthreads();
  int cvec = C / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c0 = (int)(i % cvec) * 8;
    float xv[8], d[8];
    ld8(x, i * 8, xv);
    ld8(dy, i * 8, d);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      d[j] = cf[c0 + j] * d[j] + cf[C + c0 + j] * xv[j] + cf[2 * C + c0 + j];
    st8(dx, i * 8, d);
  }
}

template <class T>
__global__ void k_concat_v8(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ y,
                            int64_t vox, int Ca, int Cb) {
  int cy = (Ca + Cb) / 8, ca = Ca / 8;
  int64_t total = vox * cy;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = i / cy;
    int c = (int)(i % cy);
    const uint4* src = c < ca ? reinterpret_cast<const uint4*>(a + v * Ca + c * 8)
                              : reinterpret_cast<const uint4*>(b + v * Cb + (c - ca) * 8);
    uint4* dst = reinterpret_cast<uint4*>(y + i * 8);
    constexpr int kWords = sizeof(T) * 8 / 16;   // 1 uint4 for bf16, 2 for fp32
#pragma unroll
    for (int k = 0; k < kWords; ++k) dst[k] = src[k];
  }
}

template <class T>
__global__ void k_pool_fwd_v8(const T* __restrict__ x, T* __restrict__ y, int N, int D, int H,
                              int W, int C) {
  int Do = D / 2, Ho = H / 2, Wo = W / 2, cv = C / 8;
  int64_t total = (int64_t)N * Do * Ho * Wo * cv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c0 = (int)(i % cv) * 8;
    int64_t r = i / cv;
    int xo = (int)(r % Wo); r /= Wo;
    int yo = (int)(r % Ho); r /= Ho;
    int zo = (int)(r % Do);
    int n = (int)(r / Do);
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = -INFINITY;
    for (int k = 0; k < 8; ++k) {
      int64_t vi = (((int64_t)n * D + 2 * zo + (k >> 2)) * H + 2 * yo + ((k >> 1) & 1)) * W +
                   2 * xo + (k & 1);
      float v[8];
      ld8(x, vi * C + c0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (v[j] > m[j] || v[j] != v[j]) m[j] = v[j];
    }
    st8(y, i * 8, m);
  }
}

// 8 consecutive elements of a 16-byte (bf16) vector as floats
__device__ __forceinline__ void unpack8(const uint4& u, float (&v)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
}

template <class T, bool BNS = false>
__global__ void k_pool_bwd_v8(const T* __restrict__ x, const T* __restrict__ dy,
                              const T* __restrict__ dcat, int dcat_cs, int dcat_co,
                              T* __restrict__ dx, int N, int D, int H, int W, int C, int relu,
                              const T* __restrict__ bnx = nullptr,
                              const float* __restrict__ bn_stat = nullptr,
                              float* __restrict__ bn_part = nullptr) {
  int Do = D / 2, Ho = H / 2, Wo = W / 2, cv = C / 8;
  int64_t total = (int64_t)N * Do * Ho * Wo * cv;
  // BNS: fused BN-backward sums of dx.  The grid stride is a multiple of cv, so a thread
  // keeps one 8-channel group and accumulates it in registers.
  float bs1[8], bs2[8], mean[8], rstd[8];
  if (BNS) {
    const int c0 = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) % cv) * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      bs1[j] = bs2[j] = 0.f;
      mean[j] = bn_stat[c0 + j];
      rstd[j] = bn_stat[C + c0 + j];
    }
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c0 = (int)(i % cv) * 8;
    int64_t r = i / cv;
    int xo = (int)(r % Wo); r /= Wo;
    int yo = (int)(r % Ho); r /= Ho;
    int zo = (int)(r % Do);
    int n = (int)(r / Do);
    float m[8];
    int best[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      m[j] = -INFINITY;
      best[j] = 0;
    }
    int64_t vidx[8];
    uint32_t pos[8];   // bit j: channel c0 + j of window position k is > 0 (ReLU mask)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      vidx[k] = (((int64_t)n * D + 2 * zo + (k >> 2)) * H + 2 * yo + ((k >> 1) & 1)) * W +
                2 * xo + (k & 1);
    // every load of the window (x, the concat gradient, dy) is issued before any use:
    // one memory round trip per output voxel instead of two
    uint4 xr[8], cr[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      xr[k] = __ldg(reinterpret_cast<const uint4*>(x + vidx[k] * C + c0));
      cr[k] = dcat ? __ldg(reinterpret_cast<const uint4*>(dcat + vidx[k] * dcat_cs + dcat_co +
                                                          c0))
                   : make_uint4(0u, 0u, 0u, 0u);
    }
    const uint4 gr = __ldg(reinterpret_cast<const uint4*>(dy + i * 8));
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float v[8];
      unpack8(xr[k], v);
      pos[k] = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (v[j] > 0.f) pos[k] |= 1u << j;
        if (v[j] > m[j] || v[j] != v[j]) {
          m[j] = v[j];
          best[j] = k;
        }
      }
    }
    float g[8];
    unpack8(gr, g);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float o[8];
      unpack8(cr[k], o);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o[j] += (best[j] == k) ? g[j] : 0.f;
        if (relu && !((pos[k] >> j) & 1u)) o[j] = 0.f;   // fused ReLU backward
      }
      st8(dx, vidx[k] * C + c0, o);
      if (BNS) {
        float xb[8];
        ld8(bnx, vidx[k] * C + c0, xb);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = __bfloat162float(__float2bfloat16(o[j]));   // as stored
          bs1[j] += d;
          bs2[j] += d * ((xb[j] - mean[j]) * rstd[j]);
        }
      }
    }
  }
  if (BNS) {   // deterministic block reduction: per-thread rows, fixed-order column sums
    extern __shared__ float bred[];   // [blockDim][16]
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      bred[threadIdx.x * 16 + j] = bs1[j];
      bred[threadIdx.x * 16 + 8 + j] = bs2[j];
    }
    __syncthreads();
    const int g0 = (int)((blockIdx.x * (int64_t)blockDim.x) % cv);   // group of thread 0
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      const int grp = c / 8, j = c % 8;
      float a = 0.f, b = 0.f;
      for (int t = (grp - g0 + cv) % cv; t < (int)blockDim.x; t += cv) {
        a += bred[t * 16 + j];
        b += bred[t * 16 + 8 + j];
      }
      bn_part[(int64_t)blockIdx.x * 2 * C + c] = a;
      bn_part[(int64_t)blockIdx.x * 2 * C + C + c] = b;
    }
  }
}

// ------------------------------------------------------------------ soft Dice loss
// One warp per voxel at a time; lanes stride over channels.  Per block partial
// sums part[block][3*ncls] = (sum p*g, sum p, sum g) per class.
constexpr int kMaxCls = 8;
constexpr int kLossWarps = 8;

template <class T>
__global__ void k_loss_fwd(const T* __restrict__ act, const uint8_t* __restrict__ labels,
                           const float* __restrict__ hw, const float* __restrict__ hb,
                           float* __restrict__ part, int64_t nvox, int C, int ncls) {
  extern __shared__ float w_s[];  // [ncls*C]
  __shared__ float red[kLossWarps][3 * kMaxCls];
  for (int i = threadIdx.x; i < ncls * C; i += blockDim.x) w_s[i] = hw[i];
  __syncthreads();
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float acc[3 * kMaxCls];
  for (int j = 0; j < 3 * kMaxCls; ++j) acc[j] = 0.f;
  int64_t gw = (int64_t)blockIdx.x * kLossWarps + warp, nw = (int64_t)gridDim.x * kLossWarps;
  for (int64_t v = gw; v < nvox; v += nw) {
    float z[kMaxCls];
    for (int k = 0; k < ncls; ++k) z[k] = 0.f;
    for (int c = lane; c < C; c += 32) {
      float a = ld(act, v * C + c);
      for (int k = 0; k < ncls; ++k) z[k] += a * w_s[k * C + c];
    }
    for (int k = 0; k < ncls; ++k)
      for (int o = 16; o; o >>= 1) z[k] += __shfl_xor_sync(0xffffffffu, z[k], o);
    if (lane == 0) {
      float mx = -INFINITY;
      for (int k = 0; k < ncls; ++k) {
        z[k] += hb[k];
        mx = fmaxf(mx, z[k]);
      }
      float se = 0.f;
      for (int k = 0; k < ncls; ++k) {
        z[k] = __expf(z[k] - mx);
        se += z[k];
      }
      int g = labels[v];
      for (int k = 0; k < ncls; ++k) {
        float p = z[k] / se;
        acc[k] += (g == k) ? p : 0.f;
        acc[kMaxCls + k] += p;
        acc[2 * kMaxCls + k] += (g == k) ? 1.f : 0.f;
      }
    }
  }
  if (lane == 0)
    for (int j = 0; j < 3 * kMaxCls; ++j) red[warp][j] = acc[j];
  __syncthreads();
  if (threadIdx.x < 3 * ncls) {
    int j = threadIdx.x, which = j / ncls, k = j % ncls;
    float s = 0.f;
    for (int w = 0; w < kLossWarps; ++w) s += red[w][which * kMaxCls + k];
    part[(int64_t)blockIdx.x * 3 * ncls + j] = s;
  }
}

__global__ void k_loss_finalize(const float* __restrict__ part, int nparts, int ncls, double eps,
                                double* __restrict__ dice, float* __restrict__ loss) {
  __shared__ double sums[3 * kMaxCls];
  int j = threadIdx.x;
  if (j < 3 * ncls) {
    double s = 0;
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * 3 * ncls + j];
    sums[j] = s;
    dice[j] = s;
  }
  __syncthreads();
  if (j == 0) {
    double acc = 0;
    for (int k = 0; k < ncls; ++k)
      acc += (2.0 * sums[k] + eps) / (sums[ncls + k] + sums[2 * ncls + k] + eps);
    double l = 1.0 - acc / ncls;
    dice[3 * ncls] = l;
    loss[0] = (float)l;
  }
}

template <class T>
__global__ void k_loss_bwd(const T* __restrict__ act, const uint8_t* __restrict__ labels,
                           const float* __restrict__ hw, const float* __restrict__ hb,
                           const double* __restrict__ dice, T* __restrict__ dact,
                           float* __restrict__ part, int64_t nvox, int C, int ncls, double eps,
                           int relu) {
  extern __shared__ float sm[];  // w_s[ncls*C], gacc[kLossWarps][ncls*C + ncls]
  float* w_s = sm;
  float* gacc = sm + ncls * C;
  int stride = ncls * C + ncls;
  for (int i = threadIdx.x; i < ncls * C; i += blockDim.x) w_s[i] = hw[i];
  for (int i = threadIdx.x; i < kLossWarps * stride; i += blockDim.x) gacc[i] = 0.f;
  __syncthreads();
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float cA[kMaxCls], cB[kMaxCls];  // dL/dp_k = cA_k * g_k + cB_k
  for (int k = 0; k < ncls; ++k) {
    double I = dice[k], P = dice[ncls + k], G = dice[2 * ncls + k];
    double den = P + G + eps;
    cA[k] = (float)(-(2.0 / ncls) / den);
    cB[k] = (float)((1.0 / ncls) * (2.0 * I + eps) / (den * den));
  }
  float* ga = gacc + warp * stride;
  int64_t gw = (int64_t)blockIdx.x * kLossWarps + warp, nw = (int64_t)gridDim.x * kLossWarps;
  for (int64_t v = gw; v < nvox; v += nw) {
    float z[kMaxCls];
    for (int k = 0; k < ncls; ++k) z[k] = 0.f;
    for (int c = lane; c < C; c += 32) {
      float a = ld(act, v * C + c);
      for (int k = 0; k < ncls; ++k) z[k] += a * w_s[k * C + c];
    }
    for (int k = 0; k < ncls; ++k)
      for (int o = 16; o; o >>= 1) z[k] += __shfl_xor_sync(0xffffffffu, z[k], o);
    float mx = -INFINITY;
    for (int k = 0; k < ncls; ++k) {
      z[k] += hb[k];
      mx = fmaxf(mx, z[k]);
    }
    float se = 0.f;
    for (int k = 0; k < ncls; ++k) {
      z[k] = __expf(z[k] - mx);
      se += z[k];
    }
    int g = labels[v];
    float dp[kMaxCls], dot = 0.f;
    for (int k = 0; k < ncls; ++k) {
      z[k] /= se;  // p_k
      dp[k] = cA[k] * (g == k ? 1.f : 0.f) + cB[k];
      dot += z[k] * dp[k];
    }
    for (int k = 0; k < ncls; ++k) z[k] = z[k] * (dp[k] - dot);  // dlogit_k
    for (int c = lane; c < C; c += 32) {
      float a = ld(act, v * C + c);
      float d = 0.f;
      for (int k = 0; k < ncls; ++k) {
        d += z[k] * w_s[k * C + c];
        ga[k * C + c] += z[k] * a;
      }
      if (relu && !(a > 0.f)) d = 0.f;   // fused ReLU backward (act is the ReLU output)
      st(dact, v * C + c, d);
    }
    if (lane < ncls) ga[ncls * C + lane] += z[lane];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < stride; i += blockDim.x) {
    float s = 0.f;
    for (int w = 0; w < kLossWarps; ++w) s += gacc[w * stride + i];
    part[(int64_t)blockIdx.x * stride + i] = s;
  }
}

// Thread-per-voxel variants (C % 8 == 0, C <= kVC): each thread reads its voxel's
// channel row with 16-byte loads; the head weights sit in shared memory.
constexpr int kVC = 64;
constexpr int kVWarps = 4;

template <class T, int NC>
__device__ __forceinline__ void head_logits(const T* act, int64_t v, int C, const float* w_s,
                                            const float* hb, float (&z)[NC],
                                            float* row /* may be null */) {
#pragma unroll
  for (int k = 0; k < NC; ++k) z[k] = hb[k];
  for (int c0 = 0; c0 < C; c0 += 8) {
    float a[8];
    ld8(act, v * C + c0, a);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (row) row[c0 + j] = a[j];
#pragma unroll
      for (int k = 0; k < NC; ++k) z[k] += a[j] * w_s[k * C + c0 + j];
    }
  }
}

template <int NC>
__device__ __forceinline__ void softmax_inplace(float (&z)[NC]) {
  float mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < NC; ++k) mx = fmaxf(mx, z[k]);
  float se = 0.f;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    z[k] = __expf(z[k] - mx);
    se += z[k];
  }
  float inv = 1.f / se;
#pragma unroll
  for (int k = 0; k < NC; ++k) z[k] *= inv;
}

template <class T, int NC>
__global__ void k_loss_fwd_v(const T* __restrict__ act, const uint8_t* __restrict__ labels,
                             const float* __restrict__ hw, const float* __restrict__ hb,
                             float* __restrict__ part, int64_t nvox, int C) {
  __shared__ float w_s[NC * kVC];
  __shared__ float red[kVWarps][3 * NC];
  for (int i = threadIdx.x; i < NC * C; i += blockDim.x) w_s[i] = hw[i];
  __syncthreads();
  float acc[3 * NC];
#pragma unroll
  for (int j = 0; j < 3 * NC; ++j) acc[j] = 0.f;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvox;
       v += (int64_t)gridDim.x * blockDim.x) {
    float z[NC];
    head_logits<T, NC>(act, v, C, w_s, hb, z, nullptr);
    softmax_inplace<NC>(z);
    int g = labels[v];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      acc[k] += (g == k) ? z[k] : 0.f;
      acc[NC + k] += z[k];
      acc[2 * NC + k] += (g == k) ? 1.f : 0.f;
    }
  }
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#pragma unroll
  for (int j = 0; j < 3 * NC; ++j) {
    float s = acc[j];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp][j] = s;
  }
  __syncthreads();
  if (threadIdx.x < 3 * NC) {
    int j = threadIdx.x;
    float s = 0.f;
    for (int w = 0; w < kVWarps; ++w) s += red[w][j];
    part[(int64_t)blockIdx.x * 3 * NC + j] = s;
  }
}

template <class T, int NC>
__global__ void k_loss_bwd_v(const T* __restrict__ act, const uint8_t* __restrict__ labels,
                             const float* __restrict__ hw, const float* __restrict__ hb,
                             const double* __restrict__ dice, T* __restrict__ dact,
                             float* __restrict__ part, int64_t nvox, int C, double eps, int relu) {
  constexpr int ncls = NC;
  __shared__ float w_s[NC * kVC];
  __shared__ float rows[kVWarps][32][kVC + 1];      // staged activations of the warp's voxels
  __shared__ float dzs[kVWarps][32][NC];
  __shared__ float red[kVWarps][NC * kVC + NC];
  for (int i = threadIdx.x; i < ncls * C; i += blockDim.x) w_s[i] = hw[i];
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float cA[NC], cB[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    double I = dice[k], P = dice[ncls + k], G = dice[2 * ncls + k];
    double den = P + G + eps;
    cA[k] = (float)(-(2.0 / ncls) / den);
    cB[k] = (float)((1.0 / ncls) * (2.0 * I + eps) / (den * den));
  }
  float gw[NC][kVC / 32];   // lane owns channels lane, lane + 32
  float gb[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    gb[k] = 0.f;
    for (int q = 0; q < kVC / 32; ++q) gw[k][q] = 0.f;
  }
  const int64_t per_iter = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < nvox; base += per_iter) {
    int64_t v = base + threadIdx.x;
    bool ok = v < nvox;
    float z[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) z[k] = 0.f;
    if (ok) {
      head_logits<T, NC>(act, v, C, w_s, hb, z, rows[warp][lane]);
      softmax_inplace<NC>(z);
      int g = labels[v];
      float dp[NC], dot = 0.f;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        dp[k] = cA[k] * (g == k ? 1.f : 0.f) + cB[k];
        dot += z[k] * dp[k];
      }
#pragma unroll
      for (int k = 0; k < NC; ++k) z[k] = z[k] * (dp[k] - dot);   // dlogit
      for (int c0 = 0; c0 < C; c0 += 8) {
        float d[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float s = 0.f;
#pragma unroll
          for (int k = 0; k < NC; ++k) s += z[k] * w_s[k * C + c0 + j];
          d[j] = (relu && !(rows[warp][lane][c0 + j] > 0.f)) ? 0.f : s;   // fused ReLU bwd
        }
        st8(dact, v * C + c0, d);
      }
    } else {
      for (int c = 0; c < C; ++c) rows[warp][lane][c] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      dzs[warp][lane][k] = z[k];
      gb[k] += z[k];
    }
    __syncwarp();
    for (int r = 0; r < 32; ++r)
      for (int q = 0; q < kVC / 32; ++q) {
        int c = lane + 32 * q;
        if (c < C) {
          float a = rows[warp][r][c];
#pragma unroll
          for (int k = 0; k < NC; ++k) gw[k][q] += dzs[warp][r][k] * a;
        }
      }
    __syncwarp();
  }
  // block reduction of the head-gradient partials
#pragma unroll
  for (int k = 0; k < NC; ++k) {
#pragma unroll
    for (int q = 0; q < kVC / 32; ++q) {
      int c = lane + 32 * q;
      if (c < C) red[warp][k * C + c] = gw[k][q];
    }
    float s = gb[k];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp][ncls * C + k] = s;
  }
  __syncthreads();
  int stride = ncls * C + ncls;
  for (int i = threadIdx.x; i < stride; i += blockDim.x) {
    float s = 0.f;
    for (int w = 0; w < kVWarps; ++w) s += red[w][i];
    part[(int64_t)blockIdx.x * stride + i] = s;
  }
}

// Tiled variants for the paper's head (bf16, C = 64).  A block streams 256-voxel tiles
// (32 KB, contiguous in NDHWC) through two shared buffers with 1-D bulk copies: the copy
// of tile k+1 is in flight while tile k is computed, so HBM sees a continuous stream
// instead of load/compute bursts.  Each thread owns one voxel row (reading its 16-byte
// chunks in a rotated order, chunk (j + t) & 7, so 8 consecutive rows hit 8 different
// bank groups); the backward rewrites the tile in place as dact and bulk-stores it, and
// accumulates the head weight gradient from the tile (thread = channel pair x row
// group).
constexpr int kLT = 256;
constexpr int kLTileBytes = kLT * 64 * 2;

template <int NC, bool BWD>
__global__ void __launch_bounds__(kLT, 2) k_loss_tile(
    const __nv_bfloat16* __restrict__ act, const uint8_t* __restrict__ labels,
    const float* __restrict__ hw, const float* __restrict__ hb, const double* __restrict__ dice,
    __nv_bfloat16* __restrict__ dact, float* __restrict__ part, int64_t nvox, double eps,
    int relu, const __nv_bfloat16* __restrict__ bnx = nullptr,
    const float* __restrict__ bn_stat = nullptr, float* __restrict__ bn_part = nullptr) {
  // bn_part (BWD): fused BN-backward sums of dact (per block rows of (sum d, sum d*xhat))
  constexpr int C = 64;
  extern __shared__ __align__(128) uint8_t loss_smem[];
  uint4* tiles = reinterpret_cast<uint4*>(loss_smem);    // [2][kLT * 8]
  __shared__ __align__(8) uint64_t full[2];
  // head weights [c][k], each 8-channel group padded by 4 floats: threads reading their
  // rows in rotated chunk order hit 8 different groups at once, and the padding puts the
  // 8 groups in 8 different bank quads (no conflicts).
  constexpr int kGrp = 8 * NC + 4;
  __shared__ __align__(16) float w_s[8 * kGrp];
  __shared__ float dz_s[kLT][NC];
  const int t = threadIdx.x;
  for (int i = t; i < C * NC; i += kLT) {
    const int c = i % C;
    w_s[(c >> 3) * kGrp + (c & 7) * NC + i / C] = hw[i];
  }
  if (t == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_barrier_init();
  }
  float bias[NC], cA[NC], cB[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    bias[k] = hb[k];
    if (BWD) {
      double I = dice[k], P = dice[NC + k], G = dice[2 * NC + k];
      double den = P + G + eps;
      cA[k] = (float)(-(2.0 / NC) / den);
      cB[k] = (float)((1.0 / NC) * (2.0 * I + eps) / (den * den));
    }
  }
  float acc[3 * NC];   // FWD: I,P,G ; BWD: gb[k], gw[k][2]
#pragma unroll
  for (int j = 0; j < 3 * NC; ++j) acc[j] = 0.f;
  const int cp = t & 31, grp = t >> 5;   // BWD weight-gradient ownership
  float bsum[4] = {0.f, 0.f, 0.f, 0.f}, bm[2] = {0.f, 0.f}, br[2] = {0.f, 0.f};
  if (BWD && bn_part) {
    bm[0] = bn_stat[2 * cp];
    bm[1] = bn_stat[2 * cp + 1];
    br[0] = bn_stat[C + 2 * cp];
    br[1] = bn_stat[C + 2 * cp + 1];
  }
  __syncthreads();
  const int64_t step = (int64_t)gridDim.x * kLT;
  auto rows_of = [&](int64_t base) { return (int)(nvox - base < kLT ? nvox - base : kLT); };
  if (t == 0 && (int64_t)blockIdx.x * kLT < nvox) {
    const int64_t b0 = (int64_t)blockIdx.x * kLT;
    const uint32_t bytes = (uint32_t)rows_of(b0) * 128;
    mbar_arrive_expect_tx(&full[0], bytes);
    bulk_load(tiles, act + b0 * C, bytes, &full[0]);
  }
  int k = 0;
  for (int64_t base = (int64_t)blockIdx.x * kLT; base < nvox; base += step, ++k) {
    const int buf = k & 1;
    uint4* tile = tiles + buf * kLT * 8;
    const int nv = rows_of(base);
    if (t == 0 && base + step < nvox) {   // prefetch the next tile into the other buffer
      if (BWD) tma_store_wait_read<0>();   // its previous dact store has left smem
      const uint32_t bytes = (uint32_t)rows_of(base + step) * 128;
      mbar_arrive_expect_tx(&full[buf ^ 1], bytes);
      bulk_load(tiles + (buf ^ 1) * kLT * 8, act + (base + step) * C, bytes, &full[buf ^ 1]);
    }
    mbar_wait(&full[buf], (uint32_t)(k >> 1) & 1u);
    float z[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) z[q] = bias[q];
    const bool own = t < nv;
    if (own) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int jj = (j + t) & 7;
        const uint4 u = tile[t * 8 + jj];
        const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e]));
          const float* wr = w_s + jj * kGrp + 2 * e * NC;
#pragma unroll
          for (int q = 0; q < NC; ++q) z[q] += f.x * wr[q] + f.y * wr[NC + q];
        }
      }
      float mx = -INFINITY;
#pragma unroll
      for (int q = 0; q < NC; ++q) mx = fmaxf(mx, z[q]);
      float se = 0.f;
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        z[q] = __expf(z[q] - mx);
        se += z[q];
      }
      const float inv = 1.f / se;
      const int g = labels[base + t];
      if (!BWD) {
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          const float pk = z[q] * inv;
          acc[q] += (g == q) ? pk : 0.f;
          acc[NC + q] += pk;
          acc[2 * NC + q] += (g == q) ? 1.f : 0.f;
        }
      } else {
        float dp[NC], dot = 0.f;
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          z[q] *= inv;
          dp[q] = cA[q] * (g == q ? 1.f : 0.f) + cB[q];
          dot += z[q] * dp[q];
        }
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          z[q] = z[q] * (dp[q] - dot);   // dlogit
          acc[q] += z[q];
        }
      }
    }
    if (BWD) {
#pragma unroll
      for (int q = 0; q < NC; ++q) dz_s[t][q] = own ? z[q] : 0.f;
      __syncthreads();   // dz_s complete
      // head weight gradient: thread owns channels 2cp, 2cp+1 over rows grp, grp+8, ...
      const uint32_t* tw = reinterpret_cast<const uint32_t*>(tile);
      for (int r = grp; r < nv; r += 8) {
        const uint32_t pr = tw[r * 32 + cp];
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pr));
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          const float d = dz_s[r][q];
          acc[NC + 2 * q] += d * a.x;
          acc[NC + 2 * q + 1] += d * a.y;
        }
      }
      __syncthreads();   // all tile reads done: each thread now rewrites its own row as dact
      if (own) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int jj = (j + t) & 7;
          uint4& u = tile[t * 8 + jj];
          const uint4 uv = u;
          const uint32_t av[4] = {uv.x, uv.y, uv.z, uv.w};
          uint32_t ov[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&av[e]));
            const float* wr = w_s + jj * kGrp + 2 * e * NC;
            float d0 = 0.f, d1 = 0.f;
#pragma unroll
            for (int q = 0; q < NC; ++q) {
              d0 += z[q] * wr[q];
              d1 += z[q] * wr[NC + q];
            }
            if (relu) {   // fused ReLU backward (act is the ReLU output)
              if (!(a.x > 0.f)) d0 = 0.f;
              if (!(a.y > 0.f)) d1 = 0.f;
            }
            __nv_bfloat162 h = __floats2bfloat162_rn(d0, d1);
            ov[e] = *reinterpret_cast<uint32_t*>(&h);
          }
          u = make_uint4(ov[0], ov[1], ov[2], ov[3]);
        }
      }
      fence_proxy_async_smem();   // generic-proxy writes -> bulk-copy reads
    }
    __syncthreads();   // tile consumed (FWD) / rewritten (BWD)
    if (BWD && t == 0) {
      bulk_store(dact + base * C, tile, (uint32_t)nv * 128);
      tma_store_commit();
    }
    if (BWD && bn_part) {   // BN-backward sums over the rewritten tile (as stored)
      const uint32_t* tw = reinterpret_cast<const uint32_t*>(tile);
      const uint32_t* xw = reinterpret_cast<const uint32_t*>(bnx + base * C);
      for (int r = grp; r < nv; r += 8) {
        const uint32_t dp = tw[r * 32 + cp], xp = xw[r * 32 + cp];
        const float2 d = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&dp));
        const float2 xv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xp));
        bsum[0] += d.x;
        bsum[1] += d.y;
        bsum[2] += d.x * ((xv.x - bm[0]) * br[0]);
        bsum[3] += d.y * ((xv.y - bm[1]) * br[1]);
      }
      __syncthreads();   // the tile is refilled by the next prefetch
    }
  }
  if (t == 0) tma_store_wait<0>();
  __syncthreads();
  float* red = reinterpret_cast<float*>(tiles);   // reuse the tiles for the block reduction
  const int lane = t & 31, warp = t >> 5;
  if (!BWD) {
#pragma unroll
    for (int j = 0; j < 3 * NC; ++j) {
      float v = acc[j];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp * 3 * NC + j] = v;
    }
    __syncthreads();
    if (t < 3 * NC) {
      float v = 0.f;
      for (int w = 0; w < kLT / 32; ++w) v += red[w * 3 * NC + t];
      part[(int64_t)blockIdx.x * 3 * NC + t] = v;
    }
  } else {
    constexpr int stride = NC * C + NC;
    // gw partials: red[grp][k*C + c]; gb partials: red[8*NC*C + warp*NC + k]
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      red[grp * NC * C + q * C + 2 * cp] = acc[NC + 2 * q];
      red[grp * NC * C + q * C + 2 * cp + 1] = acc[NC + 2 * q + 1];
      float v = acc[q];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[8 * NC * C + warp * NC + q] = v;
    }
    __syncthreads();
    for (int i = t; i < stride; i += kLT) {
      float v = 0.f;
      if (i < NC * C)
        for (int gq = 0; gq < 8; ++gq) v += red[gq * NC * C + i];
      else
        for (int w = 0; w < kLT / 32; ++w) v += red[8 * NC * C + w * NC + (i - NC * C)];
      part[(int64_t)blockIdx.x * stride + i] = v;
    }
    if (bn_part) {
      __syncthreads();
      float* bred = red + 8 * NC * C + 8 * NC;   // [grp][4][32]
#pragma unroll
      for (int q = 0; q < 4; ++q) bred[(grp * 4 + q) * 32 + cp] = bsum[q];
      __syncthreads();
      if (t < 2 * C) {   // t = which * 64 + c
        const int which = t / C, c = t % C, q = which * 2 + (c & 1), l = c >> 1;
        float v = 0.f;
        for (int gq = 0; gq < 8; ++gq) v += bred[(gq * 4 + q) * 32 + l];
        bn_part[(int64_t)blockIdx.x * 2 * C + t] = v;
      }
    }
  }
}

// Octet variants (bf16, C0 = 64, no smem staging): 8 lanes per voxel, lane o = channels
// 8o..8o+7, so a warp reads 4 consecutive voxel rows (512 B) per 16-byte load and 4
// iterations of loads are in flight per thread.  The head weights of a lane's 8 channels
// live in registers; logits are reduced across the octet with 3 shuffles per class.  The
// backward keeps its head-gradient partials (8 channels x NC) in registers too.
constexpr int kLO = 256;   // threads per block
constexpr int kLU = 4;     // iterations of loads in flight

template <int NC, bool BWD>
__global__ void __launch_bounds__(kLO, 2) k_loss_oct(
    const __nv_bfloat16* __restrict__ act, const uint8_t* __restrict__ labels,
    const float* __restrict__ hw, const float* __restrict__ hb, const double* __restrict__ dice,
    __nv_bfloat16* __restrict__ dact, float* __restrict__ part, int64_t nvox, double eps,
    int relu) {
  constexpr int C = 64;
  __shared__ float red[kLO / 32][8][BWD ? 8 * NC + NC : 3 * NC];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, o = lane & 7, vsub = lane >> 3;
  float w[NC][8], bias[NC], cA[NC], cB[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    bias[k] = hb[k];
#pragma unroll
    for (int j = 0; j < 8; ++j) w[k][j] = hw[k * C + 8 * o + j];
    if (BWD) {
      const double I = dice[k], P = dice[NC + k], G = dice[2 * NC + k];
      const double den = P + G + eps;
      cA[k] = (float)(-(2.0 / NC) / den);
      cB[k] = (float)((1.0 / NC) * (2.0 * I + eps) / (den * den));
    }
  }
  constexpr int kAcc = BWD ? 8 * NC + NC : 3 * NC;   // BWD: gw[k][8], gb[k] ; FWD: I,P,G
  float acc[kAcc];
#pragma unroll
  for (int j = 0; j < kAcc; ++j) acc[j] = 0.f;
  const uint4* src = reinterpret_cast<const uint4*>(act);
  uint4* dst = reinterpret_cast<uint4*>(dact);
  // voxel of (iteration it, thread): 4 voxels per warp, 32 per block
  const int64_t vstep = (int64_t)gridDim.x * (kLO / 8);
  for (int64_t v0 = (int64_t)blockIdx.x * (kLO / 8) + warp * 4 + vsub; v0 < nvox;
       v0 += kLU * vstep) {
    uint4 in[kLU];
    int lab[kLU];
#pragma unroll
    for (int u = 0; u < kLU; ++u) {
      const int64_t v = v0 + u * vstep;
      in[u] = v < nvox ? __ldg(src + v * 8 + o) : make_uint4(0u, 0u, 0u, 0u);
      lab[u] = v < nvox ? labels[v] : -1;
    }
#pragma unroll
    for (int u = 0; u < kLU; ++u) {
      const int64_t v = v0 + u * vstep;
      const bool ok = v < nvox;   // uniform across the octet
      float a[8];
      {
        const uint32_t wv[4] = {in[u].x, in[u].y, in[u].z, in[u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e]));
          a[2 * e] = f.x;
          a[2 * e + 1] = f.y;
        }
      }
      float z[NC];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) s += a[j] * w[k][j];
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        z[k] = s + bias[k];
      }
      float mx = -INFINITY;
#pragma unroll
      for (int k = 0; k < NC; ++k) mx = fmaxf(mx, z[k]);
      float se = 0.f;
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        z[k] = __expf(z[k] - mx);
        se += z[k];
      }
      const float inv = 1.f / se;
      const int g = lab[u];
      if (!BWD) {
        if (ok && o == 0) {
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            const float pk = z[k] * inv;
            acc[k] += (g == k) ? pk : 0.f;
            acc[NC + k] += pk;
            acc[2 * NC + k] += (g == k) ? 1.f : 0.f;
          }
        }
      } else if (ok) {
        float dp[NC], dot = 0.f;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          z[k] *= inv;
          dp[k] = cA[k] * (g == k ? 1.f : 0.f) + cB[k];
          dot += z[k] * dp[k];
        }
#pragma unroll
        for (int k = 0; k < NC; ++k) z[k] = z[k] * (dp[k] - dot);   // dlogit
        uint32_t ov[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float d0 = 0.f, d1 = 0.f;
#pragma unroll
          for (int k = 0; k < NC; ++k) {
            d0 += z[k] * w[k][2 * e];
            d1 += z[k] * w[k][2 * e + 1];
          }
          if (relu) {   // fused ReLU backward (act is the ReLU output)
            if (!(a[2 * e] > 0.f)) d0 = 0.f;
            if (!(a[2 * e + 1] > 0.f)) d1 = 0.f;
          }
          __nv_bfloat162 h = __floats2bfloat162_rn(d0, d1);
          ov[e] = *reinterpret_cast<uint32_t*>(&h);
        }
        dst[v * 8 + o] = make_uint4(ov[0], ov[1], ov[2], ov[3]);
#pragma unroll
        for (int k = 0; k < NC; ++k) {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[k * 8 + j] += z[k] * a[j];
          if (o == 0) acc[8 * NC + k] += z[k];
        }
      }
    }
  }
  // block reduction: across the 4 voxel lanes of an octet position, then across warps
#pragma unroll
  for (int j = 0; j < kAcc; ++j) {
    float v = acc[j];
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    if (vsub == 0) red[warp][o][j] = v;
  }
  __syncthreads();
  if (!BWD) {
    if (t < 3 * NC) {
      float v = 0.f;
      for (int wq = 0; wq < kLO / 32; ++wq) v += red[wq][0][t];
      part[(int64_t)blockIdx.x * 3 * NC + t] = v;
    }
  } else {
    constexpr int stride = NC * C + NC;
    for (int i = t; i < stride; i += kLO) {
      float v = 0.f;
      if (i < NC * C) {   // gw[k][c], c = 8 oo + j
        const int k = i / C, c = i % C, oo = c / 8, j = c % 8;
        for (int wq = 0; wq < kLO / 32; ++wq) v += red[wq][oo][k * 8 + j];
      } else {
        for (int wq = 0; wq < kLO / 32; ++wq) v += red[wq][0][8 * NC + (i - NC * C)];
      }
      part[(int64_t)blockIdx.x * stride + i] = v;
    }
  }
}

__global__ void k_sum_parts(const float* __restrict__ part, int nparts, int stride,
                            float* __restrict__ out_a, int na, float* __restrict__ out_b) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= stride) return;
  double s = 0;
  for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * stride + i];
  if (i < na) out_a[i] = (float)s;
  else out_b[i - na] = (float)s;
}

// ------------------------------------------------------------------ optimizer
__device__ __forceinline__ float adam_one(float& p, float g, float& m, float& v, float lr, float b1,
                                          float b2, float eps, float c1, float c2) {
  m = b1 * m + (1.f - b1) * g;
  v = b2 * v + (1.f - b2) * g * g;
  p = p - lr * (m / c1) / (sqrtf(v / c2) + eps);
  return p;
}

// Adam over a (bucket) range; 16-byte vectors for the aligned body, scalars for the
// unaligned head/tail (a bucket starts at an arbitrary element offset).
__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, __nv_bfloat16* __restrict__ pb, int64_t n, float lr,
                       float b1, float b2, float eps, const float* __restrict__ corr) {
  const float c1 = corr[0], c2 = corr[1];   // bias corrections 1 - beta^t (per step)
  int64_t head = (int64_t)((16 - ((uintptr_t)p & 15)) & 15) / 4;
  if (head > n) head = n;
  const int64_t n4 = (n - head) / 4;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  float4* p4 = reinterpret_cast<float4*>(p + head);
  const float4* g4 = reinterpret_cast<const float4*>(g + head);
  float4* m4 = reinterpret_cast<float4*>(m + head);
  float4* v4 = reinterpret_cast<float4*>(v + head);
  for (int64_t i = tid; i < n4; i += nth) {
    float4 pi = p4[i], gi = g4[i], mi = m4[i], vi = v4[i];
    adam_one(pi.x, gi.x, mi.x, vi.x, lr, b1, b2, eps, c1, c2);
    adam_one(pi.y, gi.y, mi.y, vi.y, lr, b1, b2, eps, c1, c2);
    adam_one(pi.z, gi.z, mi.z, vi.z, lr, b1, b2, eps, c1, c2);
    adam_one(pi.w, gi.w, mi.w, vi.w, lr, b1, b2, eps, c1, c2);
    p4[i] = pi;
    m4[i] = mi;
    v4[i] = vi;
    if (pb) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(pi.x, pi.y), hi = __floats2bfloat162_rn(pi.z, pi.w);
      __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(pb + head + 4 * i);
      d[0] = lo;   // pb + head is 4-byte aligned: bf16 copy offsets equal fp32 offsets
      d[1] = hi;
    }
  }
  // scalar head [0, head) and tail [head + 4 n4, n)
  const int64_t ns = head + (n - head - 4 * n4);
  for (int64_t j = tid; j < ns; j += nth) {
    const int64_t i = j < head ? j : head + 4 * n4 + (j - head);
    float pi = p[i], mi = m[i], vi = v[i];
    adam_one(pi, g[i], mi, vi, lr, b1, b2, eps, c1, c2);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
    if (pb) pb[i] = __float2bfloat16(pi);
  }
}

__global__ void k_cast(const float* __restrict__ p, __nv_bfloat16* __restrict__ pb, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    pb[i] = __float2bfloat16(p[i]);
}

__global__ void k_scale(float* __restrict__ g, int64_t n, float s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    g[i] *= s;
}

}  // namespace

// ================================================================== launchers
cudaError_t input_ncdhw(cudaStream_t s, int dtype, const float* src, void* dst, int N, int C,
                        int D, int H, int W, int Cdst, const int* aug) {
  int64_t vox = (int64_t)N * D * H * W;
  DISPATCH_T(dtype, k_input_ncdhw<T><<<grid_for(vox), kT, 0, s>>>(src, (T*)dst, N, C, D, H, W,
                                                                   Cdst, aug));
  return cudaGetLastError();
}

cudaError_t labels_aug(cudaStream_t s, const uint8_t* src, uint8_t* dst, int N, int D, int H,
                       int W, const int* aug) {
  k_labels_aug<<<grid_for((int64_t)N * D * H * W), kT, 0, s>>>(src, dst, N, D, H, W, aug);
  return cudaGetLastError();
}

cudaError_t pad_channels(cudaStream_t s, int dtype, const void* src, void* dst, int64_t vox,
                         int C, int Cdst) {
  if (Cdst % 8 == 0) {
    DISPATCH_T(dtype, k_pad_v8<T><<<grid_for(vox * (Cdst / 8)), kT, 0, s>>>(
                          (const T*)src, (T*)dst, vox, C, Cdst));
    return cudaGetLastError();
  }
  DISPATCH_T(dtype, k_pad<T><<<grid_for(vox), kT, 0, s>>>((const T*)src, (T*)dst, vox, C, Cdst));
  return cudaGetLastError();
}

int conv_stat_parts_direct(const ConvShape& sh) {
  return chan_sum_blocks((int64_t)sh.N * sh.D * sh.H * sh.W, sh.Cout);
}

// Channel statistics of a conv output computed by a separate pass (direct path).
cudaError_t chan_stats(cudaStream_t s, int dtype, const void* y, float* part, int64_t vox, int C,
                       int blocks) {
  cudaError_t e;
  DISPATCH_T(dtype, e = launch_chan_sums<T>(s, (const T*)y, (const T*)nullptr, nullptr, part, vox,
                                            C, 0, blocks));
  return e;
}

cudaError_t bn_stats_finalize(cudaStream_t s, const float* part, int nparts, int C, double count,
                              float* stat, double eps) {
  k_bn_finalize<<<(C + 31) / 32, 32 * kFinLanes, 0, s>>>(part, nparts, C, count, stat, eps);
  return cudaGetLastError();
}

cudaError_t norm_act(cudaStream_t s, int dtype, const void* x, const float* stat,
                     const float* gamma, const float* beta, void* norm, void* act, int64_t vox,
                     int C) {
  int64_t n = vox * C;
  if (dtype == 2 && C % 8 == 0) {
    k_norm_act_v8<<<grid_for(n / 8), kT, 2 * C * sizeof(float), s>>>(
        (const uint4*)x, stat, gamma, beta, (uint4*)norm, (uint4*)act, n / 8, C);
  } else {
    DISPATCH_T(dtype, k_norm_act<T><<<grid_for(n), kT, 0, s>>>((const T*)x, stat, gamma, beta,
                                                               (T*)norm, (T*)act, n, C));
  }
  return cudaGetLastError();
}

// BN apply + ReLU of the layer feeding the head, fused with the head's forward: each lane
// owns 8 channels of one voxel (C = 64: an octet of consecutive lanes per voxel), writes
// the ReLU output, and the octet reduces its 8-channel partial logits by shuffles; lane 0
// of the octet adds the voxel's softmax to the Dice partials (I, P, G per class).  The
// loss forward then only finalizes the partial rows -- the act tensor is not re-read.
template <int NC>
__global__ void __launch_bounds__(256) k_norm_act_loss(
    const uint4* __restrict__ x, const float* __restrict__ stat, const float* __restrict__ gamma,
    const float* __restrict__ beta, uint4* __restrict__ norm, uint4* __restrict__ act,
    const uint8_t* __restrict__ labels,
    const float* __restrict__ hw, const float* __restrict__ hb, float* __restrict__ part,
    int64_t nvox) {
  constexpr int C = 64;
  __shared__ float red[8][3 * NC];
  const int t = threadIdx.x, lane = t & 31, o = lane & 7;
  float a[8], b[8], w[NC][8], bias[NC], acc[3 * NC];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = 8 * o + j;
    a[j] = stat[C + c] * gamma[c];
    b[j] = beta[c] - stat[c] * a[j];
  }
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    bias[k] = hb[k];
#pragma unroll
    for (int j = 0; j < 8; ++j) w[k][j] = hw[k * C + 8 * o + j];
  }
#pragma unroll
  for (int j = 0; j < 3 * NC; ++j) acc[j] = 0.f;
  const int64_t nvec = nvox * 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;   // multiple of 8: o is fixed
  constexpr int kU = 4;
  // warp-uniform trip count (the octet shuffles need every lane): lane 0's index decides
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + t; i0 - lane < nvec; i0 += kU * stride) {
    uint4 in[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * stride;
      in[u] = i < nvec ? __ldg(x + i) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * stride;
      const bool ok = i < nvec;   // uniform across the octet (nvec % 8 == 0)
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&in[u]);
      uint4 oa, on;
      __nv_bfloat162* ha = reinterpret_cast<__nv_bfloat162*>(&oa);
      __nv_bfloat162* hn = reinterpret_cast<__nv_bfloat162*>(&on);
      float r[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        const float y0 = f.x * a[2 * j] + b[2 * j], y1 = f.y * a[2 * j + 1] + b[2 * j + 1];
        hn[j] = __floats2bfloat162_rn(y0, y1);
        ha[j] = __floats2bfloat162_rn(y0 > 0.f ? y0 : 0.f, y1 > 0.f ? y1 : 0.f);
        const float2 q = __bfloat1622float2(ha[j]);   // the head sees the stored values
        r[2 * j] = q.x;
        r[2 * j + 1] = q.y;
      }
      if (ok) {
        act[i] = oa;
        if (norm) norm[i] = on;
      }
      float z[NC];
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        float sz = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) sz += r[j] * w[k][j];
        sz += __shfl_xor_sync(0xffffffffu, sz, 1);
        sz += __shfl_xor_sync(0xffffffffu, sz, 2);
        sz += __shfl_xor_sync(0xffffffffu, sz, 4);
        z[k] = sz + bias[k];
      }
      if (ok && o == 0) {
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < NC; ++k) mx = fmaxf(mx, z[k]);
        float se = 0.f;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          z[k] = __expf(z[k] - mx);
          se += z[k];
        }
        const float inv = 1.f / se;
        const int g = labels[i / 8];
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          const float pk = z[k] * inv;
          acc[k] += (g == k) ? pk : 0.f;
          acc[NC + k] += pk;
          acc[2 * NC + k] += (g == k) ? 1.f : 0.f;
        }
      }
    }
  }
  const int warp = t >> 5;
#pragma unroll
  for (int j = 0; j < 3 * NC; ++j) {
    float v = acc[j];
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp][j] = v;
  }
  __syncthreads();
  if (t < 3 * NC) {
    float v = 0.f;
    for (int wq = 0; wq < 8; ++wq) v += red[wq][t];
    part[(int64_t)blockIdx.x * 3 * NC + t] = v;
  }
}

int norm_act_loss_parts(int64_t vox) { return grid_for(vox); }   // vox * 8 vectors / 256

cudaError_t norm_act_loss(cudaStream_t s, const void* x, const float* stat, const float* gamma,
                          const float* beta, void* norm, void* act, const uint8_t* labels,
                          const float* hw, const float* hb, float* part, int64_t vox, int C,
                          int ncls, int* rows) {
  if (C != 64 || ncls < 2 || ncls > 8) return cudaErrorInvalidValue;
  const int grid = norm_act_loss_parts(vox);
#define NAL(NCV)                                                                        \
  if (ncls == NCV)                                                                      \
    k_norm_act_loss<NCV><<<grid, 256, 0, s>>>((const uint4*)x, stat, gamma, beta, (uint4*)norm, \
                                              (uint4*)act, \
                                              labels, hw, hb, part, vox);
  NAL(2) NAL(3) NAL(4) NAL(5) NAL(6) NAL(7) NAL(8)
#undef NAL
  if (rows) *rows = grid;
  return cudaGetLastError();
}

cudaError_t loss_finalize(cudaStream_t s, const float* part, int nparts, int ncls, double eps,
                          double* dice, float* loss) {
  k_loss_finalize<<<1, 32, 0, s>>>(part, nparts, ncls, eps, dice, loss);
  return cudaGetLastError();
}

cudaError_t relu_fwd(cudaStream_t s, int dtype, const void* x, void* y, int64_t n) {
  if (n % 8 == 0) {
    DISPATCH_T(dtype, k_relu_fwd_v8<T><<<grid_for(n / 8), kT, 0, s>>>((const T*)x, (T*)y, n / 8));
    return cudaGetLastError();
  }
  DISPATCH_T(dtype, k_relu_fwd<T><<<grid_for(n), kT, 0, s>>>((const T*)x, (T*)y, n));
  return cudaGetLastError();
}

cudaError_t relu_bwd(cudaStream_t s, int dtype, const void* dy, const void* y, void* dx,
                     int64_t n) {
  if (n % 8 == 0) {
    DISPATCH_T(dtype, k_relu_bwd_v8<T><<<grid_for(n / 8), kT, 0, s>>>((const T*)dy, (const T*)y,
                                                                      (T*)dx, n / 8));
    return cudaGetLastError();
  }
  DISPATCH_T(dtype, k_relu_bwd<T><<<grid_for(n), kT, 0, s>>>((const T*)dy, (const T*)y, (T*)dx, n));
  return cudaGetLastError();
}

int bn_bwd_parts(int64_t vox, int C) { return chan_sum_blocks(vox, C); }

// fused producers write one row per CTA: persistent conv kernels <= 148, the loss <= 296,
// the pool backward grid_for() <= 148 * 16
int bn_bwd_rows_max(int64_t vox, int C) { return std::max(bn_bwd_parts(vox, C), 148 * 16); }

cudaError_t bn_bwd_sums(cudaStream_t s, int dtype, const void* x, const void* dy,
                        const float* stat, float* part, int64_t vox, int C, int* rows) {
  const int nparts = bn_bwd_parts(vox, C);
  cudaError_t e;
  DISPATCH_T(dtype, e = launch_chan_sums<T>(s, (const T*)x, (const T*)dy, stat, part, vox, C, 1,
                                            nparts));
  if (rows) *rows = nparts;
  return e;
}

cudaError_t bn_bwd(cudaStream_t s, int dtype, const void* x, const void* dy, const float* stat,
                   const float* gamma, float* ggamma, float* gbeta, void* dx, float* part,
                   int64_t vox, int C, int npre) {
  int nparts = npre;
  cudaError_t e;
  if (npre <= 0) {   // (sum dy, sum dy*xhat) not precomputed by dy's producer
    e = bn_bwd_sums(s, dtype, x, dy, stat, part, vox, C, &nparts);
    if (e != cudaSuccess) return e;
  }
  float* coef = part + (int64_t)nparts * 2 * C;
  k_bn_bwd_finalize<<<(C + 31) / 32, 32 * kFinLanes, 0, s>>>(part, nparts, C, (double)vox, stat, gamma,
                                                    ggamma, gbeta, coef);
  int64_t n = vox * C;
  if (C % 8 == 0) {
    DISPATCH_T(dtype, k_bn_bwd_apply_v8<T><<<grid_for(n / 8), kT, 3 * C * sizeof(float), s>>>(
                          (const T*)x, (const T*)dy, stat, coef, (T*)dx, n / 8, C));
    return cudaGetLastError();
  }
  DISPATCH_T(dtype, k_bn_bwd_apply<T><<<grid_for(n), kT, 0, s>>>((const T*)x, (const T*)dy, stat,
                                                                 coef, (T*)dx, n, C));
  return cudaGetLastError();
}

cudaError_t pool_fwd(cudaStream_t s, int dtype, const void* x, void* y, int N, int D, int H, int W,
                     int C) {
  int64_t total = (int64_t)N * (D / 2) * (H / 2) * (W / 2) * C;
  if (C % 8 == 0) {
    DISPATCH_T(dtype, k_pool_fwd_v8<T><<<grid_for(total / 8), kT, 0, s>>>((const T*)x, (T*)y, N,
                                                                          D, H, W, C));
    return cudaGetLastError();
  }
  DISPATCH_T(dtype, k_pool_fwd<T><<<grid_for(total), kT, 0, s>>>((const T*)x, (T*)y, N, D, H, W,
                                                                 C));
  return cudaGetLastError();
}

cudaError_t pool_bwd(cudaStream_t s, int dtype, const void* x, const void* dy, const void* dcat,
                     int dcat_cs, int dcat_co, void* dx, int N, int D, int H, int W, int C,
                     int relu, const BnSums* bn) {
  int64_t total = (int64_t)N * (D / 2) * (H / 2) * (W / 2) * C;
  if (bn && bn->part) {
    if (dtype == 2 && C % 8 == 0 && C <= 1024 && dcat_cs % 8 == 0 && dcat_co % 8 == 0 &&
        kT % (C / 8) == 0) {
      const int grid = grid_for(total / 8);   // <= bn_bwd_rows_max
      k_pool_bwd_v8<__nv_bfloat16, true><<<grid, kT, kT * 16 * sizeof(float), s>>>(
          (const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)dcat, dcat_cs,
          dcat_co, (__nv_bfloat16*)dx, N, D, H, W, C, relu, (const __nv_bfloat16*)bn->x,
          bn->stat, bn->part);
      if (bn->rows) *bn->rows = grid;
      return cudaGetLastError();
    }
    if (bn->rows) *bn->rows = 0;   // caller runs the chan sums pass
  }
  if (dtype == 2 && C % 8 == 0 && dcat_cs % 8 == 0 && dcat_co % 8 == 0) {
    using B = __nv_bfloat16;
    k_pool_bwd_v8<B><<<grid_for(total / 8), kT, 0, s>>>(
        (const B*)x, (const B*)dy, (const B*)dcat, dcat_cs, dcat_co, (B*)dx, N, D, H, W, C, relu);
    return cudaGetLastError();
  }
  DISPATCH_T(dtype, k_pool_bwd<T><<<grid_for(total), kT, 0, s>>>(
                        (const T*)x, (const T*)dy, (const T*)dcat, dcat_cs, dcat_co, (T*)dx, N, D,
                        H, W, C, relu));
  return cudaGetLastError();
}

template <class T>
__global__ void k_copy_channels_v8(const T* __restrict__ src, T* __restrict__ y, int64_t vox,
                                   int C, int Cy, int co) {
  const int cv = C / 8;
  const int64_t total = vox * cv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / cv;
    const int c = (int)(i % cv) * 8;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + v * C + c);
    uint4* d4 = reinterpret_cast<uint4*>(y + v * Cy + co + c);
    constexpr int kWords = sizeof(T) * 8 / 16;
#pragma unroll
    for (int k = 0; k < kWords; ++k) d4[k] = s4[k];
  }
}

cudaError_t copy_channels(cudaStream_t s, int dtype, const void* src, void* y, int64_t vox, int C,
                          int Cy, int co) {
  if (C % 8 || Cy % 8 || co % 8) return cudaErrorInvalidValue;
  DISPATCH_T(dtype, k_copy_channels_v8<T><<<grid_for(vox * C / 8), kT, 0, s>>>(
                        (const T*)src, (T*)y, vox, C, Cy, co));
  return cudaGetLastError();
}

cudaError_t concat2(cudaStream_t s, int dtype, const void* a, const void* b, void* y, int64_t vox,
                    int Ca, int Cb) {
  if (Ca % 8 == 0 && Cb % 8 == 0) {
    DISPATCH_T(dtype, k_concat_v8<T><<<grid_for(vox * (Ca + Cb) / 8), kT, 0, s>>>(
                          (const T*)a, (const T*)b, (T*)y, vox, Ca, Cb));
    return cudaGetLastError();
  }
  DISPATCH_T(dtype, k_concat<T><<<grid_for(vox * (Ca + Cb)), kT, 0, s>>>(
                        (const T*)a, (const T*)b, (T*)y, vox, Ca, Cb));
  return cudaGetLastError();
}

int loss_parts(int64_t vox) {
  // one resident wave: the tiled kernel runs 2 blocks of 256 threads (64 KB tiles) per SM
  int64_t b = (vox + kLossWarps * 64 - 1) / (kLossWarps * 64);
  if (b < 1) b = 1;
  if (b > 148 * 2) b = 148 * 2;
  return (int)b;
}

cudaError_t loss_fwd(cudaStream_t s, int dtype, const void* act, const uint8_t* labels,
                     const float* hw, const float* hb, float* part, double* dice, float* loss,
                     int N, int64_t vox, int C, int ncls, double eps) {
  if (ncls > kMaxCls) return cudaErrorInvalidValue;
  int64_t nvox = (int64_t)N * vox;
  int nparts = loss_parts(nvox);
  size_t smem = (size_t)ncls * C * sizeof(float);
  // forward: the smem-tiled kernel measures faster (r01: 0.30 vs 0.43 ms at 192^3, the
  // octet kernel's per-voxel shuffles and redundant softmax dominate without a store)
  if (dtype == 2 && C == 64 && ncls >= 2 && ncls <= 8 && getenv("US_LOSS_OCT_FWD")) {
#define LOSS_FWD_O(NCV)                                                                  \
  if (ncls == NCV)                                                                       \
    k_loss_oct<NCV, false><<<nparts, kLO, 0, s>>>((const __nv_bfloat16*)act, labels, hw, hb, \
                                                  nullptr, nullptr, part, nvox, eps, 0);
    LOSS_FWD_O(2) LOSS_FWD_O(3) LOSS_FWD_O(4) LOSS_FWD_O(5) LOSS_FWD_O(6) LOSS_FWD_O(7)
    LOSS_FWD_O(8)
#undef LOSS_FWD_O
  } else if (dtype == 2 && C == 64 && ncls >= 2 && ncls <= 8) {
#define LOSS_FWD_T(NCV)                                                               \
  if (ncls == NCV) {                                                                   \
    static bool attr = false;                                                         \
    if (!attr) {                                                                      \
      cudaFuncSetAttribute(k_loss_tile<NCV, false>,                                    \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kLTileBytes); \
      attr = true;                                                                    \
    }                                                                                 \
    k_loss_tile<NCV, false><<<nparts, kLT, 2 * kLTileBytes, s>>>(                      \
        (const __nv_bfloat16*)act, labels, hw, hb, nullptr, nullptr, part, nvox, eps, 0);          \
  }
    LOSS_FWD_T(2) LOSS_FWD_T(3) LOSS_FWD_T(4) LOSS_FWD_T(5) LOSS_FWD_T(6) LOSS_FWD_T(7)
    LOSS_FWD_T(8)
#undef LOSS_FWD_T
  } else if (C % 8 == 0 && C <= kVC && ncls >= 2 && ncls <= 8) {
#define LOSS_FWD_NC(NCV)                                                              \
  if (ncls == NCV)                                                                    \
    DISPATCH_T(dtype, k_loss_fwd_v<T, NCV><<<nparts, kVWarps * 32, 0, s>>>(            \
                          (const T*)act, labels, hw, hb, part, nvox, C));
    LOSS_FWD_NC(2) LOSS_FWD_NC(3) LOSS_FWD_NC(4) LOSS_FWD_NC(5) LOSS_FWD_NC(6)
    LOSS_FWD_NC(7) LOSS_FWD_NC(8)
#undef LOSS_FWD_NC
  } else {
    DISPATCH_T(dtype, k_loss_fwd<T><<<nparts, kLossWarps * 32, smem, s>>>(
                          (const T*)act, labels, hw, hb, part, nvox, C, ncls));
  }
  k_loss_finalize<<<1, 32, 0, s>>>(part, nparts, ncls, eps, dice, loss);
  return cudaGetLastError();
}

cudaError_t loss_bwd(cudaStream_t s, int dtype, const void* act, const uint8_t* labels,
                     const float* hw, const float* hb, const double* dice, void* dact,
                     float* ghw, float* ghb, float* part, int N, int64_t vox, int C, int ncls,
                     double eps, int relu, const BnSums* bn) {
  if (ncls > kMaxCls) return cudaErrorInvalidValue;
  if (bn && bn->rows) *bn->rows = 0;   // only the tiled kernel fuses the BN sums
  // backward: the octet kernel (r01: 0.64 vs 0.75 ms for the tiled one); the tiled kernel
  // still serves fused BN sums
  if (dtype == 2 && C == 64 && ncls >= 2 && ncls <= 8 && !(bn && bn->part) &&
      !getenv("US_LOSS_TILE")) {
    const int64_t nvox_ = (int64_t)N * vox;
    const int nparts_ = loss_parts(nvox_);
    const int stride_ = ncls * C + ncls;
#define LOSS_BWD_O(NCV)                                                                  \
  if (ncls == NCV)                                                                       \
    k_loss_oct<NCV, true><<<nparts_, kLO, 0, s>>>((const __nv_bfloat16*)act, labels, hw, hb, \
                                                  dice, (__nv_bfloat16*)dact, part, nvox_, eps, \
                                                  relu);
    LOSS_BWD_O(2) LOSS_BWD_O(3) LOSS_BWD_O(4) LOSS_BWD_O(5) LOSS_BWD_O(6) LOSS_BWD_O(7)
    LOSS_BWD_O(8)
#undef LOSS_BWD_O
    k_sum_parts<<<(stride_ + 127) / 128, 128, 0, s>>>(part, nparts_, stride_, ghw, ncls * C,
                                                      ghb);
    return cudaGetLastError();
  }
  int64_t nvox = (int64_t)N * vox;
  int nparts = loss_parts(nvox);
  int stride = ncls * C + ncls;
  if (dtype == 2 && C == 64 && ncls >= 2 && ncls <= 8) {
#define LOSS_BWD_T(NCV)                                                               \
  if (ncls == NCV) {                                                                   \
    static bool attr = false;                                                         \
    if (!attr) {                                                                      \
      cudaFuncSetAttribute(k_loss_tile<NCV, true>,                                    \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kLTileBytes); \
      attr = true;                                                                    \
    }                                                                                 \
    k_loss_tile<NCV, true><<<nparts, kLT, 2 * kLTileBytes, s>>>(                      \
        (const __nv_bfloat16*)act, labels, hw, hb, dice, (__nv_bfloat16*)dact, part, nvox, eps, relu, \
        bn && bn->part ? (const __nv_bfloat16*)bn->x : nullptr, bn ? bn->stat : nullptr,          \
        bn ? bn->part : nullptr);          \
  }
    LOSS_BWD_T(2) LOSS_BWD_T(3) LOSS_BWD_T(4) LOSS_BWD_T(5) LOSS_BWD_T(6) LOSS_BWD_T(7)
    LOSS_BWD_T(8)
#undef LOSS_BWD_T
    if (bn && bn->part && bn->rows) *bn->rows = nparts;
    k_sum_parts<<<(stride + 127) / 128, 128, 0, s>>>(part, nparts, stride, ghw, ncls * C, ghb);
    return cudaGetLastError();
  }
  if (C % 8 == 0 && C <= kVC && ncls >= 2 && ncls <= 8) {
#define LOSS_BWD_NC(NCV)                                                              \
  if (ncls == NCV)                                                                    \
    DISPATCH_T(dtype, k_loss_bwd_v<T, NCV><<<nparts, kVWarps * 32, 0, s>>>(            \
                          (const T*)act, labels, hw, hb, dice, (T*)dact, part, nvox, C, eps,     \
                          relu));
    LOSS_BWD_NC(2) LOSS_BWD_NC(3) LOSS_BWD_NC(4) LOSS_BWD_NC(5) LOSS_BWD_NC(6)
    LOSS_BWD_NC(7) LOSS_BWD_NC(8)
#undef LOSS_BWD_NC
    k_sum_parts<<<(stride + 127) / 128, 128, 0, s>>>(part, nparts, stride, ghw, ncls * C, ghb);
    return cudaGetLastError();
  }
  size_t smem = (size_t)(ncls * C + kLossWarps * stride) * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t e;
    DISPATCH_T(dtype, e = cudaFuncSetAttribute(k_loss_bwd<T>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem));
    if (e != cudaSuccess) return e;
  }
  DISPATCH_T(dtype, k_loss_bwd<T><<<nparts, kLossWarps * 32, smem, s>>>(
                        (const T*)act, labels, hw, hb, dice, (T*)dact, part, nvox, C, ncls, eps,
                        relu));
  k_sum_parts<<<(stride + 127) / 128, 128, 0, s>>>(part, nparts, stride, ghw, ncls * C, ghb);
  return cudaGetLastError();
}

cudaError_t adam(cudaStream_t s, float* p, const float* g, float* m, float* v,
                 __nv_bfloat16* pb, int64_t n, float lr, float b1, float b2, float eps,
                 const float* corr) {
  k_adam<<<grid_for((n + 3) / 4, kT, 148 * 8), kT, 0, s>>>(p, g, m, v, pb, n, lr, b1, b2, eps,
                                                           corr);
  return cudaGetLastError();
}

cudaError_t cast_bf16(cudaStream_t s, const float* p, __nv_bfloat16* pb, int64_t n) {
  k_cast<<<grid_for(n, kT, 148 * 32), kT, 0, s>>>(p, pb, n);
  return cudaGetLastError();
}

cudaError_t scale_f32(cudaStream_t s, float* g, int64_t n, float scale) {
  k_scale<<<grid_for(n, kT, 148 * 32), kT, 0, s>>>(g, n, scale);
  return cudaGetLastError();
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace us
