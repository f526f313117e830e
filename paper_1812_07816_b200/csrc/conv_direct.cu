// Direct CUDA-core convolutions (fp32 accumulate) for the fp32 check mode and
// for layers whose channel counts the tensor-core path does not cover
// (channels not a multiple of 16, e.g. the base-8 oracle configuration).
// Weight layout: [Cout][27][Cin], tap = kd*9 + kh*3 + kw.
//   conv  (k3 s1 p1):            y[o]  = sum_t,ci x[o + t - 1] W[co][t][ci]
//   convT (k3 s2 p1 op1):        y[o]  = sum over (i, k) with o = 2i - 1 + k of x[i] W[co][k][ci]
// Backward passes are the exact adjoints (dgrad) and input x output-grad
// correlations (wgrad) of those definitions.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace us {
cudaError_t chan_stats(cudaStream_t s, int dtype, const void* y, float* part, int64_t vox, int C,
                       int blocks);

namespace {

constexpr int kT = 256;

__device__ __forceinline__ float ldf(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ldf(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}
__device__ __forceinline__ void stf(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void stf(__nv_bfloat16* p, int64_t i, float v) {
  p[i] = __float2bfloat16(v);
}

inline int grid_for(int64_t work) {
  int64_t b = (work + kT - 1) / kT;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return (int)b;
}

// Decompose a linear NDHWC element index over (n, z, y, x, c).
struct Pos {
  int n, z, y, x, c;
};
__device__ __forceinline__ Pos unflat(int64_t i, int D, int H, int W, int C) {
  Pos p;
  p.c = (int)(i % C); i /= C;
  p.x = (int)(i % W); i /= W;
  p.y = (int)(i % H); i /= H;
  p.z = (int)(i % D);
  p.n = (int)(i / D);
  return p;
}

template <class T, class WT>
__global__ void k_conv_fwd(const T* __restrict__ x, const WT* __restrict__ w, T* __restrict__ y,
                           ConvShape sh) {
  int64_t total = (int64_t)sh.N * sh.D * sh.H * sh.W * sh.Cout;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    Pos p = unflat(i, sh.D, sh.H, sh.W, sh.Cout);
    float acc = 0.f;
    for (int kd = 0; kd < 3; ++kd) {
      int z = p.z + kd - 1;
      if (z < 0 || z >= sh.D) continue;
      for (int kh = 0; kh < 3; ++kh) {
        int yy = p.y + kh - 1;
        if (yy < 0 || yy >= sh.H) continue;
        for (int kw = 0; kw < 3; ++kw) {
          int xx = p.x + kw - 1;
          if (xx < 0 || xx >= sh.W) continue;
          int64_t vi = (((int64_t)p.n * sh.D + z) * sh.H + yy) * sh.W + xx;
          const WT* wr = w + ((int64_t)p.c * 27 + kd * 9 + kh * 3 + kw) * sh.Cin;
          for (int ci = 0; ci < sh.Cin; ++ci)
            acc += ldf(x, vi * sh.x_cs + sh.x_co + ci) * ldf(wr, ci);
        }
      }
    }
    stf(y, i, acc);
  }
}

template <class T, class WT>
__global__ void k_conv_dgrad(const T* __restrict__ dy, const WT* __restrict__ w,
                             T* __restrict__ dx, ConvShape sh) {
  int64_t total = (int64_t)sh.N * sh.D * sh.H * sh.W * sh.Cin;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    Pos p = unflat(i, sh.D, sh.H, sh.W, sh.Cin);
    float acc = 0.f;
    for (int kd = 0; kd < 3; ++kd) {
      int z = p.z - kd + 1;
      if (z < 0 || z >= sh.D) continue;
      for (int kh = 0; kh < 3; ++kh) {
        int yy = p.y - kh + 1;
        if (yy < 0 || yy >= sh.H) continue;
        for (int kw = 0; kw < 3; ++kw) {
          int xx = p.x - kw + 1;
          if (xx < 0 || xx >= sh.W) continue;
          int64_t vo = (((int64_t)p.n * sh.D + z) * sh.H + yy) * sh.W + xx;
          int tap = kd * 9 + kh * 3 + kw;
          for (int co = 0; co < sh.Cout; ++co)
            acc += ldf(dy, vo * sh.dy_cs + sh.dy_co + co) *
                   ldf(w, ((int64_t)co * 27 + tap) * sh.Cin + p.c);
        }
      }
    }
    stf(dx, i, acc);
  }
}

// One block per (co, tap, ci) weight; threads reduce over voxels.
template <class T>
__global__ void k_conv_wgrad(const T* __restrict__ x, const T* __restrict__ dy,
                             float* __restrict__ gw, ConvShape sh) {
  int idx = blockIdx.x;
  int ci = idx % sh.Cin;
  int tap = (idx / sh.Cin) % 27;
  int co = idx / (sh.Cin * 27);
  int kd = tap / 9, kh = (tap / 3) % 3, kw = tap % 3;
  int64_t vox = (int64_t)sh.N * sh.D * sh.H * sh.W;
  float acc = 0.f;
  for (int64_t v = threadIdx.x; v < vox; v += blockDim.x) {
    int64_t r = v;
    int xx = (int)(r % sh.W); r /= sh.W;
    int yy = (int)(r % sh.H); r /= sh.H;
    int z = (int)(r % sh.D);
    int n = (int)(r / sh.D);
    int zi = z + kd - 1, yi = yy + kh - 1, xi = xx + kw - 1;
    if (zi < 0 || zi >= sh.D || yi < 0 || yi >= sh.H || xi < 0 || xi >= sh.W) continue;
    int64_t vi = (((int64_t)n * sh.D + zi) * sh.H + yi) * sh.W + xi;
    acc += ldf(x, vi * sh.x_cs + sh.x_co + ci) * ldf(dy, v * sh.dy_cs + sh.dy_co + co);
  }
  __shared__ float red[kT];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) gw[idx] = red[0];
}

// Transposed conv: low-res grid (D,H,W) -> (2D,2H,2W).
template <class T, class WT>
__global__ void k_convt_fwd(const T* __restrict__ x, const WT* __restrict__ w, T* __restrict__ y,
                            ConvShape sh) {
  int D2 = 2 * sh.D, H2 = 2 * sh.H, W2 = 2 * sh.W;
  int64_t total = (int64_t)sh.N * D2 * H2 * W2 * sh.Cout;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    Pos p = unflat(i, D2, H2, W2, sh.Cout);
    float acc = 0.f;
    for (int kd = 0; kd < 3; ++kd) {
      int tz = p.z + 1 - kd;
      if (tz < 0 || (tz & 1) || (tz >> 1) >= sh.D) continue;
      for (int kh = 0; kh < 3; ++kh) {
        int ty = p.y + 1 - kh;
        if (ty < 0 || (ty & 1) || (ty >> 1) >= sh.H) continue;
        for (int kw = 0; kw < 3; ++kw) {
          int tx = p.x + 1 - kw;
          if (tx < 0 || (tx & 1) || (tx >> 1) >= sh.W) continue;
          int64_t vi = (((int64_t)p.n * sh.D + (tz >> 1)) * sh.H + (ty >> 1)) * sh.W + (tx >> 1);
          const WT* wr = w + ((int64_t)p.c * 27 + kd * 9 + kh * 3 + kw) * sh.Cin;
          for (int ci = 0; ci < sh.Cin; ++ci) acc += ldf(x, vi * sh.Cin + ci) * ldf(wr, ci);
        }
      }
    }
    stf(y, i, acc);
  }
}

template <class T, class WT>
__global__ void k_convt_dgrad(const T* __restrict__ dy, const WT* __restrict__ w,
                              T* __restrict__ dx, ConvShape sh) {
  int D2 = 2 * sh.D, H2 = 2 * sh.H, W2 = 2 * sh.W;
  int64_t total = (int64_t)sh.N * sh.D * sh.H * sh.W * sh.Cin;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    Pos p = unflat(i, sh.D, sh.H, sh.W, sh.Cin);
    float acc = 0.f;
    for (int kd = 0; kd < 3; ++kd) {
      int oz = 2 * p.z - 1 + kd;
      if (oz < 0 || oz >= D2) continue;
      for (int kh = 0; kh < 3; ++kh) {
        int oy = 2 * p.y - 1 + kh;
        if (oy < 0 || oy >= H2) continue;
        for (int kw = 0; kw < 3; ++kw) {
          int ox = 2 * p.x - 1 + kw;
          if (ox < 0 || ox >= W2) continue;
          int64_t vo = (((int64_t)p.n * D2 + oz) * H2 + oy) * W2 + ox;
          int tap = kd * 9 + kh * 3 + kw;
          for (int co = 0; co < sh.Cout; ++co)
            acc += ldf(dy, vo * sh.dy_cs + sh.dy_co + co) *
                   ldf(w, ((int64_t)co * 27 + tap) * sh.Cin + p.c);
        }
      }
    }
    stf(dx, i, acc);
  }
}

template <class T>
__global__ void k_convt_wgrad(const T* __restrict__ x, const T* __restrict__ dy,
                              float* __restrict__ gw, ConvShape sh) {
  int idx = blockIdx.x;
  int ci = idx % sh.Cin;
  int tap = (idx / sh.Cin) % 27;
  int co = idx / (sh.Cin * 27);
  int kd = tap / 9, kh = (tap / 3) % 3, kw = tap % 3;
  int D2 = 2 * sh.D, H2 = 2 * sh.H, W2 = 2 * sh.W;
  int64_t vox = (int64_t)sh.N * sh.D * sh.H * sh.W;
  float acc = 0.f;
  for (int64_t v = threadIdx.x; v < vox; v += blockDim.x) {
    int64_t r = v;
    int xx = (int)(r % sh.W); r /= sh.W;
    int yy = (int)(r % sh.H); r /= sh.H;
    int z = (int)(r % sh.D);
    int n = (int)(r / sh.D);
    int oz = 2 * z - 1 + kd, oy = 2 * yy - 1 + kh, ox = 2 * xx - 1 + kw;
    if (oz < 0 || oz >= D2 || oy < 0 || oy >= H2 || ox < 0 || ox >= W2) continue;
    int64_t vo = (((int64_t)n * D2 + oz) * H2 + oy) * W2 + ox;
    acc += ldf(x, v * sh.Cin + ci) * ldf(dy, vo * sh.dy_cs + sh.dy_co + co);
  }
  __shared__ float red[kT];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) gw[idx] = red[0];
}

}  // namespace

#define DISPATCH_TW(dtype, ...)                 \
  do {                                          \
    if ((dtype) == 2) {                         \
      using T = __nv_bfloat16;                  \
      using WT = __nv_bfloat16;                 \
      __VA_ARGS__;                              \
    } else {                                    \
      using T = float;                          \
      using WT = float;                         \
      __VA_ARGS__;                              \
    }                                           \
  } while (0)

cudaError_t conv_fwd_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* x,
                            const void* w, void* y, float* part, int nparts) {
  int64_t vox = (int64_t)sh.N * sh.D * sh.H * sh.W;
  DISPATCH_TW(dtype, k_conv_fwd<T, WT><<<grid_for(vox * sh.Cout), kT, 0, s>>>(
                         (const T*)x, (const WT*)w, (T*)y, sh));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !part) return e;
  return chan_stats(s, dtype, y, part, vox, sh.Cout, nparts);
}

cudaError_t conv_dgrad_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* dy,
                              const void* w, void* dx) {
  int64_t vox = (int64_t)sh.N * sh.D * sh.H * sh.W;
  DISPATCH_TW(dtype, k_conv_dgrad<T, WT><<<grid_for(vox * sh.Cin), kT, 0, s>>>(
                         (const T*)dy, (const WT*)w, (T*)dx, sh));
  return cudaGetLastError();
}

cudaError_t conv_wgrad_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* x,
                              const void* dy, float* gw) {
  int blocks = sh.Cout * 27 * sh.Cin;
  DISPATCH_TW(dtype, k_conv_wgrad<T><<<blocks, kT, 0, s>>>((const T*)x, (const T*)dy, gw, sh));
  return cudaGetLastError();
}

cudaError_t convt_fwd_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* x,
                             const void* w, void* y) {
  int64_t vox2 = (int64_t)sh.N * 8 * sh.D * sh.H * sh.W;
  DISPATCH_TW(dtype, k_convt_fwd<T, WT><<<grid_for(vox2 * sh.Cout), kT, 0, s>>>(
                         (const T*)x, (const WT*)w, (T*)y, sh));
  return cudaGetLastError();
}

cudaError_t convt_dgrad_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* dy,
                               const void* w, void* dx) {
  int64_t vox = (int64_t)sh.N * sh.D * sh.H * sh.W;
  DISPATCH_TW(dtype, k_convt_dgrad<T, WT><<<grid_for(vox * sh.Cin), kT, 0, s>>>(
                         (const T*)dy, (const WT*)w, (T*)dx, sh));
  return cudaGetLastError();
}

cudaError_t convt_wgrad_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* x,
                               const void* dy, float* gw) {
  int blocks = sh.Cout * 27 * sh.Cin;
  DISPATCH_TW(dtype, k_convt_wgrad<T><<<blocks, kT, 0, s>>>((const T*)x, (const T*)dy, gw, sh));
  return cudaGetLastError();
}

}  // namespace us
