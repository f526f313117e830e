// Implicit-GEMM 3x3x3 convolutions on the 5th-generation tensor cores.
//
// Data layout: activations NDHWC bf16, weights [Cout][27][Cin] bf16.
//
// k_igemm  -- output-stationary implicit GEMM (per-tap operands): conv fprop / dgrad on
//             small grids (split-K over taps), convT dgrad (8 parity views) and the
//             sub-pixel convT fprop (one GEMM for all 8 output parity classes, per-n-tile
//             tap masks; convT_subpixel_mode).
//   GEMM M = voxels of an output-space grid, tiled as a 128-voxel box; N = output
//   channels (tile BN <= 256); K = taps x input channels.  Per (tap, channel chunk) a
//   warp-specialised pipeline stages A (the tap-shifted box, one 5-D TMA load, zero fill
//   = padding) and B (the tap's weight slice), and one elected thread issues
//   tcgen05.mma (M=128 or a CTA pair's 256, N=BN, K=16) into double-buffered fp32 TMEM.
//   Four epilogue warps drain TMEM with tcgen05.ld, convert, store NDHWC (strided /
//   scattered for the transposed conv) and accumulate BatchNorm sum / sum^2.
// k_igemm_halo / k_halo_z2 -- conv fprop / dgrad on wide grids: the input halo of a tile
//   is staged once and the 27 taps are descriptor views of it (z2: two output planes per
//   tile, 1-voxel-deep halo slabs in a ring, 64 output channels).
// k_wgrad_hv / k_wgrad_halo / k_wgrad_halo_a / k_wgrad -- weight gradients (K = voxels),
//   fp32 partials per K split reduced in a fixed order: halo-view (both operands shifted
//   views, 128x192x16 MMAs), tap-pair halo (Cout 64), 8-tap halo, per-tap.
// k_stem_* -- the 4-channel input layer (in-smem im2col).
//
// Roles: warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
// warps 2..5 = epilogue.  Persistent grid of min(tiles, #SMs) CTAs (or CTA pairs).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "kernels.h"
#include "sm100.cuh"

namespace us {
namespace {

constexpr int kThreads = 192;
constexpr int kSmemBudget = 190 * 1024;
constexpr int kIgEpiBytes = 4 * 32 * 128;   // k_igemm: per epilogue warp, 32 rows x 128 B

struct Maps {
  CUtensorMap a[9];   // activations: igemm uses a[0..7] (parity views), wgrad a[0] = X, a[1..8] = dY
  CUtensorMap b;      // weights (igemm)
  CUtensorMap x2;     // dual-source conv input (a concat never materialised): channels
  int split_c;        // [split_c, Cin) of the input come from x2; 0 = one source
};

// The tensor map a load through activation map `idx` at channel `c` must use: the conv
// input's channels at or past split_c live in its second source (c is rebased to it).
__device__ __forceinline__ const CUtensorMap* act_map(const Maps& m, int idx, int& c) {
  if (idx == 0 && m.split_c > 0 && c >= m.split_c) {
    c -= m.split_c;
    return &m.x2;
  }
  return &m.a[idx];
}

struct Taps {
  int8_t dx[27], dy[27], dz[27], map[27];
  int16_t w[27];
};

struct IgParams {
  Taps taps;
  int n_taps;
  int Nb, Md, Mh, Mw;          // GEMM-M grid (batch, D, H, W)
  int bd, bh, bw;              // voxel box of one M tile (bd*bh*bw == 128)
  int td, th, tw;              // tiles per dim
  int m_tiles, n_tiles;
  int k_chunks;                // input channel chunks per tap
  int a_c0;                    // channel offset of A inside its tensor (slices)
  int w_cin;                   // Cin of the weight layout (tap stride)
  int b_n0;                    // (unused, reserved)
  __nv_bfloat16* out;
  const __nv_bfloat16* mask;   // fused ReLU backward: out = acc * (mask > 0), mask laid out like out
  const __nv_bfloat16* bnx;    // dgrad: fused BatchNorm-backward sums -- the BN input, laid out
                               // like out with Nout channels; stats then receives per-CTA rows
                               // (sum d, sum d * xhat), xhat = (bnx - mean) * rstd
  const float* bn_stat;        // mean[Nout], rstd[Nout] of that BN
  int out_cs, out_co;
  int oD, oH, oW, os, ooz, ooy, oox;
  float* stats;                // [gridDim.x][2][Nout] or null ([m_tiles][2][Nout] if split)
  int Nout;
  int splits;                  // split-K over taps (small grids); 1 = off
  float* split_part;           // [splits][m_tiles][n_tiles][128][BN] fp32 partial tiles
  int scatter_c;               // > 0: sub-pixel convT -- GEMM column p*scatter_c + co goes to
                               // output voxel 2v + p (pz,py,px bits), channel co
  int ig_pair;                 // conv fprop: run as a CTA pair (see k_igemm PAIR)
  int staged_epi;               // 1: coalesced epilogue stores through shared memory (set by
                               // dispatch_ig; US_IG_STAGED=0 turns it off)
  int sp_direct;                // sub-pixel convT: 1 = per-class weight rows straight from W
                               // (exact 27 blocks); 0 = one box of the re-laid W' (zero
                               // blocks included, full-N MMAs)
  uint8_t nt_mask[32];         // sub-pixel convT: window taps n tile j uses (bit t); nonzero
                               // turns the tiles n-major so every CTA gets the same mix of
                               // short and long tiles
};

// Sub-pixel transposed conv (k3 s2 p1 op1): output parity class c = (pz, py, px) reads the
// 2x2x2 input window tap t = (dz, dy, dx) iff t's bits lie within c's (per axis: p = 0
// takes kernel tap 1 at d = 0; p = 1 takes tap 2 at d = 0 and tap 0 at d = 1), through
// kernel tap convt_ktap(t, c).  27 of the 64 (t, c) pairs are used.
__host__ __device__ __forceinline__ bool convt_uses(int t, int c) { return (t & ~c) == 0; }
__host__ __device__ __forceinline__ int convt_ktap(int t, int c) {
  int k = 0;
  for (int a = 2; a >= 0; --a) {
    const int p = (c >> a) & 1, d = (t >> a) & 1;
    k = k * 3 + (p == 0 ? 1 : (d ? 0 : 2));
  }
  return k;
}

__device__ __forceinline__ void ig_decode(const IgParams& p, int mt, int& n, int& x0, int& y0,
                                          int& z0) {
  int tx = mt % p.tw;
  int r = mt / p.tw;
  int ty = r % p.th;
  r /= p.th;
  int tz = r % p.td;
  n = r / p.td;
  x0 = tx * p.bw;
  y0 = ty * p.bh;
  z0 = tz * p.bd;
}

// Fused ReLU backward in a dgrad epilogue: zero v[j] where the ReLU output is not > 0.
__device__ __forceinline__ void apply_relu_mask(float (&v)[32], const __nv_bfloat16* m, int n) {
  const uint4* m4 = reinterpret_cast<const uint4*>(m);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (8 * q >= n) break;
    uint4 w = __ldg(m4 + q);
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      // bf16 > 0  <=>  sign bit clear and not +0
      if ((u[e] & 0x8000u) || !(u[e] & 0x7FFFu)) v[8 * q + 2 * e] = 0.f;
      if ((u[e] & 0x80000000u) || !(u[e] & 0x7FFF0000u)) v[8 * q + 2 * e + 1] = 0.f;
    }
  }
}

// 32 bf16 (64 bytes) into registers -- issued ahead of the TMEM load in the dgrad
// epilogues so the mask / BN-input latency overlaps it
__device__ __forceinline__ void load32_bf16(const __nv_bfloat16* p, uint4 (&r)[4]) {
  const uint4* p4 = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int q = 0; q < 4; ++q) r[q] = __ldg(p4 + q);
}
__device__ __forceinline__ void apply_relu_mask_reg(float (&v)[32], const uint4 (&m)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t u[4] = {m[q].x, m[q].y, m[q].z, m[q].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if ((u[e] & 0x8000u) || !(u[e] & 0x7FFFu)) v[8 * q + 2 * e] = 0.f;
      if ((u[e] & 0x80000000u) || !(u[e] & 0x7FFF0000u)) v[8 * q + 2 * e + 1] = 0.f;
    }
  }
}

// Column sums across the 32 lanes of a warp: on return lane j holds sum of v[j].
__device__ __forceinline__ float warp_colsum32(float (&v)[32]) {
  const unsigned full = 0xffffffffu;
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    bool up = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < s; ++j) {
      float send = up ? v[j] : v[j + s];
      float keep = up ? v[j + s] : v[j];
      v[j] = keep + __shfl_xor_sync(full, send, s);
    }
  }
  return v[0];
}

// BatchNorm-backward partial sums of one 32-column chunk of a dgrad epilogue row (the
// chan_sums pass of BN_BWD folded into the kernel that produces its dy): d = the stored
// (bf16-rounded) gradient, x = the BN input at the same voxel.  Lane l returns
// (sum d, sum d * (x - mean) * rstd) of column c0 + l over the warp's 32 rows.
__device__ __forceinline__ void bn_bwd_colsums(const float (&v)[32], bool valid,
                                               const __nv_bfloat16* xrow, const float* stat,
                                               int nout, int c0, float& s1, float& s2) {
  float a[32], b[32];
  if (valid) {
    const uint4* x4 = reinterpret_cast<const uint4*>(xrow);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 u = x4[q];
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
        const int j = 8 * q + 2 * e;
        const float d0 = __bfloat162float(__float2bfloat16(v[j]));
        const float d1 = __bfloat162float(__float2bfloat16(v[j + 1]));
        a[j] = d0;
        a[j + 1] = d1;
        b[j] = d0 * ((f.x - __ldg(stat + c0 + j)) * __ldg(stat + nout + c0 + j));
        b[j + 1] = d1 * ((f.y - __ldg(stat + c0 + j + 1)) * __ldg(stat + nout + c0 + j + 1));
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = b[j] = 0.f;
  }
  s1 = warp_colsum32(a);
  s2 = warp_colsum32(b);
}

// Same from a preloaded BN-input chunk; mean / rstd of the chunk's 32 channels.
__device__ __forceinline__ void bn_bwd_colsums_reg(const float (&v)[32], bool valid,
                                                   const uint4 (&xr)[4], const float* mean,
                                                   const float* rstd, float& s1, float& s2) {
  float a[32], b[32];
  if (valid) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 m0 = __ldg(reinterpret_cast<const float4*>(mean) + 2 * q);
      const float4 m1 = __ldg(reinterpret_cast<const float4*>(mean) + 2 * q + 1);
      const float4 r0 = __ldg(reinterpret_cast<const float4*>(rstd) + 2 * q);
      const float4 r1 = __ldg(reinterpret_cast<const float4*>(rstd) + 2 * q + 1);
      const float mm[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
      const float rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
      const uint32_t w[4] = {xr[q].x, xr[q].y, xr[q].z, xr[q].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
        const int j = 8 * q + 2 * e;
        const float d0 = __bfloat162float(__float2bfloat16(v[j]));
        const float d1 = __bfloat162float(__float2bfloat16(v[j + 1]));
        a[j] = d0;
        a[j + 1] = d1;
        b[j] = d0 * ((f.x - mm[2 * e]) * rr[2 * e]);
        b[j + 1] = d1 * ((f.y - mm[2 * e + 1]) * rr[2 * e + 1]);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = b[j] = 0.f;
  }
  s1 = warp_colsum32(a);
  s2 = warp_colsum32(b);
}

// PAIR (fprop, K-major weights, no sub-pixel scatter): a CTA pair takes two M tiles of the
// same (split, n tile) with M = 256 MMAs, each CTA staging half of the BN weight rows -- the
// small deep-level grids re-read their weights from L2 once per M tile, so this halves the
// dominant traffic.
template <int BN, int CK, bool B_MN, bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_igemm(const __grid_constant__ Maps maps, const __grid_constant__ IgParams p) {
  constexpr int kRowBytes = CK * 2;
  constexpr int kABytes = 128 * kRowBytes;
  constexpr int kBBytes = (PAIR ? BN / 2 : BN) * kRowBytes;
  constexpr int kStageBytes = kABytes + kBBytes;
  constexpr int kStagesRaw = kSmemBudget / kStageBytes;
  constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                 : (2 * BN <= 256) ? 256 : 512;
  static_assert(kStages >= 2, "pipeline too shallow");
  constexpr int kEpiOff = kStages * kStageBytes;   // + kIgEpiBytes: epilogue store staging

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ float stat_s[4][2 * 1024];   // per epilogue warp: deterministic BN sums

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int mn_tiles = p.m_tiles * p.n_tiles;
  const int total_tiles = mn_tiles * p.splits;
  // tile -> (split, m tile, n tile); a split covers taps [t0, t1)
  const bool nt_major = p.nt_mask[0] != 0;
  auto tile_mn = [&](int tile, int& mt, int& nt) {
    const int r = tile % mn_tiles;
    if (nt_major) {
      nt = r / p.m_tiles;
      mt = r % p.m_tiles;
    } else {
      mt = r / p.n_tiles;
      nt = r % p.n_tiles;
    }
  };
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int pm_tiles = (p.m_tiles + 1) / 2;
  const int n_items = PAIR ? p.splits * pm_tiles * p.n_tiles : total_tiles;
  const int item0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int item_step = PAIR ? gridDim.x / 2 : gridDim.x;
  auto item_tile = [&](int it, bool& real) {   // -> tile index (split, mt, nt)
    real = true;
    if (!PAIR) return it;
    const int sp = it / (pm_tiles * p.n_tiles), r = it % (pm_tiles * p.n_tiles);
    // both CTAs of a pair share the n tile (and with it the sub-pixel tap mask)
    const int mt = 2 * (r / p.n_tiles) + (int)rank, nt = r % p.n_tiles;
    real = mt < p.m_tiles;
    const int mtt = real ? mt : p.m_tiles - 1;
    return sp * mn_tiles + (nt_major ? nt * p.m_tiles + mtt : mtt * p.n_tiles + nt);
  };
  auto tap_range = [&](int tile, int& t0, int& t1) {
    const int sp = tile / mn_tiles;
    t0 = sp * p.n_taps / p.splits;
    t1 = (sp + 1) * p.n_taps / p.splits;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], PAIR ? 256 : 128);
    }
    fence_barrier_init();
  }
  if (p.stats)
    for (int i = threadIdx.x; i < 8 * p.Nout; i += blockDim.x) stat_s[i / (2 * p.Nout)][i % (2 * p.Nout)] = 0.f;
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair<kTmemCols>(&tmem_base_s);
    else tmem_alloc<kTmemCols>(&tmem_base_s);
  }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 8; ++i) tma_prefetch(&maps.a[i]);
    tma_prefetch(&maps.b);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  auto lead = [&](uint64_t* bar) { return PAIR ? mapa_shared(smem_u32(bar), 0) : smem_u32(bar); };

  if (warp == 0) {
    // ===================== TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = item0; it < n_items; it += item_step) {
        bool real;
        const int tile = item_tile(it, real);
        int mt, nt;
        tile_mn(tile, mt, nt);
        int n, x0, y0, z0;
        ig_decode(p, mt, n, x0, y0, z0);
        int ta, tb;
        tap_range(tile, ta, tb);
        for (int t = ta; t < tb; ++t) {
          if (nt_major && !((p.nt_mask[nt] >> t) & 1)) continue;
          int ax = x0 + p.taps.dx[t], ay = y0 + p.taps.dy[t], az = z0 + p.taps.dz[t];
          int wcol = p.taps.w[t] * p.w_cin;
          for (int kc = 0; kc < p.k_chunks; ++kc) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * kStageBytes;
            uint8_t* sb = sa + kABytes;
            int ac = p.a_c0 + kc * CK;
            const CUtensorMap* am = act_map(maps, p.taps.map[t], ac);
            if (!B_MN && !PAIR && p.sp_direct) {
              // sub-pixel convT, one parity class per n tile (host: Cout % BN == 0): the
              // class's weight rows straight from W[co][k][ci] at its kernel tap k (the tile
              // only visits taps its class uses, nt_mask)
              const int col0 = nt * BN, cls = col0 / p.scatter_c, co0 = col0 % p.scatter_c;
              mbar_arrive_expect_tx(&full_bar[stage], kStageBytes);
              tma_load_5d(sa, am, &full_bar[stage], ac, ax, ay, az, n);
              tma_load_2d(sb, &maps.b, &full_bar[stage], convt_ktap(t, cls) * p.w_cin + kc * CK,
                          co0);
            } else if (PAIR) {
              if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * kStageBytes);
              tma_load_5d_pair(sa, am, lead(&full_bar[stage]), ac, ax, ay, az, n);
              if (!B_MN) {   // K-major weights: this CTA's half of the BN rows
                tma_load_2d_pair(sb, &maps.b, lead(&full_bar[stage]), wcol + kc * CK,
                                 nt * BN + (BN / 2) * (int)rank);
              } else {       // MN-major (dgrad): this CTA's 64-column chunks of the BN
#pragma unroll
                for (int j = 0; j < BN / 128; ++j)
                  tma_load_2d_pair(sb + j * (CK * 128), &maps.b, lead(&full_bar[stage]),
                                   wcol + nt * BN + ((int)rank * (BN / 128) + j) * 64, kc * CK);
              }
            } else {
            mbar_arrive_expect_tx(&full_bar[stage], kStageBytes);
            tma_load_5d(sa, am, &full_bar[stage], ac, ax, ay, az, n);
            if (!B_MN) {
              tma_load_2d(sb, &maps.b, &full_bar[stage], wcol + kc * CK, nt * BN);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_2d(sb + j * (CK * 128), &maps.b, &full_bar[stage],
                            wcol + nt * BN + j * 64, kc * CK);
            }
            }
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ===================== MMA issuer
    constexpr uint32_t kLayout = swizzle_code(kRowBytes);
    constexpr uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, BN, 0, B_MN ? 1 : 0);
    const uint32_t smem_base = smem_u32(smem);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int it = item0; it < n_items; it += item_step) {
      bool real;
      const int tile = item_tile(it, real);
      mbar_wait(&tempty_bar[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t dtmem = tmem_base + acc * BN;
      int kiter = 0;
      int ta, tb;
      tap_range(tile, ta, tb);
      int nt_i = 0;
      if (nt_major) {
        int mt_i;
        tile_mn(tile, mt_i, nt_i);
      }
      for (int t = ta; t < tb; ++t) {
        if (nt_major && !((p.nt_mask[nt_i] >> t) & 1)) continue;
        for (int kc = 0; kc < p.k_chunks; ++kc, ++kiter) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_base + stage * kStageBytes;
            const uint32_t sb = sa + kABytes;
#pragma unroll
            for (int k = 0; k < CK / 16; ++k) {
              uint64_t ad = smem_desc(sa + k * 32, 16, 8 * kRowBytes, kLayout);
              uint64_t bd = B_MN ? smem_desc(sb + k * 2048, CK * 128, 1024, 2)
                                 : smem_desc(sb + k * 32, 16, 8 * kRowBytes, kLayout);
              if (PAIR) umma_bf16_pair(dtmem, ad, bd, idesc, (kiter | k) != 0);
              else umma_bf16(dtmem, ad, bd, idesc, (kiter | k) != 0);
            }
            if (PAIR) umma_commit_pair(&empty_bar[stage], 0x3);
            else umma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (elect_one()) {
        if (PAIR) umma_commit_pair(&tfull_bar[acc], 0x3);
        else umma_commit(&tfull_bar[acc]);
      }
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  } else if (warp >= 2) {
    // ===================== epilogue (warps 2..5)
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;       // accumulator row == voxel within the tile
    const int lx = row % p.bw, ly = (row / p.bw) % p.bh, lz = row / (p.bw * p.bh);
    int acc = 0;
    uint32_t aphase = 0;
    for (int it = item0; it < n_items; it += item_step) {
      bool real;
      const int tile = item_tile(it, real);
      int mt, nt;
      tile_mn(tile, mt, nt);
      if (p.splits > 1) {   // fp32 partial tile; k_igemm_split_reduce finishes it
        float* dst = p.split_part +
                     ((((int64_t)(tile / mn_tiles) * p.m_tiles + mt) * p.n_tiles + nt) * 128 + row) * BN;
        mbar_wait(&tfull_bar[acc], aphase);
        tc_fence_after();
        constexpr int kColS = BN < 32 ? BN : 32;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += kColS) {
          uint32_t r[32];
          const uint32_t taddr = tmem_base + acc * BN + c0 + ((uint32_t)(q * 32) << 16);
          if (kColS == 32) tmem_ld32(taddr, r);
          else tmem_ld16(taddr, r);
          tmem_ld_wait();
          float4* d4 = reinterpret_cast<float4*>(dst + c0);
          if (real) {
#pragma unroll
            for (int j = 0; j < kColS / 4; ++j)
              d4[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                  __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
          }
        }
        tc_fence_before();
        if (PAIR && !leader) mbar_arrive_cluster(lead(&tempty_bar[acc]));
        else mbar_arrive(&tempty_bar[acc]);
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
        continue;
      }
      int n, x0, y0, z0;
      ig_decode(p, mt, n, x0, y0, z0);
      int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
      bool valid = real && gx < p.Mw && gy < p.Mh && gz < p.Md;
      int64_t ovox = (((int64_t)n * p.oD + gz * p.os + p.ooz) * p.oH + gy * p.os + p.ooy) * p.oW +
                     gx * p.os + p.oox;
      __nv_bfloat16* orow = p.out + ovox * p.out_cs + p.out_co + nt * BN;
      mbar_wait(&tfull_bar[acc], aphase);
      tc_fence_after();
      if (BN % 64 == 0 && p.staged_epi && !p.mask && !p.stats) {
        // Coalesced stores through shared memory (no ReLU mask / BN sums to fold in): each
        // 64-column group is 128 contiguous bytes of the thread's output row; the warp
        // stages its 32 rows (XOR-swizzled 16-byte chunks, conflict-free) and writes them
        // back 8 threads per row -- 4 full 128-byte segments per store instruction instead
        // of 32 scattered 16-byte pieces (the transposed conv's parity-scattered rows were
        // store-bound: ncu long-scoreboard stalls on the epilogue's global stores).
        uint8_t* epi = smem + kEpiOff + (warp - 2) * 4096;
        const unsigned full = 0xffffffffu;
#pragma unroll 1
        for (int g = 0; g < BN; g += 64) {
          __nv_bfloat16* dst = orow + g;
          if (p.scatter_c) {   // sub-pixel convT: parity class pc, channels co .. co + 63
            const int col = nt * BN + g, pc = col / p.scatter_c, co = col % p.scatter_c;
            const int64_t hv = (((int64_t)n * p.oD + 2 * gz + (pc >> 2)) * p.oH + 2 * gy +
                                ((pc >> 1) & 1)) * p.oW + 2 * gx + (pc & 1);
            dst = p.out + hv * p.out_cs + p.out_co + co;
          }
          uint32_t ra[32], rb[32];
          const uint32_t taddr = tmem_base + acc * BN + g + ((uint32_t)(q * 32) << 16);
          tmem_ld32(taddr, ra);
          tmem_ld32(taddr + 32, rb);
          tmem_ld_wait();
          uint8_t* myrow = epi + lane * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t* r = j < 4 ? ra + 8 * j : rb + 8 * (j - 4);
            uint4 w;
            w.x = pack_bf16(__uint_as_float(r[0]), __uint_as_float(r[1]));
            w.y = pack_bf16(__uint_as_float(r[2]), __uint_as_float(r[3]));
            w.z = pack_bf16(__uint_as_float(r[4]), __uint_as_float(r[5]));
            w.w = pack_bf16(__uint_as_float(r[6]), __uint_as_float(r[7]));
            *reinterpret_cast<uint4*>(myrow + ((j ^ (lane & 7)) << 4)) = w;
          }
          __syncwarp();
          const unsigned long long du = reinterpret_cast<unsigned long long>(dst);
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int rr = it * 4 + (lane >> 3), cc = lane & 7;
            const unsigned long long d = __shfl_sync(full, du, rr);
            const int vv = __shfl_sync(full, (int)valid, rr);
            const uint4 w =
                *reinterpret_cast<const uint4*>(epi + rr * 128 + ((cc ^ (rr & 7)) << 4));
            if (vv) *reinterpret_cast<uint4*>(d + (unsigned long long)cc * 16) = w;
          }
          __syncwarp();
        }
        tc_fence_before();
        if (PAIR && !leader) mbar_arrive_cluster(lead(&tempty_bar[acc]));
        else mbar_arrive(&tempty_bar[acc]);
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
        continue;
      }
      constexpr int kCol = BN < 32 ? BN : 32;   // columns per TMEM load
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += kCol) {
        if (p.scatter_c) {   // sub-pixel convT: this chunk is parity class pc, channels co..
          const int col = nt * BN + c0, pc = col / p.scatter_c, co = col % p.scatter_c;
          const int64_t hv = (((int64_t)n * p.oD + 2 * gz + (pc >> 2)) * p.oH + 2 * gy +
                              ((pc >> 1) & 1)) * p.oW + 2 * gx + (pc & 1);
          orow = p.out + hv * p.out_cs + p.out_co + co - c0;
        }
        uint32_t r[32];
        const uint32_t taddr = tmem_base + acc * BN + c0 + ((uint32_t)(q * 32) << 16);
        if (kCol == 32) {
          tmem_ld32(taddr, r);
        } else {
          tmem_ld16(taddr, r);
#pragma unroll
          for (int j = 16; j < 32; ++j) r[j] = 0u;
        }
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = valid ? __uint_as_float(r[j]) : 0.f;
        if (p.mask && valid) apply_relu_mask(v, p.mask + (orow - p.out) + c0, kCol);
        if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
          for (int j = 0; j < kCol / 8; ++j) {
            uint4 w;
            w.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
            w.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
            w.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
            w.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
            dst[j] = w;
          }
        }
        if (p.stats) {
          float s1, s2;
          if (p.bnx) {
            bn_bwd_colsums(v, valid, p.bnx + ovox * p.Nout + nt * BN + c0, p.bn_stat, p.Nout,
                           nt * BN + c0, s1, s2);
          } else {
            float sq[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) sq[j] = v[j] * v[j];
            s1 = warp_colsum32(v);
            s2 = warp_colsum32(sq);
          }
          int ch = nt * BN + c0 + lane;
          if (lane < kCol) {
            stat_s[warp - 2][ch] += s1;
            stat_s[warp - 2][p.Nout + ch] += s2;
          }
        }
      }
      tc_fence_before();
      if (PAIR && !leader) mbar_arrive_cluster(lead(&tempty_bar[acc]));
      else mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.stats && p.splits == 1)
    for (int i = threadIdx.x; i < 2 * p.Nout; i += blockDim.x)
      p.stats[(int64_t)blockIdx.x * 2 * p.Nout + i] =
          ((stat_s[0][i] + stat_s[1][i]) + stat_s[2][i]) + stat_s[3][i];
  if (PAIR) {
    cluster_sync();
    if (warp == 1) tmem_dealloc_pair<kTmemCols>(tmem_base);
  } else if (warp == 1) {
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// Split-K finish: block = (M tile, 64 output channels), 256 threads = 64 channels x 4 row
// groups.  Sums the split partials (fixed order), applies the fused ReLU mask, stores
// bf16 and writes the tile's BN partial sums (fixed-order combination: deterministic).
template <int BN>
__global__ void __launch_bounds__(256) k_igemm_split_reduce(const IgParams p) {
  __shared__ float red[2][4][64];
  const int mt = blockIdx.x;
  const int c = blockIdx.y * 64 + (threadIdx.x & 63), rg = threadIdx.x >> 6;
  int n, x0, y0, z0;
  ig_decode(p, mt, n, x0, y0, z0);
  const int64_t split_stride = (int64_t)p.m_tiles * p.n_tiles * 128 * BN;
  const int nt = c / BN, cc = c % BN;
  const float* src = p.split_part + (((int64_t)mt * p.n_tiles + nt) * 128) * BN + cc;
  float s1 = 0.f, s2 = 0.f;
  for (int row = rg; row < 128; row += 4) {
    const int lx = row % p.bw, ly = (row / p.bw) % p.bh, lz = row / (p.bw * p.bh);
    const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
    if (gx >= p.Mw || gy >= p.Mh || gz >= p.Md) continue;
    float v = 0.f;
    for (int sp = 0; sp < p.splits; ++sp) v += src[sp * split_stride + (int64_t)row * BN];
    const int64_t ovox = (((int64_t)n * p.oD + gz * p.os + p.ooz) * p.oH + gy * p.os + p.ooy) *
                             p.oW + gx * p.os + p.oox;
    const int64_t o = ovox * p.out_cs + p.out_co + c;
    if (p.mask && !(__bfloat162float(p.mask[o]) > 0.f)) v = 0.f;
    p.out[o] = __float2bfloat16(v);
    if (p.bnx) {   // fused BN-backward sums (d rounded as stored)
      const float d = __bfloat162float(__float2bfloat16(v));
      const float xh = (__bfloat162float(p.bnx[ovox * p.Nout + c]) - p.bn_stat[c]) *
                       p.bn_stat[p.Nout + c];
      s1 += d;
      s2 += d * xh;
    } else {
      s1 += v;
      s2 += v * v;
    }
  }
  if (!p.stats) return;
  red[0][rg][threadIdx.x & 63] = s1;
  red[1][rg][threadIdx.x & 63] = s2;
  __syncthreads();
  if (rg == 0) {
    const int k = threadIdx.x & 63;
    p.stats[(int64_t)mt * 2 * p.Nout + c] =
        ((red[0][0][k] + red[0][1][k]) + red[0][2][k]) + red[0][3][k];
    p.stats[(int64_t)mt * 2 * p.Nout + p.Nout + c] =
        ((red[1][0][k] + red[1][1][k]) + red[1][2][k]) + red[1][3][k];
  }
}

// ---------------------------------------------------------------- halo igemm
// Stride-1 3x3x3 conv (fprop, or dgrad with mirrored taps) with the input halo
// staged ONCE per 64-channel chunk: the output tile is 8(w) x 16(h) x 1(d)
// voxels; the halo is a 10 x 18 x 3 box (one 5-D TMA load, zero fill = padding)
// laid out as 540 rows of 128 B (SWIZZLE_128B).  Each of the 27 taps is a
// *view* of that buffer: start row (kd*18 + kh)*10 + kw, 16 groups of 8 rows at
// a 10-row (1280 B) stride -- the hardware swizzle is address based, so any
// 128-B-aligned row offset is a valid K-major operand (csrc/selftest_umma.cu T6).
// This cuts the A-operand L2->SM traffic from 27 x 16 KB to 69 KB per tile.
constexpr int kHW = 10, kHH = 18, kHD = 3;          // halo box
constexpr int kHaloRows = kHW * kHH * kHD;          // 540
constexpr int kHaloBytes = kHaloRows * 128;         // 69120 (64 channels)
constexpr int kHaloStride = (kHaloBytes + 1023) / 1024 * 1024;

constexpr int kHaloXposeBytes = 4 * 32 * 36 * 4;
constexpr bool halo_xpose_fits(int bn, int na, int nb, int tps) {
  return na * kHaloStride + nb * tps * bn * 128 + kHaloXposeBytes + 1024 + 4096 <= 232448;
}
constexpr size_t halo_smem_bytes(int bn, int na, int nb, int tps) {
  return (size_t)na * kHaloStride + (size_t)nb * tps * bn * 128 +
         (halo_xpose_fits(bn, na, nb, tps) ? kHaloXposeBytes : 0) + 1024;
}

struct HaloParams {
  int Nb, Md, Mh, Mw;        // conv grid
  int tw, th, td;            // tiles per dim (8 x 16 x 1 boxes)
  int m_tiles, n_tiles;
  int k_chunks;              // 64-channel chunks of the A operand
  int a_c0;                  // channel offset of A inside its tensor
  int w_cin;                 // Cin of the weight layout
  int mirror;                // 0 fprop (tap reads x[v + k - 1]), 1 dgrad (x[v - k + 1])
  __nv_bfloat16* out;
  const __nv_bfloat16* mask; // fused ReLU backward (dgrad): out = acc * (mask > 0)
  const __nv_bfloat16* bnx;  // fused BN-backward sums (dgrad), see IgParams
  const float* bn_stat;
  int b_rows_tap;            // CTA-pair dgrad: B map rows are (tap, ci) of transposed weights
  int out_cs;
  float* stats;              // [gridDim.x][2][Nout] or null
  int Nout;
};

// PAIR: CTA pair (cluster of 2, cta_group::2) as in k_halo_z2 -- two tiles per M = 256 MMA,
// each CTA stages its own halo and half of the BN weight rows (one N tile only).
template <int BN, bool B_MN, int NA, int NB, int TPS, bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_igemm_halo(const __grid_constant__ Maps maps, const __grid_constant__ HaloParams p) {
  static_assert(!(PAIR && B_MN), "the CTA-pair variant splits K-major weights only");
  constexpr int kTapBytes = (PAIR ? BN / 2 : BN) * 128;   // one tap's 64-channel K chunk
  constexpr int kBBytes = TPS * kTapBytes;          // TPS taps per B stage (more MMAs per wait)
  constexpr uint32_t kTmemCols = (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  constexpr bool kXpose = halo_xpose_fits(BN, NA, NB, TPS);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* a_buf = smem;
  uint8_t* b_buf = smem + NA * kHaloStride;
  // per epilogue warp: 32x32 transpose for the BN column sums (when it fits; else shuffles)
  float (*xpose)[32][36] = reinterpret_cast<float (*)[32][36]>(b_buf + NB * kBBytes);
  __shared__ __align__(8) uint64_t a_full[NA], a_empty[NA], b_full[NB], b_empty[NB];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ float stat_w[4][2][BN];

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int total_tiles = p.m_tiles * p.n_tiles;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int n_items = PAIR ? (total_tiles + 1) / 2 : total_tiles;   // PAIR: n_tiles == 1
  const int item0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int item_step = PAIR ? gridDim.x / 2 : gridDim.x;
  auto item_tile = [&](int it, bool& real) {
    const int t = PAIR ? 2 * it + (int)rank : it;
    real = t < total_tiles;
    return real ? t : total_tiles - 1;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NA; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < NB; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], PAIR ? 256 : 128);
    }
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 4 * 2 * BN; i += blockDim.x) (&stat_w[0][0][0])[i] = 0.f;
  if (p.stats)
    for (int i = threadIdx.x; i < 2 * p.Nout; i += blockDim.x)
      p.stats[(int64_t)blockIdx.x * 2 * p.Nout + i] = 0.f;
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair<kTmemCols>(&tmem_base_s);
    else tmem_alloc<kTmemCols>(&tmem_base_s);
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&maps.a[0]);
    tma_prefetch(&maps.b);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  auto lead = [&](uint64_t* bar) { return PAIR ? mapa_shared(smem_u32(bar), 0) : smem_u32(bar); };

  // tile order: n-tile major, so a CTA's N columns change rarely (stats flush)
  auto decode = [&](int tile, int& nt, int& n, int& x0, int& y0, int& z0) {
    nt = tile / p.m_tiles;
    int mt = tile % p.m_tiles;
    int tx = mt % p.tw;
    int r = mt / p.tw;
    int ty = r % p.th;
    r /= p.th;
    z0 = r % p.td;
    n = r / p.td;
    x0 = tx * 8;
    y0 = ty * 16;
  };

  if (warp == 0) {
    if (elect_one()) {
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      for (int it = item0; it < n_items; it += item_step) {
        bool real;
        const int tile = item_tile(it, real);
        int nt, n, x0, y0, z0;
        decode(tile, nt, n, x0, y0, z0);
        for (int kc = 0; kc < p.k_chunks; ++kc) {
          mbar_wait(&a_empty[as], aph ^ 1);
          int ac = p.a_c0 + kc * 64;
          const CUtensorMap* am = act_map(maps, 0, ac);
          if (PAIR) {
            if (leader) mbar_arrive_expect_tx(&a_full[as], 2 * kHaloBytes);
            tma_load_5d_pair(a_buf + as * kHaloStride, am, lead(&a_full[as]), ac, x0 - 1,
                             y0 - 1, z0 - 1, n);
          } else {
            mbar_arrive_expect_tx(&a_full[as], kHaloBytes);
            tma_load_5d(a_buf + as * kHaloStride, am, &a_full[as], ac, x0 - 1, y0 - 1, z0 - 1,
                        n);
          }
          if (++as == NA) {
            as = 0;
            aph ^= 1;
          }
          for (int t0 = 0; t0 < 27; t0 += TPS) {
            mbar_wait(&b_empty[bs], bph ^ 1);
            uint8_t* sb0 = b_buf + bs * kBBytes;
            if (!PAIR || leader) mbar_arrive_expect_tx(&b_full[bs], (PAIR ? 2 : 1) * kBBytes);
#pragma unroll
            for (int tt = 0; tt < TPS; ++tt) {
              const int t = t0 + tt;
              uint8_t* sb = sb0 + tt * kTapBytes;
              if (PAIR && p.b_rows_tap) {   // dgrad: W^T rows (t, ci), this CTA's half
                tma_load_2d_pair(sb, &maps.b, lead(&b_full[bs]), kc * 64,
                                 t * p.w_cin + (BN / 2) * (int)rank);
              } else if (PAIR) {            // fprop: output channel rows of this CTA's half
                tma_load_2d_pair(sb, &maps.b, lead(&b_full[bs]), t * p.w_cin + kc * 64,
                                 (BN / 2) * (int)rank);
              } else if (!B_MN) {
                tma_load_2d(sb, &maps.b, &b_full[bs], t * p.w_cin + kc * 64, nt * BN);
              } else {
#pragma unroll
                for (int j = 0; j < BN / 64; ++j)
                  tma_load_2d(sb + j * 8192, &maps.b, &b_full[bs], t * p.w_cin + nt * BN + j * 64,
                              kc * 64);
              }
            }
            if (++bs == NB) {
              bs = 0;
              bph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    constexpr uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, BN, 0, B_MN ? 1 : 0);
    const uint32_t a_base = smem_u32(a_buf), b_base = smem_u32(b_buf);
    int as = 0, bs = 0, acc = 0;
    uint32_t aph = 0, bph = 0, tph = 0;
    for (int it = item0; it < n_items; it += item_step) {
      mbar_wait(&tempty_bar[acc], tph ^ 1);
      tc_fence_after();
      const uint32_t dtmem = tmem_base + acc * BN;
      for (int kc = 0; kc < p.k_chunks; ++kc) {
        mbar_wait(&a_full[as], aph);
        tc_fence_after();
        // descriptors are built once per stage; each tap / K-step only adds its
        // (compile-time) byte offset >> 4 to the start-address field
        const uint64_t a_desc0 = smem_desc(a_base + as * kHaloStride, 16, kHW * 128, 2);
#pragma unroll
        for (int t0 = 0; t0 < 27; t0 += TPS) {
          mbar_wait(&b_full[bs], bph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t b_desc0 = B_MN ? smem_desc(b_base + bs * kBBytes, 8192, 1024, 2)
                                          : smem_desc(b_base + bs * kBBytes, 16, 1024, 2);
#pragma unroll
            for (int tt = 0; tt < TPS; ++tt) {
              const int t = t0 + tt;
              constexpr int kHWB = kHW * 128, kHHB = kHH * kHW * 128;
              const uint32_t off_f = ((t / 9) * kHHB + ((t / 3) % 3) * kHWB + (t % 3) * 128);
              const uint32_t off_m = ((2 - t / 9) * kHHB + (2 - (t / 3) % 3) * kHWB +
                                      (2 - t % 3) * 128);
              const uint32_t view = p.mirror ? off_m : off_f;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t ad = a_desc0 + ((view + k * 32) >> 4);
                const uint64_t bd = b_desc0 + ((tt * kTapBytes + k * (B_MN ? 2048 : 32)) >> 4);
                if (PAIR) umma_bf16_pair(dtmem, ad, bd, idesc, (kc | t | k) != 0);
                else umma_bf16(dtmem, ad, bd, idesc, (kc | t | k) != 0);
              }
            }
            if (PAIR) {
              umma_commit_pair(&b_empty[bs], 0x3);
              if (t0 + TPS >= 27) umma_commit_pair(&a_empty[as], 0x3);
            } else {
              umma_commit(&b_empty[bs]);
              if (t0 + TPS >= 27) umma_commit(&a_empty[as]);
            }
          }
          __syncwarp();
          if (++bs == NB) {
            bs = 0;
            bph ^= 1;
          }
        }
        if (++as == NA) {
          as = 0;
          aph ^= 1;
        }
      }
      if (elect_one()) {
        if (PAIR) umma_commit_pair(&tfull_bar[acc], 0x3);
        else umma_commit(&tfull_bar[acc]);
      }
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        tph ^= 1;
      }
    }
  } else if (warp >= 2) {
    const int q = warp & 3;
    const int ew = warp - 2;
    const int row = q * 32 + lane;
    const int lx = row & 7, ly = row >> 3;
    int acc = 0, cur_nt = -1;
    uint32_t tph = 0;
    auto flush = [&](int nt) {
      if (nt < 0 || !p.stats) return;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int i = threadIdx.x - 64; i < 2 * BN; i += 128) {
        int which = i / BN, c = i % BN;
        float s = ((stat_w[0][which][c] + stat_w[1][which][c]) + stat_w[2][which][c]) +
                  stat_w[3][which][c];
        p.stats[(int64_t)blockIdx.x * 2 * p.Nout + which * p.Nout + nt * BN + c] += s;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int i = threadIdx.x - 64; i < 4 * 2 * BN; i += 128) (&stat_w[0][0][0])[i] = 0.f;
      asm volatile("bar.sync 1, 128;" ::: "memory");
    };
    for (int it = item0; it < n_items; it += item_step) {
      bool real;
      const int tile = item_tile(it, real);
      int nt, n, x0, y0, z0;
      decode(tile, nt, n, x0, y0, z0);
      if (nt != cur_nt) {
        flush(cur_nt);
        cur_nt = nt;
      }
      int gx = x0 + lx, gy = y0 + ly, gz = z0;
      bool valid = real && gx < p.Mw && gy < p.Mh;
      int64_t ovox = (((int64_t)n * p.Md + gz) * p.Mh + gy) * p.Mw + gx;
      __nv_bfloat16* orow = p.out + ovox * p.out_cs + nt * BN;
      mbar_wait(&tfull_bar[acc], tph);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint4 mk[4], xb[4];
        if (p.mask && valid) load32_bf16(p.mask + (orow - p.out) + c0, mk);
        if (p.bnx && valid) load32_bf16(p.bnx + ovox * p.Nout + nt * BN + c0, xb);
        uint32_t r[32];
        tmem_ld32(tmem_base + acc * BN + c0 + ((uint32_t)(q * 32) << 16), r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = valid ? __uint_as_float(r[j]) : 0.f;
        if (p.mask && valid) apply_relu_mask_reg(v, mk);
        if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 w;
            w.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
            w.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
            w.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
            w.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
            dst[j] = w;
          }
        }
        if (p.stats && p.bnx) {   // dgrad: fused BN-backward sums
          float s1, s2;
          bn_bwd_colsums_reg(v, valid, xb, p.bn_stat + nt * BN + c0,
                             p.bn_stat + p.Nout + nt * BN + c0, s1, s2);
          stat_w[ew][0][c0 + lane] += s1;
          stat_w[ew][1][c0 + lane] += s2;
        } else if (p.stats && !kXpose) {
          float sq[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) sq[j] = v[j] * v[j];
          const float s1 = warp_colsum32(v);
          const float s2 = warp_colsum32(sq);
          stat_w[ew][0][c0 + lane] += s1;
          stat_w[ew][1][c0 + lane] += s2;
        } else if (p.stats) {
          // column sums through a padded smem transpose (conflict-free both ways):
          // lane = row writes its 32 values, then lane = column sums 32 rows
          float* xp = &xpose[ew][0][0];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(xp + lane * 36 + 4 * j) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          __syncwarp();
          float s1 = 0.f, s2 = 0.f;
#pragma unroll
          for (int r2 = 0; r2 < 32; ++r2) {
            const float x = xp[r2 * 36 + lane];
            s1 += x;
            s2 = fmaf(x, x, s2);
          }
          __syncwarp();
          stat_w[ew][0][c0 + lane] += s1;
          stat_w[ew][1][c0 + lane] += s2;
        }
      }
      tc_fence_before();
      if (PAIR && !leader) mbar_arrive_cluster(lead(&tempty_bar[acc]));
      else mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        tph ^= 1;
      }
    }
    flush(cur_nt);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) {
    cluster_sync();
    if (warp == 1) tmem_dealloc_pair<kTmemCols>(tmem_base);
  } else if (warp == 1) {
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------- z-pair halo igemm (N = 64)
// With 64 output channels the tensor pipe is fed from shared memory (A 4 KB + B 2 KB
// per K16 MMA: 48 clk against 32 of math) and a 128-voxel tile streams all 27 taps of
// weights (27 x 8 KB per 64-channel chunk) -- 3x its own input halo.  This variant
// computes TWO output planes (z0, z0+1) per tile into two TMEM accumulators that share
// every weight stage: weight bytes per voxel halve and each weight stage covers twice
// the MMA time, so the same ring hides twice the L2 latency (measured: the 8x16x1
// kernel is bound by weight-stage latency -- one more stage bought 13%).  The input
// arrives as 1-voxel-deep halo slabs (10 x 18 rows, 23 KB, one 5-D TMA box each) in a
// 6-slab ring; a tile needs slabs z0-1 .. z0+2 (slab j = plane z0-1+j).  Step s = 0..2
// multiplies slab s (output plane z0) and slab s+1 (plane z0+1) by the 9 taps of
// kd = s (fprop) or kd = 2-s (dgrad: mirrored taps), then releases slab s (slab 3
// after the last step), so slab loads of the next tile overlap this tile's math.
constexpr int kSlabBytes = kHW * kHH * 128;                        // 23040
constexpr int kSlabStride = (kSlabBytes + 1023) / 1024 * 1024;     // 23552
constexpr size_t z2_smem(int slabs, int nb) {
  return (size_t)slabs * kSlabStride + (size_t)nb * 3 * 64 * 128 + 1024;
}

// kZ2Slabs: slab ring (>= 5: 4 per tile + the next tile's first); kZ2NB: 3-tap weight stages
// PAIR: a CTA pair (cluster of 2, cta_group::2) computes two tiles with M = 256 MMAs: each
// CTA stages its own input slabs and HALF of every weight tap (32 of the 64 output
// channels); the leader issues the MMAs, which read A from both CTAs and B halves from
// both, so each SM's shared memory feeds 4 + 1 KB per K16 step instead of 4 + 2 KB.  Both
// CTAs' TMA loads complete on the leader's barriers; the commits multicast to both.
template <bool B_MN, int kZ2Slabs, int kZ2NB, bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_halo_z2(const __grid_constant__ Maps maps, const __grid_constant__ HaloParams p) {
  static_assert(!(PAIR && B_MN), "the CTA-pair variant splits K-major weights only");
  constexpr int BN = 64;
  constexpr int kTapBytes = (PAIR ? BN / 2 : BN) * 128;
  constexpr int kBBytes = 3 * kTapBytes;
  constexpr int kHWB = kHW * 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* s_buf = smem;
  uint8_t* b_buf = smem + kZ2Slabs * kSlabStride;
  __shared__ __align__(8) uint64_t s_full[kZ2Slabs], s_empty[kZ2Slabs], b_full[kZ2NB],
      b_empty[kZ2NB];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ float stat_w[4][2][BN];

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int total_tiles = p.m_tiles;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  // work items: tiles, or (PAIR) tile pairs -- CTA `rank` takes tile 2 * pair + rank; an odd
  // last tile leaves the peer a dummy tile (loads a real one, stores nothing)
  const int n_items = PAIR ? (total_tiles + 1) / 2 : total_tiles;
  const int item0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int item_step = PAIR ? gridDim.x / 2 : gridDim.x;
  auto item_tile = [&](int it, bool& real) {
    const int t = PAIR ? 2 * it + (int)rank : it;
    real = t < total_tiles;
    return real ? t : total_tiles - 1;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < kZ2Slabs; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 1);
    }
    for (int i = 0; i < kZ2NB; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], PAIR ? 256 : 128);   // PAIR: both CTAs' epilogues
    }
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 4 * 2 * BN; i += blockDim.x) (&stat_w[0][0][0])[i] = 0.f;
  if (p.stats)
    for (int i = threadIdx.x; i < 2 * p.Nout; i += blockDim.x)
      p.stats[(int64_t)blockIdx.x * 2 * p.Nout + i] = 0.f;
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair<256>(&tmem_base_s);
    else tmem_alloc<256>(&tmem_base_s);
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&maps.a[0]);
    tma_prefetch(&maps.b);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();   // the leader's barriers are initialised before any peer signal
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  // mbarrier of the leader CTA (TMA completion, tempty) in the cluster address space
  auto lead = [&](uint64_t* bar) { return PAIR ? mapa_shared(smem_u32(bar), 0) : smem_u32(bar); };

  auto decode = [&](int tile, int& n, int& x0, int& y0, int& z0) {
    const int tx = tile % p.tw;
    int r = tile / p.tw;
    const int ty = r % p.th;
    r /= p.th;
    z0 = (r % p.td) * 2;
    n = r / p.td;
    x0 = tx * 8;
    y0 = ty * 16;
  };

  if (warp == 0) {
    if (elect_one()) {
      int ss = 0, bs = 0;
      uint32_t sph = 0, bph = 0;
      for (int it = item0; it < n_items; it += item_step) {
        bool real;
        const int tile = item_tile(it, real);
        int n, x0, y0, z0;
        decode(tile, n, x0, y0, z0);
        for (int kc = 0; kc < p.k_chunks; ++kc) {
          for (int st = 0; st < 3; ++st) {
            for (int j = (st == 0 ? 0 : st + 1); j <= st + 1; ++j) {   // slabs 0,1 | 2 | 3
              mbar_wait(&s_empty[ss], sph ^ 1);
              int ac = p.a_c0 + kc * 64;
              const CUtensorMap* am = act_map(maps, 0, ac);
              if (PAIR) {
                if (leader) mbar_arrive_expect_tx(&s_full[ss], 2 * kSlabBytes);
                tma_load_5d_pair(s_buf + ss * kSlabStride, am, lead(&s_full[ss]), ac, x0 - 1,
                                 y0 - 1, z0 - 1 + j, n);
              } else {
                mbar_arrive_expect_tx(&s_full[ss], kSlabBytes);
                tma_load_5d(s_buf + ss * kSlabStride, am, &s_full[ss], ac, x0 - 1, y0 - 1,
                            z0 - 1 + j, n);
              }
              if (++ss == kZ2Slabs) {
                ss = 0;
                sph ^= 1;
              }
            }
            const int kd = p.mirror ? 2 - st : st;
            for (int kh = 0; kh < 3; ++kh) {
              mbar_wait(&b_empty[bs], bph ^ 1);
              uint8_t* sb0 = b_buf + bs * kBBytes;
              if (!PAIR || leader) mbar_arrive_expect_tx(&b_full[bs], (PAIR ? 2 : 1) * kBBytes);
#pragma unroll
              for (int kw = 0; kw < 3; ++kw) {
                const int t = kd * 9 + kh * 3 + kw;
                uint8_t* sb = sb0 + kw * kTapBytes;
                if (PAIR && p.b_rows_tap)   // dgrad: rows (t, ci) of W^T, ci half of rank
                  tma_load_2d_pair(sb, &maps.b, lead(&b_full[bs]), kc * 64,
                                   t * p.w_cin + 32 * (int)rank);
                else if (PAIR)   // this CTA's half: output channels [32 rank, 32 rank + 32)
                  tma_load_2d_pair(sb, &maps.b, lead(&b_full[bs]), t * p.w_cin + kc * 64,
                                   32 * (int)rank);
                else if (!B_MN)
                  tma_load_2d(sb, &maps.b, &b_full[bs], t * p.w_cin + kc * 64, 0);
                else
                  tma_load_2d(sb, &maps.b, &b_full[bs], t * p.w_cin, kc * 64);
              }
              if (++bs == kZ2NB) {
                bs = 0;
                bph ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    constexpr uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, BN, 0, B_MN ? 1 : 0);
    const uint32_t s_base = smem_u32(s_buf), b_base = smem_u32(b_buf);
    int ss = 0, bs = 0, acc = 0;
    uint32_t sph = 0, bph = 0, tph = 0;
    auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc_) {
      if (PAIR) umma_bf16_pair(d, a, b, idesc, acc_);
      else umma_bf16(d, a, b, idesc, acc_);
    };
    auto commit = [&](uint64_t* bar) {
      if (PAIR) umma_commit_pair(bar, 0x3);
      else umma_commit(bar);
    };
    for (int it = item0; it < n_items; it += item_step) {
      mbar_wait(&tempty_bar[acc], tph ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem_base + acc * 2 * BN, d1 = d0 + BN;
      for (int kc = 0; kc < p.k_chunks; ++kc) {
        // this chunk's 4 slabs sit at ring positions ss .. ss+3 (mod kZ2Slabs)
        auto slot = [&](int j) { return ss + j < kZ2Slabs ? ss + j : ss + j - kZ2Slabs; };
        auto phase = [&](int j) { return ss + j < kZ2Slabs ? sph : sph ^ 1u; };
#pragma unroll 1
        for (int st = 0; st < 3; ++st) {
          if (st == 0) mbar_wait(&s_full[slot(0)], phase(0));
          mbar_wait(&s_full[slot(st + 1)], phase(st + 1));
          tc_fence_after();
          const int sa = slot(st), sb = slot(st + 1);
          const uint64_t a0 = smem_desc(s_base + sa * kSlabStride, 16, kHWB, 2);
          const uint64_t a1 = smem_desc(s_base + sb * kSlabStride, 16, kHWB, 2);
#pragma unroll 1
          for (int kh = 0; kh < 3; ++kh) {
            mbar_wait(&b_full[bs], bph);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t b_desc0 = B_MN ? smem_desc(b_base + bs * kBBytes, 8192, 1024, 2)
                                            : smem_desc(b_base + bs * kBBytes, 16, 1024, 2);
              const int vh = p.mirror ? 2 - kh : kh;
#pragma unroll
              for (int kw = 0; kw < 3; ++kw) {
                const int vw = p.mirror ? 2 - kw : kw;
                const uint32_t view = vh * kHWB + vw * 128;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const uint64_t bd = b_desc0 + ((kw * kTapBytes + k * (B_MN ? 2048 : 32)) >> 4);
                  const uint32_t accum = (kc | st | kh | kw | k) != 0;
                  mma(d0, a0 + ((view + k * 32) >> 4), bd, accum);
                  mma(d1, a1 + ((view + k * 32) >> 4), bd, accum);
                }
              }
              commit(&b_empty[bs]);
              if (kh == 2) {
                commit(&s_empty[sa]);
                if (st == 2) commit(&s_empty[sb]);
              }
            }
            __syncwarp();
            if (++bs == kZ2NB) {
              bs = 0;
              bph ^= 1;
            }
          }
        }
        ss += 4;
        if (ss >= kZ2Slabs) {
          ss -= kZ2Slabs;
          sph ^= 1;
        }
      }
      if (elect_one()) commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        tph ^= 1;
      }
    }
  } else if (warp >= 2) {
    const int q = warp & 3;
    const int ew = warp - 2;
    const int row = q * 32 + lane;
    const int lx = row & 7, ly = row >> 3;
    int acc = 0;
    uint32_t tph = 0;
    for (int it = item0; it < n_items; it += item_step) {
      bool real;
      const int tile = item_tile(it, real);
      int n, x0, y0, z0;
      decode(tile, n, x0, y0, z0);
      const int gx = x0 + lx, gy = y0 + ly;
      mbar_wait(&tfull_bar[acc], tph);
      tc_fence_after();
#pragma unroll 1
      for (int a = 0; a < 2; ++a) {
        const int gz = z0 + a;
        const bool valid = real && gx < p.Mw && gy < p.Mh && gz < p.Md;
        const int64_t ovox = (((int64_t)n * p.Md + gz) * p.Mh + gy) * p.Mw + gx;
        __nv_bfloat16* orow = p.out + ovox * p.out_cs;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint4 mk[4], xb[4];
          if (p.mask && valid) load32_bf16(p.mask + (orow - p.out) + c0, mk);
          if (p.bnx && valid) load32_bf16(p.bnx + ovox * p.Nout + c0, xb);
          uint32_t r[32];
          tmem_ld32(tmem_base + acc * 2 * BN + a * BN + c0 + ((uint32_t)(q * 32) << 16), r);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = valid ? __uint_as_float(r[j]) : 0.f;
          if (p.mask && valid) apply_relu_mask_reg(v, mk);
          if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 w;
              w.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
              w.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
              w.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
              w.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
              dst[j] = w;
            }
          }
          if (p.stats) {
            float s1, s2;
            if (p.bnx) {   // dgrad: fused BN-backward sums
              bn_bwd_colsums_reg(v, valid, xb, p.bn_stat + c0, p.bn_stat + p.Nout + c0, s1, s2);
            } else {
              float sq[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) sq[j] = v[j] * v[j];
              s1 = warp_colsum32(v);
              s2 = warp_colsum32(sq);
            }
            stat_w[ew][0][c0 + lane] += s1;
            stat_w[ew][1][c0 + lane] += s2;
          }
        }
      }
      tc_fence_before();
      if (PAIR && !leader) mbar_arrive_cluster(lead(&tempty_bar[acc]));
      else mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        tph ^= 1;
      }
    }
    if (p.stats) {
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int i = threadIdx.x - 64; i < 2 * BN; i += 128) {
        const int which = i / BN, c = i % BN;
        const float sum = ((stat_w[0][which][c] + stat_w[1][which][c]) + stat_w[2][which][c]) +
                          stat_w[3][which][c];
        p.stats[(int64_t)blockIdx.x * 2 * p.Nout + which * p.Nout + c] += sum;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) {
    cluster_sync();   // the peer's TMEM is read and its barriers idle before the pair frees
    if (warp == 1) tmem_dealloc_pair<256>(tmem_base);
  } else if (warp == 1) {
    tmem_dealloc<256>(tmem_base);
  }
}

// ---------------------------------------------------------------- halo wgrad
// dW[co][t][ci] = sum_v dY[v][co] X[v + off(t)][ci] for Cout == 64, Cin % 64 == 0.
// K = voxels in 8(w) x 16(h) x 1(d) blocks.  Per K block the producer stages the
// X halo of one 64-channel chunk (10 x 18 x 3 rows, 69 KB) and the dY tile (128
// rows x 64 channels); every tap operand is an MN-major *view* of the halo (8-row
// K groups at a 10-row stride).  One accumulator covers a tap pair: its M = 128
// rows are two 64-channel MN chunks (tap a, tap b) whose LBO is the row delta of
// the two views.  A work unit owns 7 tap pairs (taps 0-13 or 14-26) of one
// channel chunk for a K range, all 7 accumulators resident in TMEM (448 cols).
constexpr int kWgPairs = 7;

struct WgHaloParams {
  int Nb, D, H, W;
  int tw, th;                // K blocks per (w, h) ; depth uses D directly
  int kblocks;               // Nb * D * th * tw
  int chunks;                // Cin / 64
  int units;                 // 2 * chunks
  int splits;
  int x_c0, dy_c0;
  float* part;               // [splits][units][kWgPairs][128][64]
};

// Descriptor deltas, added to a per-stage base descriptor (start-address field =
// byte offset >> 4, LBO field at bit 16): tap view offsets, and for the tap-pair
// wgrad the (view of tap a, LBO = row distance to tap b) of each pair.
__constant__ uint32_t c_halo_off[27] = {
#define HO(t) (uint32_t)((((t) / 9 * kHH + ((t) / 3) % 3) * kHW + (t) % 3) * 128)
    HO(0),  HO(1),  HO(2),  HO(3),  HO(4),  HO(5),  HO(6),  HO(7),  HO(8),
    HO(9),  HO(10), HO(11), HO(12), HO(13), HO(14), HO(15), HO(16), HO(17),
    HO(18), HO(19), HO(20), HO(21), HO(22), HO(23), HO(24), HO(25), HO(26)};
#define PD(a, b) ((uint64_t)(HO(a) >> 4) | ((uint64_t)((HO(b) - HO(a)) >> 4) << 16))
__constant__ uint64_t c_pair_desc[2][7] = {
    {PD(0, 1), PD(2, 3), PD(4, 5), PD(6, 7), PD(8, 9), PD(10, 11), PD(12, 13)},
    {PD(14, 15), PD(16, 17), PD(18, 19), PD(20, 21), PD(22, 23), PD(24, 25), PD(26, 26)}};
#undef PD
#undef HO

// PAIR (Cin % 128 == 0): a CTA pair takes the same tap group and K range for two channel
// chunks (rank r: chunk 2 cp + r); M = 256 MMAs read each CTA's own halo views, and the dY
// tile is split by N (32 output channels per CTA, 64-byte SWIZZLE_64B rows), so each SM
// feeds 4 + 1 KB per K16 step and stages half the dY bytes.
template <bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_wgrad_halo(const __grid_constant__ Maps maps, const __grid_constant__ WgHaloParams p) {
  constexpr int kDyBytes = PAIR ? 128 * 64 : 128 * 128;
  constexpr int kStage = kHaloStride + kDyBytes;
  constexpr int kStages = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int kper = (p.kblocks + p.splits - 1) / p.splits;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  // work items: (unit, split); PAIR: (unit pair = (group, chunk pair), split)
  const int units_i = PAIR ? p.units / 2 : p.units;
  const int work = units_i * p.splits;
  const int item0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int item_step = PAIR ? gridDim.x / 2 : gridDim.x;
  auto item_unit = [&](int u, int& split) {   // unit = chunk * 2 + group of this CTA
    const int ui = u % units_i;
    split = u / units_i;
    if (!PAIR) return ui;
    const int group = ui & 1, cp = ui >> 1;
    return (2 * cp + (int)rank) * 2 + group;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&tfull_bar, 1);
    mbar_init(&tempty_bar, PAIR ? 256 : 128);
    fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair<512>(&tmem_base_s);
    else tmem_alloc<512>(&tmem_base_s);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  auto lead = [&](uint64_t* bar) { return PAIR ? mapa_shared(smem_u32(bar), 0) : smem_u32(bar); };

  if (warp == 0) {
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      for (int u = item0; u < work; u += item_step) {
        int split;
        const int unit = item_unit(u, split);
        int chunk = unit >> 1;
        int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
        for (int kb = kb0; kb < kb1; ++kb) {
          int tx = kb % p.tw;
          int r = kb / p.tw;
          int ty = r % p.th;
          r /= p.th;
          int z = r % p.D;
          int n = r / p.D;
          mbar_wait(&empty_bar[st], ph ^ 1);
          uint8_t* s0 = smem + st * kStage;
          int xc = p.x_c0 + chunk * 64;
          const CUtensorMap* xm = act_map(maps, 0, xc);
          if (PAIR) {
            if (leader) mbar_arrive_expect_tx(&full_bar[st], 2 * (kHaloBytes + kDyBytes));
            tma_load_5d_pair(s0, xm, lead(&full_bar[st]), xc, tx * 8 - 1, ty * 16 - 1, z - 1, n);
            tma_load_5d_pair(s0 + kHaloStride, &maps.a[1], lead(&full_bar[st]),
                             p.dy_c0 + 32 * (int)rank, tx * 8, ty * 16, z, n);
          } else {
            mbar_arrive_expect_tx(&full_bar[st], kHaloBytes + kDyBytes);
            tma_load_5d(s0, xm, &full_bar[st], xc, tx * 8 - 1, ty * 16 - 1, z - 1, n);
            tma_load_5d(s0 + kHaloStride, &maps.a[1], &full_bar[st], p.dy_c0, tx * 8, ty * 16,
                        z, n);
          }
          if (++st == kStages) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    constexpr uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, 64, 1, 1);
    const uint32_t base = smem_u32(smem);
    int st = 0;
    uint32_t ph = 0, tph = 0;
    for (int u = item0; u < work; u += item_step) {
      int split;
      const int unit = item_unit(u, split);
      int group = unit & 1;
      int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
      mbar_wait(&tempty_bar, tph ^ 1);
      tc_fence_after();
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[st], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t hx = base + st * kStage;
          const uint64_t hx_desc = smem_desc(hx, 0, kHW * 128, 2);
          // dY as MN-major B: 128-byte rows (64 co), or PAIR 64-byte rows (32 co, SW64)
          const uint64_t dy_desc = PAIR ? smem_desc(hx + kHaloStride, 4096, 512, 4)
                                        : smem_desc(hx + kHaloStride, 8192, 1024, 2);
#pragma unroll
          for (int q = 0; q < kWgPairs; ++q) {
            const uint64_t a0 = hx_desc + c_pair_desc[group][q];
            const uint32_t dtm = tmem_base + q * 64;
#pragma unroll
            for (int k = 0; k < 8; ++k) {   // 16 voxels per MMA: two 8-voxel h rows
              const uint64_t ad = a0 + ((k * 2 * kHW * 128) >> 4);
              const uint64_t bd = dy_desc + ((k * 16 * (kDyBytes / 128)) >> 4);
              if (PAIR) umma_bf16_pair(dtm, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
              else umma_bf16(dtm, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
            }
          }
          if (PAIR) umma_commit_pair(&empty_bar[st], 0x3);
          else umma_commit(&empty_bar[st]);
        }
        __syncwarp();
        if (++st == kStages) {
          st = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) {
        if (PAIR) umma_commit_pair(&tfull_bar, 0x3);
        else umma_commit(&tfull_bar);
      }
      __syncwarp();
      tph ^= 1;
    }
  } else if (warp >= 2) {
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    uint32_t tph = 0;
    for (int u = item0; u < work; u += item_step) {
      int split;
      const int unit = item_unit(u, split);
      int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
      bool empty = kb1 <= kb0;
      mbar_wait(&tfull_bar, tph);
      tc_fence_after();
#pragma unroll 1
      for (int q = 0; q < kWgPairs; ++q) {
        float* dst = p.part + ((((int64_t)split * p.units + unit) * kWgPairs + q) * 128 + row) * 64;
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(tmem_base + q * 64 + c0 + ((uint32_t)(q4 * 32) << 16), r);
          tmem_ld_wait();
          float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            d4[j] = empty ? make_float4(0.f, 0.f, 0.f, 0.f)
                          : make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                        __uint_as_float(r[4 * j + 2]),
                                        __uint_as_float(r[4 * j + 3]));
        }
      }
      tc_fence_before();
      if (PAIR && !leader) mbar_arrive_cluster(lead(&tempty_bar));
      else mbar_arrive(&tempty_bar);
      tph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) {
    cluster_sync();
    if (warp == 1) tmem_dealloc_pair<512>(tmem_base);
  } else if (warp == 1) {
    tmem_dealloc<512>(tmem_base);
  }
}

__global__ void k_wgrad_halo_reduce(WgHaloParams p, int Cin, float* __restrict__ gw) {
  int64_t per_unit = (int64_t)kWgPairs * 128 * 64;
  int64_t total = per_unit * p.units;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int unit = (int)(i / per_unit);
    int rem = (int)(i % per_unit);
    int q = rem / (128 * 64);
    int m = (rem / 64) % 128;
    int co = rem % 64;
    int group = unit & 1, chunk = unit >> 1;
    int tap = group * 14 + 2 * q + (m >= 64 ? 1 : 0);
    if (tap >= 27) continue;
    int ci = chunk * 64 + (m & 63);
    float s = 0.f;
    for (int sp = 0; sp < p.splits; ++sp)
      s += p.part[((int64_t)sp * p.units) * per_unit + i];
    gw[((int64_t)co * 27 + tap) * Cin + ci] = s;
  }
}

// Halo wgrad for Cout >= 128: D[128 co][64 ci] per tap, A = dY tile (two 64-channel
// MN chunks), B = halo view of one 64-channel X chunk.  A work unit owns 8 taps of
// one (co block, ci chunk) pair -- 8 accumulators x 64 columns = all 512 TMEM
// columns -- for a K range; per K block: 8 taps x 8 MMAs from one 101 KB stage.
constexpr int kWgTaps = 8;

struct WgHaloAParams {
  int Nb, D, H, W;
  int tw, th, kblocks;
  int cchunks, coblocks;     // Cin / 64, Cout / 128
  int units;                 // cchunks * 4 * coblocks
  int splits;
  int x_c0, dy_c0, Cin;
  float* part;               // [splits][units][kWgTaps][128][64]
};

__global__ void __launch_bounds__(kThreads, 1)
    k_wgrad_halo_a(const __grid_constant__ Maps maps, const __grid_constant__ WgHaloAParams p) {
  constexpr int kDyBytes = 2 * 128 * 128;   // 128 voxels x 128 channels
  constexpr int kStage = kHaloStride + kDyBytes;
  constexpr int kStages = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int work = p.units * p.splits;
  const int kper = (p.kblocks + p.splits - 1) / p.splits;
  // unit -> (ci chunk, tap group, co block)
  auto decode = [&](int unit, int& cc, int& tg, int& cb) {
    cc = unit % p.cchunks;
    int r = unit / p.cchunks;
    tg = r % 4;
    cb = r / 4;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&tfull_bar, 1);
    mbar_init(&tempty_bar, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;

  if (warp == 0) {
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < work; u += gridDim.x) {
        int unit = u % p.units, split = u / p.units;
        int cc, tg, cb;
        decode(unit, cc, tg, cb);
        int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
        for (int kb = kb0; kb < kb1; ++kb) {
          int tx = kb % p.tw;
          int r = kb / p.tw;
          int ty = r % p.th;
          r /= p.th;
          int z = r % p.D;
          int n = r / p.D;
          mbar_wait(&empty_bar[st], ph ^ 1);
          uint8_t* s0 = smem + st * kStage;
          mbar_arrive_expect_tx(&full_bar[st], kHaloBytes + kDyBytes);
          int xc = p.x_c0 + cc * 64;
          const CUtensorMap* xm = act_map(maps, 0, xc);
          tma_load_5d(s0, xm, &full_bar[st], xc, tx * 8 - 1, ty * 16 - 1, z - 1, n);
#pragma unroll
          for (int j = 0; j < 2; ++j)
            tma_load_5d(s0 + kHaloStride + j * 16384, &maps.a[1], &full_bar[st],
                        p.dy_c0 + cb * 128 + j * 64, tx * 8, ty * 16, z, n);
          if (++st == kStages) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, 64, 1, 1);
    const uint32_t base = smem_u32(smem);
    int st = 0;
    uint32_t ph = 0, tph = 0;
    for (int u = blockIdx.x; u < work; u += gridDim.x) {
      int unit = u % p.units, split = u / p.units;
      int cc, tg, cb;
      decode(unit, cc, tg, cb);
      int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
      int ntaps = min(kWgTaps, 27 - tg * kWgTaps);
      mbar_wait(&tempty_bar, tph ^ 1);
      tc_fence_after();
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[st], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t hx = base + st * kStage;
          const uint64_t dy_desc = smem_desc(hx + kHaloStride, 16384, 1024, 2);
          const uint64_t hx_desc = smem_desc(hx, 16, kHW * 128, 2);
#pragma unroll 1
          for (int q = 0; q < ntaps; ++q) {
            const uint64_t b0 = hx_desc + (c_halo_off[tg * kWgTaps + q] >> 4);
            const uint32_t dtm = tmem_base + q * 64;
#pragma unroll
            for (int k = 0; k < 8; ++k)
              umma_bf16(dtm, dy_desc + ((k * 2048) >> 4), b0 + ((k * 2 * kHW * 128) >> 4), idesc,
                        (kb != kb0 || k != 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[st]);
        }
        __syncwarp();
        if (++st == kStages) {
          st = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull_bar);
      __syncwarp();
      tph ^= 1;
    }
  } else {
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    uint32_t tph = 0;
    for (int u = blockIdx.x; u < work; u += gridDim.x) {
      int unit = u % p.units, split = u / p.units;
      int cc, tg, cb;
      decode(unit, cc, tg, cb);
      int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
      bool empty = kb1 <= kb0;
      int ntaps = min(kWgTaps, 27 - tg * kWgTaps);
      mbar_wait(&tfull_bar, tph);
      tc_fence_after();
#pragma unroll 1
      for (int q = 0; q < ntaps; ++q) {
        float* dst = p.part + ((((int64_t)split * p.units + unit) * kWgTaps + q) * 128 + row) * 64;
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(tmem_base + q * 64 + c0 + ((uint32_t)(q4 * 32) << 16), r);
          tmem_ld_wait();
          float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            d4[j] = empty ? make_float4(0.f, 0.f, 0.f, 0.f)
                          : make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                        __uint_as_float(r[4 * j + 2]),
                                        __uint_as_float(r[4 * j + 3]));
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar);
      tph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem_base);
}

__global__ void k_wgrad_halo_a_reduce(WgHaloAParams p, float* __restrict__ gw) {
  int64_t per_unit = (int64_t)kWgTaps * 128 * 64;
  int64_t total = per_unit * p.units;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int unit = (int)(i / per_unit);
    int rem = (int)(i % per_unit);
    int q = rem / (128 * 64);
    int m = (rem / 64) % 128;
    int nn = rem % 64;
    int cc = unit % p.cchunks;
    int r = unit / p.cchunks;
    int tg = r % 4, cb = r / 4;
    int tap = tg * kWgTaps + q;
    if (tap >= 27) continue;
    int co = cb * 128 + m, ci = cc * 64 + nn;
    float s = 0.f;
    for (int sp = 0; sp < p.splits; ++sp)
      s += p.part[((int64_t)sp * p.units) * per_unit + i];
    gw[((int64_t)co * 27 + tap) * p.Cin + ci] = s;
  }
}

// ---------------------------------------------------------------- halo-view wgrad
// Weight gradient with BOTH operands as shifted views, so every MMA is 128 x 192 x 16 and
// tensor-bound (the N = 64 halo kernels above are shared-memory-feed bound: 6 KB of operands
// per 32 tensor clocks).  K = voxels in 8(w) x 8(h) x 2(d) blocks (128 voxels).
//
//   XA (Cout == 64): A = X views of (kd, kh) pairs -- M = 2 views x 64 ci, MN-major, the
//     two views LBO apart -- from an (8, 10, 4) X box with no w halo; B = the 3 w-shifted
//     views of a (10, 8, 2) dY box, N = 3 x 64 co, LBO = one 128-byte row.  The product of
//     X[u + (kd-1, kh-1, 0)] and dY[u + (0, 0, s)] summed over u is tap (kd, kh, 1 - s).
//     5 view pairs (the 9th view paired with itself) per 64-channel X chunk.
//   XB (Cout % 128 == 0): A = dY (M = 128 co, two 64-co chunks), B = the kw = 0, 1, 2
//     views of (kd, kh) in a (10, 10, 4) X box, N = 3 x 64 ci.  9 views per (co block,
//     ci chunk).
//
// A work unit owns 2 accumulators (2 x 192 TMEM columns) of one chunk for a K range;
// the fp32 partials are reduced in a fixed order by k_wgrad_hv_reduce.
constexpr int kHvAcc = 2;                         // accumulators per unit
constexpr int kHvN = 192;                         // 3 views x 64 channels
constexpr int kHvXaXRows = 8 * 10 * 4;            // XA X box rows (w, h, d)
constexpr int kHvXaDyRows = 10 * 8 * 2;           // XA dY box rows
constexpr int kHvXbXRows = 10 * 10 * 4;           // XB X box rows
constexpr int kHvXaStage = (kHvXaXRows + kHvXaDyRows) * 128;   // 61440
constexpr int kHvXbStage = kHvXbXRows * 128 + 2 * 128 * 128;  // 83968
constexpr int kHvXaStages = 3, kHvXbStages = 2;

struct WgHvParams {
  int Nb, D, H, W;
  int tw, th, td;          // K blocks per dim (8, 8, 2 voxels)
  int kblocks;
  int cchunks, coblocks;   // Cin / 64, XB: Cout / 128 (XA: 1)
  int groups;              // units per chunk: XA 3 (pairs {0,1},{2,3},{4}), XB 5
  int units;               // cchunks * coblocks * groups
  int splits;
  int x_c0, dy_c0, Cin;
  float* part;             // [splits][units][kHvAcc][128][kHvN]
};

// First row of view v = (kd, kh) = (v / 3, v % 3) in the X box: XA (8, 10, 4) box without
// a w halo, XB (10, 10, 4) box (its kw views are the next rows)
__device__ __forceinline__ int hv_view_row_xa(int v) { return ((v / 3) * 10 + v % 3) * 8; }
__device__ __forceinline__ int hv_view_row_xb(int v) { return ((v / 3) * 10 + v % 3) * 10; }

template <bool XA>
__global__ void __launch_bounds__(kThreads, 1)
    k_wgrad_hv(const __grid_constant__ Maps maps, const __grid_constant__ WgHvParams p) {
  constexpr int kStage = XA ? kHvXaStage : kHvXbStage;
  constexpr int kStages = XA ? kHvXaStages : kHvXbStages;
  constexpr int kXBytes = (XA ? kHvXaXRows : kHvXbXRows) * 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int work = p.units * p.splits;
  const int kper = (p.kblocks + p.splits - 1) / p.splits;
  // unit -> (ci chunk, co block, group); accumulators in the group
  auto decode = [&](int unit, int& cc, int& cb, int& grp) {
    cc = unit % p.cchunks;
    const int r = unit / p.cchunks;
    grp = r % p.groups;
    cb = r / p.groups;
  };
  auto n_acc = [&](int grp) { return grp == p.groups - 1 ? 1 : kHvAcc; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&tfull_bar, 1);
    mbar_init(&tempty_bar, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_s);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&maps.a[0]);
    tma_prefetch(&maps.a[1]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;

  if (warp == 0) {
    if (elect_one()) {
      int st = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < work; u += gridDim.x) {
        const int unit = u % p.units, split = u / p.units;
        int cc, cb, grp;
        decode(unit, cc, cb, grp);
        const int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
        for (int kb = kb0; kb < kb1; ++kb) {
          const int tx = kb % p.tw;
          int r = kb / p.tw;
          const int ty = r % p.th;
          r /= p.th;
          const int tz = r % p.td;
          const int n = r / p.td;
          mbar_wait(&empty_bar[st], ph ^ 1);
          uint8_t* s0 = smem + st * kStage;
          mbar_arrive_expect_tx(&full_bar[st], kStage);
          int xc = p.x_c0 + cc * 64;
          const CUtensorMap* xm = act_map(maps, 0, xc);
          if (XA) {
            tma_load_5d(s0, xm, &full_bar[st], xc, tx * 8, ty * 8 - 1, tz * 2 - 1, n);
            tma_load_5d(s0 + kXBytes, &maps.a[1], &full_bar[st], p.dy_c0, tx * 8 - 1, ty * 8,
                        tz * 2, n);
          } else {
            tma_load_5d(s0, xm, &full_bar[st], xc, tx * 8 - 1, ty * 8 - 1, tz * 2 - 1, n);
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_5d(s0 + kXBytes + j * 16384, &maps.a[1], &full_bar[st],
                          p.dy_c0 + cb * 128 + j * 64, tx * 8, ty * 8, tz * 2, n);
          }
          if (++st == kStages) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, kHvN, 1, 1);
    const uint32_t base = smem_u32(smem);
    int st = 0;
    uint32_t ph = 0, tph = 0;
    for (int u = blockIdx.x; u < work; u += gridDim.x) {
      const int unit = u % p.units, split = u / p.units;
      int cc, cb, grp;
      decode(unit, cc, cb, grp);
      const int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
      const int nacc = n_acc(grp);
      mbar_wait(&tempty_bar, tph ^ 1);
      tc_fence_after();
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[st], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sx = base + st * kStage;
          const uint32_t sy = sx + kXBytes;
#pragma unroll 1
          for (int a = 0; a < nacc; ++a) {
            const int v0 = 2 * (grp * kHvAcc + a);   // XA: first view of the pair
            const uint32_t dtm = tmem_base + a * 256;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const int d = kk >> 2, h = 2 * (kk & 3);   // K rows h, h+1 of plane d
              uint64_t ad, bd;
              if (XA) {
                const int va = v0, vb = min(v0 + 1, 8);
                const uint32_t ra = hv_view_row_xa(va) + (d * 10 + h) * 8;
                ad = smem_desc(sx + ra * 128, (hv_view_row_xa(vb) - hv_view_row_xa(va)) * 128,
                               8 * 128, 2);
                bd = smem_desc(sy + (d * 8 + h) * 10 * 128, 128, 10 * 128, 2);
              } else {
                const int v = grp * kHvAcc + a;   // XB: one (kd, kh) view per accumulator
                ad = smem_desc(sy + kk * 2048, 16384, 1024, 2);
                bd = smem_desc(sx + (hv_view_row_xb(v) + (d * 10 + h) * 10) * 128, 128,
                               10 * 128, 2);
              }
              umma_bf16(dtm, ad, bd, idesc, (kb != kb0 || kk != 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty_bar[st]);
        }
        __syncwarp();
        if (++st == kStages) {
          st = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull_bar);
      __syncwarp();
      tph ^= 1;
    }
  } else {
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    uint32_t tph = 0;
    for (int u = blockIdx.x; u < work; u += gridDim.x) {
      const int unit = u % p.units, split = u / p.units;
      int cc, cb, grp;
      decode(unit, cc, cb, grp);
      const int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
      const bool empty = kb1 <= kb0;
      const int nacc = n_acc(grp);
      mbar_wait(&tfull_bar, tph);
      tc_fence_after();
#pragma unroll 1
      for (int a = 0; a < nacc; ++a) {
        float* dst = p.part + ((((int64_t)split * p.units + unit) * kHvAcc + a) * 128 + row) * kHvN;
#pragma unroll 1
        for (int c0 = 0; c0 < kHvN; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(tmem_base + a * 256 + c0 + ((uint32_t)(q4 * 32) << 16), r);
          tmem_ld_wait();
          float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            d4[j] = empty ? make_float4(0.f, 0.f, 0.f, 0.f)
                          : make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                        __uint_as_float(r[4 * j + 2]),
                                        __uint_as_float(r[4 * j + 3]));
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar);
      tph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem_base);
}

// gw[co][tap][ci] = sum over splits (fixed order) of the partial element that holds it.
template <bool XA>
__global__ void k_wgrad_hv_reduce(WgHvParams p, float* __restrict__ gw) {
  const int64_t per_unit = (int64_t)kHvAcc * 128 * kHvN;
  const int64_t total = per_unit * p.units;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int unit = (int)(i / per_unit);
    const int rem = (int)(i % per_unit);
    const int a = rem / (128 * kHvN);
    const int m = (rem / kHvN) % 128;
    const int nn = rem % kHvN;
    const int cc = unit % p.cchunks;
    const int r = unit / p.cchunks;
    const int grp = r % p.groups, cb = r / p.groups;
    if (grp == p.groups - 1 && a > 0) continue;
    int co, ci, tap;
    if (XA) {
      const int v0 = 2 * (grp * kHvAcc + a);
      const int v = m < 64 ? v0 : v0 + 1;
      if (v > 8) continue;                       // the 9th view's duplicate half
      const int kw = 2 - nn / 64;                // N chunk j = w shift j - 1 = tap kw 2 - j
      tap = v * 3 + kw;
      ci = cc * 64 + (m & 63);
      co = nn % 64;
    } else {
      const int v = grp * kHvAcc + a;
      tap = v * 3 + nn / 64;
      ci = cc * 64 + nn % 64;
      co = cb * 128 + m;
    }
    float s = 0.f;
    for (int sp = 0; sp < p.splits; ++sp) s += p.part[((int64_t)sp * p.units) * per_unit + i];
    gw[((int64_t)co * 27 + tap) * p.Cin + ci] = s;
  }
}

// ---------------------------------------------------------------- wgrad
struct WgParams {
  int mode;                    // 0: conv (X shifted by tap), 1: convT (dY parity view shifted)
  int caseA;                   // 1: A = dY (2 chunks of Cout), B = X/taps ; 0: A = X, B = dY
  int Cin, Cout;
  int bnp;                     // N' of the tile (multiple of 64)
  int tiles, splits, kblocks;  // tiles, K splits, K blocks in the grid
  int Nb, D, H, W;             // K grid (voxels)
  int kbd, kbh, kbw, ktd, kth, ktw;
  int x_c0, dy_c0;             // channel offsets (slices)
  int aw;                      // channels per A chunk (64, or 32 for a 32-channel input)
  int gw_co_stride, gw_cmax;   // gw[co * gw_co_stride + tap * Cin + ci], ci < gw_cmax
  float* part;                 // [splits][rtiles][128][bnp]
  float* gw;                   // splits == 1: the epilogue writes gw[co][tap][ci] directly
  int tt;                      // taps per work unit (convT, Cout == 64: the X chunk is shared
                               // by all taps, so a unit loads it once for tt taps' dY views)
  int rtiles;                  // tiles of the part / gw layout (== tiles when tt == 1)
};

struct Chunk {
  int map;   // 0 = X map, 1..8 = dY (conv: 1; convT: 1 + parity index)
  int c0;
  int dx, dy, dz;
};

__device__ __forceinline__ void tap_shift(int mode, int tap, int& map, int& dx, int& dy, int& dz) {
  int kd = tap / 9, kh = (tap / 3) % 3, kw = tap % 3;
  if (mode == 0) {
    map = 0;
    dx = kw - 1; dy = kh - 1; dz = kd - 1;
  } else {  // dY[2i-1+k]: k=0 -> odd view j=i-1 ; k=1 -> even j=i ; k=2 -> odd j=i
    int pz = kd != 1, py = kh != 1, px = kw != 1;
    map = 1 + (pz * 4 + py * 2 + px);
    dz = kd == 0 ? -1 : 0; dy = kh == 0 ? -1 : 0; dx = kw == 0 ? -1 : 0;
  }
}

// Describe the A (128/aw chunks of aw channels) and B (bnp/64 chunks) operands of a tile.
__device__ void wg_tile(const WgParams& p, int tile, Chunk (&a)[4], Chunk (&b)[4], int& nb) {
  nb = p.bnp / 64;
  const int na = 128 / p.aw;
  if (p.caseA) {
    // tiles over (tap, co-block of 128, ci-block of bnp)
    int cblocks = p.Cin / p.bnp, nblocks = p.Cout / 128;
    int cb = tile % cblocks;
    int r = tile / cblocks;
    int nbk = r % nblocks;
    int tap = r / nblocks;
    int smap, sdx, sdy, sdz;
    tap_shift(p.mode, tap, smap, sdx, sdy, sdz);
    for (int j = 0; j < na; ++j) {   // A = dY channels
      a[j].c0 = p.dy_c0 + nbk * 128 + j * p.aw;
      if (p.mode == 1) { a[j].map = smap; a[j].dx = sdx; a[j].dy = sdy; a[j].dz = sdz; }
      else { a[j].map = 1; a[j].dx = a[j].dy = a[j].dz = 0; }
    }
    for (int j = 0; j < nb; ++j) {  // B = X channels
      b[j].c0 = p.x_c0 + cb * p.bnp + j * 64;
      if (p.mode == 0) { b[j].map = smap; b[j].dx = sdx; b[j].dy = sdy; b[j].dz = sdz; }
      else { b[j].map = 0; b[j].dx = b[j].dy = b[j].dz = 0; }
    }
  } else {
    // Cout == 64: A = X chunks -- several taps of a narrow Cin (<= 64), or
    // 128-channel blocks of one tap.
    int tapA[4], cA[4];
    if (p.Cin <= 64) {
      for (int j = 0; j < na; ++j) {
        int t = na * tile + j;
        tapA[j] = t < 27 ? t : 26;
        cA[j] = 0;
      }
    } else {
      int cblocks = p.Cin / 128;
      int cb = tile % cblocks;
      for (int j = 0; j < na; ++j) {
        tapA[j] = tile / cblocks;
        cA[j] = cb * 128 + j * p.aw;
      }
    }
    for (int j = 0; j < na; ++j) {
      a[j].c0 = p.x_c0 + cA[j];
      if (p.mode == 0) {
        tap_shift(0, tapA[j], a[j].map, a[j].dx, a[j].dy, a[j].dz);
      } else {
        a[j].map = 0; a[j].dx = a[j].dy = a[j].dz = 0;
      }
    }
    nb = 1;
    b[0].c0 = p.dy_c0;
    if (p.mode == 0) {
      b[0].map = 1; b[0].dx = b[0].dy = b[0].dz = 0;
    } else {
      tap_shift(1, tapA[0], b[0].map, b[0].dx, b[0].dy, b[0].dz);
    }
  }
}

// gw index of element (m, nn) of tile `tile`, or -1 when it is padding.
__device__ __forceinline__ int64_t wg_out_index(const WgParams& p, int tile, int m, int nn) {
  int co, ci, tap;
  if (p.caseA) {
    int cblocks = p.Cin / p.bnp, nblocks = p.Cout / 128;
    int cb = tile % cblocks;
    int r = tile / cblocks;
    int nbk = r % nblocks;
    tap = r / nblocks;
    co = nbk * 128 + m;
    ci = cb * p.bnp + nn;
  } else {
    co = nn;
    if (p.Cin <= 64) {
      tap = (128 / p.aw) * tile + m / p.aw;
      if (tap >= 27) return -1;
      ci = m % p.aw;
    } else {
      int cblocks = p.Cin / 128;
      tap = tile / cblocks;
      ci = (tile % cblocks) * 128 + m;
    }
  }
  if (ci >= p.gw_cmax) return -1;
  return (int64_t)co * p.gw_co_stride + (int64_t)tap * p.Cin + ci;
}

// PAIR (caseA, Cout >= 256): a CTA pair takes the same (tap, ci block, K range) for two
// output-channel blocks (rank r: block 2 pb + r); M = 256 MMAs read each CTA's own dY chunks
// (A) and half of the X chunks (B, split by N: ci chunks 2r, 2r+1 of the block).
template <int BNP, int KB, int AW, int TT = 1, bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_wgrad(const __grid_constant__ Maps maps, const __grid_constant__ WgParams p) {
  // TT > 1 (convT, Cout == 64, BNP == 64): a unit = (ci block, group of TT taps); per K
  // block one X chunk (A) and TT dY parity views (B), TT accumulators
  constexpr int kChunkBytes = KB * 128;             // B chunk: 64 channels x KB voxels
  constexpr int kAChunk = KB * AW * 2;              // A chunk: AW channels x KB voxels
  constexpr int kNA = 128 / AW;
  constexpr int kNB = BNP / 64 * TT / (PAIR ? 2 : 1);
  static_assert(!PAIR || (TT == 1 && BNP == 256), "pair: caseA with 256-wide N tiles");
  constexpr int kABytes = kNA * kAChunk;
  constexpr int kStageBytes = kABytes + kNB * kChunkBytes;
  constexpr int kStagesRaw = kSmemBudget / kStageBytes;
  constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
  constexpr int kAccCols = TT * BNP;
  constexpr uint32_t kTmemCols = (2 * kAccCols <= 128) ? 128 : (2 * kAccCols <= 256) ? 256 : 512;
  static_assert(TT == 1 || BNP == 64, "multi-tap units are for 64 output channels");
  static_assert(2 * kAccCols <= 512, "accumulators exceed TMEM");
  static_assert(kStages >= 2, "pipeline too shallow");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int kper = (p.kblocks + p.splits - 1) / p.splits;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int tiles_i = PAIR ? p.tiles / 2 : p.tiles;   // work items per split
  const int units = tiles_i * p.splits;
  const int item0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int item_step = PAIR ? gridDim.x / 2 : gridDim.x;
  auto item_tile = [&](int u, int& split) {
    const int ti = u % tiles_i;
    split = u / tiles_i;
    if (!PAIR) return ti;
    const int cblocks = p.Cin / p.bnp, nblocks = p.Cout / 128;
    const int cb = ti % cblocks, r = ti / cblocks;
    const int pnb = r % (nblocks / 2), tap = r / (nblocks / 2);
    return (tap * nblocks + 2 * pnb + (int)rank) * cblocks + cb;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], PAIR ? 256 : 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair<kTmemCols>(&tmem_base_s);
    else tmem_alloc<kTmemCols>(&tmem_base_s);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  auto lead = [&](uint64_t* bar) { return PAIR ? mapa_shared(smem_u32(bar), 0) : smem_u32(bar); };

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = item0; u < units; u += item_step) {
        int split;
        const int tile = item_tile(u, split);
        Chunk a[4], b[4];
        int nb;
        const int cblocks = p.Cin / 128;
        if (TT > 1) {   // tile = (tap group, ci block): A from the group's first tap
          wg_tile(p, (tile / cblocks) * TT * cblocks + tile % cblocks, a, b, nb);
        } else {
          wg_tile(p, tile, a, b, nb);
        }
        Chunk bt[TT];
        if (TT > 1) {
#pragma unroll
          for (int j = 0; j < TT; ++j) {
            int tap = (tile / cblocks) * TT + j;
            if (tap > 26) tap = 26;   // padding tap: loaded, accumulated, never written
            bt[j].c0 = p.dy_c0;
            tap_shift(1, tap, bt[j].map, bt[j].dx, bt[j].dy, bt[j].dz);
          }
        }
        int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
        for (int kb = kb0; kb < kb1; ++kb) {
          int tx = kb % p.ktw;
          int r = kb / p.ktw;
          int ty = r % p.kth;
          r /= p.kth;
          int tz = r % p.ktd;
          int n = r / p.ktd;
          int x0 = tx * p.kbw, y0 = ty * p.kbh, z0 = tz * p.kbd;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* s0 = smem + stage * kStageBytes;
          if (PAIR) {
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * kStageBytes);
#pragma unroll
            for (int j = 0; j < kNA; ++j) {
              int c0 = a[j].c0;
              const CUtensorMap* m = act_map(maps, a[j].map, c0);
              tma_load_5d_pair(s0 + j * kAChunk, m, lead(&full_bar[stage]), c0, x0 + a[j].dx,
                               y0 + a[j].dy, z0 + a[j].dz, n);
            }
#pragma unroll
            for (int j = 0; j < kNB; ++j) {   // this CTA's half of the X chunks
              const Chunk& c = b[kNB * (int)rank + j];
              int c0 = c.c0;
              const CUtensorMap* m = act_map(maps, c.map, c0);
              tma_load_5d_pair(s0 + kABytes + j * kChunkBytes, m, lead(&full_bar[stage]), c0,
                               x0 + c.dx, y0 + c.dy, z0 + c.dz, n);
            }
          } else {
          mbar_arrive_expect_tx(&full_bar[stage], kStageBytes);
#pragma unroll
          for (int j = 0; j < kNA; ++j) {
            int c0 = a[j].c0;
            const CUtensorMap* m = act_map(maps, a[j].map, c0);
            tma_load_5d(s0 + j * kAChunk, m, &full_bar[stage], c0, x0 + a[j].dx,
                        y0 + a[j].dy, z0 + a[j].dz, n);
          }
          if (TT > 1) {
#pragma unroll
            for (int j = 0; j < TT; ++j)
              tma_load_5d(s0 + kABytes + j * kChunkBytes, &maps.a[bt[j].map], &full_bar[stage],
                          bt[j].c0, x0 + bt[j].dx, y0 + bt[j].dy, z0 + bt[j].dz, n);
          } else {
#pragma unroll
            for (int j = 0; j < kNB; ++j) {
              int c0 = b[j].c0;
              const CUtensorMap* m = act_map(maps, b[j].map, c0);
              tma_load_5d(s0 + kABytes + j * kChunkBytes, m, &full_bar[stage], c0,
                          x0 + b[j].dx, y0 + b[j].dy, z0 + b[j].dz, n);
            }
          }
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    constexpr uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, BNP, 1, 1);
    const uint32_t smem_base = smem_u32(smem);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int u = item0; u < units; u += item_step) {
      int split;
      item_tile(u, split);
      int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
      mbar_wait(&tempty_bar[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t dtmem = tmem_base + acc * kAccCols;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_base + stage * kStageBytes;
          const uint32_t sb = sa + kABytes;
#pragma unroll
          for (int j = 0; j < TT; ++j) {
#pragma unroll
            for (int k = 0; k < KB / 16; ++k) {
              uint64_t ad = smem_desc(sa + k * 16 * AW * 2, kAChunk, 8 * AW * 2,
                                      swizzle_code(AW * 2));
              uint64_t bd = smem_desc(sb + j * kChunkBytes + k * 2048, kChunkBytes, 1024, 2);
              if (PAIR) umma_bf16_pair(dtmem + j * BNP, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
              else umma_bf16(dtmem + j * BNP, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
            }
          }
          if (PAIR) umma_commit_pair(&empty_bar[stage], 0x3);
          else umma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) {
        if (PAIR) umma_commit_pair(&tfull_bar[acc], 0x3);
        else umma_commit(&tfull_bar[acc]);
      }
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  } else if (warp >= 2) {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int acc = 0;
    uint32_t aphase = 0;
    for (int u = item0; u < units; u += item_step) {
      int split;
      const int utile = item_tile(u, split);
      int kb0 = split * kper, kb1 = min(p.kblocks, kb0 + kper);
      mbar_wait(&tfull_bar[acc], aphase);
      tc_fence_after();
#pragma unroll 1
      for (int jt = 0; jt < TT; ++jt) {
      int tile = utile;
      if (TT > 1) {   // real (tap, ci block) tile of accumulator jt
        const int cblocks = p.Cin / 128;
        const int tap = (utile / cblocks) * TT + jt;
        if (tap > 26) break;
        tile = tap * cblocks + utile % cblocks;
      }
      float* dst = p.part + (((int64_t)split * p.rtiles + tile) * 128 + row) * BNP;
#pragma unroll 1
      for (int c0 = 0; c0 < BNP; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + acc * kAccCols + jt * BNP + c0 + ((uint32_t)(q * 32) << 16), r);
        tmem_ld_wait();
        bool empty = kb1 <= kb0;
        if (p.gw) {   // single K split: scatter straight into the gradient buffer
          if (p.caseA) {   // row = co, the 32 columns are consecutive ci
            const int64_t o = wg_out_index(p, tile, row, c0);
            float4* g4 = reinterpret_cast<float4*>(p.gw + o);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              g4[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                  __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int64_t o = wg_out_index(p, tile, row, c0 + j);
              if (o >= 0) p.gw[o] = __uint_as_float(r[j]);
            }
          }
          continue;
        }
        float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          d4[j] = empty ? make_float4(0.f, 0.f, 0.f, 0.f)
                        : make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                      __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
      }
      }
      tc_fence_before();
      if (PAIR && !leader) mbar_arrive_cluster(lead(&tempty_bar[acc]));
      else mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) {
    cluster_sync();
    if (warp == 1) tmem_dealloc_pair<kTmemCols>(tmem_base);
  } else if (warp == 1) {
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// Sum K-splits and scatter each (tile, m, n) to gw[co][tap][ci].
__global__ void k_wgrad_reduce(WgParams p, float* __restrict__ gw) {
  int64_t per_tile = 128 * (int64_t)p.bnp;
  int64_t total = per_tile * p.rtiles;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int tile = (int)(i / per_tile);
    const int64_t o = wg_out_index(p, tile, (int)((i % per_tile) / p.bnp), (int)(i % p.bnp));
    if (o < 0) continue;
    float s = 0.f;
    for (int sp = 0; sp < p.splits; ++sp) s += p.part[((int64_t)sp * p.rtiles) * per_tile + i];
    gw[o] = s;
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
  }
  return fn;
}

CUtensorMapSwizzle swz(int row_bytes) {
  return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
         : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
         : row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                           : CU_TENSOR_MAP_SWIZZLE_NONE;
}

// 5-D map over an NDHWC bf16 activation viewed as (C, W, H, D, N); `step`
// multiplies the spatial strides (parity views of a 2x grid use step 2).
bool map_act(CUtensorMap* m, const void* base, int C_total, int N, int D, int H, int W,
             int64_t sW, int64_t sH, int64_t sD, int64_t sN, int box_c, int bw, int bh, int bd) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[5] = {(cuuint64_t)C_total, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)D,
                        (cuuint64_t)N};
  cuuint64_t strides[4] = {(cuuint64_t)sW * 2, (cuuint64_t)sH * 2, (cuuint64_t)sD * 2,
                           (cuuint64_t)sN * 2};
  cuuint32_t box[5] = {(cuuint32_t)box_c, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bd, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz(box_c * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool map_act_dense(CUtensorMap* m, const void* base, int C_total, int N, int D, int H, int W,
                   int box_c, int bw, int bh, int bd) {
  int64_t sW = C_total, sH = sW * W, sD = sH * H, sN = sD * D;
  return map_act(m, base, C_total, N, D, H, W, sW, sH, sD, sN, box_c, bw, bh, bd);
}

// Dual-source conv input (ConvShape::x2): the conv reads channels [0, x_split) from x and
// [x_split, Cin) from x2 -- the concat of the U-Net's synthesis levels never materialised.
bool map_x2(Maps& maps, const ConvShape& sh, int box_c, int bw, int bh, int bd) {
  maps.split_c = 0;
  if (!sh.x2) return true;
  if (sh.x_split <= 0 || sh.x_split % 64 || sh.x_co != 0 || sh.x_cs != sh.x_split ||
      sh.x_split >= sh.Cin)
    return false;
  maps.split_c = sh.x_split;
  return map_act_dense(&maps.x2, sh.x2, sh.Cin - sh.x_split, sh.N, sh.D, sh.H, sh.W, box_c, bw,
                       bh, bd);
}

// Weights [Cout][27*Cin] as a 2-D map with box (box_cols, box_rows).
bool map_w(CUtensorMap* m, const void* w, int Cout, int Cin, int box_cols, int box_rows,
           int taps = 27) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)taps * Cin, (cuuint64_t)Cout};
  cuuint64_t strides[1] = {(cuuint64_t)taps * Cin * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz(box_cols * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Pick a power-of-two voxel box (bd, bh, bw) with bd*bh*bw == target that
// wastes the least padded volume on (D, H, W); ties prefer wider boxes.
void choose_box(int D, int H, int W, int target, int& bd, int& bh, int& bw) {
  int64_t best = -1;
  for (int w = 1; w <= 256 && w <= target; w *= 2)
    for (int h = 1; h <= 256 && w * h <= target; h *= 2) {
      int d = target / (w * h);
      if (d > 256 || d * w * h != target) continue;
      int64_t padded = (int64_t)((D + d - 1) / d) * d * ((H + h - 1) / h) * h * ((W + w - 1) / w) * w;
      if (best < 0 || padded < best || (padded == best && w > bw)) {
        best = padded;
        bd = d; bh = h; bw = w;
      }
    }
}

// Split-K over taps for grids too small to fill the GPU (12^3 / 24^3 levels with wide
// channels): enough splits to cover the SMs, >= 3 taps each, at most 4.
int ig_splits(int mn_tiles, int n_taps, int nout) {
  if (mn_tiles * 2 >= num_sms() || nout % 64) return 1;
  // the split count with the shortest makespan: waves of the persistent grid x taps per
  // split (rounding the CTA count up, e.g. 56 tiles x 3 splits on 148 SMs, leaves 20 CTAs
  // with two tiles -- worse than 2 splits in one wave)
  const int smax = std::max(1, std::min(4, n_taps / 3));
  int best = 1;
  long best_cost = -1;
  for (int sp = 1; sp <= smax; ++sp) {
    const long waves = (mn_tiles * sp + num_sms() - 1) / num_sms();
    const long cost = waves * ((n_taps + sp - 1) / sp);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = sp;
    }
  }
  return best;
}

bool z2_pair_enabled();

// CTA-pair per-tap implicit GEMM (fprop): K-major weights, BN >= 64 so each CTA keeps >= 32
// weight rows; the sub-pixel transposed conv can pair over its re-laid W' (n-major tiles,
// both CTAs on one n tile), the direct per-class form cannot
// The ONE pair predicate: the launcher (ig_pair_ok<BN, B_MN>), the weight-map setup and the
// BN-partials row count (ig_bn_sums, conv_stat_parts_tc) all call it, so the rows a fused
// BN-sums epilogue writes always match the grid that ran.
bool ig_pair_ok_host(int bn, bool b_mn, const IgParams& p) {
  return (b_mn ? bn >= 128 : bn >= 64) && p.ig_pair && p.sp_direct == 0 &&
         (p.scatter_c == 0 || !b_mn) && z2_pair_enabled();
}
template <int BN, bool B_MN>
bool ig_pair_ok(const IgParams& p) { return ig_pair_ok_host(BN, B_MN, p); }
int ig_pair_grid(const IgParams& p) {
  const int items = p.splits * ((p.m_tiles + 1) / 2) * p.n_tiles;
  return std::min(2 * items, num_sms() / 2 * 2);
}
template <int BN, int CK>
constexpr int kStagesP = std::min(8, kSmemBudget / (128 * CK * 2 + BN / 2 * CK * 2));

template <int BN, int CK, bool B_MN>
cudaError_t launch_ig(cudaStream_t s, const Maps& maps, IgParams& p, int* grid_out) {
  constexpr int kStageBytes = 128 * CK * 2 + BN * CK * 2;
  constexpr int kStagesRaw = kSmemBudget / kStageBytes;
  constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  size_t smem = (size_t)kStages * kStageBytes + kIgEpiBytes + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_igemm<BN, CK, B_MN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (p.splits < 1) p.splits = 1;
  int tiles = p.m_tiles * p.n_tiles * p.splits;
  int grid = std::min(tiles, num_sms());
  cudaError_t e;
  if (ig_pair_ok<BN, B_MN>(p)) {
    constexpr size_t smem_p =
        (size_t)kStagesP<BN, CK> * (128 * CK * 2 + BN / 2 * CK * 2) + kIgEpiBytes + 1024;
    auto kern = k_igemm<BN, CK, B_MN, true>;
    static bool configured_p = false;
    if (!configured_p) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
      if (e != cudaSuccess) return e;
      configured_p = true;
    }
    grid = ig_pair_grid(p);
    if (grid_out) *grid_out = grid;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem_p;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, maps, p);
  } else {
    if (grid_out) *grid_out = grid;
    k_igemm<BN, CK, B_MN><<<grid, kThreads, smem, s>>>(maps, p);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess || p.splits == 1) return e;
  k_igemm_split_reduce<BN><<<dim3(p.m_tiles, p.Nout / 64), 256, 0, s>>>(p);
  return cudaGetLastError();
}

template <bool B_MN>
cudaError_t dispatch_ig(cudaStream_t s, const Maps& maps, IgParams& p, int BN, int CK) {
  static int staged = -1;
  if (staged < 0) {
    const char* e = getenv("US_IG_STAGED");
    staged = (e && e[0] == '0') ? 0 : 1;
  }
  p.staged_epi = staged;
#define IG_CASE(bn, ck) \
  if (BN == bn && CK == ck) return launch_ig<bn, ck, B_MN>(s, maps, p, nullptr);
  if constexpr (!B_MN) {
    IG_CASE(16, 16) IG_CASE(32, 16) IG_CASE(16, 32) IG_CASE(32, 32)
    IG_CASE(16, 64) IG_CASE(32, 64)
  }
  // MN-major B (dgrad) needs BN in multiples of the 64-channel swizzle chunk.
  IG_CASE(64, 16) IG_CASE(128, 16) IG_CASE(256, 16)
  IG_CASE(64, 32) IG_CASE(128, 32) IG_CASE(256, 32)
  IG_CASE(64, 64) IG_CASE(128, 64) IG_CASE(256, 64)
#undef IG_CASE
  return cudaErrorInvalidConfiguration;
}

int pick_bn(int n) { return n >= 256 ? 256 : n; }

// ConvT sub-pixel weights W'[(c*Cout + co)][t][ci] = W[co][convt_ktap(t, c)][ci], zero where
// class c does not use window tap t (the re-laid form of the Cout = 64 sub-pixel GEMM).
__global__ void k_convt_subpixel_w(const __nv_bfloat16* __restrict__ w,
                                   __nv_bfloat16* __restrict__ wp, int Cin, int Cout) {
  const int64_t total = (int64_t)8 * Cout * 8 * Cin;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ci = (int)(i % Cin);
    const int t = (int)((i / Cin) % 8);
    const int col = (int)(i / ((int64_t)8 * Cin));
    const int c = col / Cout, co = col % Cout;
    wp[i] = convt_uses(t, c) ? w[((int64_t)co * 27 + convt_ktap(t, c)) * Cin + ci]
                             : __float2bfloat16(0.f);
  }
}

// Transposed-conv fprop form: 2 = sub-pixel, weights straight from W, exact 27 blocks
// (Cout % 256 == 0: one parity class per 256-column n tile -- measured r02 24^3 512->256
// 0.165 -> 0.105 ms, 12^3 1024->512 0.214 -> 0.096 ms against the 8 class launches);
// 1 = sub-pixel over the re-laid W' with full-N MMAs (Cout == 64: 4 classes per tile; runs
// of N = 64..256 MMAs measured slower, 0.64 vs 1.10 ms at 96^3 128->64); 0 = one launch per
// parity class (Cout == 128 and the rest).  US_CONVT_CLASSES=1 forces 0.
int convt_subpixel_mode(const ConvShape& sh) {
  static int off = -1;
  if (off < 0) {
    const char* e = getenv("US_CONVT_CLASSES");
    off = (e && e[0] == '1') ? 1 : 0;
  }
  if (off || sh.Cin % 64) return 0;
  if (sh.Cout % 256 == 0 && 8 * sh.Cout / 256 <= 32) return 2;
  if (sh.Cout == 64) return 1;
  return 0;
}
bool convt_subpixel_ok(const ConvShape& sh) { return convt_subpixel_mode(sh) != 0; }
int pick_ck(int c) { return c >= 64 ? 64 : c; }

void fill_grid(IgParams& p, int Nb, int D, int H, int W) {
  p.Nb = Nb; p.Md = D; p.Mh = H; p.Mw = W;
  choose_box(D, H, W, 128, p.bd, p.bh, p.bw);
  p.td = (D + p.bd - 1) / p.bd;
  p.th = (H + p.bh - 1) / p.bh;
  p.tw = (W + p.bw - 1) / p.bw;
  p.m_tiles = Nb * p.td * p.th * p.tw;
}

void conv_taps(Taps& t, int sign) {
  for (int k = 0; k < 27; ++k) {
    int kd = k / 9, kh = (k / 3) % 3, kw = k % 3;
    t.dz[k] = (int8_t)(sign * (kd - 1));
    t.dy[k] = (int8_t)(sign * (kh - 1));
    t.dx[k] = (int8_t)(sign * (kw - 1));
    t.map[k] = 0;
    t.w[k] = (int16_t)k;
  }
}

// ---- halo path selection and launch
bool halo_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("US_NO_HALO");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool halo_eligible(const ConvShape& sh, bool dgrad) {
  if (halo_disabled()) return false;
  int ca = dgrad ? sh.Cout : sh.Cin;       // channels of the A operand (reduced)
  int nout = dgrad ? sh.Cin : sh.Cout;     // output channels
  if (ca % 64 || nout % 64) return false;
  return sh.W >= 32 && sh.H >= 16;         // dense 8x16 tiles
}

bool z2_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("US_NO_Z2");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// the z-pair kernel takes every N = 64 halo conv (fprop Cout = 64, dgrad Cin = 64)
bool halo_z2(const ConvShape& sh, bool dgrad) {
  return !z2_disabled() && (dgrad ? sh.Cin : sh.Cout) == 64;
}

void halo_grid(const ConvShape& sh, bool dgrad, HaloParams& p, int& bn) {
  int nout = dgrad ? sh.Cin : sh.Cout;
  bn = nout >= 256 ? 256 : nout;
  if (nout % bn) bn = 64;
  p.Nb = sh.N; p.Md = sh.D; p.Mh = sh.H; p.Mw = sh.W;
  p.tw = (sh.W + 7) / 8;
  p.th = (sh.H + 15) / 16;
  p.td = halo_z2(sh, dgrad) ? (sh.D + 1) / 2 : sh.D;
  p.m_tiles = sh.N * p.td * p.th * p.tw;
  p.n_tiles = nout / bn;
  p.Nout = nout;
}

template <int BN, bool B_MN, int NA, int NB, int TPS>
cudaError_t launch_halo(cudaStream_t s, const Maps& maps, const HaloParams& p) {
  size_t smem = halo_smem_bytes(BN, NA, NB, TPS);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_igemm_halo<BN, B_MN, NA, NB, TPS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int grid = std::min(p.m_tiles * p.n_tiles, num_sms());
  k_igemm_halo<BN, B_MN, NA, NB, TPS><<<grid, kThreads, smem, s>>>(maps, p);
  return cudaGetLastError();
}

template <bool B_MN, int R, int NB>
cudaError_t launch_z2_cfg(cudaStream_t s, const Maps& maps, const HaloParams& p) {
  constexpr size_t smem = z2_smem(R, NB);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_halo_z2<B_MN, R, NB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int grid = std::min(p.m_tiles, num_sms());
  k_halo_z2<B_MN, R, NB><<<grid, kThreads, smem, s>>>(maps, p);
  return cudaGetLastError();
}

// W[co][t][ci] -> W^T[t][ci][co]: the dgrad's B operand K-major (rows = ci), so the CTA
// pair can split it by rows like the fprop weights
__global__ void k_transpose_w(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ wt,
                              int Cin, int Cout) {
  const int64_t total = (int64_t)27 * Cin * Cout;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int co = (int)(i % Cout);
    const int64_t r = i / Cout;   // t * Cin + ci
    const int ci = (int)(r % Cin), t = (int)(r / Cin);
    wt[i] = w[((int64_t)co * 27 + t) * Cin + ci];
  }
}

// CTA-pair fprop (cluster of 2): grid even, one row of BN partials per CTA
int z2_pair_grid(int m_tiles) { return std::min(2 * ((m_tiles + 1) / 2), num_sms() / 2 * 2); }

bool z2_pair_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("US_NO_Z2_PAIR");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

cudaError_t launch_z2_pair(cudaStream_t s, const Maps& maps, const HaloParams& p) {
  constexpr int R = 5, NB = 6;
  constexpr size_t smem = (size_t)R * kSlabStride + (size_t)NB * 3 * 32 * 128 + 1024;
  auto kern = k_halo_z2<false, R, NB, true>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(z2_pair_grid(p.m_tiles));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, maps, p);
}

template <bool B_MN>
cudaError_t launch_z2(cudaStream_t s, const Maps& maps, const HaloParams& p) {
  // 5 slabs + 4 weight stages and 6 + 3 measure the same (r01): neither ring is the limit
  return launch_z2_cfg<B_MN, 5, 4>(s, maps, p);
}

// CTA-pair launch of the 8x16x1 halo kernel (BN = 128, one N tile)
bool halo_pair_ok(const ConvShape& sh, bool dgrad) {
  const int nout = dgrad ? sh.Cin : sh.Cout;
  return z2_pair_enabled() && !halo_z2(sh, dgrad) && (nout == 128 || nout == 256);
}

template <int BN, int NB>
cudaError_t launch_halo_pair(cudaStream_t s, const Maps& maps, const HaloParams& p) {
  constexpr int NA = 2, TPS = 1;
  static_assert(!halo_xpose_fits(BN, NA, NB, TPS), "pair smem layout assumes no transpose");
  constexpr size_t smem = (size_t)NA * kHaloStride + (size_t)NB * TPS * (BN / 2) * 128 + 1024;
  auto kern = k_igemm_halo<BN, false, NA, NB, TPS, true>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(z2_pair_grid(p.m_tiles));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, maps, p);
}

cudaError_t run_halo(cudaStream_t s, const ConvShape& sh, bool dgrad, const __nv_bfloat16* a,
                     const __nv_bfloat16* w, __nv_bfloat16* out, float* stats,
                     void* scratch = nullptr) {
  HaloParams p{};
  int bn;
  halo_grid(sh, dgrad, p, bn);
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  int a_cs = dgrad ? sh.dy_cs : sh.x_cs;
  if (halo_z2(sh, dgrad)) {
    if (!map_act_dense(&maps.a[0], a, a_cs, sh.N, sh.D, sh.H, sh.W, 64, kHW, kHH, 1) ||
        (!dgrad && !map_x2(maps, sh, 64, kHW, kHH, 1)))
      return cudaErrorInvalidValue;
    const bool pair = z2_pair_enabled() && (!dgrad || scratch);
    if (pair && dgrad) {   // W^T [27 * Cin rows][Cout] in the scratch, rows split by the pair
      __nv_bfloat16* wt = (__nv_bfloat16*)scratch;
      const int64_t total = (int64_t)27 * sh.Cin * sh.Cout;
      k_transpose_w<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, s>>>(
          w, wt, sh.Cin, sh.Cout);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      if (!map_w(&maps.b, wt, 27 * sh.Cin, sh.Cout, 64, 32, 1)) return cudaErrorInvalidValue;
      p.b_rows_tap = 1;
    } else if (!map_w(&maps.b, w, sh.Cout, sh.Cin, 64, pair ? 32 : 64)) {
      return cudaErrorInvalidValue;
    }
    p.k_chunks = (dgrad ? sh.Cout : sh.Cin) / 64;
    p.a_c0 = dgrad ? sh.dy_co : sh.x_co;
    p.w_cin = sh.Cin;
    p.mirror = dgrad ? 1 : 0;
    p.out = out;
    p.mask = dgrad ? (const __nv_bfloat16*)sh.relu_mask : nullptr;
    p.out_cs = dgrad ? sh.Cin : sh.Cout;
    p.stats = stats;
    if (dgrad && sh.bn_part) {
      p.bnx = (const __nv_bfloat16*)sh.bn_x;
      p.bn_stat = sh.bn_stat;
      p.stats = sh.bn_part;
      if (sh.bn_rows) *sh.bn_rows = pair ? z2_pair_grid(p.m_tiles) : std::min(p.m_tiles, num_sms());
    }
    if (pair) return launch_z2_pair(s, maps, p);
    return dgrad ? launch_z2<true>(s, maps, p) : launch_z2<false>(s, maps, p);
  }
  if (!map_act_dense(&maps.a[0], a, a_cs, sh.N, sh.D, sh.H, sh.W, 64, kHW, kHH, kHD) ||
      (!dgrad && !map_x2(maps, sh, 64, kHW, kHH, kHD)))
    return cudaErrorInvalidValue;
  const bool pair = halo_pair_ok(sh, dgrad) && (!dgrad || scratch);
  if (pair && dgrad) {   // W^T [27 * Cin rows][Cout], rows split by the pair
    __nv_bfloat16* wt = (__nv_bfloat16*)scratch;
    const int64_t total = (int64_t)27 * sh.Cin * sh.Cout;
    k_transpose_w<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, s>>>(
        w, wt, sh.Cin, sh.Cout);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (!map_w(&maps.b, wt, 27 * sh.Cin, sh.Cout, 64, bn / 2, 1)) return cudaErrorInvalidValue;
    p.b_rows_tap = 1;
  } else if (pair) {
    if (!map_w(&maps.b, w, sh.Cout, sh.Cin, 64, bn / 2)) return cudaErrorInvalidValue;
  } else if (!dgrad) {
    if (!map_w(&maps.b, w, sh.Cout, sh.Cin, 64, bn)) return cudaErrorInvalidValue;
  } else {
    if (!map_w(&maps.b, w, sh.Cout, sh.Cin, 64, 64)) return cudaErrorInvalidValue;
  }
  p.k_chunks = (dgrad ? sh.Cout : sh.Cin) / 64;
  p.a_c0 = dgrad ? sh.dy_co : sh.x_co;
  p.w_cin = sh.Cin;
  p.mirror = dgrad ? 1 : 0;
  p.out = out;
  p.mask = dgrad ? (const __nv_bfloat16*)sh.relu_mask : nullptr;
  p.out_cs = dgrad ? sh.Cin : sh.Cout;
  p.stats = stats;
  if (dgrad && sh.bn_part) {
    p.bnx = (const __nv_bfloat16*)sh.bn_x;
    p.bn_stat = sh.bn_stat;
    p.stats = sh.bn_part;
    if (sh.bn_rows)
      *sh.bn_rows = pair ? z2_pair_grid(p.m_tiles) : std::min(p.m_tiles * p.n_tiles, num_sms());
  }
  if (pair) return bn == 128 ? launch_halo_pair<128, 8>(s, maps, p)
                             : launch_halo_pair<256, 5>(s, maps, p);
  // B-stage depth is what bounds these kernels (r01 sweep, tools/probe_halo_variants.sh):
  // 64 columns: 3 stages of 3 taps (BN stats by warp shuffles: the transpose buffer
  // does not fit next to them); 128 columns: 5 single-tap stages.
  if (!dgrad) {
    if (bn == 64) return launch_halo<64, false, 2, 3, 3>(s, maps, p);
    if (bn == 128) return launch_halo<128, false, 2, 5, 1>(s, maps, p);
    return launch_halo<256, false, 1, 3, 1>(s, maps, p);
  }
  if (bn == 64) return launch_halo<64, true, 2, 3, 3>(s, maps, p);
  if (bn == 128) return launch_halo<128, true, 2, 5, 1>(s, maps, p);
  return launch_halo<256, true, 1, 3, 1>(s, maps, p);
}

}  // namespace

bool tc_supported(const ConvShape& sh) {
  return encode_fn() != nullptr && sh.Cin % 16 == 0 && sh.Cout % 16 == 0;
}

int conv_stat_parts_tc(const ConvShape& sh) {
  if (halo_eligible(sh, false)) {
    HaloParams hp{};
    int bn;
    halo_grid(sh, false, hp, bn);
    if ((halo_z2(sh, false) && z2_pair_enabled()) || halo_pair_ok(sh, false))
      return z2_pair_grid(hp.m_tiles);
    return std::min(hp.m_tiles * hp.n_tiles, num_sms());
  }
  IgParams p{};
  fill_grid(p, sh.N, sh.D, sh.H, sh.W);
  int bn = pick_bn(sh.Cout);
  int tiles = p.m_tiles * (sh.Cout / bn);
  p.n_tiles = sh.Cout / bn;
  p.splits = ig_splits(tiles, 27, sh.Cout);
  if (p.splits > 1) return p.m_tiles;   // split-K: partials per M tile
  p.ig_pair = 1;
  if (ig_pair_ok_host(bn, false, p)) return ig_pair_grid(p);
  return std::min(tiles, num_sms());
}

size_t convt_fwd_scratch_bytes(const ConvShape& sh) {
  // the re-laid W' of mode 1; mode 2 reads W directly
  return convt_subpixel_mode(sh) == 1 ? (size_t)8 * sh.Cout * 8 * sh.Cin * 2 : 0;
}

size_t conv_split_scratch_bytes(const ConvShape& sh, bool dgrad) {
  if (halo_eligible(sh, dgrad)) {   // CTA-pair dgrad: transposed weights
    return dgrad && ((halo_z2(sh, true) && z2_pair_enabled()) || halo_pair_ok(sh, true))
               ? (size_t)27 * sh.Cin * sh.Cout * sizeof(__nv_bfloat16) : 0;
  }
  IgParams p{};
  fill_grid(p, sh.N, sh.D, sh.H, sh.W);
  const int nout = dgrad ? sh.Cin : sh.Cout;
  const int bn = pick_bn(nout);
  const int splits = ig_splits(p.m_tiles * (nout / bn), 27, nout);
  if (splits == 1) return 0;
  return (size_t)splits * p.m_tiles * 128 * nout * sizeof(float);
}

cudaError_t conv_fwd_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                        const __nv_bfloat16* w, __nv_bfloat16* y, float* part,
                        float* split_scratch) {
  if (sh.Cin % 16 || sh.Cout % 16 || sh.Cout > 1024) return cudaErrorInvalidValue;
  if (halo_eligible(sh, false)) return run_halo(s, sh, false, x, w, y, part);
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  IgParams p{};
  fill_grid(p, sh.N, sh.D, sh.H, sh.W);
  int ck = pick_ck(sh.Cin), bn = pick_bn(sh.Cout);
  if (!map_act_dense(&maps.a[0], x, sh.x_cs, sh.N, sh.D, sh.H, sh.W, ck, p.bw, p.bh, p.bd) ||
      !map_x2(maps, sh, ck, p.bw, p.bh, p.bd))
    return cudaErrorInvalidValue;
  for (int i = 1; i < 8; ++i) maps.a[i] = maps.a[0];
  if (!map_w(&maps.b, w, sh.Cout, sh.Cin, ck, bn)) return cudaErrorInvalidValue;
  conv_taps(p.taps, +1);
  p.n_taps = 27;
  p.n_tiles = sh.Cout / bn;
  p.k_chunks = sh.Cin / ck;
  p.a_c0 = sh.x_co;
  p.w_cin = sh.Cin;
  p.out = y; p.out_cs = sh.Cout; p.out_co = 0;
  p.oD = sh.D; p.oH = sh.H; p.oW = sh.W; p.os = 1; p.ooz = p.ooy = p.oox = 0;
  p.stats = part;
  p.Nout = sh.Cout;
  p.splits = ig_splits(p.m_tiles * p.n_tiles, 27, sh.Cout);
  if (p.splits > 1) {
    if (!split_scratch) return cudaErrorInvalidValue;
    p.split_part = split_scratch;
  }
  p.ig_pair = 1;
  if (ig_pair_ok_host(bn, false, p)) {   // weights TMA box: half the rows per CTA
    if (!map_w(&maps.b, w, sh.Cout, sh.Cin, ck, bn / 2)) return cudaErrorInvalidValue;
  }
  return dispatch_ig<false>(s, maps, p, bn, ck);
}

// dgrad on the per-tap kernel: BN-backward sums in the epilogue (per CTA) or, split-K,
// in the split reduce (per M tile)
static void ig_bn_sums(const ConvShape& sh, IgParams& p, bool pair = false) {
  if (!sh.bn_part) return;
  p.bnx = (const __nv_bfloat16*)sh.bn_x;
  p.bn_stat = sh.bn_stat;
  p.stats = sh.bn_part;
  if (sh.bn_rows)
    *sh.bn_rows = p.splits > 1 ? p.m_tiles
                : pair         ? ig_pair_grid(p)
                               : std::min(p.m_tiles * p.n_tiles, num_sms());
}

cudaError_t conv_dgrad_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* dy,
                          const __nv_bfloat16* w, __nv_bfloat16* dx, float* split_scratch) {
  // dX = sum_t dY[v - off(t)] W[:, t, :]  (A = dY K-major, B = W MN-major)
  if (sh.Cin % 64 || sh.Cout % 16 || sh.Cin > 1024) return cudaErrorInvalidValue;
  if (halo_eligible(sh, true)) return run_halo(s, sh, true, dy, w, dx, nullptr, split_scratch);
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  IgParams p{};
  fill_grid(p, sh.N, sh.D, sh.H, sh.W);
  int ck = pick_ck(sh.Cout), bn = pick_bn(sh.Cin);
  if (!map_act_dense(&maps.a[0], dy, sh.dy_cs, sh.N, sh.D, sh.H, sh.W, ck, p.bw, p.bh, p.bd))
    return cudaErrorInvalidValue;
  for (int i = 1; i < 8; ++i) maps.a[i] = maps.a[0];
  if (!map_w(&maps.b, w, sh.Cout, sh.Cin, 64, ck)) return cudaErrorInvalidValue;
  conv_taps(p.taps, -1);
  p.n_taps = 27;
  p.n_tiles = sh.Cin / bn;
  p.k_chunks = sh.Cout / ck;
  p.a_c0 = sh.dy_co;
  p.w_cin = sh.Cin;
  p.out = dx; p.out_cs = sh.Cin; p.out_co = 0;
  p.mask = (const __nv_bfloat16*)sh.relu_mask;
  p.oD = sh.D; p.oH = sh.H; p.oW = sh.W; p.os = 1; p.ooz = p.ooy = p.oox = 0;
  p.stats = nullptr;
  p.Nout = sh.Cin;
  p.splits = ig_splits(p.m_tiles * p.n_tiles, 27, sh.Cin);
  if (p.splits > 1) {
    if (!split_scratch) return cudaErrorInvalidValue;
    p.split_part = split_scratch;
  }
  p.ig_pair = 1;   // CTA pair when bn >= 128 (each CTA stages its 64-column weight chunks)
  ig_bn_sums(sh, p, ig_pair_ok_host(bn, true, p));
  return dispatch_ig<true>(s, maps, p, bn, ck);
}

cudaError_t convt_fwd_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                         const __nv_bfloat16* w, __nv_bfloat16* y, void* scratch, int y_cs,
                         int y_co) {
  if (y_cs < y_co + sh.Cout || y_cs % 8 || y_co % 8) return cudaErrorInvalidValue;
  // Output parity class (pz,py,px): o = 2j + p; p=0 -> tap 1 at i=j ; p=1 -> taps 0 (i=j+1), 2 (i=j).
  if (sh.Cin % 16 || sh.Cout % 16) return cudaErrorInvalidValue;
  if (convt_subpixel_ok(sh)) {
    // Sub-pixel form: ONE GEMM over the low-res grid with a 2x2x2 input window (8 taps
    // t = (dz, dy, dx), input j + t) and 8 x Cout output columns (parity class c, channel
    // co), n tiles of 256 columns; a tile skips the taps none of its classes use (nt_mask).
    // Mode 2 (direct, one class per tile): the class's rows come straight from W at kernel
    // tap convt_ktap(t, c) -- exactly the 27 used (t, c) blocks.  Mode 1 (Cout 64, four
    // classes per tile): full-N MMAs over the re-laid W' (zero blocks of the tile included).
    const bool direct = convt_subpixel_mode(sh) == 2;   // Cout % 256 == 0
    const int Np = 8 * sh.Cout, bn = 256;
    Maps maps;
    std::memset(&maps, 0, sizeof maps);
    IgParams p{};
    fill_grid(p, sh.N, sh.D, sh.H, sh.W);
    const int ck = pick_ck(sh.Cin);
    if (!map_act_dense(&maps.a[0], x, sh.Cin, sh.N, sh.D, sh.H, sh.W, ck, p.bw, p.bh, p.bd))
      return cudaErrorInvalidValue;
    for (int i = 1; i < 8; ++i) maps.a[i] = maps.a[0];
    if (direct) {
      if (!map_w(&maps.b, w, sh.Cout, sh.Cin, ck, bn)) return cudaErrorInvalidValue;
    } else {
      __nv_bfloat16* wp = (__nv_bfloat16*)scratch;
      if (!wp) return cudaErrorInvalidValue;
      const int64_t total = (int64_t)Np * 8 * sh.Cin;
      k_convt_subpixel_w<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(
          w, wp, sh.Cin, sh.Cout);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    p.sp_direct = direct ? 1 : 0;
    // (a CTA pair, half the W' rows per CTA, measured no faster: 0.640 vs 0.624 ms at
    // 96^3 128->64; US_CONVT_PAIR=1 turns it on for A/B runs)
    static const int convt_pair = getenv("US_CONVT_PAIR") && getenv("US_CONVT_PAIR")[0] == '1';
    p.ig_pair = direct ? 0 : convt_pair;
    for (int t = 0; t < 8; ++t) {
      p.taps.dz[t] = (int8_t)((t >> 2) & 1);
      p.taps.dy[t] = (int8_t)((t >> 1) & 1);
      p.taps.dx[t] = (int8_t)(t & 1);
      p.taps.map[t] = 0;
      p.taps.w[t] = (int16_t)(direct ? 0 : t);   // direct: per class, convt_ktap
    }
    p.n_taps = 8;
    p.n_tiles = Np / bn;
    p.splits = 1;
    for (int j = 0; j < p.n_tiles; ++j) {
      const int cls0 = j * bn / sh.Cout;   // the tile's classes: cls0 .. (4 for Cout = 64)
      uint8_t m = 0;
      for (int i = 0; i < std::max(1, bn / sh.Cout); ++i)
        for (int t = 0; t < 8; ++t)
          if (convt_uses(t, cls0 + i)) m |= (uint8_t)(1u << t);
      p.nt_mask[j] = m;
    }
    p.k_chunks = sh.Cin / ck;
    p.a_c0 = 0;
    p.w_cin = sh.Cin;
    p.out = y; p.out_cs = y_cs; p.out_co = y_co;
    p.oD = 2 * sh.D; p.oH = 2 * sh.H; p.oW = 2 * sh.W; p.os = 2;
    p.scatter_c = sh.Cout;
    p.stats = nullptr;
    p.Nout = Np;
    if (!direct) {   // W' rows of the tile (a CTA pair: half of them per CTA)
      const int box = ig_pair_ok_host(bn, false, p) ? bn / 2 : bn;
      if (!map_w(&maps.b, scratch, Np, sh.Cin, ck, box, 8)) return cudaErrorInvalidValue;
    }
    return dispatch_ig<false>(s, maps, p, bn, ck);
  }
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  IgParams base{};
  fill_grid(base, sh.N, sh.D, sh.H, sh.W);
  int ck = pick_ck(sh.Cin), bn = pick_bn(sh.Cout);
  if (!map_act_dense(&maps.a[0], x, sh.Cin, sh.N, sh.D, sh.H, sh.W, ck, base.bw, base.bh, base.bd))
    return cudaErrorInvalidValue;
  for (int i = 1; i < 8; ++i) maps.a[i] = maps.a[0];
  if (!map_w(&maps.b, w, sh.Cout, sh.Cin, ck, bn)) return cudaErrorInvalidValue;
  for (int cls = 0; cls < 8; ++cls) {
    int pz = (cls >> 2) & 1, py = (cls >> 1) & 1, px = cls & 1;
    IgParams p = base;
    int kz[2], oz[2], nz = 0, ky[2], oy[2], ny = 0, kx[2], ox[2], nx = 0;
    auto fill = [](int par, int* k, int* o, int& n) {
      if (par == 0) { k[0] = 1; o[0] = 0; n = 1; }
      else { k[0] = 0; o[0] = 1; k[1] = 2; o[1] = 0; n = 2; }
    };
    fill(pz, kz, oz, nz);
    fill(py, ky, oy, ny);
    fill(px, kx, ox, nx);
    int t = 0;
    for (int a = 0; a < nz; ++a)
      for (int b = 0; b < ny; ++b)
        for (int c = 0; c < nx; ++c, ++t) {
          p.taps.dz[t] = (int8_t)oz[a];
          p.taps.dy[t] = (int8_t)oy[b];
          p.taps.dx[t] = (int8_t)ox[c];
          p.taps.map[t] = 0;
          p.taps.w[t] = (int16_t)(kz[a] * 9 + ky[b] * 3 + kx[c]);
        }
    p.n_taps = t;
    p.n_tiles = sh.Cout / bn;
    p.k_chunks = sh.Cin / ck;
    p.a_c0 = 0;
    p.w_cin = sh.Cin;
    p.out = y; p.out_cs = y_cs; p.out_co = y_co;
    p.oD = 2 * sh.D; p.oH = 2 * sh.H; p.oW = 2 * sh.W; p.os = 2;
    p.ooz = pz; p.ooy = py; p.oox = px;
    p.stats = nullptr;
    p.Nout = sh.Cout;
    cudaError_t e = dispatch_ig<false>(s, maps, p, bn, ck);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t convt_dgrad_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* dy,
                           const __nv_bfloat16* w, __nv_bfloat16* dx) {
  // dX[i] = sum_k dY[2i-1+k] Wt[:, k, :] ; dY read through 8 parity views.
  if (sh.Cin % 64 || sh.Cout % 16) return cudaErrorInvalidValue;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  IgParams p{};
  fill_grid(p, sh.N, sh.D, sh.H, sh.W);
  int ck = pick_ck(sh.Cout), bn = pick_bn(sh.Cin);
  int D2 = 2 * sh.D, H2 = 2 * sh.H, W2 = 2 * sh.W;
  int64_t cs = sh.dy_cs;
  for (int par = 0; par < 8; ++par) {
    int pz = (par >> 2) & 1, py = (par >> 1) & 1, px = par & 1;
    const __nv_bfloat16* b0 = dy + (((int64_t)pz * H2 + py) * W2 + px) * cs;
    if (!map_act(&maps.a[par], b0, (int)cs, sh.N, sh.D, sh.H, sh.W, 2 * cs, 2 * cs * W2,
                 2 * cs * W2 * H2, cs * W2 * H2 * D2, ck, p.bw, p.bh, p.bd))
      return cudaErrorInvalidValue;
  }
  if (!map_w(&maps.b, w, sh.Cout, sh.Cin, 64, ck)) return cudaErrorInvalidValue;
  for (int k = 0; k < 27; ++k) {
    int kd = k / 9, kh = (k / 3) % 3, kw = k % 3;
    int pz = kd != 1, py = kh != 1, px = kw != 1;
    p.taps.map[k] = (int8_t)(pz * 4 + py * 2 + px);
    p.taps.dz[k] = (int8_t)(kd == 0 ? -1 : 0);
    p.taps.dy[k] = (int8_t)(kh == 0 ? -1 : 0);
    p.taps.dx[k] = (int8_t)(kw == 0 ? -1 : 0);
    p.taps.w[k] = (int16_t)k;
  }
  p.n_taps = 27;
  p.n_tiles = sh.Cin / bn;
  p.k_chunks = sh.Cout / ck;
  p.a_c0 = sh.dy_co;
  p.w_cin = sh.Cin;
  p.out = dx; p.out_cs = sh.Cin; p.out_co = 0;
  p.mask = (const __nv_bfloat16*)sh.relu_mask;
  p.oD = sh.D; p.oH = sh.H; p.oW = sh.W; p.os = 1; p.ooz = p.ooy = p.oox = 0;
  p.stats = nullptr;
  p.Nout = sh.Cin;
  ig_bn_sums(sh, p);
  return dispatch_ig<true>(s, maps, p, bn, ck);
}

// ---------------------------------------------------------------- wgrad host
namespace {

constexpr int kWgTT = 4;   // taps per unit of the multi-tap convT weight gradient

bool wg_setup(const ConvShape& sh, bool transposed, WgParams& p, int& bnp, int& kb) {
  bool narrow = !transposed && sh.Cin == 32 && sh.Cout == 64;
  if ((sh.Cin % 64 && !narrow) || sh.Cout % 64) return false;
  if (transposed && sh.Cout < 128 && sh.Cin < 128) return false;
  std::memset(&p, 0, sizeof p);
  p.aw = narrow ? 32 : 64;
  p.mode = transposed ? 1 : 0;
  p.Cin = sh.Cin;
  p.Cout = sh.Cout;
  p.caseA = sh.Cout >= 128;
  if (p.caseA) {
    bnp = std::min(sh.Cin, 256);
    if (sh.Cin % bnp) bnp = 64;
    p.tiles = 27 * (sh.Cout / 128) * (sh.Cin / bnp);
  } else {
    bnp = 64;
    p.tiles = sh.Cin <= 64 ? (27 + (128 / p.aw) - 1) / (128 / p.aw) : 27 * (sh.Cin / 128);
  }
  p.bnp = bnp;
  kb = bnp >= 256 ? 64 : 128;
  p.tt = 1;
  p.rtiles = p.tiles;
  if (transposed && !p.caseA && sh.Cin % 128 == 0 && !getenv("US_WG_TT1")) {
    // X (A) is the same for every tap: 4 taps per unit share it, 64-voxel K blocks
    p.tt = kWgTT;
    p.tiles = (27 + kWgTT - 1) / kWgTT * (sh.Cin / 128);
    kb = 64;
  }
  p.Nb = sh.N; p.D = sh.D; p.H = sh.H; p.W = sh.W;
  choose_box(sh.D, sh.H, sh.W, kb, p.kbd, p.kbh, p.kbw);
  p.ktd = (sh.D + p.kbd - 1) / p.kbd;
  p.kth = (sh.H + p.kbh - 1) / p.kbh;
  p.ktw = (sh.W + p.kbw - 1) / p.kbw;
  p.kblocks = sh.N * p.ktd * p.kth * p.ktw;
  int target_units = 2 * num_sms();
  int splits = (target_units + p.tiles - 1) / p.tiles;
  splits = std::max(1, std::min(splits, p.kblocks));
  p.splits = splits;
  p.x_c0 = sh.x_co;
  p.dy_c0 = sh.dy_co;
  p.gw_co_stride = 27 * sh.Cin;
  p.gw_cmax = sh.Cin;
  return true;
}

cudaError_t launch_wg_pair(cudaStream_t s, const Maps& maps, const WgParams& p) {
  constexpr int BNP = 256, KB = 64, AW = 64;
  constexpr int kStageBytes = (128 / AW) * KB * AW * 2 + (BNP / 64 / 2) * KB * 128;
  constexpr int kStagesRaw = kSmemBudget / kStageBytes;
  constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
  const size_t smem = (size_t)kStages * kStageBytes + 1024;
  auto kern = k_wgrad<BNP, KB, AW, 1, true>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(p.tiles * p.splits, num_sms() / 2 * 2));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, maps, p);
}

template <int BNP, int KB, int AW, int TT = 1>
cudaError_t launch_wg(cudaStream_t s, const Maps& maps, const WgParams& p) {
  constexpr int kStageBytes = (128 / AW) * KB * AW * 2 + (BNP / 64) * TT * KB * 128;
  constexpr int kStagesRaw = kSmemBudget / kStageBytes;
  constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
  size_t smem = (size_t)kStages * kStageBytes + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_wgrad<BNP, KB, AW, TT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int units = p.tiles * p.splits;
  int grid = std::min(units, num_sms());
  k_wgrad<BNP, KB, AW, TT><<<grid, kThreads, smem, s>>>(maps, p);
  return cudaGetLastError();
}

cudaError_t wgrad_run(cudaStream_t s, const ConvShape& sh, bool transposed,
                      const __nv_bfloat16* x, const __nv_bfloat16* dy, float* gw, float* work) {
  WgParams p;
  int bnp, kb;
  if (!wg_setup(sh, transposed, p, bnp, kb)) return cudaErrorInvalidValue;
  p.part = work;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  // map 0: X (K grid == X grid in both modes)
  if (!map_act_dense(&maps.a[0], x, sh.x_cs, sh.N, sh.D, sh.H, sh.W, p.aw, p.kbw, p.kbh,
                     p.kbd) ||
      (!transposed && !map_x2(maps, sh, p.aw, p.kbw, p.kbh, p.kbd)))
    return cudaErrorInvalidValue;
  if (!transposed) {
    if (!map_act_dense(&maps.a[1], dy, sh.dy_cs, sh.N, sh.D, sh.H, sh.W, 64, p.kbw, p.kbh, p.kbd))
      return cudaErrorInvalidValue;
  } else {
    int D2 = 2 * sh.D, H2 = 2 * sh.H, W2 = 2 * sh.W;
    int64_t cs = sh.dy_cs;
    for (int par = 0; par < 8; ++par) {   // maps 1..8: parity views (pz,py,px) of dY
      int pz = (par >> 2) & 1, py = (par >> 1) & 1, px = par & 1;
      const __nv_bfloat16* b0 = dy + (((int64_t)pz * H2 + py) * W2 + px) * cs;
      if (!map_act(&maps.a[1 + par], b0, (int)cs, sh.N, sh.D, sh.H, sh.W, 2 * cs, 2 * cs * W2,
                   2 * cs * W2 * H2, cs * W2 * H2 * D2, 64, p.kbw, p.kbh, p.kbd))
        return cudaErrorInvalidValue;
    }
  }
  if (p.splits == 1) p.gw = gw;   // no K split: the epilogue writes the gradient itself
  cudaError_t e;
  if (p.aw == 32) e = launch_wg<64, 128, 32>(s, maps, p);
  else if (p.tt == kWgTT) e = launch_wg<64, 64, 64, kWgTT>(s, maps, p);
  else if (bnp == 64 && kb == 128) e = launch_wg<64, 128, 64>(s, maps, p);
  else if (bnp == 128 && kb == 128) e = launch_wg<128, 128, 64>(s, maps, p);
  else if (bnp == 256 && kb == 64 && p.caseA && (p.Cout / 128) % 2 == 0 &&
           z2_pair_enabled() && p.splits * p.tiles % 2 == 0)
    e = launch_wg_pair(s, maps, p);
  else if (bnp == 256 && kb == 64) e = launch_wg<256, 64, 64>(s, maps, p);
  else return cudaErrorInvalidConfiguration;
  if (e != cudaSuccess) return e;
  if (p.gw) return cudaSuccess;
  int64_t total = 128LL * bnp * p.rtiles;
  int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_wgrad_reduce<<<grid, 256, 0, s>>>(p, gw);
  return cudaGetLastError();
}

}  // namespace

namespace {
bool wgrad_halo_ok(const ConvShape& sh, bool transposed) {
  return !transposed && !halo_disabled() && sh.Cout == 64 && sh.Cin % 64 == 0 &&
         sh.W >= 32 && sh.H >= 16;
}

void wgrad_halo_setup(const ConvShape& sh, WgHaloParams& p) {
  std::memset(&p, 0, sizeof p);
  p.Nb = sh.N; p.D = sh.D; p.H = sh.H; p.W = sh.W;
  p.tw = (sh.W + 7) / 8;
  p.th = (sh.H + 15) / 16;
  p.kblocks = sh.N * sh.D * p.th * p.tw;
  p.chunks = sh.Cin / 64;
  p.units = 2 * p.chunks;
  p.splits = std::max(1, std::min(p.kblocks, (2 * num_sms() + p.units - 1) / p.units));
  p.x_c0 = sh.x_co;
  p.dy_c0 = sh.dy_co;
}

cudaError_t wgrad_halo_run(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                           const __nv_bfloat16* dy, float* gw, float* work) {
  WgHaloParams p;
  wgrad_halo_setup(sh, p);
  p.part = work;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  if (!map_act_dense(&maps.a[0], x, sh.x_cs, sh.N, sh.D, sh.H, sh.W, 64, kHW, kHH, kHD) ||
      !map_x2(maps, sh, 64, kHW, kHH, kHD))
    return cudaErrorInvalidValue;
  const bool pair = z2_pair_enabled() && p.chunks % 2 == 0;
  if (!map_act_dense(&maps.a[1], dy, sh.dy_cs, sh.N, sh.D, sh.H, sh.W, pair ? 32 : 64, 8, 16, 1))
    return cudaErrorInvalidValue;
  cudaError_t e;
  if (pair) {
    const size_t smem = 2 * ((size_t)kHaloStride + 128 * 64) + 1024;
    static bool configured = false;
    if (!configured) {
      e = cudaFuncSetAttribute(k_wgrad_halo<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
      if (e != cudaSuccess) return e;
      configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(std::min(p.units * p.splits, num_sms() / 2 * 2));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_wgrad_halo<true>, maps, p);
  } else {
    const size_t smem = 2 * ((size_t)kHaloStride + 128 * 128) + 1024;
    static bool configured = false;
    if (!configured) {
      e = cudaFuncSetAttribute(k_wgrad_halo<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
      if (e != cudaSuccess) return e;
      configured = true;
    }
    int grid = std::min(p.units * p.splits, num_sms());
    k_wgrad_halo<false><<<grid, kThreads, smem, s>>>(maps, p);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return e;
  int64_t total = (int64_t)kWgPairs * 128 * 64 * p.units;
  k_wgrad_halo_reduce<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(
      p, sh.Cin, gw);
  return cudaGetLastError();
}
}  // namespace

namespace {
bool wgrad_halo_a_ok(const ConvShape& sh, bool transposed) {
  // wins where the per-tap path is L2/smem bound (Cin <= 128); wider inputs keep the
  // per-tap kernel, whose 256-wide N tiles already reach ~1 PFLOP/s
  return !transposed && !halo_disabled() && sh.Cout % 128 == 0 && sh.Cin % 64 == 0 &&
         sh.Cin <= 128 && sh.W >= 32 && sh.H >= 16;
}

void wgrad_halo_a_setup(const ConvShape& sh, WgHaloAParams& p) {
  std::memset(&p, 0, sizeof p);
  p.Nb = sh.N; p.D = sh.D; p.H = sh.H; p.W = sh.W;
  p.tw = (sh.W + 7) / 8;
  p.th = (sh.H + 15) / 16;
  p.kblocks = sh.N * sh.D * p.th * p.tw;
  p.cchunks = sh.Cin / 64;
  p.coblocks = sh.Cout / 128;
  p.units = p.cchunks * 4 * p.coblocks;
  p.splits = std::max(1, std::min(p.kblocks, (2 * num_sms() + p.units - 1) / p.units));
  p.x_c0 = sh.x_co;
  p.dy_c0 = sh.dy_co;
  p.Cin = sh.Cin;
}

cudaError_t wgrad_halo_a_run(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                             const __nv_bfloat16* dy, float* gw, float* work) {
  WgHaloAParams p;
  wgrad_halo_a_setup(sh, p);
  p.part = work;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  if (!map_act_dense(&maps.a[0], x, sh.x_cs, sh.N, sh.D, sh.H, sh.W, 64, kHW, kHH, kHD) ||
      !map_x2(maps, sh, 64, kHW, kHH, kHD))
    return cudaErrorInvalidValue;
  if (!map_act_dense(&maps.a[1], dy, sh.dy_cs, sh.N, sh.D, sh.H, sh.W, 64, 8, 16, 1))
    return cudaErrorInvalidValue;
  size_t smem = 2 * ((size_t)kHaloStride + 2 * 128 * 128) + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_wgrad_halo_a,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int grid = std::min(p.units * p.splits, num_sms());
  k_wgrad_halo_a<<<grid, kThreads, smem, s>>>(maps, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int64_t total = (int64_t)kWgTaps * 128 * 64 * p.units;
  k_wgrad_halo_a_reduce<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(
      p, gw);
  return cudaGetLastError();
}
}  // namespace


namespace {
// Halo-view weight gradient (k_wgrad_hv): every stride-1 conv wgrad with Cout == 64 or
// Cout % 128 == 0 on grids wide enough for 8 x 8 x 2 voxel K blocks (US_NO_HV=1: the
// earlier tap-pair / 8-tap halo kernels, for A/B measurements).
bool hv_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("US_NO_HV");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool hv_xa_enabled() {   // US_HV_XA=1: the Cout == 64 variant too (measured r02: on par with
  static int v = -1;       // the CTA-pair tap-pair kernel, 1.40 vs 1.37 ms at 192^3 64->64)
  if (v < 0) {
    const char* e = getenv("US_HV_XA");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool wgrad_hv_ok(const ConvShape& sh, bool transposed) {
  // measured r02 (1 B200): XB beats the 8-tap halo / per-tap kernels at 48^3..96^3
  // (256->128 @96^3 1.78 -> 1.38 ms, 512->256 @48^3 0.81 -> 0.68 ms) but not at 24^3, where
  // the 8 x 8 x 2 K blocks leave too few units per SM
  const bool xa = sh.Cout == 64;
  return !transposed && !halo_disabled() && !hv_disabled() && sh.Cin % 64 == 0 &&
         (xa ? hv_xa_enabled() : sh.Cout % 128 == 0) && sh.W >= 32 && sh.H >= 16 &&
         sh.D >= 2;
}

void wgrad_hv_setup(const ConvShape& sh, WgHvParams& p) {
  std::memset(&p, 0, sizeof p);
  const bool xa = sh.Cout == 64;
  p.Nb = sh.N; p.D = sh.D; p.H = sh.H; p.W = sh.W;
  p.tw = (sh.W + 7) / 8;
  p.th = (sh.H + 7) / 8;
  p.td = (sh.D + 1) / 2;
  p.kblocks = sh.N * p.td * p.th * p.tw;
  p.cchunks = sh.Cin / 64;
  p.coblocks = xa ? 1 : sh.Cout / 128;
  p.groups = xa ? 3 : 5;
  p.units = p.cchunks * p.coblocks * p.groups;
  // ~3 work items per SM: with 3 groups per chunk and 148 SMs every CTA then gets one item
  // of each group (balanced although the last group holds one accumulator, not two)
  p.splits = std::max(1, std::min(p.kblocks, (3 * num_sms() + p.units - 1) / p.units));
  p.x_c0 = sh.x_co;
  p.dy_c0 = sh.dy_co;
  p.Cin = sh.Cin;
}

size_t wgrad_hv_workspace(const ConvShape& sh) {
  WgHvParams p;
  wgrad_hv_setup(sh, p);
  return (size_t)p.splits * p.units * kHvAcc * 128 * kHvN * sizeof(float);
}

template <bool XA>
cudaError_t launch_hv(cudaStream_t s, const Maps& maps, const WgHvParams& p, float* gw) {
  constexpr size_t smem = (size_t)(XA ? kHvXaStages * kHvXaStage : kHvXbStages * kHvXbStage) + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_wgrad_hv<XA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int grid = std::min(p.units * p.splits, num_sms());
  k_wgrad_hv<XA><<<grid, kThreads, smem, s>>>(maps, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t total = (int64_t)kHvAcc * 128 * kHvN * p.units;
  k_wgrad_hv_reduce<XA><<<(int)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(p, gw);
  return cudaGetLastError();
}

cudaError_t wgrad_hv_run(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                         const __nv_bfloat16* dy, float* gw, float* work) {
  WgHvParams p;
  wgrad_hv_setup(sh, p);
  p.part = work;
  const bool xa = sh.Cout == 64;
  Maps maps;
  std::memset(&maps, 0, sizeof maps);
  const int xbw = xa ? 8 : 10;   // XA: no w halo on X (the w shift is on dY)
  if (!map_act_dense(&maps.a[0], x, sh.x_cs, sh.N, sh.D, sh.H, sh.W, 64, xbw, 10, 4) ||
      !map_x2(maps, sh, 64, xbw, 10, 4))
    return cudaErrorInvalidValue;
  if (!map_act_dense(&maps.a[1], dy, sh.dy_cs, sh.N, sh.D, sh.H, sh.W, 64, xa ? 10 : 8, 8, 2))
    return cudaErrorInvalidValue;
  return xa ? launch_hv<true>(s, maps, p, gw) : launch_hv<false>(s, maps, p, gw);
}
}  // namespace

size_t wgrad_tc_workspace(const ConvShape& sh, bool transposed) {
  if (wgrad_hv_ok(sh, transposed)) return wgrad_hv_workspace(sh);
  if (wgrad_halo_a_ok(sh, transposed)) {
    WgHaloAParams hp;
    wgrad_halo_a_setup(sh, hp);
    return (size_t)hp.splits * hp.units * kWgTaps * 128 * 64 * sizeof(float);
  }
  if (wgrad_halo_ok(sh, transposed)) {
    WgHaloParams hp;
    wgrad_halo_setup(sh, hp);
    return (size_t)hp.splits * hp.units * kWgPairs * 128 * 64 * sizeof(float);
  }
  WgParams p;
  int bnp, kb;
  if (!wg_setup(sh, transposed, p, bnp, kb)) return 0;
  if (p.splits == 1) return 16;   // written straight into the gradient buffer
  return (size_t)p.splits * p.rtiles * 128 * bnp * sizeof(float);
}

cudaError_t conv_wgrad_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                          const __nv_bfloat16* dy, float* gw, float* work) {
  if (wgrad_hv_ok(sh, false)) return wgrad_hv_run(s, sh, x, dy, gw, work);
  if (wgrad_halo_a_ok(sh, false)) return wgrad_halo_a_run(s, sh, x, dy, gw, work);
  if (wgrad_halo_ok(sh, false)) return wgrad_halo_run(s, sh, x, dy, gw, work);
  return wgrad_run(s, sh, false, x, dy, gw, work);
}

cudaError_t convt_wgrad_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                           const __nv_bfloat16* dy, float* gw, float* work) {
  return wgrad_run(s, sh, true, x, dy, gw, work);
}



// ---------------------------------------------------------------- stem (4-channel input layer)
// The 4-modality input layer is a 3x3x3 conv over 4 channels: its implicit GEMM has
// K = 108, far too narrow for per-tap tcgen05 operands (8-byte channel rows).  It
// runs as ONE GEMM with K = 128 (27 taps x 4 channels, zero padded) whose A operand
// is an im2col tile built by threads in shared memory (never materialised in HBM).
// Weights [Cout][27][4] are exactly the im2col column order, so the forward only
// pads each weight row to 128 columns and the weight gradient is written straight
// into the [Cout][27][4] gradient slot.
namespace {
constexpr int kStemK = 128;
}  // namespace

namespace {
// ---- fused 4-channel stem.  A tile is a bw x bh x 1 block of 128 voxels (bw 32 or
// 16).  Its input halo -- (bw+4) x (bh+2) x 3 voxels x 4 channels, one 5-D TMA box
// whose out-of-volume part is zero filled (= the conv padding; the box starts 2
// voxels left of the tile because a TMA box must start on a 16-byte boundary,
// csrc/selftest_umma.cu T8) -- is staged by the producer warp several tiles ahead.  Four gather warps then assemble the im2col
// tile: thread r writes row r = 128 K-columns (27 taps x 4 channels + 20 zero) as
// two 64-column SWIZZLE_128B chunks (16-byte piece p of a 128-byte line at
// p ^ (r & 7), the layout a SWIZZLE_128B TMA box would produce).  The same stage
// is the K-major A operand of the forward GEMM (M = voxels) and the MN-major A
// operand of the weight gradient (M = K-columns, K = voxels).
constexpr int kStemStageA = 2 * 128 * 128;     // 32 KB
constexpr int kStemThreads = 320;              // w0 TMA, w1 MMA, w2-5 epilogue, w6-9 gather
constexpr int kStemHaloStride = 6144;          // >= 36 x 6 x 3 x 8 B, 1 KB aligned
constexpr int kStemHaloStages = 6;

struct StemGeo {
  int Nb, D, H, W;
  int bw, bh;          // tile box (bw * bh == 128)
  int tx, ty;          // tiles along W, H
  int tiles;
  int halo_bytes;      // (bw+4)*(bh+2)*3*8
};

__device__ __forceinline__ void stem_origin(const StemGeo& g, int tile, int& n, int& z, int& y0,
                                            int& x0) {
  int xb = tile % g.tx;
  int r = tile / g.tx;
  int yb = r % g.ty;
  r /= g.ty;
  z = r % g.D;
  n = r / g.D;
  x0 = xb * g.bw;
  y0 = yb * g.bh;
}

__device__ __forceinline__ void stem_halo_tma(const StemGeo& g, const CUtensorMap* xmap,
                                              uint8_t* dst, uint64_t* bar, int tile) {
  int n, z, y0, x0;
  stem_origin(g, tile, n, z, y0, x0);
  mbar_arrive_expect_tx(bar, g.halo_bytes);
  tma_load_5d(dst, xmap, bar, (x0 - 2) * 4, y0 - 1, z - 1, n, 0);
}

__device__ __forceinline__ void stem_build_row(const StemGeo& g, const uint2* hs, uint8_t* stage,
                                               int r, bool ones_col) {
  const int HX = g.bw + 4, HY = g.bh + 2;
  const int lx = r % g.bw, ly = r / g.bw;
  const uint2* c = hs + ly * HX + lx + 1;   // halo x starts at x0 - 2
  uint2 v[32];
#pragma unroll
  for (int t = 0; t < 32; ++t)
    v[t] = t < 27 ? c[((t / 9) * HY + (t / 3) % 3) * HX + t % 3] : make_uint2(0u, 0u);
  if (ones_col) v[31].y = 0x3F800000u;   // bf16 1.0 in K-column 127 (tap 31, channel 3)
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int hh = j >> 3, pc = j & 7;
    *reinterpret_cast<uint4*>(stage + hh * (128 * 128) + r * 128 + ((pc ^ (r & 7)) << 4)) =
        make_uint4(v[2 * j].x, v[2 * j].y, v[2 * j + 1].x, v[2 * j + 1].y);
  }
}

// Gather-warp loop: tiles in this CTA's order; halo stage hs and A stage `stage`.
template <int STAGES, class NextTile>
__device__ __forceinline__ void stem_gather_loop(const StemGeo& g, uint8_t* stages,
                                                 int stage_stride, uint64_t* full,
                                                 uint64_t* empty, uint8_t* halo, uint64_t* hfull,
                                                 uint64_t* hempty, int first, NextTile next,
                                                 bool ones_col) {
  const int r = threadIdx.x - 192;
  int stage = 0, hs = 0;
  uint32_t phase = 0, hphase = 0;
  for (int tile = first; tile >= 0; tile = next(tile)) {
    mbar_wait(&hfull[hs], hphase);
    mbar_wait(&empty[stage], phase ^ 1);
    stem_build_row(g, reinterpret_cast<const uint2*>(halo + hs * kStemHaloStride),
                   stages + stage * stage_stride, r, ones_col);
    fence_proxy_async_smem();
    mbar_arrive(&full[stage]);
    mbar_arrive(&hempty[hs]);
    if (++stage == STAGES) { stage = 0; phase ^= 1; }
    if (++hs == kStemHaloStages) { hs = 0; hphase ^= 1; }
  }
}

// BatchNorm statistics without a per-tile reduction: the gather puts a 1.0 in the
// (zero-weight) K-column 127 of every row, and a second MMA per tile accumulates
// the Gram matrix G = Xcol^T Xcol (128 x 128, TMEM columns 128..255).  Then for
// channel c with weight row w_c:  sum_v y = G[127] . w_c  and  sum_v y^2 = w_c^T G w_c,
// evaluated once per CTA.  The tensor core does the statistics at 2x the GEMM's
// (tiny) MMA time instead of a per-tile cross-lane reduction in the epilogue.
template <int STAGES>
__global__ void __launch_bounds__(kStemThreads, 1)
    k_stem_fwd(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
               const __nv_bfloat16* __restrict__ w, float* __restrict__ stats, const StemGeo g) {
  constexpr int kCout = 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sB = smem;                       // 2 chunks x 64 rows x 128 B
  uint8_t* sA = smem + 2 * 64 * 128;
  uint8_t* sH = sA + STAGES * kStemStageA;  // halo stages
  // output staging for TMA stores: 2 x (128 rows x 128 B), SWIZZLE_128B like the y map
  uint8_t* sO = sH + kStemHaloStages * kStemHaloStride;
  __shared__ __align__(8) uint64_t afull[STAGES], aempty[STAGES], tfull[2], tempty[2], gdone;
  __shared__ __align__(8) uint64_t hfull[kStemHaloStages], hempty[kStemHaloStages];
  __shared__ uint32_t tmem_base_s;
  __shared__ float wf[kCout][kStemK + 1];   // fp32 weights for the statistics
  __shared__ float stat_s[4][2 * kCout];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool want_stats = stats != nullptr;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&afull[s], 128);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < kStemHaloStages; ++s) {
      mbar_init(&hfull[s], 1);
      mbar_init(&hempty[s], 128);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    mbar_init(&gdone, 1);
    fence_barrier_init();
  }
  // weights [64][108] -> K-major SWIZZLE_128B operand, K zero-padded to 128
  for (int i = threadIdx.x; i < kCout * 16; i += blockDim.x) {
    const int o = i / 16, j = i % 16, hh = j >> 3, pc = j & 7;
    __align__(16) __nv_bfloat16 v8[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int k = j * 8 + e;
      v8[e] = k < 108 ? w[o * 108 + k] : __float2bfloat16(0.f);
      wf[o][k] = __bfloat162float(v8[e]);
    }
    *reinterpret_cast<uint4*>(sB + hh * (64 * 128) + o * 128 + ((pc ^ (o & 7)) << 4)) =
        *reinterpret_cast<const uint4*>(v8);
  }
  fence_proxy_async_smem();
  if (warp == 1) tmem_alloc<256>(&tmem_base_s);
  if (warp == 0 && lane == 0) tma_prefetch(&xmap);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  const uint32_t tmem_g = tmem_base + 128;

  if (warp == 0) {
    if (elect_one()) {
      int hs = 0;
      uint32_t hphase = 0;
      for (int tile = blockIdx.x; tile < g.tiles; tile += gridDim.x) {
        mbar_wait(&hempty[hs], hphase ^ 1);
        stem_halo_tma(g, &xmap, sH + hs * kStemHaloStride, &hfull[hs], tile);
        if (++hs == kStemHaloStages) { hs = 0; hphase ^= 1; }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, kCout, 0, 0);
    constexpr uint32_t idesc_g = idesc_bf16(128, 128, 1, 1);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    int stage = 0, acc = 0;
    uint32_t phase = 0, aphase = 0;
    bool first = true;
    for (int tile = blockIdx.x; tile < g.tiles; tile += gridDim.x) {
      mbar_wait(&tempty[acc], aphase ^ 1);
      mbar_wait(&afull[stage], phase);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = a0 + stage * kStemStageA;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          uint64_t ad = smem_desc(sa + (k >> 2) * (128 * 128) + (k & 3) * 32, 16, 1024, 2);
          uint64_t bd = smem_desc(b0 + (k >> 2) * (64 * 128) + (k & 3) * 32, 16, 1024, 2);
          umma_bf16(tmem_base + acc * kCout, ad, bd, idesc, k != 0);
        }
        umma_commit(&tfull[acc]);
        if (want_stats) {
          // G += Xcol^T Xcol: the stage viewed MN-major (M = N = K-columns, K = voxels)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            uint64_t gd = smem_desc(sa + k * 2048, 128 * 128, 1024, 2);
            umma_bf16(tmem_g, gd, gd, idesc_g, (first && k == 0) ? 0u : 1u);
          }
        }
        umma_commit(&aempty[stage]);
      }
      __syncwarp();
      first = false;
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    if (elect_one()) umma_commit(&gdone);
    __syncwarp();
  } else if (warp >= 6) {
    const int step = gridDim.x, tiles = g.tiles;
    stem_gather_loop<STAGES>(g, sA, kStemStageA, afull, aempty, sH, hfull, hempty,
                             blockIdx.x < tiles ? (int)blockIdx.x : -1,
                             [=](int t) { return t + step < tiles ? t + step : -1; },
                             want_stats);
  } else if (warp >= 2) {
    const int q = warp & 3, row = q * 32 + lane;
    int acc = 0;
    uint32_t aphase = 0;
    bool any = false;
    const bool leader = threadIdx.x == 64;
    int stg = 0;
    for (int tile = blockIdx.x; tile < g.tiles; tile += gridDim.x) {
      int n, z, y0, x0;
      stem_origin(g, tile, n, z, y0, x0);
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      uint32_t rr[2][32];
      tmem_ld32(tmem_base + acc * kCout + ((uint32_t)(q * 32) << 16), rr[0]);
      tmem_ld32(tmem_base + acc * kCout + 32 + ((uint32_t)(q * 32) << 16), rr[1]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      // the staging buffer of two tiles ago must have been read by its TMA store
      if (leader) tma_store_wait_read<1>();
      asm volatile("bar.sync 2, 128;" ::: "memory");
      uint8_t* stage = sO + stg * (128 * 128);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int chunk = hh * 4 + j;   // 16-byte piece of the 128-byte row
          *reinterpret_cast<uint4*>(stage + row * 128 + ((chunk ^ (row & 7)) << 4)) = make_uint4(
              pack_bf16(__uint_as_float(rr[hh][8 * j]), __uint_as_float(rr[hh][8 * j + 1])),
              pack_bf16(__uint_as_float(rr[hh][8 * j + 2]), __uint_as_float(rr[hh][8 * j + 3])),
              pack_bf16(__uint_as_float(rr[hh][8 * j + 4]), __uint_as_float(rr[hh][8 * j + 5])),
              pack_bf16(__uint_as_float(rr[hh][8 * j + 6]), __uint_as_float(rr[hh][8 * j + 7])));
        }
      fence_proxy_async_smem();
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (leader) {
        for (int j = 0; j < g.bh; ++j) {   // one box per output row of the tile
          const int64_t v0 = (((int64_t)n * g.D + z) * g.H + y0 + j) * g.W + x0;
          tma_store_2d(&ymap, stage + j * g.bw * 128, 0, (int)v0);
        }
        tma_store_commit();
      }
      stg ^= 1;
      any = true;
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    if (leader) tma_store_wait<0>();
    if (want_stats) {
      // thread k owns Gram row k: t_c = G[k] . w_c ; sum y = t_c of row 127,
      // sum y^2 = sum_k w_c[k] t_c (reduced over the 128 rows below)
      float gk[kStemK];
      if (any) {
        mbar_wait(&gdone, 0);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < kStemK; c0 += 32) {
          uint32_t rr[32];
          tmem_ld32(tmem_g + c0 + ((uint32_t)(q * 32) << 16), rr);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) gk[c0 + j] = __uint_as_float(rr[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < kStemK; ++j) gk[j] = 0.f;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < kCout; c0 += 32) {
        float s2[32], s1[32];
#pragma unroll 1
        for (int j = 0; j < 32; ++j) {
          const float* wc = wf[c0 + j];
          float t = 0.f;
#pragma unroll
          for (int l = 0; l < 108; ++l) t = fmaf(gk[l], wc[l], t);
          s2[j] = wc[row] * t;
          s1[j] = row == 127 ? t : 0.f;
        }
        float a1 = warp_colsum32(s1);
        float a2 = warp_colsum32(s2);
        stat_s[q][c0 + lane] = a1;
        stat_s[q][kCout + c0 + lane] = a2;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (want_stats)
    for (int i = threadIdx.x; i < 2 * kCout; i += blockDim.x)
      stats[(int64_t)blockIdx.x * 2 * kCout + i] =
          ((stat_s[0][i] + stat_s[1][i]) + stat_s[2][i]) + stat_s[3][i];
  if (warp == 1) tmem_dealloc<256>(tmem_base);
}

// dW[k][co] = sum_v Xcol[v][k] dY[v][co]: A = gathered Xcol stage (MN-major, M = k),
// B = the tile's dY rows [128 voxels x 64] by TMA (bh boxes of bw voxels, MN-major).
// CTA u accumulates tiles [u*kper, (u+1)*kper) and writes one fp32 partial [128][64].
template <int STAGES>
__global__ void __launch_bounds__(kStemThreads, 1)
    k_stem_wgrad(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap dymap,
                 float* __restrict__ part, const StemGeo g, int splits) {
  constexpr int kB = 128 * 128;                      // dY stage: 128 voxels x 64 ch
  constexpr int kStage = kStemStageA + kB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sH = smem + STAGES * kStage;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ __align__(8) uint64_t hfull[kStemHaloStages], hempty[kStemHaloStages];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kper = (g.tiles + splits - 1) / splits;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 129);     // 128 gather threads + the dY TMA
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kStemHaloStages; ++s) {
      mbar_init(&hfull[s], 1);
      mbar_init(&hempty[s], 128);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<128>(&tmem_base_s);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&dymap);
    tma_prefetch(&xmap);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  const int step = gridDim.x, tiles = g.tiles;
  auto next_tile = [=](int t) {
    int u = t / kper;
    if (t + 1 < min(tiles, (u + 1) * kper)) return t + 1;
    for (u += step; u < splits; u += step)
      if (u * kper < tiles) return u * kper;
    return -1;
  };
  auto first_tile = [=](int u) {
    for (; u < splits; u += step)
      if (u * kper < tiles) return u * kper;
    return -1;
  };

  if (warp == 0) {
    if (elect_one()) {
      // halos run ahead of the dY loads by up to kStemHaloStages tiles
      int stage = 0, hs = 0, ht = first_tile((int)blockIdx.x);
      uint32_t phase = 0, hphase = 0;
      int hissued = 0, dissued = 0;
      for (int t = first_tile((int)blockIdx.x); t >= 0; t = next_tile(t)) {
        while (ht >= 0 && hissued < dissued + kStemHaloStages) {
          mbar_wait(&hempty[hs], hphase ^ 1);
          stem_halo_tma(g, &xmap, sH + hs * kStemHaloStride, &hfull[hs], ht);
          if (++hs == kStemHaloStages) { hs = 0; hphase ^= 1; }
          ht = next_tile(ht);
          ++hissued;
        }
        int n, z, y0, x0;
        stem_origin(g, t, n, z, y0, x0);
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], kB);
        uint8_t* sb = smem + stage * kStage + kStemStageA;
        for (int j = 0; j < g.bh; ++j) {
          const int64_t v = (((int64_t)n * g.D + z) * g.H + y0 + j) * g.W + x0;
          tma_load_2d(sb + j * g.bw * 128, &dymap, &full[stage], 0, (int)v);
        }
        ++dissued;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, 64, 1, 1);
    const uint32_t base = smem_u32(smem);
    int stage = 0, acc = 0;
    uint32_t phase = 0, aphase = 0;
    for (int u = blockIdx.x; u < splits; u += gridDim.x) {
      const int kb0 = u * kper, kb1 = min(g.tiles, kb0 + kper);
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = base + stage * kStage, sb = sa + kStemStageA;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            uint64_t ad = smem_desc(sa + k * 2048, 128 * 128, 1024, 2);
            uint64_t bd = smem_desc(sb + k * 2048, kB, 1024, 2);
            umma_bf16(tmem_base + acc * 64, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  } else if (warp >= 6) {
    stem_gather_loop<STAGES>(g, smem, kStage, full, empty, sH, hfull, hempty,
                             first_tile((int)blockIdx.x), next_tile, false);
  } else if (warp >= 2) {
    const int q = warp & 3, row = q * 32 + lane;
    int acc = 0;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < splits; u += gridDim.x) {
      const int kb0 = u * kper, kb1 = min(g.tiles, kb0 + kper);
      float* dst = part + ((int64_t)u * 128 + row) * 64;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t rr[32];
        tmem_ld32(tmem_base + acc * 64 + c0 + ((uint32_t)(q * 32) << 16), rr);
        tmem_ld_wait();
        float4* d4 = reinterpret_cast<float4*>(dst + c0);
        const bool empty_unit = kb1 <= kb0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          d4[j] = empty_unit ? make_float4(0.f, 0.f, 0.f, 0.f)
                             : make_float4(__uint_as_float(rr[4 * j]), __uint_as_float(rr[4 * j + 1]),
                                           __uint_as_float(rr[4 * j + 2]), __uint_as_float(rr[4 * j + 3]));
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<128>(tmem_base);
}

constexpr int kStemFwdStages = 3;
constexpr int kStemWgStages = 3;

bool stem_geo(const ConvShape& sh, StemGeo& g) {
  // (the dense 4-channel input layout x_cs == 4 is checked at launch; the workspace
  // query does not carry it)
  if (sh.Cin != 4 || sh.Cout != 64) return false;
  g.Nb = sh.N; g.D = sh.D; g.H = sh.H; g.W = sh.W;
  if (sh.W % 32 == 0 && sh.H % 4 == 0) { g.bw = 32; g.bh = 4; }
  else if (sh.W % 16 == 0 && sh.H % 8 == 0) { g.bw = 16; g.bh = 8; }
  else return false;
  g.tx = sh.W / g.bw;
  g.ty = sh.H / g.bh;
  int64_t tiles = (int64_t)sh.N * sh.D * g.ty * g.tx;
  if (tiles >= (1LL << 31)) return false;
  g.tiles = (int)tiles;
  g.halo_bytes = (g.bw + 4) * (g.bh + 2) * 3 * 8;
  return true;
}

// 5-D map over the 4-channel NDHWC input viewed as (W*4, H, D, N, 1) with a halo box.
bool stem_xmap(CUtensorMap* m, const __nv_bfloat16* x, const StemGeo& g) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[5] = {(cuuint64_t)g.W * 4, (cuuint64_t)g.H, (cuuint64_t)g.D, (cuuint64_t)g.Nb, 1};
  cuuint64_t rowb = (cuuint64_t)g.W * 4 * 2;
  cuuint64_t strides[4] = {rowb, rowb * g.H, rowb * g.H * g.D, rowb * g.H * g.D * g.Nb};
  cuuint32_t box[5] = {(cuuint32_t)(g.bw + 4) * 4, (cuuint32_t)(g.bh + 2), 3, 1, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<__nv_bfloat16*>(x), dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool stem_fused(const ConvShape& sh) {
  StemGeo g{};
  return stem_geo(sh, g);
}

int stem_fused_splits(const ConvShape& sh) {
  StemGeo g{};
  if (!stem_geo(sh, g)) return 1;
  return std::max(1, std::min(g.tiles, num_sms()));
}
}  // namespace

bool stem_supported(const ConvShape& sh, bool wgrad) {
  (void)wgrad;
  return encode_fn() != nullptr && stem_fused(sh);
}

int stem_stat_parts(const ConvShape& sh) { return stem_fused_splits(sh); }

size_t stem_fwd_workspace(const ConvShape& sh) {
  return (size_t)stem_stat_parts(sh) * 2 * sh.Cout * sizeof(float);
}

cudaError_t conv_fwd_stem(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                          const __nv_bfloat16* w, __nv_bfloat16* y, void* work) {
  StemGeo g{};
  if (!stem_supported(sh, false) || !stem_geo(sh, g) || sh.x_cs != 4 || sh.x_co != 0)
    return cudaErrorInvalidValue;
  constexpr size_t smem = 2 * 64 * 128 + (size_t)kStemFwdStages * kStemStageA +
                         (size_t)kStemHaloStages * kStemHaloStride + 2 * 128 * 128 + 1024;
  CUtensorMap xmap, ymap;
  if (!stem_xmap(&xmap, x, g)) return cudaErrorInvalidValue;
  {  // output y as [nvox][64] bf16, box 64 channels x bw voxels, SWIZZLE_128B
    auto fn = encode_fn();
    const int64_t nvox = (int64_t)sh.N * sh.D * sh.H * sh.W;
    cuuint64_t dims[2] = {64, (cuuint64_t)nvox};
    cuuint64_t strides[1] = {64 * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)g.bw};
    cuuint32_t es[2] = {1, 1};
    if (fn(&ymap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_stem_fwd<kStemFwdStages>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k_stem_fwd<kStemFwdStages><<<stem_stat_parts(sh), kStemThreads, smem, s>>>(xmap, ymap, w,
                                                                             (float*)work, g);
  return cudaGetLastError();
}

size_t stem_wgrad_workspace(const ConvShape& sh) {
  return (size_t)stem_fused_splits(sh) * 128 * 64 * sizeof(float);
}

cudaError_t conv_wgrad_stem(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                            const __nv_bfloat16* dy, float* gw, void* work) {
  StemGeo g{};
  if (!stem_supported(sh, true) || !stem_geo(sh, g) || sh.x_cs != 4 || sh.x_co != 0)
    return cudaErrorInvalidValue;
  const int splits = stem_fused_splits(sh);
  const int64_t nvox = (int64_t)sh.N * sh.D * sh.H * sh.W;
  CUtensorMap dymap;
  {
    auto fn = encode_fn();
    cuuint64_t dims[2] = {(cuuint64_t)sh.dy_cs, (cuuint64_t)nvox};
    cuuint64_t strides[1] = {(cuuint64_t)sh.dy_cs * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)g.bw};
    cuuint32_t es[2] = {1, 1};
    if (fn(&dymap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(dy) + sh.dy_co,
           dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  constexpr size_t smem = (size_t)kStemWgStages * (kStemStageA + 128 * 128) +
                         (size_t)kStemHaloStages * kStemHaloStride + 1024;
  CUtensorMap xmap;
  if (!stem_xmap(&xmap, x, g)) return cudaErrorInvalidValue;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_stem_wgrad<kStemWgStages>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k_stem_wgrad<kStemWgStages><<<splits, kStemThreads, smem, s>>>(xmap, dymap, (float*)work, g,
                                                                 splits);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // reduce the per-CTA [128 K-columns][64] partials into gw[co][27][4] (columns < 108)
  WgParams p;
  std::memset(&p, 0, sizeof p);
  p.caseA = 0;
  p.Cin = kStemK;
  p.Cout = 64;
  p.bnp = 64;
  p.aw = 64;
  p.tiles = 1;
  p.rtiles = 1;
  p.tt = 1;
  p.splits = splits;
  p.gw_co_stride = 108;
  p.gw_cmax = 108;
  p.part = (float*)work;
  k_wgrad_reduce<<<(128 * 64 + 255) / 256, 256, 0, s>>>(p, gw);
  return cudaGetLastError();
}

}  // namespace us
