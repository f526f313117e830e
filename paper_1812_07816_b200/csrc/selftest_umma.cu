// Descriptor self-test for the tcgen05 paths the conv kernels rely on.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o selftest_umma selftest_umma.cu -lcuda
// Each case loads A and B tiles with TMA, issues tcgen05.mma with the
// descriptor parameters under test and compares D against a host GEMM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>
#include "sm100.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(2);} } while (0)

struct Box { int map; int c0, c1; int smem_off; int bytes; };
struct Operand { uint32_t start, lbo, sbo, layout, base_off, kstep; };
struct Params {
  Box boxes[8]; int nboxes; int total_bytes;
  Operand a, b; int M, N, K; int a_mn, b_mn;
};

__global__ void __launch_bounds__(128) umma_test(const __grid_constant__ CUtensorMap m0,
                                                 const __grid_constant__ CUtensorMap m1,
                                                 const __grid_constant__ CUtensorMap m2,
                                                 Params p, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    us::mbar_init(&bar_load, 1);
    us::mbar_init(&bar_mma, 1);
    us::fence_barrier_init();
  }
  if (warp == 1) us::tmem_alloc<256>(&tmem_base);
  us::tc_fence_before();
  __syncthreads();
  us::tc_fence_after();
  uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    us::mbar_arrive_expect_tx(&bar_load, p.total_bytes);
    for (int i = 0; i < p.nboxes; ++i) {
      const CUtensorMap* m = p.boxes[i].map == 0 ? &m0 : p.boxes[i].map == 1 ? &m1 : &m2;
      us::tma_load_2d(smem + p.boxes[i].smem_off, m, &bar_load, p.boxes[i].c0, p.boxes[i].c1);
    }
  }
  us::mbar_wait(&bar_load, 0);
  us::tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t base = us::smem_u32(smem);
    uint32_t idesc = us::idesc_bf16(p.M, p.N, p.a_mn, p.b_mn);
    for (int k = 0; k < p.K / 16; ++k) {
      uint64_t ad = us::smem_desc(base + p.a.start + k * p.a.kstep, p.a.lbo, p.a.sbo,
                                  p.a.layout, p.a.base_off);
      uint64_t bd = us::smem_desc(base + p.b.start + k * p.b.kstep, p.b.lbo, p.b.sbo,
                                  p.b.layout, p.b.base_off);
      us::umma_bf16(tmem, ad, bd, idesc, k > 0);
    }
    us::umma_commit(&bar_mma);
  }
  __syncwarp();
  us::mbar_wait(&bar_mma, 0);
  us::tc_fence_after();
  int row = warp * 32 + (threadIdx.x & 31);
  for (int c = 0; c < p.N; c += 32) {
    uint32_t v[32];
    us::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    us::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[row * p.N + c + j] = __uint_as_float(v[j]);
  }
  us::tc_fence_before();
  __syncthreads();
  if (warp == 1) us::tmem_dealloc<256>(tmem);
}


// T9: CTA pair (cta_group::2): M = 256 (128 A rows per CTA), N = 64 (32 B rows per CTA),
// K = 64, both CTAs' TMA loads complete on the leader's mbarrier, the leader issues the MMA,
// the commit is multicast to both CTAs, each reads its 128 rows x 64 columns of D.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128)
    pair_test(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
              float* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = us::cluster_ctarank();
  if (threadIdx.x == 0) {
    us::mbar_init(&bar_load, 1);
    us::mbar_init(&bar_mma, 1);
    us::fence_barrier_init();
  }
  if (warp == 1) us::tmem_alloc_pair<128>(&tmem_base);
  us::tc_fence_before();
  us::cluster_sync();
  us::tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t leader_bar = us::mapa_shared(us::smem_u32(&bar_load), 0);
  if (threadIdx.x == 0) {
    if (rank == 0) us::mbar_arrive_expect_tx(&bar_load, 2 * (16384 + 4096));
    us::tma_load_2d_pair(smem, &ma, leader_bar, 0, 128 * rank);
    us::tma_load_2d_pair(smem + 16384, &mb, leader_bar, 0, 32 * rank);
  }
  if (rank == 0 && threadIdx.x == 0) {
    us::mbar_wait(&bar_load, 0);
    us::tc_fence_after();
    const uint32_t base = us::smem_u32(smem);
    const uint32_t idesc = us::idesc_bf16(256, 64, 0, 0);
    for (int k = 0; k < 4; ++k) {
      uint64_t ad = us::smem_desc(base + k * 32, 16, 1024, 2);
      uint64_t bd = us::smem_desc(base + 16384 + k * 32, 16, 1024, 2);
      us::umma_bf16_pair(tmem, ad, bd, idesc, k > 0);
    }
    us::umma_commit_pair(&bar_mma, 0x3);
  }
  __syncwarp();
  us::mbar_wait(&bar_mma, 0);
  us::tc_fence_after();
  const int row = warp * 32 + (threadIdx.x & 31);
  for (int c = 0; c < 64; c += 32) {
    uint32_t v[32];
    us::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    us::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[(128 * rank + row) * 64 + c + j] = __uint_as_float(v[j]);
  }
  us::tc_fence_before();
  us::cluster_sync();
  if (warp == 1) us::tmem_dealloc_pair<128>(tmem);
}

// T10: CTA pair with an MN-major B split by N: B stored [K=64][N=64] (N contiguous), each
// CTA stages its 32 columns as 64-byte rows (SWIZZLE_64B) -- the layout of a halved dY tile.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128)
    pair_mn_test(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                 float* D, uint32_t lbo, uint32_t sbo) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = us::cluster_ctarank();
  if (threadIdx.x == 0) {
    us::mbar_init(&bar_load, 1);
    us::mbar_init(&bar_mma, 1);
    us::fence_barrier_init();
  }
  if (warp == 1) us::tmem_alloc_pair<128>(&tmem_base);
  us::tc_fence_before();
  us::cluster_sync();
  us::tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t leader_bar = us::mapa_shared(us::smem_u32(&bar_load), 0);
  if (threadIdx.x == 0) {
    if (rank == 0) us::mbar_arrive_expect_tx(&bar_load, 2 * (16384 + 4096));
    us::tma_load_2d_pair(smem, &ma, leader_bar, 0, 128 * rank);
    us::tma_load_2d_pair(smem + 16384, &mb, leader_bar, 32 * rank, 0);
  }
  if (rank == 0 && threadIdx.x == 0) {
    us::mbar_wait(&bar_load, 0);
    us::tc_fence_after();
    const uint32_t base = us::smem_u32(smem);
    const uint32_t idesc = us::idesc_bf16(256, 64, 0, 1);
    for (int k = 0; k < 4; ++k) {
      uint64_t ad = us::smem_desc(base + k * 32, 16, 1024, 2);
      uint64_t bd = us::smem_desc(base + 16384 + k * 16 * 64, lbo, sbo, 4);
      us::umma_bf16_pair(tmem, ad, bd, idesc, k > 0);
    }
    us::umma_commit_pair(&bar_mma, 0x3);
  }
  __syncwarp();
  us::mbar_wait(&bar_mma, 0);
  us::tc_fence_after();
  const int row = warp * 32 + (threadIdx.x & 31);
  for (int c = 0; c < 64; c += 32) {
    uint32_t v[32];
    us::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    us::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[(128 * rank + row) * 64 + c + j] = __uint_as_float(v[j]);
  }
  us::tc_fence_before();
  us::cluster_sync();
  if (warp == 1) us::tmem_dealloc_pair<128>(tmem);
}

// T8: 5-D halo box over a 4-channel NDHWC volume viewed as (W*4, H, D, N, 1), with
// negative start coordinates (zero fill), as the stem conv stages its input.
__global__ void halo_test(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, int bytes,
                          uint16_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    us::mbar_init(&bar, 1);
    us::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    us::mbar_arrive_expect_tx(&bar, bytes);
    us::tma_load_5d(smem, &m, &bar, c0, c1, c2, 0, 0);
  }
  us::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = ((uint16_t*)smem)[i];
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q));
  }
  return fn;
}

// 2-D bf16 map over [rows][cols] with box [box_rows][box_cols] and swizzle.
static CUtensorMap make_map(void* gptr, int rows, int cols, int box_rows, int box_cols,
                            int swz_bytes) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUtensorMapSwizzle sw = swz_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                        : swz_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                        : swz_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                          : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, gptr, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(2); }
  return m;
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

struct HostMat {
  int rows, cols; std::vector<float> f; std::vector<__nv_bfloat16> h; void* d = nullptr;
  HostMat(int r, int c, unsigned seed) : rows(r), cols(c), f(r * c), h(r * c) {
    srand(seed);
    for (int i = 0; i < r * c; ++i) {
      f[i] = bf(((rand() % 2001) - 1000) / 1000.0f);
      h[i] = __float2bfloat16(f[i]);
    }
    CK(cudaMalloc(&d, r * c * 2));
    CK(cudaMemcpy(d, h.data(), r * c * 2, cudaMemcpyHostToDevice));
  }
};

static int run(const char* name, const CUtensorMap& m0, const CUtensorMap& m1,
               const CUtensorMap& m2, Params p, const std::vector<float>& ref) {
  float* dD;
  CK(cudaMalloc(&dD, p.M * p.N * 4));
  CK(cudaMemset(dD, 0, p.M * p.N * 4));
  CK(cudaFuncSetAttribute(umma_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  umma_test<<<1, 128, 200 * 1024>>>(m0, m1, m2, p, dD);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> out(p.M * p.N);
  CK(cudaMemcpy(out.data(), dD, out.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  for (size_t i = 0; i < out.size(); ++i) maxerr = fmax(maxerr, fabs(out[i] - ref[i]));
  printf("%-48s max|err| = %.3e  %s\n", name, maxerr, maxerr < 1e-2 ? "PASS" : "FAIL");
  CK(cudaFree(dD));
  return maxerr < 1e-2 ? 0 : 1;
}

int main() {
  int fails = 0;
  // ---- T1: K-major SW128, A[128 x 64], B[N=64 x 64]
  {
    HostMat A(136, 64, 1), B(64, 64, 2);
    CUtensorMap ma = make_map(A.d, 136, 64, 136, 64, 128);
    CUtensorMap mb = make_map(B.d, 64, 64, 64, 64, 128);
    for (int shift = 0; shift < 8; ++shift) {
      Params p{};
      p.nboxes = 2; p.total_bytes = 136 * 128 + 64 * 128;
      p.boxes[0] = {0, 0, 0, 0, 136 * 128};
      p.boxes[1] = {1, 0, 0, 32768, 64 * 128};
      p.M = 128; p.N = 64; p.K = 64; p.a_mn = 0; p.b_mn = 0;
      p.a = {(uint32_t)(shift * 128), 16, 1024, 2, (uint32_t)shift, 32};
      p.b = {32768, 16, 1024, 2, 0, 32};
      std::vector<float> ref(128 * 64, 0.f);
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          float s = 0;
          for (int k = 0; k < 64; ++k) s += A.f[(m + shift) * 64 + k] * B.f[n * 64 + k];
          ref[m * 64 + n] = s;
        }
      char nm[96];
      snprintf(nm, sizeof nm, "K-major SW128, A row shift %d (base_off)", shift);
      run(nm, ma, mb, mb, p, ref);
      if (shift) {  // same shift without base offset: expected to differ if HW needs it
        p.a.base_off = 0;
        snprintf(nm, sizeof nm, "  (shift %d with base_off=0)", shift);
        run(nm, ma, mb, mb, p, ref);
      }
    }
  }
  // ---- T2: MN-major B (SW128): B stored [K=64][N=128], two 64-col chunks
  {
    HostMat A(128, 64, 3), B(64, 128, 4);
    CUtensorMap ma = make_map(A.d, 128, 64, 128, 64, 128);
    CUtensorMap mb = make_map(B.d, 64, 128, 64, 64, 128);
    Params p{};
    p.nboxes = 3; p.total_bytes = 128 * 128 + 2 * 64 * 128;
    p.boxes[0] = {0, 0, 0, 0, 128 * 128};
    p.boxes[1] = {1, 0, 0, 16384, 8192};
    p.boxes[2] = {1, 64, 0, 16384 + 8192, 8192};
    p.M = 128; p.N = 128; p.K = 64; p.a_mn = 0; p.b_mn = 1;
    p.a = {0, 16, 1024, 2, 0, 32};
    p.b = {16384, 8192, 1024, 2, 0, 16 * 128};
    std::vector<float> ref(128 * 128, 0.f);
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        float s = 0;
        for (int k = 0; k < 64; ++k) s += A.f[m * 64 + k] * B.f[k * 128 + n];
        ref[m * 128 + n] = s;
      }
    fails += run("K-major A SW128 x MN-major B SW128 (2 chunks)", ma, mb, mb, p, ref);
  }
  // ---- T3: MN-major A and B (wgrad shape): A^T stored [K=128][M=128], B stored [K=128][N=64]
  {
    HostMat A(128, 128, 5), B(128, 64, 6);
    CUtensorMap ma = make_map(A.d, 128, 128, 128, 64, 128);
    CUtensorMap mb = make_map(B.d, 128, 64, 128, 64, 128);
    Params p{};
    p.nboxes = 3; p.total_bytes = 2 * 128 * 128 + 128 * 128;
    p.boxes[0] = {0, 0, 0, 0, 16384};
    p.boxes[1] = {0, 64, 0, 16384, 16384};
    p.boxes[2] = {1, 0, 0, 32768, 16384};
    p.M = 128; p.N = 64; p.K = 128; p.a_mn = 1; p.b_mn = 1;
    p.a = {0, 16384, 1024, 2, 0, 16 * 128};
    p.b = {32768, 16384, 1024, 2, 0, 16 * 128};
    std::vector<float> ref(128 * 64, 0.f);
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        float s = 0;
        for (int k = 0; k < 128; ++k) s += A.f[k * 128 + m] * B.f[k * 64 + n];
        ref[m * 64 + n] = s;
      }
    fails += run("MN-major A x MN-major B, SW128", ma, mb, mb, p, ref);
  }
  // ---- T4: K-major SW32 (16 channels per row) and SW64 (32 per row)
  for (int rb = 32; rb <= 64; rb *= 2) {
    int kc = rb / 2;
    HostMat A(128, kc, 7), B(64, kc, 8);
    CUtensorMap ma = make_map(A.d, 128, kc, 128, kc, rb);
    CUtensorMap mb = make_map(B.d, 64, kc, 64, kc, rb);
    Params p{};
    p.nboxes = 2; p.total_bytes = 128 * rb + 64 * rb;
    p.boxes[0] = {0, 0, 0, 0, 128 * rb};
    p.boxes[1] = {1, 0, 0, 16384, 64 * rb};
    p.M = 128; p.N = 64; p.K = kc; p.a_mn = 0; p.b_mn = 0;
    p.a = {0, 16, (uint32_t)(8 * rb), us::swizzle_code(rb), 0, 32};
    p.b = {16384, 16, (uint32_t)(8 * rb), us::swizzle_code(rb), 0, 32};
    std::vector<float> ref(128 * 64, 0.f);
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        float s = 0;
        for (int k = 0; k < kc; ++k) s += A.f[m * kc + k] * B.f[n * kc + k];
        ref[m * 64 + n] = s;
      }
    char nm[64];
    snprintf(nm, sizeof nm, "K-major SW%d (%d ch/row)", rb, kc);
    fails += run(nm, ma, mb, mb, p, ref);
  }
  // ---- T5: MN-major SW32 chunks (16 wide): A^T stored [K=64][M=128] in 8 chunks of 16
  {
    HostMat A(64, 128, 9), B(64, 64, 10);
    CUtensorMap ma = make_map(A.d, 64, 128, 64, 16, 32);
    CUtensorMap mb = make_map(B.d, 64, 64, 64, 64, 128);
    Params p{};
    p.nboxes = 0;
    for (int c = 0; c < 8; ++c) p.boxes[p.nboxes++] = {0, c * 16, 0, c * 2048, 2048};
    p.boxes[p.nboxes++] = {1, 0, 0, 16384, 8192};
    p.total_bytes = 8 * 2048 + 8192;
    p.M = 128; p.N = 64; p.K = 64; p.a_mn = 1; p.b_mn = 1;
    p.a = {0, 2048, 256, 6, 0, 16 * 32};
    p.b = {16384, 8192, 1024, 2, 0, 16 * 128};
    std::vector<float> ref(128 * 64, 0.f);
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        float s = 0;
        for (int k = 0; k < 64; ++k) s += A.f[k * 128 + m] * B.f[k * 64 + n];
        ref[m * 64 + n] = s;
      }
    fails += run("MN-major A SW32 (8 chunks of 16) x MN-major B", ma, mb, mb, p, ref);
  }
  // ---- T6: K-major SW128 halo view: 8-row groups at a 10-row (1280 B) stride, shifted by s rows
  {
    HostMat A(176, 64, 11), B(64, 64, 12);
    CUtensorMap ma = make_map(A.d, 176, 64, 176, 64, 128);
    CUtensorMap mb = make_map(B.d, 64, 64, 64, 64, 128);
    for (int shift = 0; shift < 12; shift += 1) {
      Params p{};
      p.nboxes = 2; p.total_bytes = 176 * 128 + 64 * 128;
      p.boxes[0] = {0, 0, 0, 0, 176 * 128};
      p.boxes[1] = {1, 0, 0, 32768, 64 * 128};
      p.M = 128; p.N = 64; p.K = 64; p.a_mn = 0; p.b_mn = 0;
      p.a = {(uint32_t)(shift * 128), 16, 1280, 2, 0, 32};
      p.b = {32768, 16, 1024, 2, 0, 32};
      std::vector<float> ref(128 * 64, 0.f);
      for (int m = 0; m < 128; ++m) {
        int row = shift + (m / 8) * 10 + (m % 8);
        for (int n = 0; n < 64; ++n) {
          float s = 0;
          for (int k = 0; k < 64; ++k) s += A.f[row * 64 + k] * B.f[n * 64 + k];
          ref[m * 64 + n] = s;
        }
      }
      char nm[96];
      snprintf(nm, sizeof nm, "K-major SW128 halo view SBO=1280 shift %d", shift);
      fails += run(nm, ma, mb, mb, p, ref);
    }
  }
  // ---- T7: MN-major SW32/SW64 A with LBO/SBO both ways
  for (int rb = 32; rb <= 64; rb *= 2) {
    int w = rb / 2, nch = 128 / w, chunk = 64 * rb;
    HostMat A(64, 128, 13), B(64, 64, 14);
    CUtensorMap ma = make_map(A.d, 64, 128, 64, w, rb);
    CUtensorMap mb = make_map(B.d, 64, 64, 64, 64, 128);
    for (int variant = 0; variant < 2; ++variant) {
      Params p{};
      p.nboxes = 0;
      for (int c = 0; c < nch; ++c) p.boxes[p.nboxes++] = {0, c * w, 0, c * chunk, chunk};
      p.boxes[p.nboxes++] = {1, 0, 0, 16384, 8192};
      p.total_bytes = nch * chunk + 8192;
      p.M = 128; p.N = 64; p.K = 64; p.a_mn = 1; p.b_mn = 1;
      uint32_t lbo = variant ? (uint32_t)(8 * rb) : (uint32_t)chunk;
      uint32_t sbo = variant ? (uint32_t)chunk : (uint32_t)(8 * rb);
      p.a = {0, lbo, sbo, us::swizzle_code(rb), 0, (uint32_t)(16 * rb)};
      p.b = {16384, 8192, 1024, 2, 0, 16 * 128};
      std::vector<float> ref(128 * 64, 0.f);
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          float s = 0;
          for (int k = 0; k < 64; ++k) s += A.f[k * 128 + m] * B.f[k * 64 + n];
          ref[m * 64 + n] = s;
        }
      char nm[96];
      snprintf(nm, sizeof nm, "MN-major A SW%d chunks, %s", rb,
               variant ? "LBO=atom SBO=chunk" : "LBO=chunk SBO=atom");
      fails += run(nm, ma, mb, mb, p, ref);
    }
  }
  {  // ---- T9: CTA pair MMA
    HostMat A(256, 64, 11), B(64, 64, 12);
    CUtensorMap ma = make_map(A.d, 256, 64, 128, 64, 128);
    CUtensorMap mb = make_map(B.d, 64, 64, 32, 64, 128);
    float* dD;
    CK(cudaMalloc(&dD, 256 * 64 * 4));
    CK(cudaMemset(dD, 0, 256 * 64 * 4));
    CK(cudaFuncSetAttribute(pair_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024));
    pair_test<<<2, 128, 40 * 1024>>>(ma, mb, dD);
    cudaError_t le = cudaDeviceSynchronize();
    printf("T9 launch: %s\n", cudaGetErrorString(le));
    std::vector<float> out(256 * 64);
    double maxerr = 1e9;
    if (le == cudaSuccess) {
      CK(cudaMemcpy(out.data(), dD, out.size() * 4, cudaMemcpyDeviceToHost));
      maxerr = 0;
      for (int m = 0; m < 256; ++m)
        for (int n = 0; n < 64; ++n) {
          float s = 0;
          for (int k = 0; k < 64; ++k) s += A.f[m * 64 + k] * B.f[n * 64 + k];
          maxerr = fmax(maxerr, fabs(out[m * 64 + n] - s));
        }
    }
    printf("%-48s max|err| = %.3e  %s\n", "T9 CTA-pair M=256 N=64 (B split by N)", maxerr,
           maxerr < 1e-2 ? "PASS" : "FAIL");
    fails += maxerr < 1e-2 ? 0 : 1;
  }
  {  // ---- T10: CTA pair, MN-major B halves (SW64)
    HostMat A(256, 64, 13), B(64, 64, 14);   // B[k][n]
    CUtensorMap ma = make_map(A.d, 256, 64, 128, 64, 128);
    CUtensorMap mb = make_map(B.d, 64, 64, 64, 32, 64);
    uint32_t lbos[2] = {4096, 16}, sbos[2] = {512, 512};
    for (int v = 0; v < 2; ++v) {
      float* dD;
      CK(cudaMalloc(&dD, 256 * 64 * 4));
      CK(cudaMemset(dD, 0, 256 * 64 * 4));
      CK(cudaFuncSetAttribute(pair_mn_test, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              40 * 1024));
      pair_mn_test<<<2, 128, 40 * 1024>>>(ma, mb, dD, lbos[v], sbos[v]);
      cudaError_t le = cudaDeviceSynchronize();
      double maxerr = 1e9;
      if (le == cudaSuccess) {
        std::vector<float> out(256 * 64);
        CK(cudaMemcpy(out.data(), dD, out.size() * 4, cudaMemcpyDeviceToHost));
        maxerr = 0;
        for (int m = 0; m < 256; ++m)
          for (int n = 0; n < 64; ++n) {
            float s = 0;
            for (int k = 0; k < 64; ++k) s += A.f[m * 64 + k] * B.f[k * 64 + n];
            maxerr = fmax(maxerr, fabs(out[m * 64 + n] - s));
          }
      }
      char nm[96];
      snprintf(nm, sizeof nm, "T10 pair, MN-major B SW64 halves, LBO=%u SBO=%u", lbos[v], sbos[v]);
      printf("%-48s max|err| = %.3e  %s (%s)\n", nm, maxerr, maxerr < 1e-2 ? "PASS" : "FAIL",
             cudaGetErrorString(le));
      CK(cudaFree(dD));
    }
  }
  {  // ---- T8: stem halo box
    const int W = 32, H = 8, D = 4, bw = 32, bh = 4;
    std::vector<uint16_t> vol(W * H * D * 4);
    for (size_t i = 0; i < vol.size(); ++i) vol[i] = (uint16_t)(i % 60000 + 1);
    void* dv;
    CK(cudaMalloc(&dv, vol.size() * 2));
    CK(cudaMemcpy(dv, vol.data(), vol.size() * 2, cudaMemcpyHostToDevice));
    CUtensorMap m;
    cuuint64_t dims[5] = {(cuuint64_t)W * 4, (cuuint64_t)H, (cuuint64_t)D, 1, 1};
    cuuint64_t rowb = (cuuint64_t)W * 4 * 2;
    cuuint64_t strides[4] = {rowb, rowb * H, rowb * H * D, rowb * H * D};
    cuuint32_t box[5] = {(cuuint32_t)(bw + 2) * 4, (cuuint32_t)(bh + 2), 3, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, dv, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("T8 encode: %d\n", (int)r);
    const int HX = bw + 2, HY = bh + 2, bytes = HX * HY * 3 * 8;
    uint16_t* dout;
    CK(cudaMalloc(&dout, bytes));
    int bad = 0;
    int shifts[3] = {0, -8, -4};   // element offsets of the box start along W*4
    for (int si = 0; si < 3; ++si) {
      int z = 1, y0 = 4;
      CK(cudaFuncSetAttribute(halo_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
      halo_test<<<1, 128, 16384>>>(m, shifts[si], y0 - 1, z - 1, bytes, dout);
      cudaError_t le = cudaDeviceSynchronize();
      printf("T8 start element %d: %s\n", shifts[si], cudaGetErrorString(le));
      if (le != cudaSuccess) break;
      int x0 = shifts[si] / 4 + 1;
      std::vector<uint16_t> got(bytes / 2);
      CK(cudaMemcpy(got.data(), dout, bytes, cudaMemcpyDeviceToHost));
      for (int hz = 0; hz < 3; ++hz)
        for (int hy = 0; hy < HY; ++hy)
          for (int hx = 0; hx < HX; ++hx)
            for (int c = 0; c < 4; ++c) {
              int gz = z - 1 + hz, gy = y0 - 1 + hy, gx = x0 - 1 + hx;
              uint16_t want = (gz >= 0 && gz < D && gy >= 0 && gy < H && gx >= 0 && gx < W)
                                  ? vol[(((size_t)gz * H + gy) * W + gx) * 4 + c] : 0;
              if (got[((hz * HY + hy) * HX + hx) * 4 + c] != want) ++bad;
            }
    }
    printf("%-48s %d mismatches  %s\n", "T8 stem halo 5-D box (zero-filled border)", bad,
           bad ? "FAIL" : "PASS");
    fails += bad ? 1 : 0;
  }
  printf("selftest %s (%d failing cases)\n", fails ? "FAILED" : "PASSED", fails);
  return fails ? 1 : 0;
}
