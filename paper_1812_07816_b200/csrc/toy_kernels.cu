// Toy-semantics kernels (fp64): the device restatement of the reference's
// executor arithmetic (pkg/src/swapsim/numeric.py).  They exist so the swap
// engine can be proven bit-exact against the reference's own run_numeric():
// every reduction reproduces numpy's summation order
//   * axis-0 sums of reshape(reps, n) are sequential over reps
//     (numeric.py:67 _affine_forward, numeric.py:80 _affine_backward),
//   * 1-D sums / means use numpy's pairwise summation (blocks of <=128 with
//     8 accumulators, split at n/2 rounded down to a multiple of 8)
//     (numeric.py:214 norm, numeric.py:217 pool, numeric.py:268 norm grad),
// and products/sums are issued with explicit round-to-nearest intrinsics so
// the compiler cannot contract them into FMAs numpy does not perform.
#include "kernels.h"
#include <vector>

namespace us {
namespace {

constexpr int kThreads = 256;

inline int blocks_for(int64_t n, int per = kThreads) {
  int64_t b = (n + per - 1) / per;
  return (int)(b < 1 ? 1 : (b > 65535 * 8 ? 65535 * 8 : b));
}

// numpy pairwise_sum leaf (n <= 128).
__device__ double pw_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = __dadd_rn(r0, a[i + 0]); r1 = __dadd_rn(r1, a[i + 1]);
    r2 = __dadd_rn(r2, a[i + 2]); r3 = __dadd_rn(r3, a[i + 3]);
    r4 = __dadd_rn(r4, a[i + 4]); r5 = __dadd_rn(r5, a[i + 5]);
    r6 = __dadd_rn(r6, a[i + 6]); r7 = __dadd_rn(r7, a[i + 7]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// Same leaf over squares (for the sum-of-squares loss).
__device__ double pw_leaf_sq(const double* a, int64_t n) {
  auto sq = [](double v) { return __dmul_rn(v, v); };
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, sq(a[i]));
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = sq(a[j]);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sq(a[i + j]));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, sq(a[i]));
  return res;
}

// Full pairwise sum for short rows (k <= a few thousand), recursive like numpy.
__device__ double pw_sum(const double* a, int64_t n) {
  if (n <= 128) return pw_leaf(a, n);
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_sum(a, n2), pw_sum(a + n2, n - n2));
}

__global__ void k_pw_leaves(const double* x, const int64_t* leaves, int n_leaves, double* out,
                            int squares) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_leaves) return;
  const double* a = x + leaves[2 * i];
  int64_t len = leaves[2 * i + 1];
  out[i] = squares ? pw_leaf_sq(a, len) : pw_leaf(a, len);
}

// Post-order combine of the leaf sums; writes the total to out[0].
__global__ void k_pw_combine(const double* leaf_sums, const int* ops, int n_ops, double* out) {
  double stack[64];
  int sp = 0;
  for (int i = 0; i < n_ops; ++i) {
    int op = ops[i];
    if (op >= 0) {
      stack[sp++] = leaf_sums[op];
    } else {
      double b = stack[--sp];
      double a = stack[--sp];
      stack[sp++] = __dadd_rn(a, b);
    }
  }
  out[0] = stack[0];
}

__global__ void k_center(const double* x, double* y, int64_t n, const double* total) {
  double mean = __ddiv_rn(total[0], (double)n);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dsub_rn(x[i], mean);
}

__global__ void k_sumsq_finish(const double* total, double* acc, int first) {
  acc[0] = first ? total[0] : __dadd_rn(acc[0], total[0]);
}

// y[j] = a * sum_r x[r*n_out + j] + b  (zero padded), or a * x[j % n_in] + b.
__global__ void k_affine(const double* x, double* y, int64_t n_in, int64_t n_out, double a,
                         double b) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_out;
       j += (int64_t)gridDim.x * blockDim.x) {
    double v;
    if (n_in >= n_out) {
      int64_t reps = (n_in + n_out - 1) / n_out;
      v = (j < n_in) ? x[j] : 0.0;
      for (int64_t r = 1; r < reps; ++r) {
        int64_t idx = r * n_out + j;
        v = __dadd_rn(v, idx < n_in ? x[idx] : 0.0);
      }
    } else {
      v = x[j % n_in];
    }
    y[j] = __dadd_rn(__dmul_rn(a, v), b);
  }
}

// dx[i] = a * dy[i % n_dy] (n_dx >= n_dy), else a * sum_r dy[r*n_dx + i] (zero padded).
__global__ void k_affine_bwd(const double* dy, double* dx, int64_t n_dx, int64_t n_dy, double a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_dx;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v;
    if (n_dx >= n_dy) {
      v = dy[i % n_dy];
    } else {
      int64_t reps = (n_dy + n_dx - 1) / n_dx;
      v = (i < n_dy) ? dy[i] : 0.0;
      for (int64_t r = 1; r < reps; ++r) {
        int64_t idx = r * n_dx + i;
        v = __dadd_rn(v, idx < n_dy ? dy[idx] : 0.0);
      }
    }
    dx[i] = __dmul_rn(a, v);
  }
}

__global__ void k_relu(const double* x, double* y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (x[i] >= 0.0 || x[i] != x[i]) ? x[i] : 0.0;   // np.maximum(x, 0.0)
}

// numpy: incoming * (reuse > 0.0) multiplies by 1.0 / 0.0 (sign of zero preserved).
__global__ void k_relu_bwd(const double* dy, const double* y, double* dx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dx[i] = __dmul_rn(dy[i], y[i] > 0.0 ? 1.0 : 0.0);
}

__global__ void k_pool(const double* x, double* y, int64_t n_out, int64_t k) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_out;
       j += (int64_t)gridDim.x * blockDim.x)
    y[j] = __ddiv_rn(pw_sum(x + j * k, k), (double)k);
}

__global__ void k_pool_bwd(const double* dy, double* dx, int64_t n_dx, int64_t k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_dx;
       i += (int64_t)gridDim.x * blockDim.x)
    dx[i] = __ddiv_rn(dy[i / k], (double)k);
}

__global__ void k_copy(const double* s, double* d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

__global__ void k_add(const double* a, const double* b, double* d, int64_t n, double sb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = __dadd_rn(a[i], sb == 1.0 ? b[i] : __dmul_rn(sb, b[i]));
}

void plan_rec(int64_t lo, int64_t n, std::vector<int64_t>& leaves, std::vector<int>& ops) {
  if (n <= 128) {
    ops.push_back((int)(leaves.size() / 2));
    leaves.push_back(lo);
    leaves.push_back(n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  plan_rec(lo, n2, leaves, ops);
  plan_rec(lo + n2, n - n2, leaves, ops);
  ops.push_back(-1);
}

}  // namespace

PairwisePlan make_pairwise_plan(int64_t n) {
  PairwisePlan p;
  std::vector<int64_t> leaves;
  std::vector<int> ops;
  plan_rec(0, n, leaves, ops);
  p.n = n;
  p.n_leaves = (int)(leaves.size() / 2);
  p.n_ops = (int)ops.size();
  cudaMalloc(&p.d_leaves, leaves.size() * sizeof(int64_t));
  cudaMalloc(&p.d_ops, ops.size() * sizeof(int));
  cudaMemcpy(p.d_leaves, leaves.data(), leaves.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  cudaMemcpy(p.d_ops, ops.data(), ops.size() * sizeof(int), cudaMemcpyHostToDevice);
  return p;
}

void free_pairwise_plan(PairwisePlan& p) {
  if (p.d_leaves) cudaFree(p.d_leaves);
  if (p.d_ops) cudaFree(p.d_ops);
  p = PairwisePlan{};
}

cudaError_t toy_affine(cudaStream_t s, const double* x, double* y, int64_t n_in, int64_t n_out,
                       double a, double b) {
  k_affine<<<blocks_for(n_out), kThreads, 0, s>>>(x, y, n_in, n_out, a, b);
  return cudaGetLastError();
}
cudaError_t toy_affine_bwd(cudaStream_t s, const double* dy, double* dx, int64_t n_dx,
                           int64_t n_dy, double a) {
  k_affine_bwd<<<blocks_for(n_dx), kThreads, 0, s>>>(dy, dx, n_dx, n_dy, a);
  return cudaGetLastError();
}
cudaError_t toy_relu(cudaStream_t s, const double* x, double* y, int64_t n) {
  k_relu<<<blocks_for(n), kThreads, 0, s>>>(x, y, n);
  return cudaGetLastError();
}
cudaError_t toy_relu_bwd(cudaStream_t s, const double* dy, const double* y, double* dx, int64_t n) {
  k_relu_bwd<<<blocks_for(n), kThreads, 0, s>>>(dy, y, dx, n);
  return cudaGetLastError();
}
cudaError_t toy_center(cudaStream_t s, const double* x, double* y, const PairwisePlan& plan,
                       double* scratch) {
  k_pw_leaves<<<blocks_for(plan.n_leaves, 128), 128, 0, s>>>(x, plan.d_leaves, plan.n_leaves,
                                                               scratch + 1, 0);
  k_pw_combine<<<1, 1, 0, s>>>(scratch + 1, plan.d_ops, plan.n_ops, scratch);
  k_center<<<blocks_for(plan.n), kThreads, 0, s>>>(x, y, plan.n, scratch);
  return cudaGetLastError();
}
cudaError_t toy_pool(cudaStream_t s, const double* x, double* y, int64_t n_out, int64_t k) {
  k_pool<<<blocks_for(n_out), kThreads, 0, s>>>(x, y, n_out, k);
  return cudaGetLastError();
}
cudaError_t toy_pool_bwd(cudaStream_t s, const double* dy, double* dx, int64_t n_dx, int64_t k) {
  k_pool_bwd<<<blocks_for(n_dx), kThreads, 0, s>>>(dy, dx, n_dx, k);
  return cudaGetLastError();
}
cudaError_t toy_copy(cudaStream_t s, const double* src, double* dst, int64_t n) {
  k_copy<<<blocks_for(n), kThreads, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}
cudaError_t toy_add(cudaStream_t s, const double* a, const double* b, double* dst, int64_t n,
                    double scale_b) {
  k_add<<<blocks_for(n), kThreads, 0, s>>>(a, b, dst, n, scale_b);
  return cudaGetLastError();
}
cudaError_t toy_sumsq(cudaStream_t s, const double* x, int64_t n, double* acc, int first,
                      const PairwisePlan& plan, double* scratch) {
  k_pw_leaves<<<blocks_for(plan.n_leaves, 128), 128, 0, s>>>(x, plan.d_leaves, plan.n_leaves,
                                                               scratch + 1, 1);
  k_pw_combine<<<1, 1, 0, s>>>(scratch + 1, plan.d_ops, plan.n_ops, scratch);
  k_sumsq_finish<<<1, 1, 0, s>>>(scratch, acc, first);
  return cudaGetLastError();
}

}  // namespace us
