// Launchers for every device kernel of libunetswap.  All launch on the given
// stream and return the launch status; shapes are NDHWC unless noted.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <vector>

namespace us {

// ---------------------------------------------------------------- toy (fp64)
// Reference semantics: pkg/src/swapsim/numeric.py:62-81 (affine), 208-222
// (forward kinds), 255-276 (grads).  Summations follow numpy's order so the
// results are bit-identical to the reference's.
struct PairwisePlan {          // numpy pairwise-summation tree for one length
  int64_t n = 0;
  int n_leaves = 0;
  int n_ops = 0;
  int64_t* d_leaves = nullptr;  // [2 * n_leaves] (lo, len)
  int* d_ops = nullptr;         // post-order: >=0 push leaf, -1 add
};
PairwisePlan make_pairwise_plan(int64_t n);
void free_pairwise_plan(PairwisePlan& p);

cudaError_t toy_affine(cudaStream_t s, const double* x, double* y, int64_t n_in, int64_t n_out,
                       double a, double b);
cudaError_t toy_affine_bwd(cudaStream_t s, const double* dy, double* dx, int64_t n_dx,
                           int64_t n_dy, double a);
cudaError_t toy_relu(cudaStream_t s, const double* x, double* y, int64_t n);
cudaError_t toy_relu_bwd(cudaStream_t s, const double* dy, const double* y, double* dx, int64_t n);
cudaError_t toy_center(cudaStream_t s, const double* x, double* y, const PairwisePlan& plan,
                       double* scratch /* >= n_leaves + 1 doubles */);
cudaError_t toy_pool(cudaStream_t s, const double* x, double* y, int64_t n_out, int64_t k);
cudaError_t toy_pool_bwd(cudaStream_t s, const double* dy, double* dx, int64_t n_dx, int64_t k);
cudaError_t toy_copy(cudaStream_t s, const double* src, double* dst, int64_t n);
cudaError_t toy_add(cudaStream_t s, const double* a, const double* b, double* dst, int64_t n,
                    double scale_b);
cudaError_t toy_sumsq(cudaStream_t s, const double* x, int64_t n, double* acc, int first,
                      const PairwisePlan& plan, double* scratch);

// ---------------------------------------------------------------- real ops
// dtype: 1 = fp32 storage, 2 = bf16 storage (activations and gradients).
// aug: device {flip mask (bit 0 x, 1 y, 2 z), permutation index} or null (no augmentation)
cudaError_t input_ncdhw(cudaStream_t s, int dtype, const float* src, void* dst, int N, int C,
                        int D, int H, int W, int Cdst, const int* aug);
cudaError_t labels_aug(cudaStream_t s, const uint8_t* src, uint8_t* dst, int N, int D, int H,
                       int W, const int* aug);
cudaError_t pad_channels(cudaStream_t s, int dtype, const void* src, void* dst, int64_t vox,
                         int C, int Cdst);
cudaError_t bn_stats_finalize(cudaStream_t s, const float* part, int nparts, int C, double count,
                              float* stat /* mean[C], rstd[C] */, double eps);
cudaError_t norm_act(cudaStream_t s, int dtype, const void* x, const float* stat,
                     const float* gamma, const float* beta, void* norm, void* act, int64_t vox,
                     int C);
cudaError_t pool_fwd(cudaStream_t s, int dtype, const void* x, void* y, int N, int D, int H, int W,
                     int C);
// relu != 0: x is a ReLU output and dx is the gradient of its input (fused ReLU backward)
// Fused BN-backward sums of a produced gradient (see ConvShape::bn_*): x = BN input laid
// out like the gradient, stat = mean[C], rstd[C]; part receives *rows rows (0 = unsupported)
struct BnSums {
  const void* x = nullptr;
  const float* stat = nullptr;
  float* part = nullptr;
  int* rows = nullptr;
};
cudaError_t pool_bwd(cudaStream_t s, int dtype, const void* x, const void* dy, const void* dcat,
                     int dcat_cs, int dcat_co, void* dx, int N, int D, int H, int W, int C,
                     int relu, const BnSums* bn = nullptr);
// y[v][co + c] = src[v][c] for c < C (y has Cy channels)
cudaError_t copy_channels(cudaStream_t s, int dtype, const void* src, void* y, int64_t vox, int C,
                          int Cy, int co);
// BN backward with its (sum dy, sum dy*xhat) partials already in part (npre rows, from
// the kernel that produced dy) -- npre = 0: compute them here (chan sums pass)
int bn_bwd_rows_max(int64_t vox, int C);
cudaError_t bn_bwd_sums(cudaStream_t s, int dtype, const void* x, const void* dy,
                        const float* stat, float* part, int64_t vox, int C, int* rows);
cudaError_t concat2(cudaStream_t s, int dtype, const void* a, const void* b, void* y, int64_t vox,
                    int Ca, int Cb);
cudaError_t relu_fwd(cudaStream_t s, int dtype, const void* x, void* y, int64_t n);
cudaError_t relu_bwd(cudaStream_t s, int dtype, const void* dy, const void* y, void* dx,
                     int64_t n);
// BN backward: part scratch >= 2 * C * bn_bwd_parts() floats.
int bn_bwd_parts(int64_t vox, int C);
cudaError_t bn_bwd(cudaStream_t s, int dtype, const void* x, const void* dy, const float* stat,
                   const float* gamma, float* ggamma, float* gbeta, void* dx, float* part,
                   int64_t vox, int C, int npre = 0);
// Soft-Dice loss over a 1x1x1 head + softmax.  dice holds per-(n,class) sums
// [N][3][ncls] (intersection, sum p, sum g) followed by the loss scalar.
int loss_parts(int64_t vox);
// BN apply + ReLU of the head's input layer fused with the head forward (bf16, C = 64):
// writes act and *rows rows of Dice partials into part; loss_finalize completes LOSS_FWD
int norm_act_loss_parts(int64_t vox);
cudaError_t norm_act_loss(cudaStream_t s, const void* x, const float* stat, const float* gamma,
                          const float* beta, void* norm, void* act, const uint8_t* labels,
                          const float* hw, const float* hb, float* part, int64_t vox, int C,
                          int ncls, int* rows);
cudaError_t loss_finalize(cudaStream_t s, const float* part, int nparts, int ncls, double eps,
                          double* dice, float* loss);
cudaError_t loss_fwd(cudaStream_t s, int dtype, const void* act, const uint8_t* labels,
                     const float* hw, const float* hb, float* part, double* dice, float* loss,
                     int N, int64_t vox, int C, int ncls, double eps);
cudaError_t loss_bwd(cudaStream_t s, int dtype, const void* act, const uint8_t* labels,
                     const float* hw, const float* hb, const double* dice, void* dact,
                     float* ghw, float* ghb, float* part, int N, int64_t vox, int C, int ncls,
                     double eps, int relu, const BnSums* bn = nullptr);
cudaError_t adam(cudaStream_t s, float* p, const float* g, float* m, float* v,
                 __nv_bfloat16* pb, int64_t n, float lr, float b1, float b2, float eps,
                 const float* corr /* device [1 - b1^t, 1 - b2^t] */);
cudaError_t cast_bf16(cudaStream_t s, const float* p, __nv_bfloat16* pb, int64_t n);
cudaError_t scale_f32(cudaStream_t s, float* g, int64_t n, float scale);

// ---------------------------------------------------------------- convolutions
// Weight layout for conv and transposed conv: [Cout][27][Cin] (tap = kd*9+kh*3+kw).
// Conv: k3 s1 p1.  ConvT: k3 s2 p1 output_padding 1 (low-res grid Dl,Hl,Wl -> 2x).
struct ConvShape {
  int N, D, H, W;       // grid of the conv input (conv) / low-res input (convT)
  int Cin, Cout;
  int x_cs, x_co;       // channel stride/offset of x   (NDHWC, elements)
  // dual-source input (tcgen05 conv fprop / wgrad): channels [x_split, Cin) come from x2
  // (its own NDHWC tensor of Cin - x_split channels); x then holds x_split == x_cs channels
  const void* x2 = nullptr;
  int x_split = 0;
  int dy_cs, dy_co;     // channel stride/offset of dy
  const void* relu_mask = nullptr;   // dgrad: zero dx where mask <= 0 (fused ReLU backward;
                                     // mask = the ReLU output, laid out like dx)
  // dgrad (tcgen05): fused BatchNorm-backward sums of dx -- bn_x = the BN input laid out
  // like dx, bn_stat = its mean[Cin], rstd[Cin]; bn_part receives *bn_rows rows of
  // (sum dx, sum dx * xhat) per channel (*bn_rows = 0: this path cannot, run chan sums)
  const void* bn_x = nullptr;
  const float* bn_stat = nullptr;
  float* bn_part = nullptr;
  int* bn_rows = nullptr;
};
// Direct (CUDA-core) kernels, fp32 accumulate; dtype of activations 1 or 2;
// weights are fp32 (dtype 1) or bf16 (dtype 2).
cudaError_t conv_fwd_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* x,
                            const void* w, void* y, float* part, int nparts);
cudaError_t conv_dgrad_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* dy,
                              const void* w, void* dx);
cudaError_t conv_wgrad_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* x,
                              const void* dy, float* gw);
cudaError_t convt_fwd_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* x,
                             const void* w, void* y);
cudaError_t convt_dgrad_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* dy,
                               const void* w, void* dx);
cudaError_t convt_wgrad_direct(cudaStream_t s, int dtype, const ConvShape& sh, const void* x,
                               const void* dy, float* gw);
int conv_stat_parts_direct(const ConvShape& sh);

// Tensor-core (tcgen05) implicit-GEMM kernels: bf16 activations and weights.
struct TcWorkspace { void* ptr; size_t bytes; };
int conv_stat_parts_tc(const ConvShape& sh);
size_t wgrad_tc_workspace(const ConvShape& sh, bool transposed);
// split_scratch: conv_split_scratch_bytes() of fp32 scratch for split-K small grids
size_t conv_split_scratch_bytes(const ConvShape& sh, bool dgrad);
cudaError_t conv_fwd_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                        const __nv_bfloat16* w, __nv_bfloat16* y, float* part,
                        float* split_scratch);
cudaError_t conv_dgrad_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* dy,
                          const __nv_bfloat16* w, __nv_bfloat16* dx, float* split_scratch);
cudaError_t conv_wgrad_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                          const __nv_bfloat16* dy, float* gw, float* work);
// scratch: convt_fwd_scratch_bytes() for the sub-pixel weight re-layout (or null)
size_t convt_fwd_scratch_bytes(const ConvShape& sh);
// y: the channel slice [y_co, y_co + Cout) of a y_cs-channel tensor
cudaError_t convt_fwd_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                         const __nv_bfloat16* w, __nv_bfloat16* y, void* scratch, int y_cs,
                         int y_co);
cudaError_t convt_dgrad_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* dy,
                           const __nv_bfloat16* w, __nv_bfloat16* dx);
cudaError_t convt_wgrad_tc(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                           const __nv_bfloat16* dy, float* gw, float* work);
bool tc_supported(const ConvShape& sh);
// Narrow-input layer (27*Cin <= 128): im2col + a single tcgen05 GEMM; the workspace
// starts with the BN partials (stem_stat_parts of them), then the im2col matrix.
bool stem_supported(const ConvShape& sh, bool wgrad);
int stem_stat_parts(const ConvShape& sh);
size_t stem_fwd_workspace(const ConvShape& sh);
size_t stem_wgrad_workspace(const ConvShape& sh);
cudaError_t conv_fwd_stem(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                          const __nv_bfloat16* w, __nv_bfloat16* y, void* work);
cudaError_t conv_wgrad_stem(cudaStream_t s, const ConvShape& sh, const __nv_bfloat16* x,
                            const __nv_bfloat16* dy, float* gw, void* work);

int num_sms();

}  // namespace us
