// Program opcodes of libunetswap (parsed by paper_1812_07816_b200/_native.py).
// Tensor operand order and integer/float arguments are documented per op;
// "R" operands are read (residency-checked), "W" operands written (allocated
// on first write), "P" operands must be persistent buffers.
#pragma once

// ---- control / residency (reference numeric.py:178-188, _Tape numeric.py:84-113)
#define US_OP_SLOT_BEGIN 0     // i: slot, phase(0 fwd,1 bwd,2 other)
#define US_OP_SLOT_END 1       // i: slot
#define US_OP_SWAP_OUT 2       // R t ; i: io_id   D2H copy issued after the producer
#define US_OP_SWAP_RELEASE 3   // t ; device copy released (tensor becomes host-resident)
#define US_OP_SWAP_IN 4        // t src(host), W dst ; i: io_id, trigger_slot
#define US_OP_FREE 5           // t
#define US_OP_COPY_IN 6        // P src, W dst ; i: bytes
#define US_OP_CAPTURE 7        // R src, P dst ; i: bytes, dst_offset
#define US_OP_ZERO 8           // W t
#define US_OP_TOUCH 9          // R t ; residency read with no kernel (waits for a pending prefetch)

// ---- toy semantics in fp64 (reference numeric.py:6-13, 62-81, 189-276)
#define US_OP_TOY_AFFINE 10    // R x, W y ; i: n_in, n_out ; f: a, b
#define US_OP_TOY_AFFINE_BWD 11 // R dy, W dx ; i: n_dx, n_dy ; f: a
#define US_OP_TOY_RELU 12      // R x, W y ; i: n
#define US_OP_TOY_RELU_BWD 13  // R dy, R y, W dx ; i: n
#define US_OP_TOY_CENTER 14    // R x, W y ; i: n          y = x - mean(x) (numpy pairwise order)
#define US_OP_TOY_POOL 15      // R x, W y ; i: n_out, k   block mean
#define US_OP_TOY_POOL_BWD 16  // R dy, W dx ; i: n_dx, k
#define US_OP_TOY_COPY 17      // R src, W dst ; i: n, src_off, dst_off (dst written, maybe partially)
#define US_OP_TOY_ADD 18       // R a, R b, W dst ; i: n ; f: scale_b     dst = a + scale_b*b
#define US_OP_TOY_SUMSQ 19     // R x, P acc ; i: n, first, acc_index

// ---- real U-Net ops (bf16 or fp32 storage, NDHWC activations)
#define US_OP_INPUT_NCDHW 20   // P src(f32 NCDHW), W dst ; i: N,C,D,H,W,Cdst [; f: flips, perm]
                               //   with fargs: per-step flip/permute augmentation (dynamic)
#define US_OP_PAD_CH 21        // R src, W dst ; i: vox, C, Cdst
#define US_OP_CONV_FWD 22      // R x, P w, W y, W part[, O x2] ; i: N,D,H,W,Cin,Cout,w_off,algo,x_cs,x_co
                               //   x2: dual-source input -- channels [x_cs, Cin) read from x2
                               //   (a concat never materialised; tcgen05 only)
#define US_OP_BN_STATS 23      // R part, P stat ; i: nparts, C, count, stat_off ; f: eps
#define US_OP_NORM_ACT 24      // R x, P stat, P params, w norm, w act[, O labels, w part] ; i: vox,C,stat_off,gamma_off,beta_off[,ncls,hw_off,hb_off]
                               //   labels/part: fused head forward (bf16, C = 64) -- Dice partials
                               //   for a following LOSS_FWD with pre = 1
                               //   (w = optional output, -1 skips it: recompute clones)
#define US_OP_POOL_FWD 25      // R x, W y ; i: N,D,H,W,C
#define US_OP_CONCAT 26        // R a, O b, W y ; i: vox, Ca, Cb[, b_in_place] (1: the producer of b
                               //   wrote y[:, Ca:] itself, b = -1; only a is copied)
#define US_OP_CONVT_FWD 27     // R x, P w, W y ; i: N,Dl,Hl,Wl,Cin,Cout,w_off,algo[,y_cs,y_co]
                               //   (tcgen05: y written as the channel slice [y_co, y_co+Cout)
                               //   of a y_cs-channel tensor, e.g. straight into a concat)
#define US_OP_LOSS_FWD 28      // R act, P labels, P params, W part, P dice, P loss ; i: N,vox,C,ncls,hw_off,hb_off[,pre] ; f: eps
#define US_OP_LOSS_BWD 29      // R act, P labels, P params, P dice, W dact, P grads, W part[, BN] ; i: N,vox,C,ncls,hw_off,hb_off,ghw_off,ghb_off[,relu[,stat_off]] ; f: eps
#define US_OP_RELU_BWD 30      // R dy, R y, W dx ; i: n
#define US_OP_BN_BWD 31        // R x, R dy, P stat, P params, P grads, W dx, W part ; i: vox,C,stat_off,gamma_off,ggamma_off,gbeta_off[,pre]
                               //   pre = 1: part already holds dy's (sum dy, sum dy*xhat) rows, written
                               //   by the op that produced dy through its optional BN operands
#define US_OP_CONV_DGRAD 32    // R dy, P w, W dx, O mask|-1[, BN] ; i: N,D,H,W,Cin,Cout,w_off,algo,dy_cs,dy_co[,stat_off]
                               //   mask: ReLU output laid out like dx -> dx = dgrad * (mask > 0)
#define US_OP_CONV_WGRAD 33    // R x, R dy, P grads, W part[, O x2] ; i: N,D,H,W,Cin,Cout,g_off,algo,dy_cs,dy_co[,x_cs]
                               //   x2: dual-source input, x holds x_cs channels
#define US_OP_CONVT_DGRAD 34   // R dy, P w, W dx, O mask|-1[, BN] ; i: N,Dl,Hl,Wl,Cin,Cout,w_off,algo,dy_cs,dy_co[,stat_off]
#define US_OP_CONVT_WGRAD 35   // R x, R dy, P grads, W part ; i: N,Dl,Hl,Wl,Cin,Cout,g_off,algo,dy_cs,dy_co
#define US_OP_POOL_BWD 36      // R x, R dy, R dcat|-1, W dx[, BN] ; i: N,D,H,W,C,dcat_cs,dcat_co[,relu[,stat_off]]
                               //   relu: x is a ReLU output, dx = grad of its input
// [, BN] = three optional trailing operands (O bn_x, O stat, w part): the BN input laid out
// like the produced gradient, the statistics buffer (mean at stat_off, rstd at +C) and a
// partials tensor receiving (sum g, sum g*xhat) rows for the following BN_BWD (pre = 1).
// Trailing optional operands may be omitted from us_op (the engine pads them with -1).
#define US_OP_ADAM 37          // P p, P g, P m, P v, P pb ; i: n, write_bf16[, offset, bucket] ; f: lr,b1,b2,eps,step
                               //   bucket=1: update [offset, offset+n) on the comm stream
#define US_OP_ALLREDUCE 38     // P g ; i: offset, count[, bucket] ; f: scale   bucket=1: on the
                               //   comm stream after the compute stream wrote it; ADAM waits
#define US_OP_CAST_W 39        // P p, P pb ; i: n            fp32 master -> bf16 kernel copy
#define US_OP_RELU_FWD 40      // R x, W y ; i: n             recompute clone of an activation
#define US_OP_LABELS_AUG 41    // P labels, P labels_aug (u8) ; i: N,D,H,W ; f: flips, perm (dynamic)

#define US_OP_COUNT 42

// conv algorithms
#define US_ALGO_DIRECT 0       // CUDA-core direct convolution (any channel count, fp32 accumulate)
#define US_ALGO_TCGEN05 1      // implicit GEMM on tcgen05 tensor cores (bf16, channels % 16 == 0)
#define US_ALGO_IM2COL 2       // narrow-input conv (27*Cin <= 128): im2col + one tcgen05 GEMM (bf16)
