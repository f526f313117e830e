/*
 * libunetswap -- C ABI of the B200 swap engine and training-step kernels.
 *
 * The reference (arxiv 1812.07816 artifact, pkg/src/swapsim) has no FFI: its
 * train-step entry point is the Python function
 *     run_numeric(tg, plan=None, seed=0, inputs=None) -> (loss, {input: grad})
 *         (pkg/src/swapsim/numeric.py:153)
 * whose hot loop walks the serial order with swap_out/swap_in residency
 * moves (numeric.py:178-222, _Tape numeric.py:84-113) and whose timeline
 * contract is simulate()/stall_report() (sim.py:114, sim.py:308).  This
 * library is the device side that replaces that loop: the Python host layer
 * (paper_1812_07816_b200/lowering.py) compiles a TrainingGraph + RewritePlan
 * into a flat program of tensors and ops, and us_run() executes one step of
 * it on one GPU: kernels on a compute stream, swap-outs on a D2H copy stream,
 * prefetches on an H2D copy stream, all ordered with CUDA events and a
 * budget-capped device arena.
 *
 * Conventions: plain pointers and sizes only; every entry point returns an
 * int status (US_OK or a US_ERR_* code) and us_last_error() returns the
 * message of the last failure on the calling thread.  One context per GPU
 * per process, driven from one host thread.  The context owns the device
 * arena, persistent buffers and the pinned host pool; pointers passed in are
 * borrowed for the duration of the call.
 */
#ifndef UNETSWAP_H_
#define UNETSWAP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define US_ABI_VERSION 1

/* Status codes (mirrors the reference's exception families). */
#define US_OK 0
#define US_ERR_DOMAIN 1 /* use-after-swap / budget exhausted (GraphError family) */
#define US_ERR_USAGE 2  /* malformed program or arguments */
#define US_ERR_CUDA 3   /* CUDA runtime or driver failure */
#define US_ERR_NCCL 4   /* collective failure */

/* Tensor storage classes for us_tensor(). */
#define US_TENSOR_ARENA 0   /* step-scoped, allocated from the budgeted arena when first written */
#define US_TENSOR_PERSIST 1 /* lives for the context: parameters, optimizer state, inputs */

/* Element types. */
#define US_DT_F64 0
#define US_DT_F32 1
#define US_DT_BF16 2
#define US_DT_U8 3

/* Timeline channels (same numbering as the reference's trace tids, sim.py:30). */
#define US_CH_COMPUTE 0
#define US_CH_D2H 1
#define US_CH_H2D 2
#define US_CH_STALL 3 /* compute stream blocked on a copy; `node` = slot that waited */
#define US_CH_OP 4    /* one compute op's kernels (US_FLAG_OP_TIMES); `node` = op index */

/* Context flags (us_ctx_create / us_set_flags). */
#define US_FLAG_OP_TIMES 1u /* bracket every compute op with events (per-kernel timeline) */
#define US_FLAG_GRAPH 2u    /* capture the step as a CUDA graph (third run on) and replay it */
#define US_FLAG_NO_TIMELINE 4u /* no per-slot / per-copy timestamps (only the step's start and
                                  end): timed events stall ~40 us each while PCIe is saturated */
#define US_FLAG_POISON 8u      /* debug: fill every released arena region (freed, or swapped out
                                  once its D2H copy is done) with 0xFF bytes -- NaN in bf16 / fp32
                                  / fp64 -- so a read that bypasses the residency checks shows */

typedef struct us_ctx us_ctx;

typedef struct {
  int32_t node;    /* slot id (compute/stall) or io id (d2h/h2d) as given in the program */
  int32_t channel; /* US_CH_* */
  double start_s;  /* seconds since the step's start event */
  double end_s;
} us_event;

typedef struct {
  uint64_t arena_bytes;       /* budget of the step-scoped arena */
  uint64_t arena_peak_bytes;  /* high-water mark of the last step */
  uint64_t persistent_bytes;  /* parameters, optimizer state, inputs, scratch */
  uint64_t host_pool_bytes;   /* pinned host slots for swapped tensors */
  uint64_t d2h_bytes;         /* swap-out traffic of the last step */
  uint64_t h2d_bytes;         /* prefetch traffic of the last step */
  double step_s;              /* device time of the last step */
  double stall_s;             /* compute-stream time spent waiting on copies */
  int32_t kernels;            /* kernels launched by the last step */
  int32_t events;             /* timeline entries available from us_timeline */
  double host_enqueue_s;      /* host time us_run spent issuing the last enqueued step */
  int32_t host_numa_node;     /* NUMA node the pinned host pool is bound to (-1: unbound) */
  int32_t dp_nranks;          /* ranks of the data-parallel NCCL communicator (0: none) */
} us_stats;

const char* us_last_error(void);
int us_abi_version(void);

/* Context: one per GPU.  arena_bytes is the HBM budget for step tensors. */
int us_ctx_create(int32_t device, uint64_t arena_bytes, uint32_t flags, us_ctx** out);
int us_ctx_destroy(us_ctx* ctx);
int us_set_flags(us_ctx* ctx, uint32_t flags);

/* Program definition (replaces the reference's per-node Python dispatch,
 * numeric.py:178-222).  Tensor ids and slot ids are small non-negative ints
 * chosen by the caller; names are used in error messages only. */
int us_prog_reset(us_ctx* ctx);
int us_tensor(us_ctx* ctx, int32_t tid, uint64_t bytes, int32_t storage, int32_t dtype,
              const char* name);
/* Static arena placement (optional, all arena tensors or none): the tensor occupies
 * [offset, offset + bytes rounded to 1 KiB) of the arena whenever it is resident.  The
 * host planner guarantees that regions of tensors live at the same time in program
 * order do not overlap; the engine still waits on the pending copies of whatever was
 * released there before (lowering.Program.place). */
int us_tensor_place(us_ctx* ctx, int32_t tid, uint64_t offset);
int us_slot_name(us_ctx* ctx, int32_t slot, const char* name);
int us_op(us_ctx* ctx, int32_t opcode, const int32_t* tensors, int32_t n_tensors,
          const int64_t* iargs, int32_t n_iargs, const double* fargs, int32_t n_fargs);
int us_prog_finalize(us_ctx* ctx);
/* Patch one float argument of an already defined op (e.g. Adam's step count). */
int us_op_set_farg(us_ctx* ctx, int32_t op_index, int32_t k, double value);

/* Persistent tensor access (parameters, inputs, results). */
int us_upload(us_ctx* ctx, int32_t tid, const void* host, uint64_t bytes, uint64_t offset);
int us_download(us_ctx* ctx, int32_t tid, void* host, uint64_t bytes, uint64_t offset);
int us_tensor_ptr(us_ctx* ctx, int32_t tid, void** device_ptr);

/* Bytes of the workspace ("part") operand an op needs, from its iargs. */
int us_workspace_bytes(int32_t opcode, const int64_t* iargs, int32_t n_iargs, uint64_t* bytes);

/* Execution: enqueue one step; us_sync waits for it and collects the timeline.
 * Steps are pipelined: us_run returns once the step is enqueued and reads back
 * the previous step's timeline/stats while the GPU works. */
int us_run(us_ctx* ctx);
int us_sync(us_ctx* ctx);
/* Device-timed window on the compute stream: us_mark(0) opens, us_mark(1) closes. */
int us_mark(us_ctx* ctx, int32_t which);
int us_elapsed(us_ctx* ctx, double* seconds);
int us_stats_get(us_ctx* ctx, us_stats* out);
int us_timeline(us_ctx* ctx, us_event* out, int32_t capacity, int32_t* count);

/* Data-parallel gradient reduction: ncclUniqueId bytes from rank 0 (broadcast
 * by the caller, e.g. over torch.distributed); afterwards the program's
 * allreduce ops reduce over all ranks.  Returns US_ERR_NCCL if NCCL is absent. */
int us_dp_init(us_ctx* ctx, const void* nccl_unique_id, int32_t id_bytes, int32_t nranks,
               int32_t rank);
int us_dp_unique_id(void* out, int32_t capacity, int32_t* id_bytes);

#ifdef __cplusplus
}
#endif
#endif /* UNETSWAP_H_ */
