// libunetswap runtime: context, budgeted device arena, pinned host pool,
// program executor and swap engine.
//
// The executor is the device-side replacement of the reference's train-step
// loop (pkg/src/swapsim/numeric.py:153-229): it walks the program produced by
// paper_1812_07816_b200/lowering.py, enforcing the same residency discipline
// as _Tape (numeric.py:84-113 -- a read of a swapped-out or freed tensor is a
// use-after-swap error), and maps the simulator's three channels
// (sim.py:1-17) onto three CUDA streams:
//   compute : kernels in serial-slot order
//   d2h     : swap-outs, FIFO in producer order, issued when the producer ends
//   h2d     : prefetches, FIFO in trigger order, each waiting on its own D2H
// Cross-stream ordering uses CUDA events only; memory handed back by a
// swap-out or free carries the events that must complete before the bytes may
// be reused, so the allocator never makes the host wait.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/unetswap.h"
#include "kernels.h"
#include "opcodes.h"

struct us_ctx;

namespace {

thread_local std::string g_last_error;

struct UsError {
  int code;
  std::string msg;
};

std::string fmt(const char* f, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}

#define US_FAIL(code, ...) throw UsError{code, fmt(__VA_ARGS__)}
#define CUDA_OK(x)                                                                        \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      throw UsError{US_ERR_CUDA, fmt("%s failed: %s", #x, cudaGetErrorString(e_))};       \
  } while (0)

// S_COMM: bucketed gradient all-reduce (NCCL), overlapped with the rest of the backward.
enum Stream { S_COMP = 0, S_D2H = 1, S_H2D = 2, S_COMM = 3, S_COUNT = 4 };

struct Mark {              // an event recorded on a stream, with a global sequence number
  cudaEvent_t ev = nullptr;   // dependency edge (cudaStreamWaitEvent)
  uint64_t seq = 0;
  cudaEvent_t ext = nullptr;  // observable from the host (timing / sync): == ev unless the
                              // step is being captured as a graph, where it is a separate
                              // external event-record node
};

struct Block {
  uint64_t size;
  bool free;
  Mark pend[S_COUNT];      // last use per stream that must finish before reuse
};

struct Tensor {
  bool defined = false;
  std::string name;
  uint64_t bytes = 0;
  int storage = US_TENSOR_ARENA;
  int dtype = US_DT_F32;
  void* pptr = nullptr;    // persistent storage
  // per-step state
  int state = 0;           // 0 unallocated, 1 device, 2 host, 3 freed
  uint64_t off = 0;
  Mark d2h_done;
  int d2h_stream = 1;
  Mark h2d_done;
  bool pending_h2d = false;
  int64_t host_off = -1;
  int64_t fixed_off = -1;  // static arena placement (us_tensor_place), -1 = best fit
};

struct Op {
  int code;
  std::vector<int> t;
  std::vector<int64_t> i;
  std::vector<double> f;
};

struct Rec {
  int node, channel;
  cudaEvent_t a, b;
};

// NCCL entry points resolved at runtime (torch ships libnccl.so.2).
struct Nccl {
  void* lib = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  // ncclUniqueId is a 128-byte struct passed BY VALUE (not a pointer)
  struct UniqueId {
    char internal[128];
  };
  int (*commInitRank)(void**, int, UniqueId, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*errStr)(int) = nullptr;
  bool load() {
    if (lib) return true;
    const char* env = getenv("US_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n) continue;
      lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (lib) break;
    }
    if (!lib) return false;
    getUniqueId = (int (*)(void*))dlsym(lib, "ncclGetUniqueId");
    commInitRank = (int (*)(void**, int, UniqueId, int))dlsym(lib, "ncclCommInitRank");
    allReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
        lib, "ncclAllReduce");
    commDestroy = (int (*)(void*))dlsym(lib, "ncclCommDestroy");
    errStr = (const char* (*)(int))dlsym(lib, "ncclGetErrorString");
    return getUniqueId && commInitRank && allReduce && commDestroy;
  }
};
Nccl g_nccl;

const char* state_name(int s) {
  return s == 0 ? "not yet produced" : s == 2 ? "host-resident" : s == 3 ? "freed" : "device";
}

}  // namespace

struct us_ctx {
  int device = 0;
  cudaStream_t st[S_COUNT] = {};
  // arena
  char* arena = nullptr;
  uint64_t arena_cap = 0, in_use = 0, peak = 0;
  std::map<uint64_t, Block> blocks;
  bool fixed_layout = false;   // every arena tensor carries a planned offset
  // host pool
  char* host_pool = nullptr;
  uint64_t host_map_bytes = 0;   // mmap length of host_pool (NUMA-bound, page-locked)
  int host_numa_node = -1;       // NUMA node the pool's pages were bound to (-1: default)
  uint64_t host_cap = 0;
  // program
  std::vector<Tensor> tensors;
  std::vector<Op> ops;
  std::unordered_map<int, std::string> slot_names;
  bool finalized = false;
  uint64_t persistent_bytes = 0;
  std::map<int64_t, us::PairwisePlan> pw_plans;
  double* toy_scratch = nullptr;
  size_t toy_scratch_elems = 0;
  // events (two pools so step k's timeline survives enqueueing step k+1)
  std::vector<cudaEvent_t> pool[2];    // dependency events (no timing), per parity
  std::vector<cudaEvent_t> tpool[2];   // timed events, per parity
  size_t tpool_next = 0;
  size_t pool_next = 0;
  int parity = 0;
  uint32_t flags = 0;   // US_FLAG_*
  double host_enqueue_s = 0;
  double host_op_s[US_OP_COUNT] = {};   // US_HOST_PROFILE: host time per opcode
  long host_op_n[US_OP_COUNT] = {};
  uint64_t seq = 0;
  std::vector<Rec> recs;
  struct StepRec {
    std::vector<Rec> recs;
    cudaEvent_t start = nullptr, end = nullptr;
    uint64_t d2h = 0, h2d = 0, peak = 0;
    int kernels = 0;
    bool valid = false;
  } inflight;
  struct Done {
    double step_s = 0, stall_s = 0;
    uint64_t d2h = 0, h2d = 0, peak = 0;
    int kernels = 0;
  } done;
  // CUDA graph of the whole step (US_FLAG_GRAPH), one per event-pool parity: captured
  // on the third run, replayed afterwards with a single cudaGraphLaunch.  The host
  // logic (allocation, residency checks, waits) runs once at capture time; per-step
  // values (Adam's bias correction) reach the graph through pinned host scalars that
  // a captured memcpy node reads at replay time.
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    StepRec rec;
  } graph[2];
  int runs = 0;
  cudaEvent_t step_start = nullptr, step_end = nullptr;
  Mark comm_done;   // last gradient-bucket all-reduce of the step (comm stream)
  float* split_scratch = nullptr;   // split-K partial tiles of small-grid convs
  size_t split_cap = 0;
  bool capturing = false;
  // per-step values of "dynamic" ops, two 32-bit words each at dyn_slot[op]: Adam's
  // bias corrections (float) and the augmentation's flip mask / permutation (int)
  uint32_t* dyn_host[2] = {nullptr, nullptr};   // pinned, per parity
  uint32_t* dyn_dev = nullptr;
  int n_dyn = 0;
  std::vector<int> dyn_slot;                    // op index -> slot or -1
  static bool dynamic_op(const Op& op) {
    return op.code == US_OP_ADAM || op.code == US_OP_LABELS_AUG ||
           (op.code == US_OP_INPUT_NCDHW && op.f.size() >= 2);
  }
  void drop_graphs() {
    for (auto& g : graph) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
    runs = 0;
  }
  void set_dyn_scalars(int par) {
    for (size_t j = 0; j < ops.size(); ++j) {
      const int k = dyn_slot.empty() ? -1 : dyn_slot[j];
      if (k < 0) continue;
      const Op& op = ops[j];
      uint32_t* w = dyn_host[par] + 2 * k;
      if (op.code == US_OP_ADAM) {
        const float step = (float)op.f[4];
        const float c[2] = {1.f - powf((float)op.f[1], step), 1.f - powf((float)op.f[2], step)};
        std::memcpy(w, c, sizeof c);
      } else {
        w[0] = (uint32_t)op.f[0];   // flip mask
        w[1] = (uint32_t)op.f[1];   // permutation index
      }
    }
  }
  // Device copy of op j's per-step words, refreshed on stream s by a (capturable) memcpy
  // from this step's pinned host slots.
  const void* dyn_words(int j, cudaStream_t s) {
    const int k = dyn_slot[j];
    CUDA_OK(cudaMemcpyAsync(dyn_dev + 2 * k, dyn_host[parity] + 2 * k, 2 * sizeof(uint32_t),
                            cudaMemcpyHostToDevice, s));
    return dyn_dev + 2 * k;
  }
  cudaEvent_t window_start = nullptr, window_end = nullptr;
  std::unordered_map<int, Mark> slot_end;
  std::unordered_map<int, int> bn_rows;   // fused BN-backward partials: tensor -> rows written
  int cur_slot = -1;
  // per-step counters of the step being enqueued
  uint64_t d2h_bytes = 0, h2d_bytes = 0, step_peak = 0;
  int kernels = 0;
  std::vector<us_event> timeline;   // of the last collected step
  // data parallel
  void* nccl_comm = nullptr;
  int nranks = 1, rank = 0;

  // ------------------------------------------------------------ events
  // Two kinds of events.  Dependency events (cross-stream waits, allocator frontier)
  // are created with cudaEventDisableTiming: recording one is a cheap on-device
  // semaphore.  A timed event writes a timestamp over the host interface, and while a
  // swap copy saturates PCIe each one stalls the stream by ~40 us (tools/
  // event_interference.py) -- so timed events are recorded only where the timeline
  // needs them and only with the timeline enabled (US_FLAG_NO_TIMELINE turns them off,
  // except the step's start/end).  During graph capture a timed event is an external
  // event-record node, so it stays observable from the host.
  cudaEvent_t take(std::vector<cudaEvent_t>& p, size_t& next, unsigned evflags) {
    if (next == p.size()) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreateWithFlags(&e, evflags));
      p.push_back(e);
    }
    return p[next++];
  }
  bool timeline_on() const { return (flags & US_FLAG_NO_TIMELINE) == 0; }
  Mark record(int s, bool timed = false, bool force = false) {
    Mark m{take(pool[parity], pool_next, cudaEventDisableTiming), ++seq, nullptr};
    if (timed && (force || timeline_on())) {
      m.ext = take(tpool[parity], tpool_next, cudaEventDefault);
      if (capturing)
        CUDA_OK(cudaEventRecordWithFlags(m.ext, st[s], cudaEventRecordExternal));
      else
        CUDA_OK(cudaEventRecord(m.ext, st[s]));
    }
    CUDA_OK(cudaEventRecord(m.ev, st[s]));
    issued[s].push_back(m);
    return m;
  }
  void add_rec(int node, int channel, const Mark& a, const Mark& b) {
    if (a.ext && b.ext) recs.push_back(Rec{node, channel, a.ext, b.ext});
  }

  // Completion frontier per stream: marks complete in issue order on their stream,
  // so each one is polled until it completes and never again (the allocator asks
  // "is this block's last user done?" without one cudaEventQuery per free block).
  std::deque<Mark> issued[S_COUNT];
  uint64_t done_seq[S_COUNT] = {};
  void poll_done() {
    if (capturing) return;   // no event queries inside a stream capture
    for (int k = 0; k < S_COUNT; ++k) {
      auto& q = issued[k];
      while (!q.empty()) {
        cudaError_t r = cudaEventQuery(q.front().ev);
        if (r != cudaSuccess) {
          (void)cudaGetLastError();   // cudaErrorNotReady is a status, not a failure
          break;
        }
        done_seq[k] = q.front().seq;
        q.pop_front();
      }
    }
  }
  void forget_marks() {   // step boundary: every earlier mark is ordered before new work
    for (int k = 0; k < S_COUNT; ++k) {
      issued[k].clear();
      done_seq[k] = seq;
    }
  }

  // ------------------------------------------------------------ arena
  void arena_reset() {
    blocks.clear();
    blocks[0] = Block{arena_cap, true, {}};
    in_use = 0;
    step_peak = 0;
  }

  // Best-fit allocation for stream s; `waits` receives the events s must wait on.
  // Static placement: the planner (lowering.Program.place) gave every arena tensor an
  // offset whose region is free at this point of the program.  The region may span
  // several free blocks released by different tensors; the stream waits on exactly
  // their pending events (free blocks are not merged in this mode, so a region that was
  // never touched by a pending swap-out does not wait for one).
  uint64_t arena_alloc_fixed(uint64_t off, uint64_t bytes, int s, std::vector<Mark>& waits,
                             const Tensor& t) {
    const uint64_t end = off + bytes;
    if (end > arena_cap)
      US_FAIL(US_ERR_USAGE, "placement of '%s' [%llu, %llu) exceeds the %llu-byte arena",
              t.name.c_str(), (unsigned long long)off, (unsigned long long)end,
              (unsigned long long)arena_cap);
    // the blocks partition [0, arena_cap); key 0 always exists
    auto it = std::prev(blocks.upper_bound(off));
    std::vector<std::map<uint64_t, Block>::iterator> cover;
    uint64_t pos = it->first;
    for (auto jt = it; pos < end; ++jt) {
      if (jt == blocks.end() || jt->first != pos)
        US_FAIL(US_ERR_USAGE, "arena block map corrupt at %llu", (unsigned long long)pos);
      if (!jt->second.free)
        US_FAIL(US_ERR_USAGE, "placement of '%s' at %llu overlaps a live tensor",
                t.name.c_str(), (unsigned long long)off);
      cover.push_back(jt);
      pos += jt->second.size;
    }
    for (auto c : cover)
      for (int k = 0; k < S_COUNT; ++k)
        if (c->second.pend[k].ev && k != s) waits.push_back(c->second.pend[k]);
    const uint64_t first_off = cover.front()->first, last_off = cover.back()->first;
    const Block first = cover.front()->second, last = cover.back()->second;
    for (auto c : cover) blocks.erase(c);
    if (first_off < off) {
      Block lead = first;
      lead.size = off - first_off;
      blocks[first_off] = lead;
    }
    if (last_off + last.size > end) {
      Block tail = last;
      tail.size = last_off + last.size - end;
      blocks[end] = tail;
    }
    blocks[off] = Block{bytes, false, {}};
    in_use += bytes;
    if (in_use > step_peak) step_peak = in_use;
    return off;
  }

  uint64_t arena_alloc(uint64_t bytes, int s, std::vector<Mark>& waits, const Tensor& t) {
    bytes = (bytes + 1023) & ~uint64_t(1023);
    if (bytes == 0) bytes = 1024;
    if (t.fixed_off >= 0) return arena_alloc_fixed((uint64_t)t.fixed_off, bytes, s, waits, t);
    // Best fit among free blocks whose previous users on other streams are done;
    // only if none fits, reuse a block the stream has to wait for (a real
    // memory-pressure stall, e.g. under a capped budget).
    poll_done();
    // wait class of a free block for stream s: 0 = its other-stream users are done,
    // 1 = it waits only for compute-stream work, 2 = it waits for a copy (a D2H of a
    // swapped tensor can be tens of milliseconds away).  Best fit in the lowest class.
    auto wait_class = [&](Block& b) {
      int cls = 0;
      for (int k = 0; k < S_COUNT; ++k) {
        if (!b.pend[k].ev || k == s) continue;
        if (b.pend[k].seq <= done_seq[k]) {
          b.pend[k] = Mark{};
          continue;
        }
        cls = std::max(cls, k == S_COMP || k == S_COMM ? 1 : 2);
      }
      return cls;
    };
    auto best = blocks.end();
    int best_cls = 3;
    for (auto it = blocks.begin(); it != blocks.end(); ++it) {
      Block& b = it->second;
      if (!b.free || b.size < bytes) continue;
      const int cls = wait_class(b);
      if (cls < best_cls || (cls == best_cls && b.size < best->second.size)) {
        best = it;
        best_cls = cls;
      }
    }
    if (best == blocks.end()) {
      uint64_t largest = 0;
      for (auto& kv : blocks)
        if (kv.second.free && kv.second.size > largest) largest = kv.second.size;
      // the reference's two budget failures (sim.py:33-43): a tensor larger than the whole
      // budget can never fit (infeasible); otherwise every byte is held by tensors that
      // are only released after this allocation in program order (or the free bytes are
      // fragmented), so nothing in flight can ever make room (deadlock)
      if (bytes > arena_cap)
        US_FAIL(US_ERR_DOMAIN,
                "budget exhausted: infeasible: tensor '%s' needs %llu bytes, which can never "
                "fit in the %llu-byte budget", t.name.c_str(), (unsigned long long)bytes,
                (unsigned long long)arena_cap);
      US_FAIL(US_ERR_DOMAIN,
              "budget exhausted: deadlock: tensor '%s' needs %llu bytes; arena %llu, in use "
              "%llu, largest free block %llu, nothing in flight frees more",
              t.name.c_str(), (unsigned long long)bytes, (unsigned long long)arena_cap,
              (unsigned long long)in_use, (unsigned long long)largest);
    }
    uint64_t off = best->first;
    Block b = best->second;
    if (b.size > bytes) {
      Block rest = b;
      rest.size = b.size - bytes;
      blocks[off + bytes] = rest;
    }
    best->second = Block{bytes, false, {}};
    for (int k = 0; k < S_COUNT; ++k)
      if (b.pend[k].ev && k != s) waits.push_back(b.pend[k]);
    in_use += bytes;
    if (in_use > step_peak) step_peak = in_use;
    return off;
  }

  void arena_release(uint64_t off, const Mark* ev) {
    auto it = blocks.find(off);
    if (it == blocks.end() || it->second.free) US_FAIL(US_ERR_USAGE, "double free in arena");
    in_use -= it->second.size;
    it->second.free = true;
    for (int k = 0; k < S_COUNT; ++k) it->second.pend[k] = ev[k];
    if (fixed_layout) return;   // keep per-tensor pending events exact (arena_alloc_fixed)
    auto merge = [](Block& into, const Block& from) {
      into.size += from.size;
      for (int k = 0; k < S_COUNT; ++k)
        if (from.pend[k].seq > into.pend[k].seq) into.pend[k] = from.pend[k];
    };
    auto nx = std::next(it);
    if (nx != blocks.end() && nx->second.free) {
      merge(it->second, nx->second);
      blocks.erase(nx);
    }
    if (it != blocks.begin()) {
      auto pv = std::prev(it);
      if (pv->second.free) {
        merge(pv->second, it->second);
        blocks.erase(it);
      }
    }
  }

  // ------------------------------------------------------------ tensors
  Tensor& T(int tid) {
    if (tid < 0 || tid >= (int)tensors.size() || !tensors[tid].defined)
      US_FAIL(US_ERR_USAGE, "op references undefined tensor %d", tid);
    return tensors[tid];
  }
  void* ptr(int tid) {
    Tensor& t = T(tid);
    if (t.storage == US_TENSOR_PERSIST) return t.pptr;
    if (t.state != 1) US_FAIL(US_ERR_USAGE, "tensor '%s' has no device buffer", t.name.c_str());
    return arena + t.off;
  }
  void check_read(int tid, int op_index, std::vector<Mark>& waits) {
    Tensor& t = T(tid);
    if (t.storage == US_TENSOR_PERSIST) return;
    if (t.state != 1) {
      std::string slot = slot_names.count(cur_slot) ? slot_names[cur_slot] : fmt("op%d", op_index);
      US_FAIL(US_ERR_DOMAIN, "use-after-swap: node '%s' read tensor '%s' which is %s, "
              "not device-resident", slot.c_str(), t.name.c_str(), state_name(t.state));
    }
    if (t.pending_h2d) {
      waits.push_back(t.h2d_done);
      t.pending_h2d = false;
    }
  }
  void ensure_written(int tid, int s, std::vector<Mark>& waits) {
    Tensor& t = T(tid);
    if (t.storage == US_TENSOR_PERSIST) return;
    if (t.state == 1) return;
    if (t.state == 2 || t.state == 3)
      US_FAIL(US_ERR_USAGE, "tensor '%s' written after it was %s", t.name.c_str(),
              state_name(t.state));
    t.off = arena_alloc(t.bytes, s, waits, t);
    t.state = 1;
  }
  void release_tensor(Tensor& t, int new_state) {
    Mark ev[S_COUNT];
    if (flags & US_FLAG_POISON) {
      // debug poison: once every reader and the swap-out copy are done, the
      // region reads as NaN until its next owner writes it -- the next owner's allocation
      // waits on this (compute-stream) release mark, so it can only see its own data
      if (t.d2h_done.ev) CUDA_OK(cudaStreamWaitEvent(st[S_COMP], t.d2h_done.ev, 0));
      if (t.pending_h2d) CUDA_OK(cudaStreamWaitEvent(st[S_COMP], t.h2d_done.ev, 0));
      CUDA_OK(cudaMemsetAsync(arena + t.off, 0xFF, t.bytes, st[S_COMP]));
    }
    ev[S_COMP] = record(S_COMP);
    if (t.d2h_done.ev) ev[t.d2h_stream] = t.d2h_done;
    if (t.pending_h2d) ev[S_H2D] = t.h2d_done;   // prefetched but never read
    arena_release(t.off, ev);
    t.state = new_state;
    t.pending_h2d = false;
  }

  // Make stream s wait on `waits`; on the compute stream the wait is timed as a stall.
  void apply_waits(int s, std::vector<Mark>& waits) {
    if (waits.empty()) return;
    Mark pre;
    if (s == S_COMP) pre = record(S_COMP, true);
    for (auto& m : waits) CUDA_OK(cudaStreamWaitEvent(st[s], m.ev, 0));
    if (s == S_COMP) add_rec(cur_slot, US_CH_STALL, pre, record(S_COMP, true));
    waits.clear();
  }

  us::PairwisePlan& pw_plan(int64_t n) {
    auto it = pw_plans.find(n);
    if (it != pw_plans.end()) return it->second;
    us::PairwisePlan p = us::make_pairwise_plan(n);
    CUDA_OK(cudaGetLastError());
    if ((size_t)p.n_leaves + 1 > toy_scratch_elems) {
      if (toy_scratch) CUDA_OK(cudaFree(toy_scratch));
      toy_scratch_elems = (size_t)p.n_leaves + 64;
      CUDA_OK(cudaMalloc(&toy_scratch, toy_scratch_elems * sizeof(double)));
    }
    return pw_plans[n] = p;
  }

  void run_op(int index, const Op& op);

  // Operands of a fused BN-backward-sums request (BN input, stat + offset, partials out).
  us::BnSums bn_sums(const Op& op, int kx, int kstat, int kpart, int64_t stat_off, int C,
                     int* rows) {
    (void)C;
    us::BnSums b;
    b.x = ptr(op.t[kx]);
    b.stat = (const float*)ptr(op.t[kstat]) + stat_off;
    b.part = (float*)ptr(op.t[kpart]);
    b.rows = rows;
    return b;
  }
  // After dy's producer: if its kernel could not fold the sums in (rows == 0), run the
  // chan sums pass here; BN_BWD later reads bn_rows[part] rows.
  cudaError_t bn_sums_finish(const Op& op, int kpart, const us::BnSums& b, int rows,
                             const void* dy, int64_t vox, int C) {
    cudaError_t e = cudaSuccess;
    if (rows <= 0)
      e = us::bn_bwd_sums(st[S_COMP], T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, b.x, dy, b.stat,
                          b.part, vox, C, &rows);
    bn_rows[op.t[kpart]] = rows;
    return e;
  }
  void run_step();
  void enqueue_step();
  void collect();
};

namespace {

// Operand roles per opcode: 'R' read, 'W' written, 'P' persistent, 'O' optional read.
const char* op_roles(int code) {
  switch (code) {
    case US_OP_COPY_IN: return "PW";
    case US_OP_CAPTURE: return "RP";
    case US_OP_ZERO: return "W";
    case US_OP_TOUCH: return "R";
    case US_OP_TOY_AFFINE: case US_OP_TOY_AFFINE_BWD: case US_OP_TOY_RELU:
    case US_OP_TOY_CENTER: case US_OP_TOY_POOL: case US_OP_TOY_POOL_BWD:
    case US_OP_TOY_COPY: return "RW";
    case US_OP_TOY_RELU_BWD: case US_OP_TOY_ADD: return "RRW";
    case US_OP_TOY_SUMSQ: return "RP";
    case US_OP_INPUT_NCDHW: return "PW";
    case US_OP_PAD_CH: return "RW";
    case US_OP_CONV_FWD: return "RPWWO";
    case US_OP_BN_STATS: return "RP";
    case US_OP_NORM_ACT: return "RPPwwOw";
    case US_OP_POOL_FWD: case US_OP_RELU_FWD: return "RW";
    case US_OP_CONCAT: return "ROW";
    case US_OP_CONVT_FWD: return "RPW";
    case US_OP_LOSS_FWD: return "RPPWPP";
    case US_OP_LOSS_BWD: return "RPPPWPWOOw";
    case US_OP_RELU_BWD: return "RRW";
    case US_OP_BN_BWD: return "RRPPPWW";
    case US_OP_CONV_DGRAD: case US_OP_CONVT_DGRAD: return "RPWOOOw";
    case US_OP_CONV_WGRAD: case US_OP_CONVT_WGRAD: return "RRPWO";
    case US_OP_POOL_BWD: return "RROWOOw";
    case US_OP_ADAM: return "PPPPP";
    case US_OP_ALLREDUCE: return "P";
    case US_OP_CAST_W: case US_OP_LABELS_AUG: return "PP";
    default: return nullptr;
  }
}

us::ConvShape conv_shape(const Op& op) {
  us::ConvShape sh{};
  sh.N = (int)op.i[0]; sh.D = (int)op.i[1]; sh.H = (int)op.i[2]; sh.W = (int)op.i[3];
  sh.Cin = (int)op.i[4]; sh.Cout = (int)op.i[5];
  sh.x_cs = sh.Cin; sh.x_co = 0; sh.dy_cs = sh.Cout; sh.dy_co = 0;
  return sh;
}

}  // namespace

void us_ctx::run_op(int index, const Op& op) {
  cudaStream_t cs = st[S_COMP];
  std::vector<Mark> waits;
  switch (op.code) {
    case US_OP_SLOT_BEGIN: {
      cur_slot = (int)op.i[0];
      {
        auto nm = slot_names.find(cur_slot);
        nvtxRangePushA(nm != slot_names.end() ? nm->second.c_str() : "slot");
      }
      Mark m = record(S_COMP, true);
      if (m.ext) recs.push_back(Rec{cur_slot, US_CH_COMPUTE, m.ext, nullptr});
      return;
    }
    case US_OP_SLOT_END: {
      nvtxRangePop();
      Mark m = record(S_COMP, true);
      slot_end[(int)op.i[0]] = m;
      if (m.ext)
        for (auto it = recs.rbegin(); it != recs.rend(); ++it)
        if (it->channel == US_CH_COMPUTE && it->node == (int)op.i[0] && !it->b) {
          it->b = m.ext;
          break;
        }
      return;
    }
    case US_OP_SWAP_OUT: {
      Tensor& t = T(op.t[0]);
      if (t.state != 1 || t.pending_h2d)
        US_FAIL(US_ERR_DOMAIN, "use-after-swap: swap_out of tensor '%s' which is %s",
                t.name.c_str(), state_name(t.state));
      const int lane = S_D2H;
      Mark produced = record(S_COMP);
      CUDA_OK(cudaStreamWaitEvent(st[lane], produced.ev, 0));
      Mark a = record(lane, true);
      CUDA_OK(cudaMemcpyAsync(host_pool + t.host_off, arena + t.off, t.bytes,
                              cudaMemcpyDeviceToHost, st[lane]));
      t.d2h_done = record(lane, true);
      t.d2h_stream = lane;
      add_rec((int)op.i[0], US_CH_D2H, a, t.d2h_done);
      d2h_bytes += t.bytes;
      return;
    }
    case US_OP_SWAP_RELEASE: {
      Tensor& t = T(op.t[0]);
      if (t.state != 1 || !t.d2h_done.ev)
        US_FAIL(US_ERR_USAGE, "swap release of '%s' without a swap-out", t.name.c_str());
      release_tensor(t, 2);
      return;
    }
    case US_OP_SWAP_IN: {
      Tensor& src = T(op.t[0]);
      Tensor& dst = T(op.t[1]);
      if (src.state != 2 || !src.d2h_done.ev)
        US_FAIL(US_ERR_DOMAIN, "use-after-swap: swap_in of tensor '%s' which is %s",
                src.name.c_str(), src.state == 1 ? "still device-resident (no swap-out)"
                                                 : state_name(src.state));
      if (dst.bytes != src.bytes) US_FAIL(US_ERR_USAGE, "swap_in size mismatch");
      int trig = (int)op.i[1];
      auto te = slot_end.find(trig);
      if (te == slot_end.end())
        US_FAIL(US_ERR_USAGE, "swap_in of '%s' triggered by slot %d before it ran",
                src.name.c_str(), trig);
      CUDA_OK(cudaStreamWaitEvent(st[S_H2D], te->second.ev, 0));
      CUDA_OK(cudaStreamWaitEvent(st[S_H2D], src.d2h_done.ev, 0));
      dst.off = arena_alloc(dst.bytes, S_H2D, waits, dst);
      dst.state = 1;
      apply_waits(S_H2D, waits);
      Mark a = record(S_H2D, true);
      CUDA_OK(cudaMemcpyAsync(arena + dst.off, host_pool + src.host_off, dst.bytes,
                              cudaMemcpyHostToDevice, st[S_H2D]));
      dst.h2d_done = record(S_H2D, true);
      dst.pending_h2d = true;
      add_rec((int)op.i[0], US_CH_H2D, a, dst.h2d_done);
      h2d_bytes += dst.bytes;
      return;
    }
    case US_OP_FREE: {
      Tensor& t = T(op.t[0]);
      if (t.storage != US_TENSOR_ARENA) return;
      if (t.state != 1) US_FAIL(US_ERR_USAGE, "free of tensor '%s' which is %s", t.name.c_str(),
                                state_name(t.state));
      release_tensor(t, 3);
      return;
    }
    default:
      break;
  }

  const char* roles = op_roles(op.code);
  if (!roles) US_FAIL(US_ERR_USAGE, "unknown opcode %d", op.code);
  if ((int)op.t.size() != (int)strlen(roles))
    US_FAIL(US_ERR_USAGE, "opcode %d expects %zu tensors, got %zu", op.code, strlen(roles),
            op.t.size());
  for (size_t k = 0; k < op.t.size(); ++k) {
    char r = roles[k];
    int tid = op.t[k];
    if (r == 'O' && tid < 0) continue;
    if (r == 'P') {
      if (T(tid).storage != US_TENSOR_PERSIST)
        US_FAIL(US_ERR_USAGE, "opcode %d operand %zu must be persistent", op.code, k);
    } else if (r == 'R' || r == 'O') {
      check_read(tid, index, waits);
    }
  }
  for (size_t k = 0; k < op.t.size(); ++k)
    if (roles[k] == 'W' || (roles[k] == 'w' && op.t[k] >= 0))
      ensure_written(op.t[k], S_COMP, waits);
  apply_waits(S_COMP, waits);

  auto P = [&](int k) { return op.t[k] < 0 && roles[k] == 'w' ? nullptr : ptr(op.t[k]); };
  Mark op_a;
  if (flags & US_FLAG_OP_TIMES) op_a = record(S_COMP, true, true);
  auto D = [&](int k) { return (double*)ptr(op.t[k]); };
  const auto& I = op.i;
  const auto& F = op.f;
  cudaError_t e = cudaSuccess;
  switch (op.code) {
    case US_OP_COPY_IN:
      e = cudaMemcpyAsync(P(1), P(0), (size_t)I[0], cudaMemcpyDeviceToDevice, cs);
      break;
    case US_OP_CAPTURE:
      e = cudaMemcpyAsync((char*)P(1) + I[1], P(0), (size_t)I[0], cudaMemcpyDeviceToDevice, cs);
      break;
    case US_OP_ZERO:
      e = cudaMemsetAsync(P(0), 0, T(op.t[0]).bytes, cs);
      break;
    case US_OP_TOUCH:
      return;
    case US_OP_TOY_AFFINE: e = us::toy_affine(cs, D(0), D(1), I[0], I[1], F[0], F[1]); break;
    case US_OP_TOY_AFFINE_BWD: e = us::toy_affine_bwd(cs, D(0), D(1), I[0], I[1], F[0]); break;
    case US_OP_TOY_RELU: e = us::toy_relu(cs, D(0), D(1), I[0]); break;
    case US_OP_TOY_RELU_BWD: e = us::toy_relu_bwd(cs, D(0), D(1), D(2), I[0]); break;
    case US_OP_TOY_CENTER: {
      auto& plan = pw_plan(I[0]);
      e = us::toy_center(cs, D(0), D(1), plan, toy_scratch);
      break;
    }
    case US_OP_TOY_POOL: e = us::toy_pool(cs, D(0), D(1), I[0], I[1]); break;
    case US_OP_TOY_POOL_BWD: e = us::toy_pool_bwd(cs, D(0), D(1), I[0], I[1]); break;
    case US_OP_TOY_COPY: e = us::toy_copy(cs, D(0) + I[1], D(1) + I[2], I[0]); break;
    case US_OP_TOY_ADD: e = us::toy_add(cs, D(0), D(1), D(2), I[0], F[0]); break;
    case US_OP_TOY_SUMSQ: {
      auto& plan = pw_plan(I[0]);
      e = us::toy_sumsq(cs, D(0), I[0], D(1) + I[2], (int)I[1], plan, toy_scratch);
      break;
    }
    case US_OP_INPUT_NCDHW:
      e = us::input_ncdhw(cs, T(op.t[1]).dtype == US_DT_BF16 ? 2 : 1, (const float*)P(0), P(1),
                          (int)I[0], (int)I[1], (int)I[2], (int)I[3], (int)I[4], (int)I[5],
                          dynamic_op(op) ? (const int*)dyn_words(index, cs) : nullptr);
      break;
    case US_OP_LABELS_AUG:
      e = us::labels_aug(cs, (const uint8_t*)P(0), (uint8_t*)P(1), (int)I[0], (int)I[1],
                         (int)I[2], (int)I[3], (const int*)dyn_words(index, cs));
      break;
    case US_OP_PAD_CH:
      e = us::pad_channels(cs, T(op.t[1]).dtype == US_DT_BF16 ? 2 : 1, P(0), P(1), I[0],
                           (int)I[1], (int)I[2]);
      break;
    case US_OP_CONV_FWD: {
      us::ConvShape sh = conv_shape(op);
      sh.x_cs = (int)I[8]; sh.x_co = (int)I[9];
      int dt = T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1;
      const char* wb = (const char*)P(1) + I[6] * (dt == 2 ? 2 : 4);
      if (op.t.size() > 4 && op.t[4] >= 0) {   // dual-source input: [x | x2] along channels
        if (I[7] != US_ALGO_TCGEN05) US_FAIL(US_ERR_USAGE, "a dual-source conv needs tcgen05");
        sh.x2 = P(4);
        sh.x_split = sh.x_cs;
      }
      if (I[7] == US_ALGO_TCGEN05)
        e = us::conv_fwd_tc(cs, sh, (const __nv_bfloat16*)P(0), (const __nv_bfloat16*)wb,
                            (__nv_bfloat16*)P(2), (float*)P(3), split_scratch);
      else if (I[7] == US_ALGO_IM2COL)
        e = us::conv_fwd_stem(cs, sh, (const __nv_bfloat16*)P(0), (const __nv_bfloat16*)wb,
                              (__nv_bfloat16*)P(2), P(3));
      else
        e = us::conv_fwd_direct(cs, dt, sh, P(0), wb, P(2), (float*)P(3),
                                us::conv_stat_parts_direct(sh));
      break;
    }
    case US_OP_BN_STATS:
      e = us::bn_stats_finalize(cs, (const float*)P(0), (int)I[0], (int)I[1], (double)I[2],
                                (float*)P(1) + I[3], F[0]);
      break;
    case US_OP_NORM_ACT: {
      const float* prm = (const float*)P(2);
      if (op.t[6] >= 0) {   // fused head forward: Dice partials for the LOSS_FWD that follows
        if (op.t[4] < 0 || T(op.t[0]).dtype != US_DT_BF16)
          US_FAIL(US_ERR_USAGE, "fused norm+head needs bf16 and the ReLU output");
        int rows = 0;
        e = us::norm_act_loss(cs, P(0), (const float*)P(1) + I[2], prm + I[3], prm + I[4], P(3), P(4),
                              (const uint8_t*)P(5), prm + I[6], prm + I[7], (float*)P(6), I[0],
                              (int)I[1], (int)I[5], &rows);
        bn_rows[op.t[6]] = rows;
        break;
      }
      e = us::norm_act(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0),
                       (const float*)P(1) + I[2], prm + I[3], prm + I[4], P(3), P(4), I[0],
                       (int)I[1]);
      break;
    }
    case US_OP_POOL_FWD:
      e = us::pool_fwd(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0), P(1), (int)I[0],
                       (int)I[1], (int)I[2], (int)I[3], (int)I[4]);
      break;
    case US_OP_CONCAT:
      if (I.size() > 3 && I[3] == 1) {   // b already sits in y[:, Ca:] (its producer wrote it)
        e = us::copy_channels(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0), P(2), I[0],
                              (int)I[1], (int)(I[1] + I[2]), 0);
      } else {
        if (op.t[1] < 0) US_FAIL(US_ERR_USAGE, "concat without its second input");
        e = us::concat2(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0), P(1), P(2), I[0],
                        (int)I[1], (int)I[2]);
      }
      break;
    case US_OP_CONVT_FWD: {
      us::ConvShape sh = conv_shape(op);
      int dt = T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1;
      const char* wb = (const char*)P(1) + I[6] * (dt == 2 ? 2 : 4);
      const int y_cs = I.size() > 9 ? (int)I[8] : sh.Cout;
      const int y_co = I.size() > 9 ? (int)I[9] : 0;
      if (I[7] == US_ALGO_TCGEN05)
        e = us::convt_fwd_tc(cs, sh, (const __nv_bfloat16*)P(0), (const __nv_bfloat16*)wb,
                             (__nv_bfloat16*)P(2), split_scratch, y_cs, y_co);
      else if (y_cs != sh.Cout || y_co != 0)
        US_FAIL(US_ERR_USAGE, "convT into a channel slice needs the tcgen05 kernel");
      else
        e = us::convt_fwd_direct(cs, dt, sh, P(0), wb, P(2));
      break;
    }
    case US_OP_LOSS_FWD: {
      const float* prm = (const float*)P(2);
      if (I.size() > 6 && I[6] == 1) {   // partials written by the fused NORM_ACT
        auto it = bn_rows.find(op.t[3]);
        if (it == bn_rows.end() || it->second <= 0)
          US_FAIL(US_ERR_USAGE, "loss forward: no precomputed partials in '%s'",
                  T(op.t[3]).name.c_str());
        e = us::loss_finalize(cs, (const float*)P(3), it->second, (int)I[3], F[0], (double*)P(4),
                              (float*)P(5));
        break;
      }
      e = us::loss_fwd(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0), (const uint8_t*)P(1),
                       prm + I[4], prm + I[5], (float*)P(3), (double*)P(4), (float*)P(5),
                       (int)I[0], I[1], (int)I[2], (int)I[3], F[0]);
      break;
    }
    case US_OP_LOSS_BWD: {
      const float* prm = (const float*)P(2);
      float* g = (float*)P(5);
      int rows = 0;
      us::BnSums bn;
      if (op.t[9] >= 0) bn = bn_sums(op, 7, 8, 9, I[9], (int)I[2], &rows);
      e = us::loss_bwd(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0), (const uint8_t*)P(1),
                       prm + I[4], prm + I[5], (const double*)P(3), P(4), g + I[6], g + I[7],
                       (float*)P(6), (int)I[0], I[1], (int)I[2], (int)I[3], F[0],
                       I.size() > 8 ? (int)I[8] : 0, op.t[9] >= 0 ? &bn : nullptr);
      if (e == cudaSuccess && op.t[9] >= 0)
        e = bn_sums_finish(op, 9, bn, rows, P(4), I[0] * I[1], (int)I[2]);
      break;
    }
    case US_OP_RELU_FWD:
      e = us::relu_fwd(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0), P(1), I[0]);
      break;
    case US_OP_RELU_BWD:
      e = us::relu_bwd(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0), P(1), P(2), I[0]);
      break;
    case US_OP_BN_BWD: {
      const float* prm = (const float*)P(3);
      float* g = (float*)P(4);
      int npre = 0;
      if (I.size() > 6 && I[6] == 1) {   // partials written by dy's producer into P(6)
        auto it = bn_rows.find(op.t[6]);
        if (it == bn_rows.end() || it->second <= 0)
          US_FAIL(US_ERR_USAGE, "BN backward of '%s': no precomputed partials in '%s'",
                  T(op.t[0]).name.c_str(), T(op.t[6]).name.c_str());
        npre = it->second;
      }
      e = us::bn_bwd(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0), P(1),
                     (const float*)P(2) + I[2], prm + I[3], g + I[4], g + I[5], P(5),
                     (float*)P(6), I[0], (int)I[1], npre);
      break;
    }
    case US_OP_CONV_DGRAD:
    case US_OP_CONVT_DGRAD: {
      us::ConvShape sh = conv_shape(op);
      sh.dy_cs = (int)I[8]; sh.dy_co = (int)I[9];
      int dt = T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1;
      const char* wb = (const char*)P(1) + I[6] * (dt == 2 ? 2 : 4);
      bool tc = I[7] == US_ALGO_TCGEN05;
      if (op.t.size() > 3 && op.t[3] >= 0) {   // fused ReLU backward (tcgen05 epilogue)
        if (!tc || dt != 2) US_FAIL(US_ERR_USAGE, "fused ReLU mask needs the bf16 tcgen05 dgrad");
        sh.relu_mask = P(3);
      }
      int rows = 0;
      us::BnSums bn;
      if (op.t[6] >= 0) {   // fused BN-backward sums of dx (tcgen05 epilogue)
        bn = bn_sums(op, 4, 5, 6, I[10], sh.Cin, &rows);
        if (tc && dt == 2) {
          sh.bn_x = bn.x;
          sh.bn_stat = bn.stat;
          sh.bn_part = bn.part;
          sh.bn_rows = &rows;
        }
      }
      if (op.code == US_OP_CONV_DGRAD)
        e = tc ? us::conv_dgrad_tc(cs, sh, (const __nv_bfloat16*)P(0), (const __nv_bfloat16*)wb,
                                   (__nv_bfloat16*)P(2), split_scratch)
               : us::conv_dgrad_direct(cs, dt, sh, P(0), wb, P(2));
      else
        e = tc ? us::convt_dgrad_tc(cs, sh, (const __nv_bfloat16*)P(0), (const __nv_bfloat16*)wb,
                                    (__nv_bfloat16*)P(2))
               : us::convt_dgrad_direct(cs, dt, sh, P(0), wb, P(2));
      if (e == cudaSuccess && op.t[6] >= 0)
        e = bn_sums_finish(op, 6, bn, rows, P(2), (int64_t)sh.N * sh.D * sh.H * sh.W, sh.Cin);
      break;
    }
    case US_OP_CONV_WGRAD:
    case US_OP_CONVT_WGRAD: {
      us::ConvShape sh = conv_shape(op);
      sh.dy_cs = (int)I[8]; sh.dy_co = (int)I[9];
      int dt = T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1;
      float* gw = (float*)P(2) + I[6];
      bool tc = I[7] == US_ALGO_TCGEN05;
      if (op.t.size() > 4 && op.t[4] >= 0) {   // dual-source input: x holds I[10] channels
        if (!tc || op.code != US_OP_CONV_WGRAD || I.size() < 11)
          US_FAIL(US_ERR_USAGE, "a dual-source weight gradient needs the tcgen05 conv");
        sh.x2 = P(4);
        sh.x_cs = sh.x_split = (int)I[10];
      }
      if (op.code == US_OP_CONV_WGRAD && I[7] == US_ALGO_IM2COL)
        e = us::conv_wgrad_stem(cs, sh, (const __nv_bfloat16*)P(0), (const __nv_bfloat16*)P(1),
                                gw, P(3));
      else if (op.code == US_OP_CONV_WGRAD)
        e = tc ? us::conv_wgrad_tc(cs, sh, (const __nv_bfloat16*)P(0),
                                   (const __nv_bfloat16*)P(1), gw, (float*)P(3))
               : us::conv_wgrad_direct(cs, dt, sh, P(0), P(1), gw);
      else
        e = tc ? us::convt_wgrad_tc(cs, sh, (const __nv_bfloat16*)P(0),
                                    (const __nv_bfloat16*)P(1), gw, (float*)P(3))
               : us::convt_wgrad_direct(cs, dt, sh, P(0), P(1), gw);
      break;
    }
    case US_OP_POOL_BWD: {
      int rows = 0;
      us::BnSums bn;
      if (op.t[6] >= 0) bn = bn_sums(op, 4, 5, 6, I[8], (int)I[4], &rows);
      e = us::pool_bwd(cs, T(op.t[0]).dtype == US_DT_BF16 ? 2 : 1, P(0), P(1),
                       op.t[2] >= 0 ? P(2) : nullptr, (int)I[5], (int)I[6], P(3), (int)I[0],
                       (int)I[1], (int)I[2], (int)I[3], (int)I[4], I.size() > 7 ? (int)I[7] : 0,
                       op.t[6] >= 0 ? &bn : nullptr);
      if (e == cudaSuccess && op.t[6] >= 0)
        e = bn_sums_finish(op, 6, bn, rows, P(3), (int64_t)I[0] * I[1] * I[2] * I[3], (int)I[4]);
      break;
    }
    case US_OP_ADAM: {
      // i[3] == 1: one gradient bucket's update on the comm stream, issued as soon as the
      // backward has written (and, data parallel, reduced) it -- the optimizer overlaps
      // the rest of the backward.  Otherwise the whole buffer after every bucket.
      const int64_t off = I.size() > 2 ? I[2] : 0;
      const bool bucket = I.size() > 3 && I[3] == 1;
      cudaStream_t ss = cs;
      if (bucket) {
        Mark ready = record(S_COMP);
        CUDA_OK(cudaStreamWaitEvent(st[S_COMM], ready.ev, 0));
        ss = st[S_COMM];
      } else if (comm_done.ev) {
        CUDA_OK(cudaStreamWaitEvent(cs, comm_done.ev, 0));   // all buckets reduced
      }
      const float* corr = (const float*)dyn_words(index, ss);
      e = us::adam(ss, (float*)P(0) + off, (const float*)P(1) + off, (float*)P(2) + off,
                   (float*)P(3) + off, I[1] ? (__nv_bfloat16*)P(4) + off : nullptr, I[0],
                   (float)F[0], (float)F[1], (float)F[2], (float)F[3], corr);
      if (bucket) comm_done = record(S_COMM);
      break;
    }
    case US_OP_CAST_W:
      e = us::cast_bf16(cs, (const float*)P(0), (__nv_bfloat16*)P(1), I[0]);
      break;
    case US_OP_ALLREDUCE: {
      // i[2] == 1: a gradient bucket, reduced on the comm stream once the compute stream
      // has written it (the backward keeps running); ADAM waits for all buckets.
      float* g = (float*)P(0) + I[0];
      const bool async = I.size() > 2 && I[2] == 1;
      cudaStream_t ss = cs;
      if (async) {
        Mark ready = record(S_COMP);
        CUDA_OK(cudaStreamWaitEvent(st[S_COMM], ready.ev, 0));
        ss = st[S_COMM];
      }
      if (nccl_comm) {
        int r = g_nccl.allReduce(g, g, (size_t)I[1], /*ncclFloat32*/ 7, /*ncclSum*/ 0,
                                 nccl_comm, ss);
        if (r != 0)
          US_FAIL(US_ERR_NCCL, "ncclAllReduce failed: %s", g_nccl.errStr ? g_nccl.errStr(r) : "?");
      }
      if (F.size() && F[0] != 1.0) e = us::scale_f32(ss, g, I[1], (float)F[0]);
      if (async) comm_done = record(S_COMM);
      break;
    }
    default:
      US_FAIL(US_ERR_USAGE, "unhandled opcode %d", op.code);
  }
  if (e != cudaSuccess)
    US_FAIL(US_ERR_CUDA, "launch of opcode %d (op %d) failed: %s", op.code, index,
            cudaGetErrorString(e));
  if (op_a.ev) add_rec(index, US_CH_OP, op_a, record(S_COMP, true, true));
  ++kernels;
}

void us_ctx::run_step() {
  if (!finalized) US_FAIL(US_ERR_USAGE, "program not finalized");
  CUDA_OK(cudaSetDevice(device));
  // NVTX (no-op unless a tool such as nsys is attached): one range per step, and per slot
  // while an eager step is enqueued (SLOT_BEGIN / SLOT_END below)
  struct StepRange {
    StepRange() { nvtxRangePushA("us_run step"); }
    ~StepRange() { nvtxRangePop(); }
  } step_range;
  parity ^= 1;
  set_dyn_scalars(parity);
  const bool use_graph = (flags & US_FLAG_GRAPH) != 0;
  if (use_graph && graph[parity].exec) {
    // replay: one launch; the recorded events and stats are the captured ones
    const auto h0 = std::chrono::steady_clock::now();
    CUDA_OK(cudaGraphLaunch(graph[parity].exec, st[S_COMP]));
    host_enqueue_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
    collect();
    inflight = graph[parity].rec;
    ++runs;
    return;
  }
  // Graphs are captured only without the per-slot timeline: its timed events become
  // external event-record nodes, which serialise the copy and compute branches of the
  // replay (paper-c4: 198 ms replayed untimed, 284 ms replayed with the timeline).
  const bool capture = use_graph && runs >= 2 && !timeline_on();
  if (capture) {
    CUDA_OK(cudaStreamBeginCapture(st[S_COMP], cudaStreamCaptureModeRelaxed));
    capturing = true;
  }
  try {
    enqueue_step();
  } catch (...) {
    if (capture) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(st[S_COMP], &g);
      if (g) cudaGraphDestroy(g);
      capturing = false;
      (void)cudaGetLastError();
    }
    throw;
  }
  if (capture) {
    capturing = false;
    cudaGraph_t g = nullptr;
    CUDA_OK(cudaStreamEndCapture(st[S_COMP], &g));
    size_t n_nodes = 0;
    CUDA_OK(cudaGraphGetNodes(g, nullptr, &n_nodes));
    std::vector<cudaGraphNode_t> nodes(n_nodes);
    CUDA_OK(cudaGraphGetNodes(g, nodes.data(), &n_nodes));
    int n_kernels = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType ty;
      CUDA_OK(cudaGraphNodeGetType(nd, &ty));
      n_kernels += ty == cudaGraphNodeTypeKernel;
    }
    kernels = n_kernels;   // exact kernel launches of the step (ops may launch several)
    cudaError_t ie = cudaGraphInstantiate(&graph[parity].exec, g, 0);
    cudaGraphDestroy(g);
    CUDA_OK(ie);
    CUDA_OK(cudaGraphLaunch(graph[parity].exec, st[S_COMP]));
  }
  // The previous step's events live in the other pool; read them back only
  // now, after this step is enqueued, so the GPU never idles on the host.
  collect();
  inflight.recs.swap(recs);
  inflight.start = step_start;
  inflight.end = step_end;
  inflight.d2h = d2h_bytes;
  inflight.h2d = h2d_bytes;
  inflight.peak = step_peak;
  inflight.kernels = kernels;
  inflight.valid = true;
  if (capture) graph[parity].rec = inflight;
  ++runs;
}

void us_ctx::enqueue_step() {
  pool_next = 0;
  tpool_next = 0;
  recs.clear();
  slot_end.clear();
  cur_slot = -1;
  d2h_bytes = h2d_bytes = 0;
  kernels = 0;
  arena_reset();
  forget_marks();
  for (auto& t : tensors) {
    t.state = 0;
    t.d2h_done = Mark{};
    t.h2d_done = Mark{};
    t.pending_h2d = false;
  }
  Mark start = record(S_COMP, true, true);
  // copy streams may only start once the previous step fully retired
  CUDA_OK(cudaStreamWaitEvent(st[S_D2H], start.ev, 0));
  CUDA_OK(cudaStreamWaitEvent(st[S_H2D], start.ev, 0));
  CUDA_OK(cudaStreamWaitEvent(st[S_COMM], start.ev, 0));
  comm_done = Mark{};
  const auto h0 = std::chrono::steady_clock::now();
  static const bool host_prof = getenv("US_HOST_PROFILE") != nullptr;
  for (size_t k = 0; k < ops.size(); ++k) {
    if (!host_prof) {
      run_op((int)k, ops[k]);
      continue;
    }
    const auto t0 = std::chrono::steady_clock::now();
    run_op((int)k, ops[k]);
    host_op_s[ops[k].code] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    host_op_n[ops[k].code] += 1;
  }
  host_enqueue_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
  Mark d = record(S_D2H), h = record(S_H2D), cm = record(S_COMM);
  CUDA_OK(cudaStreamWaitEvent(st[S_COMP], cm.ev, 0));
  CUDA_OK(cudaStreamWaitEvent(st[S_COMP], d.ev, 0));
  CUDA_OK(cudaStreamWaitEvent(st[S_COMP], h.ev, 0));
  Mark end = record(S_COMP, true, true);
  step_start = start.ext;
  step_end = end.ext;
}

void us_ctx::collect() {
  if (!inflight.valid) return;
  StepRec& r = inflight;
  CUDA_OK(cudaEventSynchronize(r.end));
  r.valid = false;
  float ms = 0;
  CUDA_OK(cudaEventElapsedTime(&ms, r.start, r.end));
  done.step_s = ms * 1e-3;
  done.d2h = r.d2h;
  done.h2d = r.h2d;
  done.peak = r.peak;
  done.kernels = r.kernels;
  timeline.clear();
  double stall = 0;
  for (auto& x : r.recs) {
    if (!x.a || !x.b) continue;
    float a = 0, b = 0;
    CUDA_OK(cudaEventElapsedTime(&a, r.start, x.a));
    CUDA_OK(cudaEventElapsedTime(&b, r.start, x.b));
    us_event ev{x.node, x.channel, a * 1e-3, b * 1e-3};
    if (x.channel == US_CH_STALL) stall += ev.end_s - ev.start_s;
    timeline.push_back(ev);
  }
  done.stall_s = stall;
}

// ============================================================== C ABI
namespace {
template <class F>
int guard(F&& f) {
  try {
    f();
    return US_OK;
  } catch (const UsError& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return US_ERR_USAGE;
  }
}

// NUMA node of the GPU's PCIe attachment (sysfs), -1 when unknown.
int gpu_numa_node(int device) {
  if (const char* e = getenv("US_HOST_NUMA")) return atoi(e);   // override; -1 = unbound
  char bus[32] = {};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return -1;
  for (char* p = bus; *p; ++p) *p = (char)tolower(*p);
  FILE* f = fopen((std::string("/sys/bus/pci/devices/") + bus + "/numa_node").c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  return node;
}

// Pinned host pool for the swapped tensors, on the GPU's own NUMA node (SURVEY 7 H7:
// eight ranks swapping at once must not pull their pools across the socket link).  The
// pages are reserved with mmap, bound to the node with mbind (MPOL_PREFERRED: fall back
// to another node rather than fail when the local one is full), then faulted in and
// page-locked by cudaHostRegister.  Without a known node: plain cudaHostAlloc.
void alloc_host_pool(us_ctx* c, uint64_t bytes) {
  const int node = gpu_numa_node(c->device);
  c->host_numa_node = -1;
  if (node >= 0 && node < 1024) {
    const uint64_t len = (bytes + (2u << 20) - 1) & ~uint64_t((2u << 20) - 1);
    void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p != MAP_FAILED) {
      unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {};
      mask[node / (8 * sizeof(unsigned long))] |= 1ul << (node % (8 * sizeof(unsigned long)));
      const long mpol_preferred = 1;
      const bool bound = syscall(SYS_mbind, p, len, mpol_preferred, mask, 1024ul, 0u) == 0;
      madvise(p, len, MADV_HUGEPAGE);
      if (cudaHostRegister(p, len, cudaHostRegisterDefault) == cudaSuccess) {
        c->host_pool = (char*)p;
        c->host_map_bytes = len;
        c->host_numa_node = bound ? node : -1;
        return;
      }
      cudaGetLastError();   // clear the registration failure, fall back below
      munmap(p, len);
    }
  }
  CUDA_OK(cudaHostAlloc((void**)&c->host_pool, bytes, cudaHostAllocDefault));
}

void free_host_pool(us_ctx* c) {
  if (!c->host_pool) return;
  if (c->host_map_bytes) {
    cudaHostUnregister(c->host_pool);
    munmap(c->host_pool, c->host_map_bytes);
  } else {
    cudaFreeHost(c->host_pool);
  }
  c->host_pool = nullptr;
  c->host_map_bytes = 0;
  c->host_numa_node = -1;
}
}  // namespace

extern "C" {

const char* us_last_error(void) { return g_last_error.c_str(); }
int us_abi_version(void) { return US_ABI_VERSION; }

int us_set_flags(us_ctx* c, uint32_t flags) {
  return guard([&] {
    if (flags != c->flags) {
      c->collect();
      CUDA_OK(cudaStreamSynchronize(c->st[S_COMP]));
      c->drop_graphs();
    }
    c->flags = flags;
  });
}

int us_ctx_create(int32_t device, uint64_t arena_bytes, uint32_t flags, us_ctx** out) {
  return guard([&] {
    if (!out) US_FAIL(US_ERR_USAGE, "null out pointer");
    int n = 0;
    CUDA_OK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) US_FAIL(US_ERR_USAGE, "device %d out of range (%d)", device, n);
    CUDA_OK(cudaSetDevice(device));
    auto* c = new us_ctx();
    c->device = device;
    c->flags = flags;
    for (int s = 0; s < S_COUNT; ++s)
      CUDA_OK(cudaStreamCreateWithFlags(&c->st[s], cudaStreamNonBlocking));
    c->arena_cap = (arena_bytes + 1023) & ~uint64_t(1023);
    if (c->arena_cap) CUDA_OK(cudaMalloc(&c->arena, c->arena_cap));
    c->arena_reset();
    *out = c;
  });
}

int us_ctx_destroy(us_ctx* c) {
  if (c && getenv("US_HOST_PROFILE")) {
    for (int k = 0; k < US_OP_COUNT; ++k)
      if (c->host_op_n[k])
        fprintf(stderr, "[host] opcode %2d: %8.3f ms total, %6ld calls, %7.1f us/call\n", k,
                1e3 * c->host_op_s[k], c->host_op_n[k], 1e6 * c->host_op_s[k] / c->host_op_n[k]);
  }
  return guard([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    for (int s = 0; s < S_COUNT; ++s)
      if (c->st[s]) cudaStreamSynchronize(c->st[s]);
    for (auto& t : c->tensors)
      if (t.pptr) cudaFree(t.pptr);
    for (auto& kv : c->pw_plans) us::free_pairwise_plan(kv.second);
    if (c->toy_scratch) cudaFree(c->toy_scratch);
    if (c->arena) cudaFree(c->arena);
    free_host_pool(c);
    c->drop_graphs();
    for (auto& h : c->dyn_host)
      if (h) cudaFreeHost(h);
    if (c->dyn_dev) cudaFree(c->dyn_dev);
    if (c->split_scratch) cudaFree(c->split_scratch);
    for (auto& p : c->pool)
      for (auto e : p) cudaEventDestroy(e);
    for (auto& p : c->tpool)
      for (auto e : p) cudaEventDestroy(e);
    if (c->nccl_comm && g_nccl.commDestroy) g_nccl.commDestroy(c->nccl_comm);
    for (int s = 0; s < S_COUNT; ++s)
      if (c->st[s]) cudaStreamDestroy(c->st[s]);
    delete c;
  });
}

int us_prog_reset(us_ctx* c) {
  return guard([&] {
    c->collect();
    c->drop_graphs();
    CUDA_OK(cudaSetDevice(c->device));
    CUDA_OK(cudaDeviceSynchronize());
    for (auto& t : c->tensors)
      if (t.pptr) CUDA_OK(cudaFree(t.pptr));
    c->tensors.clear();
    c->ops.clear();
    c->slot_names.clear();
    c->finalized = false;
    c->persistent_bytes = 0;
    free_host_pool(c);
    c->host_cap = 0;
  });
}

int us_tensor(us_ctx* c, int32_t tid, uint64_t bytes, int32_t storage, int32_t dtype,
              const char* name) {
  return guard([&] {
    if (c->finalized) US_FAIL(US_ERR_USAGE, "program already finalized");
    if (tid < 0) US_FAIL(US_ERR_USAGE, "negative tensor id");
    if ((int)c->tensors.size() <= tid) c->tensors.resize(tid + 1);
    Tensor& t = c->tensors[tid];
    if (t.defined) US_FAIL(US_ERR_USAGE, "tensor %d defined twice", tid);
    t.defined = true;
    t.name = name ? name : fmt("t%d", tid);
    t.bytes = bytes;
    t.storage = storage;
    t.dtype = dtype;
    if (storage == US_TENSOR_PERSIST) {
      CUDA_OK(cudaSetDevice(c->device));
      CUDA_OK(cudaMalloc(&t.pptr, bytes ? bytes : 16));
      CUDA_OK(cudaMemset(t.pptr, 0, bytes ? bytes : 16));
      c->persistent_bytes += bytes;
    }
  });
}

int us_tensor_place(us_ctx* c, int32_t tid, uint64_t offset) {
  return guard([&] {
    if (c->finalized) US_FAIL(US_ERR_USAGE, "program already finalized");
    if (tid < 0 || tid >= (int)c->tensors.size() || !c->tensors[tid].defined)
      US_FAIL(US_ERR_USAGE, "placement of undefined tensor %d", tid);
    Tensor& t = c->tensors[tid];
    if (t.storage != US_TENSOR_ARENA)
      US_FAIL(US_ERR_USAGE, "placement of persistent tensor '%s'", t.name.c_str());
    if (offset % 1024) US_FAIL(US_ERR_USAGE, "placement offset must be 1024-aligned");
    t.fixed_off = (int64_t)offset;
  });
}

int us_slot_name(us_ctx* c, int32_t slot, const char* name) {
  return guard([&] { c->slot_names[slot] = name ? name : ""; });
}

int us_op(us_ctx* c, int32_t opcode, const int32_t* tensors, int32_t nt, const int64_t* iargs,
          int32_t ni, const double* fargs, int32_t nf) {
  return guard([&] {
    if (c->finalized) US_FAIL(US_ERR_USAGE, "program already finalized");
    if (opcode < 0 || opcode >= US_OP_COUNT) US_FAIL(US_ERR_USAGE, "bad opcode %d", opcode);
    Op op;
    op.code = opcode;
    op.t.assign(tensors, tensors + nt);
    // trailing optional operands ('O' read, 'w' write) may be left out: absent = -1
    if (const char* roles = op_roles(opcode)) {
      const size_t nr = strlen(roles);
      for (size_t k = op.t.size(); k < nr; ++k) {
        if (roles[k] != 'O' && roles[k] != 'w')
          US_FAIL(US_ERR_USAGE, "opcode %d expects %zu tensors, got %d", opcode, nr, nt);
        op.t.push_back(-1);
      }
    }
    op.i.assign(iargs, iargs + ni);
    op.f.assign(fargs, fargs + nf);
    c->ops.push_back(std::move(op));
  });
}

int us_prog_finalize(us_ctx* c) {
  return guard([&] {
    // static placement is all or nothing: a best-fit block could land on a planned region
    std::vector<char> used(c->tensors.size(), 0);
    for (auto& op : c->ops)
      for (int tid : op.t)
        if (tid >= 0 && tid < (int)used.size()) used[tid] = 1;
    int placed = 0, arena_tensors = 0;
    for (size_t j = 0; j < c->tensors.size(); ++j) {
      auto& t = c->tensors[j];
      if (!t.defined || t.storage != US_TENSOR_ARENA || !used[j]) continue;
      ++arena_tensors;
      if (t.fixed_off >= 0) {
        ++placed;
        if ((uint64_t)t.fixed_off + ((t.bytes + 1023) & ~uint64_t(1023)) > c->arena_cap)
          US_FAIL(US_ERR_DOMAIN, "budget exhausted: infeasible: tensor '%s' is placed at "
                  "%lld, past the %llu-byte budget", t.name.c_str(), (long long)t.fixed_off,
                  (unsigned long long)c->arena_cap);
      }
    }
    if (placed && placed != arena_tensors)
      US_FAIL(US_ERR_USAGE, "%d of %d arena tensors placed: place all or none", placed,
              arena_tensors);
    c->fixed_layout = placed > 0;
    // Host slots for every swapped-out tensor, 4 KiB aligned, in program order.
    uint64_t off = 0;
    for (auto& op : c->ops) {
      if (op.code != US_OP_SWAP_OUT) continue;
      Tensor& t = c->T(op.t[0]);
      if (t.host_off >= 0) continue;
      t.host_off = (int64_t)off;
      off += (t.bytes + 4095) & ~uint64_t(4095);
    }
    for (auto& op : c->ops) {
      const char* roles = op_roles(op.code);
      if (roles && op.t.size() != strlen(roles))
        US_FAIL(US_ERR_USAGE, "opcode %d expects %zu tensors, got %zu", op.code, strlen(roles),
                op.t.size());
      for (int tid : op.t)
        if (tid >= 0) c->T(tid);
    }
    CUDA_OK(cudaSetDevice(c->device));
    c->drop_graphs();
    size_t split_need = 0;
    for (auto& op : c->ops)
      if ((op.code == US_OP_CONV_FWD || op.code == US_OP_CONV_DGRAD) && op.i.size() > 7 &&
          op.i[7] == US_ALGO_TCGEN05)
        split_need = std::max(split_need, us::conv_split_scratch_bytes(
                                              conv_shape(op), op.code == US_OP_CONV_DGRAD));
    for (auto& op : c->ops)   // sub-pixel convT weight re-layout shares the scratch
      if (op.code == US_OP_CONVT_FWD && op.i.size() > 7 && op.i[7] == US_ALGO_TCGEN05)
        split_need = std::max(split_need, us::convt_fwd_scratch_bytes(conv_shape(op)));
    if (split_need > c->split_cap) {
      if (c->split_scratch) CUDA_OK(cudaFree(c->split_scratch));
      CUDA_OK(cudaMalloc((void**)&c->split_scratch, split_need));
      c->split_cap = split_need;
    }
    int n_dyn = 0;
    c->dyn_slot.assign(c->ops.size(), -1);
    for (size_t j = 0; j < c->ops.size(); ++j)
      if (us_ctx::dynamic_op(c->ops[j])) c->dyn_slot[j] = n_dyn++;
    if (n_dyn > c->n_dyn) {
      for (auto& h : c->dyn_host)
        if (h) CUDA_OK(cudaFreeHost(h));
      if (c->dyn_dev) CUDA_OK(cudaFree(c->dyn_dev));
      for (auto& h : c->dyn_host) CUDA_OK(cudaMallocHost((void**)&h, 2 * n_dyn * sizeof(uint32_t)));
      CUDA_OK(cudaMalloc((void**)&c->dyn_dev, 2 * n_dyn * sizeof(uint32_t)));
      c->n_dyn = n_dyn;
    }
    if (off) alloc_host_pool(c, off);
    c->host_cap = off;
    c->finalized = true;
  });
}

int us_op_set_farg(us_ctx* c, int32_t op_index, int32_t k, double value) {
  return guard([&] {
    if (op_index < 0 || op_index >= (int)c->ops.size()) US_FAIL(US_ERR_USAGE, "bad op index");
    auto& f = c->ops[op_index].f;
    if (k < 0 || k >= (int)f.size()) US_FAIL(US_ERR_USAGE, "bad farg index");
    if (f[k] != value && !us_ctx::dynamic_op(c->ops[op_index])) c->drop_graphs();
    f[k] = value;
  });
}

int us_upload(us_ctx* c, int32_t tid, const void* host, uint64_t bytes, uint64_t offset) {
  return guard([&] {
    Tensor& t = c->T(tid);
    if (t.storage != US_TENSOR_PERSIST) US_FAIL(US_ERR_USAGE, "upload to a step tensor");
    if (offset + bytes > t.bytes) US_FAIL(US_ERR_USAGE, "upload out of range for '%s'", t.name.c_str());
    CUDA_OK(cudaMemcpyAsync((char*)t.pptr + offset, host, bytes, cudaMemcpyHostToDevice,
                            c->st[S_COMP]));
  });
}

int us_download(us_ctx* c, int32_t tid, void* host, uint64_t bytes, uint64_t offset) {
  return guard([&] {
    Tensor& t = c->T(tid);
    if (t.storage != US_TENSOR_PERSIST) US_FAIL(US_ERR_USAGE, "download of a step tensor");
    if (offset + bytes > t.bytes) US_FAIL(US_ERR_USAGE, "download out of range for '%s'", t.name.c_str());
    CUDA_OK(cudaMemcpyAsync(host, (char*)t.pptr + offset, bytes, cudaMemcpyDeviceToHost,
                            c->st[S_COMP]));
    CUDA_OK(cudaStreamSynchronize(c->st[S_COMP]));
  });
}

int us_tensor_ptr(us_ctx* c, int32_t tid, void** out) {
  return guard([&] {
    Tensor& t = c->T(tid);
    if (t.storage != US_TENSOR_PERSIST) US_FAIL(US_ERR_USAGE, "pointer of a step tensor");
    *out = t.pptr;
  });
}

int us_workspace_bytes(int32_t opcode, const int64_t* I, int32_t ni, uint64_t* out) {
  return guard([&] {
    auto need = [&](int n) {
      if (ni < n) US_FAIL(US_ERR_USAGE, "opcode %d needs %d iargs", opcode, n);
    };
    uint64_t b = 16;
    switch (opcode) {
      case US_OP_CONV_FWD: {
        need(8);
        us::ConvShape sh{};
        sh.N = (int)I[0]; sh.D = (int)I[1]; sh.H = (int)I[2]; sh.W = (int)I[3];
        sh.Cin = (int)I[4]; sh.Cout = (int)I[5];
        if (I[7] == US_ALGO_IM2COL) {
          b = us::stem_fwd_workspace(sh);
          break;
        }
        int parts = I[7] == US_ALGO_TCGEN05 ? us::conv_stat_parts_tc(sh)
                                            : us::conv_stat_parts_direct(sh);
        b = (uint64_t)parts * 2 * sh.Cout * sizeof(float);
        break;
      }
      case US_OP_BN_BWD: {
        need(2);
        // room for precomputed partials from dy's producer as well (bn_bwd_rows_max)
        int parts = us::bn_bwd_rows_max(I[0], (int)I[1]);
        b = ((uint64_t)parts * 2 + 3) * I[1] * sizeof(float);
        break;
      }
      case US_OP_LOSS_FWD: {
        need(4);   // room for the fused NORM_ACT's partial rows as well
        const int rows = std::max(us::loss_parts(I[0] * I[1]), us::norm_act_loss_parts(I[0] * I[1]));
        b = (uint64_t)rows * 3 * I[3] * sizeof(float);
        break;
      }
      case US_OP_LOSS_BWD: {
        need(4);
        b = (uint64_t)us::loss_parts(I[0] * I[1]) * (I[3] * I[2] + I[3]) * sizeof(float);
        break;
      }
      case US_OP_CONV_WGRAD:
      case US_OP_CONVT_WGRAD: {
        need(8);
        us::ConvShape sh{};
        sh.N = (int)I[0]; sh.D = (int)I[1]; sh.H = (int)I[2]; sh.W = (int)I[3];
        sh.Cin = (int)I[4]; sh.Cout = (int)I[5];
        if (I[7] == US_ALGO_TCGEN05)
          b = us::wgrad_tc_workspace(sh, opcode == US_OP_CONVT_WGRAD);
        else if (I[7] == US_ALGO_IM2COL && opcode == US_OP_CONV_WGRAD)
          b = us::stem_wgrad_workspace(sh);
        break;
      }
      default:
        break;
    }
    *out = b < 16 ? 16 : b;
  });
}

int us_run(us_ctx* c) {
  return guard([&] { c->run_step(); });
}

int us_sync(us_ctx* c) {
  return guard([&] {
    c->collect();
    CUDA_OK(cudaStreamSynchronize(c->st[S_COMP]));
    CUDA_OK(cudaGetLastError());
  });
}

int us_mark(us_ctx* c, int32_t which) {
  return guard([&] {
    CUDA_OK(cudaSetDevice(c->device));
    cudaEvent_t& e = which == 0 ? c->window_start : c->window_end;
    if (!e) CUDA_OK(cudaEventCreate(&e));
    CUDA_OK(cudaEventRecord(e, c->st[S_COMP]));
  });
}

int us_elapsed(us_ctx* c, double* seconds) {
  return guard([&] {
    if (!c->window_start || !c->window_end) US_FAIL(US_ERR_USAGE, "timing window not marked");
    CUDA_OK(cudaEventSynchronize(c->window_end));
    float ms = 0;
    CUDA_OK(cudaEventElapsedTime(&ms, c->window_start, c->window_end));
    *seconds = ms * 1e-3;
  });
}

int us_stats_get(us_ctx* c, us_stats* s) {
  return guard([&] {
    std::memset(s, 0, sizeof *s);
    s->arena_bytes = c->arena_cap;
    s->arena_peak_bytes = c->done.peak;
    s->persistent_bytes = c->persistent_bytes;
    s->host_pool_bytes = c->host_cap;
    s->d2h_bytes = c->done.d2h;
    s->h2d_bytes = c->done.h2d;
    s->step_s = c->done.step_s;
    s->stall_s = c->done.stall_s;
    s->kernels = c->done.kernels;
    s->events = (int32_t)c->timeline.size();
    s->host_enqueue_s = c->host_enqueue_s;
    s->host_numa_node = c->host_numa_node;
    s->dp_nranks = c->nccl_comm ? c->nranks : 0;
  });
}

int us_timeline(us_ctx* c, us_event* out, int32_t cap, int32_t* count) {
  return guard([&] {
    int n = (int)c->timeline.size();
    if (count) *count = n;
    for (int k = 0; k < n && k < cap; ++k) out[k] = c->timeline[k];
  });
}

int us_dp_unique_id(void* out, int32_t cap, int32_t* id_bytes) {
  return guard([&] {
    if (!g_nccl.load()) US_FAIL(US_ERR_NCCL, "libnccl not found (set US_NCCL_LIB)");
    if (cap < 128) US_FAIL(US_ERR_USAGE, "need 128 bytes for the NCCL unique id");
    int r = g_nccl.getUniqueId(out);
    if (r) US_FAIL(US_ERR_NCCL, "ncclGetUniqueId failed (%d)", r);
    if (id_bytes) *id_bytes = 128;
  });
}

int us_dp_init(us_ctx* c, const void* uid, int32_t id_bytes, int32_t nranks, int32_t rank) {
  return guard([&] {
    // nranks == 1 still builds a (single-rank) communicator, so the bucketed all-reduce
    // path runs through NCCL on one GPU exactly as it does on eight
    if (nranks < 1 || rank < 0 || rank >= nranks) US_FAIL(US_ERR_USAGE, "bad rank %d of %d", rank, nranks);
    if (!g_nccl.load()) US_FAIL(US_ERR_NCCL, "libnccl not found (set US_NCCL_LIB)");
    if (id_bytes != 128) US_FAIL(US_ERR_USAGE, "NCCL unique id must be 128 bytes");
    Nccl::UniqueId id;
    std::memcpy(id.internal, uid, 128);
    CUDA_OK(cudaSetDevice(c->device));
    int r = g_nccl.commInitRank(&c->nccl_comm, nranks, id, rank);
    if (r) US_FAIL(US_ERR_NCCL, "ncclCommInitRank failed: %s", g_nccl.errStr ? g_nccl.errStr(r) : "?");
    c->nranks = nranks;
    c->rank = rank;
  });
}

}  // extern "C"
