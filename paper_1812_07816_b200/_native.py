"""ctypes binding of libunetswap.so (include/unetswap.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_1812_07816_b200/csrc``).  There is deliberately no fallback: if the
shared object is missing or no CUDA device is present, ``Engine`` raises.
Opcode numbers are parsed from ``csrc/opcodes.h`` so host and device can
never disagree.
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libunetswap.so")
_OPCODES_H = os.path.join(_HERE, "csrc", "opcodes.h")


def _parse_defines(path: str) -> dict:
    out = {}
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            m = re.match(r"\s*#define\s+(US_\w+)\s+(-?\d+)", line)
            if m:
                out[m.group(1)] = int(m.group(2))
    return out


OP = _parse_defines(_OPCODES_H)
_H = _parse_defines(os.path.join(_HERE, "..", "include", "unetswap.h")) \
    if os.path.exists(os.path.join(_HERE, "..", "include", "unetswap.h")) else {}

US_OK, US_ERR_DOMAIN, US_ERR_USAGE, US_ERR_CUDA, US_ERR_NCCL = 0, 1, 2, 3, 4
ARENA, PERSIST = 0, 1
DT_F64, DT_F32, DT_BF16, DT_U8 = 0, 1, 2, 3
CH_COMPUTE, CH_D2H, CH_H2D, CH_STALL, CH_OP = 0, 1, 2, 3, 4
FLAG_OP_TIMES = 1
FLAG_GRAPH = 2
FLAG_NO_TIMELINE = 4
FLAG_POISON = 8
ALGO_DIRECT = OP["US_ALGO_DIRECT"]
ALGO_TCGEN05 = OP["US_ALGO_TCGEN05"]
ALGO_IM2COL = OP["US_ALGO_IM2COL"]


class EngineError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class us_event(ctypes.Structure):
    _fields_ = [("node", ctypes.c_int32), ("channel", ctypes.c_int32),
                ("start_s", ctypes.c_double), ("end_s", ctypes.c_double)]


class us_stats(ctypes.Structure):
    _fields_ = [("arena_bytes", ctypes.c_uint64), ("arena_peak_bytes", ctypes.c_uint64),
                ("persistent_bytes", ctypes.c_uint64), ("host_pool_bytes", ctypes.c_uint64),
                ("d2h_bytes", ctypes.c_uint64), ("h2d_bytes", ctypes.c_uint64),
                ("step_s", ctypes.c_double), ("stall_s", ctypes.c_double),
                ("kernels", ctypes.c_int32), ("events", ctypes.c_int32),
                ("host_enqueue_s", ctypes.c_double), ("host_numa_node", ctypes.c_int32),
                ("dp_nranks", ctypes.c_int32)]


_lib = None


def load_library() -> ctypes.CDLL:
    """Load the CUDA library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EngineError(US_ERR_USAGE, f"{LIB_PATH} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, U64, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32
    sig = {
        "us_last_error": (ctypes.c_char_p, []),
        "us_abi_version": (ctypes.c_int, []),
        "us_ctx_create": (ctypes.c_int, [I32, U64, U32, ctypes.POINTER(P)]),
        "us_ctx_destroy": (ctypes.c_int, [P]),
        "us_set_flags": (ctypes.c_int, [P, U32]),
        "us_prog_reset": (ctypes.c_int, [P]),
        "us_tensor": (ctypes.c_int, [P, I32, U64, I32, I32, ctypes.c_char_p]),
        "us_slot_name": (ctypes.c_int, [P, I32, ctypes.c_char_p]),
        "us_tensor_place": (ctypes.c_int, [P, I32, U64]),
        "us_op": (ctypes.c_int, [P, I32, ctypes.POINTER(I32), I32, ctypes.POINTER(ctypes.c_int64),
                                 I32, ctypes.POINTER(ctypes.c_double), I32]),
        "us_prog_finalize": (ctypes.c_int, [P]),
        "us_op_set_farg": (ctypes.c_int, [P, I32, I32, ctypes.c_double]),
        "us_upload": (ctypes.c_int, [P, I32, P, U64, U64]),
        "us_download": (ctypes.c_int, [P, I32, P, U64, U64]),
        "us_tensor_ptr": (ctypes.c_int, [P, I32, ctypes.POINTER(P)]),
        "us_workspace_bytes": (ctypes.c_int, [I32, ctypes.POINTER(ctypes.c_int64), I32,
                                              ctypes.POINTER(U64)]),
        "us_run": (ctypes.c_int, [P]),
        "us_sync": (ctypes.c_int, [P]),
        "us_mark": (ctypes.c_int, [P, I32]),
        "us_elapsed": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_double)]),
        "us_stats_get": (ctypes.c_int, [P, ctypes.POINTER(us_stats)]),
        "us_timeline": (ctypes.c_int, [P, ctypes.POINTER(us_event), I32, ctypes.POINTER(I32)]),
        "us_dp_unique_id": (ctypes.c_int, [P, I32, ctypes.POINTER(I32)]),
        "us_dp_init": (ctypes.c_int, [P, P, I32, I32, I32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    """Names declared in include/unetswap.h (the C ABI surface)."""
    hdr = os.path.join(_HERE, "..", "include", "unetswap.h")
    with open(hdr, encoding="utf-8") as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(us_\w+)\s*\(", text)))


def _check(rc: int):
    if rc != US_OK:
        msg = load_library().us_last_error().decode(errors="replace")
        raise EngineError(rc, msg)


def workspace_bytes(opcode: int, iargs) -> int:
    lib = load_library()
    arr = (ctypes.c_int64 * len(iargs))(*[int(v) for v in iargs])
    out = ctypes.c_uint64(0)
    _check(lib.us_workspace_bytes(opcode, arr, len(iargs), ctypes.byref(out)))
    return int(out.value)


class Engine:
    """One libunetswap context (one GPU, one program at a time)."""

    def __init__(self, device: int = 0, arena_bytes: int = 0, flags: int = 0):
        self.lib = load_library()
        self.ctx = ctypes.c_void_p()
        self.flags = int(flags)
        _check(self.lib.us_ctx_create(device, int(arena_bytes), self.flags,
                                      ctypes.byref(self.ctx)))
        self.arena_bytes = int(arena_bytes)
        self.device = device

    def set_flags(self, flags: int):
        """US_FLAG_OP_TIMES: bracket every compute op with events (channel CH_OP);
        US_FLAG_GRAPH: capture the step as a CUDA graph and replay it."""
        _check(self.lib.us_set_flags(self.ctx, int(flags)))
        self.flags = int(flags)

    def close(self):
        if self.ctx:
            _check(self.lib.us_ctx_destroy(self.ctx))
            self.ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- program ---------------------------------------------------------
    def reset(self):
        _check(self.lib.us_prog_reset(self.ctx))

    def tensor(self, tid: int, nbytes: int, storage: int, dtype: int, name: str = ""):
        _check(self.lib.us_tensor(self.ctx, tid, int(nbytes), storage, dtype, name.encode()))

    def place(self, tid: int, offset: int):
        _check(self.lib.us_tensor_place(self.ctx, tid, int(offset)))

    def slot_name(self, slot: int, name: str):
        _check(self.lib.us_slot_name(self.ctx, slot, name.encode()))

    def op(self, opcode: int, tensors=(), iargs=(), fargs=()):
        t = (ctypes.c_int32 * max(1, len(tensors)))(*tensors)
        i = (ctypes.c_int64 * max(1, len(iargs)))(*[int(v) for v in iargs])
        f = (ctypes.c_double * max(1, len(fargs)))(*[float(v) for v in fargs])
        _check(self.lib.us_op(self.ctx, opcode, t, len(tensors), i, len(iargs), f, len(fargs)))

    def finalize(self):
        _check(self.lib.us_prog_finalize(self.ctx))

    def set_farg(self, op_index: int, k: int, value: float):
        _check(self.lib.us_op_set_farg(self.ctx, op_index, k, float(value)))

    # -- data ------------------------------------------------------------
    def upload(self, tid: int, arr: np.ndarray, offset: int = 0):
        a = np.ascontiguousarray(arr)
        _check(self.lib.us_upload(self.ctx, tid, a.ctypes.data, a.nbytes, offset))

    def upload_ptr(self, tid: int, ptr: int, nbytes: int, offset: int = 0):
        _check(self.lib.us_upload(self.ctx, tid, ctypes.c_void_p(ptr), nbytes, offset))

    def download(self, tid: int, nbytes: int, dtype, offset: int = 0) -> np.ndarray:
        out = np.empty(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
        _check(self.lib.us_download(self.ctx, tid, out.ctypes.data, out.nbytes, offset))
        return out

    def download_ptr(self, tid: int, ptr: int, nbytes: int, offset: int = 0):
        _check(self.lib.us_download(self.ctx, tid, ctypes.c_void_p(ptr), nbytes, offset))

    def tensor_ptr(self, tid: int) -> int:
        p = ctypes.c_void_p()
        _check(self.lib.us_tensor_ptr(self.ctx, tid, ctypes.byref(p)))
        return int(p.value or 0)

    # -- execution -------------------------------------------------------
    def run(self):
        _check(self.lib.us_run(self.ctx))

    def sync(self):
        _check(self.lib.us_sync(self.ctx))

    def mark(self, which: int):
        _check(self.lib.us_mark(self.ctx, which))

    def elapsed(self) -> float:
        s = ctypes.c_double(0)
        _check(self.lib.us_elapsed(self.ctx, ctypes.byref(s)))
        return s.value

    def stats(self) -> dict:
        st = us_stats()
        _check(self.lib.us_stats_get(self.ctx, ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in us_stats._fields_}

    def timeline(self) -> list[tuple[int, int, float, float]]:
        n = ctypes.c_int32(0)
        _check(self.lib.us_timeline(self.ctx, None, 0, ctypes.byref(n)))
        buf = (us_event * max(1, n.value))()
        _check(self.lib.us_timeline(self.ctx, buf, n.value, ctypes.byref(n)))
        return [(e.node, e.channel, e.start_s, e.end_s) for e in buf[:n.value]]

    # -- data parallel ---------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = load_library()
        buf = ctypes.create_string_buffer(128)
        n = ctypes.c_int32(0)
        _check(lib.us_dp_unique_id(buf, 128, ctypes.byref(n)))
        return buf.raw[:n.value]

    def dp_init(self, uid: bytes, nranks: int, rank: int):
        buf = ctypes.create_string_buffer(uid, len(uid))
        _check(self.lib.us_dp_init(self.ctx, buf, len(uid), nranks, rank))
