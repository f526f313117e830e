"""CPU interpreter of libunetswap *toy* programs -- TEST INFRASTRUCTURE ONLY.

It executes a ``lowering.Program`` op list with numpy, applying the same
residency rules as the CUDA engine (read of a swapped-out / freed tensor is a
use-after-swap), so the CPU test suite can check the lowering's placement
logic against the reference fixtures without a GPU.  The product path never
imports this module.
"""
import numpy as np

from paper_1812_07816_b200._native import ARENA, OP

INV = {v: k[len("US_OP_"):] for k, v in OP.items() if k.startswith("US_OP_")}


class MockUseAfterSwap(Exception):
    pass


def run_program(prog, inputs: dict):
    """inputs: staging tid -> np.ndarray.  Returns persistent buffers by tid."""
    defs = prog.by_tid()
    persist = {tid: np.zeros(d.nbytes // 8) for tid, d in defs.items() if d.storage != ARENA}
    for tid, arr in inputs.items():
        persist[tid] = np.asarray(arr, dtype=np.float64).copy()
    dev, host, state = {}, {}, {}
    stats = {"d2h": 0, "h2d": 0, "peak": 0, "cur": 0}

    def read(t):
        if defs[t].storage != ARENA:
            return persist[t]
        if state.get(t) != 1:
            raise MockUseAfterSwap(f"use-after-swap: tensor {defs[t].name!r} is "
                                   f"{ {0: 'not yet produced', 2: 'host-resident', 3: 'freed'}.get(state.get(t, 0))}")
        return dev[t]

    def write(t, arr):
        if defs[t].storage != ARENA:
            persist[t][:] = arr
            return
        if state.get(t, 0) == 0:
            stats["cur"] += defs[t].nbytes
            stats["peak"] = max(stats["peak"], stats["cur"])
        elif state[t] != 1:
            raise MockUseAfterSwap(f"write after release of {defs[t].name!r}")
        state[t] = 1
        dev[t] = arr

    def release(t, new_state):
        stats["cur"] -= defs[t].nbytes
        state[t] = new_state
        dev.pop(t, None)

    for code, tids, ia, fa in prog.ops:
        name = INV[code]
        if name in ("SLOT_BEGIN", "SLOT_END"):
            continue
        if name == "SWAP_OUT":
            host[tids[0]] = read(tids[0]).copy()
            stats["d2h"] += defs[tids[0]].nbytes
        elif name == "SWAP_RELEASE":
            if tids[0] not in host:
                raise MockUseAfterSwap("release without swap-out")
            release(tids[0], 2)
        elif name == "SWAP_IN":
            if state.get(tids[0]) != 2:
                raise MockUseAfterSwap(f"use-after-swap: swap_in of {defs[tids[0]].name!r}")
            write(tids[1], host[tids[0]].copy())
            stats["h2d"] += defs[tids[1]].nbytes
        elif name == "FREE":
            release(tids[0], 3)
        elif name == "COPY_IN":
            write(tids[1], read(tids[0]).copy())
        elif name == "CAPTURE":
            persist[tids[1]][:] = read(tids[0])
        elif name == "TOUCH":
            read(tids[0])
        elif name == "ZERO":
            write(tids[0], np.zeros(defs[tids[0]].nbytes // 8))
        elif name == "TOY_AFFINE":
            x = read(tids[0])
            n_in, n_out = ia
            a, b = fa
            if n_in >= n_out:
                reps = -(-n_in // n_out)
                pad = np.zeros(reps * n_out)
                pad[:n_in] = x
                y = a * pad.reshape(reps, n_out).sum(axis=0) + b
            else:
                y = a * np.tile(x, -(-n_out // n_in))[:n_out] + b
            write(tids[1], y)
        elif name == "TOY_AFFINE_BWD":
            dy = read(tids[0])
            n_dx, n_dy = ia
            a = fa[0]
            if n_dx >= n_dy:
                dx = (a * np.tile(dy, -(-n_dx // n_dy))[:n_dx]).copy()
            else:
                reps = -(-n_dy // n_dx)
                pad = np.zeros(reps * n_dx)
                pad[:n_dy] = dy
                dx = a * pad.reshape(reps, n_dx).sum(axis=0)
            write(tids[1], dx)
        elif name == "TOY_RELU":
            write(tids[1], np.maximum(read(tids[0]), 0.0))
        elif name == "TOY_RELU_BWD":
            write(tids[2], read(tids[0]) * (read(tids[1]) > 0.0))
        elif name == "TOY_CENTER":
            x = read(tids[0])
            write(tids[1], x - x.mean())
        elif name == "TOY_POOL":
            x = read(tids[0])
            n_out, k = ia
            write(tids[1], x[:k * n_out].reshape(n_out, k).mean(axis=1))
        elif name == "TOY_POOL_BWD":
            dy = read(tids[0])
            n_dx, k = ia
            write(tids[1], np.repeat(dy / k, k)[:n_dx])
        elif name == "TOY_COPY":
            src = read(tids[0])
            n, so, do = ia
            if defs[tids[1]].storage == ARENA and state.get(tids[1]) == 1:
                dst = dev[tids[1]].copy()
            else:
                dst = np.zeros(defs[tids[1]].nbytes // 8)
            dst[do:do + n] = src[so:so + n]
            write(tids[1], dst)
        elif name == "TOY_ADD":
            a, b = read(tids[0]), read(tids[1])
            write(tids[2], a + (b if fa[0] == 1.0 else fa[0] * b))
        elif name == "TOY_SUMSQ":
            x = read(tids[0])
            n, first, idx = ia
            acc = persist[tids[1]]
            acc[idx] = (0.0 if first else acc[idx]) + float(np.dot(x, x))
        else:
            raise AssertionError(f"mock cannot run op {name}")
    return persist, stats


# Operand roles per opcode (mirrors op_roles() in csrc/engine.cu).
ROLES = {
    "COPY_IN": "PW", "CAPTURE": "RP", "ZERO": "W", "TOUCH": "R",
    "TOY_AFFINE": "RW", "TOY_AFFINE_BWD": "RW", "TOY_RELU": "RW", "TOY_CENTER": "RW",
    "TOY_POOL": "RW", "TOY_POOL_BWD": "RW", "TOY_COPY": "RW", "TOY_RELU_BWD": "RRW",
    "TOY_ADD": "RRW", "TOY_SUMSQ": "RP", "INPUT_NCDHW": "PW", "PAD_CH": "RW",
    "CONV_FWD": "RPWWO", "BN_STATS": "RP", "NORM_ACT": "RPPwwOw", "POOL_FWD": "RW",
    "CONCAT": "ROW", "CONVT_FWD": "RPW", "LOSS_FWD": "RPPWPP", "LOSS_BWD": "RPPPWPWOOw",
    "RELU_BWD": "RRW", "BN_BWD": "RRPPPWW", "CONV_DGRAD": "RPWOOOw", "CONVT_DGRAD": "RPWOOOw",
    "CONV_WGRAD": "RRPWO", "CONVT_WGRAD": "RRPWO", "POOL_BWD": "RROWOOw", "ADAM": "PPPPP",
    "ALLREDUCE": "P", "CAST_W": "PP", "RELU_FWD": "RW", "LABELS_AUG": "PP",
}


def dry_run(prog):
    """Residency-only execution of any program: returns (peak bytes, d2h bytes, h2d bytes).
    Raises MockUseAfterSwap on a read of a non-resident tensor."""
    defs = prog.by_tid()
    state, cur, peak, d2h, h2d = {}, 0, 0, 0, 0
    for code, tids, ia, fa in prog.ops:
        name = INV[code]
        if name in ("SLOT_BEGIN", "SLOT_END"):
            continue
        if name == "SWAP_OUT":
            if state.get(tids[0]) != 1:
                raise MockUseAfterSwap(f"use-after-swap: swap_out of {defs[tids[0]].name}")
            d2h += defs[tids[0]].nbytes
            continue
        if name == "SWAP_RELEASE":
            state[tids[0]] = 2
            cur -= defs[tids[0]].nbytes
            continue
        if name == "SWAP_IN":
            if state.get(tids[0]) != 2:
                raise MockUseAfterSwap(f"use-after-swap: swap_in of {defs[tids[0]].name}")
            state[tids[1]] = 1
            cur += defs[tids[1]].nbytes
            peak = max(peak, cur)
            h2d += defs[tids[1]].nbytes
            continue
        if name == "FREE":
            if defs[tids[0]].storage == ARENA:
                if state.get(tids[0]) != 1:
                    raise MockUseAfterSwap(f"free of non-resident {defs[tids[0]].name}")
                state[tids[0]] = 3
                cur -= defs[tids[0]].nbytes
            continue
        roles = ROLES[name]
        # trailing optional operands may be left out (the engine pads them with -1)
        assert len(tids) <= len(roles) and all(r in "Ow" for r in roles[len(tids):]), \
            (name, tids)
        tids = tuple(tids) + (-1,) * (len(roles) - len(tids))
        for r, t in zip(roles, tids):
            if r in "Ow" and t < 0:
                continue
            if r == "P":
                assert defs[t].storage != ARENA, (name, defs[t].name)
            elif r in "RO" and defs[t].storage == ARENA and state.get(t) != 1:
                raise MockUseAfterSwap(f"use-after-swap: {name} read {defs[t].name} "
                                       f"(state {state.get(t, 0)})")
        for r, t in zip(roles, tids):
            if r == "w":
                if t < 0:
                    continue
                r = "W"
            if r == "W" and defs[t].storage == ARENA and state.get(t, 0) == 0:
                state[t] = 1
                cur += defs[t].nbytes
                peak = max(peak, cur)
            elif r == "W" and defs[t].storage == ARENA and state.get(t) != 1:
                raise MockUseAfterSwap(f"write to released {defs[t].name}")
    return peak, d2h, h2d
