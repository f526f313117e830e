"""Does the host page size of the pinned swap pool change the PCIe copy rates?  torch's
cudaHostAlloc buffers vs mmap + MADV_HUGEPAGE + cudaHostRegister, each direction alone and
both at once (1 GiB per copy, best of 3)."""
import json
import mmap
import time

import torch

n = 1 << 30
cudart = torch.cuda.cudart()


def hugepage_pinned():
    m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    t = torch.frombuffer(m, dtype=torch.uint8)
    t.fill_(1)   # fault the pages in (huge where the kernel grants them)
    err = cudart.cudaHostRegister(t.data_ptr(), n, 0)
    assert int(err) == 0, err
    return m, t


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
out = {}
try:
    thp = open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
except OSError:
    thp = "?"
out["thp"] = thp
bufs = {"cudaHostAlloc": (None, torch.empty(n, dtype=torch.uint8, pin_memory=True),
                          torch.empty(n, dtype=torch.uint8, pin_memory=True))}
m1, h1 = hugepage_pinned()
m2, h2 = hugepage_pinned()
bufs["mmap+hugepage+register"] = (None, h1, h2)
for name, (_, ha, hb) in bufs.items():
    def d2h():
        with torch.cuda.stream(s1):
            ha.copy_(d1, non_blocking=True)

    def h2d():
        with torch.cuda.stream(s2):
            d2.copy_(hb, non_blocking=True)
    r = {"pinned": bool(ha.is_pinned()),
         "d2h": n / timed(d2h) / 1e9, "h2d": n / timed(h2d) / 1e9,
         "duplex_per_dir": n / timed(lambda: (d2h(), h2d())) / 1e9}
    out[name] = r
try:
    out["AnonHugePages"] = [l for l in open("/proc/meminfo") if "AnonHugePages" in l][0].strip()
except OSError:
    pass
print(json.dumps(out))
