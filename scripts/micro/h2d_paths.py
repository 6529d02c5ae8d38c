"""Host<->device copy paths for the public numpy spmv (dev aid): what an
8 MB x in / 8 MB y out costs through each route."""
import time

import numpy as np
import torch

n = 989777
x = np.random.default_rng(0).standard_normal(n)
xd = torch.empty(n, dtype=torch.float64, device="cuda")
yd = torch.randn(n, dtype=torch.float64, device="cuda")
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
s = torch.cuda.Stream()


def t(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


print("threads", torch.get_num_threads())
print("A pageable H2D (from_numpy.to)      %7.1f us" % t(lambda: xd.copy_(torch.from_numpy(x))))
print("B memcpy->pinned + H2D              %7.1f us" % t(lambda: (pin.copy_(torch.from_numpy(x)), xd.copy_(pin, non_blocking=True))))
print("  memcpy numpy->pinned only         %7.1f us" % t(lambda: pin.copy_(torch.from_numpy(x))))
print("  H2D pinned only                   %7.1f us" % t(lambda: xd.copy_(pin, non_blocking=True)))


def chunked(k=8):
    c = (n + k - 1) // k
    xt = torch.from_numpy(x)
    for i in range(k):
        sl = slice(i * c, min(n, (i + 1) * c))
        pin[sl].copy_(xt[sl])
        xd[sl].copy_(pin[sl], non_blocking=True)


print("C chunked memcpy/H2D pipeline (8)   %7.1f us" % t(chunked))
print("D D2H to fresh pageable (cpu())     %7.1f us" % t(lambda: yd.cpu().numpy()))
print("E D2H to fresh pinned (cached)      %7.1f us" % t(lambda: torch.empty(n, dtype=torch.float64, pin_memory=True).copy_(yd, non_blocking=True)))
cr = torch.cuda.cudart()


def reg():
    ptr = x.ctypes.data
    cr.cudaHostRegister(ptr, x.nbytes, 0)
    xd.copy_(torch.from_numpy(x), non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(ptr)


print("F register + H2D + unregister       %7.1f us" % t(reg))
