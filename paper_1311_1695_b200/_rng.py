"""Start / restart vectors drawn exactly as the reference draws them, with
the next draw prepared off the critical path.

The reference solvers draw every random vector as rng.standard_normal(n)
from one numpy Generator, in a fixed order (dacg.py:161,203; jd.py:112,144;
irlm.py:236,250).  Iteration counts only match the reference if the same
numbers arrive in the same order, so the stream is kept; what changes is
when the next vector is computed: a worker thread draws it from a copy of
the generator state while the device iterates (numpy fills the array with
the GIL released), and the caller's generator is advanced to the state after
that draw when the vector is taken.  Any other use of the generator in
between must call `invalidate()` first, which discards the prepared vector.
"""

import concurrent.futures as cf

import numpy as np

_pool = None


def _executor():
    global _pool
    if _pool is None:
        _pool = cf.ThreadPoolExecutor(max_workers=1, thread_name_prefix="lapb200-rng")
    return _pool


def _draw(state, n):
    g = np.random.Generator(np.random.PCG64())
    g.bit_generator.state = state
    v = g.standard_normal(n)
    return v, g.bit_generator.state


class NormalStream:
    """rng.standard_normal(n), one vector at a time, prefetched."""

    def __init__(self, rng, n):
        self.rng = rng
        self.n = int(n)
        self._fut = None
        self._ok = isinstance(rng.bit_generator, np.random.PCG64)
        self._prefetch()

    def invalidate(self):
        self._fut = None

    def draw(self):
        fut, self._fut = self._fut, None
        if fut is not None:
            v, state = fut.result()
            self.rng.bit_generator.state = state
        else:
            v = self.rng.standard_normal(self.n)
        self._prefetch()
        return v

    def _prefetch(self):
        if self._ok and self.n >= 1 << 16:
            self._fut = _executor().submit(_draw, self.rng.bit_generator.state, self.n)
