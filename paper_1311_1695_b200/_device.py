"""Device plumbing: CUDA availability, streams, workspaces, vector buffers.

PyTorch provides device memory (the caching allocator), pinned host memory
and the current stream; every computation is a liblapb200 kernel.  Vectors on
the device are 1-D float64 torch tensors; column blocks (deflation bases,
search spaces) are 2-D tensors of shape (k, n), i.e. column-major n x k with
leading dimension n, so a column is a contiguous row of the tensor.
"""

import ctypes
import threading

import numpy as np

from . import _native as nat

_state = threading.local()
_checked = False


def torch():
    import torch as _t
    return _t


def require_cuda():
    """Fail loudly when no CUDA device is present (no CPU fallback)."""
    global _checked
    if _checked:
        return
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "paper_1311_1695_b200 needs a CUDA device (B200 / sm_100a); "
            "there is no CPU fallback")
    nat.load()
    _checked = True


def device():
    require_cuda()
    return torch().device("cuda", torch().cuda.current_device())


def stream_ptr():
    """cudaStream_t of torch's current stream (as an int for ctypes).  Inside
    solver_stream() the pointer is cached per thread: torch's
    current_stream() costs ~10 us a call, and a solve makes thousands."""
    s = getattr(_state, "stream", None)
    if s is not None:
        return s
    return torch().cuda.current_stream().cuda_stream


class Workspace:
    """An lg_ws handle (deterministic-reduction scratch) bound to a stream."""

    def __init__(self):
        require_cuda()
        h = ctypes.c_void_p()
        nat.call("lg_ws_create", ctypes.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and h.value and nat._lib is not None:
            nat._lib.lg_ws_destroy(h)


def workspace():
    """The workspace of the current stream (one per stream per thread)."""
    cache = getattr(_state, "ws", None)
    if cache is None:
        cache = _state.ws = {}
    s = stream_ptr()
    ws = cache.get(s)
    if ws is None:
        ws = cache[s] = Workspace()
    return ws


def empty(n, dtype=None):
    t = torch()
    return t.empty(n, dtype=dtype or t.float64, device=device())


def zeros(n, dtype=None):
    t = torch()
    return t.zeros(n, dtype=dtype or t.float64, device=device())


def is_device_array(x):
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def to_device(x):
    """float64 contiguous device tensor from numpy / torch input."""
    t = torch()
    if isinstance(x, t.Tensor):
        x = x.to(device=device(), dtype=t.float64)
        return x.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if not arr.flags.writeable:
        arr = arr.copy()
    return t.from_numpy(arr).to(device())


def to_host(x):
    t = torch()
    if isinstance(x, t.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x, dtype=np.float64)


def columns_to_host(rows, n):
    """Device rows (a list of 1-D tensors or a 2-D (m, n) tensor) as the
    host matrix np.column_stack(rows) -- transposed on the device, one copy."""
    t = torch()
    if isinstance(rows, (list, tuple)):
        if not rows:
            return np.zeros((n, 0))
        rows = t.stack(list(rows))
    if rows.shape[0] == 0:
        return np.zeros((n, 0))
    m = rows.t().contiguous()
    # a pinned (already mapped, cached by torch's host allocator) result
    # buffer: the copy runs at PCIe speed instead of page-faulting a fresh
    # pageable array; the numpy array keeps the buffer alive
    out = t.empty(m.shape, dtype=m.dtype, pin_memory=True)
    out.copy_(m)
    return out.numpy()


def ptr(x):
    return x.data_ptr() if x is not None else None


class Pinned:
    """Pinned host mirror of a small device array (status readbacks)."""

    def __init__(self, dev_tensor):
        t = torch()
        self.dev = dev_tensor
        self.host = t.empty(dev_tensor.shape, dtype=dev_tensor.dtype, pin_memory=True)
        self.np = self.host.numpy()
        self.nbytes = dev_tensor.numel() * dev_tensor.element_size()

    def fetch(self, stream=None):
        nat.call("lg_readback", self.dev.data_ptr(), self.host.data_ptr(),
                 self.nbytes, stream if stream is not None else stream_ptr())
        return self.np

    def push(self, stream=None):
        nat.call("lg_upload", self.dev.data_ptr(), self.host.data_ptr(),
                 self.nbytes, stream if stream is not None else stream_ptr())


class _Staging:
    __slots__ = ("n", "xd", "yd")

    def __init__(self, n):
        self.n = n
        self.xd = empty(n)
        self.yd = empty(n)


def staging(n):
    """Per-thread device buffers for host-array products of length n (reused
    across calls; the product is synchronous, so reuse is safe)."""
    cache = getattr(_state, "staging", None)
    if cache is None:
        cache = _state.staging = {}
    key = (n, torch().cuda.current_device())
    st = cache.get(key)
    if st is None:
        if len(cache) >= 4:
            cache.clear()
        st = cache[key] = _Staging(n)
    return st


class _PinnedPool:
    """Page-locked host buffers handed out as fresh numpy arrays (results of
    the host-buffer products, DMA'd into directly); a buffer goes back to the
    pool when its array is collected.  A few buffers per size are kept."""

    KEEP = 8

    def __init__(self):
        self.free = {}
        self.lock = threading.Lock()

    def array(self, n):
        import weakref
        t = torch()
        with self.lock:
            lst = self.free.get(n)
            buf = lst.pop() if lst else None
        if buf is None:
            buf = t.empty(n, dtype=t.float64, pin_memory=True)
        arr = buf.numpy()
        weakref.finalize(arr, self._give_back, n, buf)
        return arr

    def _give_back(self, n, buf):
        with self.lock:
            lst = self.free.setdefault(n, [])
            if len(lst) < self.KEEP:
                lst.append(buf)


_pinned_pool = _PinnedPool()


def pinned_array(n):
    """A fresh float64 numpy array of length n in page-locked memory."""
    return _pinned_pool.array(n)


_solver_streams = {}


def solver_stream():
    """Context manager running device work on a dedicated (capturable)
    stream of the current device, ordered after the caller's stream."""
    t = torch()
    d = t.cuda.current_device()
    key = (d, threading.get_ident())     # one per thread (simulated ranks)
    s = _solver_streams.get(key)
    if s is None:
        s = _solver_streams[key] = t.cuda.Stream(device=d)
    s.wait_stream(t.cuda.current_stream())
    return _StreamCtx(t, s)


class _StreamCtx:
    def __init__(self, t, s):
        self.t, self.s = t, s
        self.prev = None

    def __enter__(self):
        self.cm = self.t.cuda.stream(self.s)
        self.cm.__enter__()
        self.prev = getattr(_state, "stream", None)
        _state.stream = self.s.cuda_stream
        return self.s

    def __exit__(self, *exc):
        _state.stream = self.prev
        self.cm.__exit__(*exc)
        self.t.cuda.current_stream().wait_stream(self.s)
