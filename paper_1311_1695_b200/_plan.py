"""Prebuilt device launches: fused vector passes, scalar programs, SpMV,
IC(0) apply.

A solver iteration is a fixed sequence of launches whose operands are fixed
device buffers and whose scalar coefficients live in a device slot file, so
each launch's argument block is built once (ctypes structs) and replayed;
the Python cost of an iteration is one ctypes call per launch.

    Slots     named double slots + int flags in device memory
    Prog      assembler for the device scalar interpreter (csrc/lg_scalar.cu)
    Fused     one lg_fused pass
    Spmv      one lg_spmv launch (optionally with epilogue dots)
    Ic0Apply  one lg_ic0_apply (or Jacobi) launch
"""

import ctypes
import struct

import numpy as np

from . import _device as dev
from . import _native as nat

OPS = {
    "NOP": 0, "MOV": 1, "IMM": 2, "ADD": 3, "SUB": 4, "MUL": 5, "DIV": 6,
    "SQRT": 7, "NEG": 8, "HYPOT": 9, "ABS": 10, "MAX": 11, "MIN": 12,
    "LE": 13, "LT": 14, "EQ": 15, "SEL": 16, "AND": 17, "OR": 18, "NOT": 19,
    "FLAG": 20, "FLAGOR": 21, "LDFLAG": 22, "HALTIF": 23, "DIVZ": 24,
    "INC": 25, "RECIP": 26, "NE": 27, "GT": 28, "GE": 29,
}


def _addr(x):
    """Integer device address of a tensor / sentinel / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


class Slots:
    """Named scalar slots (device doubles) and flags (device int32)."""

    NSLOT = 256     # addressable by the scalar interpreter (uint8 indices)
    NFLAG = 32

    def __init__(self, names=(), flags=(), capacity=1024):
        t = dev.torch()
        self.cap = max(capacity, self.NSLOT)
        # one device buffer: [flags (int32) | slots (double)] so a status
        # readback is a single copy + synchronisation
        self.buf = dev.zeros(4 * self.NFLAG + 8 * self.cap, dtype=t.uint8)
        self.f = self.buf[:4 * self.NFLAG].view(t.int32)
        self.s = self.buf[4 * self.NFLAG:].view(t.float64)
        self.idx = {}
        self.fidx = {}
        for nm in names:
            self.add(nm)
        for nm in flags:
            self.add_flag(nm)
        self.pin = dev.Pinned(self.buf)
        self._hf = self.pin.host[:4 * self.NFLAG].view(t.int32).numpy()
        self._hs = self.pin.host[4 * self.NFLAG:].view(t.float64).numpy()

    def add(self, name, count=1):
        """Allocate `count` consecutive slots under `name` (idempotent)."""
        if name in self.idx:
            return self.idx[name]
        base = getattr(self, "_next", 0)
        if base + count > self.cap:
            raise ValueError("scalar slot file exhausted")
        self.idx[name] = base
        self._next = base + count
        return base

    def add_flag(self, name):
        if name not in self.fidx:
            if len(self.fidx) >= self.NFLAG:
                raise ValueError("flag file exhausted")
            self.fidx[name] = len(self.fidx)
        return self.fidx[name]

    def p(self, name, off=0):
        """Device address of slot `name` (+ offset)."""
        return self.s.data_ptr() + 8 * (self.idx[name] + off)

    def fp(self, name):
        return self.f.data_ptr() + 4 * self.fidx[name]

    # host access (synchronising)
    def fetch(self):
        """(slots, flags) as host arrays after one copy + sync."""
        self.pin.fetch(dev.stream_ptr())
        return self._hs, self._hf

    def read(self, *names):
        s, _ = self.fetch()
        return [float(s[self.idx[n]]) for n in names]

    def set(self, **values):
        """Write slots from the host (synchronous small upload)."""
        for k, v in values.items():
            self.s[self.idx[k]] = float(v)

    def set_vec(self, name, values):
        i = self.idx[name]
        vals = np.asarray(values, dtype=np.float64)
        self.s[i:i + vals.size] = dev.torch().from_numpy(vals).to(self.s.device)

    def clear_flags(self):
        self.f.zero_()

    def setflag(self, name, value):
        self.f[self.fidx[name]] = int(value)


class Prog:
    """Assembler for a device scalar program."""

    def __init__(self, slots, skip=None):
        self.S = slots
        self.ops = []
        self.imm = []
        self.skip = skip
        self._built = None

    def _s(self, name):
        if isinstance(name, int):
            return name
        if name not in self.S.idx:
            self.S.add(name)
        i = self.S.idx[name]
        if i >= Slots.NSLOT:
            raise ValueError(f"slot {name!r} is beyond the interpreter's 256-slot window")
        return i

    def emit(self, op, dst=0, a=0, b=0):
        self.ops.append(OPS[op] | (dst << 8) | (a << 16) | (b << 24))
        self._built = None
        return self

    def const(self, dst, value):
        if len(self.imm) >= nat.LG_MAXIMM:
            raise ValueError("too many immediates")
        self.imm.append(float(value))
        return self.emit("IMM", self._s(dst), len(self.imm) - 1)

    def __getattr__(self, opname):
        up = opname.upper()
        if up not in OPS:
            raise AttributeError(opname)

        def f(dst, a=0, b=0):
            if up in ("FLAG", "FLAGOR"):
                return self.emit(up, self.S.fidx[dst], self._s(a))
            if up == "LDFLAG":
                return self.emit(up, self._s(dst), self.S.fidx[a])
            if up == "HALTIF":
                return self.emit(up, 0, self._s(dst))
            return self.emit(up, self._s(dst), self._s(a), self._s(b) if b != 0 else 0)

        return f

    def build(self):
        if len(self.ops) > nat.LG_MAXOPS:
            raise ValueError("scalar program too long")
        ops = (ctypes.c_uint32 * max(1, len(self.ops)))(*self.ops)
        imm = (ctypes.c_double * max(1, len(self.imm)))(*self.imm)
        skip = self.S.fp(self.skip) if self.skip else None
        self._built = (self.S.s.data_ptr(), self.S.f.data_ptr(), ctypes.cast(ops, ctypes.c_void_p),
                       len(self.ops), ctypes.cast(imm, ctypes.c_void_p), len(self.imm), skip,
                       ops, imm)
        return self

    def __call__(self, stream=None):
        if self._built is None:
            self.build()
        b = self._built
        nat.check(nat.load().lg_scalar_prog(b[0], b[1], b[2], b[3], b[4], b[5], b[6],
                                            stream if stream is not None else dev.stream_ptr()),
                  "lg_scalar_prog")


class Fused:
    """One fused streaming pass (lg_fused), built once and replayed.

    outs:   list of dicts {out, terms: [(vec, h, dslot)], upd: (Q, k, cptr, cscale),
                           post: (dptr, mode)}
    dots:   list of (a, b, c) -> (a - c) . b   (b None: a . a)
    blocks: list of (Q, k, vec) -> Q[:, :k]^T vec
    Q is a (kcap, n) tensor (column-major n x kcap) or (address, ld) tuple.
    """

    def __init__(self, n, outs=(), dots=(), blocks=(), result=None, skip=None, prog=None):
        a = nat.FusedArgs()
        a.n = n
        self._keep = []
        for k, o in enumerate(outs):
            if o is None:
                continue
            oa = a.o[k]
            oa.out = _addr(o["out"])
            terms = o.get("terms", ())
            if len(terms) > nat.LG_MAXT:
                raise ValueError("too many terms")
            oa.nterms = len(terms)
            for t, term in enumerate(terms):
                v, h = term[0], term[1]
                d = term[2] if len(term) > 2 else None
                oa.t[t].v = _addr(v)
                oa.t[t].h = float(h)
                oa.t[t].d = d
            upd = o.get("upd")
            if upd is not None:
                q, kk, cptr = upd[0], upd[1], upd[2]
                cs = upd[3] if len(upd) > 3 else 1.0
                qa, ld = self._qaddr(q)
                oa.uq, oa.uld, oa.uk, oa.uc, oa.cscale = qa, ld, int(kk), cptr, float(cs)
            upd2 = o.get("upd2")
            if upd2 is not None:
                qa, ld = self._qaddr(upd2[0])
                oa.uq2, oa.uld2, oa.uk2, oa.uc2 = qa, ld, int(upd2[1]), upd2[2]
                if upd is None:
                    oa.cscale = float(upd2[3]) if len(upd2) > 3 else 1.0
            post = o.get("post")
            if post is not None:
                oa.d_post, oa.post_mode = post[0], int(post[1])
        if len(dots) > nat.LG_MAXD:
            raise ValueError("too many dots")
        a.ndots = len(dots)
        for d, dot in enumerate(dots):
            x = dot[0]
            y = dot[1] if len(dot) > 1 else None
            c = dot[2] if len(dot) > 2 else None
            a.da[d] = _addr(x)
            a.db[d] = _addr(y)
            a.dc[d] = _addr(c)
        a.nblocks = len(blocks)
        for b, blk in enumerate(blocks):
            q, kk, v = blk
            qa, ld = self._qaddr(q)
            a.b[b].q, a.b[b].ld, a.b[b].k, a.b[b].v = qa, ld, int(kk), _addr(v)
        a.result = _addr(result)
        a.skip = skip
        self.args = a
        self.argp = ctypes.byref(a)
        self.nres = len(dots) + sum(int(b[1]) for b in blocks)
        # a scalar program run by the pass's finishing CTA (its own skip flag
        # must be the pass's: one predicate covers both)
        self.prog = None
        if prog is not None:
            if not dots and not blocks:
                raise ValueError("a folded program needs a pass with dot products")
            pskip = prog.S.fp(prog.skip) if prog.skip else None
            if pskip != skip:
                raise ValueError("folded program and pass must share the skip flag")
            self.prog = prog.build()

    @staticmethod
    def _qaddr(q):
        if isinstance(q, tuple):
            return q[0], q[1]
        return q.data_ptr(), q.shape[-1]

    def set_k(self, block=None, upd=None, upd2=None):
        """Change the live column count of a block dot / update (e.g. after a
        deflation basis grew) without rebuilding."""
        if block is not None:
            bi, k = block
            self.args.b[bi].k = int(k)
        if upd is not None:
            oi, k = upd
            self.args.o[oi].uk = int(k)
        if upd2 is not None:
            oi, k = upd2
            self.args.o[oi].uk2 = int(k)
        self.nres = self.args.ndots + sum(self.args.b[i].k for i in range(self.args.nblocks))

    def __call__(self, ws=None, stream=None):
        ws = ws or dev.workspace()
        st = stream if stream is not None else dev.stream_ptr()
        if self.prog is None:
            nat.check(nat.load().lg_fused(self.argp, ws.handle, st), "lg_fused")
            return
        b = self.prog._built
        nat.check(nat.load().lg_fused_prog(self.argp, b[0], b[1], b[2], b[3], b[4], b[5],
                                           ws.handle, st), "lg_fused_prog")


class Spmv:
    """One lg_spmv launch: y = A x - theta x (+ epilogue dots into result)."""

    def __init__(self, csr, x, y, theta=0.0, theta_d=None, theta_neg=False, dots=(),
                 q=None, nq=0, result=None, skip=None):
        self.csr = csr
        self.h = csr.handle
        self.x, self.y = _addr(x), _addr(y)
        self.theta = float(theta)
        self.theta_d = theta_d
        self.neg = 1 if theta_neg else 0
        self.nd = len(dots)
        self.dv = (ctypes.c_void_p * max(1, len(dots)))(*[_addr(d) for d in dots])
        if q is not None:
            self.q, self.ldq = Fused._qaddr(q)
        else:
            self.q, self.ldq = None, 0
        self.nq = int(nq)
        self.result = _addr(result)
        self.skip = skip

    def __call__(self, ws=None, stream=None):
        ws = ws or dev.workspace()
        nat.check(nat.load().lg_spmv(self.h, self.x, self.y, self.theta, self.theta_d, self.neg,
                                     self.nd, self.dv, self.q, self.ldq, self.nq, self.result,
                                     ws.handle, self.skip,
                                     stream if stream is not None else dev.stream_ptr()),
                  "lg_spmv")


class PrecApply:
    """z = M^{-1} r for the device preconditioner of an Ic0Factor."""

    def __init__(self, dfac, r, z, skip=None):
        self.d = dfac
        self.r, self.z = _addr(r), _addr(z)
        self.skip = skip

    def __call__(self, ws=None, stream=None):
        self.d.apply_raw(self.r, self.z, self.skip,
                         stream if stream is not None else dev.stream_ptr())


def _graph_note(msg):
    import os
    import sys
    if os.environ.get("LG_DEBUG"):
        print(f"[lapb200] {msg}", file=sys.stderr)


class Graph:
    """A fixed launch sequence captured into a CUDA graph and replayed.

    Capture requires a non-legacy stream: solvers run inside
    `with dev.solver_stream():`.  Every launch object must be replay-safe
    (fixed buffers, coefficients read from device slots).  If capture fails
    (e.g. a launch type the driver cannot capture) the sequence is replayed
    eagerly instead -- same kernels, more host overhead.
    """

    captured = 0     # graphs captured / capture failures (process-wide, for tests)
    failed = 0

    def __init__(self, fns):
        self.fns = list(fns)
        self.exec = None
        self.stream = None
        self.eager = False
        self.calls = 0

    def _capture(self, stream):
        lib = nat.load()
        h = ctypes.c_void_p()
        rc = lib.lg_capture_begin(stream)
        if rc != 0:
            self.eager = True
            Graph.failed += 1
            _graph_note("capture begin failed: " + nat.last_error())
            return
        try:
            for f in self.fns:
                f(stream=stream)
        except Exception as exc:   # a launch refused under capture (e.g. a collective)
            _graph_note(f"capture raised {exc!r}")
        finally:
            rc = lib.lg_capture_end(stream, ctypes.byref(h))
        if rc != 0:
            self.eager = True
            Graph.failed += 1
            _graph_note("capture failed, replaying eagerly: " + nat.last_error())
            return
        self.exec = h
        self.stream = stream
        Graph.captured += 1

    def __call__(self, stream=None):
        stream = stream if stream is not None else dev.stream_ptr()
        self.calls += 1
        # the first replay runs eagerly (lazy scratch allocations happen
        # outside capture); the second captures
        if not stream or self.eager or self.calls == 1:
            for f in self.fns:
                f(stream=stream)
            return
        if self.exec is None or self.stream != stream:
            self.release()
            self._capture(stream)
            if self.eager:
                for f in self.fns:
                    f(stream=stream)
                return
        nat.check(nat.load().lg_graph_launch(self.exec, stream), "lg_graph_launch")

    def release(self):
        if self.exec is not None and nat._lib is not None:
            nat._lib.lg_graph_destroy(self.exec)
        self.exec = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Execution context: the whole vector on one GPU, or one rank's row slice.


class AllReduce:
    """Sum a slot range over the ranks (dot-product partials of a pass)."""

    def __init__(self, comm, result, count):
        self.comm = comm
        self.result = result
        self.count = count      # int or a callable (live count after set_k)

    def __call__(self, ws=None, stream=None):
        c = self.count() if callable(self.count) else self.count
        if c:
            self.comm.allreduce_(self.result[:c])


class Exchange:
    """Complete a full-length vector from every rank's slice, in place."""

    def __init__(self, comm, x):
        self.comm, self.x = comm, x

    def __call__(self, ws=None, stream=None):
        self.comm.exchange_(self.x)


class ExchangeStart:
    """Issue the slice exchange of x (completed by the paired ExchangeWait);
    work launched in between overlaps the transfer."""

    def __init__(self, comm, x):
        self.comm, self.x, self.reqs = comm, x, None

    def __call__(self, ws=None, stream=None):
        self.reqs = self.comm.exchange_start(self.x)


class ExchangeWait:
    def __init__(self, start):
        self.start = start

    def __call__(self, ws=None, stream=None):
        self.start.comm.exchange_wait(self.start.reqs)
        self.start.reqs = None


class SplitOp:
    """A rank's row block as interior (own columns + diagonal) and exterior
    (every other column) halves (dist.RowComm.solver_operator)."""

    def __init__(self, inner, outer):
        self.inner, self.outer = inner, outer
        self.n = inner.n


class SpmvAcc:
    """y += A x (lg_spmv_acc): the exterior half of a split row block."""

    def __init__(self, csr, x, y, skip=None):
        self.h = csr.handle
        self.x, self.y = _addr(x), _addr(y)
        self.skip = skip

    def __call__(self, ws=None, stream=None):
        ws = ws or dev.workspace()
        nat.check(nat.load().lg_spmv_acc(self.h, self.x, self.y, ws.handle, self.skip,
                                         stream if stream is not None else dev.stream_ptr()),
                  "lg_spmv_acc")


class Seq:
    """Launches run in order (one plan entry of a row-partitioned solver)."""

    def __init__(self, steps):
        self.steps = [s for s in steps if s is not None]
        self.fused = next((s for s in self.steps if isinstance(s, Fused)), None)

    def set_k(self, **kw):
        self.fused.set_k(**kw)

    @property
    def nres(self):
        return self.fused.nres

    def __call__(self, ws=None, stream=None):
        for s in self.steps:
            s(stream=stream)


class Ctx:
    """Where a solver's n-vector work runs.

    comm None: every pass covers the whole vector (one GPU) and a scalar
    program folds into the finishing CTA of the pass it reads.
    comm given (dist.RowComm): passes cover this rank's rows [r0, r1) of the
    same full-length buffers, their dot partials are all-reduced before the
    program (then a launch of its own), and an SpMV first completes its input
    from the other ranks' slices and multiplies the rank's row block.
    """

    def __init__(self, n, comm=None):
        self.n = n
        self.comm = comm if (comm is not None and (comm.world > 1 or
                                                    getattr(comm, "force_dist", False))) else None
        self.lo = self.comm.r0 if self.comm else 0
        self.nl = self.comm.nl if self.comm else n

    @property
    def dist(self):
        return self.comm is not None

    @property
    def eager(self):
        """Launch sequences with collectives that cannot be captured."""
        return self.comm is not None and not self.comm.graph_safe

    def v(self, t):
        """A vector operand restricted to this rank's rows (a tensor, or a raw
        device address; small ints are references to a pass's own outputs)."""
        if self.comm is None or t is None:
            return t
        if isinstance(t, int):
            return t if t < 16 else t + 8 * self.lo
        return t[self.lo:self.lo + self.nl]

    def q(self, c):
        """A column block (k, n) restricted to this rank's rows."""
        if self.comm is None or c is None:
            return c
        if isinstance(c, tuple):
            return (c[0] + 8 * self.lo, c[1])
        return (c.data_ptr() + 8 * self.lo, c.shape[-1])

    def fused(self, outs=(), dots=(), blocks=(), result=None, skip=None, prog=None):
        if self.comm is None:
            return Fused(self.n, outs=outs, dots=dots, blocks=blocks, result=result,
                         skip=skip, prog=prog)
        o2 = []
        for o in outs:
            if o is None:
                o2.append(None)
                continue
            d = dict(o)
            d["out"] = self.v(o["out"])
            d["terms"] = [(self.v(t[0]),) + tuple(t[1:]) for t in o.get("terms", ())]
            for key in ("upd", "upd2"):
                if o.get(key) is not None:
                    u = o[key]
                    d[key] = (self.q(u[0]),) + tuple(u[1:])
            o2.append(d)
        d2 = [tuple(self.v(x) for x in dt) for dt in dots]
        b2 = [(self.q(b[0]), b[1], self.v(b[2])) for b in blocks]
        f = Fused(self.nl, outs=o2, dots=d2, blocks=b2, result=result, skip=skip)
        steps = [f]
        if result is not None and (dots or blocks):
            steps.append(AllReduce(self.comm, result, lambda: f.nres))
        if prog is not None:
            steps.append(prog.build() if prog._built is None else prog)
        return Seq(steps)

    def spmv(self, csr, x, y, theta=0.0, theta_d=None, theta_neg=False, dots=(), q=None,
             nq=0, result=None, skip=None):
        if self.comm is None:
            return Spmv(csr, x, y, theta=theta, theta_d=theta_d, theta_neg=theta_neg,
                        dots=dots, q=q, nq=nq, result=result, skip=skip)
        if isinstance(csr, SplitOp):
            # the interior product (own slice of x, diagonal, theta shift)
            # overlaps the exchange; the exterior product accumulates after it
            st = ExchangeStart(self.comm, x)
            steps = [st,
                     Spmv(csr.inner, x, y, theta=theta, theta_d=theta_d, theta_neg=theta_neg,
                          skip=skip),
                     ExchangeWait(st),
                     SpmvAcc(csr.outer, x, y, skip=skip)]
        else:
            steps = [Exchange(self.comm, x),
                     Spmv(csr, x, y, theta=theta, theta_d=theta_d, theta_neg=theta_neg,
                          skip=skip)]
        if dots or nq:
            steps.append(self.fused(dots=[(y, d) for d in dots],
                                    blocks=[(q, nq, y)] if nq else (), result=result,
                                    skip=skip))
        return Seq(steps)

    def prec_apply(self, prec, r, z, skip=None):
        """z = M^{-1} r over this rank's rows: a local preconditioner gets the
        slices; one whose apply needs other ranks' rows (dist.DistFsai)
        contributes its own launch sequence with the exchanges."""
        if self.comm is not None and hasattr(prec, "dist_steps"):
            return Seq(prec.dist_steps(r, z, skip))
        return PrecApply(prec, self.v(r), self.v(z), skip=skip)

    def project(self, c, k, v, out, slots, name=None):
        """out = v - C (C^T v) over this rank's rows (two passes)."""
        name = name or f"_pc{k}"
        if name not in slots.idx:
            slots.add(name, max(k, 1))
        res = slots.s[slots.idx[name]:]
        self.fused(blocks=[(c, k, v)], result=res)()
        self.fused(outs=[dict(out=out, terms=[(v, 1.0)], upd=(c, k, slots.p(name)))])()
        return out

    def gather(self, x):
        """Complete a full-length vector from the ranks' slices."""
        if self.comm is not None:
            self.comm.exchange_(x)
        return x
