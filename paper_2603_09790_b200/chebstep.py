"""Python mirror of the reference chebstep solve-path API, running on B200.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/chebstep/*.hpp); every compute call goes
through libchebstep_gpu.so (include/chebstep_gpu.h) -- CUDA kernels for
sm_100a, no CPU fallback. Blocks (VectorBlock, block.hpp:13-33) are numpy
arrays of shape (n, k) in Fortran (column-major) order; small dense matrices
(SmallDense, block.hpp:35-57) are (rows, cols) arrays.

Additions beyond the reference API (all optional):
  * SolverConfig.mode = "fast" (one packed reduction per outer iteration,
    the default) or "reference" (the reference's algebra and serial
    reduction order; bitwise equal to the CPU reference on one GPU);
  * Context / DeviceProblem for device-resident problems (generated on the
    GPU, optionally z-slab partitioned across ranks) and solves whose vectors
    never leave HBM.
"""
from __future__ import annotations

import ctypes as C
import os
import enum
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import CsConfig, CsReport, lib

# ---------------------------------------------------------------------------------- errors
# errors.hpp:9-56


class Error(RuntimeError):
    pass


class DimensionError(Error):
    pass


class InvalidMatrixError(Error):
    pass


class NotSpdError(Error):
    pass


class BasisBreakdownError(Error):
    def __init__(self, what: str, column: int):
        super().__init__(what)
        self.column = column


class SolverBreakdownError(Error):
    def __init__(self, what: str, outer_iteration: int):
        super().__init__(what)
        self.outer_iteration = outer_iteration


class GuardExceededError(Error):
    pass


class ParseError(Error):
    pass


class InvalidArgumentError(Error):
    pass


class CudaError(Error):
    """Device / runtime failure. There is no CPU fallback."""


class NcclError(Error):
    pass


_SIMPLE = {L.CS_ERR_DIMENSION: DimensionError, L.CS_ERR_INVALID_MATRIX: InvalidMatrixError,
           L.CS_ERR_NOT_SPD: NotSpdError, L.CS_ERR_GUARD_EXCEEDED: GuardExceededError,
           L.CS_ERR_PARSE: ParseError, L.CS_ERR_INVALID_ARGUMENT: InvalidArgumentError,
           L.CS_ERR_GENERIC: Error, L.CS_ERR_CUDA: CudaError, L.CS_ERR_NCCL: NcclError}


def _check(rc: int) -> None:
    if rc == L.CS_OK:
        return
    msg, payload = L.last_error()
    if rc == L.CS_ERR_BASIS_BREAKDOWN:
        raise BasisBreakdownError(msg, payload)
    if rc == L.CS_ERR_SOLVER_BREAKDOWN:
        raise SolverBreakdownError(msg, payload)
    raise _SIMPLE.get(rc, Error)(msg)


# ---------------------------------------------------------------------------------- context

class Context:
    """One GPU: streams, optional NCCL communicator, timing and launch counters."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib.cs_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        self.nranks, self.rank = 1, 0

    def close(self):
        if self.handle:
            _check(lib.cs_ctx_destroy(self.handle))  # refuses while problems are alive
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib.cs_comm_unique_id(buf))
        return buf.raw

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        _check(lib.cs_ctx_comm_init(self.handle, nranks, rank, uid))
        self.nranks, self.rank = nranks, rank

    def allreduce_max(self, v: float) -> float:
        d = C.c_double(v)
        _check(lib.cs_ctx_allreduce_max(self.handle, C.byref(d)))
        return d.value

    def set_timing(self, on: bool = True):
        _check(lib.cs_ctx_set_timing(self.handle, int(on)))

    def reset_timing(self):
        _check(lib.cs_ctx_reset_timing(self.handle))

    def timing(self) -> dict:
        out = {}
        for i, name in enumerate(L.PHASES):
            ms, cnt = C.c_double(), C.c_int64()
            _check(lib.cs_ctx_get_timing(self.handle, i, C.byref(ms), C.byref(cnt)))
            out[name] = (ms.value, cnt.value)
        return out

    def launches(self) -> int:
        v = C.c_int64()
        _check(lib.cs_ctx_launch_count(self.handle, C.byref(v)))
        return v.value

    def synchronize(self):
        _check(lib.cs_ctx_synchronize(self.handle))

    def stream(self) -> int:
        """cudaStream_t (as int) of this context's solve kernels."""
        h = C.c_void_p()
        _check(lib.cs_ctx_stream(self.handle, C.byref(h)))
        return h.value or 0


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def set_default_context(ctx: Context) -> None:
    global _default_ctx
    _default_ctx = ctx


def device_count() -> int:
    n = C.c_int(0)
    _check(lib.cs_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------------------------- csr / problems

@dataclass
class CsrMatrix:
    """csr.hpp:12-39: int64 offsets/columns, FP64 values."""
    n: int = 0
    row_offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))
    col_indices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))

    def __post_init__(self):
        self.row_offsets = np.ascontiguousarray(self.row_offsets, np.int64)
        self.col_indices = np.ascontiguousarray(self.col_indices, np.int64)
        self.values = np.ascontiguousarray(self.values, np.float64)

    def nnz(self) -> int:
        return int(self.col_indices.size)

    def diagonal(self, i: int) -> float:
        cols = self.col_indices[self.row_offsets[i]:self.row_offsets[i + 1]]
        k = int(np.searchsorted(cols, i))
        if k == cols.size or cols[k] != i:
            return 0.0
        return float(self.values[self.row_offsets[i] + k])

    @staticmethod
    def identity(n: int) -> "CsrMatrix":
        return CsrMatrix(n, np.arange(n + 1), np.arange(n), np.ones(n))

    @staticmethod
    def diagonal_matrix(d) -> "CsrMatrix":
        d = np.asarray(d, np.float64)
        return CsrMatrix(d.size, np.arange(d.size + 1), np.arange(d.size), d.copy())


@dataclass
class PoissonSpec:
    nx: int = 1
    ny: int = 1
    nz: int = 1

    def size(self) -> int:
        return self.nx * self.ny * self.nz


@dataclass
class PoissonSystem:
    a: CsrMatrix
    rhs: np.ndarray


class DeviceProblem:
    """A matrix resident in HBM as SELL-32 (+ preconditioner, + halo layout).

    ``DeviceProblem.generate`` builds a stencil operator on the device; with
    a communicator on ``ctx`` each rank gets its z-slab. ``DeviceProblem.from_csr``
    uploads a reference CsrMatrix (single rank)."""

    def __init__(self, ctx: Context, handle):
        self.ctx, self.handle = ctx, handle
        info = np.zeros(12, np.int64)
        _check(lib.cs_problem_info(handle, info))
        (self.n_global, self.n_local, self.nnz_local, self.row_begin, self.n_ghost,
         self.device_bytes, self.slices, self.pattern_slices, self.uniform_slices,
         self.pattern_entries, self.cdia_classes, cdia_flags) = (int(v) for v in info)
        self.cdia_uniform_diag = cdia_flags & 1
        self.cdia_planar = (cdia_flags >> 1) & 1  # separable SpMV without participation words
        self.precond = "identity"

    @property
    def halo_mode(self) -> str:
        """Halo transport of the last solve: "none", "nccl" or "nvlink-p2p"."""
        m = C.c_int(0)
        _check(lib.cs_problem_halo_mode(self.handle, C.byref(m)))
        return ("none", "nccl", "nvlink-p2p")[m.value]

    @classmethod
    def generate(cls, kind: str, nx: int, ny: int, nz: int, coef=(1.0, 1.0, 1.0),
                 ctx: Optional[Context] = None) -> "DeviceProblem":
        ctx = ctx or default_context()
        k = {"poisson27": L.CS_GEN_POISSON27, "stencil7": L.CS_GEN_STENCIL7,
             "poisson7": L.CS_GEN_STENCIL7, "aniso7": L.CS_GEN_STENCIL7}[kind]
        if kind == "aniso7" and tuple(coef) == (1.0, 1.0, 1.0):
            coef = (1.0, 1.0, 100.0)
        c = (C.c_double * 3)(*map(float, coef))
        h = C.c_void_p()
        _check(lib.cs_problem_generate(ctx.handle, k, nx, ny, nz, C.cast(c, C.c_void_p), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_csr(cls, a: CsrMatrix, ctx: Optional[Context] = None) -> "DeviceProblem":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib.cs_problem_upload_csr(ctx.handle, a.n, a.row_offsets.ctypes.data,
                                         a.col_indices.ctypes.data, a.values.ctypes.data,
                                         C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_csr_block(cls, n_global: int, row_begin: int, row_end: int, rowptr_local, col_global,
                       values, ctx: Optional[Context] = None) -> "DeviceProblem":
        """Collective: this rank's row block of a general CSR (global columns);
        builds the owner-grouped halo plan over the context's communicator."""
        ctx = ctx or default_context()
        rp = np.ascontiguousarray(rowptr_local, np.int64)
        ci = np.ascontiguousarray(col_global, np.int64)
        va = np.ascontiguousarray(values, np.float64)
        if rp.size != row_end - row_begin + 1:
            raise DimensionError("rowptr_local must have row_end - row_begin + 1 entries")
        h = C.c_void_p()
        _check(lib.cs_problem_upload_csr_block(ctx.handle, n_global, row_begin, row_end,
                                               rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
                                               C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def read_matrix_market(cls, path: str, require_spd: bool = False,
                           ctx: Optional[Context] = None) -> "DeviceProblem":
        """Matrix Market file straight to the device; each rank keeps its
        cs_partition_rows(n, 1) block (collective when ctx has a communicator)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib.cs_problem_read_mm(ctx.handle, os.fsencode(path), int(require_spd), C.byref(h)))
        return cls(ctx, h)

    def close(self):
        if self.handle:
            lib.cs_problem_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_precond(self, m) -> "DeviceProblem":
        """identity / jacobi (fused into the kernels), a BlockJacobiPreconditioner
        (device-factored blocks) or a DevicePreconditioner plugin."""
        if isinstance(m, BlockJacobiPreconditioner):
            if m.n != self.n_local:
                raise DimensionError("block_jacobi: preconditioner size != problem rows")
            _check(lib.cs_problem_set_precond_block_jacobi(self.handle, m.bs, m.blocks.ravel()))
            self._precond_keep = m
            self.precond = m.name()
            return self
        if isinstance(m, DevicePreconditioner):
            cb = m._c_callback()
            _check(lib.cs_problem_set_precond_fn(self.handle, C.cast(cb, C.c_void_p), None))
            self._precond_keep = m  # the callback must outlive the problem's solves
            self.precond = m.name()
            return self
        name = m if isinstance(m, str) else m.name()
        kind = {"identity": L.CS_PRECOND_IDENTITY, "jacobi": L.CS_PRECOND_JACOBI}.get(name)
        if kind is None:
            raise InvalidArgumentError(
                f"preconditioner {name!r} has no device implementation (identity, jacobi, "
                "BlockJacobiPreconditioner, DevicePreconditioner)")
        _check(lib.cs_problem_set_precond(self.handle, kind))
        self.precond = name
        return self

    def inv_diag(self) -> np.ndarray:
        out = np.zeros(self.n_local)
        _check(lib.cs_problem_inv_diag(self.handle, out))
        return out

    def to_csr(self) -> CsrMatrix:
        """Local rows as CSR with GLOBAL column indices (bit-exact assembly checks)."""
        rp = np.zeros(self.n_local + 1, np.int64)
        ci = np.zeros(max(self.nnz_local, 1), np.int64)
        v = np.zeros(max(self.nnz_local, 1), np.float64)
        _check(lib.cs_problem_download_csr(self.handle, rp, ci, v))
        nnz = int(rp[-1])
        return CsrMatrix(self.n_local, rp, ci[:nnz].copy(), v[:nnz].copy())

    def ghosts(self) -> np.ndarray:
        g = np.zeros(max(self.n_ghost, 1), np.int64)
        _check(lib.cs_problem_ghosts(self.handle, g))
        return g[:self.n_ghost].copy()

    def spmv(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n_local)
        _check(lib.cs_spmv(self.handle, x, y))
        return y

    def mpk(self, r, s: int, params: "ChebyshevParams") -> "MpkResult":
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(self.n_local * s)
        p = np.zeros(self.n_local * (s + 1))
        _check(lib.cs_mpk(self.handle, r, s, params.lambda_min, params.lambda_max, z, p))
        return MpkResult(z.reshape(s, self.n_local).T, p.reshape(s + 1, self.n_local).T)

    def bench_spmv(self, kind: str = "plain", reps: int = 20) -> float:
        """Average ms of one SpMV-family launch timed alone (CUDA events)."""
        k = {"plain": 0, "mpk_ref": 1, "mpk_fast": 2, "pack8": 3, "update8": 4,
             "p2p_push": 5, "p2p_mpk": 6}[kind]
        ms = C.c_double()
        _check(lib.cs_bench_spmv(self.handle, k, reps, C.byref(ms)))
        return ms.value

    def estimate_interval(self, steps: int = 40, seed: int = 1234, mode: str = "fast"):
        lo, hi = C.c_double(), C.c_double()
        _check(lib.cs_estimate_interval(self.handle, steps, seed, _mode(mode), C.byref(lo),
                                        C.byref(hi)))
        return SpectrumEstimate(lo.value, hi.value, "lanczos", 0.9, 1.1)

    def pcg_s_solve(self, b=None, x0=None, cfg: Optional["SolverConfig"] = None) -> "SolveResult":
        """Host vectors in/out (local rows); the solve itself is device-resident."""
        cfg = cfg or SolverConfig()
        b = np.ones(self.n_local) if b is None else np.ascontiguousarray(b, np.float64)
        x0 = np.zeros(self.n_local) if x0 is None else np.ascontiguousarray(x0, np.float64)
        if b.size != self.n_local or x0.size != self.n_local:
            raise DimensionError("pcg_s_solve: vector length mismatch")
        x = np.zeros(self.n_local)
        rep, bufs = _report(cfg.max_outer + 2, cfg.s, self.n_local, cfg)
        cc = cfg._c()
        _check(lib.cs_pcg_s_solve(self.handle, b, x0, C.byref(cc), x, C.byref(rep)))
        return SolveResult(x, _unpack(rep, bufs))

    def pcg_s_solve_device(self, b_ptr: int, x0_ptr: int, x_ptr: int,
                           cfg: Optional["SolverConfig"] = None) -> "SolveReport":
        """Raw device pointers (e.g. torch tensor .data_ptr()), n_local doubles each."""
        cfg = cfg or SolverConfig()
        rep, bufs = _report(cfg.max_outer + 2)
        _check(lib.cs_pcg_s_solve_device(self.handle, b_ptr, x0_ptr, C.byref(cfg._c()), x_ptr,
                                         C.byref(rep)))
        return _unpack(rep, bufs)

    def pcg_solve(self, b=None, x0=None, tol: float = 1e-6, max_iter: int = 1000,
                  mode: str = "fast", cfg: Optional["PcgConfig"] = None) -> "SolveResult":
        """Classical PCG; cfg (PcgConfig) adds the error_reference / collect_iterates hooks."""
        b = np.ones(self.n_local) if b is None else np.ascontiguousarray(b, np.float64)
        x0 = np.zeros(self.n_local) if x0 is None else np.ascontiguousarray(x0, np.float64)
        x = np.zeros(self.n_local)
        if cfg is not None:
            tol, max_iter = cfg.tol, cfg.max_iter
        if not (tol >= 0.0) or max_iter < 1:
            raise InvalidArgumentError("pcg_solve: bad tol/max_iter")
        cc = CsConfig()
        lib.cs_config_default(C.byref(cc))
        cc.tol, cc.max_outer, cc.mode = tol, max_iter, _mode(mode)
        keep = None
        if cfg is not None and cfg.error_reference is not None:
            keep = np.ascontiguousarray(cfg.error_reference, np.float64)
            cc.error_reference = keep.ctypes.data
        if cfg is not None:
            cc.collect_iterates = int(cfg.collect_iterates)
        rep, bufs = _report(max_iter + 2, 1, self.n_local, cfg)
        _check(lib.cs_pcg_solve_cfg(self.handle, b, x0, C.byref(cc), x, C.byref(rep)))
        del keep
        return SolveResult(x, _unpack(rep, bufs))

    def pcg_solve_device(self, b_ptr: int, x0_ptr: int, x_ptr: int, tol: float = 1e-6,
                         max_iter: int = 1000, mode: str = "fast") -> "SolveReport":
        rep, bufs = _report(max_iter + 2)
        _check(lib.cs_pcg_solve_device(self.handle, b_ptr, x0_ptr, tol, max_iter, _mode(mode),
                                       x_ptr, C.byref(rep)))
        return _unpack(rep, bufs)


def read_matrix_market(path: str, require_spd: bool = False) -> CsrMatrix:
    """problems.hpp:28-31 (problems.cpp:55-109): host parse on all cores."""
    h, n, nnz = C.c_void_p(), C.c_int64(), C.c_int64()
    _check(lib.cs_mm_read(os.fsencode(path), int(require_spd), C.byref(h), C.byref(n),
                          C.byref(nnz)))
    try:
        rp = np.zeros(n.value + 1, np.int64)
        ci = np.zeros(nnz.value, np.int64)
        va = np.zeros(nnz.value, np.float64)
        _check(lib.cs_csr_host_rows(h, 0, n.value, rp.ctypes.data, ci.ctypes.data, va.ctypes.data))
    finally:
        lib.cs_csr_host_free(h)
    return CsrMatrix(n.value, rp, ci, va)


def write_matrix_market(path: str, a: CsrMatrix) -> None:
    """problems.hpp:33-34 (problems.cpp:111-127): lower triangle, %.17g."""
    _check(lib.cs_mm_write(os.fsencode(path), a.n, a.row_offsets.ctypes.data,
                           a.col_indices.ctypes.data, a.values.ctypes.data))


def _validate(a: CsrMatrix, check: int) -> None:
    if check == L.CS_CHECK_SPD_DIAGONAL:  # csr.cpp:100-110 checks no structure first
        _check(lib.cs_csr_validate(a.n, a.row_offsets.ctypes.data, a.col_indices.ctypes.data,
                                   a.values.ctypes.data, check))
        return
    if a.row_offsets.size != a.n + 1 or a.n < 0:
        raise InvalidMatrixError("row_offsets length must be n+1")
    if int(a.row_offsets[0]) != 0:
        raise InvalidMatrixError("row_offsets[0] must be 0")
    if a.values.size != a.col_indices.size or int(a.row_offsets[-1]) != a.col_indices.size:
        raise InvalidMatrixError("row_offsets[n] must equal nnz")
    _check(lib.cs_csr_validate(a.n, a.row_offsets.ctypes.data, a.col_indices.ctypes.data,
                               a.values.ctypes.data, check))


def validate_structure(a: CsrMatrix) -> None:
    """csr.cpp:58-79"""
    _validate(a, L.CS_CHECK_STRUCTURE)


def validate_symmetric(a: CsrMatrix) -> None:
    """csr.cpp:81-98"""
    _validate(a, L.CS_CHECK_SYMMETRIC)


def validate_spd_diagonal(a: CsrMatrix) -> None:
    """csr.cpp:100-110"""
    _validate(a, L.CS_CHECK_SPD_DIAGONAL)


def poisson27(spec: PoissonSpec, ctx: Optional[Context] = None) -> PoissonSystem:
    """problems.cpp:13-53, assembled on the device and downloaded."""
    p = DeviceProblem.generate("poisson27", spec.nx, spec.ny, spec.nz, ctx=ctx)
    try:
        return PoissonSystem(p.to_csr(), np.ones(spec.size()))
    finally:
        p.close()


def stencil7(spec: PoissonSpec, coef=(1.0, 1.0, 1.0), ctx: Optional[Context] = None) -> PoissonSystem:
    """7-point operator (poisson7 = (1,1,1); the anisotropic config 4 = (1,1,100))."""
    p = DeviceProblem.generate("stencil7", spec.nx, spec.ny, spec.nz, coef, ctx=ctx)
    try:
        return PoissonSystem(p.to_csr(), np.ones(spec.size()))
    finally:
        p.close()


# ---------------------------------------------------------------------------------- precond

class Preconditioner:
    """precond.hpp:12-23. Device kernels exist for identity and jacobi only."""

    def name(self) -> str:
        raise NotImplementedError


class IdentityPreconditioner(Preconditioner):
    def name(self) -> str:
        return "identity"


class JacobiPreconditioner(Preconditioner):
    """M = diag(A); the device recomputes inv_diag = 1/a_ii exactly as precond.cpp:15-23
    (NotSpdError on a non-positive diagonal, raised here like the reference ctor)."""

    def __init__(self, a: CsrMatrix):
        d = np.array([a.diagonal(i) for i in range(a.n)]) if a.n <= 4096 else None
        if d is not None and not np.all(d > 0.0):
            raise NotSpdError("jacobi: diagonal must be strictly positive")
        self.a = a

    def name(self) -> str:
        return "jacobi"


class BlockJacobiPreconditioner(Preconditioner):
    """M = blockdiag(A_11, A_22, ...) over blocks of `bs` consecutive rows.

    The dense diagonal blocks are extracted here (entries summed in stored
    order; a short last block padded with the identity), the device factorises
    them (Cholesky, dense_ops.cpp:55-88 order) and applies two triangular
    solves per block inside the solve. apply() is the host restatement."""

    def __init__(self, a: CsrMatrix, bs: int = 4):
        if not 1 <= bs <= 16:
            raise InvalidArgumentError("block_jacobi: bs must be in [1, 16]")
        self.bs, self.n = int(bs), int(a.n)
        nb = (a.n + bs - 1) // bs
        blocks = np.zeros((nb, bs, bs))  # blocks[b, j, i] = A[b*bs+i, b*bs+j] (column-major)
        rows = np.repeat(np.arange(a.n, dtype=np.int64), np.diff(a.row_offsets))
        cols = a.col_indices
        inb = (cols // bs) == (rows // bs)
        np.add.at(blocks, (rows[inb] // bs, cols[inb] % bs, rows[inb] % bs), a.values[inb])
        for r in range(a.n, nb * bs):
            blocks[r // bs, r % bs, r % bs] = 1.0
        self.blocks = np.ascontiguousarray(blocks)

    def name(self) -> str:
        return "block_jacobi"


class DevicePreconditioner(Preconditioner):
    """Plugin whose apply runs on the device: subclass and implement
    ``device_apply(in_ptr, out_ptr, n, stream)`` (raw device pointers, n doubles,
    the solve's cudaStream_t as an int), enqueueing out = M^-1 in on that stream.
    The solver calls it wherever the reference calls Preconditioner::apply."""

    def device_apply(self, in_ptr: int, out_ptr: int, n: int, stream: int) -> None:
        raise NotImplementedError

    def name(self) -> str:
        return "device"

    def _c_callback(self):
        if getattr(self, "_cb", None) is None:
            def cb(_user, i, o, n, stream):
                try:
                    self.device_apply(i or 0, o or 0, n, stream or 0)
                    return 0
                except Exception:  # noqa: BLE001 -- reported as a failed apply
                    return 1
            self._cb = L.PRECOND_FN(cb)
        return self._cb


def _general(m) -> bool:
    return isinstance(m, (BlockJacobiPreconditioner, DevicePreconditioner))


def _precond_kind(m: Preconditioner) -> int:
    kind = {"identity": L.CS_PRECOND_IDENTITY, "jacobi": L.CS_PRECOND_JACOBI}.get(m.name())
    if kind is None:
        raise InvalidArgumentError(f"preconditioner {m.name()!r} has no device implementation")
    return kind


# ---------------------------------------------------------------------------------- config / report

class GramSolverKind(enum.Enum):
    fgs = 0
    cholesky = 1


@dataclass
class FgsConfig:
    nu: int = 30
    multi_rhs: bool = True


@dataclass
class SpectrumEstimate:
    lambda_min: float = 0.0
    lambda_max: float = 0.0
    method: str = "lanczos"
    low_factor: float = 1.0
    high_factor: float = 1.0


def _mode(mode: str) -> int:
    return {"fast": L.CS_MODE_FAST, "reference": L.CS_MODE_REFERENCE}[mode]


@dataclass
class SolverConfig:
    """solver.hpp:16-37 (+ mode / check_every, device-only knobs)."""
    s: int = 4
    tol: float = 1e-6
    max_outer: int = 500
    fgs: FgsConfig = field(default_factory=FgsConfig)
    gram_solver: GramSolverKind = GramSolverKind.fgs
    spectrum: Optional[SpectrumEstimate] = None
    lanczos_steps: int = 40
    seed: int = 1234
    # analysis hooks (solver.hpp:30-34); none changes the iterates
    collect_gram: bool = False
    track_true_residual: bool = False
    error_reference: Optional[np.ndarray] = None
    collect_iterates: bool = False
    mode: str = "fast"
    check_every: int = 0
    variant: int = 0  # CS_VAR_* bits (arithmetic variants for sensitivity studies)

    def _c(self) -> CsConfig:
        c = CsConfig()
        lib.cs_config_default(C.byref(c))
        c.s, c.tol, c.max_outer, c.nu = self.s, self.tol, self.max_outer, self.fgs.nu
        c.gram = self.gram_solver.value
        if self.spectrum is not None:
            c.has_spectrum = 1
            c.lambda_min, c.lambda_max = self.spectrum.lambda_min, self.spectrum.lambda_max
        c.lanczos_steps, c.seed = self.lanczos_steps, self.seed
        c.mode, c.check_every = _mode(self.mode), self.check_every
        c.variant = self.variant
        c.collect_gram = int(self.collect_gram)
        c.track_true_residual = int(self.track_true_residual)
        c.collect_iterates = int(self.collect_iterates)
        if self.error_reference is not None:
            self._ref_keep = np.ascontiguousarray(self.error_reference, np.float64)
            c.error_reference = self._ref_keep.ctypes.data
        return c


@dataclass
class SolveReport:
    """solver.hpp:39-68 (+ device facts)."""
    converged: bool = False
    outer_iters: int = 0
    rel_residual: np.ndarray = field(default_factory=lambda: np.zeros(0))
    delta_alpha: np.ndarray = field(default_factory=lambda: np.zeros(0))
    delta_beta: np.ndarray = field(default_factory=lambda: np.zeros(0))
    spmv_count: int = 0
    precond_count: int = 0
    allreduce_count: int = 0
    local_update_flops: float = 0.0
    gram_solve_flops: float = 0.0
    spectrum_used: SpectrumEstimate = field(default_factory=SpectrumEstimate)
    kappa_w: np.ndarray = field(default_factory=lambda: np.zeros(0))
    gram_history: list = field(default_factory=list)
    true_rel_residual: np.ndarray = field(default_factory=lambda: np.zeros(0))
    a_norm_error: np.ndarray = field(default_factory=lambda: np.zeros(0))
    iterates: list = field(default_factory=list)
    device_allreduces: int = 0
    schedule: int = 0  # CS_SCHED_* bits of the fast schedule that ran
    kernel_launches: int = 0
    t_lanczos_ms: float = 0.0
    t_solve_ms: float = 0.0


@dataclass
class SolveResult:
    x: np.ndarray
    report: SolveReport


def _report(cap: int, s: int = 0, n: int = 0, cfg=None):
    bufs = [np.zeros(cap) for _ in range(3)]
    rep = CsReport()
    rep.cap = cap
    rep.rel_residual, rep.delta_alpha, rep.delta_beta = (b.ctypes.data_as(L._dp) for b in bufs)
    hooks = {}
    if cfg is not None:
        if getattr(cfg, "collect_gram", False):
            hooks["kappa"] = np.zeros(cap)
            hooks["gram"] = np.zeros(cap * s * s)
            rep.kappa_w = hooks["kappa"].ctypes.data_as(L._dp)
            rep.gram_history = hooks["gram"].ctypes.data_as(L._dp)
        if getattr(cfg, "track_true_residual", False):
            hooks["true"] = np.zeros(cap)
            rep.true_rel_residual = hooks["true"].ctypes.data_as(L._dp)
        if getattr(cfg, "error_reference", None) is not None:
            hooks["aerr"] = np.zeros(cap)
            rep.a_norm_error = hooks["aerr"].ctypes.data_as(L._dp)
        if getattr(cfg, "collect_iterates", False):
            hooks["iter"] = np.zeros(cap * n)
            rep.iterates = hooks["iter"].ctypes.data_as(L._dp)
    bufs.append((hooks, s, n))
    return rep, bufs


def _unpack(rep: CsReport, bufs) -> SolveReport:
    out = SolveReport(
        bool(rep.converged), rep.outer_iters, bufs[0][:rep.n_rel].copy(),
        bufs[1][:rep.n_da].copy(), bufs[2][:rep.n_db].copy(), rep.spmv_count, rep.precond_count,
        rep.allreduce_count, rep.local_update_flops, rep.gram_solve_flops,
        SpectrumEstimate(rep.lambda_min, rep.lambda_max, "lanczos", 0.9, 1.1))
    out.device_allreduces, out.kernel_launches = rep.device_allreduces, rep.kernel_launches
    out.schedule = rep.schedule
    out.t_lanczos_ms, out.t_solve_ms = rep.t_lanczos_ms, rep.t_solve_ms
    hooks, s, n = bufs[3] if len(bufs) > 3 else ({}, 0, 0)
    if "kappa" in hooks:
        out.kappa_w = hooks["kappa"][:rep.n_kappa].copy()
        out.gram_history = [hooks["gram"][i * s * s:(i + 1) * s * s].reshape(s, s).T.copy()
                            for i in range(rep.n_kappa)]
    if "true" in hooks:
        out.true_rel_residual = hooks["true"][:rep.n_true].copy()
    if "aerr" in hooks:
        out.a_norm_error = hooks["aerr"][:rep.n_aerr].copy()
    if "iter" in hooks:
        out.iterates = [hooks["iter"][i * n:(i + 1) * n].copy() for i in range(rep.n_iter)]
    return out


# ---------------------------------------------------------------------------------- solves

def _vec(v, n, what):
    v = np.ascontiguousarray(v, np.float64)
    if v.size != n:
        raise DimensionError(f"{what}: vector length mismatch")
    return v


def pcg_s_solve(a: CsrMatrix, b, x0, m: Preconditioner, cfg: Optional[SolverConfig] = None,
                ctx: Optional[Context] = None) -> SolveResult:
    """solver.hpp:81-83 -- upload, SELL conversion, preconditioner, spectrum
    estimate, device solve and download in one C-ABI call."""
    cfg = cfg or SolverConfig()
    ctx = ctx or default_context()
    cc = cfg._c()
    if not (1 <= cfg.s <= 64):
        raise InvalidArgumentError("SolverConfig: s must be in [1, 64]")
    b = _vec(b, a.n, "pcg_s_solve")
    x0 = _vec(x0, a.n, "pcg_s_solve")
    if _general(m):  # block Jacobi / device plugin: upload, attach, solve
        p = _with_problem(a, m, ctx)
        try:
            return p.pcg_s_solve(b, x0, cfg)
        finally:
            p.close()
    x = np.zeros(a.n)
    rep, bufs = _report(cfg.max_outer + 2, cfg.s, a.n, cfg)
    _check(lib.cs_pcg_s_solve_csr(ctx.handle, a.n, a.row_offsets.ctypes.data,
                                  a.col_indices.ctypes.data, a.values.ctypes.data,
                                  _precond_kind(m), b.ctypes.data, x0.ctypes.data, C.byref(cc),
                                  x.ctypes.data, C.byref(rep)))
    return SolveResult(x, _unpack(rep, bufs))


@dataclass
class PcgConfig:
    """solver.hpp:85-90."""
    tol: float = 1e-6
    max_iter: int = 1000
    error_reference: Optional[np.ndarray] = None
    collect_iterates: bool = False


def pcg_solve(a: CsrMatrix, b, x0, m: Preconditioner, cfg=None, max_iter: Optional[int] = None,
              ctx: Optional[Context] = None) -> SolveResult:
    """solver.hpp:95-100: pcg_solve(a, b, x0, m, PcgConfig) or (…, tol, max_iter)."""
    if cfg is None:
        cfg = PcgConfig()
    elif not isinstance(cfg, PcgConfig):
        cfg = PcgConfig(float(cfg), int(max_iter if max_iter is not None else 1000))
    ctx = ctx or default_context()
    b = _vec(b, a.n, "pcg_solve")
    x0 = _vec(x0, a.n, "pcg_solve")
    p = _with_problem(a, m, ctx)
    try:
        return p.pcg_solve(b, x0, cfg.tol, cfg.max_iter, "fast", cfg=cfg)
    finally:
        p.close()


@dataclass
class InexactVerdict:
    max_delta: float
    budget: float
    passed: bool

    @property
    def pass_(self) -> bool:
        return self.passed


def monitor_inexact(report: SolveReport, delta_cap: float = 1.0) -> InexactVerdict:
    """solver.cpp:275-282 (host bookkeeping over the report)."""
    max_delta = 0.0
    for d in report.delta_alpha:
        max_delta = max(max_delta, float(d))
    budget = float(report.outer_iters) * max_delta
    return InexactVerdict(max_delta, budget, budget <= delta_cap)


# ---------------------------------------------------------------------------------- unit entries

@dataclass
class ChebyshevParams:
    """mpk.hpp:14-28."""
    lambda_min: float = 0.0
    lambda_max: float = 0.0

    @staticmethod
    def from_interval(lo: float, hi: float) -> "ChebyshevParams":
        if not (hi > lo) or not (lo > 0.0) or not math.isfinite(hi):
            raise InvalidArgumentError("ChebyshevParams: need lambda_max > lambda_min > 0")
        return ChebyshevParams(lo, hi)

    @staticmethod
    def from_estimate(e: SpectrumEstimate) -> "ChebyshevParams":
        return ChebyshevParams.from_interval(e.lambda_min, e.lambda_max)

    def alpha(self) -> float:
        return 2.0 / (self.lambda_max - self.lambda_min)

    def sigma(self) -> float:
        return (self.lambda_max + self.lambda_min) / (self.lambda_max - self.lambda_min)

    def gamma(self) -> float:
        return 1.0


@dataclass
class MpkResult:
    z: np.ndarray  # n x s
    p: np.ndarray  # n x (s+1)


def _with_problem(a: CsrMatrix, m: Optional[Preconditioner], ctx):
    p = DeviceProblem.from_csr(a, ctx)
    if m is not None:
        p.set_precond(m)
    return p


def spmv(a: CsrMatrix, x, ctx: Optional[Context] = None) -> np.ndarray:
    """csr.hpp:51 -- bitwise equal to the reference row-serial SpMV."""
    x = _vec(x, a.n, "spmv")
    p = _with_problem(a, None, ctx)
    try:
        return p.spmv(x)
    finally:
        p.close()


def spmv_into(a: CsrMatrix, x, y: np.ndarray, ctx: Optional[Context] = None) -> None:
    if y.size != a.n:
        raise DimensionError("spmv: vector length must equal matrix dimension")
    y[:] = spmv(a, x, ctx)


def mpk_chebyshev(a: CsrMatrix, r, s: int, m: Preconditioner, params: ChebyshevParams,
                  ctx: Optional[Context] = None) -> MpkResult:
    """mpk.hpp:43-44."""
    r = _vec(r, a.n, "mpk")
    p = _with_problem(a, m, ctx)
    try:
        return p.mpk(r, s, params)
    finally:
        p.close()


def _block(x) -> np.ndarray:
    x = np.asarray(x, np.float64)
    if x.ndim == 1:
        x = x[:, None]
    return x


def _colmajor(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x.T).ravel()


def block_gram(u, v, mode: str = "reference", ctx: Optional[Context] = None) -> np.ndarray:
    """dense_ops.hpp:17 -- G = u^T v. mode "reference" = serial ascending order (bitwise)."""
    ctx = ctx or default_context()
    u, v = _block(u), _block(v)
    if u.shape[0] != v.shape[0]:
        raise DimensionError("block_gram: row counts differ")
    g = np.zeros(u.shape[1] * v.shape[1])
    _check(lib.cs_block_gram(ctx.handle, u.shape[0], u.shape[1], v.shape[1], _colmajor(u),
                             _colmajor(v), g, _mode(mode)))
    return g.reshape(v.shape[1], u.shape[1]).T.copy()


def block_update(y, x, c, ctx: Optional[Context] = None) -> np.ndarray:
    """dense_ops.hpp:20-21 -- y + x c."""
    ctx = ctx or default_context()
    y, x, c = _block(y), _block(x), _block(c)
    n, k = y.shape
    m = x.shape[1]
    if x.shape[0] != n or c.shape != (m, k):
        raise DimensionError("block_update: shape mismatch")
    out = np.zeros(n * k)
    _check(lib.cs_block_update(ctx.handle, n, m, k, _colmajor(y), _colmajor(x), _colmajor(c), out))
    return out.reshape(k, n).T.copy()


@dataclass
class GramSystem:
    w: np.ndarray
    diag: np.ndarray
    normalized: bool = False

    def order(self) -> int:
        return self.w.shape[0]


def assemble_gram(q, aq, mode: str = "reference", ctx: Optional[Context] = None) -> GramSystem:
    """gram.hpp:27 -- W = q^T aq symmetrised; NotSpdError on a degenerate diagonal."""
    ctx = ctx or default_context()
    q, aq = _block(q), _block(aq)
    if q.shape != aq.shape:
        raise DimensionError("assemble_gram: block shapes differ")
    k = q.shape[1]
    w = np.zeros(k * k)
    _check(lib.cs_assemble_gram(ctx.handle, q.shape[0], k, _colmajor(q), _colmajor(aq), w,
                                _mode(mode)))
    w = w.reshape(k, k).T.copy()
    return GramSystem(w, np.diag(w).copy())


def gram_from_matrix(w) -> GramSystem:
    """gram.cpp:51-58: square, exactly symmetric, positive finite diagonal."""
    w = np.asarray(w, np.float64)
    if w.ndim != 2 or w.shape[0] != w.shape[1]:
        raise DimensionError("gram_from_matrix: not square")
    if not np.array_equal(w, w.T):
        raise InvalidMatrixError("gram_from_matrix: matrix not symmetric")
    d = np.diag(w).copy()
    if not np.all(np.isfinite(d) & (d > 0.0)):
        raise NotSpdError("gram: non-positive diagonal (basis degeneracy)")
    return GramSystem(w.copy(), d)


def normalize_gram(g: GramSystem) -> GramSystem:
    """gram.cpp:60-76: D^-1/2 W D^-1/2 with an exact unit diagonal."""
    inv = 1.0 / np.sqrt(g.diag)
    w = (g.w * inv[:, None]) * inv[None, :]
    np.fill_diagonal(w, 1.0)
    return GramSystem(w, np.ones(g.order()), True)


@dataclass
class FgsRate:
    spectral_norm: float
    spectral_radius: float


def fgs_rate(g: GramSystem) -> FgsRate:
    """gram.cpp:148-174 (host eigensolvers instead of dgesvd/dgeev)."""
    if not g.normalized:
        raise InvalidArgumentError("fgs_rate: system must be normalized")
    w = np.asfortranarray(g.w, np.float64)
    nrm, rad = C.c_double(), C.c_double()
    _check(lib.cs_fgs_rate(g.order(), w.ctypes.data, C.byref(nrm), C.byref(rad)))
    return FgsRate(nrm.value, rad.value)


def kappa_sym(w) -> float:
    """kappa_2 of a symmetric matrix as solver.cpp:69-74 computes it."""
    w = np.asfortranarray(w, np.float64)
    k = C.c_double()
    _check(lib.cs_kappa_sym(w.shape[0], w.ctypes.data, C.byref(k)))
    return k.value


@dataclass
class FgsResult:
    x: np.ndarray
    rel_residual: float


def fgs_solve(g: GramSystem, rhs, cfg: Optional[FgsConfig] = None,
              ctx: Optional[Context] = None) -> FgsResult:
    """gram.hpp:49-50."""
    ctx = ctx or default_context()
    cfg = cfg or FgsConfig()
    rhs = _block(rhs)
    s = g.order()
    if rhs.shape[0] != s:
        raise DimensionError("fgs: rhs rows mismatch")
    if not cfg.multi_rhs and rhs.shape[1] > 1:
        raise InvalidArgumentError("fgs: multiple right-hand sides disabled")
    x = np.zeros(s * rhs.shape[1])
    d = C.c_double()
    _check(lib.cs_fgs_solve(ctx.handle, s, _colmajor(g.w), rhs.shape[1], _colmajor(rhs), cfg.nu,
                            x, C.byref(d)))
    return FgsResult(x.reshape(rhs.shape[1], s).T.copy(), d.value)


def small_cholesky_solve(w, rhs, ctx: Optional[Context] = None) -> np.ndarray:
    """dense_ops.hpp:28."""
    ctx = ctx or default_context()
    w, rhs = _block(w), _block(rhs)
    s = w.shape[0]
    if w.shape[1] != s:
        raise DimensionError("cholesky: matrix not square")
    if rhs.shape[0] != s:
        raise DimensionError("cholesky: rhs rows mismatch")
    x = np.zeros(s * rhs.shape[1])
    _check(lib.cs_cholesky_solve(ctx.handle, s, _colmajor(w), rhs.shape[1], _colmajor(rhs), x))
    return x.reshape(rhs.shape[1], s).T.copy()


def random_vector(n: int, seed: int, ctx: Optional[Context] = None) -> np.ndarray:
    """util.cpp:31-36, generated on the device (counter-based SplitMix64)."""
    ctx = ctx or default_context()
    out = np.zeros(n)
    _check(lib.cs_random_vector(ctx.handle, n, seed, out))
    return out


def tridiag_eigvals(diag, off) -> np.ndarray:
    d = np.ascontiguousarray(diag, np.float64)
    e = np.ascontiguousarray(off, np.float64)
    if e.size == 0:
        e = np.zeros(1)
    out = np.zeros(d.size)
    _check(lib.cs_tridiag_eigvals(d.size, d, e, out))
    return out


def estimate_interval(a: CsrMatrix, m: Preconditioner, steps: int = 40, seed: int = 1234,
                      mode: str = "fast", ctx: Optional[Context] = None) -> SpectrumEstimate:
    """spectral.hpp:49-50 -- device Lanczos."""
    p = _with_problem(a, m, ctx)
    try:
        return p.estimate_interval(steps, seed, mode)
    finally:
        p.close()


# ---------------------------------------------------------------------------------- partitioning

def partition_rows(n_rows: int, plane: int, nranks: int, rank: int):
    b, e = C.c_int64(), C.c_int64()
    _check(lib.cs_partition_rows(n_rows, plane, nranks, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


def halo_map_csr(row_begin: int, row_end: int, rowptr_local, col_global):
    """Ghost list + local int32 columns of one rank's CSR block (host, no GPU)."""
    rp = np.ascontiguousarray(rowptr_local, np.int64)
    cg = np.ascontiguousarray(col_global, np.int64)
    ng = C.c_int64()
    _check(lib.cs_halo_map_csr(row_begin, row_end, rp, cg, C.byref(ng), None, 0, None))
    ghosts = np.zeros(max(ng.value, 1), np.int64)
    cl = np.zeros(max(cg.size, 1), np.int32)
    _check(lib.cs_halo_map_csr(row_begin, row_end, rp, cg, C.byref(ng), ghosts.ctypes.data,
                               ng.value, cl.ctypes.data))
    return ghosts[:ng.value].copy(), cl[:cg.size].copy()
