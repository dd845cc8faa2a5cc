"""oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes front-end over the two CPU oracles that implement oracle/oracle_abi.h:

* ``Oracle("port")``: oracle/lib/libcs_oracle.so, the plain-C restatement
  (oracle/cs_oracle.c) -- always available (builds from this repo alone);
* ``Oracle("ref")``: oracle/_ref/libchebstep_ref.so, the unmodified reference
  library compiled from /root/reference/proj/src by oracle/Makefile -- built in
  the development container and shipped (git-ignored) to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm import this module, and only as the checker or the CPU baseline. The
product package (paper_2603_09790_b200) must never import it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "port": os.path.join(HERE, "lib", "libcs_oracle.so"),
    "ref": os.path.join(HERE, "_ref", "libchebstep_ref.so"),
}
PREFIX = {"port": "orc_", "ref": "ref_"}

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_dp = C.POINTER(C.c_double)


class OcCfg(C.Structure):
    _fields_ = [("s", C.c_int), ("tol", C.c_double), ("max_outer", C.c_int), ("nu", C.c_int),
                ("gram", C.c_int), ("has_spectrum", C.c_int), ("lambda_min", C.c_double),
                ("lambda_max", C.c_double), ("lanczos_steps", C.c_int), ("seed", C.c_uint64)]


class OcReport(C.Structure):
    _fields_ = [("converged", C.c_int), ("outer_iters", C.c_int), ("spmv_count", C.c_int64),
                ("precond_count", C.c_int64), ("allreduce_count", C.c_int64),
                ("local_update_flops", C.c_double), ("gram_solve_flops", C.c_double),
                ("lambda_min", C.c_double), ("lambda_max", C.c_double), ("cap", C.c_int),
                ("n_rel", C.c_int), ("n_da", C.c_int), ("n_db", C.c_int),
                ("rel_residual", _dp), ("delta_alpha", _dp), ("delta_beta", _dp)]


class OcHooks(C.Structure):
    _fields_ = [("collect_gram", C.c_int), ("track_true_residual", C.c_int),
                ("collect_iterates", C.c_int), ("error_reference", C.c_void_p), ("cap", C.c_int),
                ("kappa_w", _dp), ("gram_history", _dp), ("true_rel_residual", _dp),
                ("a_norm_error", _dp), ("iterates", _dp), ("n_kappa", C.c_int),
                ("n_true", C.c_int), ("n_aerr", C.c_int), ("n_iter", C.c_int)]


class OracleError(RuntimeError):
    def __init__(self, code: int, payload: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code, self.payload, self.msg = code, payload, msg


@dataclass
class Csr:
    n: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])


@dataclass
class Report:
    converged: bool
    outer_iters: int
    spmv_count: int
    precond_count: int
    allreduce_count: int
    local_update_flops: float
    gram_solve_flops: float
    lambda_min: float
    lambda_max: float
    rel_residual: np.ndarray = field(repr=False)
    delta_alpha: np.ndarray = field(repr=False)
    delta_beta: np.ndarray = field(repr=False)


def build(which: str = "port") -> None:
    target = {"port": "port", "ref": "ref", "all": "all"}[which]
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def available(which: str) -> bool:
    return os.path.exists(LIBS[which])


def nnz27(nx, ny, nz) -> int:
    f = lambda m: 3 * m - 2 if m > 1 else 1  # noqa: E731
    return f(nx) * f(ny) * f(nz)


def nnz7(nx, ny, nz) -> int:
    n = nx * ny * nz
    return n + 2 * ((nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1))


class Oracle:
    def __init__(self, which: str = "port"):
        path = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run make -C oracle)")
        self.which = which
        self.lib = C.CDLL(path)
        p = PREFIX[which]
        self._f = lambda name: getattr(self.lib, p + name)
        L = self._f
        sig = {
            "poisson27_fill": [C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, _f64p],
            "spmv": [C.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p],
            "jacobi_invdiag": [C.c_int64, _i64p, _i64p, _f64p, _f64p],
            "mpk": [C.c_int64, _i64p, _i64p, _f64p, C.c_int, _f64p, C.c_int, C.c_double,
                    C.c_double, _f64p, _f64p],
            "block_gram": [C.c_int64, C.c_int, C.c_int, _f64p, _f64p, _f64p],
            "block_update": [C.c_int64, C.c_int, C.c_int, _f64p, _f64p, _f64p, _f64p],
            "assemble_gram": [C.c_int64, C.c_int, _f64p, _f64p, _f64p],
            "fgs_solve": [C.c_int, _f64p, C.c_int, _f64p, C.c_int, _f64p, _dp],
            "cholesky_solve": [C.c_int, _f64p, C.c_int, _f64p, _f64p],
            "random_vector": [C.c_int64, C.c_uint64, _f64p],
            "tridiag_eigvals": [C.c_int, _f64p, _f64p, _f64p],
            "estimate_interval": [C.c_int64, _i64p, _i64p, _f64p, C.c_int, C.c_int, C.c_uint64,
                                  _dp, _dp],
            "pcg_s_solve": [C.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p, C.c_int,
                            C.POINTER(OcCfg), _f64p, C.POINTER(OcReport)],
            "pcg_solve": [C.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p, C.c_int, C.c_double,
                          C.c_int, _f64p, C.POINTER(OcReport)],
        }
        for name, args in sig.items():
            fn = L(name)
            fn.argtypes = args
            fn.restype = C.c_int
        le = L("last_error")
        le.argtypes = [C.POINTER(C.c_int)]
        le.restype = C.c_char_p
        if which == "port":
            self.lib.orc_stencil7_fill.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                                   C.c_double, C.c_double, _i64p, _i64p, _f64p]
            self.lib.orc_stencil7_fill.restype = C.c_int

    def _check(self, rc: int) -> None:
        if rc != 0:
            payload = C.c_int(0)
            msg = self._f("last_error")(C.byref(payload)).decode()
            raise OracleError(rc, payload.value, msg)

    # ---------------------------------------------------------------- problems
    def poisson27(self, nx, ny=None, nz=None) -> Csr:
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        n = nx * ny * nz
        nnz = nnz27(nx, ny, nz)
        rp = np.zeros(n + 1, np.int64)
        ci = np.zeros(nnz, np.int64)
        v = np.zeros(nnz, np.float64)
        self._check(self._f("poisson27_fill")(nx, ny, nz, rp, ci, v))
        return Csr(n, rp, ci, v)

    def stencil7(self, nx, ny=None, nz=None, coef=(1.0, 1.0, 1.0)) -> Csr:
        """Restatement-only generator (port library), see cs_oracle.c."""
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        n = nx * ny * nz
        nnz = nnz7(nx, ny, nz)
        rp = np.zeros(n + 1, np.int64)
        ci = np.zeros(nnz, np.int64)
        v = np.zeros(nnz, np.float64)
        lib = self.lib if self.which == "port" else Oracle("port").lib
        self._check(lib.orc_stencil7_fill(nx, ny, nz, *map(float, coef), rp, ci, v))
        return Csr(n, rp, ci, v)

    # ---------------------------------------------------------------- kernels
    def spmv(self, a: Csr, x) -> np.ndarray:
        y = np.zeros(a.n)
        self._check(self._f("spmv")(a.n, a.rowptr, a.col, a.val, np.ascontiguousarray(x, np.float64), y))
        return y

    def jacobi_invdiag(self, a: Csr) -> np.ndarray:
        out = np.zeros(a.n)
        self._check(self._f("jacobi_invdiag")(a.n, a.rowptr, a.col, a.val, out))
        return out

    def mpk(self, a: Csr, r, s: int, lo: float, hi: float, precond: int = 1):
        z = np.zeros((s, a.n))
        p = np.zeros((s + 1, a.n))
        self._check(self._f("mpk")(a.n, a.rowptr, a.col, a.val, precond,
                                    np.ascontiguousarray(r, np.float64), s, lo, hi, z, p))
        return z, p  # row j of the array == column j of the column-major block

    def block_gram(self, u: np.ndarray, v: np.ndarray) -> np.ndarray:
        """u: (ku, n), v: (kv, n) stacks of columns -> G (ku x kv)."""
        ku, n = u.shape
        kv = v.shape[0]
        g = np.zeros((kv, ku))
        self._check(self._f("block_gram")(n, ku, kv, np.ascontiguousarray(u), np.ascontiguousarray(v), g))
        return g.T.copy()

    def block_update(self, y: np.ndarray, x: np.ndarray, c: np.ndarray) -> np.ndarray:
        """y: (k, n), x: (m, n), c: (m x k) -> (k, n) = y + x c."""
        k, n = y.shape
        m = x.shape[0]
        out = np.zeros((k, n))
        cf = np.asfortranarray(c).ravel(order="F").copy()
        self._check(self._f("block_update")(n, m, k, np.ascontiguousarray(y), np.ascontiguousarray(x), cf, out))
        return out

    def assemble_gram(self, q: np.ndarray, aq: np.ndarray) -> np.ndarray:
        k, n = q.shape
        w = np.zeros((k, k))
        self._check(self._f("assemble_gram")(n, k, np.ascontiguousarray(q), np.ascontiguousarray(aq), w))
        return w.T.copy()

    def fgs_solve(self, w: np.ndarray, rhs: np.ndarray, nu: int):
        s = w.shape[0]
        rhs = rhs.reshape(s, -1)
        k = rhs.shape[1]
        x = np.zeros(s * k)
        d = C.c_double(0.0)
        self._check(self._f("fgs_solve")(s, np.asfortranarray(w).ravel(order="F").copy(), k,
                                          rhs.ravel(order="F").copy(), nu, x, C.byref(d)))
        return x.reshape(k, s).T.copy(), d.value

    def cholesky_solve(self, w: np.ndarray, rhs: np.ndarray) -> np.ndarray:
        s = w.shape[0]
        rhs = rhs.reshape(s, -1)
        k = rhs.shape[1]
        x = np.zeros(s * k)
        self._check(self._f("cholesky_solve")(s, np.asfortranarray(w).ravel(order="F").copy(), k,
                                               rhs.ravel(order="F").copy(), x))
        return x.reshape(k, s).T.copy()

    def random_vector(self, n: int, seed: int) -> np.ndarray:
        out = np.zeros(n)
        self._check(self._f("random_vector")(n, seed, out))
        return out

    def tridiag_eigvals(self, d, e) -> np.ndarray:
        d = np.ascontiguousarray(d, np.float64)
        e = np.ascontiguousarray(e, np.float64)
        if e.size == 0:
            e = np.zeros(1)
        out = np.zeros(d.size)
        self._check(self._f("tridiag_eigvals")(d.size, d, e, out))
        return out

    def estimate_interval(self, a: Csr, precond: int = 1, steps: int = 40, seed: int = 1234):
        lo, hi = C.c_double(), C.c_double()
        self._check(self._f("estimate_interval")(a.n, a.rowptr, a.col, a.val, precond, steps, seed,
                                                  C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    # ---------------------------------------------------------------- solvers
    @staticmethod
    def _report(cap: int):
        bufs = [np.zeros(cap) for _ in range(3)]
        rep = OcReport()
        rep.cap = cap
        rep.rel_residual, rep.delta_alpha, rep.delta_beta = (
            b.ctypes.data_as(_dp) for b in bufs)
        return rep, bufs

    @staticmethod
    def _unpack(rep: OcReport, bufs) -> Report:
        return Report(bool(rep.converged), rep.outer_iters, rep.spmv_count, rep.precond_count,
                      rep.allreduce_count, rep.local_update_flops, rep.gram_solve_flops,
                      rep.lambda_min, rep.lambda_max, bufs[0][:rep.n_rel].copy(),
                      bufs[1][:rep.n_da].copy(), bufs[2][:rep.n_db].copy())

    def pcg_s_solve(self, a: Csr, b=None, x0=None, *, s=4, tol=1e-6, max_outer=500, nu=30,
                    gram="fgs", spectrum=None, lanczos_steps=40, seed=1234, precond=1):
        b = np.ones(a.n) if b is None else np.ascontiguousarray(b, np.float64)
        x0 = np.zeros(a.n) if x0 is None else np.ascontiguousarray(x0, np.float64)
        cfg = OcCfg(s, tol, max_outer, nu, 1 if gram == "cholesky" else 0,
                    1 if spectrum else 0, *(spectrum or (0.0, 0.0)), lanczos_steps, seed)
        rep, bufs = self._report(max_outer + 2)
        x = np.zeros(a.n)
        self._check(self._f("pcg_s_solve")(a.n, a.rowptr, a.col, a.val, b, x0, precond,
                                            C.byref(cfg), x, C.byref(rep)))
        return x, self._unpack(rep, bufs)

    # ---------------------------------------------------------------- ingestion (ref only)
    def mm_read(self, path: str, require_spd: bool = False) -> Csr:
        assert self.which == "ref"
        f = self.lib.ref_mm_read
        f.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                      C.c_void_p, C.c_void_p, C.c_void_p]
        n, nnz = C.c_int64(), C.c_int64()
        self._check(f(os.fsencode(path), int(require_spd), C.byref(n), C.byref(nnz), None, None, None))
        rp = np.zeros(n.value + 1, np.int64)
        ci = np.zeros(nnz.value, np.int64)
        v = np.zeros(nnz.value)
        self._check(f(os.fsencode(path), int(require_spd), C.byref(n), C.byref(nnz),
                      rp.ctypes.data, ci.ctypes.data, v.ctypes.data))
        return Csr(n.value, rp, ci, v)

    def mm_write(self, path: str, a: Csr) -> None:
        assert self.which == "ref"
        f = self.lib.ref_mm_write
        f.argtypes = [C.c_char_p, C.c_int64, _i64p, _i64p, _f64p]
        self._check(f(os.fsencode(path), a.n, a.rowptr, a.col, a.val))

    def csr_validate(self, a: Csr, check: int) -> None:
        assert self.which == "ref"
        f = self.lib.ref_csr_validate
        f.argtypes = [C.c_int64, _i64p, _i64p, _f64p, C.c_int64, C.c_int]
        self._check(f(a.n, a.rowptr, a.col, a.val, a.col.size, check))

    def pcg_s_solve_hooks(self, a: Csr, *, s=4, tol=1e-6, max_outer=500, nu=30, gram="fgs",
                          spectrum=None, precond=1, collect_gram=False, track_true_residual=False,
                          error_reference=None, collect_iterates=False, classical=False):
        """Reference library only: solve with SolverConfig/PcgConfig analysis hooks."""
        assert self.which == "ref"
        b, x0 = np.ones(a.n), np.zeros(a.n)
        cap = max_outer + 2
        bufs = {"kappa": np.zeros(cap), "gram": np.zeros(cap * s * s), "true": np.zeros(cap),
                "aerr": np.zeros(cap), "iter": np.zeros(cap * a.n) if collect_iterates else None}
        hk = OcHooks()
        hk.collect_gram, hk.track_true_residual = int(collect_gram), int(track_true_residual)
        hk.collect_iterates = int(collect_iterates)
        ref = None
        if error_reference is not None:
            ref = np.ascontiguousarray(error_reference, np.float64)
            hk.error_reference = ref.ctypes.data
        hk.cap = cap
        hk.kappa_w, hk.gram_history = (bufs["kappa"].ctypes.data_as(_dp), bufs["gram"].ctypes.data_as(_dp))
        hk.true_rel_residual = bufs["true"].ctypes.data_as(_dp)
        hk.a_norm_error = bufs["aerr"].ctypes.data_as(_dp)
        if collect_iterates:
            hk.iterates = bufs["iter"].ctypes.data_as(_dp)
        rep, rb = self._report(cap)
        x = np.zeros(a.n)
        if classical:
            fn = self.lib.ref_pcg_solve_hooks
            fn.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p, C.c_int, C.c_double,
                           C.c_int, C.POINTER(OcHooks), _f64p, C.POINTER(OcReport)]
            self._check(fn(a.n, a.rowptr, a.col, a.val, b, x0, precond, tol, max_outer,
                           C.byref(hk), x, C.byref(rep)))
        else:
            cfg = OcCfg(s, tol, max_outer, nu, 1 if gram == "cholesky" else 0,
                        1 if spectrum else 0, *(spectrum or (0.0, 0.0)), 40, 1234)
            fn = self.lib.ref_pcg_s_solve_hooks
            fn.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p, C.c_int, C.POINTER(OcCfg),
                           C.POINTER(OcHooks), _f64p, C.POINTER(OcReport)]
            self._check(fn(a.n, a.rowptr, a.col, a.val, b, x0, precond, C.byref(cfg), C.byref(hk),
                           x, C.byref(rep)))
        out = {"kappa": bufs["kappa"][:hk.n_kappa].copy(),
               "gram": [bufs["gram"][i * s * s:(i + 1) * s * s].reshape(s, s).T.copy()
                        for i in range(hk.n_kappa)],
               "true": bufs["true"][:hk.n_true].copy(), "aerr": bufs["aerr"][:hk.n_aerr].copy(),
               "iter": [bufs["iter"][i * a.n:(i + 1) * a.n].copy() for i in range(hk.n_iter)]
               if collect_iterates else []}
        return x, self._unpack(rep, rb), out

    def pcg_solve(self, a: Csr, b=None, x0=None, *, tol=1e-6, max_iter=1000, precond=1):
        b = np.ones(a.n) if b is None else np.ascontiguousarray(b, np.float64)
        x0 = np.zeros(a.n) if x0 is None else np.ascontiguousarray(x0, np.float64)
        rep, bufs = self._report(max_iter + 2)
        x = np.zeros(a.n)
        self._check(self._f("pcg_solve")(a.n, a.rowptr, a.col, a.val, b, x0, precond, tol, max_iter,
                                          x, C.byref(rep)))
        return x, self._unpack(rep, bufs)
