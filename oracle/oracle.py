"""ctypes wrapper of oracle/liboracle_dd.so (TEST INFRASTRUCTURE ONLY).

Marshalling only; every step of the oracle runs in dd_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_dd.so")
_SRC = os.path.join(_HERE, "dd_oracle.c")
_SHIM = os.path.join(_HERE, "dd_shim.c")       # the SURVEY 8(b) dd_* ABI over ddo_*

SCHED_FIXED = 0
SCHED_LADDER = 1
OK, EINVAL, ENOCONV, ENUMERIC, ENOMEM = 0, 1, 2, 3, 6


def build_oracle(force: bool = False) -> str:
    """Compile the oracle (plain C11, fp64, OpenMP).  No -ffast-math: IEEE RN."""
    srcs = [_SRC, _SHIM, os.path.join(_HERE, "dd_oracle.h")]
    if force or not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(f) for f in srcs):
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO, _SRC, _SHIM, "-lm"])
    return _SO


class _Opt(C.Structure):
    _fields_ = [("err_tol", C.c_double), ("trunc_tau", C.c_double),
                ("max_inner_iter", C.c_int), ("n_threads", C.c_int),
                ("schedule", C.c_int), ("eps_start", C.c_double),
                ("coarsest_side", C.c_int), ("no_truncate", C.c_int), ("empty_init", C.c_int),
                ("check_every", C.c_int), ("warm_refine", C.c_int), ("safeguard", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("cells", C.c_longlong), ("iters_sum", C.c_longlong),
                ("iters_max", C.c_int), ("failed", C.c_int),
                ("err_x_sum", C.c_double), ("entries", C.c_longlong),
                ("safeguarded", C.c_int), ("pad_", C.c_int)]


class _Info(C.Structure):
    _fields_ = [("side", C.c_int), ("s", C.c_int), ("nb", C.c_int),
                ("last_partition", C.c_int), ("half_index", C.c_longlong),
                ("entries", C.c_longlong), ("eps", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build_oracle())
        d, i, ll, p = C.c_double, C.c_int, C.c_longlong, C.c_void_p
        dp = C.POINTER(C.c_double)
        _lib.ddo_sinkhorn_dense.argtypes = [i, i, dp, dp, dp, d, d, i, dp, dp,
                                            C.POINTER(i), dp]
        _lib.ddo_build_schedule.argtypes = [i, i, d, d, C.POINTER(i), dp, C.POINTER(i), i]
        _lib.ddo_init.argtypes = [C.POINTER(p), i, dp, dp, d, i, C.POINTER(_Opt)]
        _lib.ddo_set_eps.argtypes = [p, d]
        _lib.ddo_set_cost.argtypes = [p, i, p, p]
        _lib.ddo_iterate.argtypes = [p, i]
        _lib.ddo_solve_cells.argtypes = [p, i, i, p, p]
        _lib.ddo_solve_cells_par.argtypes = [p, i, i, p, p]
        _lib.ddo_dual_gap.argtypes = [p, dp, dp, dp]
        _lib.ddo_refine.argtypes = [p]
        _lib.ddo_run_schedule.argtypes = [p]
        _lib.ddo_primal_cost.argtypes = [p, dp, dp]
        _lib.ddo_marginal_error.argtypes = [p, dp, dp]
        _lib.ddo_fetch_plan_coo.argtypes = [p, C.POINTER(ll), p, p, p]
        _lib.ddo_get_stats.argtypes = [p, C.POINTER(_Stats)]
        _lib.ddo_get_state_info.argtypes = [p, C.POINTER(_Info)]
        _lib.ddo_get_state.argtypes = [p, p, p, p, p, p]
        _lib.ddo_set_state.argtypes = [p, i, ll, i, p, p, p, p, p]
        _lib.ddo_get_layer_marginals.argtypes = [p, p, p]
        _lib.ddo_free.argtypes = [p]
        _lib.ddo_last_error.argtypes = [p]
        _lib.ddo_last_error.restype = C.c_char_p
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def sinkhorn_dense(a, b, cost, eps, tol, max_iter=100000, f0=None):
    """Dense log-domain Sinkhorn of the oracle (returns f, g, iters, err, rc)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    nx, ny = a.size, b.size
    f = np.zeros(nx) if f0 is None else np.array(f0, dtype=np.float64)
    g = np.zeros(ny)
    it = C.c_int(0)
    err = C.c_double(0)
    rc = lib().ddo_sinkhorn_dense(nx, ny, _dp(a), _dp(b), _dp(cost), eps, tol, max_iter,
                                  _dp(f), _dp(g), C.byref(it), C.byref(err))
    return f, g, it.value, err.value, rc


def build_schedule(n_final, coarsest_side, kappa_final, eps_start=0.0):
    m = 512
    side = (C.c_int * m)()
    kap = (C.c_double * m)()
    sw = (C.c_int * m)()
    k = lib().ddo_build_schedule(n_final, coarsest_side, kappa_final, eps_start,
                                 side, kap, sw, m)
    return [(side[j], kap[j], sw[j]) for j in range(min(k, m))]


class Oracle:
    """One oracle context (same call names as the product binding)."""

    def __init__(self, mu, nu, eps, cell_size, *, err_tol=1e-6, trunc_tau=1e-15,
                 max_inner_iter=10000, n_threads=0, schedule=SCHED_FIXED, eps_start=0.0,
                 coarsest_side=8, no_truncate=False, empty_init=False, check_every=1, warm_refine=False,
                 safeguard=False):
        self.mu = np.ascontiguousarray(mu, dtype=np.float64)
        self.nu = np.ascontiguousarray(nu, dtype=np.float64)
        n = self.mu.shape[0]
        opt = _Opt(err_tol, trunc_tau, max_inner_iter, n_threads, schedule, eps_start,
                   coarsest_side, 1 if no_truncate else 0, 1 if empty_init else 0, check_every,
                   1 if warm_refine else 0, 1 if safeguard else 0)
        self._h = C.c_void_p()
        rc = lib().ddo_init(C.byref(self._h), n, _dp(self.mu), _dp(self.nu), eps, cell_size,
                            C.byref(opt))
        if rc:
            msg = self.last_error()
            lib().ddo_free(self._h)
            self._h = None
            raise ValueError(f"ddo_init failed rc={rc}: {msg}")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ddo_free(self._h)
            self._h = None

    def last_error(self):
        return lib().ddo_last_error(self._h).decode()

    def _check(self, rc, what, allow=(OK,)):
        if rc not in allow:
            raise RuntimeError(f"{what} failed rc={rc}: {self.last_error()}")
        return rc

    def set_eps(self, eps):
        return self._check(lib().ddo_set_eps(self._h, eps), "set_eps")

    def set_cost(self, h1=None, h2=None):
        """General separable cost c = h1(|x1-y1|) + h2(|x2-y2|): tables over
        finest-grid pixel differences 0..n-1 in [0,1]^2 cost units; None = |x-y|^2."""
        if h1 is None:
            return self._check(lib().ddo_set_cost(self._h, 0, None, None), "set_cost")
        self._h1 = np.ascontiguousarray(h1, dtype=np.float64)
        self._h2 = np.ascontiguousarray(h2, dtype=np.float64)
        return self._check(lib().ddo_set_cost(self._h, self._h1.size, _dp(self._h1), _dp(self._h2)),
                           "set_cost")

    def iterate(self, k=1):
        return self._check(lib().ddo_iterate(self._h, k), "iterate", (OK, ENOCONV))

    def dual_gap(self):
        """(KL - ||K||, J - ||K||, relative PD gap) of eq. RelPDGap."""
        a, b, r = C.c_double(), C.c_double(), C.c_double()
        self._check(lib().ddo_dual_gap(self._h, C.byref(a), C.byref(b), C.byref(r)), "dual_gap")
        return a.value, b.value, r.value

    def solve_cells(self, part, cells, concurrent=False):
        """Algorithm 2 lines 8-13 for the listed cells of partition part only
        (concurrent: one OpenMP thread per cell, as in a sweep; else one cell
        at a time, each half-iteration's outputs spread over the threads)."""
        cells = np.ascontiguousarray(cells, np.int32)
        iters = np.zeros(max(cells.size, 1), np.int32)
        fn = lib().ddo_solve_cells_par if concurrent else lib().ddo_solve_cells
        self._check(fn(self._h, part, cells.size, cells.ctypes.data, iters.ctypes.data),
                    "solve_cells", (OK, ENOCONV))
        return iters[:cells.size]

    def refine(self):
        return self._check(lib().ddo_refine(self._h), "refine")

    def run_schedule(self):
        return self._check(lib().ddo_run_schedule(self._h), "run_schedule", (OK, ENOCONV))

    def primal_cost(self):
        a, b = C.c_double(), C.c_double()
        self._check(lib().ddo_primal_cost(self._h, C.byref(a), C.byref(b)), "primal_cost")
        return a.value, b.value

    def marginal_error(self):
        a, b = C.c_double(), C.c_double()
        self._check(lib().ddo_marginal_error(self._h, C.byref(a), C.byref(b)), "marginal_error")
        return a.value, b.value

    def fetch_plan_coo(self):
        cnt = C.c_longlong(0)
        self._check(lib().ddo_fetch_plan_coo(self._h, C.byref(cnt), None, None, None), "plan")
        n = cnt.value
        xi = np.zeros(n, np.int32)
        yi = np.zeros(n, np.int32)
        m = np.zeros(n, np.float64)
        self._check(lib().ddo_fetch_plan_coo(self._h, C.byref(cnt), xi.ctypes.data,
                                             yi.ctypes.data, m.ctypes.data), "plan")
        return xi, yi, m

    def plan_dense(self):
        info = self.state_info()
        n2 = info["side"] ** 2
        xi, yi, m = self.fetch_plan_coo()
        P = np.zeros((n2, n2))
        np.add.at(P, (xi, yi), m)
        return P

    def stats(self):
        st = _Stats()
        self._check(lib().ddo_get_stats(self._h, C.byref(st)), "stats")
        return {k: getattr(st, k) for k, _ in _Stats._fields_}

    def state_info(self):
        inf = _Info()
        self._check(lib().ddo_get_state_info(self._h, C.byref(inf)), "state_info")
        return {k: getattr(inf, k) for k, _ in _Info._fields_}

    def get_state(self):
        info = self.state_info()
        nb, side = info["nb"], info["side"]
        boxes = np.zeros((nb * nb, 4), np.int32)
        offs = np.zeros(nb * nb, np.int64)
        vals = np.zeros(max(info["entries"], 1), np.float64)
        aA = np.zeros((side, side))
        aB = np.zeros((side, side))
        self._check(lib().ddo_get_state(self._h, boxes.ctypes.data, offs.ctypes.data,
                                        vals.ctypes.data, aA.ctypes.data, aB.ctypes.data),
                    "get_state")
        return dict(info=info, boxes=boxes, offsets=offs, values=vals[:info["entries"]],
                    alpha_A=aA, alpha_B=aB)

    def set_state(self, st):
        info = st["info"]
        boxes = np.ascontiguousarray(st["boxes"], np.int32)
        offs = np.ascontiguousarray(st["offsets"], np.int64)
        vals = np.ascontiguousarray(st["values"], np.float64)
        if vals.size == 0:
            vals = np.zeros(1)
        aA = np.ascontiguousarray(st["alpha_A"], np.float64)
        aB = np.ascontiguousarray(st["alpha_B"], np.float64)
        self._check(lib().ddo_set_state(self._h, info["side"], info["half_index"],
                                        info["last_partition"], boxes.ctypes.data,
                                        offs.ctypes.data, vals.ctypes.data, aA.ctypes.data,
                                        aB.ctypes.data), "set_state")

    def layer_marginals(self):
        side = self.state_info()["side"]
        mu = np.zeros((side, side))
        nu = np.zeros((side, side))
        lib().ddo_get_layer_marginals(self._h, mu.ctypes.data, nu.ctypes.data)
        return mu, nu

    def basic_marginals_dense(self):
        """nu_i as a dense (nb*nb, side*side) array (small sizes only)."""
        st = self.get_state()
        side = st["info"]["side"]
        nb = st["info"]["nb"]
        out = np.zeros((nb * nb, side, side))
        for i in range(nb * nb):
            y0, x0, hr, hc = st["boxes"][i]
            if hr * hc:
                o = st["offsets"][i]
                out[i, y0:y0 + hr, x0:x0 + hc] = st["values"][o:o + hr * hc].reshape(hr, hc)
        return out.reshape(nb * nb, side * side)
