"""One ctypes harness for the SURVEY.md 8(b) C-ABI, usable on either library:
libdd_gpu.so (the product) or liboracle_dd.so (the oracle's dd_* shim,
oracle/dd_shim.c).  Declares only the entry points both export; the same
call sequence then runs on both and the tests compare the results.
(Test infrastructure: the product package never imports this.)"""
from __future__ import annotations

import ctypes as C

import numpy as np

OK, EINVAL, ENOCONV = 0, 1, 2
SCHED_FIXED, SCHED_LADDER = 0, 1
PLAN_BASIC_MARGINALS, PLAN_COO = 0, 1

COMMON = ["dd_init", "dd_iterate", "dd_set_eps", "dd_refine", "dd_run_schedule", "dd_reset",
          "dd_primal_cost", "dd_dual_gap", "dd_marginal_error", "dd_fetch_plan", "dd_get_stats",
          "dd_get_totals", "dd_reset_totals", "dd_get_state_info", "dd_get_state", "dd_set_state",
          "dd_build_schedule", "dd_synchronize", "dd_free", "dd_last_error", "dd_version"]


class Options(C.Structure):
    _fields_ = [("err_tol", C.c_double), ("trunc_tau", C.c_double),
                ("max_inner_iter", C.c_int), ("check_every", C.c_int), ("n_gpus", C.c_int),
                ("schedule", C.c_int), ("eps_start", C.c_double), ("coarsest_side", C.c_int),
                ("no_truncate", C.c_int), ("flags", C.c_uint), ("device", C.c_int),
                ("pool_capacity", C.c_longlong), ("stream", C.c_void_p),
                ("reserved", C.c_int * 8)]


class Stats(C.Structure):
    _fields_ = [("cells", C.c_longlong), ("iters_sum", C.c_longlong), ("iters_max", C.c_int),
                ("failed", C.c_int), ("err_x_sum", C.c_double), ("entries", C.c_longlong),
                ("ms", C.c_double), ("mufu_ops", C.c_double), ("solve_ms", C.c_double),
                ("launches", C.c_longlong), ("big_cells", C.c_longlong), ("max_box", C.c_int),
                ("reserved_i", C.c_int), ("cluster_cells", C.c_longlong)]


class Info(C.Structure):
    _fields_ = [("side", C.c_int), ("s", C.c_int), ("nb", C.c_int), ("last_partition", C.c_int),
                ("half_index", C.c_longlong), ("entries", C.c_longlong), ("eps", C.c_double)]


def load(path):
    L = C.CDLL(path)
    d, i, ll, p = C.c_double, C.c_int, C.c_longlong, C.c_void_p
    dp = C.POINTER(d)
    L.dd_init.argtypes = [C.POINTER(p), i, p, p, i, d, i, C.POINTER(Options)]
    for n in ("dd_refine", "dd_run_schedule", "dd_reset", "dd_synchronize", "dd_reset_totals", "dd_free"):
        getattr(L, n).argtypes = [p]
    L.dd_iterate.argtypes = [p, i]
    L.dd_set_eps.argtypes = [p, d]
    L.dd_primal_cost.argtypes = [p, dp, dp]
    L.dd_marginal_error.argtypes = [p, dp, dp]
    L.dd_dual_gap.argtypes = [p, dp, dp, dp]
    L.dd_fetch_plan.argtypes = [p, i, p, C.POINTER(C.c_size_t)]
    L.dd_get_stats.argtypes = [p, C.POINTER(Stats)]
    L.dd_get_totals.argtypes = [p, C.POINTER(Stats)]
    L.dd_get_state_info.argtypes = [p, C.POINTER(Info)]
    L.dd_get_state.argtypes = [p, p, p, p, p, p]
    L.dd_set_state.argtypes = [p, i, ll, i, p, p, p, ll, p, p]
    L.dd_build_schedule.argtypes = [i, i, d, d, p, p, p, i]
    L.dd_last_error.argtypes = [p]
    L.dd_last_error.restype = C.c_char_p
    L.dd_version.restype = C.c_char_p
    return L


class Solver:
    """The same calls on either library."""

    def __init__(self, L, mu, nu, eps, s, **kw):
        self.L = L
        o = Options()
        o.err_tol = kw.get("err_tol", 1e-6)
        o.trunc_tau = kw.get("trunc_tau", 1e-15)
        o.max_inner_iter = kw.get("max_inner_iter", 10000)
        o.check_every = kw.get("check_every", 1)
        o.schedule = kw.get("schedule", SCHED_FIXED)
        o.eps_start = kw.get("eps_start", 0.0)
        o.coarsest_side = kw.get("coarsest_side", 8)
        o.reserved[2] = 1 if kw.get("cold_refine", False) else 0
        self.mu = np.ascontiguousarray(mu, np.float64)
        self.nu = np.ascontiguousarray(nu, np.float64)
        self.h = C.c_void_p()
        rc = L.dd_init(C.byref(self.h), self.mu.shape[0], self.mu.ctypes.data, self.nu.ctypes.data, 0, eps, s,
                       C.byref(o))
        if rc:
            msg = L.dd_last_error(self.h)
            L.dd_free(self.h)
            self.h = None
            raise ValueError(f"dd_init rc={rc}: {msg}")

    def close(self):
        if self.h:
            self.L.dd_free(self.h)
            self.h = None

    def rc(self, name, *args):
        return getattr(self.L, name)(self.h, *args)

    def iterate(self, k):
        return self.rc("dd_iterate", k)

    def synchronize(self):
        return self.rc("dd_synchronize")

    def primal_cost(self):
        a, b = C.c_double(), C.c_double()
        assert self.rc("dd_primal_cost", C.byref(a), C.byref(b)) == OK
        return a.value, b.value

    def marginal_error(self):
        a, b = C.c_double(), C.c_double()
        assert self.rc("dd_marginal_error", C.byref(a), C.byref(b)) == OK
        return a.value, b.value

    def stats(self):
        st = Stats()
        rc = self.rc("dd_get_stats", C.byref(st))
        return rc, {k: getattr(st, k) for k, _ in Stats._fields_}

    def info(self):
        inf = Info()
        assert self.rc("dd_get_state_info", C.byref(inf)) == OK
        return {k: getattr(inf, k) for k, _ in Info._fields_}

    def basic_marginals(self):
        """DD_PLAN_BASIC_MARGINALS through dd_fetch_plan, as dense (nb^2, side, side)."""
        inf = self.info()
        n = C.c_size_t(0)
        assert self.rc("dd_fetch_plan", PLAN_BASIC_MARGINALS, None, C.byref(n)) == OK
        buf = np.zeros(n.value, np.uint8)
        assert self.rc("dd_fetch_plan", PLAN_BASIC_MARGINALS, C.c_void_p(buf.ctypes.data), C.byref(n)) == OK
        nb, side = inf["nb"], inf["side"]
        nb2 = nb * nb
        boxes = buf[:16 * nb2].view(np.int32).reshape(nb2, 4)
        offs = buf[16 * nb2:24 * nb2].view(np.int64)
        vals = buf[24 * nb2:].view(np.float64)
        out = np.zeros((nb2, side, side))
        for i in range(nb2):
            y0, x0, hr, hc = boxes[i]
            if hr * hc:
                out[i, y0:y0 + hr, x0:x0 + hc] = vals[offs[i]:offs[i] + hr * hc].reshape(hr, hc)
        return out
