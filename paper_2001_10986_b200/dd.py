"""Thin ctypes binding of libdd_gpu.so (include/dd.h).

Argument marshalling only: every step of the path runs in the CUDA library.
There is no CPU fallback -- if the library or an sm_100 device is missing,
construction raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("DD_LIB", os.path.join(_HERE, "libdd_gpu.so"))   # DD_LIB: diagnostic builds

OK, EINVAL, ENOCONV, ENUMERIC, ECUDA, ENCCL, ENOMEM = 0, 1, 2, 3, 4, 5, 6
COST_SQEUCLID = 0
SCHED_FIXED, SCHED_LADDER = 0, 1
FLAG_DEVICE_INPUT = 1
FLAG_SAFEGUARD = 2
PLAN_BASIC_MARGINALS, PLAN_COO = 0, 1

# every symbol include/dd.h declares (checked by tests/test_abi.py)
EXPORTS = ["dd_init", "dd_iterate", "dd_set_eps", "dd_set_max_inner_iter", "dd_set_cost", "dd_refine", "dd_run_schedule", "dd_run_schedule_batch", "dd_reset",
           "dd_primal_cost", "dd_dual_gap", "dd_marginal_error", "dd_fetch_plan", "dd_get_stats", "dd_get_totals",
           "dd_reset_totals", "dd_set_stripe", "dd_clear_rows", "dd_export_rows",
           "dd_import_rows", "dd_export_rows_slab", "dd_import_rows_slab", "dd_compact", "dd_copy_alpha", "dd_y_accumulate", "dd_y_l1", "dd_phase_profile", "dd_get_cell_stats", "dd_get_state_info", "dd_get_state", "dd_set_state",
           "dd_build_schedule", "dd_measure_mufu_peak", "dd_synchronize", "dd_free",
           "dd_last_error", "dd_version"]


class NotConverged(RuntimeError):
    """DD_ENOCONV: some cell hit max_inner_iter (reading A6); the state stays Y-feasible."""


class Options(C.Structure):
    _fields_ = [("err_tol", C.c_double), ("trunc_tau", C.c_double),
                ("max_inner_iter", C.c_int), ("check_every", C.c_int), ("n_gpus", C.c_int),
                ("schedule", C.c_int), ("eps_start", C.c_double), ("coarsest_side", C.c_int),
                ("no_truncate", C.c_int), ("flags", C.c_uint), ("device", C.c_int),
                ("pool_capacity", C.c_longlong), ("stream", C.c_void_p),
                ("reserved", C.c_int * 8)]


class SweepStats(C.Structure):
    _fields_ = [("cells", C.c_longlong), ("iters_sum", C.c_longlong), ("iters_max", C.c_int),
                ("failed", C.c_int), ("err_x_sum", C.c_double), ("entries", C.c_longlong),
                ("ms", C.c_double), ("mufu_ops", C.c_double), ("solve_ms", C.c_double),
                ("launches", C.c_longlong), ("big_cells", C.c_longlong), ("max_box", C.c_int),
                ("reserved_i", C.c_int), ("cluster_cells", C.c_longlong)]


class StateInfo(C.Structure):
    _fields_ = [("side", C.c_int), ("s", C.c_int), ("nb", C.c_int), ("last_partition", C.c_int),
                ("half_index", C.c_longlong), ("entries", C.c_longlong), ("eps", C.c_double)]


_lib = None


def lib():
    """Load libdd_gpu.so (fails loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"{SO_PATH} missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(SO_PATH)
        d, i, ll, p = C.c_double, C.c_int, C.c_longlong, C.c_void_p
        L.dd_init.argtypes = [C.POINTER(p), i, p, p, i, d, i, C.POINTER(Options)]
        L.dd_iterate.argtypes = [p, i]
        L.dd_set_eps.argtypes = [p, d]
        L.dd_set_cost.argtypes = [p, i, p, p]
        if hasattr(L, "dd_set_max_inner_iter"):
            L.dd_set_max_inner_iter.argtypes = [p, i]
        L.dd_refine.argtypes = [p]
        L.dd_run_schedule.argtypes = [p]
        if hasattr(L, "dd_run_schedule_batch"):     # (older A/B variant builds lack it)
            L.dd_run_schedule_batch.argtypes = [C.POINTER(C.c_void_p), C.c_int]
        L.dd_reset.argtypes = [p]
        L.dd_primal_cost.argtypes = [p, C.POINTER(d), C.POINTER(d)]
        L.dd_marginal_error.argtypes = [p, C.POINTER(d), C.POINTER(d)]
        L.dd_dual_gap.argtypes = [p, C.POINTER(d), C.POINTER(d), C.POINTER(d)]
        L.dd_fetch_plan.argtypes = [p, i, p, C.POINTER(C.c_size_t)]
        L.dd_get_stats.argtypes = [p, C.POINTER(SweepStats)]
        L.dd_get_totals.argtypes = [p, C.POINTER(SweepStats)]
        L.dd_reset_totals.argtypes = [p]
        L.dd_get_cell_stats.argtypes = [p, p, p, p, p, p, p, i]
        L.dd_phase_profile.argtypes = [p, p]
        L.dd_set_stripe.argtypes = [p, i, i]
        L.dd_clear_rows.argtypes = [p, i, i]
        L.dd_export_rows.argtypes = [p, i, i, p, C.POINTER(C.c_size_t)]
        L.dd_import_rows.argtypes = [p, i, i, p, C.c_size_t]
        if hasattr(L, "dd_compact"):
            L.dd_compact.argtypes = [p]
        if hasattr(L, "dd_export_rows_slab"):
            L.dd_export_rows_slab.argtypes = [p, i, i, p, C.c_size_t]
            L.dd_import_rows_slab.argtypes = [p, i, i, p, C.c_size_t]
        L.dd_y_accumulate.argtypes = [p, p]
        L.dd_copy_alpha.argtypes = [p, i, i, i, p, i]
        L.dd_y_l1.argtypes = [p, p, C.POINTER(d)]
        L.dd_get_state_info.argtypes = [p, C.POINTER(StateInfo)]
        L.dd_get_state.argtypes = [p, p, p, p, p, p]
        L.dd_set_state.argtypes = [p, i, ll, i, p, p, p, ll, p, p]
        L.dd_build_schedule.argtypes = [i, i, d, d, p, p, p, i]
        L.dd_measure_mufu_peak.argtypes = [i, C.POINTER(d)]
        L.dd_synchronize.argtypes = [p]
        L.dd_free.argtypes = [p]
        L.dd_last_error.argtypes = [p]
        L.dd_last_error.restype = C.c_char_p
        L.dd_version.restype = C.c_char_p
        _lib = L
    return _lib


def build_schedule(n_final, coarsest_side, kappa_final, eps_start=0.0):
    m = 512
    side = (C.c_int * m)()
    kap = (C.c_double * m)()
    sw = (C.c_int * m)()
    k = lib().dd_build_schedule(n_final, coarsest_side, kappa_final, eps_start,
                                C.cast(side, C.c_void_p), C.cast(kap, C.c_void_p),
                                C.cast(sw, C.c_void_p), m)
    return [(side[j], kap[j], sw[j]) for j in range(min(k, m))]


def measure_mufu_peak(device=0):
    v = C.c_double(0)
    rc = lib().dd_measure_mufu_peak(device, C.byref(v))
    if rc:
        raise RuntimeError(f"dd_measure_mufu_peak rc={rc}")
    return v.value


def run_schedule_batch(dds, check=True):
    """dd_run_schedule_batch: the full schedule of several independent problems
    (contexts on distinct streams), sweeps enqueued round-robin, one wait.
    check=False accepts DD_ENOCONV (flagged cells, reading A6) and returns it."""
    arr = (C.c_void_p * len(dds))(*[d._h.value for d in dds])
    rc = lib().dd_run_schedule_batch(arr, len(dds))
    if rc != OK:
        return dds[0]._check(rc, "run_schedule_batch", (OK,) if check else (OK, ENOCONV))
    return rc


class DD:
    """One libdd_gpu context.  Same call names as the oracle's binding."""

    def __init__(self, mu, nu, eps, cell_size, *, err_tol=1e-6, trunc_tau=1e-15,
                 max_inner_iter=10000, schedule=SCHED_FIXED, eps_start=0.0, coarsest_side=8,
                 no_truncate=False, device=0, pool_capacity=0, stream=None, device_input=False,
                 bcap_main=0, bcap_big=0, cold_refine=False, check_every=1, cluster=0,
                 cluster_theta=0, n_clusters=0, safeguard=False, bcap_onchip=0):
        opt = Options()
        opt.err_tol = err_tol
        opt.trunc_tau = trunc_tau
        opt.max_inner_iter = max_inner_iter
        opt.check_every = check_every
        opt.schedule = schedule
        opt.eps_start = eps_start
        opt.coarsest_side = coarsest_side
        opt.no_truncate = 1 if no_truncate else 0
        opt.device = device
        opt.pool_capacity = pool_capacity
        opt.stream = stream
        opt.reserved[0] = bcap_main
        opt.reserved[1] = bcap_big
        opt.reserved[2] = 1 if cold_refine else 0
        opt.reserved[3] = cluster            # K1 cluster tier: 0 off, 2 auto (long poles), 1 every big-path cell
        opt.reserved[4] = cluster_theta      # routing threshold in % (0 -> default)
        opt.reserved[5] = n_clusters         # persistent clusters (0 -> default)
        opt.reserved[6] = bcap_onchip        # testing: larger boxes -> tier G (global-memory layouts)
        opt.flags = FLAG_SAFEGUARD if safeguard else 0
        self._h = C.c_void_p()
        if device_input:
            # mu, nu: objects exposing data_ptr() (device fp64) and a square shape
            opt.flags |= FLAG_DEVICE_INPUT
            n = int(mu.shape[0])
            pm, pn = C.c_void_p(mu.data_ptr()), C.c_void_p(nu.data_ptr())
            self._keep = (mu, nu)
        else:
            mu = np.ascontiguousarray(mu, dtype=np.float64)
            nu = np.ascontiguousarray(nu, dtype=np.float64)
            n = mu.shape[0]
            pm, pn = C.c_void_p(mu.ctypes.data), C.c_void_p(nu.ctypes.data)
            self._keep = (mu, nu)
        rc = lib().dd_init(C.byref(self._h), n, pm, pn, COST_SQEUCLID, eps, cell_size, C.byref(opt))
        if rc:
            msg = self.last_error()
            lib().dd_free(self._h)
            self._h = None
            if rc == EINVAL:
                raise ValueError(f"dd_init rc={rc}: {msg}")
            raise RuntimeError(f"dd_init rc={rc}: {msg}")
        self.n = n

    def __del__(self):
        if getattr(self, "_h", None):
            lib().dd_free(self._h)
            self._h = None

    def close(self):
        self.__del__()

    def last_error(self):
        return lib().dd_last_error(self._h).decode()

    def _check(self, rc, what, allow=(OK,)):
        if rc not in allow:
            if rc == ENOCONV:
                raise NotConverged(f"{what}: {self.last_error()}")
            raise RuntimeError(f"{what} failed rc={rc}: {self.last_error()}")
        return rc

    def set_eps(self, eps):
        return self._check(lib().dd_set_eps(self._h, eps), "set_eps")

    def set_cost(self, h1=None, h2=None):
        """General separable cost c = h1(|x1-y1|) + h2(|x2-y2|): tables over
        finest-grid pixel differences 0..n-1, [0,1]^2 cost units; None = |x-y|^2."""
        if h1 is None:
            return self._check(lib().dd_set_cost(self._h, 0, None, None), "set_cost")
        h1 = np.ascontiguousarray(h1, dtype=np.float64)
        h2 = np.ascontiguousarray(h2, dtype=np.float64)
        return self._check(lib().dd_set_cost(self._h, h1.size, h1.ctypes.data_as(C.c_void_p),
                                             h2.ctypes.data_as(C.c_void_p)), "set_cost")

    def set_max_inner_iter(self, k):
        return self._check(lib().dd_set_max_inner_iter(self._h, k), "set_max_inner_iter")

    def iterate(self, k=1, check=True):
        return self._check(lib().dd_iterate(self._h, k), "iterate", (OK,) if check else (OK, ENOCONV))

    def refine(self):
        return self._check(lib().dd_refine(self._h), "refine")

    def run_schedule(self, check=True):
        return self._check(lib().dd_run_schedule(self._h), "run_schedule", (OK,) if check else (OK, ENOCONV))

    def reset(self):
        return self._check(lib().dd_reset(self._h), "reset")

    def synchronize(self, check=True):
        return self._check(lib().dd_synchronize(self._h), "synchronize", (OK,) if check else (OK, ENOCONV))

    def primal_cost(self):
        a, b = C.c_double(), C.c_double()
        self._check(lib().dd_primal_cost(self._h, C.byref(a), C.byref(b)), "primal_cost")
        return a.value, b.value

    def dual_gap(self):
        """(KL - ||K||, J - ||K||, relative PD gap) of eq. RelPDGap."""
        a, b, r = C.c_double(), C.c_double(), C.c_double()
        self._check(lib().dd_dual_gap(self._h, C.byref(a), C.byref(b), C.byref(r)), "dual_gap")
        return a.value, b.value, r.value

    def marginal_error(self):
        a, b = C.c_double(), C.c_double()
        self._check(lib().dd_marginal_error(self._h, C.byref(a), C.byref(b)), "marginal_error")
        return a.value, b.value

    def _stats(self, fn):
        st = SweepStats()
        self._check(fn(self._h, C.byref(st)), "stats", (OK, ENOCONV))
        out = {k: getattr(st, k) for k, _ in SweepStats._fields_}
        out["fallbacks"] = out.pop("reserved_i")
        return out

    def stats(self):
        return self._stats(lib().dd_get_stats)

    def totals(self):
        return self._stats(lib().dd_get_totals)

    def reset_totals(self):
        return self._check(lib().dd_reset_totals(self._h), "reset_totals")

    # ---- multi-GPU stripe primitives (device buffers: objects with data_ptr())
    def set_stripe(self, row_lo, row_hi):
        return self._check(lib().dd_set_stripe(self._h, row_lo, row_hi), "set_stripe")

    def clear_rows(self, row, nrows):
        return self._check(lib().dd_clear_rows(self._h, row, nrows), "clear_rows")

    def export_rows_size(self, row, nrows):
        nbytes = C.c_size_t(0)
        self._check(lib().dd_export_rows(self._h, row, nrows, None, C.byref(nbytes)), "export_rows")
        return nbytes.value

    def export_rows(self, row, nrows, dev_buf):
        nbytes = C.c_size_t(int(dev_buf.numel() * dev_buf.element_size()))
        self._check(lib().dd_export_rows(self._h, row, nrows, C.c_void_p(dev_buf.data_ptr()),
                                         C.byref(nbytes)), "export_rows")
        return nbytes.value

    def import_rows(self, row, nrows, dev_buf, nbytes):
        return self._check(lib().dd_import_rows(self._h, row, nrows, C.c_void_p(dev_buf.data_ptr()), nbytes),
                           "import_rows")

    def compact(self):
        return self._check(lib().dd_compact(self._h), "compact")

    def export_rows_slab(self, row, nrows, slab):
        """Asynchronous export into a fixed-capacity device slab (uint8 tensor)."""
        return self._check(lib().dd_export_rows_slab(self._h, row, nrows, C.c_void_p(slab.data_ptr()),
                                                     slab.numel() * slab.element_size()), "export_rows_slab")

    def import_rows_slab(self, row, nrows, slab):
        return self._check(lib().dd_import_rows_slab(self._h, row, nrows, C.c_void_p(slab.data_ptr()),
                                                     slab.numel() * slab.element_size()), "import_rows_slab")

    def copy_alpha(self, partition, row0, nrows, dev_buf, to_ctx):
        return self._check(lib().dd_copy_alpha(self._h, partition, row0, nrows, C.c_void_p(dev_buf.data_ptr()),
                                               1 if to_ctx else 0), "copy_alpha")

    def y_accumulate(self, dev_acc):
        return self._check(lib().dd_y_accumulate(self._h, C.c_void_p(dev_acc.data_ptr())), "y_accumulate")

    def y_l1(self, dev_acc):
        v = C.c_double(0)
        self._check(lib().dd_y_l1(self._h, C.c_void_p(dev_acc.data_ptr()), C.byref(v)), "y_l1")
        return v.value

    def phase_profile(self):
        """K1 per-phase cycle counters since the last call ([2][16] uint64; see dd.h)."""
        out = np.zeros(32, np.uint64)
        self._check(lib().dd_phase_profile(self._h, out.ctypes.data), "phase_profile")
        return out.reshape(2, 16)

    def cell_stats(self, flags=False, err=False):
        """Per composite cell of the last sweep: (iters, box_side, mufu_ops, kcycles[, flags][, err_x]) arrays."""
        n = lib().dd_get_cell_stats(self._h, None, None, None, None, None, None, 0)
        if n < 0:
            raise RuntimeError(f"dd_get_cell_stats rc={-n}: {self.last_error()}")
        it = np.zeros(max(n, 1), np.int32)
        bx = np.zeros(max(n, 1), np.int32)
        mf = np.zeros(max(n, 1), np.float64)
        kc = np.zeros(max(n, 1), np.int32)
        fl = np.zeros(max(n, 1), np.int32)
        ex = np.zeros(max(n, 1), np.float32)
        lib().dd_get_cell_stats(self._h, it.ctypes.data, bx.ctypes.data, mf.ctypes.data, kc.ctypes.data,
                                fl.ctypes.data, ex.ctypes.data, n)
        out = (it[:n], bx[:n], mf[:n], kc[:n])
        if flags:
            out = out + (fl[:n],)
        if err:
            out = out + (ex[:n].astype(np.float64),)
        return out

    def state_info(self):
        inf = StateInfo()
        self._check(lib().dd_get_state_info(self._h, C.byref(inf)), "state_info")
        return {k: getattr(inf, k) for k, _ in StateInfo._fields_}

    def get_state(self):
        info = self.state_info()
        nb, side = info["nb"], info["side"]
        boxes = np.zeros((nb * nb, 4), np.int32)
        offs = np.zeros(nb * nb, np.int64)
        vals = np.zeros(max(info["entries"], 1), np.float64)
        aA = np.zeros((side, side))
        aB = np.zeros((side, side))
        self._check(lib().dd_get_state(self._h, boxes.ctypes.data, offs.ctypes.data, vals.ctypes.data,
                                       aA.ctypes.data, aB.ctypes.data), "get_state")
        return dict(info=info, boxes=boxes, offsets=offs, values=vals[:info["entries"]],
                    alpha_A=aA, alpha_B=aB)

    def set_state(self, st):
        info = st["info"]
        boxes = np.ascontiguousarray(st["boxes"], np.int32)
        offs = np.ascontiguousarray(st["offsets"], np.int64)
        vals = np.ascontiguousarray(st["values"], np.float64)
        nv = vals.size
        if nv == 0:
            vals = np.zeros(1)
        aA = np.ascontiguousarray(st["alpha_A"], np.float64)
        aB = np.ascontiguousarray(st["alpha_B"], np.float64)
        self._check(lib().dd_set_state(self._h, info["side"], info["half_index"], info["last_partition"],
                                       boxes.ctypes.data, offs.ctypes.data, vals.ctypes.data, nv,
                                       aA.ctypes.data, aB.ctypes.data), "set_state")

    def fetch_plan_coo(self):
        nbytes = C.c_size_t(0)
        self._check(lib().dd_fetch_plan(self._h, PLAN_COO, None, C.byref(nbytes)), "fetch_plan")
        n = nbytes.value // 16
        buf = np.zeros(nbytes.value, np.uint8)
        self._check(lib().dd_fetch_plan(self._h, PLAN_COO, buf.ctypes.data, C.byref(nbytes)), "fetch_plan")
        xi = buf[:4 * n].view(np.int32)
        yi = buf[4 * n:8 * n].view(np.int32)
        m = buf[8 * n:].view(np.float64)
        return xi, yi, m

    def plan_dense(self):
        side = self.state_info()["side"]
        xi, yi, m = self.fetch_plan_coo()
        P = np.zeros((side * side, side * side))
        np.add.at(P, (xi, yi), m)
        return P

    def basic_marginals_dense(self):
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
