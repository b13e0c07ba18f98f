"""Multi-GPU driver: one problem striped over ranks (DESIGN.md
"Multi-GPU").  Host orchestration only -- every sweep, the row packing and
the marginal accounting run in libdd_gpu.so; the boundary rows move as
device byte buffers through a transport:

  * TorchTransport: torch.distributed point-to-point (NCCL over NVLink on a
    GPU box, gloo for the CPU protocol tests), plus all-reduce of the
    statistics;
  * LocalTransport: several contexts of one process on one device
    ("virtual stripes"), used to check the striped algorithm against a
    single context.

Stripe geometry (rows are basic-cell rows of the current layer, nb of them):
rank p owns rows [R_p, R_p+1) with even R_p.  It solves the A-cells whose
rows lie in its stripe and the B-cells whose lower row 2q lies in it (plus
the last, one-row B row for the bottom rank).  Per B-sweep exactly one row
crosses each stripe boundary twice: row R_p - 1 moves from rank p-1 to
rank p before the sweep and back after it (P:1566-1569 cell shapes).
Layers with fewer than two basic rows per rank run replicated (every rank
does the whole layer; no exchange).  A-sweeps need no exchange.
"""
from __future__ import annotations

import numpy as np

from .dd import DD, build_schedule


# ------------------------------------------------------------------ geometry --
def stripe_bounds(nb: int, nranks: int):
    """Even row bounds [R_0 = 0, ..., R_N = nb] or None (replicated layer)."""
    if nranks <= 1 or nb < 2 * nranks:
        return None
    half = nb // 2                       # A-cell rows, distributed as evenly as possible
    b = [2 * ((p * half) // nranks) for p in range(nranks + 1)]
    b[-1] = nb
    return b


def balanced_bounds(nb: int, row_work, nranks: int, old=None):
    """Cost-aware even bounds: split the per-A-cell-row predicted work
    (row_work[q], q < nb/2) into nranks contiguous runs of nearly equal
    work (greedy on the prefix sums).  With `old` bounds, each new bound
    stays strictly between its old neighbours, so a basic row moves at most
    one rank per rebalance."""
    half = nb // 2
    w = np.asarray(row_work, dtype=np.float64)
    c = np.concatenate([[0.0], np.cumsum(w)])
    tot = c[-1]
    if not tot > 0:
        return stripe_bounds(nb, nranks)
    b = [0]
    for r in range(1, nranks):
        q = int(np.searchsorted(c, tot * r / nranks))
        if q > 0 and abs(c[q - 1] - tot * r / nranks) < abs(c[q] - tot * r / nranks):
            q -= 1
        lo_q = b[-1] // 2 + 1
        hi_q = half - (nranks - r)
        if old is not None:
            lo_q = max(lo_q, old[r - 1] // 2 + 1)
            hi_q = min(hi_q, old[r + 1] // 2 - 1)
        b.append(2 * min(max(q, lo_q), max(lo_q, hi_q)))
    b.append(nb)
    return b


def owned_cell_rows(nb: int, part: int, lo: int, hi: int):
    """Partition cell rows [q0, q1) solved by the stripe [lo, hi) (engine.cu cell_rows)."""
    q0 = lo // 2
    q1 = hi // 2 + (1 if (part == 2 and hi == nb) else 0)
    return q0, q1


def cell_basic_rows(nb: int, part: int, q: int):
    """Basic rows covered by partition cell row q."""
    if part == 1:
        return [2 * q, 2 * q + 1]
    return [r for r in (2 * q - 1, 2 * q) if 0 <= r < nb]


# ----------------------------------------------------------------- transports --
class LocalTransport:
    """All ranks in this process: messages are handed over directly."""

    def __init__(self, nranks: int):
        self.nranks = nranks

    def exchange(self, sends, expects):
        """sends: [(src, dst, tensor)]; expects: [(src, dst)] -> {(src, dst): tensor}."""
        got = {(s, d): t for s, d, t in sends}
        return {k: got[k] for k in expects}

    def exchange_fixed(self, sends, expects, recv_bufs):
        """Fixed-size slabs: the receiver reads the sender's slab (contexts on
        different streams of one device: order them by a device sync)."""
        import torch
        torch.cuda.synchronize()
        got = {(s, d): t for s, d, t in sends}
        return {k: got[k] for k in expects}

    def allreduce_sum(self, t):
        return t

    def allreduce_max(self, t):
        return t


class TorchTransport:
    """torch.distributed point-to-point + all-reduce (one rank per process)."""

    def __init__(self, dist, rank: int, nranks: int, device, staging=None):
        self.dist = dist
        self.rank = rank
        self.nranks = nranks
        self.device = device
        self.staging = staging          # "cpu": host-staged buffers (gloo); None: device buffers (NCCL)

    def exchange(self, sends, expects):
        if self.staging:
            cpu = TorchTransport(self.dist, self.rank, self.nranks, self.staging)
            got = cpu.exchange([(s, d, t.to(self.staging)) for s, d, t in sends], expects)
            return {k: v.to(self.device) for k, v in got.items()}
        import torch
        d = self.dist
        # 1) sizes
        ops, hdr_in = [], {}
        for s, dst, t in sends:
            assert s == self.rank
            ops.append(d.P2POp(d.isend, torch.tensor([t.numel()], dtype=torch.int64, device=self.device), dst))
        for s, dst in expects:
            assert dst == self.rank
            h = torch.zeros(1, dtype=torch.int64, device=self.device)
            hdr_in[(s, dst)] = h
            ops.append(d.P2POp(d.irecv, h, s))
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()
        # 2) payloads
        ops, out = [], {}
        for s, dst, t in sends:
            ops.append(d.P2POp(d.isend, t, dst))
        for k, h in hdr_in.items():
            buf = torch.empty(int(h.item()), dtype=torch.uint8, device=self.device)
            out[k] = buf
            ops.append(d.P2POp(d.irecv, buf, k[0]))
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()
        return out

    def exchange_fixed(self, sends, expects, recv_bufs):
        """One round of fixed-size slabs (NCCL needs matching counts; the
        slab's header carries the real size): no size round, no .item().
        work.wait() orders the current stream after the NCCL ops on the
        device -- no host synchronisation."""
        if self.staging:
            cpu = TorchTransport(self.dist, self.rank, self.nranks, self.staging)
            rb = {k: v.to(self.staging) for k, v in recv_bufs.items()}
            got = cpu.exchange_fixed([(s, d, t.to(self.staging)) for s, d, t in sends], expects, rb)
            for k, v in got.items():
                recv_bufs[k].copy_(v)
            return recv_bufs
        d = self.dist
        ops = [d.P2POp(d.isend, t, dst) for s, dst, t in sends]
        ops += [d.P2POp(d.irecv, recv_bufs[k], k[0]) for k in expects]
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()
        return {k: recv_bufs[k] for k in expects}

    def _reduce(self, t, op):
        if self.staging:
            h = t.to(self.staging)
            self.dist.all_reduce(h, op=op)
            t.copy_(h.to(t.device))
            return t
        self.dist.all_reduce(t, op=op)
        return t

    def allreduce_sum(self, t):
        return self._reduce(t, self.dist.ReduceOp.SUM)

    def allreduce_max(self, t):
        return self._reduce(t, self.dist.ReduceOp.MAX)


# ------------------------------------------------------------------- driver --
class StripedRun:
    """Drive one problem over `nranks` stripes.

    ranks: list of (rank, DD) owned by this process (one entry under
    torch.distributed, all ranks for LocalTransport); every DD must be in
    DD_SCHED_LADDER or FIXED mode on the same inputs."""

    def __init__(self, ranks, nranks: int, transport, device="cuda", slab_factor: float = 2.0,
                 cost_aware: bool = True):
        self.ranks = list(ranks)
        self.nranks = nranks
        self.tr = transport
        self.device = device
        self.half_index = 0
        self.bounds = None
        self.nb = None
        self.exchanged_bytes = 0
        self.cells_solved = 0
        self.slab_factor = slab_factor
        self.cost_aware = cost_aware
        self.a_work = None               # per A-cell row work of the last recorded A-sweep
        self.rebalances = 0
        self.slab_bytes = 0
        self.slabs = {}                  # (rank, "send"|"recv") -> uint8 device tensor

    # -- layer setup
    def _layer(self, prev=None):
        info = self.ranks[0][1].state_info()
        nb_prev = self.nb
        self.nb = info["nb"]
        if prev is not None and self.nb == 2 * nb_prev:
            # a striped coarse layer refines into its children only: the fine
            # stripes are the coarse ones doubled (each rank holds exactly the
            # refined rows of its own coarse rows, eq. FineBasicMarginals)
            self.bounds = [2 * x for x in prev]
        else:
            self.bounds = stripe_bounds(self.nb, self.nranks)
        for r, dd in self.ranks:
            if self.bounds is None:
                dd.set_stripe(0, 0)
            else:
                dd.set_stripe(self.bounds[r], self.bounds[r + 1])
        if self.bounds is not None:
            self._size_slabs()

    def _size_slabs(self):
        """Once per layer (the layer change synchronises anyway): the slab
        capacity = slab_factor x the largest boundary-row payload of the
        refined state, the same on every rank (max all-reduce); rounded up
        to 1 MiB.  An exchange that outgrows it is reported by the library
        (DD_ENOMEM at the next dd_synchronize), never truncated silently."""
        import torch
        b, N = self.bounds, self.nranks
        need = 0
        for r, dd in self.ranks:
            rows = ([b[r + 1] - 1] if r < N - 1 else []) + ([b[r] - 1] if r > 0 else [])
            for row in rows:
                need = max(need, dd.export_rows_size(row, 1))
        t = self.tr.allreduce_max(torch.tensor([float(need)], dtype=torch.float64, device=self.device))
        need = int(t.item())
        cap = int(need * self.slab_factor) + (1 << 16)
        cap = ((cap + (1 << 20) - 1) >> 20) << 20
        if cap != self.slab_bytes:
            self.slab_bytes = cap
            self.slabs = {}
            for r, _ in self.ranks:
                for kind in ("send", "recv_lo", "recv_hi"):
                    self.slabs[(r, kind)] = torch.empty(cap, dtype=torch.uint8, device=self.device)

    def start(self):
        """Call after init / reset (coarsest layer) or after a refine."""
        self._layer()

    def _gather_alpha(self):
        """Every rank needs the potentials of the whole layer to glue them
        (dd_refine): A-cell potentials come from the A-cell's owner,
        B-cell potentials from the B-cell's owner (basic row r lies in B-cell
        row (r + 1) // 2); one all-reduce per partition of a zero-padded image."""
        import torch
        info = self.ranks[0][1].state_info()
        side, s, nb = info["side"], info["s"], info["nb"]
        b = self.bounds
        for part in (1, 2):
            full = torch.zeros(side * side, dtype=torch.float64, device=self.device)
            for r, dd in self.ranks:
                if part == 1:
                    rows = range(b[r], b[r + 1])
                else:
                    q0, q1 = owned_cell_rows(nb, 2, b[r], b[r + 1])
                    rows = [x for q in range(q0, q1) for x in cell_basic_rows(nb, 2, q)]
                r0, r1 = min(rows) * s, (max(rows) + 1) * s
                seg = torch.empty((r1 - r0) * side, dtype=torch.float64, device=self.device)
                dd.copy_alpha(part, r0, r1 - r0, seg, to_ctx=False)
                full[r0 * side:r1 * side] += seg
            full = self.tr.allreduce_sum(full)
            for _, dd in self.ranks:
                dd.copy_alpha(part, 0, side, full, to_ctx=True)

    def refine(self):
        prev = self.bounds
        if prev is not None:
            self._gather_alpha()
            for _, dd in self.ranks:
                dd.set_stripe(0, 0)          # alpha is now global: dd_refine glues it
        for _, dd in self.ranks:
            dd.refine()
        self._layer(prev)

    def set_eps(self, eps):
        for _, dd in self.ranks:
            dd.set_eps(eps)

    # -- one sweep with the boundary-row exchange of the B partition
    def _export(self, dd, row):
        import torch
        n = dd.export_rows_size(row, 1)
        buf = torch.empty(n, dtype=torch.uint8, device=self.device)
        dd.export_rows(row, 1, buf)
        self.exchanged_bytes += n
        return buf

    def _pass_rows(self, down: bool):
        """down: row hi-1 of rank p -> rank p+1 (before a B-sweep);
        up: row lo-1 of rank p -> rank p-1 (after it).  Fixed-capacity slabs,
        packed and unpacked on the device (dd_export_rows_slab /
        dd_import_rows_slab), one send/recv round: no host synchronisation."""
        b, N = self.bounds, self.nranks
        sends, expects, recv = [], [], {}
        for r, dd in self.ranks:
            if down and r < N - 1:
                row = b[r + 1] - 1
                dd.export_rows_slab(row, 1, self.slabs[(r, "send")])
                dd.clear_rows(row, 1)
                sends.append((r, r + 1, self.slabs[(r, "send")]))
            if not down and r > 0:
                row = b[r] - 1
                dd.export_rows_slab(row, 1, self.slabs[(r, "send")])
                dd.clear_rows(row, 1)
                sends.append((r, r - 1, self.slabs[(r, "send")]))
            if down and r > 0:
                expects.append((r - 1, r))
                recv[(r - 1, r)] = self.slabs[(r, "recv_lo")]
            if not down and r < N - 1:
                expects.append((r + 1, r))
                recv[(r + 1, r)] = self.slabs[(r, "recv_hi")]
        self.exchanged_bytes += self.slab_bytes * len(sends)
        got = self.tr.exchange_fixed(sends, expects, recv)
        for r, dd in self.ranks:
            if down and r > 0:
                dd.import_rows_slab(b[r] - 1, 1, got[(r - 1, r)])
            if not down and r < N - 1:
                dd.import_rows_slab(b[r + 1] - 1, 1, got[(r + 1, r)])

    def sweep(self, record=False):
        part = 1 if self.half_index % 2 == 0 else 2
        striped = self.bounds is not None
        nca = self.nb // 2 if part == 1 else self.nb // 2 + 1
        self.cells_solved += nca * nca          # whole-problem cell solves (replicas counted once)
        if striped and part == 2:
            self._pass_rows(down=True)
        for _, dd in self.ranks:
            dd.iterate(1)
        if striped and part == 2:
            self._pass_rows(down=False)
        if record and striped and part == 1:
            self._record_a_work()
        self.half_index += 1

    # -- cost-aware stripes (tools/stripe_balance.py)
    def _record_a_work(self):
        """Per A-cell row: the algorithmic MUFU ops of the A-sweep just done
        (each rank holds its own cells' counts; summed over ranks).  One host
        synchronisation per eps stage, outside the exchange path."""
        import torch
        na = self.nb // 2
        w = np.zeros(na)
        for _, dd in self.ranks:
            _, _, mf, _ = dd.cell_stats()
            w += mf.reshape(na, na).sum(1)
        t = self.tr.allreduce_sum(torch.tensor(w, dtype=torch.float64, device=self.device))
        self.a_work = (self.nb, t.cpu().numpy())

    def rebalance(self):
        """Before an A-sweep: move the stripe bounds to balance the recorded
        A-row work (a row moves at most one rank).  Rows change owner with
        their boxes (dd_export_rows / dd_import_rows + dd_compact); the
        potentials of both partitions are gathered first, so every rank holds
        the warm start of the cells it gains.  Per-cell arithmetic is
        unchanged: the result stays bit-identical to one context."""
        if self.bounds is None or self.a_work is None or not self.cost_aware:
            return False
        nbw, w = self.a_work
        if nbw != self.nb:                        # recorded on the coarser layer: split each row in two
            w = np.repeat(w / 2.0, self.nb // nbw)
        old = list(self.bounds)
        new = balanced_bounds(self.nb, w, self.nranks, old)
        if new == old:
            return False
        self._gather_alpha()
        for _, dd in self.ranks:
            dd.compact()                          # frees the halo slots (the returned boundary row)
        b, N = old, self.nranks
        sends, expects, meta = [], [], []
        for p in range(1, N):
            if new[p] > old[p]:                   # rows [old_p, new_p) go up: p -> p-1
                lo, cnt, src, dst = old[p], new[p] - old[p], p, p - 1
            elif new[p] < old[p]:                 # rows [new_p, old_p) go down: p-1 -> p
                lo, cnt, src, dst = new[p], old[p] - new[p], p - 1, p
            else:
                continue
            meta.append((lo, cnt, src, dst))
        for lo, cnt, src, dst in meta:
            for r, dd in self.ranks:
                if r == src:
                    buf = self._export_n(dd, lo, cnt)
                    sends.append((src, dst, buf))
            if any(r == dst for r, _ in self.ranks):
                expects.append((src, dst))
        got = self.tr.exchange(sends, expects)
        for lo, cnt, src, dst in meta:
            for r, dd in self.ranks:
                if r == dst:
                    buf = got[(src, dst)]
                    dd.import_rows(lo, cnt, buf, buf.numel())   # old stripe set: slot by side
        self.bounds = new
        for r, dd in self.ranks:
            dd.set_stripe(new[r], new[r + 1])
            dd.compact()
        self.rebalances += 1
        self._size_slabs()
        return True

    def _export_n(self, dd, row, nrows):
        import torch
        n = dd.export_rows_size(row, nrows)
        buf = torch.empty(n, dtype=torch.uint8, device=self.device)
        dd.export_rows(row, nrows, buf)
        self.exchanged_bytes += n
        return buf

    def iterate(self, k, record_last_a=False):
        for j in range(k):
            last_a = record_last_a and (j == k - 1 or j == k - 2) and self.half_index % 2 == 0
            self.sweep(record=last_a)

    def run_schedule(self, n, coarsest, kappa_final, eps_start=0.0):
        self.half_index = 0
        self.a_work = None
        self.start()
        side = self.ranks[0][1].state_info()["side"]
        for sd, kappa, sweeps in build_schedule(n, coarsest, kappa_final, eps_start):
            while side < sd:
                self.refine()
                side *= 2
            self.set_eps(kappa / sd**2)
            if self.half_index % 2 == 0:
                self.rebalance()               # cost-aware bounds from the last stage's A-sweep
            self.iterate(sweeps, record_last_a=self.cost_aware)

    # -- whole-problem quantities (sums over ranks)
    def totals(self):
        """Statistics summed over ranks (a replicated coarse layer counts once
        per rank; `cells_solved` counts whole-problem cell solves)."""
        import torch
        keys = ["cells", "iters_sum", "failed", "err_x_sum", "mufu_ops"]
        v = np.zeros(len(keys))
        m = np.zeros(2)
        for _, dd in self.ranks:
            t = dd.totals()
            v += [t[k] for k in keys]
            m = np.maximum(m, [t["iters_max"], t["max_box"]])
        tv = self.tr.allreduce_sum(torch.tensor(v, dtype=torch.float64, device=self.device))
        tm = self.tr.allreduce_max(torch.tensor(m, dtype=torch.float64, device=self.device))
        out = dict(zip(keys, tv.cpu().numpy().tolist()))
        out["iters_max"], out["max_box"] = tm.cpu().numpy().tolist()
        return out

    def _halo_in(self):
        """Evaluation of the last partition (A15) on a stripe needs the plan of
        its cells as swept: after a B-sweep the row above the stripe went
        back to its owner, so fetch a read-only copy (the owner keeps it)."""
        if self.bounds is None or self.half_index == 0 or self.half_index % 2 == 1:
            return False                  # replicated, or the last sweep was an A-sweep
        b, N = self.bounds, self.nranks
        sends = [(r, r + 1, self._export(dd, b[r + 1] - 1)) for r, dd in self.ranks if r < N - 1]
        expects = [(r - 1, r) for r, _ in self.ranks if r > 0]
        got = self.tr.exchange(sends, expects)
        for r, dd in self.ranks:
            if r > 0:
                buf = got[(r - 1, r)]
                dd.import_rows(b[r] - 1, 1, buf, buf.numel())
        return True

    def _halo_out(self):
        for r, dd in self.ranks:
            if r > 0:
                dd.clear_rows(self.bounds[r] - 1, 1)

    def primal_cost(self):
        import torch
        v = np.zeros(2)
        halo = self._halo_in()
        for _, dd in self.ranks:
            v += dd.primal_cost()
        if halo:
            self._halo_out()
        t = self.tr.allreduce_sum(torch.tensor(v, dtype=torch.float64, device=self.device))
        if self.bounds is None:           # replicated layer: every rank evaluated every cell
            t = t / self.nranks
        return tuple(t.cpu().numpy().tolist())

    def marginal_error(self):
        import torch
        side = self.ranks[0][1].state_info()["side"]
        lx = 0.0
        acc = torch.zeros(side * side, dtype=torch.int64, device=self.device)
        replicated = self.bounds is None
        for i, (_, dd) in enumerate(self.ranks):       # owned rows only (before the halo copy)
            if not replicated or (i == 0 and self._is_root()):
                dd.y_accumulate(acc)
        halo = self._halo_in()
        for _, dd in self.ranks:
            lx += dd.marginal_error()[0]
        if halo:
            self._halo_out()
        lxt = self.tr.allreduce_sum(torch.tensor([lx], dtype=torch.float64, device=self.device))
        if replicated:                    # every rank holds the whole layer: count it once
            lxt = lxt / self.nranks
        acc = self.tr.allreduce_sum(acc)
        ly = self.ranks[0][1].y_l1(acc)
        return float(lxt.item()), ly

    def _is_root(self):
        return any(r == 0 for r, _ in self.ranks)

    def basic_marginals_dense(self):
        """Union of the ranks' owned rows (LocalTransport / tests)."""
        out = None
        for _, dd in self.ranks:
            d = dd.basic_marginals_dense()
            out = d if out is None else out + d
        if self.bounds is None:
            out = out / len(self.ranks)
        return out
