"""Host logic of the multi-GPU stripe path on CPU: stripe
geometry, cell ownership, the boundary-row exchange schedule, and the
torch.distributed transport protocol over gloo with world_size 2."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2001_10986_b200.striped import (TorchTransport, cell_basic_rows, owned_cell_rows,
                                           stripe_bounds)


@pytest.mark.parametrize("nb", [4, 8, 16, 32, 64, 256])
@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_stripe_bounds(nb, nranks):
    b = stripe_bounds(nb, nranks)
    if nranks == 1 or nb < 2 * nranks:
        assert b is None
        return
    assert b[0] == 0 and b[-1] == nb and len(b) == nranks + 1
    assert all(x % 2 == 0 for x in b)
    assert all(b[i + 1] - b[i] >= 2 for i in range(nranks))
    sizes = [b[i + 1] - b[i] for i in range(nranks)]
    assert max(sizes) - min(sizes) <= 2          # balanced to one A-row


@pytest.mark.parametrize("nb,nranks", [(8, 2), (16, 3), (32, 4), (256, 8)])
def test_every_cell_owned_once_and_exchange_rows(nb, nranks):
    """Each partition cell row is solved by exactly one rank; in a B-sweep the
    rows a rank touches are its own rows plus the imported row lo-1, minus
    the exported row hi-1 (which the rank below solves)."""
    b = stripe_bounds(nb, nranks)
    for part in (1, 2):
        nca = nb // 2 if part == 1 else nb // 2 + 1
        owners = [0] * nca
        for p in range(nranks):
            q0, q1 = owned_cell_rows(nb, part, b[p], b[p + 1])
            touched = sorted({r for q in range(q0, q1) for r in cell_basic_rows(nb, part, q)})
            for q in range(q0, q1):
                owners[q] += 1
            lo, hi = b[p], b[p + 1]
            if part == 1:
                assert touched == list(range(lo, hi))
            else:
                expect = set(range(lo, hi))
                if p > 0:
                    expect.add(lo - 1)
                if p < nranks - 1:
                    expect.discard(hi - 1)
                assert set(touched) == expect
        assert owners == [1] * nca


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = TorchTransport(dist, rank, world, "cpu")
        # rank r sends (r+1)*10 + k bytes to the other rank, variable sizes
        n = 37 + 11 * rank
        payload = torch.arange(n, dtype=torch.int64).to(torch.uint8) + rank
        other = 1 - rank
        got = tr.exchange([(rank, other, payload)], [(other, rank)])
        buf = got[(other, rank)]
        n_other = 37 + 11 * other
        ok = buf.numel() == n_other and torch.equal(buf, torch.arange(n_other, dtype=torch.int64).to(torch.uint8) + other)
        s = tr.allreduce_sum(torch.tensor([1.0 + rank], dtype=torch.float64))
        m = tr.allreduce_max(torch.tensor([1.0 + rank], dtype=torch.float64))
        # one-sided round: only rank 0 sends (the shape of a B-sweep at the stripe ends)
        got2 = tr.exchange([(0, 1, payload)] if rank == 0 else [], [(0, 1)] if rank == 1 else [])
        ok2 = (rank == 0 and not got2) or (rank == 1 and got2[(0, 1)].numel() == 37)
        q.put((rank, bool(ok), float(s.item()), float(m.item()), bool(ok2)))
    finally:
        dist.destroy_process_group()


def test_torch_transport_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok, s, m, ok2 in res:
        assert ok and ok2
        assert s == 3.0 and m == 2.0
