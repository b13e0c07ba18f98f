"""dd_run_schedule_batch (include/dd.h): several independent problems on one
GPU with their sweeps enqueued round-robin.  Each problem's arithmetic is
unchanged, so its final state must equal dd_run_schedule's bit for bit; the
argument checks reject mismatched contexts and a shared stream."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from ddinputs import gaussian_mixture_image  # noqa: E402


@pytest.fixture(scope="module")
def mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2001_10986_b200 import DD
    from paper_2001_10986_b200.dd import run_schedule_batch
    return DD, run_schedule_batch


def _imgs(n, k):
    return gaussian_mixture_image(n, 100 + 2 * k, 3), gaussian_mixture_image(n, 101 + 2 * k, 3)


def test_batch_equals_sequential_256(mods):
    DD, run_batch = mods
    n, s = 256, 4
    eps = 0.5 / n**2
    kw = dict(schedule=1, coarsest_side=8, max_inner_iter=100000)
    seq, bat = [], []
    for k in range(3):
        mu, nu = _imgs(n, k)
        g = DD(mu, nu, eps, s, **kw)
        g.run_schedule()
        seq.append((g.get_state(), g.primal_cost()))
        bat.append(DD(mu, nu, eps, s, **kw))
    run_batch(bat)
    for k in range(3):
        st = bat[k].get_state()
        for key in ("boxes", "offsets", "values", "alpha_A", "alpha_B"):
            assert np.array_equal(st[key], seq[k][0][key]), (k, key)
        assert bat[k].primal_cost() == seq[k][1]
    # a second batch from the reset state reproduces the first
    for g in bat:
        g.reset()
    run_batch(bat)
    assert np.array_equal(bat[1].get_state()["values"], seq[1][0]["values"])


def test_batch_argument_checks(mods):
    DD, run_batch = mods
    import torch
    mu, nu = _imgs(64, 0)
    st = torch.cuda.Stream()
    a = DD(mu, nu, 0.5 / 64**2, 4, schedule=1, coarsest_side=8, stream=st.cuda_stream)
    b = DD(mu, nu, 0.5 / 64**2, 4, schedule=1, coarsest_side=8, stream=st.cuda_stream)
    with pytest.raises(RuntimeError, match="share a stream"):
        run_batch([a, b])
    mu2, nu2 = _imgs(128, 0)
    c = DD(mu2, nu2, 0.5 / 128**2, 4, schedule=1, coarsest_side=8)
    with pytest.raises(RuntimeError, match="differs"):
        run_batch([a, c])


@pytest.mark.parametrize("n,s", [(256, 4), (128, 8)])
def test_poisoned_memory_bit_identical(mods, n, s):
    """No step of the path reads memory it did not write: with DD_POISON=1
    every state / scratch buffer starts as 0xFF bytes (NaN) and K1 fills its
    SMEM likewise; the final state must equal the clean run bit for bit (a
    stale read would change a speculative-window decision or a value)."""
    import os
    DD, _ = mods
    mu, nu = _imgs(n, 1)
    eps = 0.5 / n**2
    kw = dict(schedule=1, coarsest_side=8, max_inner_iter=100000, bcap_main=18 if s == 8 else 0)
    ref = DD(mu, nu, eps, s, **kw)
    ref.run_schedule()
    a = ref.get_state()
    os.environ["DD_POISON"] = "1"
    try:
        g = DD(mu, nu, eps, s, **kw)
    finally:
        del os.environ["DD_POISON"]
    g.run_schedule()
    b = g.get_state()
    for key in ("boxes", "offsets", "values", "alpha_A", "alpha_B"):
        assert np.array_equal(a[key], b[key]), key
