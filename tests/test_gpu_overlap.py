"""Overlapped time-slab halo (north star (d)): with NCCL the sweep of rank
r > 0 runs while the ghost x^k_{first-1} is still in flight -- with a zero ghost -- and a
step-0 kernel completes the first local step from the ghost once it has arrived.  Only one
GPU is reachable, so the same code path is driven with the manual halo
(BIOT_FLAG_MANUAL_HALO | BIOT_FLAG_DEFER_STEP0: the caller moves the slices), and the
iterates must be BITWISE those of one slab: the step-0 kernel repeats the tile kernels'
slot order, coefficient sources and epilogue.  The norms of the completed step are reduced
in another grouping (equal to rounding)."""
import numpy as np
import pytest

from paper_2310_10430_b200 import BiotSolver, FLAG_MANUAL_HALO, FLAG_DEFER_STEP0
from workloads import config_problem, make_problem, initial_iterate, load_scales

pytestmark = pytest.mark.gpu


def _seeded(prob, nt, **kw):
    s = load_scales(nt, parity=True)
    g = BiotSolver(prob, n_t=nt, load_scale=s, **kw)
    g.set_iterate(g.first_step, initial_iterate(prob.dirichlet, np.arange(g.first_step, g.first_step + g.n_tl),
                                                prob.x0_seed))
    return g


def _slabs_vs_one(prob, nt, world, precond, K):
    omega = 0.5 if precond == 2 else 0.3
    ref = _seeded(prob, nt, precond=precond, omega=omega)
    ref.iterate(K)
    xr = ref.solution()
    hr = [ref.residual_history(k) for k in range(K)]
    ranks = [_seeded(prob, nt, precond=precond, omega=omega, rank=r, world=world,
                     flags=FLAG_MANUAL_HALO | FLAG_DEFER_STEP0) for r in range(world)]
    try:
        for _ in range(K):
            slices = [g.last_slice() for g in ranks]
            for r in range(1, world):
                ranks[r].set_ghost(slices[r - 1])
            for g in ranks:
                g.iterate(1)
        xs = np.concatenate([g.solution() for g in ranks])
        assert np.array_equal(xs, xr)
        for g in ranks:
            assert np.array_equal(g.last_slice(), g.solution(g.first_step + g.n_tl - 1, 1)[0])
        for k in range(K):
            hs = np.concatenate([g.residual_history(k) for g in ranks])
            assert np.allclose(hs, hr[k], rtol=1e-12, atol=0), k
    finally:
        for g in ranks:
            g.close()
        ref.close()


@pytest.mark.parametrize("precond", [2, 1])
@pytest.mark.parametrize("world", [2, 8])
def test_deferred_step0_2d_bitwise(precond, world):
    """2D tile kernel (config 2: lognormal kappa, 256 steps; 8 slabs = 32-step slabs)."""
    _slabs_vs_one(config_problem(2), 256, world, precond, 5)


@pytest.mark.parametrize("precond", [2, 1])
def test_deferred_step0_one_step_slabs(precond):
    """N_t = world: every slab is one step, so the step-0 kernel also writes the send slice."""
    _slabs_vs_one(config_problem(1), 4, 4, precond, 4)


def test_deferred_step0_trig_multiload():
    from workloads import trig_problem
    tp = trig_problem(4, 64, 1.0 / 64)
    _slabs_vs_one(tp, 64, 4, 2, 4)
    _slabs_vs_one(tp, 64, 4, 1, 4)


@pytest.mark.parametrize("precond", [2, 1])
def test_deferred_step0_3d_bitwise(precond):
    """3D tile kernel (lognormal kappa, patches cut by the mesh edge, ragged chunks)."""
    prob = make_problem(3, 9, 80, 0.01, 4, storage=1e-3, kappa_median=1e-3, kappa_sigma=1.0,
                        kappa_seed=3, x0_seed=9)
    _slabs_vs_one(prob, 80, 4, precond, 4)
