"""Gauss-Seidel in time with the SWEEPS partitioned across ranks (BIOT_FLAG_SWEEP_SLABS):
the multi-GPU form of PAPER.md Alg. 2 that the paper pipelines over threads / MPI ranks
(Alg. 4; Alg. 5; "GPU g runs sweep g and streams each
finished slice to GPU g+1").  Rank g owns global sweeps g*K/P+1 .. (g+1)*K/P over ALL
steps; at every global wave it receives the slice its first sweep starts from and sends
the slice its last sweep finished.  Driven here with the manual halo (one GPU): rank P-1's
x^K must equal the one-context wavefront bitwise, every rank's history its sweeps', and
after the pipeline fill all P ranks work in every wave (contrast: the time-slab partition
of a K-wide wavefront keeps at most two ranks busy when K <= N_t / P)."""
import numpy as np
import pytest

from paper_2310_10430_b200 import BiotSolver, FLAG_MANUAL_HALO, FLAG_SWEEP_SLABS
from workloads import config_problem, make_problem, initial_iterate, load_scales

pytestmark = pytest.mark.gpu


def _run(prob, nt, K, P, precond, gmres_k=0):
    omega = 0.5 if precond == 2 else 0.3
    s = load_scales(nt, parity=True)
    x0 = initial_iterate(prob.dirichlet, np.arange(1, nt + 1), prob.x0_seed)
    ref = BiotSolver(prob, n_t=nt, precond=precond, omega=omega, load_scale=s)
    ref.set_iterate(1, x0)
    if gmres_k:
        ref.iterate_gs_gmres(K, gmres_k)
    else:
        ref.iterate_gs(K)
    xr = ref.solution()
    hr = [ref.residual_history(k) for k in range(K)]
    ref.close()
    ranks = [BiotSolver(prob, n_t=nt, precond=precond, omega=omega, load_scale=s, rank=r, world=P,
                        flags=FLAG_MANUAL_HALO | FLAG_SWEEP_SLABS) for r in range(P)]
    try:
        ranks[0].set_iterate(1, x0)
        for g in ranks:
            g.gs_begin(K, gmres_k)
        u0 = [r * K // P + 1 for r in range(P)]
        u1 = [(r + 1) * K // P for r in range(P)]
        waves = nt + K - 1
        busy = np.zeros((P, waves), bool)
        for W in range(waves):
            for r in range(1, P):
                t = W - u0[r] + 1
                if 0 <= t < nt:
                    ranks[r].set_ghost(ranks[r - 1].last_slice())
            for r, g in enumerate(ranks):
                wl = W - (u0[r] - 1)
                busy[r, W] = 0 <= wl < nt + (u1[r] - u0[r] + 1) - 1
                g.gs_wave()
        for g in ranks:
            g.gs_end()
        assert np.array_equal(ranks[-1].solution(), xr)
        for r in range(P):
            for u in range(u0[r], u1[r] + 1):
                assert np.allclose(ranks[r].residual_history(u - 1), hr[u - 1], rtol=1e-12, atol=0), (r, u)
        return busy
    finally:
        for g in ranks:
            g.close()


@pytest.mark.parametrize("precond", [2, 1])
def test_sweep_partition_bitwise_2d(precond):
    busy = _run(config_problem(2), 256, 16, 4, precond)
    # every rank works N_t + K/P - 1 waves; all four at once from the end of the fill
    # ((P-1) K/P waves) to the start of the drain: N_t - (P-1) K/P + K/P - 1 = 247 waves
    assert (busy.sum(axis=1) == 256 + 4 - 1).all()
    assert busy.all(axis=0).sum() == 256 - 3 * 4 + 4 - 1


def test_sweep_partition_uneven_and_3d():
    prob = make_problem(3, 7, 40, 0.01, 6, storage=1e-3, kappa_median=1e-3, kappa_sigma=1.0, kappa_seed=3, x0_seed=9)
    _run(prob, 40, 7, 3, 2)       # 7 sweeps over 3 ranks: 2, 2, 3


def test_sweep_partition_gs_gmres():
    _run(config_problem(1), 32, 6, 2, 2, gmres_k=3)
