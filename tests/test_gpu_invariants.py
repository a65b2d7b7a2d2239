"""GPU properties that hold at any size (needs a B200).

* iterate(a); iterate(b) == iterate(a+b) bitwise; run-to-run bitwise;
* time-slab decomposition (world = 2, 4, 8 contexts, halo moved by the host)
  gives x^K bitwise equal to one slab -- the multi-GPU contract checked on one
  GPU without kernels that wait on each other;
* front invariant at full size (config 3): x^0 = 0, s = 1 -> x_n^K == x_K^K, n >= K;
* monotone residual history at full size with metric inputs;
* degenerate inputs: K = 0, all DoFs Dirichlet, S = 0.
"""
import numpy as np
import pytest

from paper_2310_10430_b200 import BiotSolver, FLAG_MANUAL_HALO
from workloads import config_problem, make_problem, initial_iterate, load_scales

pytestmark = pytest.mark.gpu


def _seeded(prob, nt, **kw):
    s = load_scales(nt, parity=True)
    g = BiotSolver(prob, n_t=nt, load_scale=s, **kw)
    g.set_iterate(g.first_step, initial_iterate(prob.dirichlet, np.arange(g.first_step, g.first_step + g.n_tl),
                                                prob.x0_seed))
    return g


@pytest.mark.parametrize("precond", [1, 2])
def test_additive_and_deterministic(precond):
    prob = config_problem(2)
    g1 = _seeded(prob, prob.n_t, precond=precond)
    g1.iterate(3); g1.iterate(4)
    g2 = _seeded(prob, prob.n_t, precond=precond)
    g2.iterate(7)
    assert np.array_equal(g1.solution(), g2.solution())
    for k in range(7):
        assert np.array_equal(g1.residual_history(k), g2.residual_history(k))
    assert np.array_equal(g1.residual_norms(), g2.residual_norms())
    g0 = _seeded(prob, prob.n_t, precond=precond)
    x_before = g0.solution()
    g0.iterate(0)
    assert np.array_equal(g0.solution(), x_before)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("precond", [2, 1])
def test_time_slabs_bitwise(world, precond):
    prob = config_problem(2)
    nt, K = prob.n_t, 9
    ref = _seeded(prob, nt, precond=precond)
    ref.iterate(K)
    xr = ref.solution()
    ranks = [_seeded(prob, nt, precond=precond, rank=r, world=world, flags=FLAG_MANUAL_HALO)
             for r in range(world)]
    for _ in range(K):
        slices = [g.last_slice() for g in ranks]
        for r in range(1, world):
            ranks[r].set_ghost(slices[r - 1])
        for g in ranks:
            g.iterate(1)
    xs = np.concatenate([g.solution() for g in ranks])
    assert np.array_equal(xs, xr)
    # the send buffer written by the last sweep equals the last owned step
    for g in ranks:
        assert np.array_equal(g.last_slice(), g.solution(g.first_step + g.n_tl - 1, 1)[0])
    # norms agree to rounding (reduction grouping depends on the slab length)
    hs = np.concatenate([g.residual_history(K - 1) for g in ranks])
    assert np.allclose(hs, ref.residual_history(K - 1), rtol=1e-12, atol=0)


def test_front_invariant_full_config3():
    prob = config_problem(3)
    g = BiotSolver(prob, precond=2, omega=0.5)
    K = 5
    g.iterate(K)
    x = g.solution(K, 40)
    for r in range(1, 40):
        assert np.array_equal(x[r], x[0])
    xl = g.solution(prob.n_t - 3, 4)
    assert np.array_equal(xl[-1], x[0])
    assert not np.array_equal(g.solution(K - 1, 1)[0], x[0])


@pytest.mark.parametrize("cid", [2, 3])
def test_monotone_history_metric_inputs(cid):
    prob = config_problem(cid)
    g = BiotSolver(prob, precond=2, omega=0.5)
    g.iterate(prob.K)
    tot = np.array([np.sqrt((g.residual_history(k) ** 2).sum()) for k in range(prob.K)])
    assert np.all(np.diff(tot) <= 0) and tot[-1] < 0.5 * tot[0]
    fin = np.sqrt((g.residual_norms() ** 2).sum())
    assert fin <= tot[-1]


def test_all_dirichlet_and_zero_storage():
    prob = make_problem(2, 6, 8, 0.1, 3, storage=0.0)
    prob.dirichlet = np.ones_like(prob.dirichlet)
    g = _seeded(prob, 8)
    g.iterate(3)
    assert np.abs(g.solution()).max() == 0.0
    assert np.abs(g.residual_norms()).max() == 0.0


@pytest.mark.parametrize("cid", [1, 2])
@pytest.mark.parametrize("precond", [2, 1])
def test_kernel_variants_bitwise(cid, precond, monkeypatch):
    """Every sweep kernel shares dev::node_epilogue; generic and row-march also share the
    neighbour order (bitwise identical iterates); the TMA tile kernel walks the 10 columns
    of a row pair in its own fixed order (equal to rounding)."""
    prob = config_problem(cid)
    K = 6
    res = {}
    for kern in ("generic", "march", "tile"):
        monkeypatch.setenv("BIOT_KERNEL", kern)
        g = _seeded(prob, prob.n_t, precond=precond)
        g.iterate(K)
        res[kern] = (g.solution(), g.residual_history(K - 1), g.info.kernel_path)
        g.close()
    assert res["generic"][2] == 1 and res["march"][2] == 4 and res["tile"][2] == 5
    assert np.array_equal(res["march"][0], res["generic"][0])
    assert np.allclose(res["march"][1], res["generic"][1], rtol=1e-12, atol=0)
    x, ref = res["tile"][0], res["generic"][0]
    assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.allclose(res["tile"][1], res["generic"][1], rtol=1e-10, atol=0)


def _tile3d_cases():
    # (n cells per axis, n_t, storage, kappa sigma): ragged time tails (n_t % 32 != 0),
    # patches cut by the mesh edge (n+1 not a multiple of 4), S = 0 (zero-storage variant)
    return [(7, 40, 1e-3, 1.0), (8, 33, 0.0, 0.0), (5, 64, 1e-3, 1.5), (9, 7, 0.0, 1.0)]


@pytest.mark.parametrize("case", _tile3d_cases())
@pytest.mark.parametrize("precond", [2, 1])
def test_tile3d_vs_generic(case, precond, monkeypatch):
    """The 3D TMA tile kernel (template stencil, structural zeros skipped, boundary
    nodes out of line) against the generic BDIA kernel: equal to rounding."""
    n, nt, S, sig = case
    prob = make_problem(3, n, nt, 0.01, 6, storage=S, kappa_median=1e-3, kappa_sigma=sig,
                        kappa_seed=3, x0_seed=9)
    K = 6
    res = {}
    for kern in ("generic", "tile"):
        monkeypatch.setenv("BIOT_KERNEL", kern)
        g = _seeded(prob, nt, precond=precond)
        g.iterate(K)
        res[kern] = (g.solution(), np.stack([g.residual_history(k) for k in range(K)]),
                     g.residual_norms(), g.info.kernel_path)
        g.close()
    assert res["generic"][3] == 1 and res["tile"][3] == 7
    x, ref = res["tile"][0], res["generic"][0]
    assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.allclose(res["tile"][1], res["generic"][1], rtol=1e-10, atol=0)
    assert np.allclose(res["tile"][2], res["generic"][2], rtol=1e-10, atol=0)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("precond", [2, 1])
def test_tile3d_time_slabs_bitwise(world, precond):
    """Chunk 0 of each slab recomputes q(t0-1) from the ghost in the carry's FMA order; the
    slices moved between the contexts are the send buffers the kernels wrote (the NCCL
    data path)."""
    prob = make_problem(3, 7, 96, 0.01, 5, storage=1e-3, kappa_median=1e-3, kappa_sigma=1.0,
                        kappa_seed=3, x0_seed=9)
    nt, K = prob.n_t, 5
    ref = _seeded(prob, nt, precond=precond)
    assert ref.info.kernel_path == 7
    ref.iterate(K)
    xr = ref.solution()
    ranks = [_seeded(prob, nt, precond=precond, rank=r, world=world, flags=FLAG_MANUAL_HALO)
             for r in range(world)]
    for _ in range(K):
        slices = [g.last_slice() for g in ranks]
        for r in range(1, world):
            ranks[r].set_ghost(slices[r - 1])
        for g in ranks:
            g.iterate(1)
    xs = np.concatenate([g.solution() for g in ranks])
    assert np.array_equal(xs, xr)


@pytest.mark.parametrize("dim,world", [(2, 2), (2, 4), (3, 2)])
def test_gs_time_slabs_bitwise(dim, world):
    """Gauss-Seidel wavefront split over time slabs (one context per slab, the slice of
    each slab's last step moved to the next slab's ghost before every wave that needs
    it -- the NCCL exchange's data path) equals one slab bitwise."""
    if dim == 2:
        prob = config_problem(1)
        nt = prob.n_t
    else:
        prob = make_problem(3, 7, 24, 0.01, 5, storage=1e-3, kappa_median=1e-3, kappa_sigma=1.0,
                            kappa_seed=3, x0_seed=9)
        nt = prob.n_t
    K = 6
    ref = _seeded(prob, nt, precond=2)
    ref.iterate_gs(K)
    xr = ref.solution()
    hr = np.concatenate([ref.residual_history(k) for k in range(K)])
    ranks = [_seeded(prob, nt, precond=2, rank=r, world=world, flags=FLAG_MANUAL_HALO) for r in range(world)]
    waves = [g.gs_begin(K) for g in ranks][0]
    assert waves == nt + K - 1
    for w in range(waves):
        slices = [g.last_slice() for g in ranks]
        for r in range(1, world):
            first = ranks[r].first_step
            if w - K + 2 <= first <= w + 1:
                ranks[r].set_ghost(slices[r - 1])
        for g in ranks:
            g.gs_wave()
    for g in ranks:
        g.gs_end()
    xs = np.concatenate([g.solution() for g in ranks])
    assert np.array_equal(xs, xr)
    hs = np.concatenate([np.concatenate([g.residual_history(k) for g in ranks]) for k in range(K)])
    assert np.allclose(hs, hr, rtol=1e-12, atol=0)


def test_gs_gmres_time_slabs_bitwise():
    """Alg. 3 (Gauss-Seidel + GMRES) split over two time slabs equals one slab bitwise."""
    prob = config_problem(1)
    nt, K, k, world = prob.n_t, 4, 3, 2
    ref = _seeded(prob, nt, precond=2)
    ref.iterate_gs_gmres(K, k)
    xr = ref.solution()
    ranks = [_seeded(prob, nt, precond=2, rank=r, world=world, flags=FLAG_MANUAL_HALO) for r in range(world)]
    waves = [g.gs_begin(K, k) for g in ranks][0]
    for w in range(waves):
        slices = [g.last_slice() for g in ranks]
        for r in range(1, world):
            first = ranks[r].first_step
            if w - K + 2 <= first <= w + 1:
                ranks[r].set_ghost(slices[r - 1])
        for g in ranks:
            g.gs_wave()
    for g in ranks:
        g.gs_end()
    assert np.array_equal(np.concatenate([g.solution() for g in ranks]), xr)


@pytest.mark.parametrize("precond", [2, 1])
def test_aux_uniform_skip_bitwise(precond, monkeypatch):
    """Uniform coefficients (config 3's kind: S = 0, one kappa): row strips inside the
    aux-uniform rectangle skip the aux-record copy and read the shared record; iterates and
    norms are bitwise those of the run that streams every record (BIOT_NO_AUX_SKIP=1)."""
    prob = make_problem(2, 64, 256, 1e-3, 5, storage=0.0, kappa_median=1e-6, x0_seed=5)
    res = []
    for skip in (False, True):
        if skip:
            monkeypatch.delenv("BIOT_NO_AUX_SKIP", raising=False)
        else:
            monkeypatch.setenv("BIOT_NO_AUX_SKIP", "1")
        g = _seeded(prob, 256, precond=precond, omega=0.5 if precond == 2 else 0.3)
        g.iterate(5)
        res.append((g.solution(), [g.residual_history(k) for k in range(5)], g.residual_norms()))
        g.close()
    assert np.array_equal(res[0][0], res[1][0])
    assert all(np.array_equal(a, b) for a, b in zip(res[0][1], res[1][1]))
    assert np.array_equal(res[0][2], res[1][2])


@pytest.mark.parametrize("precond,K", [(2, 4), (1, 3), (2, 16)])
def test_gs_gmres_compact_basis_bitwise(precond, K, monkeypatch):
    """Narrow Gauss-Seidel windows keep the Krylov basis compact (row pitch = window
    width); iterates and history are bitwise those of the panel-layout basis
    (BIOT_GMRES_NO_COMPACT=1): same arithmetic, same dot order."""
    prob = config_problem(1)
    nt, k = prob.n_t, 4
    res = []
    for compact in (False, True):
        if compact:
            monkeypatch.delenv("BIOT_GMRES_NO_COMPACT", raising=False)
        else:
            monkeypatch.setenv("BIOT_GMRES_NO_COMPACT", "1")
        g = _seeded(prob, nt, precond=precond, omega=1.0)
        g.iterate_gs_gmres(K, k)
        res.append((g.solution(), [g.residual_history(i) for i in range(K)]))
        g.close()
    assert np.array_equal(res[0][0], res[1][0])
    assert all(np.array_equal(a, b) for a, b in zip(res[0][1], res[1][1]))
