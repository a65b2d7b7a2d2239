"""C-ABI surface and host-side logic of libbiot_pit.so (CPU only).

* the library loads and exports every function include/biot_pit.h declares;
* invalid arguments are rejected with BIOT_E_INVALID before any device work;
* on a machine without a GPU, biot_setup fails loudly (no CPU fallback);
* the library's own host assembly (biot_assemble_host, independent code)
  equals the oracle's operators -- both derived from the paper, sharing only
  the seeded inputs.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from paper_2310_10430_b200 import _lib, assemble_host, BiotSolver, BiotError
from workloads import make_problem, config_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "biot_pit.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(biot_[a-z_0-9]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    L = _lib.load()
    names = _declared()
    assert len(names) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (biot_\w+)", out))
    for n in names:
        assert n in exported, n
        getattr(L, n)
    assert set(_lib.EXPORTS) == set(names)
    hdr = open(os.path.join(ROOT, "include", "biot_pit.h")).read()
    assert L.biot_abi_version() == int(re.search(r"#define BIOT_PIT_ABI_VERSION (\d+)", hdr).group(1))


def test_info_struct_matches_header():
    """The ctypes mirror of biot_info has the header's field names in order."""
    hdr = open(os.path.join(ROOT, "include", "biot_pit.h")).read()
    body = hdr[hdr.index("/* Read-only facts about a context. */"):hdr.index("} biot_info;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in re.findall(r"(?:int32_t|int64_t|double)\s+([^;]+);", body):
        names += [v.strip() for v in decl.split(",")]
    assert [f[0] for f in _lib.BiotInfo._fields_] == names


def test_bc_struct_matches_header():
    """The ctypes mirror of biot_bc has the header's field names in order (ABI v3 added
    the §4.1 sources and Dirichlet data)."""
    hdr = open(os.path.join(ROOT, "include", "biot_pit.h")).read()
    body = hdr[hdr.index("typedef struct {\n    const uint8_t *dirichlet;"):hdr.index("} biot_bc;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    body = re.sub(r"void \(\*\w+\)\([^;]*\);", "void *source_eval;", body)
    body = re.sub(r"\[\d+\]", "", body)                     # arrays: keep the name
    names = [re.split(r"[\s*]+", d.strip())[-1] for d in re.findall(r"([^;{]+);", body)]
    names = [n for n in names if n]
    assert [f[0] for f in _lib.BiotBC._fields_] == names


def test_no_torch_in_signatures_and_no_oracle_link():
    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in out and "oracle" not in out and "python" not in out
    # the product sources never reference the oracle
    for root, _, files in os.walk(os.path.join(ROOT, "paper_2310_10430_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "liboracle" not in src, f


def _setup_status(prob, **kw):
    L = _lib.load()
    inp = _lib.Inputs(prob)
    o = dict(precond=2, omega=0.5, device=0, rank=0, world=1, nccl_id=None, stream=None, flags=0,
             history=0)
    o.update(kw.pop("opts", {}))
    opts = _lib.BiotOpts(**o)
    ctx = ctypes.c_void_p()
    n_t = kw.get("n_t", prob.n_t)
    dt = kw.get("dt", prob.dt)
    st = L.biot_setup(ctypes.byref(inp.mesh), ctypes.byref(inp.mat), ctypes.byref(inp.bc), dt, n_t,
                      ctypes.byref(opts), ctypes.byref(ctx))
    if ctx:
        L.biot_destroy(ctx)
    return st, L.biot_last_error(None).decode()


def test_invalid_arguments_rejected():
    prob = make_problem(2, 4, 8, 0.1, 1)
    assert _setup_status(prob, n_t=0)[0] == 1
    assert _setup_status(prob, dt=-1.0)[0] == 1
    assert _setup_status(prob, opts=dict(precond=3))[0] == 1
    assert _setup_status(prob, opts=dict(omega=0.0))[0] == 1
    assert _setup_status(prob, opts=dict(world=3))[0] == 1          # 8 % 3 != 0
    assert _setup_status(prob, opts=dict(world=2, rank=2))[0] == 1
    assert _setup_status(prob, opts=dict(world=2, rank=0))[0] == 1   # no nccl id, no manual flag
    bad = make_problem(2, 4, 8, 0.1, 1)
    bad.cells = bad.cells[:, [0, 2, 1]].copy()                       # inverted triangles
    st, msg = _setup_status(bad)
    assert st == 1 and "inverted" in msg
    bad2 = make_problem(2, 4, 8, 0.1, 1)
    bad2.cells = bad2.cells.copy(); bad2.cells[0, 0] = 10 ** 6
    assert _setup_status(bad2)[0] == 1


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="GPU present")
def test_no_gpu_fails_loudly():
    prob = make_problem(2, 4, 8, 0.1, 1)
    st, msg = _setup_status(prob)
    assert st == 3, (st, msg)                                          # BIOT_E_CUDA, no fallback
    with pytest.raises(BiotError):
        BiotSolver(prob)


def _coo_to_paper(S, coo, ndof):
    i, j, v = coo
    M = sp.coo_matrix((v, (i, j)), shape=(ndof, ndof)).tocsr()
    d, nn = S.dim, S.nn
    # permutation interleaved -> paper order
    perm = np.empty(ndof, dtype=np.int64)
    nodes = np.arange(nn)
    for c in range(d):
        perm[nodes * d + c] = nodes * (d + 1) + c
    perm[d * nn + nodes] = nodes * (d + 1) + d
    return M[perm][:, perm]


@pytest.mark.parametrize("dim,n,storage,sigma", [(2, 6, 1e-3, 1.0), (2, 5, 0.0, 0.0), (3, 3, 1e-3, 1.5)])
def test_host_assembly_matches_oracle(dim, n, storage, sigma):
    prob = make_problem(dim, n, 4, 0.01, 1, lam=1.3, mu=0.7, alpha=0.9, storage=storage,
                        kappa_median=1e-2, kappa_sigma=sigma, kappa_seed=3)
    S = oracle.OracleSystem(prob)
    A, P, f, dinv = assemble_host(prob, prob.dt)
    ndof = S.ndof
    AA = _coo_to_paper(S, A, ndof)
    AP = _coo_to_paper(S, P, ndof)
    scale = abs(S.AA).max()
    assert abs(AA - S.AA).max() < 1e-14 * scale
    assert abs(AP - S.AP).max() < 1e-14 * scale
    assert np.abs(S.to_paper(f) - S.F).max() < 1e-15
    dref = np.concatenate([S.DAinv, S.DSinv])
    assert np.allclose(S.to_paper(dinv), dref, rtol=1e-13, atol=0)


def test_host_assembly_unstructured_ell_path():
    """A renumbered (non-banded) mesh takes the ELL path; operators still match the oracle."""
    prob = make_problem(2, 6, 4, 0.01, 1)
    rng = np.random.default_rng(0)
    perm = rng.permutation(prob.coords.shape[0])
    inv = np.argsort(perm)
    prob.coords = prob.coords[perm]
    prob.cells = inv[prob.cells].astype(np.int32)
    prob.facets = inv[prob.facets].astype(np.int32)
    m = prob.dirichlet.reshape(-1, 3)[perm]
    prob.dirichlet = m.reshape(-1).copy()
    S = oracle.OracleSystem(prob)
    A, P, f, dinv = assemble_host(prob, prob.dt)
    AA = _coo_to_paper(S, A, S.ndof)
    assert abs(AA - S.AA).max() < 1e-14 * abs(S.AA).max()


@pytest.mark.parametrize("which", ["trig", "patch"])
def test_host_load_terms_match_oracle(which):
    """The library's §4.1 load terms (sources by its quadrature, Dirichlet lifting from the
    unmasked blocks; R24) equal the oracle's independent ones."""
    from paper_2310_10430_b200.solver import assemble_loads_host
    from workloads import trig_problem, linear_patch_problem
    prob = trig_problem(3, 8, 0.01) if which == "trig" else linear_patch_problem(5, 4, 0.1, lam=1.3, mu=0.7)
    S = oracle.OracleSystem(prob)
    F, kinds, src = assemble_loads_host(prob, prob.dt)
    want = {("src", q): None for q in range(prob.n_sources)}
    for j, k in enumerate(S.kinds[1:], start=1):
        want[k] = S.loads[j]
    names = {0: "src", 1: "dnow", 2: "dprev"}
    assert len(F) == len([k for k, v in want.items() if v is not None and np.abs(v).max() > 0])
    for j in range(len(F)):
        key = ("src", int(src[j])) if kinds[j] == 0 else (names[int(kinds[j])],)
        ref = S.from_paper(want[key])
        scale = np.abs(ref).max()
        assert np.abs(F[j] - ref).max() <= 1e-13 * scale, (key, np.abs(F[j] - ref).max(), scale)


@pytest.mark.parametrize("dim,n", [(2, 1), (2, 5), (3, 1), (3, 3)])
def test_structured_mesh_helper_matches_workloads(dim, n):
    """biot_mesh_structured reproduces the workload meshes (node numbering, cell vertex
    order, orientation) exactly; SURVEY §8(b) helpers."""
    from paper_2310_10430_b200.solver import mesh_structured
    from workloads import mesh
    X, C = mesh_structured(dim, n)
    Xw, Cw = mesh(dim, n)
    assert np.array_equal(X, Xw)
    assert np.array_equal(C, Cw)


@pytest.mark.parametrize("dim,n", [(2, 4), (3, 2)])
def test_bc_column_helper(dim, n):
    """biot_bc_column: the column Dirichlet mask and top facets of the workloads, and the
    traction load equal to the oracle's (total = -load * |top| = -load)."""
    from paper_2310_10430_b200.solver import mesh_structured, bc_column
    from workloads import column_dirichlet, top_facets
    X, C = mesh_structured(dim, n)
    mask, F, facets = bc_column(X, C, load=2.5)
    assert np.array_equal(mask, column_dirichlet(X))
    tf = top_facets(X, C)
    assert sorted(map(tuple, np.sort(facets, axis=1))) == sorted(map(tuple, np.sort(tf, axis=1)))
    tr = np.zeros(dim)
    tr[dim - 1] = -2.5
    Fu = oracle.traction_load(dim, X, tf, tr)                  # node-major U, d per node
    nn = X.shape[0]
    Fi = F.reshape(nn, dim + 1)
    assert np.abs(Fi[:, :dim].ravel() - Fu).max() < 1e-15
    assert np.all(Fi[:, dim] == 0.0)
    assert abs(Fi[:, dim - 1].sum() + 2.5) < 1e-13
