"""The five BASELINE.json configs as named presets.

Parity runs use seeded random x^0 (x0_seed) and s_n = 1 + 0.1 sin n; metric
runs use x^0 = 0 and s_n = 1 (BJ "zero initial state", "unit load").
"""
from __future__ import annotations

from .generators import make_problem

CONFIGS = {
    1: dict(dim=2, n=16, n_t=32, dt=1 / 32, K=50, lam=1.0, mu=1.0, alpha=1.0, storage=1e-3,
            kappa_median=1e-2, kappa_sigma=0.0, kappa_seed=0, x0_seed=11),
    2: dict(dim=2, n=128, n_t=256, dt=1 / 256, K=100, lam=1.0, mu=1.0, alpha=1.0, storage=1e-3,
            kappa_median=1e-2, kappa_sigma=1.0, kappa_seed=1, x0_seed=12),
    3: dict(dim=2, n=512, n_t=1024, dt=1e-3, K=100, lam=1.0, mu=1.0, alpha=1.0, storage=0.0,
            kappa_median=1e-6, kappa_sigma=0.0, kappa_seed=0, x0_seed=13),
    4: dict(dim=3, n=64, n_t=512, dt=1 / 512, K=50, lam=1.0, mu=1.0, alpha=1.0, storage=1e-3,
            kappa_median=1e-3, kappa_sigma=1.5, kappa_seed=2, x0_seed=14),
    5: dict(dim=3, n=128, n_t=1024, dt=1e-3, K=30, lam=2.0, mu=1.0, alpha=1.0, storage=1e-4,
            kappa_median=1e-4, kappa_sigma=0.0, kappa_seed=0, x0_seed=15),
}

DESCRIPTIONS = {
    1: "2D 16x16 P1-P1, N_t=32, K=50",
    2: "2D 128x128 P1-P1 lognormal kappa, N_t=256, K=100",
    3: "2D 512x512 P1-P1 kappa=1e-6 S=0, N_t=1024, K=100",
    4: "3D 64^3 Kuhn P1-P1 lognormal kappa, N_t=512, K=50",
    5: "3D 128^3 Kuhn P1-P1, N_t=1024, K=30",
}


def config_problem(cid: int, **overrides):
    """Build the Problem for config `cid` (1..5); overrides replace preset keys."""
    kw = dict(CONFIGS[cid])
    kw.update(overrides)
    return make_problem(name=f"config{cid}", **kw)
