"""Projected time-slab scaling from one GPU.

Only one B200 is reachable, so the P-GPU run is projected from the work one rank does:
rank P-1's slab (N_t/P steps) in the overlapped-halo form the NCCL run uses on that rank
(BIOT_FLAG_MANUAL_HALO | BIOT_FLAG_DEFER_STEP0: the sweep with a zero ghost on the SMs
left after the NCCL reservation, then the first-step completion) timed on this GPU, plus
the halo (one slice of N_dof doubles per outer iteration) at the NVLink 5 per-direction
bandwidth (900 GB/s, B200_PROFILING.md) and a fixed latency, counted as NOT overlapped
(an upper bound: in the NCCL run the exchange runs during the sweep).

    efficiency(P) = T_1 / (P * (T_slab(P) + t_halo))

    python tools/project_scaling.py [--configs 3 4] [--K 20] > profiles/r02_scaling_projection.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_10430_b200 import BiotSolver, FLAG_MANUAL_HALO, FLAG_DEFER_STEP0  # noqa: E402
from workloads import config_problem  # noqa: E402

NVLINK_GBS = 900.0          # per direction, B200 NVLink 5 (B200_PROFILING.md)
HALO_LAT_US = 15.0          # assumed send/recv latency per exchange (NCCL p2p over NVSwitch)


def slab_ms(prob, P, K, precond, omega):
    g = BiotSolver(prob, precond=precond, omega=omega, rank=P - 1, world=P,
                   flags=(FLAG_MANUAL_HALO | FLAG_DEFER_STEP0) if P > 1 else 0)
    try:
        g.iterate(3)
        best = []
        for _ in range(3):
            g.iterate(K)
            best.append(float(g.last_timing()[0]))
        best.sort()
        return best[1], g.get_info()
    finally:
        g.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[3, 4])
    ap.add_argument("--K", type=int, default=20)
    ap.add_argument("--precond", type=int, default=2)
    ap.add_argument("--P", type=int, nargs="+", default=[1, 2, 4, 8])
    args = ap.parse_args()
    out = {"what": __doc__.strip().splitlines()[0], "nvlink_gbs": NVLINK_GBS, "halo_latency_us": HALO_LAT_US,
           "precond": args.precond, "lines": []}
    for cid in args.configs:
        prob = config_problem(cid)
        omega = 0.5 if args.precond == 2 else 0.3
        t1, info1 = slab_ms(prob, 1, args.K, args.precond, omega) if 1 in args.P else (float("nan"), None)
        halo_ms = prob.n_dof * 8 / (NVLINK_GBS * 1e9) * 1e3 + HALO_LAT_US * 1e-3
        for P in args.P:
            tp, info = (t1, info1) if P == 1 else slab_ms(prob, P, args.K, args.precond, omega)
            th = 0.0 if P == 1 else halo_ms
            eff = t1 / (P * (tp + th))
            out["lines"].append({"config": cid, "P": P, "n_t_local": info.n_t_local, "ms_per_iter_slab": tp,
                                 "halo_ms": th, "projected_ms_per_iter": tp + th,
                                 "projected_efficiency": eff,
                                 # the exchange runs on the comm stream during the sweep (on the
                                 # 2 reserved SMs, already in ms_per_iter_slab): hidden if it is
                                 # shorter than the sweep, which it is by > 10x
                                 "projected_efficiency_overlapped": t1 / (P * max(tp, th)),
                                 "projected_value": prob.n_dof * prob.n_t / ((tp + th) / 1e3)})
            print(json.dumps(out["lines"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
