"""A/B of library builds (tools/build_variant.py) on one config: per-iteration and sweep
times (CUDA events inside the library) and a bitwise comparison of the iterate after K
iterations against the first build.  Each build runs in its own process (one library
per process):

    python tools/ab_variants.py --config 4 --precond 2 lib_a.so lib_b.so ...
    ('-' = the product library)

Compare against the library of the previous commit (build it from a checkout of that
commit into paper_2310_10430_b200/build/ab/), not only against a switch inside the new
build: the reverted tile3d list schedule gained 1.3% over its own fallback order while the
whole build was 3.5% slower than its predecessor (profiles/r02_ab_tile3d_schedule.txt).
"""
import argparse
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(args):
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_2310_10430_b200 import BiotSolver
    from workloads import config_problem, initial_iterate, load_scales

    prob = config_problem(args.config)
    nt = prob.n_t
    g = BiotSolver(prob, precond=args.precond, omega=args.omega, load_scale=load_scales(nt, parity=True))
    g.set_iterate(1, initial_iterate(prob.dirichlet, np.arange(1, nt + 1), 5))
    run = (lambda k: g.iterate_cheb(k, args.cheb_m)) if args.cheb_m else g.iterate
    run(args.K)
    x = g.solution()
    h = hashlib.sha1(np.ascontiguousarray(x).tobytes()).hexdigest()
    run(3)
    its, sws = [], []
    for _ in range(args.repeats):
        run(args.steps)
        it, sw = g.last_timing()
        its.append(it)
        sws.append(sw)
    path = g.info.kernel_path
    g.close()
    print(json.dumps({"sha1": h, "iter_ms": sorted(its)[len(its) // 2], "sweep_ms": sorted(sws)[len(sws) // 2],
                      "path": path}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--precond", type=int, default=2)
    ap.add_argument("--omega", type=float, default=None)
    ap.add_argument("--K", type=int, default=3)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--cheb-m", type=int, default=0, help="time biot_iterate_cheb(K, m) instead")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.omega is None:
        a.omega = 0.5 if a.precond == 2 else 0.3
    if a.child:
        return child(a)
    ref = None
    for lib in a.libs:
        env = dict(os.environ)
        env.pop("BIOT_LIB_OVERRIDE", None)
        if lib != "-":
            env["BIOT_LIB_OVERRIDE"] = os.path.abspath(lib)
        cmd = [sys.executable, os.path.abspath(__file__), "--child", "--config", str(a.config), "--precond",
               str(a.precond), "--omega", str(a.omega), "--K", str(a.K), "--steps", str(a.steps), "--repeats",
               str(a.repeats), "--cheb-m", str(a.cheb_m), "x"]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True)
        if r.returncode != 0:
            print(f"{lib}: FAILED\n{r.stderr[-2000:]}", flush=True)
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        ref = ref or d["sha1"]
        print(f"config{a.config} P~{a.precond} {lib:40s} iter {d['iter_ms']:8.3f} ms  sweep {d['sweep_ms']:8.3f} ms"
              f"  bitwise={'same' if d['sha1'] == ref else 'DIFFERENT'}", flush=True)


if __name__ == "__main__":
    main()
