"""Benchmark: space-time DoF updates/s per outer iteration (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

A "step" is one outer iteration of the inverted time-stepping scheme over every
time step of the workload (residual with previous-step coupling, block
preconditioner, damped update, per-step residual norms).  Default workload:
config 3 (2D 512x512 P1-P1, N_t = 1024, kappa=1e-6, S=0), the configuration the
metric's roofline and 8-GPU efficiency targets are quoted on that fits one GPU
(DESIGN.md "Measurement").  N > 1: one rank per GPU (under torchrun, or
self-spawned through torch.distributed.run when WORLD_SIZE is unset), time slabs
of N_t/N steps, NCCL send/recv of one slice per outer iteration (strong scaling).

Timing: W warm-up iterations, then --repeats (default 5) timed runs of exactly K
outer iterations, each bracketed by a barrier + device synchronize and timed with
CUDA events on the launching stream, max over ranks; the line reports the median
run, nvidia-smi clocks sampled across the timed runs.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "space-time DoF updates/s per outer iteration; % of HBM/fp64 roofline"
UNIT = "DoF-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--workload", default="config", choices=["config", "trig"],
                    help="config: BASELINE config --config; trig: PAPER.md §4.1 trigonometric test "
                         "(h = 2^-trig_k, N_t = 1024, tau = 1/1024; sources + Dirichlet lifting)")
    ap.add_argument("--trig-k", type=int, default=9)
    ap.add_argument("--precond", type=int, default=2)
    ap.add_argument("--omega", type=float, default=0.5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--method", default="jacobi", choices=["jacobi", "gs", "gmres", "gs_gmres", "cheb"],
                    help="jacobi: all steps at once (BASELINE metric); gs: Gauss-Seidel in time "
                         "(PAPER.md Alg. 2 literal) as a wavefront; gmres: Alg. 3 with one GMRES(k) "
                         "cycle per step and outer iteration (left P~2); gs_gmres: Alg. 3 literally "
                         "(Gauss-Seidel in time + GMRES(k)) on the wavefront")
    ap.add_argument("--gmres-k", type=int, default=10)
    ap.add_argument("--cheb-m", type=int, default=2, help="Chebyshev steps per inner inverse (--method cheb)")
    ap.add_argument("--cheb-alpha", type=float, default=30.0)
    ap.add_argument("--repeats", type=int, default=5, help="timed runs of K iterations; the median is reported")
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel directly (BIOT_FLAG_NO_GRAPH)")
    return ap.parse_args()


def spawn_ranks(n):
    """--gpus N without a launcher: re-run this command under torch.distributed.run with N
    local ranks (127.0.0.1 rendezvous); rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # communicator size visible in the NCCL INIT lines
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line))

    def start(self):
        """Start sampling every 100 ms (before the warm-up) and wait for the first sample;
        mark() opens the timed region, stop() keeps the samples taken inside it (or, for a
        region shorter than the sampling period, the last one before it, under warm-up load)."""
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        t0 = time.time()
        while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.01)

    def mark(self):
        self.t0 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        t1 = time.time()
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        t0 = getattr(self, "t0", 0.0)
        inside = [ln for ts, ln in self.lines if t0 <= ts <= t1 + 0.05]
        before = [ln for ts, ln in self.lines if ts < t0]
        out = "".join(inside if inside else before[-1:])
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sms:
            return None
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms), "in_region": bool(inside)}


KERNELS = {1: "sweep_kernel<BDIA> (generic, fused residual + P~ + update + norms)",
           2: "sweep_kernel<ELL> (generic, fused residual + P~ + update + norms)",
           4: "march2d_kernel",
           5: "tile2d_kernel (TMA row march, fused residual + P~ + update + norms)",
           7: "tile3d_kernel (TMA plane march, fused residual + P~ + update + norms)"}


def fp64_peak(sm_mhz):
    """FP64 FMA peak: DFMA microbenchmark (tools/ubench/dfma.cu, profiles/r01_ubench_dfma.txt):
    58.8 FMA/clk/SM sustained at 16-32 warps/SM x 4-8 chains; nominal 64."""
    measured = 148 * 58.8 * 2 * sm_mhz * 1e6 / 1e12
    nominal = 148 * 64 * 2 * sm_mhz * 1e6 / 1e12
    return measured, nominal


def load_traffic(cid):
    """DRAM bytes (read + write) per launch of the dominant kernel from one ncu --set full
    capture (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(p)).get(cid if isinstance(cid, str) else f"config{cid}")
        return None if t is None else float(t["bytes"])
    except Exception:
        return None


def make_problem_for(args):
    from workloads import config_problem, trig_problem
    if args.workload == "trig":
        return trig_problem(args.trig_k, 1024, 1.0 / 1024)
    return config_problem(args.config)


def oracle_loads(S, prob, w):
    """Load coefficients of the first w steps: s_n = 1 (configs) or all §4.1 terms (trig)."""
    if getattr(prob, "source_fn", None) is not None:
        return S.coefs(np.zeros(w), 1, w)
    return np.ones(w)


def cpu_baseline(prob, precond, omega, budget_s=12.0, window=64):
    """The oracle as it stands, on all host cores, over a bounded sample of the workload."""
    import oracle
    S = oracle.OracleSystem(prob)
    cores = os.cpu_count() or 1
    w = min(window, prob.n_t)
    X = np.zeros((w + 1, S.ndof))
    s = oracle_loads(S, prob, w)
    passes, t0 = 0, time.perf_counter()
    while True:
        S.iterate(X, s, 1, precond, omega, history=True, nthreads=cores)
        passes += 1
        el = time.perf_counter() - t0
        if el >= budget_s or passes >= 200:
            break
    value = S.ndof * w * passes / el
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{passes} outer iteration(s) over a {w}-step window of the full "
                      f"{prob.coords.shape[0]}-node mesh, P~{precond}, omega={omega} "
                      f"(oracle assembly excluded), {el:.1f} s wall"}


def workload_config(args, prob, world):
    from workloads import DESCRIPTIONS
    ws_gb = 2 * prob.n_dof * prob.n_t * 8 / 1e9
    name = (f"trig h=1/{prob.n}: PAPER.md §4.1 trigonometric test, {prob.n}x{prob.n} P1-P1, N_t=1024, "
            f"tau=1/1024, sources (cos t, sin t) + Dirichlet lifting (4 load terms)"
            if args.workload == "trig" else f"config{args.config}: {DESCRIPTIONS[args.config]}")
    return {"workload": name
                        + (", Gauss-Seidel in time (wavefront)" if args.method == "gs" else "")
                        + (f", per-step GMRES({args.gmres_k})" if args.method == "gmres" else "")
                        + (f", Alg. 3: Gauss-Seidel in time + GMRES({args.gmres_k})" if args.method == "gs_gmres"
                           else "")
                        + (f", P~2 with Chebyshev({args.cheb_m}) inner inverses (alpha {args.cheb_alpha})"
                           if args.method == "cheb" else ""),
            "model": f"biot-p1p1-{prob.dim}d", "n_dof": int(prob.n_dof), "n_t": int(prob.n_t),
            "global_batch": int(prob.n_dof * prob.n_t), "seq_len": int(prob.n_t),
            "precond": f"P~{args.precond}", "omega": args.omega, "parallelism": f"time-slab{world}",
            "l2": (f"inputs larger than L2 (x panels {ws_gb:.1f} GB vs 126 MB L2); no flush needed" if ws_gb > 0.5
                   else f"x panels {ws_gb * 1e3:.1f} MB fit in the 126 MB L2 (L2-resident small configuration, "
                        f"not flushed; the metric's configuration is config 3)"),
            "inputs": ("x^0 = 0, x_0 = the §4.1 initial condition, exact §4.1 data" if args.workload == "trig"
                       else "x^0 = 0, s_n = 1 (BJ metric inputs), synthetic mesh/material")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    prob = make_problem_for(args)
    import oracle
    S = oracle.OracleSystem(prob)
    cores = os.cpu_count() or 1
    w = min(16, prob.n_t)
    X = np.zeros((w + 1, S.ndof))
    s = oracle_loads(S, prob, w)
    S.iterate(X, s, 1, args.precond, args.omega, nthreads=cores)     # warm-up pass
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        S.iterate(X, s, 1, args.precond, args.omega, nthreads=cores)
        times.append(time.perf_counter() - t0)
        if sum(times) > 150:
            break
    tot = sum(times)
    value = S.ndof * w * len(times) / tot
    sample = (f"each step = 1 outer iteration of the oracle over a {w}-step window of the full "
              f"{prob.coords.shape[0]}-node mesh (bounded sample of the workload)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args, prob, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)

    from paper_2310_10430_b200 import BiotSolver, nccl_unique_id, FLAG_NO_GRAPH

    prob = make_problem_for(args)
    nccl_id = None
    if world > 1:
        from paper_2310_10430_b200.dist import broadcast_nccl_id
        nccl_id = broadcast_nccl_id(nccl_unique_id, device=dev)
    stream = torch.cuda.current_stream()
    reps = max(1, args.repeats)
    g = BiotSolver(prob, precond=args.precond, omega=args.omega, device=local, rank=rank, world=world,
                   nccl_id=nccl_id, stream=stream.cuda_stream, flags=FLAG_NO_GRAPH if args.no_graph else 0,
                   history=max(1024, reps * args.steps + args.warmup + args.e2e_steps + 8))
    info = g.info

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    if args.method == "gmres":
        step = lambda K: g.iterate_gmres(K, args.gmres_k)
    elif args.method == "gs_gmres":
        step = lambda K: g.iterate_gs_gmres(K, args.gmres_k)
    elif args.method == "cheb":
        step = lambda K: g.iterate_cheb(K, args.cheb_m, args.cheb_alpha)
    else:
        step = g.iterate_gs if args.method == "gs" else g.iterate
    clk = ClockSampler(local)
    clk.start()
    # warm-up (untimed)
    step(max(args.warmup, 3))
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    runs = []
    clk.mark()
    for _ in range(reps):
        barrier()
        ev0.record(stream)
        step(args.steps)               # K outer iterations, one library call
        ev1.record(stream)
        barrier()
        # preconditioner pass(es) of the dominant kernel, CUDA events on the launching stream
        t = torch.tensor([ev0.elapsed_time(ev1), float(g.last_timing()[1])], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        runs.append((float(t[0]), float(t[1])))
    clocks = clk.stop()
    ms, sweep_ms = sorted(runs)[len(runs) // 2]             # the median run and its kernel time
    ms_per_step = ms / args.steps
    value = prob.n_dof * prob.n_t * args.steps / (ms / 1e3)

    # end to end through the public API with host buffers: every step uploads its
    # inputs (the load scales s_n) from pinned host memory and reads back the
    # step's result (per-step residual norms)
    s_host = torch.ones(prob.n_t, dtype=torch.float64).pin_memory()
    out_host = torch.empty((info.n_t_local, 2), dtype=torch.float64).pin_memory()
    s_np, out_np = s_host.numpy(), out_host.numpy()
    from paper_2310_10430_b200 import _lib
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    trig = args.workload == "trig"        # loads fixed at setup: no per-step host input
    for _ in range(args.e2e_steps):
        if not trig:
            g.set_load_scale(s_np)
        step(1)
        _lib.check(g.lib.biot_residual_history(g.ctx, g.get_info().iterations - 1, _lib.ptr(out_np)), g.ctx)
    e1.record(stream)
    barrier()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = prob.n_dof * prob.n_t * args.e2e_steps / (float(e2e_ms[0]) / 1e3)

    if rank == 0:
        pk = peaks()
        hbm = pk["hbm_gbs"] if pk else 6650.0
        algo_bytes = info.bytes_per_iter          # per launch of the sweep kernel (this rank)
        if args.method in ("gmres", "gs_gmres"):
            # one GMRES(k) cycle = 7 + 14k + 2k^2 passes over a space-time panel
            kk = args.gmres_k
            algo_bytes = (7 + 14 * kk + 2 * kk * kk) * 8.0 * prob.n_dof * info.n_t_local
        if args.method == "cheb":
            # panel passes per outer iteration: residual 2, start 2 + 1/nc
            # (m = 1: 3 with the update), step k: 5 (+1 from k = 2 on), the last one 4 (+1)
            mm, nc = args.cheb_m, prob.dim + 1
            if args.precond == 2:   # the start is fused into the first step (reads Z directly)
                passes = 5.0 if mm == 1 else 2 + sum(
                    (3 if k == mm - 1 else 4) + (2 if k >= 2 else 0) for k in range(1, mm))
            else:   # P~1: displacement block, B^T z_u - r_p, pressure block (fractions fu, fp)
                fu, fp = (nc - 1) / nc, 1.0 / nc
                steps = lambda f, last_x: sum(((3 if k == mm - 1 and last_x else 5) + (1 if k >= 2 else 0)) * f
                                               + (2 * f if k == mm - 1 and last_x else 0) for k in range(1, mm))
                passes = (2 + (2 * fu if mm == 1 else -fu) + steps(fu, False)   # residual, u start (fused: d_0 not read)
                          + fu + fp + 2 * fu + (2 * fp if mm == 1 else 2 * fp)   # r~_p, x_u update, p start
                          + steps(fp, True))
            algo_bytes = passes * 8.0 * prob.n_dof * info.n_t_local
        achieved_gbs = algo_bytes / (sweep_ms / 1e3) / 1e9
        sm_max = (pk or {}).get("sm_max_mhz", 1965.0)
        fp64_meas_tf, fp64_nom_tf = fp64_peak(sm_max)
        achieved_tf = info.flops_per_iter / (sweep_ms / 1e3) / 1e12
        if prob.dim == 2 or args.method in ("gmres", "gs_gmres", "cheb"):   # panel-pass bound
            roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                    "frac": achieved_gbs / hbm,
                    "traffic": (load_traffic("trig" if args.workload == "trig" else args.config)
                                if args.method == "jacobi" and args.precond == 2 else None),
                    "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                                    "profiles/traffic.json)",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else "fallback 6.65 TB/s",
                    "frac_of_nominal_8tbs": achieved_gbs / 8000.0,
                    "fp64_tflops": achieved_tf, "fp64_peak_tflops_measured": fp64_meas_tf}
        else:
            roof = {"bound": "alu", "achieved": achieved_tf, "peak": fp64_meas_tf, "unit": "TFLOP/s",
                    "frac": achieved_tf / fp64_meas_tf,
                    "traffic": load_traffic(args.config) if args.method == "jacobi" and args.precond == 2 else None,
                    "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                                    "profiles/traffic.json)",
                    "peak_source": "DFMA microbenchmark 58.8 FMA/clk/SM x 148 SMs x 2 x sm_max_mhz "
                                   "(profiles/r01_ubench_dfma.txt); nominal 64 FMA/clk/SM = "
                                   f"{fp64_nom_tf:.1f} TFLOP/s",
                    "hbm_gbs": achieved_gbs, "hbm_peak": hbm}
        roof["kernel"] = KERNELS.get(info.kernel_path, f"kernel path {info.kernel_path}")
        if args.method in ("gmres", "gs_gmres", "cheb", "gs"):
            roof["kernel"] = ("whole outer iteration (events around all its kernels): " + roof["kernel"]
                              + {"gmres": " + GMRES panel kernels", "gs_gmres": " + GMRES panel kernels",
                                 "cheb": " + cheb_init/cheb_step kernels", "gs": " on the wavefront windows"}[args.method])
        roof["kernel_ms"] = sweep_ms
        roof["algorithmic"] = {"bytes_per_launch": algo_bytes, "flops_per_launch": info.flops_per_iter,
                               "per_unit": "16 B and 2*(nnz(AA)+nnz(A'))/n_dof flop per space-time DoF "
                                           "update + operator values once (DESIGN.md roofline)"}
        per_step = info.launches_per_iter
        launches = per_step * args.steps
        if info.graph and args.method == "jacobi" and args.steps >= 2:
            launches += 1 + args.steps // 2      # history counter: one set per call + one advance per replay
        if args.method == "gs":   # n_t + K - 1 waves and two checkerboard copies per call
            launches = 2 + (info.n_t_local + args.steps - 1) * per_step
        if args.method == "cheb":   # residual sweep + finalize (1-2) + start + m - 1 steps
            launches = args.steps * (info.launches_per_iter + args.cheb_m)
        if args.method in ("gmres", "gs_gmres"):   # residual + finalize, 2 + k (1 + 2 x 3 + 3) + 1 panel kernels
            launches = args.steps * (2 + 2 + 2 + args.gmres_k * (1 + 6 + 3) + 1)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(args, prob, world), "roofline": roof,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 0 if trig else int(8 * prob.n_t),
                        "d2h_bytes_per_step": int(16 * info.n_t_local),
                        "what": ("per step: biot_iterate(1) + biot_residual_history readback, host sync "
                                 "each step (the §4.1 loads are set up once)" if trig else
                                 "per step: biot_set_load_scale (host s_n) + biot_iterate(1) + "
                                 "biot_residual_history readback, host sync each step")},
                "gpu_launches": launches,
                "timing": {"repeats": reps, "runs_ms": [r[0] for r in runs], "reported": "median run",
                           "cuda_graph": bool(info.graph) and args.method == "jacobi",
                           "comm_nranks": int(info.comm_nranks) if world > 1 else None},
                "clocks": clocks}
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(prob, args.precond, args.omega)
        print(json.dumps(line), flush=True)
    g.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
