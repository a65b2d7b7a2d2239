"""Time the sweep-kernel variants (env-selected) on one config: ms/iteration and
the fused sweep kernel alone, CUDA events inside the library.  Dev tool."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2310_10430_b200 import BiotSolver  # noqa: E402
from workloads import config_problem  # noqa: E402


def main():
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    variants = sys.argv[2:] or ["generic", "march:2", "march:4", "4,2", "2,4"]
    prob = config_problem(cid)
    K = 10
    for v in variants:
        for k in ("BIOT_KERNEL", "BIOT_STENCIL_R", "BIOT_STENCIL_T", "BIOT_MARCH_T", "BIOT_MARCH_ROWS"):
            os.environ.pop(k, None)
        os.environ.pop("BIOT_TILE_CFG", None)
        os.environ.pop("BIOT_TILE_DRY", None)
        if v.endswith(":dry"):
            os.environ["BIOT_TILE_DRY"] = "1"
            v = v[:-4]
        if v in ("generic", "tile"):
            os.environ["BIOT_KERNEL"] = v
        elif v.startswith("tile:"):          # tile:r,stages,maxreg
            os.environ["BIOT_KERNEL"] = "tile"
            os.environ["BIOT_TILE_CFG"] = v.split(":")[1]
        elif v.startswith("march"):          # march[:T[:rows]]
            f = v.split(":")
            os.environ["BIOT_KERNEL"] = "march"
            if len(f) > 1:
                os.environ["BIOT_MARCH_T"] = f[1]
            if len(f) > 2:
                os.environ["BIOT_MARCH_ROWS"] = f[2]
        else:
            raise SystemExit(f"unknown variant {v}")
        for pc in (2, 1):
            if os.environ.get("BIOT_TILE_DRY") and pc == 1:
                continue
            try:
                g = BiotSolver(prob, precond=pc, omega=0.5)
            except Exception as e:  # unsupported combination
                print(f"config{cid} {v:12s} P{pc}: {e}")
                continue
            g.iterate(3)
            g.iterate(K)
            it, sw = g.last_timing()
            inf = g.info
            gbs = inf.bytes_per_iter / (sw / 1e3) / 1e9
            print(f"config{cid} {v:12s} P{pc} path={inf.kernel_path} iter {it:8.3f} ms  sweep {sw:8.3f} ms"
                  f"  algo {gbs:7.0f} GB/s  {inf.n_dof * inf.n_t_local / (it / 1e3) / 1e9:7.1f} GDoF/s",
                  flush=True)
            g.close()


if __name__ == "__main__":
    main()
