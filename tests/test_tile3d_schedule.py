"""Host logic of the tile3d static list schedule (CPU only).

`biot::tile3d_schedule` (csrc/tile3d_kernels.cu) is internal C++ (std::vector
arguments), so a ten-line g++ wrapper compiled into a temporary directory exposes it to
ctypes; the wrapper resolves the symbol from the already-loaded libbiot_pit.so.  Checked:
the table is a partition of the mesh (every (patch, plane) covered exactly once, so a
schedule bug cannot drop or double-update a node), the per-CTA slices tile the table, the
cut never makes the simulated makespan worse than plain round robin, and the function's
values on config 4's mesh (n1 = 65) for 22- and 13-plane tiles.
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from paper_2310_10430_b200 import _lib

WRAP = r"""
#include <cstdint>
#include <vector>
namespace biot {
int tile3d_schedule(int n1, int z_rows, int grid, double h, std::vector<int32_t> &tab,
                    std::vector<int32_t> &off, double *makespan, double *makespan_rr);
}
extern "C" int t3_sched(int n1, int z_rows, int grid, double h, int32_t *tab, int cap, int32_t *off,
                        double *ms, double *rr) {
    std::vector<int32_t> t, o;
    const int G = biot::tile3d_schedule(n1, z_rows, grid, h, t, o, ms, rr);
    if ((int)t.size() > cap || (int)o.size() != G + 1) return -1;
    for (size_t i = 0; i < t.size(); ++i) tab[i] = t[i];
    for (size_t i = 0; i < o.size(); ++i) off[i] = o[i];
    return (int)(t.size() / 4) * 1024 + G;   // tiles, CTAs (G <= 1023 here)
}
"""
BX, BY = 4, 3   # the kernel's patch (kBX, kBY)


@pytest.fixture(scope="module")
def sched(tmp_path_factory):
    ctypes.CDLL(_lib.LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    d = tmp_path_factory.mktemp("t3sched")
    src, so = d / "wrap.cpp", d / "libt3wrap.so"
    src.write_text(WRAP)
    subprocess.run(["g++", "-O1", "-shared", "-fPIC", str(src), "-o", str(so)], check=True)
    L = ctypes.CDLL(str(so))
    i32p, dp = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)
    L.t3_sched.argtypes = [ctypes.c_int] * 3 + [ctypes.c_double, i32p, ctypes.c_int, i32p, dp, dp]
    L.t3_sched.restype = ctypes.c_int

    def call(n1, z_rows, grid, h):
        cap = 4 * 8 * ((n1 + BX - 1) // BX) * ((n1 + BY - 1) // BY) * ((n1 + z_rows - 1) // z_rows)
        tab = np.zeros(cap, np.int32)
        off = np.zeros(grid + 2, np.int32)
        ms, rr = ctypes.c_double(), ctypes.c_double()
        r = L.t3_sched(n1, z_rows, grid, h, tab.ctypes.data_as(i32p), cap, off.ctypes.data_as(i32p),
                       ctypes.byref(ms), ctypes.byref(rr))
        assert r >= 0
        nt, G = r // 1024, r % 1024
        return tab[:4 * nt].reshape(nt, 4), off[:G + 1], ms.value, rr.value

    return call


@pytest.mark.parametrize("n1,z_rows,grid,h", [(65, 22, 148, 1.0), (65, 22, 148, 0.0), (129, 24, 148, 1.0),
                                              (17, 8, 148, 1.0), (9, 5, 148, 0.25), (33, 11, 7, 1.0),
                                              (65, 13, 148, 0.5), (6, 5, 148, 1.0)])
def test_schedule_is_a_partition(sched, n1, z_rows, grid, h):
    tab, off, ms, rr = sched(n1, z_rows, grid, h)
    G = len(off) - 1
    assert 1 <= G <= grid and off[0] == 0 and off[-1] == len(tab)
    assert np.all(np.diff(off) >= 1)                      # every launched CTA has work
    cover = np.zeros((n1, (n1 + BY - 1) // BY, (n1 + BX - 1) // BX), np.int32)   # (plane, patch y, patch x)
    for x0, y0, za, zb in tab:
        assert x0 % BX == 0 and y0 % BY == 0 and 0 <= x0 < n1 and 0 <= y0 < n1
        assert 0 <= za < zb <= n1 and zb - za <= z_rows
        cover[za:zb, y0 // BY, x0 // BX] += 1
    assert cover.min() == 1 and cover.max() == 1          # each (patch, plane) exactly once
    # the simulated makespan is the busiest CTA's planes + h per tile, never above round robin
    load = [float(np.sum(tab[off[c]:off[c + 1], 3] - tab[off[c]:off[c + 1], 2])) + h * (off[c + 1] - off[c])
            for c in range(G)]
    assert max(load) == pytest.approx(ms, abs=1e-9)
    assert ms <= rr + 1e-9
    assert ms >= (n1 * cover.shape[1] * cover.shape[2] + h * len(tab)) / G - 1e-9   # work / CTAs


def test_schedule_config4_numbers(sched):
    """Config 4's mesh (n1 = 65, 17 x 22 patches, 148 CTAs): 22-plane tiles (3 ranges, 1122
    base tiles = 7.6 rounds) with h = 1, and 13-plane tiles (5 ranges, 1870 = 12.6 rounds) with
    h = 0.25; values worked out by hand for round robin: 8 tiles of 22+1 planes less three
    21-plane ones = 181; 13 tiles of 13.25 = 172.25."""
    tab, off, ms, rr = sched(65, 22, 148, 1.0)
    assert len(off) - 1 == 148
    assert len(tab) == 1356 and rr == 181.0 and ms == 175.0
    t13, o13, ms13, rr13 = sched(65, 13, 148, 0.25)
    assert len(t13) == 2112 and rr13 == 172.25 and ms13 == 169.5
    # within a CTA the tiles keep the dealing order (spatial neighbours march concurrently):
    # the first tile of CTA c is base tile c of the first round
    npx = (65 + BX - 1) // BX
    for c in (0, 1, 17, 147):
        assert tuple(tab[off[c]][:2]) == ((c % npx) * BX, (c // npx) * BY)

