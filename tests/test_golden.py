"""Pins to numbers the paper prints (tests/golden/paper_values.json, each with its citation)."""
import json
import os

import numpy as np

import synth
from oracle import discretize as D, mlgmres

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_peak_memory_matches_paper():
    ks = G["mlgmres_memory_vector"]["value"]
    assert mlgmres.peak_vectors(G["outer_fgmres_inner"]["value"], ks[1], ks[3]) == \
        G["peak_memory_vectors_3535_ki5"]["value"]
    # Table 4 measured usage never exceeds the bound
    assert max(G["table4_measured_vectors"]["value"].values()) <= G["peak_memory_vectors_3535_ki5"]["value"]


def test_table3_grid_rule():
    """R17: n = n_lambda n_ppw + 2 n_ppw + 1 (PML = 1 wavelength per side) reproduces 13 of the 15
    printed sizes; (25,6) and (50,6) are printed as 161 / 311 (rule: 163 / 313)."""
    tab = G["table3_grid_points_per_axis"]["value"]
    miss = []
    for nl, row in tab.items():
        for ppw, n in zip((6, 8, 10), row):
            if synth.table3_grid(int(nl), ppw) != n:
                miss.append((int(nl), ppw))
    assert sorted(miss) == [(25, 6), (50, 6)]


def test_dot_test_at_paper_magnitude():
    """Table 5: relative difference of the Helmholtz adjoint test is O(1e-15)."""
    p = synth.tiny3d()
    H = D.helmholtz_matrix(p, 2 * np.pi * 8.0, D.default_pml(p.m))
    x, y = synth.random_complex(p.n_ext, 1), synth.random_complex(p.n_ext, 3)
    a, b = np.vdot(y, H @ x), np.vdot(H.conj().T @ y, x)
    rel = abs(a - b) / max(abs(a), abs(b))
    assert rel < 100 * G["table5_helmholtz_dot_test_rel_diff"]["value"]


def test_table3_workload_generator():
    """synth.table3 builds every Table 3 cell with the R17 grid rule, one
    wavelength of PML (n_ppw points) per side, h = lambda / n_ppw and a centred source."""
    for nl, ppw in synth.TABLE3_CELLS:
        p = synth.table3(nl, ppw)
        n = synth.table3_grid(nl, ppw)
        assert p.next == (n, n, n)
        assert all(w == (ppw, ppw) for w in p.pml)
        lam = 1.0 / np.sqrt(p.m.max()) / p.freqs[0]
        assert abs(lam / p.h - ppw) < 1e-12
        assert abs(p.n[0] * p.h - (nl * lam + p.h)) < 1e-9 * lam   # n_lambda wavelengths (+ one node)
        s = int(p.src[0])
        assert (s % p.n[0], (s // p.n[0]) % p.n[1], s // (p.n[0] * p.n[1])) == (p.n[0] // 2,) * 3
