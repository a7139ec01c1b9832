"""Derive the weights of the "optimal" mixed-grid stencils (DESIGN R34/R35; a
2D 9-point "optimal" stencil [23] and a 3D compact 27-point stencil [60], whose coefficients
the paper does not print). The stencil families (product forms of 1D operators, so that the
PML enters through the same stretched 1D tables T_a as STD2):

  2D: L = a (T_x + T_z) + (1 - a) (T_x A_z + A_x T_z)
      M = c I + (d/2) (E_x + E_z) + (1 - c - d) E_x E_z
  3D: L = w1 sum_a T_a + (w2/2) sum_a T_a (A_b + A_c) + (1 - w1 - w2) sum_a T_a A_b A_c
      M = m1 I + (m2/3) sum_a E_a + (m3/3) sum_{a<b} E_a E_b + (1 - m1 - m2 - m3) E_x E_y E_z
  H = L + omega^2 M diag(m)        (Eq. 7 with A = M)

T_a: stretched second difference (D4), A_a = (1/4, 1/2, 1/4), E_a = (1/2, 0, 1/2). In the
interior the plane-wave symbols are -(4/h^2) sin^2(t_a/2), cos^2(t_a/2) and cos(t_a); the
weights minimise the squared phase-velocity error sqrt(-L/(M k^2)) - 1 over propagation
directions and 4 to infinitely many points per wavelength (1/G uniform in (0, 1/4]), which
is the design criterion of the "optimal" stencils the paper cites. Prints the weights and
the worst / mean phase error at G = 4, 5, 6, 8, 10 against STD2.

    python scripts/derive_opt_stencil.py
"""
import json

import numpy as np
from scipy.optimize import least_squares

G_MIN = 4.0


def sym2(p, th_x, th_z):
    a, c, d = p
    e = 1 - c - d
    tx, tz = 4 * np.sin(th_x / 2) ** 2, 4 * np.sin(th_z / 2) ** 2
    ax, az = np.cos(th_x / 2) ** 2, np.cos(th_z / 2) ** 2
    ex, ez = np.cos(th_x), np.cos(th_z)
    negL = a * (tx + tz) + (1 - a) * (tx * az + ax * tz)
    M = c + d / 2 * (ex + ez) + e * ex * ez
    return negL, M


def sym3(p, th):
    w1, w2, m1, m2, m3 = p
    w3, m4 = 1 - w1 - w2, 1 - m1 - m2 - m3
    t = 4 * np.sin(th / 2) ** 2
    al = np.cos(th / 2) ** 2
    ep = np.cos(th)
    negL = 0.0
    for a in range(3):
        b, c = [i for i in range(3) if i != a]
        negL = negL + w1 * t[a] + w2 / 2 * t[a] * (al[b] + al[c]) + w3 * t[a] * al[b] * al[c]
    M = m1 + m2 / 3 * ep.sum(0) + m3 / 3 * (ep[0] * ep[1] + ep[0] * ep[2] + ep[1] * ep[2]) + m4 * ep[0] * ep[1] * ep[2]
    return negL, M


def samples2(n_g=24, n_phi=16):
    inv_g = np.linspace(1.0 / G_MIN, 1e-3, n_g)
    phi = np.linspace(0, np.pi / 4, n_phi)
    IG, PH = np.meshgrid(inv_g, phi, indexing="ij")
    kh = 2 * np.pi * IG
    return kh.ravel(), kh.ravel() * np.cos(PH.ravel()), kh.ravel() * np.sin(PH.ravel())


def samples3(n_g=20, n_dir=12):
    inv_g = np.linspace(1.0 / G_MIN, 1e-3, n_g)
    pol = np.linspace(0, np.pi / 2, n_dir)
    az = np.linspace(0, np.pi / 4, n_dir)
    IG, PO, AZ = np.meshgrid(inv_g, pol, az, indexing="ij")
    kh = 2 * np.pi * IG.ravel()
    d = np.stack([np.sin(PO.ravel()) * np.cos(AZ.ravel()), np.sin(PO.ravel()) * np.sin(AZ.ravel()), np.cos(PO.ravel())])
    return kh, kh * d


def phase_err2(p, kh, tx, tz):
    negL, M = sym2(p, tx, tz)
    return np.sqrt(negL / (M * kh**2)) - 1


def phase_err3(p, kh, th):
    negL, M = sym3(p, th)
    return np.sqrt(negL / (M * kh**2)) - 1


def report(err_fn, p, n_dim):
    out = {}
    for G in (4, 5, 6, 8, 10):
        kh = 2 * np.pi / G
        if n_dim == 2:
            phi = np.linspace(0, np.pi / 4, 91)
            e = err_fn(p, np.full_like(phi, kh), kh * np.cos(phi), kh * np.sin(phi))
        else:
            pol, az = np.meshgrid(np.linspace(0, np.pi / 2, 46), np.linspace(0, np.pi / 4, 46), indexing="ij")
            d = np.stack([np.sin(pol.ravel()) * np.cos(az.ravel()), np.sin(pol.ravel()) * np.sin(az.ravel()),
                          np.cos(pol.ravel())])
            e = err_fn(p, np.full(d.shape[1], kh), kh * d)
        out[G] = {"max_abs": float(np.abs(e).max()), "mean_abs": float(np.abs(e).mean())}
    return out


def main():
    # all weights (including the dependent last ones) kept non-negative: a convex combination
    # of consistent Laplacians and a non-negative mass distribution (well-posed coarse grids;
    # the unconstrained optimum has large cancelling weights of both signs)
    pen = 1e3
    kh, tx, tz = samples2()
    r2 = least_squares(lambda p: np.concatenate([phase_err2(p, kh, tx, tz), [pen * min(0.0, 1 - p[1] - p[2])]]),
                       x0=[0.5, 0.6, 0.1], bounds=([0, 0, 0], [1, 1, 1]))
    kh3, th3 = samples3()
    r3 = least_squares(lambda p: np.concatenate([phase_err3(p, kh3, th3), [pen * min(0.0, 1 - p[0] - p[1]),
                                                                         pen * min(0.0, 1 - p[2] - p[3] - p[4])]]),
                       x0=[0.3, 0.3, 0.5, 0.3, 0.15], bounds=([0] * 5, [1] * 5))
    std2_2 = report(phase_err2, [1.0, 1.0, 0.0], 2)
    std2_3 = report(phase_err3, [1.0, 0.0, 1.0, 0.0, 0.0], 3)
    res = {
        "opt9_2d": {"a": r2.x[0], "c": r2.x[1], "d": r2.x[2], "e": 1 - r2.x[1] - r2.x[2],
                    "phase_error": report(phase_err2, r2.x, 2), "std2_phase_error": std2_2},
        "opt27_3d": {"w1": r3.x[0], "w2": r3.x[1], "w3": 1 - r3.x[0] - r3.x[1], "m1": r3.x[2], "m2": r3.x[3],
                     "m3": r3.x[4], "m4": 1 - r3.x[2] - r3.x[3] - r3.x[4],
                     "phase_error": report(phase_err3, r3.x, 3), "std2_phase_error": std2_3},
    }
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
