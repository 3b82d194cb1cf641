"""Weights of the compact 27-point Helmholtz stencil (config 4's fine
operator; the reference has only the 7-point one, src/helmholtz.cpp:45-100).

Family (uniform spacing h; faces f, edges e, corners c of the 3x3x3 cell):
  Lap u ~ a1/h^2 sum_f (u_f - u_0) + a2/(4h^2) sum_e (u_e - u_0) + a3/(4h^2) sum_c (u_c - u_0)
  mass  ~ c0 M_0 u_0 + c1/6 sum_f M_0f u_f + c2/12 sum_e M_0e u_e + c3/8 sum_c M_0c u_c
with a1 + a2 + a3 = 1 and c0 + c1 + c2 + c3 = 1 (each piece consistent to
second order) and M_0j = (M_0 + M_j)/2 (complex symmetric). For a constant
medium the plane-wave symbol (h = 1, theta = k h) is
  Lap(k)  = 2 a1 sum(cos t_a - 1) + a2 sum_{a<b}(cos t_a cos t_b - 1) + 2 a3 (cx cy cz - 1)
  Mass(k) = c0 + c1/3 sum cos t_a + c2/3 sum_{a<b} cos t_a cos t_b + c3 cx cy cz
and the numerical phase velocity is v_num / v = sqrt(-Lap / Mass) / |k h|.
The five free weights minimise the squared phase-velocity error over
propagation directions (a Fibonacci sphere) and 4 to 12 grid points per
wavelength (the north star's 10 ppw sits inside). Prints the weights
(csrc/hierarchy.cu kStencil27) and the error table against the 7-point stencil.
"""
import numpy as np
from scipy.optimize import least_squares


def directions(n=200):
    i = np.arange(n) + 0.5
    phi = np.arccos(1 - 2 * i / n)
    th = np.pi * (1 + 5 ** 0.5) * i
    d = np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], 1)
    return d[d[:, 2] >= 0]  # the symbol is even


def vratio(w, ppw, dirs):
    a1, a2, c1, c2, c3 = w
    a3, c0 = 1 - a1 - a2, 1 - c1 - c2 - c3
    kh = 2 * np.pi / ppw
    t = dirs * kh
    c = np.cos(t)
    s1 = c.sum(1)
    s2 = c[:, 0] * c[:, 1] + c[:, 0] * c[:, 2] + c[:, 1] * c[:, 2]
    s3 = c.prod(1)
    lap = 2 * a1 * (s1 - 3) + a2 * (s2 - 3) + 2 * a3 * (s3 - 1)
    mass = c0 + c1 / 3 * s1 + c2 / 3 * s2 + c3 * s3
    return np.sqrt(-lap / mass) / kh


def residual(w, dirs, ppws):
    return np.concatenate([vratio(w, g, dirs) - 1.0 for g in ppws])


def main():
    dirs = directions()
    ppws = np.linspace(4.0, 12.0, 33)
    r = least_squares(residual, x0=[0.3, 0.5, 0.2, 0.1, 0.01], args=(dirs, ppws), bounds=([0, 0, 0, 0, 0], [1, 1, 1, 1, 1]))
    a1, a2, c1, c2, c3 = r.x
    print(f"a1={a1:.17g}\na2={a2:.17g}\na3={1 - a1 - a2:.17g}\nc0={1 - c1 - c2 - c3:.17g}\nc1={c1:.17g}\nc2={c2:.17g}\nc3={c3:.17g}")
    seven = [1.0, 0.0, 0.0, 0.0, 0.0]  # a1 = 1, c0 = 1: the 7-point operator
    print("ppw   max|v/v0-1| 27-pt     7-pt")
    for g in (4, 5, 6, 8, 10, 12, 20):
        print(f"{g:4d}   {np.abs(vratio(r.x, g, dirs) - 1).max():.3e}   {np.abs(vratio(seven, g, dirs) - 1).max():.3e}")


if __name__ == "__main__":
    main()
