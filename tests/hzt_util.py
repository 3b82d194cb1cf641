"""Shared helpers for the test suite."""
import numpy as np


def rel_err(a, b):
    den = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (den if den > 0 else 1.0))


# ---- compact 27-point operator (config 4): numpy restatement of the spec in
# include/hz_b200.h (hz_problem_create_ex) with the weights of
# scripts/design_27pt.py, used as the checker of the GPU operator
W27 = dict(a1=0.30896924112207297, a2=0.5974547869846899, c1=0.49495786061914238, c2=0.023557529253244218,
           c3=2.4579791982563098e-08)


def weights27(h):
    a1, a2, c1, c2, c3 = (W27[k] for k in ("a1", "a2", "c1", "c2", "c3"))
    a3, c0 = 1.0 - a1 - a2, 1.0 - c1 - c2 - c3
    ih2 = 1.0 / (h * h)
    lap = [0.0, a1 * ih2, a2 * ih2 / 4.0, a3 * ih2 / 4.0]
    lap[0] = -(6.0 * lap[1] + 12.0 * lap[2] + 8.0 * lap[3])
    mu = [c0, c1 / 6.0, c2 / 12.0, c3 / 8.0]
    return lap, mu


def csr27(cfg, shift=0.0):
    """scipy CSR of the compact 27-point operator with gamma + shift*omega."""
    import scipy.sparse as sp
    n0, n1, n2 = cfg.n
    lap, mu = weights27(cfg.h[0])
    w = cfg.omega
    gam = cfg.gamma_base + w * cfg.ramp
    M = w * w * (1.0 - 1j * gam / w) * cfg.m - 1j * shift * w * w * cfg.m
    idx = np.arange(n0 * n1 * n2).reshape(n2, n1, n0)
    rows, cols, vals = [idx.ravel()], [idx.ravel()], [lap[0] + mu[0] * M]
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                q = abs(dx) + abs(dy) + abs(dz)
                if q == 0:
                    continue
                sl_i = (slice(max(0, -dz), n2 - max(0, dz)), slice(max(0, -dy), n1 - max(0, dy)),
                        slice(max(0, -dx), n0 - max(0, dx)))
                sl_j = (slice(max(0, dz), n2 - max(0, -dz)), slice(max(0, dy), n1 - max(0, -dy)),
                        slice(max(0, dx), n0 - max(0, -dx)))
                i, j = idx[sl_i].ravel(), idx[sl_j].ravel()
                rows.append(i)
                cols.append(j)
                vals.append(lap[q] + mu[q] * 0.5 * (M[i] + M[j]))
    n = n0 * n1 * n2
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))


def symbol27(kvec, h, mval, w):
    """Plane-wave symbol of the 27-point operator (constant m, gamma = 0):
    A exp(i k.x) = S exp(i k.x) at interior nodes."""
    lap, mu = weights27(h)
    c = np.cos(np.asarray(kvec) * h)
    s1 = c.sum()
    s2 = c[0] * c[1] + c[0] * c[2] + c[1] * c[2]
    s3 = c.prod()
    L = lap[0] + lap[1] * 2 * s1 + lap[2] * 4 * s2 + lap[3] * 8 * s3
    Mk = mu[0] + mu[1] * 2 * s1 + mu[2] * 4 * s2 + mu[3] * 8 * s3
    return L + w * w * mval * Mk
