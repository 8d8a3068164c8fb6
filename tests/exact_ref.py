"""Exact rational brute force — an independent PIN for the fp64 oracle (tests only).

Pure-Python loops over ``fractions.Fraction`` for tiny clouds (N, M <= 64): exact squared
distances, exact lowest-index argmin (SPEC.md:441 brute force; R3), exact Chamfer
(SPEC.md:441 mean+mean) and exact gradients with the argmin held fixed.  Written separately
from oracle/chamfer_oracle.c (different language, exact arithmetic) so that a dropped term, a
wrong sign or index, or a transposed operand in the oracle shows up as a mismatch.
"""
from fractions import Fraction


def _frac_cloud(a):
    return [[[Fraction(float(c)) for c in p] for p in cloud] for cloud in a]


def sqdist(p, q):
    return sum((p[c] - q[c]) ** 2 for c in range(3))


def nn_exact(q, t):
    """q, t: nested lists of Fractions [B][P][3].  Returns (d, idx, d2) nested lists."""
    D, I, D2 = [], [], []
    for b in range(len(q)):
        db, ib, sb = [], [], []
        for x in q[b]:
            ds = [sqdist(x, y) for y in t[b]]
            best = min(ds)
            arg = ds.index(best)  # lowest index attaining the exact minimum
            rest = ds[:arg] + ds[arg + 1:]
            db.append(best)
            ib.append(arg)
            sb.append(min(rest) if rest else None)
        D.append(db)
        I.append(ib)
        D2.append(sb)
    return D, I, D2


def chamfer_exact(x, y, w1=1, w2=1):
    X, Y = _frac_cloud(x), _frac_cloud(y)
    dxy, ixy, sxy = nn_exact(X, Y)
    dyx, iyx, syx = nn_exact(Y, X)
    B = len(X)
    cd = [Fraction(w1) * sum(dxy[b]) / len(dxy[b]) + Fraction(w2) * sum(dyx[b]) / len(dyx[b]) for b in range(B)]
    loss = sum(cd) / B
    return dict(d_xy=dxy, idx_xy=ixy, d2_xy=sxy, d_yx=dyx, idx_yx=iyx, d2_yx=syx, cd=cd, loss=loss, X=X, Y=Y)


def grad_exact(X, Y, ixy, iyx, g, h):
    """Exact VJP: g[b][i], h[b][j] Fractions.  Returns grad_x, grad_y nested [B][P][3]."""
    B = len(X)
    gx = [[[Fraction(0)] * 3 for _ in X[b]] for b in range(B)]
    gy = [[[Fraction(0)] * 3 for _ in Y[b]] for b in range(B)]
    for b in range(B):
        for i, a in enumerate(ixy[b]):
            for c in range(3):
                diff = X[b][i][c] - Y[b][a][c]
                gx[b][i][c] += 2 * g[b][i] * diff   # d/dx_i of ||x_i - y_a||^2
                gy[b][a][c] -= 2 * g[b][i] * diff   # d/dy_a of the same term
        for j, a in enumerate(iyx[b]):
            for c in range(3):
                diff = Y[b][j][c] - X[b][a][c]
                gy[b][j][c] += 2 * h[b][j] * diff
                gx[b][a][c] -= 2 * h[b][j] * diff
    return gx, gy
