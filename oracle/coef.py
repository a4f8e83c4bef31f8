"""ORACLE / TEST INFRASTRUCTURE — restatement of the lognormal-coefficient problem
(PF_PROBLEM_LOGNORMAL, include/pf_setup.h), which the reference does not have (SURVEY.md
§0.1): "parity unpinned by the reference".  Pure-Python loops, small grids only; used by
tests/test_setup.py to pin paper_1609_04809_b200/csrc/pf_setup.cpp (build_coefficients,
coef_entry, the gcn-ordered assembly) entry by entry.

Definitions restated:
  kappa_c = exp(z_c), z_c = sqrt(-2 ln u1) cos(2 pi u2), (u1, u2) from splitmix64 keyed by
  (seed, finest gcn); finest element matrix kappa_c * K_e (K_e: 2-point Gauss Q1
  stiffness, assembly.cpp:48-92); coarse element matrix E_C = sum over children (child
  index order) of P_c^T E_c P_c; level matrix = sum over the cells sharing the two
  vertices, ascending gcn (partition.cpp:184-186).
"""
from __future__ import annotations

import math

M64 = (1 << 64) - 1
RING = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def kappa(seed: int, gcn: int) -> float:
    a = splitmix64(seed ^ splitmix64((gcn * 2 + 1) & M64))
    b = splitmix64(a)
    u1 = (float(a >> 11) + 1.0) / 9007199254740992.0
    u2 = (float(b >> 11) + 1.0) / 9007199254740992.0
    z = math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)
    return math.exp(z)


def gcn(d, n_coarse, level, x, y, z):
    S = 1 << level
    g = ((x // S) * n_coarse + (y // S)) * n_coarse + (z // S) if d == 3 else (x // S) * n_coarse + (y // S)
    for b in range(level - 1, -1, -1):
        ci = ((((x >> b) & 1) << 2) | (((y >> b) & 1) << 1) | ((z >> b) & 1)) if d == 3 else \
             ((((x >> b) & 1) << 1) | ((y >> b) & 1))
        g = g * (1 << d) + ci
    return g


def element_stiffness(d, h):
    """K_e of a cell with extents h (make_element / element_matrices, assembly.cpp:48-92)."""
    nv = 1 << d
    off = 0.5 / math.sqrt(3.0)
    pts = [0.5 - off, 0.5 + off]
    vol = 1.0
    hh = [1.0, 1.0, 1.0]
    for a in range(d):
        hh[a] = h[a]
        vol *= hh[a]
    K = [[0.0] * nv for _ in range(nv)]
    for ix in range(2):
        for iy in range(2):
            for iz in range(2 if d == 3 else 1):
                p = [pts[ix], pts[iy], pts[iz] if d == 3 else 0.0]
                w = 0.5 * 0.5
                if d == 3:
                    w *= 0.5
                qw = w * vol
                grad = []
                for v in range(nv):
                    fac = [1.0, 1.0, 1.0]
                    dfac = [0.0, 0.0, 0.0]
                    for a in range(d):
                        hi = RING[v][a] == 1
                        fac[a] = p[a] if hi else 1.0 - p[a]
                        dfac[a] = 1.0 if hi else -1.0
                    gv = []
                    for a in range(d):
                        gg = dfac[a]
                        for b2 in range(d):
                            if b2 != a:
                                gg *= fac[b2]
                        gv.append(gg)
                    grad.append(gv)
                for i in range(nv):
                    for j in range(nv):
                        gs = 0.0
                        for a in range(d):
                            gs += grad[i][a] * grad[j][a] / (hh[a] * hh[a])
                        K[i][j] += qw * gs
    return K


def coord(level, N, i):
    return float(i) * (1.0 / float(N)) if level == 0 else float(i) / float(N)


def element_matrices(d, n_coarse, n_levels, seed):
    """E[l][(cx, cy, cz)] -> 8x8 (list of lists) for every cell of every level."""
    nv = 1 << d
    L = n_levels
    E = [dict() for _ in range(L)]
    Nf = n_coarse << (L - 1)
    lvlf = L - 1
    for x in range(Nf):
        for y in range(Nf):
            for z in range(Nf if d == 3 else 1):
                h = [coord(lvlf, Nf, x + 1) - coord(lvlf, Nf, x), coord(lvlf, Nf, y + 1) - coord(lvlf, Nf, y),
                     coord(lvlf, Nf, z + 1) - coord(lvlf, Nf, z) if d == 3 else 1.0]
                Ke = element_stiffness(d, h)
                k = kappa(seed, gcn(d, n_coarse, lvlf, x, y, z))
                E[lvlf][(x, y, z)] = [[k * Ke[i][j] for j in range(nv)] for i in range(nv)]
    P = []
    for ci in range(nv):
        o = ((ci >> 2, (ci >> 1) & 1, ci & 1) if d == 3 else (ci >> 1, ci & 1, 0))
        Pc = [[0.0] * nv for _ in range(nv)]
        for k in range(nv):
            for i in range(nv):
                w = 1.0
                for a in range(d):
                    xi = float(o[a] + RING[k][a]) / 2.0
                    w *= xi if RING[i][a] else 1.0 - xi
                Pc[k][i] = w
        P.append((o, Pc))
    for l in range(L - 2, -1, -1):
        Nc = n_coarse << l
        for X in range(Nc):
            for Y in range(Nc):
                for Z in range(Nc if d == 3 else 1):
                    out = [[0.0] * nv for _ in range(nv)]
                    for o, Pc in P:
                        Ec = E[l + 1][(2 * X + o[0], 2 * Y + o[1], 2 * Z + o[2] if d == 3 else 0)]
                        T = [[0.0] * nv for _ in range(nv)]
                        for k in range(nv):
                            for j in range(nv):
                                t = 0.0
                                for m in range(nv):
                                    t += Ec[k][m] * Pc[m][j]
                                T[k][j] = t
                        for i in range(nv):
                            for j in range(nv):
                                u = 0.0
                                for k in range(nv):
                                    u += Pc[k][i] * T[k][j]
                                out[i][j] += u
                    E[l][(X, Y, Z)] = out
    return E


def ring_slot(d, o):
    for v in range(1 << d):
        if RING[v][0] == o[0] and RING[v][1] == o[1] and (d == 2 or RING[v][2] == o[2]):
            return v
    raise ValueError(o)


def matrix_entry(d, n_coarse, level, E, local_cells, p, q):
    """Assembled entry (p, q) (lattice vertices) of a level: the cells containing both that
    are local to the rank, ascending gcn, E[cell][slot p][slot q] summed from 0.0."""
    cells = []
    for cx in range(max(p[0], q[0]) - 1, min(p[0], q[0]) + 1):
        for cy in range(max(p[1], q[1]) - 1, min(p[1], q[1]) + 1):
            zr = range(max(p[2], q[2]) - 1, min(p[2], q[2]) + 1) if d == 3 else [0]
            for cz in zr:
                if (cx, cy, cz) in local_cells:
                    cells.append((gcn(d, n_coarse, level, cx, cy, cz), (cx, cy, cz)))
    v = 0.0
    for _, c in sorted(cells):
        si = ring_slot(d, (p[0] - c[0], p[1] - c[1], p[2] - c[2]))
        sj = ring_slot(d, (q[0] - c[0], q[1] - c[1], q[2] - c[2]))
        v += E[level][c][si][sj]
    return v
