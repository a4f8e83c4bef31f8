"""ORACLE / TEST INFRASTRUCTURE — numpy restatement of the Q2 and rotated-Q1 hierarchies
(include/pf_fe.h, BASELINE configs[2] and configs[3]).  The reference has neither family
(its assembly is Q1 only): "parity unpinned by the reference".  The restatement follows
the reference's Q1 algorithm (element matrices by tensor Gauss quadrature,
assembly.cpp:48-88; global entries summed over their cells in ascending cell order,
assembly.cpp:90-142; Dirichlet rows kept with identity values, assembly.cpp:162-170;
the load by the same quadrature, assembly.cpp:144-160; per-fine-dof (coarse dof, weight)
prolongation lists, multigrid.cpp:35-72) generalised to the two families, written
independently of paper_1609_04809_b200/csrc/pf_fe_setup.cpp:

  - entries are assembled by an element loop (np.add.at in cell order) instead of the
    product's per-row gather;
  - the Q2 prolongation evaluates the coarse basis at the fine nodes; the rotated-Q1 one
    integrates the coarse basis over each fine face with a 2 x 2 Gauss rule (the product
    uses closed-form weights), so it is compared within 1e-15;
  - the exact-solution dof values come from per-axis libm tables.

Small grids only (tests/test_fe_setup.py).  Only tests may import this module.
"""
from __future__ import annotations

import math

import numpy as np

from oracle.coef import kappa as lognormal_kappa

DIRICHLET, INDEP = 7, 1


def gauss(n):
    if n == 2:
        r = 0.5 / math.sqrt(3.0)
        return [0.5 - r, 0.5 + r], [0.5, 0.5]
    r = 0.5 * math.sqrt(0.6)
    return [0.5 - r, 0.5, 0.5 + r], [5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0]


class Level:
    """One level in host order: own entities first, then Dirichlet ones, each
    lexicographic.  Attributes mirror paper_1609_04809_b200.levels.LevelArrays."""

    def __init__(self, lex_keys, boundary):
        self.boundary = np.asarray(boundary, bool)
        own = np.flatnonzero(~self.boundary)
        dirs = np.flatnonzero(self.boundary)
        self.lex_of = np.concatenate([own, dirs])
        self.host_of = np.empty(len(self.lex_of), np.int64)
        self.host_of[self.lex_of] = np.arange(len(self.lex_of))
        self.n, self.n_own = len(self.lex_of), len(own)
        self.keys = np.asarray(lex_keys, np.int64)[self.lex_of]
        self.is_dir = np.zeros(self.n, np.uint8)
        self.is_dir[self.n_own:] = 1
        self.class_of = np.where(self.is_dir == 1, DIRICHLET, INDEP).astype(np.uint8)
        self.owns_row = np.ones(self.n, np.uint8)
        self.order = self.lex_of.astype(np.int64)

    def assemble(self, cell_dofs, elem):
        """cell_dofs[c] = lex entity of every local dof of cell c (cells ascending);
        elem[c] = that cell's element matrix.  Own rows: sum over cells in cell order;
        Dirichlet rows: the same pattern with identity values."""
        cell_dofs = np.asarray(cell_dofs)
        nloc = cell_dofs.shape[1]
        r = self.host_of[np.repeat(cell_dofs, nloc, axis=1)].reshape(-1)
        c = self.host_of[np.tile(cell_dofs, (1, nloc))].reshape(-1)
        v = np.asarray(elem).reshape(-1)
        key = r * self.n + c
        uniq, pos = np.unique(key, return_inverse=True)
        vals = np.zeros(len(uniq))
        np.add.at(vals, pos, v)  # sequential, in cell order
        rows, cols = uniq // self.n, uniq % self.n
        vals = np.where(rows >= self.n_own, np.where(rows == cols, 1.0, 0.0), vals)
        self.row_offsets = np.zeros(self.n + 1, np.int64)
        np.add.at(self.row_offsets, rows + 1, 1)
        self.row_offsets = np.cumsum(self.row_offsets)
        self.cols = cols.astype(np.int32)
        self.vals = vals

    def set_prolongation(self, rows):
        """rows[h] = list of (coarse host index, weight)."""
        off = [0]
        cols, w = [], []
        for row in rows:
            for c, x in sorted(row):
                cols.append(c)
                w.append(x)
            off.append(len(cols))
        self.p_offsets = np.array(off, np.int64)
        self.p_cols = np.array(cols, np.int32)
        self.p_w = np.array(w, np.float64)


# ------------------------------------------------------------------------- Q2 --

def q2_phi(i, t):
    return (1.0 - t) * (1.0 - 2.0 * t) if i == 0 else (4.0 * t) * (1.0 - t) if i == 1 else t * (2.0 * t - 1.0)


def q2_dphi(i, t):
    return 4.0 * t - 3.0 if i == 0 else 4.0 - 8.0 * t if i == 1 else 4.0 * t - 1.0


def q2_unit_stiffness():
    t, w = gauss(3)
    V = [[q2_phi(i, t[q]) for q in range(3)] for i in range(3)]
    D = [[q2_dphi(i, t[q]) for q in range(3)] for i in range(3)]
    loc = [(a // 9, (a // 3) % 3, a % 3) for a in range(27)]
    K = np.zeros((27, 27))
    for a, (ax, ay, az) in enumerate(loc):
        for b, (bx, by, bz) in enumerate(loc):
            s = 0.0
            for qx in range(3):
                for qy in range(3):
                    for qz in range(3):
                        wq = (w[qx] * w[qy]) * w[qz]
                        ga = ((D[ax][qx] * V[ay][qy]) * V[az][qz], (V[ax][qx] * D[ay][qy]) * V[az][qz],
                              (V[ax][qx] * V[ay][qy]) * D[az][qz])
                        gb = ((D[bx][qx] * V[by][qy]) * V[bz][qz], (V[bx][qx] * D[by][qy]) * V[bz][qz],
                              (V[bx][qx] * V[by][qy]) * D[bz][qz])
                        s += wq * ((ga[0] * gb[0] + ga[1] * gb[1]) + ga[2] * gb[2])
            K[a, b] = s
    return K


def q2_level(N):
    M = 2 * N + 1
    i, j, k = np.meshgrid(np.arange(M), np.arange(M), np.arange(M), indexing="ij")
    lex_keys = np.stack([np.zeros(M ** 3, np.int64), i.ravel(), j.ravel(), k.ravel()], 1)
    bnd = ((i == 0) | (j == 0) | (k == 0) | (i == M - 1) | (j == M - 1) | (k == M - 1)).ravel()
    L = Level(lex_keys, bnd)
    h = 1.0 / N
    Ke = np.array([[h * x for x in row] for row in q2_unit_stiffness()])
    cells = [(cx, cy, cz) for cx in range(N) for cy in range(N) for cz in range(N)]
    dofs = [[((2 * cx + a // 9) * M + 2 * cy + (a // 3) % 3) * M + 2 * cz + a % 3 for a in range(27)]
            for cx, cy, cz in cells]
    L.assemble(dofs, [Ke] * len(cells))
    cls = lambda x: 2 if x & 1 else (0 if x % 4 == 0 else 1)  # noqa: E731
    L.color = np.array([(cls(a) * 3 + cls(b)) * 3 + cls(c) for _, a, b, c in L.keys[:L.n_own]], np.int32)
    L.N = N
    return L


def q2_prolongation(F, Cl):
    Mc = 2 * Cl.N + 1

    def axis(i):  # coarse Q2 basis of the coarse cell containing fine node i, at i
        cell = min(i // 4, Cl.N - 1)
        t = (i - 4 * cell) / 4.0
        return [(2 * cell + m, q2_phi(m, t)) for m in range(3) if q2_phi(m, t) != 0.0]

    rows = []
    for _, i, j, k in F.keys:
        rows.append([(int(Cl.host_of[(ci * Mc + cj) * Mc + ck]), (wi * wj) * wk)
                     for ci, wi in axis(i) for cj, wj in axis(j) for ck, wk in axis(k)])
    F.set_prolongation(rows)


def q2_rhs(L):
    N, M = L.N, 2 * L.N + 1
    t, w = gauss(3)
    h = 1.0 / N
    vol, K3 = (h * h) * h, (3.0 * math.pi) * math.pi
    S = np.array([[math.sin(math.pi * ((float(c) + t[q]) * h)) for q in range(3)] for c in range(N)])
    V = [[q2_phi(i, t[q]) for q in range(3)] for i in range(3)]
    cx, cy, cz = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    cx, cy, cz = cx.ravel(), cy.ravel(), cz.ravel()
    le = np.zeros((N ** 3, 27))
    for qx in range(3):
        for qy in range(3):
            for qz in range(3):
                wq = (w[qx] * w[qy]) * w[qz]
                f = ((K3 * S[cx, qx]) * S[cy, qy]) * S[cz, qz]
                wf = (wq * vol) * f
                phi = np.array([(V[a // 9][qx] * V[(a // 3) % 3][qy]) * V[a % 3][qz] for a in range(27)])
                le += wf[:, None] * phi[None, :]
    b = np.zeros(L.n)
    for hh in range(L.n_own):
        _, i, j, k = L.keys[hh]
        acc = 0.0
        for ci in _q2_cells(i, N):
            for cj in _q2_cells(j, N):
                for ck in _q2_cells(k, N):
                    acc += le[(ci * N + cj) * N + ck, ((i - 2 * ci) * 3 + (j - 2 * cj)) * 3 + (k - 2 * ck)]
        b[hh] = acc
    s = [math.sin(math.pi * (float(p) / float(2 * N))) for p in range(M)]
    exact = np.array([((1.0 * s[i]) * s[j]) * s[k] for _, i, j, k in L.keys])
    return b, exact


def _q2_cells(i, N):
    if i & 1:
        return [(i - 1) // 2]
    return [c for c in (i // 2 - 1, i // 2) if 0 <= c < N]


# ----------------------------------------------------------------- rotated Q1 --

def rt_phi(o, sigma, X):
    p, q = [a for a in range(3) if a != o]
    return (1.0 / 6.0 + (0.5 * sigma) * X[o]) + 0.25 * ((2.0 * X[o] * X[o] - X[p] * X[p]) - X[q] * X[q])


def rt_grad(o, sigma, X):
    return [sigma + 2.0 * X[a] if a == o else -X[a] for a in range(3)]


def rt_unit_stiffness():
    t, w = gauss(2)
    K = np.zeros((6, 6))
    for a in range(6):
        for b in range(6):
            s = 0.0
            for qx in range(2):
                for qy in range(2):
                    for qz in range(2):
                        X = [2.0 * t[qx] - 1.0, 2.0 * t[qy] - 1.0, 2.0 * t[qz] - 1.0]
                        wq = (w[qx] * w[qy]) * w[qz]
                        ga = rt_grad(a // 2, 1.0 if a & 1 else -1.0, X)
                        gb = rt_grad(b // 2, 1.0 if b & 1 else -1.0, X)
                        s += wq * ((ga[0] * gb[0] + ga[1] * gb[1]) + ga[2] * gb[2])
            K[a, b] = s
    return K


def rt_faces(N):
    keys = []
    for o in range(3):
        ext = [N + (o == a) for a in range(3)]
        for a0 in range(ext[0]):
            for a1 in range(ext[1]):
                for a2 in range(ext[2]):
                    keys.append((o, a0, a1, a2))
    return keys


def rt_face_lex(N, o, a):
    per = N * N * (N + 1)
    e1, e2 = N + (o == 1), N + (o == 2)
    return o * per + (a[0] * e1 + a[1]) * e2 + a[2]


def rt_cell_faces(N, cell):
    """lex faces of a cell's local slots s = 2 o + (+ side)."""
    out = []
    for s in range(6):
        o = s // 2
        a = list(cell)
        a[o] += s & 1
        out.append(rt_face_lex(N, o, a))
    return out


def rt_kappas(N_finest, n_levels, lognormal, seed):
    """finest: the generator keyed by the lexicographic cell number; coarser: the mean of
    the 8 children (child order dx, dy, dz)."""
    Nf = N_finest
    fine = [lognormal_kappa(seed, c) if lognormal else 1.0 for c in range(Nf ** 3)]
    kap = [fine]
    N = Nf
    for _ in range(n_levels - 1):
        Nc = N // 2
        kc = []
        for c in range(Nc ** 3):
            cx, cy, cz = c // (Nc * Nc), (c // Nc) % Nc, c % Nc
            s = 0.0
            for d in range(8):
                s += kap[0][((2 * cx + (d >> 2)) * N + 2 * cy + ((d >> 1) & 1)) * N + 2 * cz + (d & 1)]
            kc.append(0.125 * s)
        kap.insert(0, kc)
        N = Nc
    return kap


def rt_level(N, kappa):
    keys = rt_faces(N)
    bnd = [a[o] in (0, N) for o, *a in [(k[0], k[1], k[2], k[3]) for k in keys]]
    L = Level(np.array(keys, np.int64), bnd)
    h = 1.0 / N
    Ke = np.array([[h * x for x in row] for row in rt_unit_stiffness()])
    cells = [(cx, cy, cz) for cx in range(N) for cy in range(N) for cz in range(N)]
    L.assemble([rt_cell_faces(N, c) for c in cells],
               [np.array([[kappa[i] * Ke[a, b] for b in range(6)] for a in range(6)]) for i in range(len(cells))])
    L.color = np.array([2 * o + (a[o] & 1) for o, *a in L.keys[:L.n_own].tolist()], np.int32)
    L.N = N
    return L


def rt_prolongation(F, Cl):
    """Mean of the coarse function over each own fine face (2 x 2 Gauss on the face in the
    coarse cell's reference coordinates), the two sides of a coarse face averaged; no
    entries for Dirichlet fine faces."""
    t, w = gauss(2)
    Nc = Cl.N
    rows = []
    for hh, (o, *a) in enumerate(F.keys.tolist()):
        if hh >= F.n_own:
            rows.append([])
            continue
        sides = []  # (coarse cell coords, X_o of the fine face in that cell)
        if a[o] & 1:
            sides.append(((a[o] - 1) // 2, 0.0))
        else:
            if a[o] // 2 - 1 >= 0:
                sides.append((a[o] // 2 - 1, 1.0))
            if a[o] // 2 < Nc:
                sides.append((a[o] // 2, -1.0))
        acc = {}
        for co, Xo in sides:
            cell = [co if ax == o else a[ax] // 2 for ax in range(3)]
            faces = rt_cell_faces(Nc, cell)
            tang = [ax for ax in range(3) if ax != o]
            for s in range(6):
                m = 0.0
                for q1 in range(2):
                    for q2 in range(2):
                        X = [0.0, 0.0, 0.0]
                        X[o] = Xo
                        for ax, q in zip(tang, (q1, q2)):
                            lo = -1.0 if (a[ax] & 1) == 0 else 0.0  # the fine face's half
                            X[ax] = lo + t[q]
                        m += (w[q1] * w[q2]) * rt_phi(s // 2, 1.0 if s & 1 else -1.0, X)
                if abs(m) < 1e-14:
                    continue
                col = int(Cl.host_of[faces[s]])
                acc[col] = acc.get(col, 0.0) + m / len(sides)
        rows.append(list(acc.items()))
    F.set_prolongation(rows)


def rt_rhs(L):
    N = L.N
    t, w = gauss(3)
    h = 1.0 / N
    vol, K3 = (h * h) * h, (3.0 * math.pi) * math.pi
    S = np.array([[math.sin(math.pi * ((float(c) + t[q]) * h)) for q in range(3)] for c in range(N)])
    cx, cy, cz = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    cx, cy, cz = cx.ravel(), cy.ravel(), cz.ravel()
    le = np.zeros((N ** 3, 6))
    for q in range(27):
        qx, qy, qz = q // 9, (q // 3) % 3, q % 3
        X = [2.0 * t[qx] - 1.0, 2.0 * t[qy] - 1.0, 2.0 * t[qz] - 1.0]
        wq = (w[qx] * w[qy]) * w[qz]
        f = ((K3 * S[cx, qx]) * S[cy, qy]) * S[cz, qz]
        wf = (wq * vol) * f
        phi = np.array([rt_phi(a // 2, 1.0 if a & 1 else -1.0, X) for a in range(6)])
        le += wf[:, None] * phi[None, :]
    b = np.zeros(L.n)
    for hh in range(L.n_own):
        o, *a = L.keys[hh].tolist()
        acc = 0.0
        for side in (0, 1):
            co = a[o] - 1 + side
            if 0 <= co < N:
                c = list(a)
                c[o] = co
                acc += le[(c[0] * N + c[1]) * N + c[2], 2 * o + (1 if side == 0 else 0)]
        b[hh] = acc
    ph = math.pi * h
    sn = [math.sin(math.pi * (float(x) * h)) for x in range(N + 1)]
    mn = [(math.cos(math.pi * (float(x) * h)) - math.cos(math.pi * (float(x + 1) * h))) / ph for x in range(N)]
    exact = []
    for o, *a in L.keys.tolist():
        u = 1.0
        for ax in range(3):
            u *= sn[a[ax]] if ax == o else mn[a[ax]]
        exact.append(u)
    return b, np.array(exact)


# ---------------------------------------------------------------------- driver --

def build(family, n_coarse, n_levels, lognormal=False, seed=2024):
    """(levels coarsest first, b, x0, exact, finest kappa) of one family; family 2 = Q2,
    3 = rotated Q1 (include/pf_fe.h)."""
    Ns = [n_coarse << l for l in range(n_levels)]
    if family == 2:
        levels = [q2_level(N) for N in Ns]
        for l in range(1, n_levels):
            q2_prolongation(levels[l], levels[l - 1])
        b, exact = q2_rhs(levels[-1])
        kap = [1.0] * Ns[-1] ** 3
    else:
        kaps = rt_kappas(Ns[-1], n_levels, lognormal, seed)
        levels = [rt_level(N, k) for N, k in zip(Ns, kaps)]
        for l in range(1, n_levels):
            rt_prolongation(levels[l], levels[l - 1])
        b, exact = rt_rhs(levels[-1])
        kap = kaps[-1]
    return levels, b, np.zeros(len(b)), exact, np.array(kap)
