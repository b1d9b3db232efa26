"""Shared test helpers: golden-fixture parsing and brute-force pins written independently of oracle/."""
from __future__ import annotations

import itertools
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_app_e():
    """Parse tests/golden/app_e_fixture.txt → dict of 0-based expectations."""
    out = {"cliques": [], "sc2": {}, "rowsum": {}, "pivot": [], "o2clique": [], "sc2clique": []}
    with open(os.path.join(GOLDEN, "app_e_fixture.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            tag, *vals = line.split()
            v = [int(x) for x in vals]
            if tag == "clique":
                out["cliques"].append([x - 1 for x in v])
            elif tag == "sc2":
                out["sc2"][(v[0] - 1, v[1] - 1)] = v[2]
            elif tag == "triangles":
                out["triangles"] = v[0]
            elif tag == "rowsum":
                out["rowsum"][v[0] - 1] = v[1]
            elif tag == "pivot":
                out["pivot"].append((v[0] - 1, v[1] - 1, v[2]))
            elif tag in ("o2clique", "sc2clique"):
                out[tag].append((v[0] - 1, v[1] - 1, v[2] - 1, v[3]))
    n = 1 + max(max(c) for c in out["cliques"])
    C = np.zeros((n, n), np.uint8)
    for c in out["cliques"]:
        for a, b in itertools.permutations(c, 2):
            C[a, b] = 1
    out["C"] = C
    return out


def py_triangles(C):
    """Brute-force 3-cliques by plain Python loops over index triples (independent of oracle/)."""
    n = C.shape[0]
    tri = []
    for i in range(n):
        for j in range(i + 1, n):
            if not C[i, j]:
                continue
            for z in range(j + 1, n):
                if C[i, z] and C[j, z]:
                    tri.append((i, j, z))
    return tri


def triangles_per_edge(C):
    """Count, for every unordered edge, the brute-force triangles containing it (App. B)."""
    cnt = {}
    for (i, j, z) in py_triangles(C):
        for e in ((i, j), (i, z), (j, z)):
            cnt[e] = cnt.get(e, 0) + 1
    return cnt


def random_rotation(rng):
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array(
        [
            [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
            [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
            [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
        ]
    )


def numpy_kabsch(P, Q):
    """Textbook Kabsch via numpy.linalg.svd (library routine), independent of oracle/'s Jacobi SVD."""
    P = np.asarray(P, np.float64)
    Q = np.asarray(Q, np.float64)
    cp, cq = P.mean(0), Q.mean(0)
    H = (P - cp).T @ (Q - cq)
    U, S, Vt = np.linalg.svd(H)
    d = np.sign(np.linalg.det(Vt.T @ U.T))
    R = Vt.T @ np.diag([1.0, 1.0, d]) @ U.T
    return R, cq - R @ cp


def rot_angle_deg(R_est, R_gt):
    """Angle between rotations, well-conditioned near 0: θ = 2 asin(||R − R_gt||_F / (2√2))."""
    d = np.linalg.norm(np.asarray(R_est, np.float64) - np.asarray(R_gt, np.float64))
    return float(np.degrees(2 * np.arcsin(min(1.0, d / (2 * np.sqrt(2))))))
