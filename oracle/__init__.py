"""TurboReg CPU oracle — TEST INFRASTRUCTURE ONLY.

Thin ctypes wrappers over ``oracle/turboreg_oracle.cpp`` (a plain, literal C++17 implementation of the
paper's definitions; see that file's header for the step list and PAPER.md citations).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module.  The product package ``paper_2507_01439_b200`` never
imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "turboreg_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library (g++, fixed float semantics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class Params(ctypes.Structure):
    _fields_ = [
        ("tau", ctypes.c_float),
        ("k1", ctypes.c_int32),
        ("k2", ctypes.c_int32),
        ("inlier_threshold", ctypes.c_float),
        ("graph_mode", ctypes.c_int32),
        ("rank_metric", ctypes.c_int32),
    ]


class Result(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_float * 9),
        ("t", ctypes.c_float * 3),
        ("inlier_count", ctypes.c_int32),
        ("clique", ctypes.c_int32 * 3),
        ("clique_weight", ctypes.c_int32),
        ("num_pivots", ctypes.c_int32),
        ("num_cliques", ctypes.c_int32),
        ("hypotheses_evaluated", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("num_edges", ctypes.c_int64),
        ("near_edges", ctypes.c_int64),
        ("f64_disagreements", ctypes.c_int64),
        ("neighbor_checks", ctypes.c_int64),
        ("best_count_f64", ctypes.c_int32),
        ("near_corr", ctypes.c_int32),
        ("mae", ctypes.c_double),
        ("mse", ctypes.c_double),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64, f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        _lib.oracle_compat.argtypes = [P, P, i32, f32, P, P, P]
        _lib.oracle_compat.restype = i64
        _lib.oracle_sc2.argtypes = [P, i32, P]
        _lib.oracle_o2.argtypes = [P, i32, P]
        _lib.oracle_select_pivots.argtypes = [P, i32, i32, P]
        _lib.oracle_select_pivots.restype = i32
        _lib.oracle_pgs.argtypes = [P, i32, P, i32, i32, P, P]
        _lib.oracle_pgs.restype = i32
        _lib.oracle_canonical.argtypes = [P, i32, i32]
        _lib.oracle_canonical.restype = i32
        _lib.oracle_triangle_degenerate.argtypes = [P, P, P]
        _lib.oracle_triangle_degenerate.restype = i32
        _lib.oracle_kabsch.argtypes = [P, P, i32, P, P]
        _lib.oracle_kabsch.restype = i32
        _lib.oracle_count_inliers.argtypes = [P, P, i32, P, P, f32]
        _lib.oracle_count_inliers.restype = i32
        _lib.oracle_brute_triangles.argtypes = [P, i32, P, i64]
        _lib.oracle_brute_triangles.restype = i64
        _lib.oracle_estimate.argtypes = [P, P, i32, ctypes.POINTER(Params), ctypes.POINTER(Result), P, P, P, P, P, P]
        _lib.oracle_hypothesis_errors.argtypes = [P, P, i32, P, P, P, P]
        _lib.oracle_estimate.restype = i32
        u64 = ctypes.c_uint64
        _lib.oracle_splitmix64.argtypes = [u64, u64]
        _lib.oracle_splitmix64.restype = u64
        _lib.oracle_ransac_triple.argtypes = [u64, i64, i32, P]
        _lib.oracle_ransac.argtypes = [P, P, i32, i32, u64, f32, ctypes.POINTER(Result), P, P]
        _lib.oracle_ransac.restype = i32
        _lib.oracle_point_resolution.argtypes = [P, i32]
        _lib.oracle_point_resolution.restype = f32
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------------------------------- step wrappers
def compat(src, dst, tau):
    """Eq. 1 → (C uint8 [n,n], n_edges, near_edges, f64_disagreements)."""
    src, dst = _f32(src), _f32(dst)
    n = src.shape[0]
    C = np.zeros((n, n), np.uint8)
    near, dis = ctypes.c_int64(), ctypes.c_int64()
    e = lib().oracle_compat(_p(src), _p(dst), n, float(np.float32(tau)), _p(C), ctypes.byref(near), ctypes.byref(dis))
    return C, int(e), int(near.value), int(dis.value)


def sc2(C):
    """Eq. 2 → Ĝ int32 [n,n]."""
    C = np.ascontiguousarray(C, dtype=np.uint8)
    n = C.shape[0]
    G = np.zeros((n, n), np.int32)
    lib().oracle_sc2(_p(C), n, _p(G))
    return G


def o2(G):
    """Def. 2 → Õ int32 [n,n] (strict upper triangle of Ĝ)."""
    G = np.ascontiguousarray(G, dtype=np.int32)
    n = G.shape[0]
    O = np.zeros((n, n), np.int32)
    lib().oracle_o2(_p(G), n, _p(O))
    return O


def select_pivots(Gbar, k1):
    """Eq. 4 → int32 [P,3] rows (i, j, w) in (w desc, i asc, j asc) order."""
    Gbar = np.ascontiguousarray(Gbar, dtype=np.int32)
    n = Gbar.shape[0]
    piv = np.zeros((max(k1, 1), 3), np.int32)
    m = lib().oracle_select_pivots(_p(Gbar), n, int(k1), _p(piv))
    return piv[:m].copy()


def pgs(Gbar, pivots, k2):
    """Alg. 1 L5-13 → (cliques int32 [K,4] rows (i,j,z,S) in pivot order, neighbour checks)."""
    Gbar = np.ascontiguousarray(Gbar, dtype=np.int32)
    pivots = np.ascontiguousarray(pivots, dtype=np.int32).reshape(-1, 3)
    n = Gbar.shape[0]
    cap = max(1, pivots.shape[0] * int(k2))
    out = np.zeros((cap, 4), np.int32)
    chk = ctypes.c_int64()
    m = lib().oracle_pgs(_p(Gbar), n, _p(pivots), pivots.shape[0], int(k2), _p(out), ctypes.byref(chk))
    return out[:m].copy(), int(chk.value)


def canonical(cliques, dedup=False):
    cl = np.ascontiguousarray(cliques, dtype=np.int32).reshape(-1, 4).copy()
    m = lib().oracle_canonical(_p(cl), cl.shape[0], 1 if dedup else 0)
    return cl[:m].copy()


def triangle_degenerate(p0, p1, p2):
    return bool(lib().oracle_triangle_degenerate(_p(_f32(p0)), _p(_f32(p1)), _p(_f32(p2))))


def kabsch(P, Q):
    """Least-squares rigid fit Q ≈ R P + t in float64 → (R [3,3], t [3]) or None if degenerate."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    R = np.zeros(9, np.float64)
    t = np.zeros(3, np.float64)
    st = lib().oracle_kabsch(_p(P), _p(Q), P.shape[0], _p(R), _p(t))
    if st != 0:
        return None
    return R.reshape(3, 3), t


def count_inliers(src, dst, R, t, thr):
    src, dst = _f32(src), _f32(dst)
    R = _f32(np.asarray(R).reshape(9))
    t = _f32(np.asarray(t).reshape(3))
    return int(lib().oracle_count_inliers(_p(src), _p(dst), src.shape[0], _p(R), _p(t), float(np.float32(thr))))


def brute_triangles(C):
    C = np.ascontiguousarray(C, dtype=np.uint8)
    n = C.shape[0]
    m = lib().oracle_brute_triangles(_p(C), n, None, 0)
    out = np.zeros((max(m, 1), 3), np.int32)
    lib().oracle_brute_triangles(_p(C), n, _p(out), m)
    return out[:m].copy()


def estimate(src, dst, tau, k1, k2, inlier_threshold, graph_mode=0, trace=False, rank_metric=0):
    """Full oracle pipeline (steps 1-9).  Returns dict with the result and, if trace, the intermediates.
    rank_metric: 0 = inlier number (Eq. 9), 1 = MAE, 2 = MSE (App. F.1, reading r20)."""
    src, dst = _f32(src), _f32(dst)
    n = src.shape[0]
    prm = Params(float(tau), int(k1), int(k2), float(inlier_threshold), int(graph_mode), int(rank_metric))
    res = Result()
    C = G = piv = cl = hyp = err = None
    if trace:
        C = np.zeros((n, n), np.uint8)
        G = np.zeros((n, n), np.int32)
        piv = np.zeros((max(k1, 1), 3), np.int32)
        cl = np.zeros((max(k1 * k2, 1), 4), np.int32)
        hyp = np.zeros((max(k1 * k2, 1), 16), np.float32)
        err = np.zeros((max(k1 * k2, 1), 2), np.float64)
    lib().oracle_estimate(_p(src), _p(dst), n, ctypes.byref(prm), ctypes.byref(res), _p(C), _p(G), _p(piv), _p(cl), _p(hyp),
                          _p(err))
    out = {
        "status": res.status,
        "R": np.array(res.R, np.float32).reshape(3, 3),
        "t": np.array(res.t, np.float32),
        "inlier_count": res.inlier_count,
        "clique": tuple(res.clique),
        "clique_weight": res.clique_weight,
        "num_pivots": res.num_pivots,
        "num_cliques": res.num_cliques,
        "hypotheses_evaluated": res.hypotheses_evaluated,
        "num_edges": res.num_edges,
        "near_edges": res.near_edges,
        "f64_disagreements": res.f64_disagreements,
        "neighbor_checks": res.neighbor_checks,
        "best_count_f64": res.best_count_f64,
        "near_corr": res.near_corr,
        "mae": res.mae,
        "mse": res.mse,
    }
    if trace:
        nc = res.num_cliques
        h = hyp[:nc]
        out.update(
            C=C,
            G=G,
            pivots=piv[: res.num_pivots].copy(),
            cliques=cl[:nc].copy(),
            hyp_R=h[:, :9].reshape(-1, 3, 3).copy(),
            hyp_t=h[:, 9:12].copy(),
            hyp_count=h[:, 12].copy().view(np.int32),
            hyp_degenerate=h[:, 13].copy().view(np.int32),
            hyp_mae=err[:nc, 0].copy(),
            hyp_mse=err[:nc, 1].copy(),
        )
    return out


def hypothesis_errors(src, dst, R, t):
    """(MAE, MSE) of a float32 hypothesis over all correspondences (reading r20)."""
    src, dst = _f32(src), _f32(dst)
    mae, mse = ctypes.c_double(), ctypes.c_double()
    lib().oracle_hypothesis_errors(_p(src), _p(dst), src.shape[0], _p(_f32(np.asarray(R).reshape(9))),
                                   _p(_f32(np.asarray(t).reshape(3))), ctypes.byref(mae), ctypes.byref(mse))
    return mae.value, mse.value


# ------------------------------------------------------------------------------------ NEXT(4) RANSAC
def splitmix64(seed, k):
    """k-th output of the counter-based SplitMix64 stream seeded with `seed` (the RANSAC sampler's draws)."""
    return int(lib().oracle_splitmix64(int(seed) & (2**64 - 1), int(k)))


def ransac_triple(seed, k, n):
    """Correspondence triple k (sorted, distinct) of the RANSAC baseline."""
    out = np.zeros(3, np.int32)
    lib().oracle_ransac_triple(int(seed) & (2**64 - 1), int(k), int(n), _p(out))
    return tuple(int(x) for x in out)


def ransac(src, dst, iters, seed, inlier_threshold, trace=False):
    """Equal-budget 3-point RANSAC baseline: `iters` sampled triples, steps 7-8 per
    triple, argmax by (count desc, (i,j,z) asc)."""
    src, dst = _f32(src), _f32(dst)
    n = src.shape[0]
    res = Result()
    cl = hyp = None
    if trace:
        cl = np.zeros((max(iters, 1), 4), np.int32)
        hyp = np.zeros((max(iters, 1), 16), np.float32)
    lib().oracle_ransac(_p(src), _p(dst), n, int(iters), int(seed) & (2**64 - 1), float(inlier_threshold),
                        ctypes.byref(res), _p(cl), _p(hyp))
    out = {
        "status": res.status,
        "R": np.array(res.R, np.float32).reshape(3, 3),
        "t": np.array(res.t, np.float32),
        "inlier_count": res.inlier_count,
        "clique": tuple(res.clique),
        "num_cliques": res.num_cliques,
        "hypotheses_evaluated": res.hypotheses_evaluated,
        "best_count_f64": res.best_count_f64,
        "near_corr": res.near_corr,
    }
    if trace:
        out.update(cliques=cl[:iters].copy(), hyp_R=hyp[:iters, :9].reshape(-1, 3, 3).copy(),
                   hyp_t=hyp[:iters, 9:12].copy(), hyp_count=hyp[:iters, 12].copy().view(np.int32),
                   hyp_degenerate=hyp[:iters, 13].copy().view(np.int32))
    return out


# ------------------------------------------------------------------------------------ NEXT(3) resolution
def point_resolution(xyz):
    """Median nearest-neighbour distance of a point cloud (lower median, float32 distances, reading r22);
    the τ initialisation of P:322 is 0.25 × this."""
    xyz = _f32(xyz)
    return float(lib().oracle_point_resolution(_p(xyz), xyz.shape[0]))
