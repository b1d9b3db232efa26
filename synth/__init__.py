"""Seeded synthetic correspondence sets (shared input generator; holds none of the method's arithmetic).

This is the only module both the CUDA path's tests/bench and the oracle consume.  It draws planted
ground-truth registration problems shaped like the paper's workloads (generator
adapted from SPEC synth S:456-478):

* numpy ``PCG64(seed)``; geometry drawn in float64, stored as float32;
* ground-truth rotation from a uniform unit quaternion, translation uniform in ±extent/2 per axis;
* source points uniform in the box [-extent/2, extent/2]^3 (per-axis extent);
* inlier targets ``R x + t + N(0, σ² I)``, redrawn while ``||noise|| > 6σ``;
* outlier targets uniform in the axis-aligned bounding box of the transformed source points;
* inlier indices are a seeded random permutation (reading r17: O2 depends on index order).

Configs A–E are BASELINE.json ``configs[0..4]``; their numeric parameters are SURVEY.md §8(d)'s table.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

GENERATOR = "numpy.random.PCG64"


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    inlier_ratio: float
    extent: tuple  # box side per axis, metres
    sigma: float  # inlier noise, metres
    tau: float  # τ of Eq. 1 (stringent, Def. 1)
    inlier_threshold: float  # g(·) residual bound
    k1: int
    k2: int
    seed: int


CONFIGS = {
    # BASELINE.json configs[0]: synthetic N=500, 90% outliers, 0.5K TurboCliques, single pair
    "A": Workload("synthetic_N500", 500, 0.10, (1.0, 1.0, 1.0), 0.005, 0.0125, 0.015, 500, 2, 1000),
    # configs[1]: 3DMatch+FCGF-shaped, N=5000, ~25% inliers, 1K TurboCliques (τ = 0.012)
    "B": Workload("3dmatch_fcgf_N5000", 5000, 0.25, (3.0, 3.0, 3.0), 0.010, 0.012, 0.10, 1000, 2, 2000),
    # configs[2]: 3DLoMatch-shaped, ~5% inliers, 2K TurboCliques
    "C": Workload("3dlomatch_N5000", 5000, 0.05, (3.0, 3.0, 3.0), 0.010, 0.012, 0.10, 2000, 2, 3000),
    # configs[3]: KITTI+FPFH-shaped outdoor, metre-scale thresholds, 1K TurboCliques
    "D": Workload("kitti_fpfh_N5000", 5000, 0.20, (80.0, 80.0, 6.0), 0.10, 0.25, 0.6, 1000, 2, 4000),
    # configs[4]: batch sweep of 1623 3DMatch-shaped pairs; pair p uses seed 100000 + p
    "E": Workload("3dmatch_batch_N5000", 5000, 0.25, (3.0, 3.0, 3.0), 0.010, 0.012, 0.10, 1000, 2, 100000),
}

BATCH_PAIRS = 1623  # 3DMatch pair count


def _rotation_from_quaternion(q):
    w, x, y, z = q / np.linalg.norm(q)
    return np.array(
        [
            [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
            [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
            [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
        ]
    )


def generate(n, inlier_ratio, extent, sigma, seed):
    """Draw one planted instance.  Returns dict(src, dst float32 [n,3]; R, t float64; inlier_mask bool)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ext = np.broadcast_to(np.asarray(extent, np.float64), (3,))
    R = _rotation_from_quaternion(rng.standard_normal(4))
    t = rng.uniform(-ext / 2, ext / 2)
    src = rng.uniform(-ext / 2, ext / 2, size=(n, 3))
    moved = src @ R.T + t
    n_in = int(round(n * inlier_ratio))
    perm = rng.permutation(n)
    mask = np.zeros(n, bool)
    mask[perm[:n_in]] = True
    dst = np.empty_like(src)
    idx_in = np.nonzero(mask)[0]
    noise = rng.standard_normal((n_in, 3)) * sigma
    if sigma > 0:
        while True:
            bad = np.linalg.norm(noise, axis=1) > 6 * sigma
            if not bad.any():
                break
            noise[bad] = rng.standard_normal((int(bad.sum()), 3)) * sigma
    dst[idx_in] = moved[idx_in] + noise
    lo, hi = moved.min(axis=0), moved.max(axis=0)
    idx_out = np.nonzero(~mask)[0]
    dst[idx_out] = rng.uniform(lo, hi, size=(idx_out.size, 3))
    return {
        "src": src.astype(np.float32),
        "dst": dst.astype(np.float32),
        "R": R,
        "t": t,
        "inlier_mask": mask,
        "seed": seed,
        "generator": GENERATOR,
    }


def workload_instance(cfg: Workload, pair: int = 0, n: int | None = None):
    """Instance ``pair`` of workload ``cfg`` (seed = cfg.seed + pair); optional size override."""
    return generate(n or cfg.n, cfg.inlier_ratio, cfg.extent, cfg.sigma, cfg.seed + pair)


def with_n(cfg: Workload, n: int) -> Workload:
    return replace(cfg, n=n)


def rotation_error_deg(R_est, R_gt):
    """RE = arccos((tr(R_gtᵀ R) − 1)/2) in degrees."""
    c = (np.trace(np.asarray(R_gt, np.float64).T @ np.asarray(R_est, np.float64)) - 1.0) / 2.0
    return float(np.degrees(np.arccos(np.clip(c, -1.0, 1.0))))


def translation_error(t_est, t_gt):
    return float(np.linalg.norm(np.asarray(t_est, np.float64) - np.asarray(t_gt, np.float64)))


def erdos_renyi(n, density, seed):
    """Symmetric 0/1 adjacency (zero diagonal) at the given edge density (SPEC acceptance 1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    up = np.triu(rng.random((n, n)) < density, 1)
    return (up | up.T).astype(np.uint8)


def fixture_app_e():
    """App. E graph as read by S:149: union of the cliques {1..5} and {2,4,6,7}; 0-based."""
    C = np.zeros((7, 7), np.uint8)
    for clique in ([0, 1, 2, 3, 4], [1, 3, 5, 6]):
        for a in clique:
            for b in clique:
                if a != b:
                    C[a, b] = 1
    return C
