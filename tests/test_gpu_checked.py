"""The checked build (lib/libturboreg_checked.so, -DTRK_CHECKS): after the SC^2 assembly every O2 edge slot
must hold its increasing neighbour j > i with C_ij = 1 and Ĝ_ij = popcount(row_i AND row_j) (Eq. 2), each
row's slot count must equal |U_i|, every TurboClique must be a 3-clique with S = the sum of its weights
(Eq. 6) and every pivot a positive O2 edge — verified on the device over configs A–D, batches, SC^2 mode,
RANSAC, the split path and Erdős–Rényi graphs; a violation traps and the run fails.  (compute-sanitizer is
closed on the GPU pool; this is the substitute for its memcheck / racecheck on index arithmetic.)
Needs a B200: `pytest -m gpu`."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_invariants():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = os.path.join(ROOT, "paper_2507_01439_b200", "lib", "libturboreg_checked.so")
    if not os.path.exists(lib):
        from paper_2507_01439_b200.build import build

        build(checked=True)
    env = dict(os.environ, TURBOREG_LIBRARY=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "--full"], env=env,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "TRK_CHECKS" not in r.stdout + r.stderr
    assert f"library {lib}" in r.stdout
