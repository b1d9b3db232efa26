import sys; sys.path.insert(0, '.')
import numpy as np, synth, oracle
from paper_2507_01439_b200 import TurboReg
from paper_2507_01439_b200._binding import I_SC2, I_STATE
cfg = synth.CONFIGS["C"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8500
inst = synth.workload_instance(cfg, pair=1, n=n)
ref = oracle.estimate(inst["src"], inst["dst"], cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, trace=True)
Gr = ref["G"]; Cr = ref["C"].astype(bool)
deg = Cr.sum(1)
tr = TurboReg(cfg.tau, cfg.k1, cfg.k2, cfg.inlier_threshold, max_n=n)
tr.set_option("sc2_path", 1)
tr.register(inst["src"], inst["dst"])
G = tr.intermediate(0, I_SC2)
U = np.triu(np.ones((n, n), bool), 1)
print("n", n, "W", tr.intermediate(0, I_STATE)["W"])
print("gpu0-ref>0", int(((G == 0) & (Gr > 0) & U).sum()), "gpu>0-ref0", int(((G > 0) & (Gr == 0) & U).sum()), "both>0 differ", int(((G > 0) & (Gr > 0) & (G != Gr) & U).sum()))
bad = np.argwhere((G != Gr) & U)
light = deg <= 64
for a, b in bad[:8]:
    print(a, b, "deg", deg[a], deg[b], "gpu", G[a, b], "ref", Gr[a, b], "C", Cr[a, b])
# per j: which j columns are affected
js = np.unique(bad[:, 1]); print("distinct j", len(js), js[:20])
ii = np.unique(bad[:, 0]); print("distinct i", len(ii), ii[:20])
# are affected pairs those where the common neighbour index k is >= 8192?
a, b = bad[0]
common = np.nonzero(Cr[a] & Cr[b])[0]; print("common nbrs of first bad", common)
