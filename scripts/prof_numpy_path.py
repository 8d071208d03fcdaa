import sys, cProfile, pstats
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1901_06110_b200 as pnp
n = 8192
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
img = np.random.default_rng(0).random((n, n))
for _ in range(2): pnp.dsg_nlm_denoise(img, p)
pr = cProfile.Profile(); pr.enable()
for _ in range(3): pnp.dsg_nlm_denoise(img, p)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
