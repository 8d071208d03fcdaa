import cProfile, pstats, sys
sys.argv = ["x"]
exec(open("scripts/admm_overhead.py").read().split("for iters in")[0])
cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=1, constraint=pnp.UNIT_BOX)
for _ in range(5):
    pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
