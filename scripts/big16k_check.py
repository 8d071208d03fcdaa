"""16384^2 adaptive denoise (k cache too large for HBM -> recompute path):
timing and a local parity window against the float64 oracle (development aid)."""
import sys, time, math
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1901_06110_b200 as pnp
import oracle
from oracle import dsg as odsg
N = 16384
p = pnp.PatchParams(7, 10, (12/255)/math.sqrt(2), 2.0)
g = torch.Generator(device="cuda").manual_seed(1)
yy = torch.linspace(0, 1, N, device="cuda")[:, None]
xx = torch.linspace(0, 1, N, device="cuda")[None, :]
clean = 0.15 + 0.7 * (0.5 + 0.5 * torch.sin(40.0 * xx + 25.0 * yy) * torch.cos(30.0 * yy))
x = (clean + (25 / 255) * torch.randn(N, N, device="cuda", generator=g)).contiguous()
torch.cuda.synchronize(); t=time.perf_counter()
out, d, alpha = pnp.dsg_nlm_denoise(x, p, return_aux=True)
torch.cuda.synchronize(); print("16384^2 denoise", round(time.perf_counter()-t,3), "s, alpha", float(alpha[0]))
# local parity on a window far from the borders (d depends on guide within 2R+p)
r0, c0, S, M = 9000, 12000, 40, 2*10+3
crop = x[r0-M:r0+S+M, c0-M:c0+S+M].double().cpu().numpy()
ref_out, ref_d, _ = oracle.dsg_nlm_denoise(crop, 7, 10, (12/255)/math.sqrt(2), patch_sigma=2.0, return_aux=True)
dd = np.abs(d[r0:r0+S, c0:c0+S].double().cpu().numpy() - ref_d[M:M+S, M:M+S]).max()
print("d max abs diff vs oracle crop:", dd, " d range", float(ref_d.min()), float(ref_d.max()))
