import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200 import _arrays as A, denoise as D
n = 8192
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
img = np.random.default_rng(0).random((n, n))
print("threads", torch.get_num_threads())
for _ in range(2): pnp.dsg_nlm_denoise(img, p)
def t(f, *a):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(*a); torch.cuda.synchronize(); return r, (time.perf_counter() - t0) * 1e3
for rep in range(3):
    _, tot = t(pnp.dsg_nlm_denoise, img, p)
    _, tv = t(A.validate, img)
    x, td = t(A.to_device, img)
    out, tk = t(pnp.dsg_nlm_denoise, x, p)
    _, tf = t(A.from_device, out, A.NUMPY)
    _, te = t(np.empty, (n, n))
    z, tz = t(np.empty, (n, n)); 
    _, tt = t(z.fill, 0.0)
    print(f"total {tot:.1f} validate {tv:.1f} to_device {td:.1f} denoise {tk:.1f} from_device {tf:.1f} np.empty+touch {tt:.1f}")
