"""Cost of page-locking a fresh 512 MB numpy result (cudaHostRegister) vs
filling it, and D2H float64 into it (diagnosis for the numpy drop-in tail)."""
import time

import numpy as np
import torch

n = 8192
cud = torch.cuda.cudart()
g64 = torch.rand(n, n, device="cuda", dtype=torch.float64)
torch.cuda.synchronize()
for rep in range(3):
    r = np.empty((n, n))
    t0 = time.perf_counter()
    torch.from_numpy(r).zero_()
    t1 = time.perf_counter()
    rc = cud.cudaHostRegister(r.ctypes.data, r.nbytes, 0)
    t2 = time.perf_counter()
    torch.from_numpy(r).copy_(g64, non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    cud.cudaHostUnregister(r.ctypes.data)
    t4 = time.perf_counter()
    r2 = np.empty((n, n))
    t5 = time.perf_counter()
    rc2 = cud.cudaHostRegister(r2.ctypes.data, r2.nbytes, 0)   # fresh, not faulted
    t6 = time.perf_counter()
    cud.cudaHostUnregister(r2.ctypes.data)
    print(f"zero {1e3*(t1-t0):.1f} register(touched) {1e3*(t2-t1):.1f} rc={rc} D2H f64 {1e3*(t3-t2):.1f} "
          f"unregister {1e3*(t4-t3):.1f} register(fresh) {1e3*(t6-t5):.1f} rc={rc2}")
p = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); p.copy_(g64, non_blocking=True); torch.cuda.synchronize()
    print("D2H f64 into pinned", round(1e3 * (time.perf_counter() - t), 1))
for rep in range(2):
    t = time.perf_counter(); q = torch.empty((n, n), dtype=torch.float64, pin_memory=True); print("pinned alloc (cached?)", round(1e3 * (time.perf_counter() - t), 1)); del q
