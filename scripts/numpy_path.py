"""Drop-in numpy path at 8192^2: dsg_nlm_denoise(float64 numpy) wall time and
its parts (development aid)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_1901_06110_b200 as pnp

n = 8192
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
img = np.random.default_rng(0).random((n, n))
pnp.dsg_nlm_denoise(img[:512, :512], p)
for _ in range(2):
    t0 = time.perf_counter()
    out = pnp.dsg_nlm_denoise(img, p)
    t1 = time.perf_counter()
    print(f"numpy drop-in 8192^2: {1e3 * (t1 - t0):.1f} ms", flush=True)
t0 = time.perf_counter(); a32 = np.asarray(img, dtype=np.float32); t1 = time.perf_counter()
print(f"  host f64->f32: {1e3 * (t1 - t0):.1f} ms")
t0 = time.perf_counter(); d = torch.from_numpy(a32).cuda(); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"  pageable H2D 256 MB: {1e3 * (t1 - t0):.1f} ms")
t0 = time.perf_counter(); h = d.cpu(); t1 = time.perf_counter()
print(f"  D2H 256 MB: {1e3 * (t1 - t0):.1f} ms")
t0 = time.perf_counter(); h64 = h.numpy().astype(np.float64); t1 = time.perf_counter()
print(f"  host f32->f64: {1e3 * (t1 - t0):.1f} ms")
t0 = time.perf_counter(); d64 = torch.from_numpy(img).cuda(); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"  pageable H2D 512 MB (f64): {1e3 * (t1 - t0):.1f} ms")
t0 = time.perf_counter(); h64b = d64.cpu().numpy(); t1 = time.perf_counter()
print(f"  D2H 512 MB (f64): {1e3 * (t1 - t0):.1f} ms")

# the staged path's pieces
from paper_1901_06110_b200 import _arrays as A
t0 = time.perf_counter(); A.validate(img); t1 = time.perf_counter()
print(f"  validate (threaded isfinite): {1e3 * (t1 - t0):.1f} ms")
t0 = time.perf_counter(); dd = A.to_device(img); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"  to_device (threaded cast to pinned + DMA): {1e3 * (t1 - t0):.1f} ms")
stage = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
t0 = time.perf_counter(); stage.copy_(torch.from_numpy(img)); t1 = time.perf_counter()
print(f"    cast into pinned: {1e3 * (t1 - t0):.1f} ms (threads {torch.get_num_threads()})")
t0 = time.perf_counter(); yd = pnp.dsg_nlm_denoise(dd, p); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"  denoise (device): {1e3 * (t1 - t0):.1f} ms")
t0 = time.perf_counter(); o = A.from_device(yd, A.NUMPY); t1 = time.perf_counter()
print(f"  from_device (device cast + pinned DMA): {1e3 * (t1 - t0):.1f} ms")
