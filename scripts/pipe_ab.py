"""A/B of the band-pipelined adaptive denoise (PNP_PIPE bands) at 8192^2.

Times dsg_nlm_denoise on the config-4 image for each band count, checks the
result is bitwise equal to the sequential path (PNP_PIPE=0), and prints one
line per setting.  Usage: python scripts/pipe_ab.py [n] [bands ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1901_06110_b200 as pnp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
bands = [int(b) for b in sys.argv[2:]] or [0, 2, 4, 8, 16]
params = pnp.PatchParams.from_h(bench.P_C4, bench.R_C4, bench.H_BW, bench.SIGMA_P)
x = torch.from_numpy(bench.make_image_rows(n, 0, n)).cuda()
units = n * n * (2 * bench.R_C4 + 1) ** 2
ref = None
for rep in range(2):
    for nb in bands:
        os.environ["PNP_PIPE"] = str(nb)
        for _ in range(3):
            out = pnp.dsg_nlm_denoise(x, params)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = 10
        e0.record()
        for _ in range(k):
            out = pnp.dsg_nlm_denoise(x, params)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        if ref is None:
            ref = out.clone()
        same = bool(torch.equal(out, ref))
        print(f"rep {rep} PNP_PIPE={nb:3d}  {ms:7.3f} ms  {units / ms / 1e9:8.1f} Gpix*off/s  "
              f"bitwise_equal={same}", flush=True)
