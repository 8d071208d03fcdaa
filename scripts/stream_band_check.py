"""DenoiseStream with / without the banded first upload: one-image and
five-image runs at 8192^2 (development aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1901_06110_b200 as pnp

n = 8192
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
host = torch.rand(n, n).pin_memory()
outs = [torch.empty_like(host).pin_memory() for _ in range(5)]
st = pnp.DenoiseStream(p, (n, n))
bands = st._bands
for label, b in (("banded", bands), ("plain", None), ("banded", bands), ("plain", None)):
    st._bands = b
    for k in (1, 5):
        st.run([host] * k, outs[:k])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.run([host] * k, outs[:k])
        e1.record()
        torch.cuda.synchronize()
        print(f"{label:7s} {k} images: {e0.elapsed_time(e1):8.2f} ms", flush=True)
