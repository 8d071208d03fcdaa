#!/bin/bash
# Debug-build hygiene run (profiles/checks_r2.log): product vs the PNP_CHECKS +
# PNP_JITTER build, twice, over every device path (scripts/checks_run.py).
set -e
python scripts/checks_run.py /tmp/chk_ref.npz
for i in 1 2; do PNP_B200_LIB=build/var_checks/libpnpb200.so python scripts/checks_run.py /tmp/chk_$i.npz; done
python - <<'PY'
import numpy as np
ref = dict(np.load("/tmp/chk_ref.npz"))
for i in (1, 2):
    got = dict(np.load(f"/tmp/chk_{i}.npz"))
    bad = [k for k in ref if not np.array_equal(ref[k], got[k], equal_nan=True)]
    print(f"debug run {i}: {len(ref)} outputs, bitwise different: {bad or 'none'}")
PY
