#!/bin/bash
# ncu --set full of one config-2 ADMM iteration's kernels (cached apply sweep,
# fixup + u-update, SR residual / adjoint, reductions), warm L2 like the real
# loop; writes gpurun_out/admm_<tag>.ncu-rep and admm_sweep_<tag>.ncu-rep.
# Run only after scripts/admm_prof.py exited 0 without ncu.
tag=${1:-r1}
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"dsg_fixup|sr_adjoint|sr_residual|reduce_partials" \
  --launch-skip 40 -c 6 -o gpurun_out/admm_$tag python scripts/admm_prof.py 30 \
  > gpurun_out/ncu_admm_$tag.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:dsg_sweep --launch-skip 10 -c 1 -o gpurun_out/admm_sweep_$tag \
  python scripts/admm_prof.py 30 > gpurun_out/ncu_admm_sweep_$tag.log 2>&1
tail -n 2 gpurun_out/ncu_admm_$tag.log gpurun_out/ncu_admm_sweep_$tag.log
