#!/bin/bash
# ncu --set full of the DSG sweep kernels at 8192^2 (config 4): k-cache path
# (sweep A + store, sweep B cached) and recompute path; writes
# gpurun_out/sweeps_<tag>.ncu-rep.  Run only after the same command exited 0
# without ncu.
tag=${1:-r1}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dsg_sweep -c 2 \
  -o gpurun_out/sweeps_cache_$tag python scripts/prof_dsg.py 8192 > gpurun_out/ncu_cache_$tag.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dsg_sweep -c 2 \
  -o gpurun_out/sweeps_nocache_$tag python scripts/prof_dsg.py 8192 --nocache > gpurun_out/ncu_nocache_$tag.log 2>&1
tail -n 1 gpurun_out/ncu_cache_$tag.log; tail -n 1 gpurun_out/ncu_nocache_$tag.log
