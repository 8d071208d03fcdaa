# ncu --set full of one config-5 iteration's kernels (64 x 1024^2, frozen guides):
# cached apply sweep, apply fixup + u/x-update, SR residual, SR adjoint
mkdir -p gpurun_out/$1
python scripts/cfg5_repeat.py 64 1 > gpurun_out/$1/plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"dsg_sweep_kernel|dsg_fixup_tile_kernel|sr_residual_kernel|sr_adjoint_kernel" \
  --launch-skip 140 -c 5 -o gpurun_out/$1/cfg5 python scripts/cfg5_repeat.py 64 1 > gpurun_out/$1/ncu.log 2>&1
tail -3 gpurun_out/$1/ncu.log
