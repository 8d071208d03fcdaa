# ncu --set full of the SR residual / adjoint kernels inside a config-5 solve
mkdir -p gpurun_out/$1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sr_adjoint_kernel --launch-skip 5 -c 1 \
  -o gpurun_out/$1/sr_adj python scripts/cfg5_repeat.py 64 1 > gpurun_out/$1/ncu_adj.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sr_residual_kernel --launch-skip 70 -c 1 \
  -o gpurun_out/$1/sr_res python scripts/cfg5_repeat.py 64 1 > gpurun_out/$1/ncu_res.log 2>&1
if [ "$2" = fix ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dsg_fixup_tile_kernel --launch-skip 5 -c 1 \
  -o gpurun_out/$1/fix5 python scripts/cfg5_repeat.py 64 1 > gpurun_out/$1/ncu_fix.log 2>&1
fi
ls gpurun_out/$1
