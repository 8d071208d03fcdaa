# ncu --set full of the 8192^2 adaptive denoise's tile fixups (RS, KXD)
mkdir -p gpurun_out/$1
cat > /tmp/one8k.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_1901_06110_b200 as pnp
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
x = torch.rand(8192, 8192, device="cuda")
pnp.dsg_nlm_denoise(x, p); torch.cuda.synchronize()
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dsg_fixup_tile_kernel -c 2 \
  -o gpurun_out/$1/fix8k python /tmp/one8k.py > gpurun_out/$1/ncu_fix8k.log 2>&1
tail -2 gpurun_out/$1/ncu_fix8k.log
