# ncu launch list of adaptive denoises at 512^2 (config-3 shape: R10 P7 Gaussian) after warm-up
mkdir -p gpurun_out/$1
cat > /tmp/ad512.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_1901_06110_b200 as pnp
p = pnp.PatchParams.from_h(7, 10, 10 / 255, 2.0)
x = torch.rand(512, 512, device="cuda")
for _ in range(8): pnp.dsg_nlm_denoise(x, p)
torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none --cache-control none --csv -s 20 python /tmp/ad512.py > gpurun_out/$1/ad512.csv 2>&1
grep -E '^"[0-9]' gpurun_out/$1/ad512.csv | python3 -c "
import sys,csv
rows=list(csv.reader(sys.stdin))
for r in rows[:60]: print(r[0], r[4][:55], r[12][:30], r[14])
"
