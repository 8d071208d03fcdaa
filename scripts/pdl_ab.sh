# PDL on/off A/B of the ADMM loop, frozen applies and the bench (development aid)
for pdl in 1 0 1; do
  echo "== PNP_PDL=$pdl"
  PNP_PDL=$pdl python scripts/admm_prof.py 30 2>&1 | grep -E "^\["
  PNP_PDL=$pdl python scripts/apply_sizes.py 256 512 1024 2048 2>&1 | tail -4
  PNP_PDL=$pdl python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); a=d['admm']
        print('bench', round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1),
              'c1', round(a['config1_denoise_256']['ms_per_denoise'],4),
              'c2', round(a['config2_sr_512']['iters_per_s']), round(a['config2_sr_512']['device_ms'],3),
              'c3', round(a['config3_qis_512']['iters_per_s']),
              'c5', round(a['config5_sr_64x1024']['image_iters_per_s']))"
done
