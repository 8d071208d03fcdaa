#!/bin/bash
# A/B of the DSG kernels: product library vs build/var_$1 (quick_perf, 8192^2, alternating)
for i in 1 2; do
  echo "== product"; python scripts/quick_perf.py 8192
  echo "== $1"; PNP_B200_LIB=build/var_$1/libpnpb200.so python scripts/quick_perf.py 8192
done
