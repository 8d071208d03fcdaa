for v in g4l2 g4l3 g2l2 g2l4 g3l3 g4l2; do
  echo "== $v"
  PNP_B200_LIB=build/var_$v/libpnpb200.so python scripts/admm_prof.py 30 2>&1 | grep -E "^\[|fixup"
  PNP_B200_LIB=build/var_$v/libpnpb200.so python scripts/apply_sizes.py 256 512 1024 2>&1 | tail -3
done
