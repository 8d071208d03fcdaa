# tile-fixup launch-bounds variants: 8192^2 launch lists (development aid)
python scripts/prof_dsg.py 8192 > /dev/null 2>&1
for v in tlb1 tlb3 tlb4; do
  echo "== $v"
  PNP_B200_LIB=build/var_$v/libpnpb200.so bash scripts/launch_times.sh 8192 cache 2>&1 | grep -E "fixup|finalize"
done
