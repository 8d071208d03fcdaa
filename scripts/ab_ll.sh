# same-box A/B of the 8192^2 launch list between library builds
for lib in "$@"; do
  echo "== $lib"
  PNP_B200_LIB=$lib bash scripts/launch_times.sh 8192 cache 2>&1 | sed -n 2,13p
done
