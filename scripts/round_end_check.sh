cd $GRAFT_REPO_ROOT
set -u
mkdir -p gpurun_out/$1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$1/gpu_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/$1/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$1/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/$1/bench.json 2> gpurun_out/$1/bench.err; echo "bench rc $?" >> gpurun_out/$1/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$1/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/$1/ncu.log 2>&1; echo "ncu rc $?" >> gpurun_out/$1/ncu.log
tail -3 gpurun_out/$1/gpu_tests.log
