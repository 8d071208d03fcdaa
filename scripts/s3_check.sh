# session-3 GPU check: gpu tests + config-5 launch summary (+ optional bench)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/$1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/$1/gpu_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/$1/gpu_tests.log
tail -3 gpurun_out/$1/gpu_tests.log
bash scripts/cfg5_launches.sh > gpurun_out/$1/cfg5_summary.txt 2>&1; head -8 gpurun_out/$1/cfg5_summary.txt
if [ "$2" = bench ]; then timeout 600 python bench.py > gpurun_out/$1/bench.json 2> gpurun_out/$1/bench.err; tail -2 gpurun_out/$1/bench.err; fi
