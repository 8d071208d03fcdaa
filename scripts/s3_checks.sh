# session-3 hygiene check: debug-build comparison + forward/ADMM/checks GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/$1
timeout 900 bash scripts/checks_compare.sh > gpurun_out/$1/checks.log 2>&1; echo "checks rc $?" >> gpurun_out/$1/checks.log
timeout 600 python -m pytest tests/test_forward_gpu.py tests/test_admm_gpu.py tests/test_checks_gpu.py -q > gpurun_out/$1/tests.log 2>&1; tail -2 gpurun_out/$1/tests.log
tail -4 gpurun_out/$1/checks.log
