set -x
timeout 900 python -m pytest tests/test_gpu_bandit.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2e_pytest.log
bash tools/p2var.sh "default nopf notw pf2" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2e_ab.log 2>&1
PHASES=1 bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2e_phases.log 2>&1
timeout 300 python tools/prof_p2_host.py > gpurun_out/r2e_host.log 2>&1; head -8 gpurun_out/r2e_host.log
