set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2f_pytest.log
bash tools/p2var.sh "default notw" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2f_ab.log 2>&1
PHASES=1 bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2f_phases.log 2>&1
timeout 300 python tools/prof_p2_host.py > gpurun_out/r2f_host.log 2>&1; head -5 gpurun_out/r2f_host.log
