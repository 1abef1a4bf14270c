# round-2 pass t: row update with its loads batched up front
set -x
timeout 2400 python -m pytest tests/test_gpu_bandit.py tests/test_gpu_cfg4.py tests/test_gpu_sharded.py tests/test_gpu_eval.py tests/test_gpu_stage1.py tests/test_gpu_budget.py -x -q --timeout 900 > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2t_pytest.log
bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2t_p2.log 2>&1; grep -E "^==|iter 2" gpurun_out/r2t_p2.log | cut -c1-120
PHASES=1 bash tools/p2var.sh "default" "cfg4" > gpurun_out/r2t_p2_phases.log 2>&1; grep -E "cycles" gpurun_out/r2t_p2_phases.log | cut -c1-300
