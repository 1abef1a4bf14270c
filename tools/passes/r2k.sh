# round-2 pass k: find the docs-scorer failure on ragged documents; wide bandit variant
set -x
timeout 900 python -m pytest tests/test_gpu_maxsim.py -x -q --timeout 120 -k "corpus or packed or resident" > gpurun_out/r2k_pytest_packed.log 2>&1; echo "pytest packed rc=$?"
tail -25 gpurun_out/r2k_pytest_packed.log
CFG=cfg2 timeout 200 python tools/ab_packed.py > gpurun_out/r2k_ab_cfg2.log 2>&1; echo "ab cfg2 rc=$?"; tail -5 gpurun_out/r2k_ab_cfg2.log
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 -k "bandit or cfg4 or sharded or stage1 or eval or budget" > gpurun_out/r2k_pytest_bandit.log 2>&1; echo "pytest bandit rc=$?"
tail -5 gpurun_out/r2k_pytest_bandit.log
bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2k_p2.log 2>&1; grep -E "^==|iter 2" gpurun_out/r2k_p2.log | cut -c1-120
PHASES=1 bash tools/p2var.sh "default" "cfg3 cfg4" > gpurun_out/r2k_p2_phases.log 2>&1; grep -E "^==|cycles" gpurun_out/r2k_p2_phases.log | cut -c1-300
