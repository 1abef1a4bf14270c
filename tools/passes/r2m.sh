# round-2 pass m: row-state prefetch (cfg4), expansion-path tests, host-side profile of run_batch
set -x
timeout 1500 python -m pytest tests/test_gpu_bandit.py tests/test_gpu_cfg4.py tests/test_gpu_sharded.py -x -q --timeout 600 > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc=$?"
tail -6 gpurun_out/r2m_pytest.log
bash tools/p2var.sh "default" "cfg4 cfg3 cfg2" > gpurun_out/r2m_p2.log 2>&1; grep -E "^==|iter 2" gpurun_out/r2m_p2.log | cut -c1-120
PHASES=1 bash tools/p2var.sh "default" "cfg4" > gpurun_out/r2m_p2_phases.log 2>&1; grep -E "^==|cycles" gpurun_out/r2m_p2_phases.log | cut -c1-300
timeout 300 python tools/prof_p2_host.py > gpurun_out/r2m_host.log 2>&1; head -40 gpurun_out/r2m_host.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bandit_kernel -c 1 -o /tmp/r2m_bandit_cfg4 -f python tools/prof_p2.py --config cfg4 --iters 1 > gpurun_out/r2m_ncu_bandit4.log 2>&1; echo "ncu bandit cfg4 rc=$?"
ncu -i /tmp/r2m_bandit_cfg4.ncu-rep --page details > gpurun_out/r2m_ncu_bandit_cfg4_details.txt 2>&1
ncu -i /tmp/r2m_bandit_cfg4.ncu-rep --page source --csv --print-source sass > gpurun_out/r2m_ncu_bandit_cfg4_sass.csv 2>&1
ls -la gpurun_out/ | head -20
