# round-2 pass n: offsets in shared memory, wide shape for big pools (cfg5), expansion tests, all-config table
set -x
timeout 1500 python -m pytest tests/test_gpu_bandit.py tests/test_gpu_cfg4.py tests/test_gpu_sharded.py tests/test_gpu_eval.py tests/test_gpu_stage1.py -x -q --timeout 600 > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc=$?"
tail -6 gpurun_out/r2n_pytest.log
bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2n_p2.log 2>&1; grep -E "^==|iter 2" gpurun_out/r2n_p2.log | cut -c1-120
PHASES=1 bash tools/p2var.sh "default" "cfg2 cfg5" > gpurun_out/r2n_p2_phases.log 2>&1; grep -E "^==|cycles" gpurun_out/r2n_p2_phases.log | cut -c1-300
timeout 1500 python tools/bench_all.py > gpurun_out/r2n_configs.jsonl 2> gpurun_out/r2n_configs.err; echo "bench_all rc=$?"; tail -3 gpurun_out/r2n_configs.err; cut -c1-200 gpurun_out/r2n_configs.jsonl
