# round-2 pass r: smoke with the resident-corpus scorer, device-side trace compaction, launch list of the repo's kernels in bench.py
set -x
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2r_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2r_smoke.log | cut -c1-300
timeout 1500 python -m pytest tests/test_gpu_bandit.py tests/test_gpu_eval.py tests/test_gpu_budget.py -x -q --timeout 900 > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2r_pytest.log
timeout 900 python bench.py > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/r2r_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|topk|bandit|plan_|stage1|warm_cells|gather|budget|norm" -c 400 --csv --log-file gpurun_out/r2r_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2r_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
