# round-2 evidence pass: GPU tests, smoke, bench, launch list, P2 per-config times, ncu capture of the bandit kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2g_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2g_smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2g_bench.err; cut -c1-600 gpurun_out/r2g_bench.json
bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2g_p2.log 2>&1; grep -E "^==|kernel" gpurun_out/r2g_p2.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-stage1 --no-p2-sharded --no-p1-sharded --no-drop-in --no-p2-host-stepped > gpurun_out/r2g_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bandit_kernel -c 1 -o gpurun_out/r2g_bandit_cfg2 -f python tools/prof_p2.py --config cfg2 --iters 1 > gpurun_out/r2g_ncu_bandit.log 2>&1; echo "ncu bandit rc=$?"
