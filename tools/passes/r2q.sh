# round-2 final pass: full GPU tests, smoke, bench (ours + reference arm), launch list, traffic captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/r2q_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2q_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2q_smoke.log | cut -c1-300
timeout 900 python bench.py > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err; echo "bench rc=$?"
tail -4 gpurun_out/r2q_bench.err; cut -c1-300 gpurun_out/r2q_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2q_bench_ref.json 2> gpurun_out/r2q_bench_ref.err; echo "bench ref rc=$?"; cut -c1-400 gpurun_out/r2q_bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2q_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-stage1 --no-p2-sharded --no-p1-sharded --no-drop-in > gpurun_out/r2q_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"maxsim_tc_kernel|maxsim_docs_kernel|bandit_kernel" -c 12 --csv --log-file gpurun_out/r2q_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-stage1 --no-p2-sharded --no-p1-sharded --no-drop-in > gpurun_out/r2q_ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
ls -la gpurun_out | head -20
