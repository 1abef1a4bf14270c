# round-2 verification pass: everything the driver runs at round end + the all-config table
set -x
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/r2v_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2v_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2v_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2v_smoke.log | cut -c1-300
timeout 900 python bench.py > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r2v_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2v_bench_ref.json 2> gpurun_out/r2v_bench_ref.err; echo "bench ref rc=$?"
timeout 1500 python tools/bench_all.py > gpurun_out/r2v_configs.jsonl 2> gpurun_out/r2v_configs.err; echo "bench_all rc=$?"; cut -c1-160 gpurun_out/r2v_configs.jsonl
