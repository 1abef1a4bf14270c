# round-2 pass z: after splitting the 16-bit bandit units per layout — full GPU tests, smoke, bench
set -x
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/r2z_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2z_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2z_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2z_smoke.log | cut -c1-200
timeout 900 python bench.py > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r2z_bench.err; cut -c1-300 gpurun_out/r2z_bench.json
