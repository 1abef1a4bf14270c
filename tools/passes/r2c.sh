set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "cfg4 or pcg64 or guard or wide or config_query or sync" > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2c_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-stage1 --no-p2-sharded --no-p1-sharded --no-e2e > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "bench rc=$?"
