# round-2 pass o: row-cache variant — parity tests, timing on/off on every config
set -x
timeout 1800 python -m pytest tests/test_gpu_bandit.py tests/test_gpu_cfg4.py -x -q --timeout 900 > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc=$?"
tail -12 gpurun_out/r2o_pytest.log | cut -c1-200
for c in cfg2 cfg3 cfg4 cfg5; do
  echo "== $c on-demand"; timeout 300 python tools/prof_p2.py --config $c --iters 3 2>&1 | grep "^iter 2" | cut -c1-260
  echo "== $c row-cache"; timeout 300 python tools/prof_p2.py --config $c --iters 3 --row-cache 2>&1 | grep "^iter 2" | cut -c1-300
done > gpurun_out/r2o_rowcache.log 2>&1
cat gpurun_out/r2o_rowcache.log
echo "== cfg2 row-cache phases"; timeout 300 python tools/prof_p2.py --config cfg2 --iters 2 --row-cache --phases 2>&1 | tail -1 | cut -c1-300
echo "== cfg4 row-cache phases"; timeout 300 python tools/prof_p2.py --config cfg4 --iters 2 --row-cache --phases 2>&1 | tail -1 | cut -c1-300
