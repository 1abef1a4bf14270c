# round-2 pass p: row-cache variant as its own instantiations; fill threshold 2 vs first touch
set -x
timeout 2400 python -m pytest tests/test_gpu_bandit.py tests/test_gpu_cfg4.py -x -q --timeout 900 > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/r2p_pytest.log | cut -c1-200
for c in cfg2 cfg3 cfg4 cfg5; do
  echo "== $c on-demand"; timeout 300 python tools/prof_p2.py --config $c --iters 3 2>&1 | grep "^iter 2" | cut -c1-110
  echo "== $c row-cache (fill at 2 revealed)"; timeout 300 python tools/prof_p2.py --config $c --iters 3 --row-cache 2 2>&1 | grep "^iter 2" | sed 's/reveals.*aggregate//' | cut -c1-200
  echo "== $c row-cache (fill at first touch)"; timeout 300 python tools/prof_p2.py --config $c --iters 3 --row-cache 0 2>&1 | grep "^iter 2" | sed 's/reveals.*aggregate//' | cut -c1-200
done > gpurun_out/r2p_rowcache.log 2>&1
cat gpurun_out/r2p_rowcache.log
