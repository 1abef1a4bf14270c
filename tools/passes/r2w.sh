# round-2 pass w: K1 with 256-token tiles — parity (GPU tests), bit-equality and timing A/B against 128-token tiles
set -x
timeout 1500 python -m pytest tests/test_gpu_maxsim.py tests/test_gpu_cfg4.py tests/test_gpu_bandit.py -x -q --timeout 600 > gpurun_out/r2w_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2w_pytest.log
for c in cfg2 cfg3 cfg4 cfg1; do
  for v in default tile128; do
    if [ $v = default ]; then unset CBX_LIB CBX_TOOLS; else export CBX_TOOLS=1 CBX_LIB=build/var_$v/libcbx.so; fi
    echo "== $c $v"; timeout 200 python tools/prof_p1.py --config $c --iters 6 2>&1 | tail -3
  done
done > gpurun_out/r2w_p1_ab.log 2>&1
unset CBX_LIB CBX_TOOLS
cat gpurun_out/r2w_p1_ab.log
CFG=cfg2 timeout 200 python tools/ab_packed.py 2>/dev/null | tail -1
CFG=cfg3 timeout 200 python tools/ab_packed.py 2>/dev/null | tail -1
timeout 900 python bench.py --no-p2-sharded --no-stage1 --no-drop-in > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err; echo "bench rc=$?"; cut -c1-330 gpurun_out/r2w_bench.json
