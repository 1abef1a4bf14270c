# round-2 pass l: docs scorer with the accumulator-barrier fix; wide bandit shapes; full tests; bench; profiles (text only)
set -x
timeout 900 python -m pytest tests/test_gpu_maxsim.py -x -q --timeout 120 > gpurun_out/r2l_pytest_maxsim.log 2>&1; echo "pytest maxsim rc=$?"
tail -4 gpurun_out/r2l_pytest_maxsim.log
for c in cfg2 cfg3 cfg5; do
  for v in default oldpk; do
    if [ $v = default ]; then unset CBX_LIB CBX_TOOLS; else export CBX_TOOLS=1 CBX_LIB=build/var_$v/libcbx.so; fi
    CFG=$c timeout 200 python tools/ab_packed.py 2>/dev/null | tail -1
  done
done > gpurun_out/r2l_packed_ab.jsonl
unset CBX_LIB CBX_TOOLS
cat gpurun_out/r2l_packed_ab.jsonl
timeout 2000 python -m pytest tests -m gpu -x -q --timeout 600 --deselect tests/test_gpu_maxsim.py > gpurun_out/r2l_pytest_rest.log 2>&1; echo "pytest rest rc=$?"
tail -4 gpurun_out/r2l_pytest_rest.log
bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2l_p2.log 2>&1; grep -E "^==|iter 2" gpurun_out/r2l_p2.log | cut -c1-120
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo "bench rc=$?"
tail -16 gpurun_out/r2l_bench.err
CFG=cfg2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:maxsim_docs_kernel -c 1 -o /tmp/r2l_docs_cfg2 -f python tools/ab_packed.py > gpurun_out/r2l_ncu_docs.log 2>&1; echo "ncu docs rc=$?"
ncu -i /tmp/r2l_docs_cfg2.ncu-rep --page details > gpurun_out/r2l_ncu_docs_cfg2_details.txt 2>&1
ncu -i /tmp/r2l_docs_cfg2.ncu-rep --page source --csv > gpurun_out/r2l_ncu_docs_cfg2_sass.csv 2>&1
ncu -i /tmp/r2l_docs_cfg2.ncu-rep --page raw --csv > gpurun_out/r2l_ncu_docs_cfg2_raw.csv 2>&1
ls -la /tmp/r2l_docs_cfg2.ncu-rep gpurun_out/
