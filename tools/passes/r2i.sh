# round-2 pass i: byte-ring doc-tile scorer + reordered MMA screen; fixed bench
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2i_pytest.log
for c in cfg2 cfg3 cfg5; do
  for v in default oldpk; do
    if [ $v = default ]; then unset CBX_LIB CBX_TOOLS; else export CBX_TOOLS=1 CBX_LIB=build/var_$v/libcbx.so; fi
    CFG=$c timeout 300 python tools/ab_packed.py 2>/dev/null | tail -1
  done
done > gpurun_out/r2i_packed_ab.jsonl
unset CBX_LIB CBX_TOOLS
cat gpurun_out/r2i_packed_ab.jsonl
bash tools/p2var.sh "default nomma" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2i_p2_ab.log 2>&1; grep -E "^==|iter 2" gpurun_out/r2i_p2_ab.log | cut -c1-120
PHASES=1 bash tools/p2var.sh "default" "cfg2 cfg4" > gpurun_out/r2i_p2_phases.log 2>&1; grep -E "^==|cycles" gpurun_out/r2i_p2_phases.log | cut -c1-300
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo "bench rc=$?"
cat gpurun_out/r2i_bench.err | tail -30; cut -c1-400 gpurun_out/r2i_bench.json
CFG=cfg2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:maxsim_docs_kernel -c 1 -o gpurun_out/r2i_docs_cfg2 -f python tools/ab_packed.py > gpurun_out/r2i_ncu_docs.log 2>&1; echo "ncu docs rc=$?"
