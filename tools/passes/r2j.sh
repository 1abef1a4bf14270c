# round-2 pass j: docs scorer with 256-row tiles; bandit MMA reload variant; ncu line profiles
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "maxsim or corpus or packed or bandit" > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2j_pytest.log
for c in cfg2 cfg3 cfg5; do
  for v in default oldpk; do
    if [ $v = default ]; then unset CBX_LIB CBX_TOOLS; else export CBX_TOOLS=1 CBX_LIB=build/var_$v/libcbx.so; fi
    CFG=$c timeout 300 python tools/ab_packed.py 2>/dev/null | tail -1
  done
done > gpurun_out/r2j_packed_ab.jsonl
unset CBX_LIB CBX_TOOLS
cat gpurun_out/r2j_packed_ab.jsonl
bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2j_p2.log 2>&1; grep -E "^==|iter 2" gpurun_out/r2j_p2.log | cut -c1-120
CFG=cfg2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:maxsim_docs_kernel -c 1 -o gpurun_out/r2j_docs_cfg2 -f python tools/ab_packed.py > gpurun_out/r2j_ncu_docs.log 2>&1; echo "ncu docs rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bandit_kernel -c 1 -o gpurun_out/r2j_bandit_cfg2 -f python tools/prof_p2.py --config cfg2 --iters 1 > gpurun_out/r2j_ncu_bandit.log 2>&1; echo "ncu bandit rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bandit_kernel -c 1 -o gpurun_out/r2j_bandit_cfg4 -f python tools/prof_p2.py --config cfg4 --iters 1 > gpurun_out/r2j_ncu_bandit4.log 2>&1; echo "ncu bandit cfg4 rc=$?"
