# round-2 pass h: MMA reveal screen + document-tile packed scorer: parity, A/B timing, sanitizer
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2h_pytest.log
for c in cfg2 cfg3 cfg5; do
  for v in default oldpk; do
    if [ $v = default ]; then unset CBX_LIB CBX_TOOLS; else export CBX_TOOLS=1 CBX_LIB=build/var_$v/libcbx.so; fi
    CFG=$c timeout 300 python tools/ab_packed.py 2>&1 | tail -1
  done
done > gpurun_out/r2h_packed_ab.jsonl 2>&1
unset CBX_LIB CBX_TOOLS
cat gpurun_out/r2h_packed_ab.jsonl
bash tools/p2var.sh "default nomma" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2h_p2_ab.log 2>&1; grep -E "^==|kernel" gpurun_out/r2h_p2_ab.log | cut -c1-220
PHASES=1 bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2h_p2_phases.log 2>&1; grep -E "^==|cycles" gpurun_out/r2h_p2_phases.log | cut -c1-300
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize.py > gpurun_out/r2h_sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/r2h_sanitize_$tool.log
done
