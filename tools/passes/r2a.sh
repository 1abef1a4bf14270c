set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2a_pytest.log
for c in cfg4 cfg2 cfg5 cfg3; do timeout 300 python tools/prof_p2.py --config $c --phases > gpurun_out/r2a_prof_$c.log 2>&1; echo "$c rc=$?"; cat gpurun_out/r2a_prof_$c.log | tail -4; done
