set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "mailbox or cfg4" > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2d_pytest.log
timeout 300 python tools/prof_p2_host.py > gpurun_out/r2d_host.log 2>&1; echo "prof rc=$?"
head -60 gpurun_out/r2d_host.log
