# round-2 pass u: tree leaf loads batched; line-level ncu profile of the cfg4 run (mapped on the box: same library)
set -x
timeout 2400 python -m pytest tests/test_gpu_bandit.py tests/test_gpu_cfg4.py tests/test_gpu_sharded.py tests/test_gpu_stage1.py -x -q --timeout 900 > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2u_pytest.log
bash tools/p2var.sh "default" "cfg2 cfg3 cfg4 cfg5" > gpurun_out/r2u_p2.log 2>&1; grep -E "^==|iter 2" gpurun_out/r2u_p2.log | cut -c1-120
PHASES=1 bash tools/p2var.sh "default" "cfg4" > gpurun_out/r2u_p2_phases.log 2>&1; grep -E "cycles" gpurun_out/r2u_p2_phases.log | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bandit_kernel -c 1 -o /tmp/r2u_bandit_cfg4 -f python tools/prof_p2.py --config cfg4 --iters 1 > gpurun_out/r2u_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/r2u_bandit_cfg4.ncu-rep --page details > gpurun_out/r2u_ncu_bandit_cfg4_details.txt 2>&1
python tools/ncu_lines.py /tmp/r2u_bandit_cfg4.ncu-rep paper_2602_02827_b200/libcbx.so _ZN3cbx13bandit_kernelI6__halfLi16ELi1ELi512ELb1ELi1ELb1ELb0EEEvNS_12BanditParamsE 60 > gpurun_out/r2u_ncu_bandit_cfg4_lines.txt 2>&1; head -40 gpurun_out/r2u_ncu_bandit_cfg4_lines.txt | cut -c1-200
OUTER=1 python tools/ncu_lines.py /tmp/r2u_bandit_cfg4.ncu-rep paper_2602_02827_b200/libcbx.so _ZN3cbx13bandit_kernelI6__halfLi16ELi1ELi512ELb1ELi1ELb1ELb0EEEvNS_12BanditParamsE 40 > gpurun_out/r2u_ncu_bandit_cfg4_lines_outer.txt 2>&1
