# round-2 pass y: ncu --set full of K1 (256-token tiles) on cfg2 and cfg3, K1d on cfg3; text exports only
set -x
for c in cfg2 cfg3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc_kernel -s 3 -c 1 -o /tmp/r2y_k1_$c -f python tools/prof_p1.py --config $c --iters 5 > gpurun_out/r2y_ncu_k1_$c.log 2>&1; echo "ncu k1 $c rc=$?"
  ncu -i /tmp/r2y_k1_$c.ncu-rep --page details > gpurun_out/r2y_ncu_k1_${c}_details.txt 2>&1
  ncu -i /tmp/r2y_k1_$c.ncu-rep --page raw --csv > gpurun_out/r2y_ncu_k1_${c}_raw.csv 2>&1
  python tools/ncu_lines.py /tmp/r2y_k1_$c.ncu-rep paper_2602_02827_b200/libcbx.so _ZN3cbx16maxsim_tc_kernelENS_7TmapSetENS_8TcParamsE 25 > gpurun_out/r2y_ncu_k1_${c}_lines.txt 2>&1
done
grep -E "Duration|DRAM Throughput|Memory Throughput|Issue Slots Busy|L2 Hit" gpurun_out/r2y_ncu_k1_cfg2_details.txt | head -8
head -12 gpurun_out/r2y_ncu_k1_cfg2_lines.txt | cut -c1-170
