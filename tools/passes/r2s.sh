# round-2 pass s: launch list of the repo's kernels inside bench.py (same command as the bench line)
set -x
timeout 900 python bench.py > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r2s_bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^(cbx::)?(bandit_kernel|gather_copy_kernel|gather_scan_kernel|maxsim_docs_kernel|maxsim_exact_kernel|maxsim_tc_kernel|plan_add_kernel|plan_blocks_kernel|plan_local_kernel|row_partial_fsum_kernel|stage1_.*|token_norm_max_kernel|topk_pass_kernel|warm_cells_kernel|warm_draw_kernel)" -c 500 --csv --log-file gpurun_out/r2s_launches.csv python bench.py --no-cpu > gpurun_out/r2s_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
wc -l gpurun_out/r2s_launches.csv
