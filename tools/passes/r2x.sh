# round-2 final verification (K1 with 256-token tiles): everything the driver runs + table + launch list + traffic
set -x
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/r2x_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2x_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2x_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2x_smoke.log | cut -c1-300
timeout 900 python bench.py > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r2x_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2x_bench_ref.json 2> gpurun_out/r2x_bench_ref.err; echo "bench ref rc=$?"
timeout 1500 python tools/bench_all.py > gpurun_out/r2x_configs.jsonl 2> gpurun_out/r2x_configs.err; echo "bench_all rc=$?"; cut -c1-160 gpurun_out/r2x_configs.jsonl
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^(cbx::)?(bandit_kernel|gather_copy_kernel|gather_scan_kernel|maxsim_docs_kernel|maxsim_exact_kernel|maxsim_tc_kernel|plan_add_kernel|plan_blocks_kernel|plan_local_kernel|row_partial_fsum_kernel|stage1_.*|token_norm_max_kernel|topk_pass_kernel|warm_cells_kernel|warm_draw_kernel)" -c 500 --csv --log-file gpurun_out/r2x_launches.csv python bench.py --no-cpu > gpurun_out/r2x_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"maxsim_tc_kernel|maxsim_docs_kernel" -c 8 --csv --log-file gpurun_out/r2x_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-stage1 --no-p2-sharded --no-p1-sharded --no-drop-in --no-bandit > gpurun_out/r2x_ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
