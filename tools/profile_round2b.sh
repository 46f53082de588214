# Round-2 final pass after the render sort rework (run under gpurun, one GPU): the GPU
# suite, the C3 headline bench line (with the C2 render sample), the reference arm, the
# C2 render launch list with DRAM bytes and a full capture of k_rsort_mid / k_rblend.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/r2b_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2b_pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_c3_reference_arm.json 2> gpurun_out/r2_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r2_launches_render_c2.csv python tools/render_diag.py > gpurun_out/r2_render_diag_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^k_r(sort_mid|blend)$" -c 2 \
    -o gpurun_out/r2_k_rmid_rblend_c2 -f python tools/render_diag.py > gpurun_out/r2_k_rmid_rblend_c2.log 2>&1
cat gpurun_out/r2_bench_c3.json gpurun_out/r2_bench_c3_reference_arm.json
