# Round-2 measurements (run under gpurun, one GPU): bench lines (C3 headline with render,
# CPU baseline and parity; the reference arm; C1; C4), a C3 launch list with DRAM bytes
# (40 of the 200 views), full ncu captures of the K4 label / grouped-bisection launches and
# of the K5 render kernels, and a C2 render launch list.
set -x
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_c3_reference_arm.json 2> gpurun_out/r2_ref.err
timeout 900 python bench.py --config C1 --no-render > gpurun_out/r2_bench_c1.json 2> gpurun_out/r2_c1.err
timeout 1800 python bench.py --config C4 --no-render --no-cpu-baseline > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r2_launches_c3_40views.csv python tools/profile_case.py --views 40 --steps 1 \
    > gpurun_out/r2_launches_run.log 2>&1
timeout 600 bash tools/ncu_full.sh "^k_eval$" r2_k_eval_label_c3 20 1 40
timeout 600 bash tools/ncu_full.sh "k_eval_group" r2_k_eval_group_c3 2 1 40
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r2_launches_render_c2.csv python tools/render_diag.py > gpurun_out/r2_render_diag_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_rcount|k_rtest|k_rsort|k_rblend" -c 5 \
    -o gpurun_out/r2_k_render_c2 -f python tools/profile_case.py --config C2 --views 1 --steps 1 --render \
    > gpurun_out/r2_k_render_c2.log 2>&1
ls -la gpurun_out | tail -30
