# Round profiles (run under gpurun): a per-launch timing list of one C3 meshing step
# (40 of the 200 views) and full captures of the label and bisection K4 launches.
set -x
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_c3_40v.csv python tools/profile_case.py --views 40 --steps 1 \
    > gpurun_out/launches_run.log 2>&1
timeout 600 bash tools/ncu_full.sh "^k_eval$" k_eval_label_c3 20 1 40
timeout 600 bash tools/ncu_full.sh "k_eval_group" k_eval_group_c3 2 1 40
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_render" -c 4 -o gpurun_out/k_render_c2 -f \
    python tools/profile_case.py --config C2 --views 1 --steps 1 --render > gpurun_out/k_render_c2.log 2>&1
