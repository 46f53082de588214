#!/bin/bash
# usage: gpu_render_cycle.sh TAG  (runs on the GPU box)
T=$1
timeout 900 python -m pytest tests/test_render_gpu.py tests/test_configs_gpu.py -q -rf --timeout 300 > gpurun_out/pytest_$T.log 2>&1; echo rc=$? >> gpurun_out/pytest_$T.log
timeout 300 python tools/render_diag.py > gpurun_out/render_diag_$T.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_render_$T.csv python tools/render_diag.py > gpurun_out/ncu_$T.log 2>&1
tail -3 gpurun_out/pytest_$T.log; cat gpurun_out/render_diag_$T.log; python tools/launch_summary.py gpurun_out/launches_render_$T.csv | head -8
