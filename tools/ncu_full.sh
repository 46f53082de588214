# Full ncu capture of selected kernels of a short C3 meshing run:
#   bash tools/ncu_full.sh <kernel regex> <output name> [launch skip] [launch count] [views]
set -e
re="$1"; out="$2"; skip="${3:-0}"; cnt="${4:-3}"; views="${5:-8}"
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k "regex:$re" -s "$skip" -c "$cnt" \
    -o "gpurun_out/$out" -f python tools/profile_case.py --views "$views" --steps 1 > "gpurun_out/$out.log" 2>&1
