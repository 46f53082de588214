# A/B of render variants: tools/_ab_render.sh <suffix>...
for rep in 1 2; do for v in "$@"; do
  echo "== variant '$v' rep $rep"
  SOF_LIB_PATH=$PWD/paper_2506_19139_b200/libsof_cuda$v.so python tools/profile_case.py --config C2 --views 3 --steps 3 --render
done; done
