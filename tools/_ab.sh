# A/B timing on one box: tools/_ab.sh <variant suffix>... (each run alternates)
for rep in 1 2; do for v in "$@"; do
  echo "== variant '$v' rep $rep"
  SOF_LIB_PATH=$PWD/paper_2506_19139_b200/libsof_cuda$v.so python tools/profile_case.py --views 200 --steps 2
done; done
