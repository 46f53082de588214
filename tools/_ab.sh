# A/B timing on one box: tools/_ab.sh <variant>... (each run alternates). A variant is a
# library suffix ("" = the default build, "_prev" = libsof_cuda_prev.so) optionally
# followed by ":ENV=VAL" (e.g. "":SOF_NO_VORDER=1).
for rep in 1 2; do for spec in "$@"; do
  v="${spec%%:*}"; envs=""; [ "$spec" != "$v" ] && envs="${spec#*:}"
  echo "== variant '$spec' rep $rep"
  env $envs SOF_LIB_PATH=$PWD/paper_2506_19139_b200/libsof_cuda$v.so python tools/profile_case.py --views 200 --steps 2 --timed 2
done; done
