for m in "irls fp32" "l1 fp64" "irls fp64"; do
  set -- $m
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:point_pass_hot -s 3 -c 1 -o gpurun_out/prof_$1_$2 python tools/one_pass.py $1 $2 > /dev/null 2>&1
done
ls gpurun_out
