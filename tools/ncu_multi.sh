#!/bin/bash
# ncu --set full captures of several kernels of one config-3 factor + solve:
#   [CFG=5] tools/ncu_multi.sh TAG "name:regex[:skip]" ...
tag=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; rest=${spec#*:}; kre=${rest%%:*}; skip=0
  [ "$rest" != "$kre" ] && skip=${rest#*:}
  timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none \
    -k "regex:$kre" --launch-skip "$skip" --launch-count 1 -f -o "gpurun_out/${tag}_${name}" \
    python tools/one_step.py "${CFG:-3}" > "gpurun_out/${tag}_${name}.log" 2>&1
done
