#!/bin/bash
mkdir -p gpurun_out
for spec in "skw:skel_warp_kernel:0" "skt64:skel_team_kernel<64:0" "skt256:skel_team_kernel<256:0"; do
  IFS=: read tag kre skip <<< "$spec"
  timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none \
    -k regex:"$kre" --launch-skip "$skip" --launch-count 1 -f -o gpurun_out/s4d_${tag} \
    python tools/one_step.py 3 > gpurun_out/s4d_${tag}.log 2>&1
done
