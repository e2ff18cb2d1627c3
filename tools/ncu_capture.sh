#!/bin/bash
# ncu --set full capture of one kernel of a BASELINE config's factor + solve
# (tools/one_step.py), run on the GPU box:
#   tools/ncu_capture.sh TAG KERNEL_REGEX [LAUNCH_SKIP] [CONFIG]
tag=$1; kre=$2; skip=${3:-0}; cfg=${4:-3}
mkdir -p gpurun_out
python -c "import paper_1307_2895_b200._build as b; b.build()" > gpurun_out/${tag}_build.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none \
  -k regex:"$kre" --launch-skip "$skip" --launch-count 1 -o gpurun_out/${tag} \
  python tools/one_step.py "$cfg" > gpurun_out/${tag}.log 2>&1
