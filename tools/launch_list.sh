#!/bin/bash
# ncu launch list (per-kernel GPU time, serialized, cold) of one factor + solve of a config
tag=$1; cfg=${2:-3}
mkdir -p gpurun_out
python -c "import paper_1307_2895_b200._build as b; b.build()" > gpurun_out/${tag}_build.log 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}.csv python tools/one_step.py "$cfg" > gpurun_out/${tag}.log 2>&1
