#!/bin/bash
# usage: tools/gpu_job.sh <tag> <what...>   (run on the GPU box via gpurun)
tag=$1; shift
mkdir -p gpurun_out
python -c "import paper_1307_2895_b200._build as b; b.build()" > gpurun_out/${tag}_build.log 2>&1
for w in "$@"; do
  case $w in
    tests) timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/${tag}_tests.log 2>&1 ;;
    testsx) timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/${tag}_tests.log 2>&1 ;;
    bench) timeout 900 python bench.py --steps 5 --warmup 2 > gpurun_out/${tag}_bench.log 2>&1 ;;
    benchq) timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-extra > gpurun_out/${tag}_bench.log 2>&1 ;;
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1 ;;
    *) eval "$w" ;;
  esac
done
