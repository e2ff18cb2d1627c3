set -x
mkdir -p gpurun_out
python -c "import paper_1307_2895_b200._build as b; b.build()" > gpurun_out/r2i_build.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:"elim_small_kernel|solve_elim_fwd_mma" --launch-count 2 -o gpurun_out/r2i_a python tools/one_step.py 3 > gpurun_out/r2i_ncu_a.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:"solve_elim_bwd_mma" --launch-skip 8 --launch-count 1 -o gpurun_out/r2i_b python tools/one_step.py 3 > gpurun_out/r2i_ncu_b.log 2>&1
