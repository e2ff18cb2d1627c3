mkdir -p gpurun_out
python -c "import paper_1307_2895_b200._build as b; b.build()" > gpurun_out/r2k_build.log 2>&1
NCU=/usr/local/cuda/bin/ncu
O="--set full --import-source on --clock-control none"
timeout 600 $NCU $O -k regex:"skel_kernel" --launch-count 1 -o gpurun_out/r2k_skel python tools/one_step.py 3 > gpurun_out/r2k_1.log 2>&1
timeout 600 $NCU $O -k regex:"elim_small_kernel" --launch-count 1 -o gpurun_out/r2k_elim python tools/one_step.py 3 > gpurun_out/r2k_2.log 2>&1
timeout 600 $NCU $O -k regex:"solve_elim_fwd_mma" --launch-count 1 -o gpurun_out/r2k_fwd python tools/one_step.py 3 > gpurun_out/r2k_3.log 2>&1
timeout 600 $NCU $O -k regex:"solve_elim_bwd_mma" --launch-skip 8 --launch-count 1 -o gpurun_out/r2k_bwd python tools/one_step.py 3 > gpurun_out/r2k_4.log 2>&1
timeout 600 $NCU $O -k regex:"sym_front_kernel" --launch-skip 4 --launch-count 2 -o gpurun_out/r2k_sym python tools/one_step.py 3 > gpurun_out/r2k_5.log 2>&1
