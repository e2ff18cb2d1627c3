mkdir -p gpurun_out
python -c "import paper_1307_2895_b200._build as b; b.build()" > gpurun_out/r2m_build.log 2>&1
NCU=/usr/local/cuda/bin/ncu
O="--set full --import-source on --clock-control none"
timeout 600 $NCU $O -k regex:"elim_small_kernel" --launch-count 1 -o gpurun_out/r2m_elim python tools/one_step.py 3 > gpurun_out/r2m_2.log 2>&1
timeout 600 $NCU $O -k regex:"solve_elim_fwd_mma" --launch-count 1 -o gpurun_out/r2m_fwd python tools/one_step.py 3 > gpurun_out/r2m_3.log 2>&1
