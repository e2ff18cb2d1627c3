tools/ncu_capture.sh r3c_skel "skel_kernel" 0 3
tools/ncu_capture.sh r3c_symc "sym_front_kernel" 2 3
