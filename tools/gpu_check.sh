timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gaussian_level -s 2 -c 1 \
  -o gpurun_out/r2_gbm_l0 python tools/prof_kernels.py --which gbml01 --reps 1 > gpurun_out/r2_ncu_l0.log 2>&1
tail -1 gpurun_out/r2_ncu_l0.log
