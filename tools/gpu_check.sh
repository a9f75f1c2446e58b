ARV_LIB_PATH=tools/checked/libarv_b200_checked.so timeout 1500 python -m pytest tests/test_gpu_mlmc.py -q -p no:cacheprovider --tb=short 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gaussian_level -s 1 -c 1 \
  -o gpurun_out/r2_gbm_v5 python tools/prof_kernels.py --which gbm --reps 1 > gpurun_out/r2_ncu_gbm.log 2>&1
tail -1 gpurun_out/r2_ncu_gbm.log
