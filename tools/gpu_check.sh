bash tools/gpu_ab.sh "--which gbmall,gbm --reps 10" 2>&1 | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg32_linsigned -s 2 -c 1 \
  -o gpurun_out/r2_headline python tools/prof_kernels.py --which sub --reps 3 > gpurun_out/r2_ncu_head.log 2>&1
tail -2 gpurun_out/r2_ncu_head.log
