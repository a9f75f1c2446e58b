set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -40 > gpurun_out/r2_gputest.log
python tools/prof_kernels.py --which gbmall,gbm,cirall --reps 10 > gpurun_out/r2_prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gaussian_level -s 1 -c 1 \
  -o gpurun_out/r2_gbm_v3 python tools/prof_kernels.py --which gbm --reps 1 > gpurun_out/r2_ncu_gbm.log 2>&1
tail -3 gpurun_out/r2_gputest.log; cat gpurun_out/r2_prof.log
