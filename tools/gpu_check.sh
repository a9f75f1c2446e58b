bash tools/gpu_ab.sh "--which gbmall,gbm --reps 10" 2>&1 | tail -12
