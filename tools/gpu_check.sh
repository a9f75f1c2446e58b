bash tools/gpu_ab.sh "--which gbmall,gbm --reps 10"
