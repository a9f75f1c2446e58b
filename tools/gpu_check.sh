timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -3
bash tools/gpu_ab.sh "--which gbmall,cirall --reps 10" 2>&1 | tail -40 | grep -E "==|all|l0|l6"
