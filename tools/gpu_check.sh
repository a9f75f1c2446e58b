timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -6
python tools/prof_kernels.py --which gbmall,gbm --reps 10
