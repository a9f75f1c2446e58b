timeout 600 python -m pytest tests/test_gpu_mlmc.py -q -p no:cacheprovider --tb=short -k beyond 2>&1 | tail -5
