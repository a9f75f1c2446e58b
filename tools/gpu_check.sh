timeout 600 python -m pytest tests/test_gpu_host.py -q -p no:cacheprovider --tb=short 2>&1 | tail -5
