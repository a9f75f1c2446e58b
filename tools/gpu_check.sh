timeout 600 python -m pytest tests/test_gpu_headline.py -q -p no:cacheprovider --tb=short -k sample_host 2>&1 | tail -8
