timeout 600 python -m pytest tests/test_gpu_graph.py -q -p no:cacheprovider --tb=short 2>&1 | tail -15
python tools/host_paths.py graph
