timeout 900 python -m pytest tests/test_gpu_mlmc.py tests/test_gpu_dist.py tests/test_gpu_experiment.py -q -p no:cacheprovider --tb=short 2>&1 | tail -3
python tools/host_paths.py suites 2>&1 | head -3
timeout 600 python bench.py --no-cpu --no-plugin --no-sustained --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:v['seconds'] for k,v in d['mlmc'].items()})"
