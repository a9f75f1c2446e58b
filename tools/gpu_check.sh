# One-shot GPU check used during development.  Writes gpurun_out/.
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -80 > gpurun_out/r2_gputest.log
bash tools/gpu_ab.sh "--which gbmall,gbm --reps 10" > gpurun_out/r2_ab.log 2>&1
python tools/level_times.py > gpurun_out/r2_levels.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -5 gpurun_out/r2_gputest.log; cat gpurun_out/r2_ab.log gpurun_out/r2_levels.log
