# One-shot GPU check used during development: GPU tests, smoke, bench lines.
# Writes gpurun_out/.
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -80 > gpurun_out/r2_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2>> gpurun_out/r2_bench.err
tail -5 gpurun_out/r2_gputest.log; cat gpurun_out/r2_smoke.log; tail -c 1500 gpurun_out/r2_bench.err
