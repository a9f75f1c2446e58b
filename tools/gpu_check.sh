set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -30 > gpurun_out/r2_gputest.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 900 python bench.py --workload config1 --no-mlmc --no-cpu --no-plugin > gpurun_out/r2_bench_c1.json 2>> gpurun_out/r2_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2>> gpurun_out/r2_bench.err
python tools/sweep_config3.py > gpurun_out/r2_sweep3.jsonl 2> gpurun_out/r2_sweep3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-mlmc --no-cpu --no-sustained --no-plugin > gpurun_out/r2_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg32_linsigned -s 5 -c 1 \
  -o gpurun_out/r2_headline python tools/prof_kernels.py --which sub --reps 3 > gpurun_out/r2_ncu_head.log 2>&1
tail -3 gpurun_out/r2_gputest.log; tail -3 gpurun_out/r2_bench.err; tail -2 gpurun_out/r2_sweep3.jsonl | cut -c1-600
