# ncu captures for profiles/ (run on the GPU box through gpurun, one GPU; each only after
# the same command has exited 0 without ncu).  Reports land in gpurun_out/<tag>_*.ncu-rep;
# tools/ncu_refresh.py turns them into profiles/ncu_summary.json + briefs.
#   bash tools/ncu_capture.sh <tag>
TAG=${1:-cap}
FP64=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
set -x
python tools/prof_kernels.py --which sub,const,gbm,cir --reps 2 > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:linlane -c 1 -s 2 \
  -o gpurun_out/${TAG}_headline -f python tools/prof_kernels.py --which sub --reps 2 > gpurun_out/${TAG}_ncu_headline.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg32_constant -c 1 -s 2 \
  -o gpurun_out/${TAG}_const -f python tools/prof_kernels.py --which const --reps 2 > gpurun_out/${TAG}_ncu_const.log 2>&1
timeout 600 ncu --set full --metrics $FP64 --clock-control none --import-source on -k regex:k_gaussian_level -c 1 -s 1 \
  -o gpurun_out/${TAG}_gbm -f python tools/prof_kernels.py --which gbm --reps 1 > gpurun_out/${TAG}_ncu_gbm.log 2>&1
# a CIR exact level is a sequence of segment kernels: FP64 counts and durations of all of one level (reps 1: warm-up + 1)
timeout 900 ncu --metrics gpu__time_duration.sum,$FP64,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio \
  --clock-control none -k regex:k_cir --csv --log-file gpurun_out/${TAG}_cir_counts.csv \
  python tools/prof_kernels.py --which cir --reps 1 > gpurun_out/${TAG}_ncu_cir.log 2>&1
