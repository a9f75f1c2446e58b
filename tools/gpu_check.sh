# GPU test suite against the checked library (device-side asserts, ARV_CHECKS=1).
set -x
ARV_LIB_PATH=tools/checked/libarv_b200_checked.so timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short \
  > gpurun_out/r2_checked_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_checked_tests.log
ARV_LIB_PATH=tools/checked/libarv_b200_checked.so timeout 900 python tools/sanitize.py --big >> gpurun_out/r2_checked_tests.log 2>&1; echo "workload rc=$?" >> gpurun_out/r2_checked_tests.log
tail -8 gpurun_out/r2_checked_tests.log
