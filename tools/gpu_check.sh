python tools/host_paths.py > gpurun_out/r2_host_paths.log 2>&1; head -12 gpurun_out/r2_host_paths.log
