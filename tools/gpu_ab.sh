# A/B timing of library variants (tools/ab/*.so, built with _build.build(defines=..., out=...))
# against the in-tree library.  Usage: bash tools/gpu_ab.sh "<prof_kernels args>"
ARGS=${1:-"--which gbmall,gbm --reps 10"}
for round in 1 2; do
  echo "== in-tree"; python tools/prof_kernels.py $ARGS
  for lib in tools/ab/*.so; do
    echo "== $lib"; ARV_LIB_PATH=$lib python tools/prof_kernels.py $ARGS
  done
done
