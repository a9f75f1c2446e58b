for r in 1 2; do
python tools/gen_tune.py
for lib in tools/ab/*.so; do ARV_LIB_PATH=$lib python tools/gen_tune.py; done
done
