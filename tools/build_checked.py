"""Build the checked library (device-side bounds / invariant asserts, ARV_CHECKS=1)
into tools/checked/, for running the GPU test suite against it:

    python tools/build_checked.py
    ARV_LIB_PATH=tools/checked/libarv_b200_checked.so python -m pytest tests -m gpu

(compute-sanitizer is closed on the GPU pool.)
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2012_09715_b200 import _build  # noqa: E402

if __name__ == "__main__":
    os.makedirs(os.path.join(HERE, "checked"), exist_ok=True)
    print(_build.build(defines=("ARV_CHECKS=1",), out=os.path.join(HERE, "checked", "libarv_b200_checked.so")))
