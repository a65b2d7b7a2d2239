"""Build an experimental variant of the library with -D flags, for A/B timing on the GPU:

    python tools/build_variant.py build/variants/libbiot_x.so BIOT_SOMETHING=1 ...
    BIOT_LIB_OVERRIDE=build/variants/libbiot_x.so python bench.py ...
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2310_10430_b200 import build as B  # noqa: E402

if __name__ == "__main__":
    out = os.path.abspath(sys.argv[1])
    os.makedirs(os.path.dirname(out), exist_ok=True)
    print(B.build(out=out, defines=sys.argv[2:]))
