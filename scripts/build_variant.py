"""Builds the library with extra nvcc defines into variants/<name>.so (A/B measurements;
select at run time with MSF_LIB_PATH=variants/<name>.so).  Usage:
    python scripts/build_variant.py NAME -DMACRO=VALUE ..."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1411_3923_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out_dir = os.path.join(ROOT, "variants")
    os.makedirs(out_dir, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        objs = []
        for src in B.sources():
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            subprocess.check_call([B.NVCC, *B.FLAGS, *defs, "-c", src, "-o", obj])
            objs.append(obj)
        out = os.path.join(out_dir, name + ".so")
        subprocess.check_call([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-o", out, *objs, "-lcudart", "-ldl"])
    print(out)


if __name__ == "__main__":
    main()
