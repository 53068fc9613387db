"""Build an experiment variant of the library with extra -D flags into
build/variant/ (the product library is untouched) and print its path.

    python tools/variant_build.py -DSK_DECODE_STAGES=2
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_06283_b200 import build as B  # noqa: E402


def main():
    flags = sys.argv[1:]
    out = os.path.join(ROOT, "build", "variant")
    os.makedirs(out, exist_ok=True)
    objs = []
    for s in B._sources():
        o = os.path.join(out, os.path.basename(s)[:-3] + ".o")
        subprocess.run([B.nvcc()] + B.ARCH + B.NVCC_FLAGS + flags + ["-c", s, "-o", o], check=True)
        objs.append(o)
    lib = os.path.join(out, "libsocket_variant.so")
    subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
