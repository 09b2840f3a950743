"""Build A/B variants of libph.so with extra -D flags into ab/ (git-ignored; travels with gpurun):
    python tools/ab_build.py NAME=DEF1,DEF2 NAME2=DEF3 ...
then on the GPU box: PH_LIB=ab/libph_NAME.so python bench.py --no-cpu --no-e2e ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2202_12309_b200 import _build  # noqa: E402


def one(spec):
    name, _, defs = spec.partition("=")
    out = os.path.join(ROOT, "ab", f"libph_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    _build.build(force=True, defines=[d for d in defs.split(",") if d], out=out)
    return out


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for o in ex.map(one, sys.argv[1:]):
            print(o)
