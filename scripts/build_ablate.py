"""Build experiment variants of the library: python scripts/build_ablate.py NAME=-DMACRO[,-DMACRO2] ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_08158_b200 import build as b  # noqa: E402


def one(spec):
    name, flags = spec.split("=", 1)
    out = os.path.join(b.HERE, f"libads_ablate_{name}.so")
    b.build(extra=flags.split(","), out=out)
    return out


with ThreadPoolExecutor(max_workers=4) as ex:
    for o in ex.map(one, sys.argv[1:]):
        print(o)
