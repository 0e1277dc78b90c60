"""Build experiment / diagnostic variants of libmxmoe.so in parallel: python tools/build_variants.py name=DEF1,DEF2 ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_05799_b200 import build as b  # noqa: E402


def one(spec):
    name, _, defs = spec.partition("=")
    out = os.path.join(ROOT, "tools", "variants", f"lib_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    try:
        b.build_variant(out, [d for d in defs.split(",") if d])
        return name, 0
    except RuntimeError as e:
        return name, str(e)


rc = 0
with ThreadPoolExecutor(max_workers=4) as ex:
    for name, r in ex.map(one, sys.argv[1:]):
        print(name, "rc", r)
        rc |= r != 0
sys.exit(rc)
