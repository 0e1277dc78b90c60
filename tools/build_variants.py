"""Build experiment / diagnostic variants of libmxmoe.so in parallel: python tools/build_variants.py name=DEF1,DEF2 ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_05799_b200 import build as b  # noqa: E402

procs = []
for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    out = os.path.join(ROOT, "tools", "variants", f"lib_{name}.so")
    cmd = [b.NVCC, *b.FLAGS, *[f"-D{d}" for d in defs.split(",") if d], "-o", out,
           *[os.path.join(b.CSRC, s) for s in b.SOURCES]]
    procs.append((name, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
rc = 0
for name, p in procs:
    out, _ = p.communicate()
    print(name, "rc", p.returncode, out[-400:] if p.returncode else "")
    rc |= p.returncode
sys.exit(rc)
