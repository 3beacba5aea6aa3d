"""Build library variants: python tools/build_variants.py file.cu name:-DX=1,-DY=2 name2:..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_02371_b200 import build as B  # noqa: E402

files = sys.argv[1].split(",")
os.makedirs(os.path.join(os.path.dirname(B.HERE), "variants"), exist_ok=True)
B.build()
for spec in sys.argv[2:]:
    name, flags = spec.split(":")
    flags = [f for f in flags.split(",") if f]
    objs = [B._compile(s, flags if os.path.basename(s) in files else []) for s in B.sources()]
    out = os.path.join(os.path.dirname(B.HERE), "variants", name + ".so")
    r = subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-cudart", "static", "-o", out, *objs],
                       capture_output=True, text=True)
    print(name, "ok" if r.returncode == 0 else r.stderr[-400:])
