"""Build a library variant with extra -D flags for ONE source file (the other
objects are the default build's): python tools/variant_lib.py ccd.cu out.so -DX=1 ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_02371_b200 import build as B  # noqa: E402

src, out, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
objs = []
for s in B.sources():
    if os.path.basename(s) == src:
        objs.append(B._compile(s, flags))
    else:
        objs.append(B._compile(s, []))
r = subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-cudart", "static", "-o", out, *objs],
                   capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(out)
