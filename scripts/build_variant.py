"""Build an A/B variant of libhelm with extra -D flags: python scripts/build_variant.py NAME -DX=1 ...
-> paper_1703_09268_b200/lib/libhelm_NAME.so (load with HELM_LIB_VARIANT=NAME). Prints march2d /
plane register and spill counts."""
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_09268_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.PKG, "lib", f"libhelm_{name}.so")
cmd = [B.nvcc(), *B.NVCC_FLAGS, "-Xptxas=-v", *defs, "-I", os.path.join(B.ROOT, "include"), "-o", out, *B.SRC]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    print(r.stderr[-3000:])
    sys.exit(1)
cur, sp = None, ""
pat = re.compile(os.environ.get("KPAT", r"_Z9k_march2dIdLi[34]ELi[2-5]E"))
for l in r.stderr.splitlines():
    m = re.search(r"Compiling entry function '([^']*)'", l)
    if m:
        cur = m.group(1) if pat.search(m.group(1)) else None
        continue
    if cur and "spill" in l:
        sp = l.split(",", 1)[0].strip() + " / " + l.strip().split(",")[1].strip()
    if cur and "Used" in l:
        print(name, cur[:26], re.search(r"Used \d+ registers", l).group(0), "|", sp)
        cur = None
print(out)
