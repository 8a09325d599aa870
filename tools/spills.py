"""Dev: map STL/LDL (register spills) of each kernel instantiation to source lines.
usage: python tools/spills.py LIB.so"""
import re, subprocess, sys, tempfile, os, glob
from collections import Counter
lib = sys.argv[1]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
txt = "".join(subprocess.run(["nvdisasm", "-g", "-c", c], capture_output=True, text=True).stdout
              for c in sorted(glob.glob(os.path.join(d, "*.cubin"))))
cur = curline = None
per = {}
for l in txt.splitlines():
    m = re.search(r'\.text\.(\S+):', l)
    if m: cur = m.group(1)
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m: curline = (os.path.basename(m.group(1)), int(m.group(2)))
    if cur and re.search(r'\b(STL|LDL)', l):
        per.setdefault(cur, Counter())[curline] += 1
for k, c in per.items():
    print(k[17:60], sum(c.values()), sorted(c.items(), key=lambda x: -x[1])[:10])
