"""Dev: per-kernel statistics of the DMMA k-loop body in SASS (accumulator renames D != C,
non-DMMA instructions, local-memory spills).  usage: python tools/kloop_stats.py LIB.so"""
import glob, os, re, subprocess, sys, tempfile
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(sys.argv[1])], cwd=d, capture_output=True)
txt = "".join(subprocess.run(["nvdisasm", "-c", c], capture_output=True, text=True).stdout
              for c in sorted(glob.glob(os.path.join(d, "*.cubin"))))
funcs, cur = {}, None
for l in txt.splitlines():
    m = re.search(r'\.text\.(\S+):', l)
    if m:
        cur = m.group(1); funcs[cur] = []
    elif cur:
        m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
        if m and 'NOP' not in m.group(2):
            funcs[cur].append(m.group(2).strip())
for name, ins in funcs.items():
    if 'dgemm_abft_kernel' not in name:
        continue
    idx = [i for i, t in enumerate(ins) if 'DMMA' in t]
    # the main k-loop body: the densest window of 128 consecutive DMMAs (thin / segment loops
    # with fewer DMMAs per stage come first in the function)
    w = min(range(len(idx) - 127), key=lambda a: idx[a + 127] - idx[a])
    loop = ins[idx[w]:idx[w + 127] + 1]
    dc = sum(1 for t in loop if (m := re.search(r'DMMA\.8x8x4 (R\d+), R\d+, R\d+, (R\d+)', t)) and m.group(1) != m.group(2))
    other = sum(1 for t in loop if 'DMMA' not in t)
    ldl = sum(1 for t in loop if 'LDL' in t or 'STL' in t)
    print(f"{name[24:40]}  D!=C {dc:3d}  other {other:3d}  LDL/STL {ldl}")
