"""Summarise the ncu source page: top instructions by stall samples, per kernel.
usage: python tools/ncu_source_top.py REP [N] [kernel-substring]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
pat = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name",')
for b in blocks[1:]:
    name, rest = b.split("\n", 1)
    if pat not in name: continue
    rows = list(csv.reader(io.StringIO(rest)))
    hdr = rows[0]; si = hdr.index("Warp Stall Sampling (All Samples)"); src = hdr.index("Source")
    cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h]
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    tot = sum(float(r[si] or 0) for r in data)
    print("==", name[:90], "total samples", tot)
    # aggregate by opcode
    agg = {}
    for r in data:
        op = r[src].strip().split()[0] if r[src].strip() else "?"
        if op.startswith("@"): op = r[src].strip().split()[1]
        op = op.split(".")[0]
        agg[op] = agg.get(op, 0) + float(r[si] or 0)
    print("  by opcode:", ", ".join(f"{k} {v/tot*100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]))
    data.sort(key=lambda r: -float(r[si] or 0))
    for r in data[:N]:
        print(f"  {float(r[si])/tot*100:5.2f}%  {r[0][-5:]}  {r[src].strip()[:70]}")
