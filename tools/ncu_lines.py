#!/usr/bin/env python3
"""Per-source-line view of an .ncu-rep: tools/ncu_lines.py X.ncu-rep [samples|inst|global|long_sb] [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; key = sys.argv[2] if len(sys.argv) > 2 else "samples"; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
cur = None; h2 = None; recs = []
for r in csv.reader(io.StringIO(src)):
    if not r: continue
    if r[0] in ("File Path", "File Name"): cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": h2 = r; continue
    if r[0] == "Function Name": continue
    if h2 and len(r) == len(h2) and r[0] != "": recs.append((cur, r))
f = lambda x: float(x or 0)
col = {"samples": "# Samples", "inst": "Instructions Executed", "global": "L2 Theoretical Sectors Global", "long_sb": "stall_long_sb", "local": "L2 Theoretical Sectors Local"}[key]
ix = h2.index(col); ie = h2.index("Instructions Executed"); te = h2.index("Thread Instructions Executed"); ss = h2.index("# Samples")
tot = sum(f(r[ix]) for _, r in recs); toti = sum(f(r[ie]) for _, r in recs); tots = sum(f(r[ss]) for _, r in recs)
print(f"total {col}: {tot:.4g}; instructions {toti:.4g}; samples {tots:.4g}")
for fn, r in sorted(recs, key=lambda x: -f(x[1][ix]))[:top]:
    i = f(r[ie])
    print("%5.1f%%  inst %4.1f%%  smp %4.1f%%  lanes %4.1f  %s:%s  %s" % (100 * f(r[ix]) / max(tot, 1), 100 * i / toti, 100 * f(r[ss]) / tots, f(r[te]) / max(i, 1), fn, r[0], r[1].strip()[:100]))
