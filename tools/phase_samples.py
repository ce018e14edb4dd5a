"""Aggregate ncu warp-stall samples between the CS2R SR_CLOCKLO phase markers (SASS order)."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
iss = hdr.index("Warp Stall Sampling (All Samples)"); isrc = hdr.index("Source"); ie = hdr.index("Instructions Executed")
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]; ci = [hdr.index(c) for c in cols]
tot = sum(float(r[iss] or 0) for r in data)
seg = 0; segs = collections.OrderedDict(); first = {}
for i, r in enumerate(data):
    if 'SR_CLOCKLO' in r[isrc]:
        seg += 1
    d = segs.setdefault(seg, [0.0, collections.Counter(), 0])
    d[0] += float(r[iss] or 0); d[2] += 1
    for c, k in zip(cols, ci): d[1][c[6:]] += float(r[k] or 0)
    first.setdefault(seg, i)
for s, (v, st, n) in segs.items():
    if v / tot < 0.005: continue
    top = ", ".join(f"{k} {x/v*100:.0f}%" for k, x in st.most_common(3))
    print(f"seg {s:3d} @{first[s]:5d} n={n:4d} {v/tot*100:5.1f}%  {top}  | {data[first[s]][isrc].strip()[:50]}")
