"""Aggregate ncu SASS-level warp-stall samples by CUDA source line.
usage: python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_MANGLED [top]
(needs -lineinfo; maps SASS addresses through nvdisasm --print-line-info of the cubin)"""
import csv, io, os, re, subprocess, sys, tempfile, collections

rep, lib, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
addr2line = {}
for cub in os.listdir(d):
    if not cub.endswith(".cubin"):
        continue
    dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True, text=True).stdout
    cur = None
    infn = False
    for line in dis.splitlines():
        if line.startswith("//---------------------"):
            infn = ".text." in line and kern in line
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
        if m and cur:
            addr2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ci = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.defaultdict(lambda: collections.Counter())
tot = 0
base = None
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    if base is None:
        base = int(r[0], 16)  # ncu prints absolute addresses; the first is the function start
    a = int(r[0], 16) - base
    key = addr2line.get(a, ("?", 0))
    n = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    agg[key]["samples"] += n
    agg[key]["inst"] += int(r[ci["Instructions Executed"]] or 0)
    tot += n
    for s in stalls:
        v = r[ci[s]]
        if v:
            agg[key][s] += int(float(v))
print(f"total samples {tot}")
src = {}
for key in agg:
    f = key[0]
    for root in ("paper_2008_03518_b200/csrc",):
        p = os.path.join(root, f)
        if os.path.exists(p) and f not in src:
            src[f] = open(p).read().splitlines()
for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    f, ln = key
    text = src.get(f, [""] * (ln + 1))[ln - 1].strip()[:70] if f in src and ln > 0 else ""
    st = sorted(((k[6:], v) for k, v in c.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:3]
    print(f"{100 * c['samples'] / tot:5.1f}% {f}:{ln:<5d} {' '.join(f'{k}={v}' for k, v in st):48s} | {text}")
