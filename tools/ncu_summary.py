"""Summarise gpurun_out ncu captures into profiles/<round>_ncu_summary.md (+ traffic json)."""
import collections, csv, io, json, subprocess, sys

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
WANT = ['gpu__time_duration.sum', 'launch__grid_size', 'launch__cluster_size', 'launch__block_size',
        'launch__registers_per_thread', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    return {h: (v, u) for h, u, v in zip(rr[0], rr[1], rr[2])}


def source(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[1], rows[2:]


def stalls(hdr, data, a, b):
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    s = collections.Counter()
    for r in data[a:b]:
        for c in cols:
            s[c[6:]] += float(r[hdr.index(c)] or 0)
    t = sum(s.values()) or 1
    return {k: v / t * 100 for k, v in s.items() if v / t > 0.01}


lines = [f"# {rnd} — ncu evidence (B200, sm_100a)\n",
         "Captures (`ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1`; the",
         "library each capture was taken with is kept beside it in gpurun_out for the line mapping):",
         "- `walk_batch`: first walk launch of the configs[1] FCFS batch (`tools/ncu_batch.py`): the first",
         "  slice's head request alone at G = 16 to completion -- the batch's critical path -- §8(a) path;",
         "- `walk_cull16`: one configs[1] request with SURVEY f1 culling on one 16-CTA cluster (`tools/ncu_cull.py 16`);",
         "- `walk_f4`: one configs[1] request with the A = 1350 action space, wide walker (`tools/ncu_f4.py`);",
         "- `walk_c5split`: configs[4] (1M plans, A = 85) one request on the full path split over the",
         "  co-resident clusters with the in-kernel exchange (`tools/ncu_c5.py`), the roofline stress.",
         "L2 traffic = lts__t_sectors.sum x 32 B.",
         "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` of `python bench.py --steps 1",
         "--warmup 3 --no-cpu-baseline --no-c4` (the headline blocks; cold-cache, serialised: compare shares,",
         "not absolutes; the configs[2..4] blocks are left out: ncu serialises the p2p ranks' kernels).\n"]
rows = list(csv.reader(open(sys.argv[2] if len(sys.argv) > 2 else 'gpurun_out/launches.csv')))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[hi]; data = rows[hi + 1:]
ik, iv, im = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name')
t = collections.defaultdict(float); n = collections.Counter()
for r in data:
    if len(r) <= iv or r[im] != 'gpu__time_duration.sum':
        continue
    name = r[ik].split('(')[0].replace('void ', '')
    t[name] += float(r[iv].replace(',', '')); n[name] += 1
tot = sum(t.values())
lines += ["## Launch list of the bench command\n", "| kernel | launches | device time (ms) | share |", "|---|---|---|---|"]
for k in sorted(t, key=lambda k: -t[k]):
    lines.append(f"| `{k}` | {n[k]} | {t[k] / 1e6:.2f} | {t[k] / tot * 100:.1f}% |")
lines.append("")
traffic = None
import os
for rep, kern, title in (('walk_batch', 'walk_kernel<3, 0>', 'configs[1] batch, first slice head (full path)'),
                         ('walk_cull16', 'walk_kernel<3, 4>', 'configs[1] request, f1 culling, G=16'),
                         ('walk_cull8', 'walk_kernel<3, 4>', 'configs[1] request, f1 culling, G=8 (the culled head size)'),
                         ('walk_f4', 'walk_kernel<10, 5>', 'configs[1] request, A = 1350 (SURVEY f4), wide walker'),
                         ('walk_c5split', 'walk_kernel<5, 2>', 'configs[4] 1M plans, A = 85, split request (full path)')):
    rep = f'{rnd}_{rep}'
    if not os.path.exists(f'gpurun_out/{rep}.ncu-rep'):
        continue
    m = raw(f'gpurun_out/{rep}.ncu-rep')
    if 'lts__t_sectors.sum' in m:
        lb = float(m['lts__t_sectors.sum'][0].replace(',', '')) * 32
        m['l2_bytes (lts__t_sectors x 32)'] = (f"{lb / 1e6:.3f}", 'Mbyte')
        WANT_ = WANT + ['l2_bytes (lts__t_sectors x 32)']
    else:
        WANT_ = WANT
    lines += [f"## {kern} — {title}\n", "| metric | value |", "|---|---|"]
    for k in WANT_:
        if k in m:
            lines.append(f"| `{k}` | {m[k][0]} {m[k][1]} |")
    if rep.endswith('walk_batch'):
        rd = float(m['dram__bytes_read.sum'][0].replace(',', '')) * (1e6 if m['dram__bytes_read.sum'][1] == 'Mbyte' else 1e3 if m['dram__bytes_read.sum'][1] == 'Kbyte' else 1e9 if m['dram__bytes_read.sum'][1] == 'Gbyte' else 1)
        wr = float(m['dram__bytes_write.sum'][0].replace(',', '')) * (1e6 if m['dram__bytes_write.sum'][1] == 'Mbyte' else 1e3 if m['dram__bytes_write.sum'][1] == 'Kbyte' else 1e9 if m['dram__bytes_write.sum'][1] == 'Gbyte' else 1)
        traffic = dict(kernel="walk_kernel<3, 0>", capture=f"{rnd} walk_batch (tools/ncu_batch.py, first launch)",
                       dram_bytes_read=int(rd), dram_bytes_write=int(wr), per_launch_bytes=int(rd + wr),
                       l2_bytes=int(float(m['lts__t_sectors.sum'][0].replace(',', '')) * 32) if 'lts__t_sectors.sum' in m else None,
                       note="DRAM traffic per launch; the kernel is FP32-pipe bound, plan rows are L2-resident")
    h, d = source(f'gpurun_out/{rep}.ncu-rep')
    iss = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed"); isrc = h.index("Source")
    # hottest compute region: skip mbarrier spin-waits (SYNCS / YIELD loops)
    ex = [0.0 if any(k in r[isrc] for k in ('SYNCS', 'YIELD', 'NANOSLEEP')) else float(r[ie] or 0) for r in d]
    mx = max(ex)
    im = ex.index(mx)  # the contiguous block around the most-executed instruction
    a = im
    while a > 0 and ex[a - 1] >= 0.9 * mx:
        a -= 1
    b = im + 1
    while b < len(ex) and ex[b] >= 0.9 * mx:
        b += 1
    ts = sum(float(r[iss] or 0) for r in d)
    hs = sum(float(r[iss] or 0) for r in d[a:b])
    st = stalls(h, d, a, b)
    allst = stalls(h, d, 0, len(d))
    ops = collections.Counter()
    for r in d[a:b]:
        tok = r[isrc].split()
        op = tok[1] if tok and tok[0].startswith('@') else (tok[0] if tok else '')
        ops[op.split('.')[0]] += 1
    if b - a < 10:
        lines += ["", "No dominant loop (latency-bound step): per-source-line stall attribution in "
                  f"profiles/{rnd}_lines_{rep}.txt (tools/ncu_lines.py).",
                  "Whole kernel: " + ", ".join(f"{k} {v:.1f}%" for k, v in sorted(allst.items(), key=lambda x: -x[1])) + ".", ""]
        continue
    lines += ["", f"Most-executed loop: {b - a} SASS instructions, {hs / ts * 100:.1f} % of warp-stall samples; "
              + "reasons: " + ", ".join(f"{k} {v:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])) + ".",
              "Instruction mix: " + ", ".join(f"{k} {v}" for k, v in ops.most_common()) + ".",
              "Whole kernel: " + ", ".join(f"{k} {v:.1f}%" for k, v in sorted(allst.items(), key=lambda x: -x[1])) + ".", ""]
open(f'profiles/{rnd}_ncu_summary.md', 'w').write("\n".join(lines) + "\n")
if traffic:
    json.dump(traffic, open(f'profiles/{rnd}_traffic.json', 'w'), indent=1)
print("\n".join(lines))
