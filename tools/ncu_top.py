"""Summarise an ncu report: headline metrics + top stall sites (SASS)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
launch = sys.argv[2] if len(sys.argv) > 2 else "0"
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
want = ['Duration', 'Compute (SM) Throughput', 'DRAM Throughput', 'L2 Cache Throughput', 'L1/TEX Cache Throughput',
        'Executed Ipc Active', 'Issue Slots Busy', 'No Eligible', 'Registers Per Thread']
for r in rows[1:]:
    if r[ix['ID']] == launch and r[ix['Metric Name']] in want:
        print(f"  {r[ix['Metric Name']]:32s} {r[ix['Metric Value']]} {r[ix['Metric Unit']]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
keys = [k for k in h if any(s in k for s in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active", "sm__inst_executed_pipe_fp64", "pipe_tensor", "smsp__inst_executed_op_dmma", "sm__throughput"))]
for row in rr[2:]:
    if row[h.index("ID")] == launch:
        for k in keys:
            print(f"  {k:60s} {row[h.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", launch, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
seen = set(); lst = []
for r in rows[2:]:
    if len(r) <= ist or r[ia] in seen: continue
    try: float(r[ist] or 0)
    except ValueError: continue
    seen.add(r[ia]); lst.append(r)
tot = sum(float(r[ist] or 0) for r in lst)
print("  top stall sites (% of samples):")
for r in sorted(lst, key=lambda r: -float(r[ist] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
    j = lst.index(r)
    ctx = " | ".join(x[isrc].strip()[:40] for x in lst[max(0, j - 3):j] if "SYNCS" in x[isrc] or "BAR" in x[isrc])
    print(f"   {r[ia][-5:]} {float(r[ist]) / tot * 100:5.1f}%  {r[isrc].strip()[:60]}  {ctx}")
