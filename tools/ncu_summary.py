"""Summarise an ncu report: key metrics + opcode mix + top stalled SASS."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
KEYS = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Avg. Active Threads Per Warp", "Issue Slots Busy", "No Eligible", "L1/TEX Hit Rate",
        "L2 Hit Rate", "L2 Cache Throughput", "DRAM Throughput", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "Branch Efficiency", "Memory Throughput",
        "Compute (SM) Throughput", "Grid Size", "Waves Per SM", "Local Memory Spilling Requests"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(out))
hdr = next(r)
ix = {h: i for i, h in enumerate(hdr)}
seen = set()
for row in r:
    m = row[ix["Metric Name"]]
    if m in KEYS and m not in seen:
        seen.add(m)
        print(f"{m:40s} {row[ix['Metric Unit']]:>12s} {row[ix['Metric Value']]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) >= 3:
    names, units, vals = rr[0], rr[1], rr[2]
    for want in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                 "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
                 "l1tex__t_bytes.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
                 "lts__t_sectors_srcunit_tex_op_write.sum", "gpu__time_duration.sum"]:
        if want in names:
            k = names.index(want)
            print(f"{want:40s} {units[k]:>12s} {vals[k]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot = collections.Counter(); st = collections.Counter(); T = S = 0
seq = []
for row in rows[2:]:
    s = row[ix["Source"]].strip()
    toks = s.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    ti = int(row[ix["Thread Instructions Executed"]] or 0)
    sm = int(row[ix["Warp Stall Sampling (All Samples)"]] or 0)
    wi = int(row[ix["Instructions Executed"]] or 0)
    tot[op] += ti; st[op] += sm; T += ti; S += sm
    seq.append((row[ix["Address"]][-5:], s, wi, ti, sm))
print(f"thread-inst {T}  stall-samples {S}")
for op, c in tot.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 16):
    print(f"  {op:10s} {100*c/T:5.1f}% thr  {100*st[op]/max(S,1):5.1f}% stall")
print("top stalls:")
for a, s, wi, ti, sm in sorted(seq, key=lambda x: -x[4])[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
    print(f"  {a} {s[:64]:64s} warp-exec {wi:9d} samples {sm}")
