"""Summarise an ncu source-page SASS CSV: executed instructions and stall samples
by opcode, plus the top instructions.  Usage: python tools/ncu_sass_summary.py rep.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
by_op = collections.Counter()
stall = collections.Counter()
thr = collections.Counter()
total = 0
tot_stall = 0
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    t = int(r[ix["Thread Instructions Executed"]] or 0)
    by_op[op] += n
    stall[op] += s
    thr[op] += t
    total += n
    tot_stall += s
print(f"total warp-instructions {total}, stall samples {tot_stall}")
print(f"{'op':10s} {'inst%':>7s} {'stall%':>7s} {'lanes':>6s}")
for op, n in by_op.most_common(30):
    print(f"{op:10s} {100*n/total:7.2f} {100*stall[op]/max(1,tot_stall):7.2f} {thr[op]/max(1,n):6.1f}")
