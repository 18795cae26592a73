"""Top source lines of an ncu report by executed warp-instructions and stall samples.
Usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
path = "?"
hdr = None
rows = []
for rec in csv.reader(io.StringIO(txt)):
    if not rec:
        continue
    if rec[0] == "File Path":
        path = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = {h: i for i, h in enumerate(rec)}
        continue
    if hdr and rec[0] and rec[0] != "-":
        try:
            n = int(rec[hdr["Instructions Executed"]] or 0)
            s = int(rec[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError, IndexError):
            continue
        rows.append((n, s, path, rec[0], rec[1].strip()[:90]))
tot = sum(r[0] for r in rows)
tots = sum(r[1] for r in rows)
print(f"total {tot} warp-inst, {tots} samples")
for n, s, p, ln, src in sorted(rows, reverse=True)[:N]:
    print(f"{100 * n / tot:5.1f}% {100 * s / max(tots, 1):5.1f}%  {p}:{ln}  {src}")
