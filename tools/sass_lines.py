"""Attribute an ncu report's executed SASS instructions to source lines, split by
opcode class (fp32 / shared-memory / control / integer / other), using the line
table of the kernel's cubin (nvdisasm -gi).  The cubin must be the build that was
profiled.  Usage: python tools/sass_lines.py rep.ncu-rep step.sm_100a.cubin [N]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
kname = next(csv.reader([lines[0]]))[1]
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = {h: i for i, h in enumerate(rows[0])}
ex = []
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    ex.append((int(r[hdr["Address"]], 16), r[hdr["Source"]].strip(), int(r[hdr["Instructions Executed"]] or 0)))
base = ex[0][0]
# mangled-name match: template args of the profiled kernel
m = re.search(r"brax_step_kernel<(?:[\w:]+::)?(\w+), (?:\(int\))?(\d+)(?:, (?:\(bool\))?(\w+))?>", kname)
lane, regs, env = m.group(1), m.group(2), m.group(3)
envbit = "1" if env in ("1", "true") else "0"
want = f"INS_3dev2{lane}ELi{regs}ELb{envbit}E" if env is not None else f"INS_3dev2{lane}ELi{regs}E"
dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
loc = {}
cur = None
func = None
for l in dis.splitlines():
    if l.startswith("\t.text.") or l.startswith(".text."):
        func = l
    mm = re.match(r"\s*//## File \"([^\"]+)\", line (\d+)(.*)", l)
    if mm:
        cur = (mm.group(1).split("/")[-1] + ":" + mm.group(2))
        inl = re.search(r"inlined at \"([^\"]+)\", line (\d+)", mm.group(3))
        if inl:
            cur += " <- " + inl.group(1).split("/")[-1] + ":" + inl.group(2)
        continue
    mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if mo and func and want in func:
        loc[int(mo.group(1), 16)] = cur


def cls(src):
    op = src.split()[0]
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    if op in ("FFMA", "FMUL", "FADD", "FFMA2", "FMUL2", "FADD2"):
        return "fp"
    if op in ("LDS", "STS"):
        return "smem"
    if op in ("BRA", "BSSY", "BSYNC", "ISETP", "PLOP3", "BAR", "EXIT", "WARPSYNC", "UISETP", "BRX", "CALL", "RET"):
        return "ctrl"
    if op in ("IADD3", "IMAD", "LEA", "LOP3", "SHF", "IABS", "UIADD3", "ULEA", "ULOP3", "USHF", "UIMAD", "VIADD", "IMNMX"):
        return "int"
    if op in ("MOV", "UMOV", "CS2R", "S2R", "S2UR", "R2UR", "LDC", "LDCU", "MOV32I"):
        return "mov"
    return "other"


by = collections.defaultdict(collections.Counter)
tot = collections.Counter()
miss = 0
for a, src, n in ex:
    key = loc.get(a - base)
    if key is None:
        miss += n
        key = "?"
    c = cls(src)
    by[key][c] += n
    by[key]["all"] += n
    tot[c] += n
    tot["all"] += n
print(f"kernel {kname}; {tot['all']} warp-inst; unmapped {miss}")
print("class totals: " + ", ".join(f"{k} {100 * v / tot['all']:.1f}%" for k, v in tot.most_common()))
print(f"{'all%':>6s} {'fp':>5s} {'smem':>5s} {'ctrl':>5s} {'int':>5s} {'mov':>5s} {'oth':>5s}  line")
for key, c in sorted(by.items(), key=lambda kv: -kv[1]["all"])[:N]:
    print(f"{100 * c['all'] / tot['all']:6.2f} " + " ".join(f"{100 * c[k] / tot['all']:5.2f}" for k in ("fp", "smem", "ctrl", "int", "mov", "other")) + f"  {key}")
