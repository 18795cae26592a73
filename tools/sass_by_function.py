"""Static SASS instruction mix per device function of the step kernel
(nvdisasm -gi line/inline info mapped to function line ranges of step_device.cuh).
Usage: python tools/sass_by_function.py step.sm_100a.cubin [ncu-report]"""
import collections
import csv
import io
import re
import subprocess
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]
dev = open(f"{ROOT}/paper_2106_13281_b200/csrc/step_device.cuh").read().splitlines()
ranges = []  # (start_line, name)
for i, l in enumerate(dev, 1):
    m = re.match(r"__device__ __forceinline__ \S+ (\w+)\(", l) or re.match(r"struct (\w+) \{", l)
    if m:
        ranges.append((i, m.group(1)))
TOP = {"kinematic", "joint", "contact", "integrate", "Acc", "stage", "load_block", "load_actions", "block_extras",
       "store_block", "stg_to_records", "records_to_stg", "seg_seg", "atan2_f", "asin_f", "iw", "rotate"}


kern = open(f"{ROOT}/paper_2106_13281_b200/csrc/step.cu").read().splitlines()


def func_of(line):
    name = None
    for start, n in ranges:
        if start <= line:
            name = n
    return name


cubin = sys.argv[1]
txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
frames = []
stats = collections.defaultdict(collections.Counter)
addr_func = {}
for l in txt.splitlines():
    if "//## File" in l:
        frames = re.findall(r'"([^"]+)", line (\d+)', l)
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", l)
    if not m:
        continue
    addr = int(m.group(1), 16)
    op = m.group(3).split(".")[0]
    owner = "kernel"
    # nvdisasm gives the innermost location "inlined at" the kernel's call site:
    # attribute by the callee named on that step.cu line
    for f, ln in frames:
        if f.endswith("step.cu"):
            src = kern[int(ln) - 1]
            for name in ("kinematic", "joint", "contact", "integrate", "acc.joint", "acc.slot", "stg_to_records",
                         "records_to_stg", "block_extras", "load_block", "load_actions", "store_block",
                         "tma_", "mbar_"):
                if name + "(" in src:
                    owner = name
                    break
            else:
                owner = f"step.cu:{ln}"
    stats[owner][op] += 1
    addr_func[addr] = owner

dyn = collections.Counter()
if len(sys.argv) > 2:
    rep = subprocess.run(["ncu", "-i", sys.argv[2], "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(rep[1:]))))
    h = {k: i for i, k in enumerate(rows[0])}
    base = None
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        a = int(r[h["Address"]], 16)
        if base is None:
            base = a
        dyn[addr_func.get(a - base, "?")] += int(r[h["Instructions Executed"]] or 0)
FP = {"FFMA", "FMUL", "FADD", "FSEL", "FMNMX", "FSETP", "MUFU", "HFMA2"}
tot_dyn = sum(dyn.values()) or 1
print(f"{'function':16s} {'static':>7s} {'fp%':>5s} {'lds/sts':>8s} {'ctrl':>5s}  {'dyn%':>6s}")
for fn, c in sorted(stats.items(), key=lambda kv: -dyn.get(kv[0], 0)):
    n = sum(c.values())
    fp = sum(v for k, v in c.items() if k in FP)
    mem = c["LDS"] + c["STS"]
    ctrl = c["BRA"] + c["BSSY"] + c["BSYNC"] + c["ISETP"]
    print(f"{fn:16s} {n:7d} {100 * fp / n:5.1f} {mem:8d} {ctrl:5d}  {100 * dyn.get(fn, 0) / tot_dyn:6.1f}")
