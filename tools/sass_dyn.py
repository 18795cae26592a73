"""Dynamic SASS profile of one step-kernel variant: every SASS instruction of the
profiled function (nvdisasm -gi line / inline info of the in-tree library)
joined with its executed count and stall samples from an ncu report.

    python tools/sass_dyn.py REPORT.ncu-rep [--kernel F2ELi96ELb0ELb1E] [--by callsite|line|op] [--ops IMAD,LEA]

--by callsite: the outermost step.cu line of the inline chain (which item code);
--by line: the innermost source line; --by op: opcode.  --ops filters opcodes.
"""
import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2106_13281_b200", "_lib", "libbrax_b200.so")


def sass_of(kernel_substr, unit="step", kname="brax_step_kernel"):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
    cub = os.path.join(tmp, f"{unit}.sm_100a.cubin")
    elf = subprocess.run(["cuobjdump", "-elf", cub], capture_output=True, text=True).stdout
    sym = None
    in_symtab = False
    for line in elf.splitlines():
        if line.startswith(".section .symtab"):
            in_symtab = True
            continue
        if in_symtab and line.startswith(".section"):
            break
        if in_symtab and kname in line and kernel_substr in line and line.split()[-1].startswith("_Z"):
            sym = line.split()[0]
            break
    if sym is None:
        raise SystemExit(f"no kernel matching {kernel_substr}")
    return subprocess.run(["nvdisasm", "-gi", "-fun", sym, cub], capture_output=True, text=True).stdout


def main():
    p = argparse.ArgumentParser()
    p.add_argument("report")
    p.add_argument("--kernel", default="F2ELi96ELb0ELb1E")
    p.add_argument("--lean", action="store_true", help="the lean kernel (step_lean.cu); --kernel e.g. ILi4ELi96E")
    p.add_argument("--by", default="callsite", choices=["callsite", "line", "op"])
    p.add_argument("--ops", default="")
    p.add_argument("--top", type=int, default=40)
    a = p.parse_args()
    src = {}
    for f in ("step.cu", "step_device.cuh", "step_lean.cu"):
        src[f] = open(os.path.join(ROOT, "paper_2106_13281_b200", "csrc", f)).read().splitlines()
    info = {}
    frames = []
    sass = sass_of(a.kernel, "step_lean", "brax_step_lean") if a.lean else sass_of(a.kernel)
    fresh = True  # nvdisasm -gi writes an inline chain as consecutive //## lines, innermost first
    for line in sass.splitlines():
        if "//## File" in line:
            if fresh:
                frames = []
                fresh = False
            frames += re.findall(r'"([^"]+)", line (\d+)', line)
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        fresh = True
        sc = [(os.path.basename(f), int(n)) for f, n in frames if os.path.basename(f) in src]
        info[int(m.group(1), 16)] = (sc[-1] if sc else ("?", 0), sc[0] if sc else ("?", 0), m.group(3).split(".")[0])
    rep = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(rep[1:]))))
    h = {k: i for i, k in enumerate(rows[0])}
    ops = set(a.ops.split(",")) if a.ops else None
    dyn, stall = collections.Counter(), collections.Counter()
    base = None
    tot = tots = 0
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        addr = int(r[h["Address"]], 16)
        base = addr if base is None else base
        n = int(r[h["Instructions Executed"]] or 0)
        s = int(r[h["Warp Stall Sampling (All Samples)"]] or 0)
        outer, inner, op = info.get(addr - base, (("?", 0), ("?", 0), "?"))
        tot += n
        tots += s
        if ops and op not in ops:
            continue
        key = {"callsite": outer, "line": inner, "op": op}[a.by]
        dyn[key] += n
        stall[key] += s
    print(f"total {tot} warp-instructions, {tots} stall samples; shown: {sum(dyn.values())}")
    for k, n in dyn.most_common(a.top):
        if isinstance(k, tuple):
            f, ln = k
            text = src[f][ln - 1].strip()[:90] if f in src and ln else ""
            label = f"{f}:{ln}  {text}"
        else:
            label = k
        print(f"{100 * n / tot:5.1f}% {100 * stall[k] / max(tots, 1):5.1f}%  {label}")


if __name__ == "__main__":
    main()
