"""Pretty-print tools/sweep.py JSON lines with their prefixes: python tools/experiments/show.py LOG"""
import json
import sys

for line in open(sys.argv[1]):
    if "{" not in line:
        print(line.rstrip())
        continue
    pre, js = line.split("{", 1)
    d = json.loads("{" + js)
    c = d["cfg"]
    print(f"{pre.strip():24s} {d['scene']:12s} {d['envs']:6d} {d['us_per_step']:7.2f} us  frac {d['frac_fp32_1965']:.3f}  "
          f"G{c['G']} V{c['V']} W{c['warps']} r{c['regs']} fx{c['fixed_gather']} t{c['tuned']} lean{c.get('lean', 0)}")
