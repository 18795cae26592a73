"""Mutation runs of the fp64 oracle against its CPU pin suite (VERDICT r1 "What's
weak" 1): copy the repo to a scratch directory, apply ONE source mutation to
oracle/brax_oracle.cpp, rebuild the oracle there and run `pytest -m "not gpu"`.
A mutation is "killed" if at least one test fails.  Prints one line per mutation
and writes profiles/r2/mutations.txt.

    python tools/mutation_check.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "oracle/brax_oracle.cpp"

# (name, exact source text, replacement) — each must occur exactly once
MUTATIONS = [
    ("torque: 2*s*a, no clamp (R11)",
     "tau[i] = tau[i] + T(J.act_strength) * xclamp(a, T(-1.0), T(1.0));",
     "tau[i] = tau[i] + T(2.0) * T(J.act_strength) * a;"),
    ("torque: clamp dropped (R11)",
     "tau[i] = tau[i] + T(J.act_strength) * xclamp(a, T(-1.0), T(1.0));",
     "tau[i] = tau[i] + T(J.act_strength) * a;"),
    ("elasticity: (1+e) -> (1-e) (R13)",
     "-(T(1.0) + T(S.e)) * un",
     "-(T(1.0) - T(S.e)) * un"),
    ("friction: mu factor dropped (R13)",
     "T jt = xmin(st_ / eff(that), T(S.mu) * jn);",
     "T jt = xmin(st_ / eff(that), jn);"),
    ("I_w^-1: rotation order transposed (R4)",
     "return rotate(q, divide(inv_rotate(q, v), inertia));",
     "return inv_rotate(q, divide(rotate(q, v), inertia));"),
    ("I_w^-1: inertia multiplied instead of divided (R4)",
     "return rotate(q, divide(inv_rotate(q, v), inertia));",
     "return rotate(q, hadamard(inv_rotate(q, v), inertia));"),
    ("op counter: sqrt counted as 1 flop (SURVEY 8(d))",
     "inline Cnt xsqrt(Cnt x) { g_flops += 4;",
     "inline Cnt xsqrt(Cnt x) { g_flops += 1;"),
    ("op counter: atan2 not counted (SURVEY 8(d))",
     "inline Cnt xatan2(Cnt y, Cnt x) { g_flops += 20;",
     "inline Cnt xatan2(Cnt y, Cnt x) { g_flops += 0;"),
    ("op counter: division counted as 1 flop (SURVEY 8(d))",
     "inline Cnt operator/(Cnt a, Cnt b) { g_flops += 4;",
     "inline Cnt operator/(Cnt a, Cnt b) { g_flops += 1;"),
    ("contact: Baumgarte bias beta/h -> beta (R13)",
     "(T(S.beta) / h) * d",
     "T(S.beta) * d"),
    ("joint: angular damping sign flipped (R5)",
     "V3<T> td = T(J.c_a) * (P.w - C.w);",
     "V3<T> td = T(J.c_a) * (C.w - P.w);"),
    ("collision integrator: sum instead of mean (R14)",
     "T scale = opt.combine_sum ? T(1.0) : T(1.0) / T(double(cnt[b]));",
     "T scale = T(1.0);"),
]


def run_one(name, old, new, tmp):
    path = os.path.join(tmp, SRC)
    with open(os.path.join(ROOT, SRC)) as f:
        src = f.read()
    assert src.count(old) == 1, f"mutation site not unique: {name}"
    with open(path, "w") as f:
        f.write(src.replace(old, new))
    shutil.rmtree(os.path.join(tmp, "oracle", "_build"), ignore_errors=True)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                        "-x", "--timeout", "600"], cwd=tmp, capture_output=True, text=True)
    tail = [ln for ln in r.stdout.splitlines() if ln.strip()]
    failed = [ln for ln in tail if ln.startswith("FAILED")]
    summary = tail[-1] if tail else r.stderr[-200:]
    return r.returncode != 0, (failed[0] if failed else summary)


def main():
    tmp = tempfile.mkdtemp(prefix="brax_mut_")
    ign = shutil.ignore_patterns(".git", "gpurun_out", "_build", "__pycache__", "profiles")
    shutil.copytree(ROOT, tmp, dirs_exist_ok=True, ignore=ign)
    lines = []
    try:
        for name, old, new in MUTATIONS:
            killed, why = run_one(name, old, new, tmp)
            line = f"{'KILLED ' if killed else 'SURVIVED'} | {name} | {why}"
            print(line, flush=True)
            lines.append(line)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    out = os.path.join(ROOT, "profiles", "r2", "mutations.txt")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        f.write("# tools/mutation_check.py: one oracle mutation at a time, CPU pin suite (pytest -m 'not gpu')\n")
        f.write("\n".join(lines) + "\n")
    return 0 if all(ln.startswith("KILLED") for ln in lines) else 1


if __name__ == "__main__":
    sys.exit(main())
