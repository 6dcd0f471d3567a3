"""Mutation check of the oracle's CPU pins (VERDICT r01 "What's weak #1").

Copies the repo (without .git / gpurun_out) to a scratch directory, applies one
plausible mistake at a time to oracle/oracle.c, rebuilds the oracle there and
runs the oracle-side CPU tests.  Every mutation must turn at least one test
red.  Usage: python tools/mutate_oracle.py [--out profiles/oracle_mutations.txt]
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = [
    ("sigma3 without -sum(x - x~)",
     "t[6] = fmax(t[6], fabs((S->s[c] - st[c]) - dx));",
     "t[6] = fmax(t[6], fabs(S->s[c] - st[c]));"),
    ("sigma1 scaled by rho2",
     "double s1 = rho[0] * t[4]", "double s1 = rho[1] * t[4]"),
    ("sigma h-term dropped",
     "s2 = rho[1] * t[5]", "s2 = 0.0 * t[5]"),
    ("r z-term dropped",
     "t[1] = fmax(t[1], fabs(S->z[e] - gfun(P, (long)e, S->x[e])));", ";"),
    ("x1 init = sum (not mean)",
     "S->x1[i] = buf[i] / (double)P->q_total;", "S->x1[i] = buf[i];"),
    ("h init without min(c, .)",
     "S->h[IJ(i, j)] = fmin(P->c[i], nsum_val(&a));", "S->h[IJ(i, j)] = nsum_val(&a);"),
    ("s init = 0",
     "S->s[JK(j, k)] = fmax(0.0, sx - P->y[JK(j, k)]);", "S->s[JK(j, k)] = 0.0;"),
    ("r consensus term dropped",
     "t[3] = fmax(t[3], fabs(S->x[IX(i, j, 0)] - S->x1[i]));", ";"),
    ("dual rescale of mu skipped",
     "for (size_t e = 0; e < NC; ++e) S->mu[e] *= f3;", ";"),
]

TESTS = ["tests/test_oracle_admm.py", "tests/test_oracle_residuals.py",
         "tests/test_oracle_quartic.py"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    lines = []
    tmp = tempfile.mkdtemp(prefix="orcmut_")
    try:
        for name, old, new in MUTATIONS:
            d = os.path.join(tmp, "repo")
            if os.path.exists(d):
                shutil.rmtree(d)
            shutil.copytree(ROOT, d, ignore=shutil.ignore_patterns(".git", "gpurun_out", "*.so",
                                                                   "__pycache__", ".pytest_cache"))
            src = os.path.join(d, "oracle", "oracle.c")
            s = open(src).read()
            assert s.count(old) == 1, f"mutation site not unique: {name}"
            open(src, "w").write(s.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                                "-m", "not gpu", *TESTS], cwd=d, capture_output=True, text=True)
            tail = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")][:1]
            verdict = "KILLED" if r.returncode != 0 else "SURVIVED"
            line = f"{verdict:8s} {name:32s} {tail[0] if tail else r.stdout.strip().splitlines()[-1]}"
            print(line, flush=True)
            lines.append(line)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write("# tools/mutate_oracle.py: each plausible oracle mistake vs the CPU pins\n")
            f.write("\n".join(lines) + "\n")
    return 0 if all(ln.startswith("KILLED") for ln in lines) else 1


if __name__ == "__main__":
    sys.exit(main())
