"""Mutation probe of the oracle's pins (round-2 VERDICT item 2): apply one plausible mistake
at a time to a scratch copy of oracle/pvro.c, build it, and run the CPU pin suites against it
(PVRO_SO). Every mutant must fail at least one named pin.

  python tools/mutation_probe.py
"""
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "pvro.c")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_pins_geometry.py", "tests/test_oracle_registration.py"]

# (name, regex, replacement): each must match exactly once in pvro.c
MUTANTS = [
    ("psf steps h_u <-> h_w (sample_pos)",
     r"abc\[0\] \* st->h\[0\] \* st->u\[d\] \+ abc\[1\] \* st->h\[1\] \* st->v\[d\] \+ abc\[2\] \* st->h\[2\] \* st->w\[d\]",
     "abc[0] * st->h[2] * st->u[d] + abc[1] * st->h[1] * st->v[d] + abc[2] * st->h[0] * st->w[d]"),
    ("through-plane offsets along u instead of w",
     r"abc\[2\] \* st->h\[2\] \* st->w\[d\]", "abc[2] * st->h[2] * st->u[d]"),
    ("init fill over 6 instead of 26 neighbours",
     r"if \(!di && !dj && !dl\) continue;\n(\s+)int i2 = i \+ di",
     r"if (!di && !dj && !dl) continue;\n\1if (abs(di) + abs(dj) + abs(dl) != 1) continue;\n\1int i2 = i + di"),
    ("diffusivity b_d from X1 instead of X0",
     r"double g = \(X0\[k2\] - X0\[k\]\) / delta;", "double g = (X1[k2] - X1[k]) / delta;"),
    ("clamp range over all y instead of live y",
     r"if \(x->kappa\[j\] >= x->tau_live\) \{\n(\s+)double yv = pixel_y", r"if (1) {\n\1double yv = pixel_y"),
]


def main():
    src = open(SRC).read()
    bad = 0
    for name, pat, rep in MUTANTS:
        mut, n = re.subn(pat, rep, src)
        if n != 1:
            print(f"[probe] {name}: pattern matched {n} times (fix the probe)")
            bad += 1
            continue
        with tempfile.TemporaryDirectory() as d:
            c = os.path.join(d, "pvro.c")
            open(c, "w").write(mut)
            subprocess.check_call(["cp", os.path.join(ROOT, "oracle", "pvro.h"), d])
            so = os.path.join(d, "libpvro_mut.so")
            subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", "-o", so, c, "-lm"])
            env = dict(os.environ, PVRO_SO=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:randomly"] + PINS,
                               cwd=ROOT, env=env, capture_output=True, text=True)
            failed = re.findall(r"^FAILED (\S+)", r.stdout, re.M)
            if r.returncode == 0 or not failed:
                print(f"[probe] {name}: SURVIVED (all pins pass)")
                bad += 1
            else:
                print(f"[probe] {name}: caught by {len(failed)} pin(s), e.g. {failed[0]}")
    print(f"[probe] {len(MUTANTS) - bad}/{len(MUTANTS)} mutants caught")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
