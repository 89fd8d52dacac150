"""Mutation check of the oracle's pins (test infrastructure, not product code): builds
scratch copies of oracle/kiops_oracle.c with one deliberate mistake each, runs the
CPU pin suites against each build (KIOPS_ORACLE_LIB) and reports which tests catch
it.  A mutation no test catches means an unpinned branch.
  python scripts/oracle_mutations.py > profiles/r02_oracle_mutations.txt"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "oracle", "kiops_oracle.c")).read()
MUTATIONS = {
    "Eq. 43 inverted as printed (log(tau/tau_old)/log(omega/omega_old))":
        ("const double o = log(om / omo) / log(tau / tau_old);", "const double o = log(tau / tau_old) / log(om / omo);"),
    "R4 floor ord >= 1 removed": ("ord = o > 1.0 ? o : 1.0;", "ord = o;"),
    "R4 fallback j/4 removed (non-positive estimates used)": ("if (isfinite(o) && o > 0.0)", "if (1)"),
    "R3 relative threshold 1e-12 -> 1e-11": ("(1e-12 * c > 1e-14) ? 1e-12 * c : 1e-14", "(1e-11 * c > 1e-14) ? 1e-11 * c : 1e-14"),
    "R3 absolute floor removed": ("(1e-12 * c > 1e-14) ? 1e-12 * c : 1e-14", "1e-12 * c"),
    "Eq. 45 exponent sign flipped": ("1.0 / (double)(j_old - j)", "1.0 / (double)(j - j_old)"),
    "Eq. 44 gamma_max 0.6 -> 0.9": ("gamma_max = 0.6", "gamma_max = 0.9"),
}
TESTS = ["tests/test_pins_controller.py", "tests/test_pins_iop.py"]
print("oracle mutation check: pin suites", " ".join(TESTS))
with tempfile.TemporaryDirectory() as d:
    for name, (a, b) in MUTATIONS.items():
        if a not in SRC:
            print(f"SKIP (pattern not found): {name}")
            continue
        src = os.path.join(d, "m.c")
        lib = os.path.join(d, f"m{abs(hash(name))}.so")
        open(src, "w").write(SRC.replace(a, b))
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-I", os.path.join(ROOT, "oracle"),
                               "-o", lib, src, "-lm"])
        env = dict(os.environ, KIOPS_ORACLE_LIB=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider"] + TESTS,
                           cwd=ROOT, env=env, capture_output=True, text=True)
        failed = sorted({ln.split("::")[1].split(" ")[0] for ln in r.stdout.splitlines() if ln.startswith("FAILED")})
        print(f"{'CAUGHT' if failed else 'MISSED'}: {name}: {', '.join(failed) or '-'}")
