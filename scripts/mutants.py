"""Mutation check of the oracle pins: apply one plausible
mistake at a time to a scratch copy of the repo and confirm that at least one
`-m "not gpu"` test fails.  Usage: python scripts/mutants.py [-k NAME]."""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, file, original, mutated)
MUTANTS = [
    ("energy_flux_vE", "oracle/physics.py", "(vn * (E + p),))", "(vn * E,))"),
    ("sound_speed_no_gamma", "oracle/physics.py", "ad.sqrt(eq.gamma * p / rho)", "ad.sqrt(p / rho)"),
    ("glf_half_lambda", "oracle/physics.py", "0.5 * (fl + fr) + lv * (l - r)", "0.5 * (fl + fr) + 0.5 * lv * (l - r)"),
    ("momentum_no_p", "oracle/physics.py", "mk * vn + (pe if k == d else 0.0)", "mk * vn"),
    ("pressure_no_half", "oracle/physics.py", "(E - 0.5 * e2 * ke / rho)", "(E - e2 * ke / rho)"),
    ("llf_lambda_min", "oracle/physics.py", "lam = ad.maxval(wave_speed(eq, wL, d), wave_speed(eq, wR, d))",
     "lam = wave_speed(eq, wL, d)"),
    ("viscous_div_factor", "oracle/physics.py", "txx = mu * (2.0 * ux - (2.0 / 3.0) * div)",
     "txx = mu * (2.0 * ux - (1.0 / 3.0) * div)"),
    ("heat_flux_dropped", "oracle/physics.py", "txx * u + txy * v + lam_T * Tx", "txx * u + txy * v"),
]


def run(name, rel, old, new, k):
    tmp = tempfile.mkdtemp(prefix="mut_")
    try:
        for d in ("oracle", "tests", "paper_2109_04804_b200"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("*.so", "build*", "csrc", "__pycache__"))
        p = os.path.join(tmp, rel)
        s = open(p).read()
        assert s.count(old) == 1, (name, old)
        open(p, "w").write(s.replace(old, new))
        args = [sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu and not slow", "-p", "no:cacheprovider",
                "tests/test_oracle_physics.py", "tests/test_oracle_dgsem.py", "tests/test_oracle_implicit.py"]
        if k:
            args += ["-k", k]
        r = subprocess.run(args, cwd=tmp, capture_output=True, text=True)
        failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
        return r.returncode != 0, failed[:3]
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default=None)
    a = ap.parse_args()
    ok = True
    for name, rel, old, new in MUTANTS:
        killed, failed = run(name, rel, old, new, a.k)
        ok &= killed
        print(f"{name:24s} {'KILLED' if killed else 'SURVIVED'}  {failed[:1]}")
    sys.exit(0 if ok else 1)
