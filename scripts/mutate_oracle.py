"""Mutation check of the oracle pins (VERDICT r1 'What's weak #1').

Each mutation is applied to a temporary copy of oracle/; the -m "not gpu" oracle tests run
against that copy and must FAIL.  Usage: python scripts/mutate_oracle.py"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MUTATIONS = {
    "transposed element moduli in local_problem":
        ("msfem.py", "E[ex * nely + ey] * K0", "E[ey * nelx + ex] * K0"),
    "D = I instead of diag(K_omega)":
        ("msfem.py", "return Kf, np.diag(Kf).copy()", "return Kf, np.ones(Kf.shape[0])"),
    "basis without chi":
        ("msfem.py", "v = chi * psi[:, a]", "v = psi[:, a]"),
    "swapped chi coordinates":
        ("msfem.py", "chi = partition_of_unity(I, J, dix, diy, cx, cy)",
         "chi = partition_of_unity(I, J, diy, dix, cx, cy)"),
    "coarse correction on r instead of r - Az":
        ("msfem.py", "z = z + self.coarse_correction(r - self.A @ z)",
         "z = z + self.coarse_correction(r)"),
}


def main():
    failed_to_catch = []
    for name, (fname, old, new) in MUTATIONS.items():
        tmp = tempfile.mkdtemp()
        for d in ("oracle", "tests", "workloads"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
        path = os.path.join(tmp, "oracle", fname)
        src = open(path).read()
        assert src.count(old) == 1, (name, old)
        open(path, "w").write(src.replace(old, new))
        env = dict(os.environ, PYTHONPATH=tmp)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                            "tests/test_oracle_msfem.py", "tests/test_oracle_fem.py"],
                           cwd=tmp, env=env, capture_output=True, text=True)
        caught = r.returncode != 0
        last = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
        print(f"{'caught ' if caught else 'MISSED '} {name}: {last[0] if last else ''}")
        if not caught:
            failed_to_catch.append(name)
        shutil.rmtree(tmp)
    sys.exit(1 if failed_to_catch else 0)


if __name__ == "__main__":
    main()
