"""Mutation check of the oracle's pins (VERDICT r1 "Next round" 1).

Each mutation permutes the per-node weights of one U-independent load term
inside a scratch copy of oracle/fo_oracle.cpp -- the kind of mistake the
totals-only pins (P4, P6) cannot see -- rebuilds it there and runs the CPU pin
suites against it.  A mutation counts as caught when at least one pin fails;
the unmutated copy must pass.  Run:  python tools/mutate_oracle.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_pins_next.py",
        "tests/test_oracle_pins_pernode.py"]

# (name, [(old, new, occurrence index)]); occurrence 0 = wedge / tet element,
# 1 = hexahedral element (the same source lines appear in both)
ROT6 = "N[(i % 3 + 1) % 3 + 3 * (i / 3)]"
ROT8 = "N[(i % 4 + 1) % 4 + 4 * (i / 4)]"
MUTATIONS = [
    ("wedge driving stress: node weights rotated (R and the energy alike)", [
        ("r[2 * i] += promote<T>(W * rg * sx * N[i]);", f"r[2 * i] += promote<T>(W * rg * sx * {ROT6});", 0),
        ("r[2 * i + 1] += promote<T>(W * rg * sy * N[i]);", f"r[2 * i + 1] += promote<T>(W * rg * sy * {ROT6});", 0),
        ("u += Ul[2 * i] * N[i]; v += Ul[2 * i + 1] * N[i];",
         f"u += Ul[2 * i] * {ROT6}; v += Ul[2 * i + 1] * {ROT6};", 0),
    ]),
    ("wedge basal beta: P1 vertex weights rotated", [
        ("double b = Lt[0] * e.beta[0] + Lt[1] * e.beta[1] + Lt[2] * e.beta[2];",
         "double b = Lt[1] * e.beta[0] + Lt[2] * e.beta[1] + Lt[0] * e.beta[2];", 0),
    ]),
    ("hex driving stress: node weights rotated (R and the energy alike)", [
        ("r[2 * i] += promote<T>(W * rg * sx * N[i]);", f"r[2 * i] += promote<T>(W * rg * sx * {ROT8});", 1),
        ("r[2 * i + 1] += promote<T>(W * rg * sy * N[i]);", f"r[2 * i + 1] += promote<T>(W * rg * sy * {ROT8});", 1),
        ("u += Ul[2 * i] * N[i]; v += Ul[2 * i + 1] * N[i];",
         f"u += Ul[2 * i] * {ROT8}; v += Ul[2 * i + 1] * {ROT8};", 1),
    ]),
    ("hex basal beta: bilinear vertex weights rotated", [
        ("b += Q[j] * e.beta[j];", "b += Q[(j + 1) % 4] * e.beta[j];", 0),
    ]),
]


def _replace_nth(src, old, new, n):
    i = -1
    for _ in range(n + 1):
        i = src.find(old, i + 1)
        if i < 0:
            raise SystemExit(f"mutation anchor not found (occurrence {n}): {old}")
    return src[:i] + new + src[i + len(old):]


def _scratch(tmp):
    shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(tmp, "oracle"),
                    ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    os.makedirs(os.path.join(tmp, "paper_2204_04321_b200"))
    for f in ("__init__.py", "meshgen.py"):
        shutil.copy(os.path.join(ROOT, "paper_2204_04321_b200", f), os.path.join(tmp, "paper_2204_04321_b200"))
    os.makedirs(os.path.join(tmp, "tests"))
    for f in ["tests/conftest.py"] + PINS:
        shutil.copy(os.path.join(ROOT, f), os.path.join(tmp, f))
    for d in ("tests/golden",):
        if os.path.isdir(os.path.join(ROOT, d)):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d))


def _run(tmp):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider"] + PINS,
                       cwd=tmp, capture_output=True, text=True)
    failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
    return r.returncode, failed, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""


def main():
    ok = True
    with tempfile.TemporaryDirectory() as tmp:
        _scratch(tmp)
        rc, failed, tail = _run(tmp)
        print(f"control (unmutated): rc={rc} {tail}")
        ok &= rc == 0
        src0 = open(os.path.join(tmp, "oracle", "fo_oracle.cpp")).read()
        for name, edits in MUTATIONS:
            src = src0
            for old, new, n in edits:
                src = _replace_nth(src, old, new, n)
            open(os.path.join(tmp, "oracle", "fo_oracle.cpp"), "w").write(src)
            lib = os.path.join(tmp, "oracle", "liboracle.so")
            if os.path.exists(lib):
                os.remove(lib)
            rc, failed, tail = _run(tmp)
            caught = rc != 0
            ok &= caught
            print(f"{'CAUGHT ' if caught else 'MISSED '} {name}: {tail}; failing pins: "
                  f"{", ".join(failed) if failed else "-"}")
        open(os.path.join(tmp, "oracle", "fo_oracle.cpp"), "w").write(src0)
    print("all mutations caught" if ok else "SOME MUTATION WAS NOT CAUGHT")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
