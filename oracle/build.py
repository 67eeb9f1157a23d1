"""Build the oracle's C helper (host row regeneration) -- test infrastructure.

gcc -O2 -fPIC -shared -ffp-contract=off -mfma -fopenmp -I include
    oracle/gen_rows.c -o oracle/_build/libgenrows.so -lm
"""

import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
SRC = HERE / "gen_rows.c"
OUT = HERE / "_build" / "libgenrows.so"
DEPS = [SRC, ROOT / "include" / "ksvd_gen.h", Path(__file__)]


def build(force: bool = False) -> Path:
    if not force and OUT.exists() and all(d.stat().st_mtime <= OUT.stat().st_mtime for d in DEPS):
        return OUT
    OUT.parent.mkdir(exist_ok=True)
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-mfma", "-fopenmp",
           f"-I{ROOT / 'include'}", str(SRC), "-o", str(OUT), "-lm"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode:
        raise RuntimeError(f"gcc failed:\n{res.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
