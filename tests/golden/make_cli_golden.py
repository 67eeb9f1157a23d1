"""Regenerate tests/golden/cli/*.csv by running the REFERENCE command line
(/root/reference/pkg, importable in the build container only) and stripping
the timing columns.  The GPU CLI tests replay each artifact's embedded
config through this package's CLI and diff the tables line by line.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py
"""

import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from krysvd.cli import main  # noqa: E402  (the reference)

from tests.cli_tables import strip_timing  # noqa: E402

CASES = {
    "rank_abs": ["rank", "--sizes", "120x100,200x150", "--rank-true", "20", "--repeats", "1",
                 "--seed", "3"],
    "rank_rel": ["rank", "--sizes", "300x200", "--rank-true", "40", "--eps", "1e-6",
                 "--mode", "relative", "--repeats", "1", "--seed", "5"],
    "rank_wide": ["rank", "--sizes", "90x240", "--rank-true", "30", "--repeats", "1",
                  "--seed", "8", "--no-with-oracle"],
    "svd_lowrank": ["svd", "--size", "100x80", "--rank-true", "15", "--r", "10",
                    "--repeats", "1", "--seed", "4"],
    "svd_budget": ["svd", "--size", "150x120", "--rank-true", "50", "--r", "8", "--k", "30",
                   "--repeats", "1", "--seed", "6"],
    "svd_dense": ["svd", "--size", "70x50", "--rank-true", "12", "--r", "6", "--method",
                  "dense", "--repeats", "1", "--seed", "2"],
    "compare": ["compare", "--sizes", "120x100,80x90", "--rank-true", "20", "--r", "5",
                "--methods", "fsvd,dense", "--repeats", "1", "--seed", "3"],
    "triplets": ["triplets", "--size", "60x50", "--rank-true", "10", "--r", "5",
                 "--methods", "dense,fsvd", "--seed", "5"],
}

if __name__ == "__main__":
    out_dir = Path(__file__).resolve().parent / "cli"
    out_dir.mkdir(exist_ok=True)
    with tempfile.TemporaryDirectory() as d:
        for name, argv in CASES.items():
            tmp = Path(d) / f"{name}.csv"
            assert main(argv + ["--out", str(tmp)]) == 0, name
            (out_dir / f"{name}.csv").write_text(strip_timing(tmp.read_text()) + "\n")
            print("wrote", name)
