"""The CLI on the GPU path against the reference's own tables: each golden
artifact (tests/golden/make_cli_golden.py ran the reference CLI) is replayed
from its embedded config through this package and diffed line by line
(tests/cli_tables.py tolerances); plus file inputs, replay determinism and
the on-device `gen` kinds."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from oracle import krylov_oracle as O
from paper_2104_10785_b200 import synth
from paper_2104_10785_b200.cli import argv_from_config, main, read_embedded_config
from tests.cli_tables import diff_tables, rows_of, sections_of, strip_timing

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden" / "cli"


def _run(argv, out):
    code = main(argv + ["--out", str(out)])
    return code, (Path(out).read_text() if Path(out).exists() else "")


@pytest.mark.parametrize("path", sorted(GOLDEN.glob("*.csv")), ids=lambda p: p.stem)
def test_replay_matches_reference_table(path, tmp_path):
    argv = argv_from_config(read_embedded_config(path))
    code, text = _run(argv, tmp_path / "ours.csv")
    assert code == 0
    problems = diff_tables(strip_timing(text), path.read_text())
    assert not problems, "\n".join(problems[:20])


def test_rerun_identical_after_timing_strip(tmp_path):
    argv = argv_from_config(read_embedded_config(GOLDEN / "compare.csv"))
    _, a = _run(argv, tmp_path / "a.csv")
    _, b = _run(argv, tmp_path / "b.csv")
    assert strip_timing(a) == strip_timing(b)
    _, j = _run(argv[:-2] + ["--format", "json"], tmp_path / "c.json")
    doc = json.loads(j)
    assert doc["config"]["command"] == "compare" and len(doc["records"]) == 4
    assert doc["records"][1]["rank_estimated"] is None


def test_rank_file_input_matches_memory(tmp_path):
    mat = tmp_path / "m.klrm"
    assert main(["gen", "--size", "80x60", "--rank-true", "12", "--seed", "3",
                 "--out", str(mat)]) == 0
    code, text = _run(["rank", "--input", str(mat), "--repeats", "1", "--seed", "3"],
                      tmp_path / "r.csv")
    assert code == 0
    row = rows_of(text)[1][0]
    assert (row["rank"], row["oracle_rank"], row["rank_true"]) == ("12", "12", "NA")
    csvm = tmp_path / "m.csv"
    np.savetxt(csvm, np.diag([5.0, 3.0, 1.0]), delimiter=",")
    code, text = _run(["svd", "--input", str(csvm), "--r", "2", "--repeats", "1"],
                      tmp_path / "s.csv")
    assert code == 0
    assert [float(r["sigma"]) for r in rows_of(text)[1]] == pytest.approx([5.0, 3.0], rel=1e-12)
    assert sections_of(text)["summary"]["rank_estimated"] == 3


@pytest.mark.parametrize("kind,p,dtype", [("harmonic", 0.0, "f64"), ("exp", 4.0, "f32"),
                                          ("geom", 3.0, "f64")])
def test_device_gen_kinds(tmp_path, kind, p, dtype):
    """gen on the device writes the same matrix synth.generate holds in HBM,
    and the rank verb recovers the planted rank from the snapshot."""
    out = tmp_path / "g.klrm"
    assert main(["gen", "--size", "3000x400", "--kind", kind, "--rank-true", "25",
                 "--s0", "10", "--p", str(p), "--dtype", dtype, "--seed", "7",
                 "--out", str(out)]) == 0
    spec = synth.GenSpec(m=3000, n=400, rank=25, seed=7, spectrum=kind, s0=10.0, p=p,
                         dtype=dtype)
    A = K.read_matrix(out)
    assert np.array_equal(A, synth.generate(spec).to_dense().astype(np.float64))
    rel = O.rank_oracle(A, eps=1e-4, mode="relative")
    assert rel.rank == 25
    code, text = _run(["rank", "--input", str(out), "--eps", "1e-4", "--mode", "relative",
                       "--repeats", "1", "--no-with-oracle"], tmp_path / "r.csv")
    assert code == 0 and rows_of(text)[1][0]["rank"] == str(rel.rank)
