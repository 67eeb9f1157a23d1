"""CLI host logic (no GPU): artifact rendering conventions, parsers, schema
pins against the reference's golden tables, replay plumbing, host `gen`
bits, and the exit codes of errors raised before any device work
(reference tests/test_bench_cli.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import harness
from paper_2104_10785_b200.cli import (_cell, argv_from_config, build_parser, main,
                                       read_embedded_config, render)
from paper_2104_10785_b200.linops import BENCH_MATRIX, derive_seed
from paper_2104_10785_b200.synth import gaussian_matrix, low_rank_synth
from tests.cli_tables import rows_of, same_value, sections_of, strip_timing

GOLDEN = Path(__file__).resolve().parent / "golden" / "cli"
COMPARE_HEADER = ("method,m,n,rank_true,r_extracted,k_used,seconds,"
                  "seconds_mean,err_res,err_res_full,err_rel,rank_estimated,seed")
RANK_HEADER = ("m,n,rank_true,rank,k_prime,eps,mode,threshold,seconds,seconds_mean,"
               "oracle_rank,oracle_seconds,seed")


def test_cell_conventions():
    assert [_cell(v) for v in (None, True, False, 5, 0.1, 1e-8, "fsvd")] == \
        ["NA", "true", "false", "5", "0.1", "1e-08", "fsvd"]


def test_render_csv_tsv_json():
    payload = {"command": "demo", "params": {"a": 1}, "columns": ["x", "y"],
               "records": [{"x": 1, "y": None}, {"x": np.int64(2), "y": np.float64(0.5)}],
               "sections": {"summary": {"n": np.int64(3)}}}
    lines = render(payload, "csv").strip().split("\n")
    assert json.loads(lines[0][len("# config: "):]) == \
        {"command": "demo", "schema": harness.SCHEMA_VERSION, "params": {"a": 1}}
    assert lines[1] == '# summary: {"n":3}'
    assert lines[2:] == ["x,y", "1,NA", "2,0.5"]
    assert render(payload, "tsv").strip().split("\n")[2] == "x\ty"
    doc = json.loads(render(payload, "json"))
    assert doc["records"] == [{"x": 1, "y": None}, {"x": 2, "y": 0.5}]
    assert doc["summary"] == {"n": 3} and doc["config"]["command"] == "demo"


def test_parse_size():
    assert harness.parse_size("1000x500") == (1000, 500)
    assert harness.parse_size("16X8") == (16, 8)
    for bad in ("abc", "1x2x3", "ax3"):
        with pytest.raises(K.ConfigError):
            harness.parse_size(bad)


def test_derive_seed_matches_reference_stream_rule():
    seq = np.random.SeedSequence(entropy=3, spawn_key=(BENCH_MATRIX, 0))
    assert derive_seed(3, BENCH_MATRIX, 0) == int(seq.generate_state(1, dtype=np.uint64)[0])


@pytest.mark.parametrize("path", sorted(GOLDEN.glob("*.csv")), ids=lambda p: p.stem)
def test_golden_tables_use_our_schema_and_replay(path):
    """Every reference artifact's columns are the ones this CLI emits, and
    its embedded config parses back into our parser unchanged."""
    cfg = read_embedded_config(path)
    cols, _ = rows_of(path.read_text())
    want = {"rank": RANK_HEADER, "compare": COMPARE_HEADER, "svd": "index,sigma",
            "triplets": "method,index,q,sigma_oracle,sigma_method"}[cfg["command"]]
    assert cols == [c for c in want.split(",") if "seconds" not in c]
    args = build_parser().parse_args(argv_from_config(cfg))
    for key, val in cfg["params"].items():
        got = getattr(args, "fmt" if key == "format" else key)
        assert got == val or (val is None and got is None), (key, got, val)


def test_replay_flags_for_booleans(tmp_path):
    cfg = {"command": "rank", "params": {"with_oracle": False, "eps": 1e-8, "input": None}}
    assert argv_from_config(cfg) == ["rank", "--no-with-oracle", "--eps", "1e-08"]
    p = tmp_path / "plain.csv"
    p.write_text("a,b\n1,2\n")
    with pytest.raises(K.ConfigError):
        read_embedded_config(p)


def test_gen_host_kinds_write_reference_bits(tmp_path):
    out = tmp_path / "m.klrm"
    assert main(["gen", "--size", "80x60", "--rank-true", "12", "--seed", "3",
                 "--out", str(out)]) == 0
    assert np.array_equal(K.read_matrix(out),
                          low_rank_synth(80, 60, 12, seed=derive_seed(3, BENCH_MATRIX, 0)))
    assert main(["gen", "--size", "7x5", "--kind", "gaussian", "--mean", "1", "--std", "2",
                 "--seed", "1", "--out", str(out)]) == 0
    assert np.array_equal(K.read_matrix(out), gaussian_matrix(
        7, 5, mean=1.0, std=2.0, seed=derive_seed(1, BENCH_MATRIX, 0)))


def test_exit_codes_before_device_work(tmp_path):
    assert main(["gen", "--size", "10x10"]) == 2                      # needs --out
    assert main(["gen", "--size", "10x10", "--max-elems", "50",
                 "--out", str(tmp_path / "x")]) == 2                   # element cap
    assert main(["rank", "--out", str(tmp_path / "o.csv")]) == 2        # no source
    assert main(["rank", "--input", str(tmp_path / "nope.klrm")]) == 2  # missing file
    bad = tmp_path / "bad.klrm"
    A = np.ones((4, 3))
    A[1, 2] = np.nan
    K.write_matrix(bad, A)
    assert main(["rank", "--input", str(bad)]) == 3                     # NaN input
    assert main(["svd", "--r", "2"]) == 2                               # size xor input
    assert main(["svd", "--size", "10x10", "--r", "2", "--method", "qr"]) == 2
    assert main(["svd", "--size", "10x10", "--r", "2", "--method", "rsvd-default",
                 "--out", str(tmp_path / "o.csv")]) == 2               # out of scope
    assert main(["compare", "--sizes", "120x100", "--rank-true", "5", "--r", "2",
                 "--max-elems", "100"]) == 2
    assert main(["triplets", "--size", "2000x2000", "--rank-true", "10", "--r", "5"]) == 2
    assert main(["rsl"]) == 2                                           # not provided


def test_table_tolerance_rules():
    assert same_value("k_used", "21", "22") and not same_value("k_used", "21", "24")
    assert same_value("err_rel", "3e-16", "7e-16") and not same_value("err_rel", "1e-3", "7e-16")
    assert same_value("sigma", "1.0000000000001", "1.0")
    assert not same_value("rank", "20", "21") and same_value("oracle_rank", "NA", "NA")
    text = (GOLDEN / "svd_lowrank.csv").read_text()
    assert strip_timing(text) == text.strip()
    assert sections_of(text)["summary"]["rank_estimated"] == 15
