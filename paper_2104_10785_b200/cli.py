"""`krysvd`-compatible command line for the GK path (reference cli.py).

Verbs gen, rank, svd, compare, triplets -- same flags, defaults, CSV/TSV/JSON
schemas, embedded `# config:` replay lines and exit codes (0 ok, 2
ConfigError or bad flags, 3 NumericalError) as the reference, so tables from
this package and from the reference/oracle diff line by line once the
"seconds" columns are stripped.  `rsl` (the similarity-learning trainer) is
out of scope.

`gen --kind harmonic|exp|geom` is the on-device seeded generator
(ksvd_matrix_generate) streamed to a KLRM snapshot by
ksvd_matrix_to_klrm -- it makes the BASELINE configs 3-5 matrices without a
host copy; `lowrank` / `gaussian` are the reference's host generators, bit
for bit.

Run as `python -m paper_2104_10785_b200.cli <verb> ...`.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import sys
from pathlib import Path

import numpy as np

from . import harness
from .errors import ConfigError, NumericalError
from .linops import BENCH_MATRIX, derive_seed
from .matrixio import read_csv_matrix, read_matrix, write_matrix

FORMATS = ("csv", "json", "tsv")
DEVICE_KINDS = ("harmonic", "exp", "geom")


# ---------------------------------------------------------------------------
# output artifacts (reference cli.py:27-107)

def to_jsonable(obj):
    """numpy scalars/arrays -> plain JSON types, recursively."""
    if isinstance(obj, dict):
        return {k: to_jsonable(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [to_jsonable(v) for v in obj]
    if isinstance(obj, np.ndarray):
        return to_jsonable(obj.tolist())
    if isinstance(obj, np.generic):
        return obj.item()
    return obj


def _cell(v) -> str:
    """Table cell text: NA for missing, true/false, repr for floats."""
    if v is None:
        return "NA"
    if v is True or v is False:
        return "true" if v else "false"
    return repr(v) if isinstance(v, float) else str(v)


def _compact(obj) -> str:
    return json.dumps(obj, separators=(",", ":"))


def render(payload: dict, fmt: str) -> str:
    """payload keys: command, params, columns, records, sections (optional)."""
    payload = to_jsonable(payload)
    config = {"command": payload["command"], "schema": harness.SCHEMA_VERSION,
              "params": payload["params"]}
    sections = payload.get("sections", {})
    if fmt == "json":
        return json.dumps({"config": config, "records": payload["records"], **sections},
                          indent=2) + "\n"
    sep = "\t" if fmt == "tsv" else ","
    out = [f"# config: {_compact(config)}"]
    out += [f"# {name}: {_compact(body)}" for name, body in sections.items()]
    out.append(sep.join(payload["columns"]))
    out += [sep.join(_cell(rec.get(c)) for c in payload["columns"])
            for rec in payload["records"]]
    return "\n".join(out) + "\n"


def write_output(payload: dict, out, fmt: str) -> None:
    text = render(payload, fmt)
    if out is None:
        sys.stdout.write(text)
    else:
        Path(out).write_text(text)


def read_embedded_config(path) -> dict:
    """The effective configuration embedded in an output artifact."""
    text = Path(path).read_text()
    if text.lstrip().startswith("{"):
        return json.loads(text)["config"]
    tag = "# config: "
    found = [ln[len(tag):] for ln in text.splitlines() if ln.startswith(tag)]
    if not found:
        raise ConfigError(f"no embedded config found in {path}")
    return json.loads(found[0])


def argv_from_config(config: dict) -> list[str]:
    """argv that replays the run an embedded config describes."""
    argv = [config["command"]]
    for key, val in config["params"].items():
        if val is None:
            continue
        flag = "--" + key.replace("_", "-")
        if isinstance(val, bool):
            argv.append(flag if val else "--no-" + flag[2:])
        else:
            argv += [flag, str(val)]
    return argv


# ---------------------------------------------------------------------------
# parser (reference cli.py:110-210, minus rsl)

_COMMON = [
    ("--seed", dict(type=int, default=0)),
    ("--repeats", dict(type=int, default=3, help="timed repetitions after one discarded warm-up")),
    ("--out", dict(default=None, help="output path (default stdout)")),
    ("--format", dict(dest="fmt", choices=FORMATS, default="csv")),
    ("--max-elems", dict(type=float, default=1e8,
                         help="refuse matrices with more entries than this")),
]
_RSVD_KNOBS = [("--power-iters", dict(type=int, default=0)),
               ("--oversampling", dict(type=int, default=None))]

_VERBS = {
    "gen": ("write a synthetic test matrix", [
        ("--size", dict(required=True, help="MxN, e.g. 1000x1000")),
        ("--kind", dict(choices=("lowrank", "gaussian") + DEVICE_KINDS, default="lowrank",
                        help="lowrank/gaussian: reference host generators; harmonic/exp/"
                             "geom: on-device P diag(s) Q^T + noise")),
        ("--rank-true", dict(type=int, default=100, help="factor rank")),
        ("--mean", dict(type=float, default=0.0)),
        ("--std", dict(type=float, default=1.0)),
        ("--s0", dict(type=float, default=1.0, help="device kinds: leading singular value")),
        ("--p", dict(type=float, default=0.0, help="device kinds: decay parameter")),
        ("--noise", dict(type=float, default=0.0, help="device kinds: noise scale")),
        ("--dtype", dict(choices=("f64", "f32"), default="f64",
                         help="device kinds: storage before the f64 snapshot")),
    ]),
    "rank": ("estimate numerical rank", [
        ("--sizes", dict(default=None, help="comma list of MxN")),
        ("--rank-true", dict(type=int, default=100)),
        ("--input", dict(default=None, help="matrix file (.klrm or .csv)")),
        ("--eps", dict(type=float, default=1e-8)),
        ("--mode", dict(choices=("absolute", "relative"), default="absolute")),
        ("--with-oracle", dict(action=argparse.BooleanOptionalAction, default=True,
                               help="also time a dense-SVD rank count")),
    ]),
    "svd": ("run one factorization method on one matrix", [
        ("--size", dict(default=None, help="MxN for a synthetic matrix")),
        ("--input", dict(default=None, help="matrix file (.klrm or .csv)")),
        ("--rank-true", dict(type=int, default=None)),
        ("--method", dict(choices=harness.METHODS, default="fsvd")),
        ("--r", dict(type=int, required=True, help="triplets to extract")),
        ("--k", dict(type=int, default=None, help="iteration budget (default min(m,n))")),
    ] + _RSVD_KNOBS),
    "compare": ("methods x sizes timing/accuracy table", [
        ("--sizes", dict(default="1000x1000")),
        ("--rank-true", dict(type=int, default=100)),
        ("--r", dict(type=int, default=20)),
        ("--methods", dict(default=",".join(harness.GPU_METHODS))),
    ] + _RSVD_KNOBS),
    "triplets": ("per-direction agreement with the dense oracle", [
        ("--size", dict(default="500x400")),
        ("--rank-true", dict(type=int, default=50)),
        ("--r", dict(type=int, default=20)),
        ("--methods", dict(default=",".join(harness.GPU_METHODS))),
    ] + _RSVD_KNOBS),
}


def build_parser() -> argparse.ArgumentParser:
    top = argparse.ArgumentParser(
        prog="krysvd", description="GPU Golub-Kahan partial SVD / rank toolkit")
    sub = top.add_subparsers(dest="command", required=True)
    for verb, (helptext, flags) in _VERBS.items():
        p = sub.add_parser(verb, help=helptext)
        for flag, kw in _COMMON + flags:
            p.add_argument(flag, **kw)
    return top


# ---------------------------------------------------------------------------
# verbs

def _items(text: str) -> list[str]:
    return [t for t in text.split(",") if t]


def _sizes(text: str) -> list[tuple[int, int]]:
    return [harness.parse_size(t) for t in _items(text)]


def load_matrix(path) -> np.ndarray:
    p = Path(path)
    if not p.exists():
        raise ConfigError(f"input file not found: {p}")
    A = read_csv_matrix(p) if p.suffix.lower() == ".csv" else read_matrix(p)
    if not np.isfinite(A).all():
        raise NumericalError(f"input matrix {p} contains NaN or Inf entries")
    return A


def _gen(a):
    if a.out is None:
        raise ConfigError("gen writes a matrix file and requires --out")
    m, n = harness.parse_size(a.size)
    if m * n > a.max_elems:
        raise ConfigError(f"size {m}x{n} exceeds the element cap {a.max_elems:g}")
    if a.kind in DEVICE_KINDS:
        from . import synth
        from .matrixio import write_matrix_device
        spec = synth.GenSpec(m=m, n=n, rank=a.rank_true, seed=a.seed, spectrum=a.kind,
                             s0=a.s0, p=a.p, noise=a.noise, dtype=a.dtype)
        write_matrix_device(a.out, synth.generate(spec))
    else:
        mseed = derive_seed(a.seed, BENCH_MATRIX, 0)
        if a.kind == "lowrank":
            A = harness.low_rank_synth(m, n, a.rank_true, seed=mseed)
        else:
            from .synth import gaussian_matrix
            A = gaussian_matrix(m, n, mean=a.mean, std=a.std, seed=mseed)
        write_matrix(a.out, A)
    print(f"wrote {a.out}: {m}x{n} kind={a.kind} seed={a.seed}")
    return None


def _rank(a):
    params = {"eps": a.eps, "mode": a.mode, "with_oracle": a.with_oracle, "seed": a.seed,
              "repeats": a.repeats, "max_elems": a.max_elems, "format": a.fmt}
    if a.input is not None:
        A = load_matrix(a.input)
        if A.size > a.max_elems:
            raise ConfigError(f"input exceeds the element cap {a.max_elems:g}")
        rows = [harness.rank_report_for_matrix(A, eps=a.eps, mode=a.mode, seed=a.seed,
                                               repeats=a.repeats, with_oracle=a.with_oracle)]
        params["input"] = str(a.input)
    elif a.sizes is not None:
        rows = harness.cmd_rank(_sizes(a.sizes), a.rank_true, eps=a.eps, mode=a.mode,
                                repeats=a.repeats, seed=a.seed, with_oracle=a.with_oracle,
                                max_elems=a.max_elems)
        params.update(sizes=a.sizes, rank_true=a.rank_true)
    else:
        raise ConfigError("rank needs --sizes or --input")
    cols = ["m", "n", "rank_true", "rank", "k_prime", "eps", "mode", "threshold", "seconds",
            "seconds_mean", "oracle_rank", "oracle_seconds", "seed"]
    return {"command": "rank", "params": params, "columns": cols, "records": rows}


def _svd(a):
    params = {"method": a.method, "r": a.r, "k": a.k, "rank_true": a.rank_true,
              "power_iters": a.power_iters, "oversampling": a.oversampling, "seed": a.seed,
              "repeats": a.repeats, "max_elems": a.max_elems, "format": a.fmt}
    if (a.size is None) == (a.input is None):
        raise ConfigError("svd needs exactly one of --size or --input")
    if a.input is not None:
        A = load_matrix(a.input)
        params["input"] = str(a.input)
    else:
        m, n = harness.parse_size(a.size)
        if m * n > a.max_elems:
            raise ConfigError(f"size {m}x{n} exceeds the element cap {a.max_elems:g}")
        rt = a.rank_true if a.rank_true is not None else min(100, m, n)
        A = harness.low_rank_synth(m, n, rt, seed=derive_seed(a.seed, BENCH_MATRIX, 0))
        params.update(size=a.size, rank_true=rt)
    rows, summary = harness.cmd_svd(A, a.method, a.r, rank_true=params["rank_true"], k=a.k,
                                    repeats=a.repeats, seed=a.seed,
                                    power_iters=a.power_iters, oversampling=a.oversampling,
                                    max_elems=a.max_elems)
    return {"command": "svd", "params": params, "columns": ["index", "sigma"],
            "records": rows, "sections": {"summary": summary}}


def _compare(a):
    params = {"sizes": a.sizes, "rank_true": a.rank_true, "r": a.r, "methods": a.methods,
              "power_iters": a.power_iters, "oversampling": a.oversampling, "seed": a.seed,
              "repeats": a.repeats, "max_elems": a.max_elems, "format": a.fmt}
    recs = harness.cmd_compare(_sizes(a.sizes), a.rank_true, a.r, _items(a.methods),
                               repeats=a.repeats, seed=a.seed, max_elems=a.max_elems,
                               power_iters=a.power_iters, oversampling=a.oversampling)
    return {"command": "compare", "params": params,
            "columns": [f.name for f in dataclasses.fields(harness.BenchRecord)],
            "records": [dataclasses.asdict(r) for r in recs]}


def _triplets(a):
    params = {"size": a.size, "rank_true": a.rank_true, "r": a.r, "methods": a.methods,
              "power_iters": a.power_iters, "oversampling": a.oversampling, "seed": a.seed,
              "max_elems": a.max_elems, "format": a.fmt}
    m, n = harness.parse_size(a.size)
    if m * n > a.max_elems:
        raise ConfigError(f"size {m}x{n} exceeds the element cap {a.max_elems:g}")
    quals = harness.cmd_triplet_quality(m, n, a.rank_true, a.r, _items(a.methods),
                                        seed=a.seed, power_iters=a.power_iters,
                                        oversampling=a.oversampling)
    rows = [{"method": t.method, "index": i + 1, "q": float(t.q[i]),
             "sigma_oracle": float(t.sigma_oracle[i]), "sigma_method": float(t.sigma_method[i])}
            for t in quals for i in range(len(t.q))]
    return {"command": "triplets", "params": params,
            "columns": ["method", "index", "q", "sigma_oracle", "sigma_method"], "records": rows}


HANDLERS = {"gen": _gen, "rank": _rank, "svd": _svd, "compare": _compare,
            "triplets": _triplets}


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:  # argparse: 2 on bad flags, 0 on --help
        return int(exc.code or 0)
    try:
        payload = HANDLERS[args.command](args)
    except (ConfigError, NumericalError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2 if isinstance(exc, ConfigError) else 3
    if payload is not None:
        write_output(payload, args.out, args.fmt)
    return 0


if __name__ == "__main__":
    sys.exit(main())
