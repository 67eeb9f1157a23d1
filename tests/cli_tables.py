"""Helpers for CLI artifacts: drop timing fields, split tables into rows."""

import json


def _scrub(doc):
    if isinstance(doc, dict):
        return {k: _scrub(v) for k, v in doc.items() if "seconds" not in k}
    if isinstance(doc, list):
        return [_scrub(v) for v in doc]
    return doc


def strip_timing(text: str, sep: str = ",") -> str:
    """Remove every column / embedded field whose name mentions seconds."""
    meta, table = [], []
    for ln in text.strip().split("\n"):
        if ln.startswith("# ") and not table:
            tag, _, body = ln[2:].partition(": ")
            meta.append(f"# {tag}: " + json.dumps(_scrub(json.loads(body)),
                                                  separators=(",", ":")))
        else:
            table.append(ln.split(sep))
    keep = [i for i, c in enumerate(table[0]) if "seconds" not in c]
    return "\n".join(meta + [sep.join(r[i] for i in keep) for r in table])


def sections_of(text: str) -> dict:
    out = {}
    for ln in text.strip().split("\n"):
        if ln.startswith("# "):
            tag, _, body = ln[2:].partition(": ")
            out[tag] = json.loads(body)
    return out


def rows_of(text: str, sep: str = ","):
    lines = [ln for ln in text.strip().split("\n") if not ln.startswith("#")]
    cols = lines[0].split(sep)
    return cols, [dict(zip(cols, ln.split(sep))) for ln in lines[1:]]


# Column tolerance classes for comparing this package's tables with the
# reference's (values are Krylov outputs: rounding-stable to ~1e-13, see
# SURVEY.md 8(c) probe 1; k' past the numerical rank is not reproducible,
# probe 5, so k_used / k_prime get a slack of 2).
_REL = {"sigma", "sigma_oracle", "sigma_method", "threshold", "eps"}
_KSLACK = {"k_used", "k_prime"}
_ERR = {"err_rel", "err_res", "err_res_full"}
_FLOOR = 1e-9


def _num(s):
    if s in ("NA", None):
        return None
    try:
        return int(s)
    except (TypeError, ValueError):
        pass
    try:
        return float(s)
    except (TypeError, ValueError):
        return s


def same_value(col, ours, ref) -> bool:
    a, b = _num(ours) if isinstance(ours, str) else ours, _num(ref) if isinstance(ref, str) else ref
    if a is None or b is None:
        return a is None and b is None
    if col in _KSLACK:
        return abs(a - b) <= 2
    if col in _ERR:
        if abs(b) < _FLOOR:
            return abs(a) < _FLOOR
        return abs(a - b) <= 1e-6 * abs(b)
    if col in _REL:
        return abs(a - b) <= 1e-10 * max(abs(b), 1e-300)
    if col == "q":
        return abs(a - b) <= 1e-8
    if isinstance(b, float) or isinstance(a, float):
        return abs(a - b) <= 1e-12 * max(abs(b), 1.0)
    return a == b


def diff_tables(ours: str, ref: str) -> list[str]:
    """Line-by-line differences beyond the column tolerances ([] = match)."""
    problems = []
    so, sr = sections_of(ours), sections_of(ref)
    if so.get("config") != sr.get("config"):
        problems.append(f"config {so.get('config')} != {sr.get('config')}")
    for name in sr:
        if name == "config":
            continue
        for k, v in (sr[name].items() if isinstance(sr[name], dict) else []):
            if not same_value(k, so.get(name, {}).get(k), v):
                problems.append(f"{name}.{k}: {so.get(name, {}).get(k)} vs {v}")
    co, ro = rows_of(ours)
    cr, rr = rows_of(ref)
    if co != cr:
        return problems + [f"columns {co} != {cr}"]
    if len(ro) != len(rr):
        return problems + [f"{len(ro)} rows vs {len(rr)}"]
    for i, (a, b) in enumerate(zip(ro, rr)):
        problems += [f"row {i} {c}: {a[c]} vs {b[c]}" for c in cr
                     if not same_value(c, a[c], b[c])]
    return problems
