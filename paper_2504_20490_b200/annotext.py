"""Pure-Python text helpers shared by the package and the benchmark's reference
arm: the reference's HetAnnotation::str() form (annotation.cpp:146-170) built
from groups/specs, parsed back, and the DType tables (common.hpp:28, BF16
appended).  No native code is loaded by importing this module.
"""
from __future__ import annotations

from fractions import Fraction
from typing import Optional, Sequence

# hshard::DType ordinals (reference common.hpp:28, BF16 appended).
DTYPES = {"f32": 0, "f64": 1, "i32": 2, "i64": 3, "bf16": 4}
DTYPE_BYTES = {"f32": 4, "f64": 8, "i32": 4, "i64": 8, "bf16": 2}

kDuplicate = -1
kPartial = -2


def _ds_str(ds) -> str:
    if isinstance(ds, str):
        return ds
    items = ds.items() if isinstance(ds, dict) else ds
    return "{" + ",".join(f"{k}:{c}" for k, c in items) + "}"


def anno(groups: Sequence[Sequence[int]], specs, hdim: int = -1,
         ratios: Optional[Sequence] = None) -> str:
    """HetAnnotation::make(groups, specs, hdim, ratios) in text form.

    specs: one per group; each a dict / list of (key, count) / "{k:c}" string.
    ratios: Fractions, (num, den) tuples or "a/b" strings.
    """
    parts = []
    for g, ds in zip(groups, specs):
        parts.append("(" + ",".join(str(d) for d in g) + ")" + _ds_str(ds))
    s = f"hsize={len(groups)} hdim={hdim} [" + "; ".join(parts) + "]"
    if ratios:
        rs = []
        for r in ratios:
            if isinstance(r, tuple):
                r = Fraction(r[0], r[1])
            r = Fraction(r)
            rs.append(str(r.numerator) if r.denominator == 1 else f"{r.numerator}/{r.denominator}")
        s += " ratios=" + ",".join(rs)
    return s


def single(group: Sequence[int], ds) -> str:
    """HetAnnotation::single(group, ds)."""
    return anno([group], [ds], -1)


def parse_annotation(text: str) -> dict:
    """Parse the str() form into {"groups", "specs", "hdim", "hsize", "ratios"} (pure Python;
    used by tests and the oracle to reason about annotations)."""
    text = text.strip()
    hdim = int(text.split("hdim=")[1].split()[0])
    body = text[text.index("[") + 1:text.rindex("]")]
    groups, specs = [], []
    for part in body.split(";"):
        part = part.strip()
        ids = part[part.index("(") + 1:part.index(")")]
        groups.append([int(x) for x in ids.split(",") if x.strip()])
        ds = part[part.index("{") + 1:part.rindex("}")]
        specs.append([tuple(int(v) for v in e.split(":")) for e in ds.split(",") if e.strip()])
    ratios = []
    tail = text[text.rindex("]") + 1:]
    if "ratios=" in tail:
        ratios = [Fraction(x) for x in tail.split("ratios=")[1].strip().split(",") if x]
    return {"groups": groups, "specs": specs, "hdim": hdim, "hsize": len(groups), "ratios": ratios}
