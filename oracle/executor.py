"""ORACLE / TEST INFRASTRUCTURE ONLY -- CPU restatement of the hshard executor.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker / reported baseline -- never on the
product path.

The reference declares execute_plan / scatter / reassemble
(/root/reference/proj/include/hshard/sim.hpp:63-79) but never defines them;
their semantics are specified in SPEC.md:467-495 and restated per step in
SURVEY.md Appendix C.  This module restates them over native-dtype numpy
shards (the reference keeps doubles, tensor.hpp:24-30):

  * placement: annotation.cpp:304-354 (subgroup_region with floor_mul
    boundaries, row-major digit refinement).
  * shard layout: dense row-major over placement(...).extents() (tensor.cpp:84-92).
  * AllReduce / ReduceScatter: value(R_d) = sum over group members in
    ASCENDING DEVICE ID order of src[m][R_d]; every member must
    cover R_d.
  * AllGather: R_d assembled from src[m] ∩ R_d; every cell exactly once.
  * SendRecv / Identity / Bsr: copies (Bsr payload order = fusion groups).
  * Split collectives, per finest slice and receiver r with bottom partial
    ordinal (p_r of P_r): sum, in ascending id order, of the contributors c
    with p_c mod P_r == p_r (SURVEY App. C rule, generalised so every
    contributor lands on exactly one receiver ordinal); zero-fill if none.
  * Arithmetic: accumulate in f32 for bf16/f32, f64 for f64, wrapping integer
    adds for i32/i64; round to the storage dtype once per plan phase (the mid
    annotation materialises between phases).
  * A step whose members cannot produce their target box (the reference's
    align_shard_specs defect) raises UnexecutableStep.

Pinned by: tests/test_oracle.py (ref_tool's reference-primitive executor
vectors in tests/golden/data.jsonl, bit-exact on the grid) and the SPEC
reassembly-invariance sweep.
"""
from __future__ import annotations

import json
from fractions import Fraction
from typing import Dict, List, Optional

import numpy as np

from . import datagen as dg


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{code}: {msg}")
        self.code = code


# ---------------------------------------------------------------- annotations
def parse(text: str) -> dict:
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
    return {"groups": groups, "specs": specs, "hdim": hdim, "hsize": len(groups),
            "ratios": ratios}


def eff_hdim(a) -> int:
    return -1 if a["hsize"] == 1 else a["hdim"]


def subgroup_region(a, shape, g):
    b = [[0, int(s)] for s in shape]
    hd = eff_hdim(a)
    if hd < 0:
        return b
    ratios = a["ratios"] or [Fraction(1, a["hsize"])] * a["hsize"]
    before = sum(ratios[:g], Fraction(0))
    ext = int(shape[hd])
    lo = (before * ext).__floor__()
    hi = ext if g == a["hsize"] - 1 else ((before + ratios[g]) * ext).__floor__()
    b[hd] = [lo, hi]
    return b


def placement(a, shape, dev) -> dict:
    """-> {"bounds", "g", "p", "P", "q", "Q"} (annotation.cpp:304-354)."""
    for g, grp in enumerate(a["groups"]):
        if dev in grp:
            break
    else:
        raise OracleError("DeviceNotInAnnotation", str(dev))
    idx = grp.index(dev)
    spec = a["specs"][g]
    digits = [0] * len(spec)
    rem = idx
    for k in range(len(spec) - 1, -1, -1):
        digits[k] = rem % spec[k][1]
        rem //= spec[k][1]
    b = subgroup_region(a, shape, g)
    p, P, q, Q = 0, 1, 0, 1
    for (key, cnt), dgt in zip(spec, digits):
        if key >= 0:
            lo, hi = b[key]
            step = (hi - lo) // cnt
            b[key] = [lo + step * dgt, lo + step * (dgt + 1)]
        elif key == -1:
            q, Q = q * cnt + dgt, Q * cnt
        else:
            p, P = p * cnt + dgt, P * cnt
    return {"bounds": b, "g": g, "p": p, "P": P, "q": q, "Q": Q}


def placements(a, shape) -> Dict[int, dict]:
    return {d: placement(a, shape, d) for grp in a["groups"] for d in grp}


def _ext(bounds):
    return tuple(hi - lo for lo, hi in bounds)


def _local(owner, box):
    return tuple(slice(lo - o, hi - o) for (lo, hi), o in zip(box, owner))


def _isect(a, b):
    out = []
    for (a0, a1), (b0, b1) in zip(a, b):
        lo, hi = max(a0, b0), min(a1, b1)
        if lo >= hi:
            return None
        out.append([lo, hi])
    return out


def _covers(outer, inner):
    return all(o0 <= i0 and i1 <= o1 for (o0, o1), (i0, i1) in zip(outer, inner))


# ---------------------------------------------------------------- data
def scatter(anno_text: str, shape, dtype: str, seed: int, tid: int = 0, mode: str = "grid"):
    """Source state: each device's shard from the counter-hash generator."""
    a = parse(anno_text)
    out = {}
    top_partial = eff_hdim(a) == -2
    for d, pl in placements(a, shape).items():
        tg = pl["g"] if top_partial else -1
        out[d] = dg.shard_values(shape, pl["bounds"], seed, tid, a["hsize"], tg, pl["g"], pl["p"],
                                 pl["P"], dtype, mode)
    return out


def reassemble(anno_text: str, shards, shape, dtype: str):
    """Logical value (float64): sum partials, concat splits; replicas and (hdim -1) extra
    subgroups are skipped (SPEC.md:476-481 semantics, equality not re-asserted here)."""
    a = parse(anno_text)
    x = np.zeros([int(s) for s in shape], dtype=np.float64)
    hd = eff_hdim(a)
    for d, pl in placements(a, shape).items():
        if pl["q"] != 0 or (hd == -1 and pl["g"] != 0):
            continue
        x[tuple(slice(lo, hi) for lo, hi in pl["bounds"])] += dg.decode(shards[d], dtype)
    return x


# ---------------------------------------------------------------- arithmetic
def _acc_dtype(dtype):
    return {"bf16": np.float32, "f32": np.float32, "f64": np.float64, "i32": np.int32,
            "i64": np.int64}[dtype]


def _widen(arr, dtype):
    if dtype == "bf16":
        return dg.bf16_bits_to_f32(arr)
    return np.array(arr, dtype=_acc_dtype(dtype), copy=True)


def _narrow(acc, dtype):
    if dtype == "bf16":
        return dg.f32_to_bf16_bits(acc)
    return acc.astype(dg.NP_DTYPE[dtype])


def _sum_terms(terms, dtype):
    """Fixed-order accumulation: acc = t0; acc += t1; ... ; round once."""
    acc = _widen(terms[0], dtype)
    with np.errstate(over="ignore"):
        for t in terms[1:]:
            acc = acc + _widen(t, dtype)
    return _narrow(acc, dtype)


# ---------------------------------------------------------------- execution
def _alloc(a, shape, dtype):
    pls = placements(a, shape)
    return pls, {d: np.zeros(_ext(pl["bounds"]), dtype=dg.NP_DTYPE[dtype]) for d, pl in pls.items()}


def _run_step(step, phase_src, src_pl, src, tgt_pl, tgt, dtype):
    kind = step["kind"]
    if kind == "Identity":
        for d in phase_src["groups"][step["sub"]]:
            tgt[d][...] = src[d]
    elif kind == "SendRecv":
        for s, r in step["pairs"]:
            tgt[r][...] = src[s]
    elif kind in ("AllReduce", "ReduceScatter"):
        for grp in step["groups"]:
            order = sorted(grp)
            for d in grp:
                box = tgt_pl[d]["bounds"]
                for m in order:
                    if not _covers(src_pl[m]["bounds"], box):
                        raise OracleError("UnexecutableStep", f"{kind} member {m} lacks {box}")
                tgt[d][...] = _sum_terms([src[m][_local([b[0] for b in src_pl[m]["bounds"]], box)]
                                          for m in order], dtype)
    elif kind == "AllGather":
        for grp in step["groups"]:
            for d in grp:
                box = tgt_pl[d]["bounds"]
                hits = np.zeros(_ext(box), dtype=np.int32)
                for m in grp:
                    isect = _isect(src_pl[m]["bounds"], box)
                    if isect is None:
                        continue
                    lt = _local([b[0] for b in box], isect)
                    tgt[d][lt] = src[m][_local([b[0] for b in src_pl[m]["bounds"]], isect)]
                    hits[lt] += 1
                if not np.all(hits == 1):
                    raise OracleError("UnexecutableStep", f"AllGather cannot assemble {box} on {d}")
    elif kind == "Bsr":
        bsr = step["bsr"]
        for dev, tid, reg in bsr["local"]:
            tgt[dev][_local([b[0] for b in tgt_pl[dev]["bounds"]], reg)] = \
                src[dev][_local([b[0] for b in src_pl[dev]["bounds"]], reg)]
        for fg in bsr["fg"]:
            for i in fg[2]:
                tid, reg, s, r, nbytes = bsr["xfer"][i]
                tgt[r][_local([b[0] for b in tgt_pl[r]["bounds"]], reg)] = \
                    src[s][_local([b[0] for b in src_pl[s]["bounds"]], reg)]
    else:  # split collectives
        for sc in step["slices"]:
            reg = sc["reg"]
            cs = sorted(sc["c"])
            for r in sc["r"]:
                pr, Pr = tgt_pl[r]["p"], tgt_pl[r]["P"]
                terms = [src[c][_local([b[0] for b in src_pl[c]["bounds"]], reg)]
                         for c in cs if src_pl[c]["p"] % Pr == pr]
                lt = _local([b[0] for b in tgt_pl[r]["bounds"]], reg)
                if terms:
                    tgt[r][lt] = _sum_terms(terms, dtype)
                else:
                    tgt[r][lt] = 0


def execute_plan(plan, src_shards, dtype: Optional[str] = None):
    """plan: canonical plan JSON (str or dict) of a CommPlan; src_shards: {dev: array}."""
    if isinstance(plan, str):
        plan = json.loads(plan)
    dtype = dtype or plan["dtype"]
    shape = plan["shape"]
    src_a = parse(plan["src"])
    cur_a, cur_pl, cur = src_a, placements(src_a, shape), dict(src_shards)
    if plan["bottom"]:
        tgt_a = parse(plan["mid"] if plan["mid"] else plan["dst"])
        tgt_pl, tgt = _alloc(tgt_a, shape, dtype)
        for step in plan["bottom"]:
            _run_step(step, cur_a, cur_pl, cur, tgt_pl, tgt, dtype)
        cur_a, cur_pl, cur = tgt_a, tgt_pl, tgt
    if plan["top"]:
        tgt_a = parse(plan["dst"])
        tgt_pl, tgt = _alloc(tgt_a, shape, dtype)
        for step in plan["top"]:
            _run_step(step, cur_a, cur_pl, cur, tgt_pl, tgt, dtype)
        cur = tgt
    return cur


def execute_switch(plan, entries, src_shards, dtype):
    """Fused switch BsrPlan: src_shards[(tid, dev)] -> dst[(tid, dev)]."""
    if isinstance(plan, str):
        plan = json.loads(plan)
    meta = {tid: (parse(s), parse(d), shp) for tid, s, d, shp in entries}
    dst, src_pl, dst_pl = {}, {}, {}
    for tid, (sa, da, shp) in meta.items():
        src_pl[tid] = placements(sa, shp)
        dst_pl[tid] = placements(da, shp)
        for d, pl in dst_pl[tid].items():
            dst[(tid, d)] = np.zeros(_ext(pl["bounds"]), dtype=dg.NP_DTYPE[dtype])
    for dev, tid, reg in plan["local"]:
        dst[(tid, dev)][_local([b[0] for b in dst_pl[tid][dev]["bounds"]], reg)] = \
            src_shards[(tid, dev)][_local([b[0] for b in src_pl[tid][dev]["bounds"]], reg)]
    for fg in plan["fg"]:
        for i in fg[2]:
            tid, reg, s, r, nbytes = plan["xfer"][i]
            dst[(tid, r)][_local([b[0] for b in dst_pl[tid][r]["bounds"]], reg)] = \
                src_shards[(tid, s)][_local([b[0] for b in src_pl[tid][s]["bounds"]], reg)]
    return dst
